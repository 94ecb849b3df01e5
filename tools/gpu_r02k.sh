TAG=${1:-r02k}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -k "tuned" -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
for t in 1 0; do
  for cfg in ieee123 batch123; do
    DOPF_NO_TUNE=$t DOPF_BENCH_NO_NCU=1 timeout 420 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
    python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('no_tune=$t', '$cfg', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['setup'])" || tail -3 gpurun_out/ab.err
  done
done
