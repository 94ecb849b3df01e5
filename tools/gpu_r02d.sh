# full non-slow GPU suite on the current build + quick benches
TAG=${1:-r02d}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; tail -4 gpurun_out/${TAG}_pytest.log
for cfg in ieee8500 ieee123; do
  DOPF_BENCH_NO_NCU=1 timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$cfg', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
done
