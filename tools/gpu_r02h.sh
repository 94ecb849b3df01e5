# batches as persistent CTA groups (with the barrier drain): parity first, then a bounded A/B
TAG=${1:-r02h}
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -k "persistent_groups" -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
if grep -q "1 passed" gpurun_out/${TAG}_pytest.log; then
  timeout 600 python -m pytest tests -m "gpu and not slow" -k "batch or scenario or timing" -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest2.log 2>&1; tail -2 gpurun_out/${TAG}_pytest2.log
  for mode in groups clusters; do
    if [ $mode = clusters ]; then export DOPF_BATCH_CLUSTERS=1; else unset DOPF_BATCH_CLUSTERS; fi
    DOPF_BENCH_NO_NCU=1 timeout 420 python bench.py --config batch123 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
    python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$mode', 'batch123', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
  done
  unset DOPF_BATCH_CLUSTERS
fi
PHASE_DUMP=gpurun_out/${TAG}_phase_dump.npz timeout 300 python tools/phase_clock.py > gpurun_out/${TAG}_phase.log 2>&1; head -11 gpurun_out/${TAG}_phase.log
DOPF_BENCH_NO_NCU=1 timeout 300 python bench.py --config ieee8500 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('ieee8500', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
