# batches as persistent CTA groups vs one cluster per scenario
TAG=${1:-r02g}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -k "batch or scenario or timing" -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
for r in 1 2; do
for mode in groups clusters; do
  if [ $mode = clusters ]; then export DOPF_BATCH_CLUSTERS=1; else unset DOPF_BATCH_CLUSTERS; fi
  DOPF_BENCH_NO_NCU=1 timeout 900 python bench.py --config batch123 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$mode', 'batch123', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
done
done
unset DOPF_BATCH_CLUSTERS
DOPF_BENCH_NO_NCU=1 timeout 600 python bench.py --config ieee8500 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('ieee8500', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
