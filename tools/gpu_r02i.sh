TAG=${1:-r02i}
mkdir -p gpurun_out
timeout 900 python tools/tune_partition.py 8 0.5 > gpurun_out/${TAG}_tune.log 2>&1; head -10 gpurun_out/${TAG}_tune.log
W=$(tail -1 gpurun_out/${TAG}_tune.log)
for r in 1 2; do
  DOPF_BENCH_NO_NCU=1 timeout 300 python bench.py --config ieee8500 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('default', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
  DOPF_BLOCK_WEIGHTS=$W DOPF_BENCH_NO_NCU=1 timeout 300 python bench.py --config ieee8500 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('tuned', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
done
