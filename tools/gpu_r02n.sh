TAG=${1:-r02n}
mkdir -p gpurun_out
for r in 1 2; do
  for t in 1 0; do
    DOPF_NO_TUNE=$t DOPF_BENCH_NO_NCU=1 timeout 900 python bench.py --config tiled --tiles 64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
    python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('no_tune=$t', 'tiled', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['setup'])" || tail -3 gpurun_out/ab.err
  done
done
