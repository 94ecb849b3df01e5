mkdir -p gpurun_out
for v in 2 3; do
  DOPF_STAGED_CTAS=$v DOPF_NO_TUNE=1 DOPF_BENCH_NO_NCU=1 timeout 900 python bench.py --config tiled --tiles 64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('staged_ctas=$v', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['kernel']['smem_bytes'])" || tail -3 gpurun_out/ab.err
done
for kb in 40 56; do
  DOPF_STAGE_KB=$kb DOPF_NO_TUNE=1 DOPF_BENCH_NO_NCU=1 timeout 900 python bench.py --config tiled --tiles 64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('stage_kb=$kb', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
done
