mkdir -p gpurun_out
for lib in ab_libs/cur ab_libs/nocheck; do
  DOPF_BENCH_NO_NCU=1 DOPF_CUDA_SO=$lib/libdopf_cuda.so timeout 900 python bench.py --config batch123 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$lib', 'batch123', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
done
