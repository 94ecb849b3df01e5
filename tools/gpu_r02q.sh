mkdir -p gpurun_out
for r in 1 2; do
  for lib in ab_libs/base ab_libs/nozfree; do
    DOPF_BENCH_NO_NCU=1 DOPF_CUDA_SO=$lib/libdopf_cuda.so timeout 300 python bench.py --config ieee8500 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
    python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$lib', 'ieee8500', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
  done
done
