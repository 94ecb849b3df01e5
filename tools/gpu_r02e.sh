# batch: A in L2 with 3 CTAs per scenario (al2) vs base (A in smem, 4 CTAs)
TAG=${1:-r02e}
mkdir -p gpurun_out
DOPF_CUDA_SO=ab_libs/al2/libdopf_cuda.so timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -k "batch or ieee8500 or fixture" -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
for lib in ab_libs/base ab_libs/al2; do
  DOPF_BENCH_NO_NCU=1 DOPF_CUDA_SO=$lib/libdopf_cuda.so timeout 900 python bench.py --config batch123 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$lib', 'batch123', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['kernel'])" || tail -3 gpurun_out/ab.err
  DOPF_BENCH_NO_NCU=1 DOPF_CUDA_SO=$lib/libdopf_cuda.so timeout 600 python bench.py --config ieee8500 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$lib', 'ieee8500', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
done
