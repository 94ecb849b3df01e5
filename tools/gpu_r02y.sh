mkdir -p gpurun_out
DOPF_CUDA_SO=ab_libs/h12/libdopf_cuda.so timeout 600 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -k "ieee8500 or fixture_solve or tuned" -x -q -p no:cacheprovider > gpurun_out/spread_pytest.log 2>&1; tail -2 gpurun_out/spread_pytest.log
for r in 1 2; do
  for lib in ab_libs/cur ab_libs/h12; do
    DOPF_BENCH_NO_NCU=1 DOPF_CUDA_SO=$lib/libdopf_cuda.so timeout 300 python bench.py --config ieee8500 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
    python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$lib', 'ieee8500', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
  done
done
