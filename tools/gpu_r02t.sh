mkdir -p gpurun_out
DOPF_CUDA_SO=ab_libs/g2/libdopf_cuda.so timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -k "batch" -x -q -p no:cacheprovider > gpurun_out/g2_pytest.log 2>&1; tail -3 gpurun_out/g2_pytest.log
for a in 1 0; do
  DOPF_BATCH_A_SMEM=$a DOPF_BENCH_NO_NCU=1 DOPF_CUDA_SO=ab_libs/g2/libdopf_cuda.so timeout 900 python bench.py --config batch123 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('a_smem_forced=$a', 'batch123', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['kernel'])" || tail -3 gpurun_out/ab.err
done
