TAG=${1:-tim}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_timings.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; tail -2 gpurun_out/${TAG}_pytest.log
for r in 1 2; do
  for lib in ab_libs/base/libdopf_cuda.so paper_2501_08293_b200/lib/libdopf_cuda.so; do
    for cfg in ieee8500 tiled; do
      DOPF_CUDA_SO=$lib timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>/dev/null
      python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$lib'.split('/')[1], '$cfg', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1))"
    done
  done
done
