TAG=${1:-r02m}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -m "gpu and not slow" -k "stream or tiled or hub or fall" -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
for r in 1 2; do
  for lib in ab_libs/base ab_libs/sfuse; do
    DOPF_BENCH_NO_NCU=1 DOPF_CUDA_SO=$lib/libdopf_cuda.so timeout 900 python bench.py --config tiled --tiles 64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
    python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$lib', 'tiled', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
  done
done
DOPF_STREAM_PROF=1 timeout 600 python tools/ncu_tiled.py 64 100 > gpurun_out/${TAG}_tiled_phase.log 2>&1; head -3 gpurun_out/${TAG}_tiled_phase.log
