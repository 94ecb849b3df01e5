# r02 session 3: new GPU tests, resident no-barrier A/B, tiled chunk-balance A/B
TAG=${1:-r02c}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_prepare.py tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_timings.py -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; tail -4 gpurun_out/${TAG}_pytest.log
timeout 300 python tools/phase_clock.py > gpurun_out/${TAG}_phase.log 2>&1; head -12 gpurun_out/${TAG}_phase.log
for r in 1 2 3; do
  for lib in ab_libs/base ab_libs/nobar ab_libs/fuse; do
    for cfg in ieee8500 ieee123; do
      DOPF_BENCH_NO_NCU=1 DOPF_CUDA_SO=$lib/libdopf_cuda.so timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
      python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$lib', '$cfg', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
    done
  done
done
for rr in 1 0; do
  if [ $rr = 1 ]; then export DOPF_STREAM_RR=1; else unset DOPF_STREAM_RR; fi
  DOPF_BENCH_NO_NCU=1 timeout 900 python bench.py --config tiled --tiles 64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('tiled RR=$rr', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
done
unset DOPF_STREAM_RR
timeout 900 python -m pytest tests/test_gpu_edge_cases.py -m "gpu and slow" -x -q -p no:cacheprovider > gpurun_out/${TAG}_slow.log 2>&1; tail -3 gpurun_out/${TAG}_slow.log
