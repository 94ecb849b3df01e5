# streaming parity mode, setup timing of the 4096-scenario batch, quick sanity bench
TAG=${1:-r02f}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prepare.py -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python tools/prepare_timing.py 4096 > gpurun_out/${TAG}_prepare_timing.log 2>&1; cat gpurun_out/${TAG}_prepare_timing.log
