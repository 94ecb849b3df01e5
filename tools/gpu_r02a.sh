# r02 session 3: f2 prepare tests, interleaved-GEMV A/B, bench with live ncu traffic
TAG=${1:-r02a}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_prepare.py -x -q -p no:cacheprovider > gpurun_out/${TAG}_prepare.log 2>&1; tail -15 gpurun_out/${TAG}_prepare.log
bash tools/gpu_resident_ab.sh ${TAG} 2
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1; tail -c 2500 gpurun_out/${TAG}_bench.log
