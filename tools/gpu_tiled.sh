# Tiled 64x IEEE-8500 on the HBM-streaming path: bench line + ncu of k_local.  usage: bash tools/gpu_tiled.sh <tag> [tiles]
TAG=${1:-tiled}
T=${2:-64}
mkdir -p gpurun_out
timeout 1500 python bench.py --config tiled --tiles $T --steps 3 --warmup 3 > gpurun_out/${TAG}_bench.log 2> gpurun_out/${TAG}_bench.err
tail -1 gpurun_out/${TAG}_bench.log | cut -c1-600; grep -E "e2e step|Error|error" gpurun_out/${TAG}_bench.err
