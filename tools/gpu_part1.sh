# One-GPU check of the partitioned (NCCL, C ABI) tiled path vs the single-GPU streaming path.
TAG=${1:-part1}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_cli.py -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_cli.log 2>&1; tail -2 gpurun_out/${TAG}_cli.log
DOPF_BENCH_PARTITIONED=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --config tiled --steps 3 --warmup 3 > gpurun_out/${TAG}_tiled_part.log 2> gpurun_out/${TAG}_tiled_part.err
tail -1 gpurun_out/${TAG}_tiled_part.log | cut -c1-600
DOPF_PART_GRAPH=unrolled DOPF_BENCH_PARTITIONED=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 bench.py --config tiled --steps 3 --warmup 3 > gpurun_out/${TAG}_tiled_part_unrolled.log 2> gpurun_out/${TAG}_tiled_part_unrolled.err
tail -1 gpurun_out/${TAG}_tiled_part_unrolled.log | cut -c1-600
timeout 1200 python bench.py --config tiled --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_tiled.log 2> gpurun_out/${TAG}_tiled.err
tail -1 gpurun_out/${TAG}_tiled.log | cut -c1-400
