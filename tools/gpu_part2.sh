TAG=${1:-part2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nccl.py tests/test_partition.py -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_nccl.log 2>&1; tail -2 gpurun_out/${TAG}_nccl.log
DOPF_BENCH_PARTITIONED=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --config tiled --steps 3 --warmup 3 > gpurun_out/${TAG}_tiled_part.log 2> gpurun_out/${TAG}_tiled_part.err
python -c "import json;d=json.loads(open('gpurun_out/${TAG}_tiled_part.log').read().strip().splitlines()[-1]);print('part', d['value'], d['e2e']['value'], d['gpu_launches'], d['config']['parallelism'][-30:])"
timeout 1200 python bench.py --config tiled --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_tiled.log 2> gpurun_out/${TAG}_tiled.err
python -c "import json;d=json.loads(open('gpurun_out/${TAG}_tiled.log').read().strip().splitlines()[-1]);print('single', d['value'], d['e2e']['value'], d['gpu_launches'])"
