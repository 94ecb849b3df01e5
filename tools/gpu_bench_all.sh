# Parity tests + bench lines for every single-GPU config.  usage: bash tools/gpu_bench_all.sh <tag>
TAG=${1:-all}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
for cfg in ieee8500 ieee123 ieee13; do
  timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_${cfg}.log 2>&1
  tail -1 gpurun_out/${TAG}_bench_${cfg}.log | cut -c1-300
done
timeout 900 python bench.py --config batch123 --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_batch123.log 2>&1
tail -1 gpurun_out/${TAG}_bench_batch123.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref_ieee8500.log 2>&1
tail -1 gpurun_out/${TAG}_ref_ieee8500.log | cut -c1-200
timeout 1500 python bench.py --config tiled --tiles 64 --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_tiled.log 2>&1
tail -1 gpurun_out/${TAG}_bench_tiled.log | cut -c1-300
