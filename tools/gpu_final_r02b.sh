# Round-2 closing evidence with the final code: every bench config + reference arm.
TAG=${1:-r02close}
mkdir -p gpurun_out
for cfg in ieee8500 ieee123 ieee13; do
  timeout 900 python bench.py --config $cfg > gpurun_out/${TAG}_bench_${cfg}.log 2>/dev/null
  tail -1 gpurun_out/${TAG}_bench_${cfg}.log | cut -c1-160
done
timeout 1500 python bench.py --config batch123 --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_batch123.log 2>/dev/null
tail -1 gpurun_out/${TAG}_bench_batch123.log | cut -c1-160
timeout 1800 python bench.py --config tiled --tiles 64 --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_tiled.log 2>/dev/null
tail -1 gpurun_out/${TAG}_bench_tiled.log | cut -c1-160
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref_ieee8500.log 2>&1
tail -1 gpurun_out/${TAG}_ref_ieee8500.log | cut -c1-160
