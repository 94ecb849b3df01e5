TAG=${1:-r02final2}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${TAG}_bench_ieee8500.log 2>gpurun_out/${TAG}_bench_ieee8500.err; tail -1 gpurun_out/${TAG}_bench_ieee8500.log
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref.log 2>&1; tail -1 gpurun_out/${TAG}_ref.log
timeout 600 python bench.py --config ieee123 > gpurun_out/${TAG}_bench_ieee123.log 2>/dev/null; tail -1 gpurun_out/${TAG}_bench_ieee123.log | cut -c1-200
