# headline evidence with the tuned split: bench (full line), launch list + ncu of the tuned kernel, phase clock
TAG=${1:-r02o}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${TAG}_bench_ieee8500.log 2>gpurun_out/${TAG}_bench_ieee8500.err; tail -1 gpurun_out/${TAG}_bench_ieee8500.log | cut -c1-300
DOPF_TUNE=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/ncu_target.py ieee8500 8500 3 > /dev/null 2>&1
DOPF_TUNE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:admm_persistent -s 1 -c 1 -o gpurun_out/${TAG}_prof python tools/ncu_target.py ieee8500 8500 2 > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref.log 2>&1; tail -1 gpurun_out/${TAG}_ref.log | cut -c1-200
