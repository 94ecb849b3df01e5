# ncu launch list + one full capture of the 8500 solve.  usage: bash tools/gpu_ncu.sh <tag>
TAG=${1:-ncu}
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/ncu_target.py ieee8500 8500 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:admm -s 1 -c 1 -o gpurun_out/${TAG}_prof python tools/ncu_target.py ieee8500 8500 2 > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
