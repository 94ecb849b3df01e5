TAG=${1:-r02q}
mkdir -p gpurun_out
W=$(DOPF_TUNE=1 timeout 300 python tools/ncu_target.py ieee8500 8500 | grep DOPF_BLOCK_WEIGHTS | cut -d= -f2)
echo "$W" > gpurun_out/${TAG}_weights.txt
DOPF_BLOCK_WEIGHTS=$W timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/ncu_target.py ieee8500 8500 3 > /dev/null 2>&1
DOPF_BLOCK_WEIGHTS=$W timeout 900 ncu --set full --clock-control none --import-source on -k regex:admm_persistent -s 1 -c 1 -o gpurun_out/${TAG}_prof python tools/ncu_target.py ieee8500 8500 2 > gpurun_out/${TAG}_ncu.log 2>&1
tail -1 gpurun_out/${TAG}_ncu.log
DOPF_BLOCK_WEIGHTS=$W timeout 300 python tools/phase_clock.py > gpurun_out/${TAG}_phase.log 2>&1; head -11 gpurun_out/${TAG}_phase.log
