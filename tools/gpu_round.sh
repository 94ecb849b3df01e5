set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
timeout 300 python tools/ncu_target.py ieee8500 8500 2 > gpurun_out/target.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/ncu_target.py ieee8500 8500 3 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:admm -s 1 -c 1 -o gpurun_out/prof8500 python tools/ncu_target.py ieee8500 8500 2 > gpurun_out/ncu_full.log 2>&1
timeout 300 python tools/phase_clock.py > gpurun_out/phase.log 2>&1
tail -3 gpurun_out/*.log
