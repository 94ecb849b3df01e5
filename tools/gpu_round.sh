# One GPU round: parity tests, bench, phase clock, ncu launch list + full capture.
# usage: bash tools/gpu_round.sh <tag>
TAG=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
tail -5 gpurun_out/${TAG}_pytest.log
timeout 300 python tools/phase_clock.py > gpurun_out/${TAG}_phase.log 2>&1; cat gpurun_out/${TAG}_phase.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1; tail -c 1500 gpurun_out/${TAG}_bench.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/ncu_target.py ieee8500 8500 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:admm -s 1 -c 1 -o gpurun_out/${TAG}_prof python tools/ncu_target.py ieee8500 8500 2 > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
