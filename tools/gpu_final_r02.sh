# Round-2 evidence: the whole GPU suite, smoke, every bench config, reference arm,
# launch lists and ncu of the resident (single + batch) and streaming kernels, phase clocks.
TAG=${1:-r02final}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_gpu.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; tail -2 gpurun_out/${TAG}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
for cfg in ieee8500 ieee123 ieee13; do
  timeout 900 python bench.py --config $cfg > gpurun_out/${TAG}_bench_${cfg}.log 2>gpurun_out/${TAG}_bench_${cfg}.err
  tail -1 gpurun_out/${TAG}_bench_${cfg}.log | cut -c1-200
done
timeout 1200 python bench.py --config batch123 --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_batch123.log 2>gpurun_out/${TAG}_bench_batch123.err
tail -1 gpurun_out/${TAG}_bench_batch123.log | cut -c1-200
timeout 1800 python bench.py --config tiled --tiles 64 --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_tiled.log 2>gpurun_out/${TAG}_bench_tiled.err
tail -1 gpurun_out/${TAG}_bench_tiled.log | cut -c1-200
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref_ieee8500.log 2>&1
tail -1 gpurun_out/${TAG}_ref_ieee8500.log | cut -c1-200
timeout 300 python tools/prepare_timing.py 4096 > gpurun_out/${TAG}_prepare_timing.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/ncu_target.py ieee8500 8500 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:admm -s 1 -c 1 -o gpurun_out/${TAG}_prof python tools/ncu_target.py ieee8500 8500 2 > gpurun_out/${TAG}_ncu.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${TAG}_batch_launches.csv python tools/ncu_batch.py 296 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:admm -s 1 -c 1 -o gpurun_out/${TAG}_batch_prof python tools/ncu_batch.py 296 2 > gpurun_out/${TAG}_batch_ncu.log 2>&1
DOPF_STREAM_NOGRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/${TAG}_tiled_launches.csv python tools/ncu_tiled.py 64 2 > /dev/null 2>&1
DOPF_STREAM_NOGRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_staged" -s 1 -c 1 -o gpurun_out/${TAG}_tiled_prof python tools/ncu_tiled.py 64 3 > gpurun_out/${TAG}_tiled_ncu.log 2>&1
DOPF_STREAM_PROF=1 timeout 600 python tools/ncu_tiled.py 64 200 > gpurun_out/${TAG}_tiled_phase.log 2>&1
timeout 300 python tools/phase_clock.py > gpurun_out/${TAG}_phase.log 2>&1
ls gpurun_out/ | grep ${TAG} | wc -l
