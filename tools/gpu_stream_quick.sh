mkdir -p gpurun_out; export DOPF_VERBOSE=1
timeout 900 python -m pytest tests -m gpu -x -q -k "stream or tiled or reupload or partition" > gpurun_out/st_pytest.log 2>&1; tail -3 gpurun_out/st_pytest.log
timeout 500 python bench.py --config tiled --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/st_bench.log 2>gpurun_out/st_bench.err; grep -E "stream layout|e2e step" gpurun_out/st_bench.err | head -3
python -c "import json,sys;d=json.loads(open(\"gpurun_out/st_bench.log\").read().strip().splitlines()[-1]);print(d[\"value\"], d[\"ms_per_step\"], d[\"roofline\"][\"frac\"], d[\"e2e\"][\"value\"])"
DOPF_STREAM_NOGRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/st_launch.csv python tools/ncu_tiled.py 64 2 > gpurun_out/st_ncu1.log 2>&1
