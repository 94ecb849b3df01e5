# Quick GPU check: parity tests, phase clock, short bench.  usage: bash tools/gpu_quick.sh <tag>
TAG=${1:-quick}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
tail -5 gpurun_out/${TAG}_pytest.log
timeout 300 python tools/phase_clock.py > gpurun_out/${TAG}_phase.log 2>&1; cat gpurun_out/${TAG}_phase.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/${TAG}_bench.log').read().strip().splitlines()[-1]);print({k:d[k] for k in ('value','time_to_converge_ms','iterations_to_converge')}, d['roofline']['frac'], d['e2e']['value'])"
