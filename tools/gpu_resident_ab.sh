# Resident-kernel change: parity tests, phase clock, A/B vs ab_libs/base.  usage: bash tools/gpu_resident_ab.sh TAG [rounds]
TAG=${1:-rab}; R=${2:-3}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; tail -2 gpurun_out/${TAG}_pytest.log
timeout 300 python tools/phase_clock.py > gpurun_out/${TAG}_phase.log 2>&1; head -12 gpurun_out/${TAG}_phase.log
for r in $(seq $R); do
  for lib in ab_libs/base/libdopf_cuda.so paper_2501_08293_b200/lib/libdopf_cuda.so; do
    for cfg in ieee8500 ieee123; do
      DOPF_CUDA_SO=$lib timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>/dev/null
      python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$lib'.split('/')[1], '$cfg', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
    done
  done
done
