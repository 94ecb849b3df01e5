# A/B of two library builds: parity of B, phase clock of B, interleaved benches.  usage: bash tools/gpu_ab2.sh TAG A.so B.so [rounds]
TAG=$1; A=$2; B=$3; R=${4:-2}
mkdir -p gpurun_out
DOPF_CUDA_SO=$B timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_timings.py -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; tail -2 gpurun_out/${TAG}_pytest.log
DOPF_CUDA_SO=$B timeout 300 python tools/phase_clock.py > gpurun_out/${TAG}_phase.log 2>&1; head -12 gpurun_out/${TAG}_phase.log
for r in $(seq $R); do
  for lib in $A $B; do
    for cfg in ieee8500 ieee123; do
      DOPF_BENCH_NO_NCU=1 DOPF_CUDA_SO=$lib timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
      python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$lib'.split('/')[-2], '$cfg', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
    done
  done
done
for lib in $A $B; do
  DOPF_BENCH_NO_NCU=1 DOPF_CUDA_SO=$lib timeout 900 python bench.py --config batch123 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$lib'.split('/')[-2], 'batch123', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
done
