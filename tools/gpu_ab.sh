# A/B of an environment toggle on both bench configs, interleaved.  usage: bash tools/gpu_ab.sh VAR [rounds]
VAR=$1; R=${2:-2}
mkdir -p gpurun_out
for r in $(seq $R); do
  for v in 0 1; do
    for cfg in ieee8500 tiled; do
      env $VAR=$v timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>/dev/null
      python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$VAR=$v', '$cfg', round(d['value'],1), round(d['roofline']['frac'],4))"
    done
  done
done
