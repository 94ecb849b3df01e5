# A/B/... of values of an environment knob on the tiled config, interleaved.  usage: bash tools/gpu_ab_vals.sh VAR "v1 v2 ..." [rounds]
VAR=$1; VALS=$2; R=${3:-2}
mkdir -p gpurun_out
for r in $(seq $R); do
  for v in $VALS; do
    env $VAR=$v timeout 600 python bench.py --config tiled --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$VAR=$v', round(d['value'],1), round(d['roofline']['frac'],4))"
  done
done
