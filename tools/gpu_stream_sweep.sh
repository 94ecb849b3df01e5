# Staged streaming kernel: pipeline-shape sweep on the tiled feeder.  usage: bash tools/gpu_stream_sweep.sh "ctas stages kb" ...
mkdir -p gpurun_out
for cfg in "$@"; do
  set -- $cfg
  tag=sw_$1_$2_$3
  DOPF_STAGED_CTAS=$1 DOPF_STAGES=$2 DOPF_STAGE_KB=$3 DOPF_VERBOSE=1 timeout 400 python bench.py --config tiled --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$tag.log 2>gpurun_out/$tag.err
  echo "ctas=$1 stages=$2 kb=$3 $(grep 'stream layout' gpurun_out/$tag.err | head -1 | cut -c1-90)"
  python -c "import json;d=json.loads(open('gpurun_out/$tag.log').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])" 2>&1 | tail -1
done
