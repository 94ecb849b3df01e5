# Staged pipeline shapes on the tiled feeder.  usage: bash tools/gpu_stream_cfgs.sh "ctas stages kb" ...
mkdir -p gpurun_out
for cfg in "$@"; do
  set -- $cfg
  DOPF_STAGED_CTAS=$1 DOPF_STAGES=$2 DOPF_STAGE_KB=$3 DOPF_VERBOSE=1 timeout 400 python bench.py --config tiled --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cf.log 2>gpurun_out/cf.err
  echo "ctas=$1 stages=$2 kb=$3 $(grep 'stream layout' gpurun_out/cf.err | head -1 | cut -c15-60)"
  python -c "import json;d=json.loads(open('gpurun_out/cf.log').read().strip().splitlines()[-1]);print('   ', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1))" 2>&1 | tail -1
done
