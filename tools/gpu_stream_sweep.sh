# Staged streaming kernel: pipeline-shape sweep on the tiled feeder.  usage: bash tools/gpu_stream_sweep.sh
mkdir -p gpurun_out
for cfg in "2 48" "3 32" "4 24" "3 24" "4 16"; do
  set -- $cfg
  DOPF_STAGES=$1 DOPF_STAGE_KB=$2 DOPF_VERBOSE=1 timeout 400 python bench.py --config tiled --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sw_$1_$2.log 2>gpurun_out/sw_$1_$2.err
  echo "stages=$1 kb=$2 $(grep 'stream layout' gpurun_out/sw_$1_$2.err | head -1)"
  python -c "import json;d=json.loads(open('gpurun_out/sw_$1_$2.log').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
done
