# A/B of two builds of libdopf_cuda.so on one config, interleaved.  usage: bash tools/gpu_ab_libs.sh A.so B.so [config] [rounds]
A=$1; B=$2; CFG=${3:-tiled}; R=${4:-2}
mkdir -p gpurun_out
for r in $(seq $R); do
  for lib in $A $B; do
    DOPF_CUDA_SO=$lib timeout 600 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$(basename $lib)', '$CFG', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1))"
  done
done
