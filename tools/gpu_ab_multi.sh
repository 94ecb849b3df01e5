# A/B/C... of several builds of libdopf_cuda.so on one config, interleaved.  usage: bash tools/gpu_ab_multi.sh config rounds lib1.so lib2.so ...
CFG=$1; R=$2; shift 2
mkdir -p gpurun_out
for r in $(seq $R); do
  for lib in "$@"; do
    DOPF_CUDA_SO=$lib DOPF_VERBOSE=1 timeout 600 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err
    echo "$(basename $lib) $(grep 'stream layout' gpurun_out/ab.err | head -1 | cut -c15-60)"
    python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('   ', '$CFG', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1))"
  done
done
