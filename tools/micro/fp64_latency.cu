// fp64 dependent-chain latency and per-SM throughput on this GPU (DADD, DMUL,
// DFMA, IEEE division).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, double a, double b, int iters, long long* cyc) {
  double x = a + threadIdx.x * 1e-9;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (OP == 0) x = __dadd_rn(x, b);
      if (OP == 1) x = __dmul_rn(x, b);
      if (OP == 2) x = __fma_rn(x, b, a);
      if (OP == 3) x = __ddiv_rn(x, b);
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 4096 * 8);
  const char* names[4] = {"DADD", "DMUL", "DFMA", "DDIV"};
  for (int op = 0; op < 4; ++op) {
    for (int warps : {1, 4, 16, 32}) {
      const int iters = 256;
      auto k = op == 0 ? chain<0> : op == 1 ? chain<1> : op == 2 ? chain<2> : chain<3>;
      k<<<1, 32 * warps>>>(out, 1.0000001, 0.9999999, iters, cyc);
      k<<<1, 32 * warps>>>(out, 1.0000001, 0.9999999, iters, cyc);
      long long h;
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      const double per = double(h) / (iters * 16);
      printf("%s warps=%2d: %.1f cycles per dependent op per warp -> %.2f warp-ops/cycle/SM\n", names[op], warps,
             per, warps / per);
    }
  }
  return 0;
}
