// L2 hit latency microbenchmark (pointer chase, one thread), plain ld.cg vs
// 128-bit relaxed.gpu loads. usage: ./l2_latency
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void chase_cg(const unsigned long long* p, int n, unsigned long long* out, long long* cyc) {
  unsigned long long i = 0;
  long long t0 = clock64();
  for (int k = 0; k < n; ++k) i = __ldcg(p + i * 2);
  long long t1 = clock64();
  *out = i;
  *cyc = t1 - t0;
}
__global__ void chase_b128(const unsigned long long* p, int n, unsigned long long* out, long long* cyc) {
  unsigned long long i = 0, hi;
  long long t0 = clock64();
  for (int k = 0; k < n; ++k) {
    asm volatile("{ .reg .b128 d; ld.relaxed.gpu.global.b128 d, [%2]; mov.b128 {%0, %1}, d; }"
                 : "=l"(i), "=l"(hi) : "l"(p + i * 2) : "memory");
  }
  long long t1 = clock64();
  *out = i + hi;
  *cyc = t1 - t0;
}
__device__ void chase_smem_flag(unsigned long long* flag, int n, long long* cyc, int role) {
  // ping-pong between two CTAs through one global word
  long long t0 = clock64();
  for (int k = 0; k < n; ++k) {
    if (role == 0) {
      while (atomicAdd(flag, 0) != 2ull * k) {}
      atomicExch(flag, 2ull * k + 1);
    } else {
      while (atomicAdd(flag, 0) != 2ull * k + 1) {}
      atomicExch(flag, 2ull * k + 2);
    }
  }
  long long t1 = clock64();
  if (role == 0) *cyc = t1 - t0;
}
__global__ void pingpong(unsigned long long* flag, int n, long long* cyc) {
  chase_smem_flag(flag, n, cyc, blockIdx.x == 0 ? 0 : 1);
}

int main() {
  const size_t N = 4u << 20;  // 4M records x 16 B = 64 MB
  std::vector<unsigned long long> h(2 * N);
  std::vector<size_t> perm(N);
  for (size_t i = 0; i < N; ++i) perm[i] = i;
  srand(1);
  for (size_t i = N - 1; i > 0; --i) { size_t j = rand() % (i + 1); std::swap(perm[i], perm[j]); }
  for (size_t i = 0; i < N; ++i) h[2 * perm[i]] = perm[(i + 1) % N], h[2 * perm[i] + 1] = 0;
  unsigned long long *d, *out; long long* cyc;
  cudaMalloc(&d, 16 * N); cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  cudaMemcpy(d, h.data(), 16 * N, cudaMemcpyHostToDevice);
  const int n = 200000;
  long long c;
  for (int rep = 0; rep < 2; ++rep) {
    chase_cg<<<1, 1>>>(d, n, out, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("ld.cg chase      : %.0f cycles/load\n", double(c) / n);
    chase_b128<<<1, 1>>>(d, n, out, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("ld.relaxed b128  : %.0f cycles/load\n", double(c) / n);
  }
  unsigned long long* flag; cudaMalloc(&flag, 8);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(flag, 0, 8);
    pingpong<<<2, 1>>>(flag, 20000, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("atomic ping-pong : %.0f cycles/round trip (2 hops)\n", double(c) / 20000);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
