// Micro-benchmark: latency (cycles) of dependent fp64 add / fma, fp32 add, shared-memory load and
// warp shuffle chains on one warp (B200, sm_100a).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
  __syncthreads();
  double a = out[threadIdx.x], b = 1e-300;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { a = a + b; a = a + b; a = a + b; a = a + b; }
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) { a = fma(a, 1.0000001, b); a = fma(a, 1.0000001, b); a = fma(a, 1.0000001, b); a = fma(a, 1.0000001, b); }
  long long t2 = clock64();
  float fa = (float)a, fb = 1e-30f;
  for (int i = 0; i < n; ++i) { fa = fa + fb; fa = fa + fb; fa = fa + fb; fa = fa + fb; }
  long long t3 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < n; ++i) { idx = ((int)sm[idx & 1023]) + (idx & 1); idx = ((int)sm[idx & 1023]) + (idx & 1); idx = ((int)sm[idx & 1023]) + (idx & 1); idx = ((int)sm[idx & 1023]) + (idx & 1); }
  long long t4 = clock64();
  double s = a;
  for (int i = 0; i < n; ++i) { s = __shfl_xor_sync(0xffffffffu, s, 1); s = __shfl_xor_sync(0xffffffffu, s, 2); s = __shfl_xor_sync(0xffffffffu, s, 4); s = __shfl_xor_sync(0xffffffffu, s, 8); }
  long long t5 = clock64();
  double d = a;
  for (int i = 0; i < n; ++i) { d = 1.0 / d; d = 1.0 / d; d = 1.0 / d; d = 1.0 / d; }
  long long t6 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; }
  out[threadIdx.x] = a + fa + idx + s + d;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMemset(o, 0, 1024 * 8); cudaMalloc(&c, 64);
  const int n = 4096;
  for (int w = 1; w <= 8; w *= 2) {
    k<<<1, 32 * w>>>(o, c, n); cudaDeviceSynchronize();
    long long h[6]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    const char* nm[6] = {"dadd", "dfma", "fadd", "lds(+cvt,iadd)", "shfl.f64", "drcp(div)"};
    printf("warps/CTA %d:", w);
    for (int i = 0; i < 6; ++i) printf("  %s %.1f", nm[i], (double)h[i] / (4.0 * n));
    printf("  cycles per dependent op\n");
  }
  return 0;
}
