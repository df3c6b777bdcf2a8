// Do DMMA.8x8x4 (FP64 tensor) and DFMA share one pipe on B200?  Warps [0, W/2) run a DMMA
// loop, warps [W/2, W) a DFMA loop (or all warps one kind); report each kind's TF/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu && ./pipes
#include <cstdio>
#include <cuda_runtime.h>

__global__ void mixed(double* out, int iters, int mode) {
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool mma = mode == 0 ? true : (mode == 1 ? false : warp < nw / 2);
  double s = 0;
  if (mma) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4, c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  } else {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters * 4; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = fma(x[i], 0.999, 1e-3);
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
  }
  if (s == 1.2345) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 4096, blocks = 148, threads = 512;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[3] = {"all DMMA", "all DFMA", "half DMMA + half DFMA"};
  for (int mode = 0; mode < 3; ++mode) {
    mixed<<<blocks, threads>>>(out, 16, mode);
    cudaEventRecord(e0);
    mixed<<<blocks, threads>>>(out, iters, mode);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = blocks * threads / 32.0;
    const double w_mma = mode == 0 ? warps : (mode == 1 ? 0 : warps / 2);
    const double w_fma = warps - w_mma;
    const double f_mma = w_mma * iters * 8 * 512.0;          // 8 DMMA x 512 flops per iter
    const double f_fma = w_fma * 32 * iters * 4 * 16 * 2.0;  // 32 lanes x 64 FMA per iter
    printf("%-24s %8.3f ms  DMMA %6.2f TF/s  DFMA %6.2f TF/s  total %6.2f TF/s\n", names[mode],
           ms, f_mma / ms / 1e9, f_fma / ms / 1e9, (f_mma + f_fma) / ms / 1e9);
  }
  return 0;
}
