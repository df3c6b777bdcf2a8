// Microbenchmarks for the B200 roofline of the TANQ hot path:
// DFMA peak, DMMA.8x8x4 (mma.sync f64) peak, HBM stream with 16 B and 32 B loads.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}

__global__ void copy16(const double2* __restrict__ in, double2* __restrict__ out, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) out[i] = in[i];
}

__global__ void copy32(const double* __restrict__ in, double* __restrict__ out, size_t n4) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n4; i += stride) {
    double a, b, c, d;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(in + 4 * i));
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(out + 4 * i), "d"(a), "d"(b), "d"(c), "d"(d));
  }
}

// in-place read-modify-write stream (the gate kernel's access pattern): x <- a*x
__global__ void rmw16(double2* p, size_t n, double a) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) { double2 v = p[i]; v.x *= a; v.y *= a; p[i] = v; }
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s sms %d cc %d.%d clock %d kHz mem %.1f GB l2 %d MB\n", prop.name, prop.multiProcessorCount,
         prop.major, prop.minor, prop.clockRate, prop.totalGlobalMem / 1e9, prop.l2CacheSize >> 20);
  int sms = prop.multiProcessorCount;
  double* dout; CK(cudaMalloc(&dout, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // DFMA
  {
    int iters = 20000, blocks = sms * 8, threads = 256;
    dfma_kernel<<<blocks, threads>>>(dout, 100, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(dout, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fma = (double)blocks * threads * iters * 16;
    printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", 2 * fma / ms / 1e9, ms);
  }
  // DMMA
  for (int wpb : {4, 8, 16}) {
    int iters = 20000, blocks = sms * (32 / wpb) , threads = 32 * wpb;
    dmma_kernel<<<blocks, threads>>>(dout, 100);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(dout, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fma = (double)blocks * (threads / 32) * iters * 8 * 256;
    printf("DMMA m8n8k4 (warps/blk %d, blocks %d): %.2f TFLOP/s (%.3f ms)\n", wpb, blocks, 2 * fma / ms / 1e9, ms);
  }
  // HBM
  size_t bytes = (size_t)8 << 30;  // 8 GiB per buffer
  double *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
  CK(cudaMemset(a, 0, bytes)); CK(cudaMemset(b, 0, bytes));
  size_t n16 = bytes / 16, n32 = bytes / 32;
  for (int rep = 0; rep < 2; ++rep) {
    for (int bpsm : {4, 8, 16}) {
      int blocks = sms * bpsm;
      copy16<<<blocks, 256>>>((double2*)a, (double2*)b, n16); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) copy16<<<blocks, 256>>>((double2*)a, (double2*)b, n16);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      printf("copy LDG.128 blocks/sm %d: %.1f GB/s\n", bpsm, 5 * 2.0 * bytes / ms / 1e6);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) copy32<<<blocks, 256>>>(a, b, n32);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      printf("copy LDG.256 blocks/sm %d: %.1f GB/s\n", bpsm, 5 * 2.0 * bytes / ms / 1e6);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) rmw16<<<blocks, 256>>>((double2*)a, n16, 1.0);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      printf("in-place rmw LDG.128 blocks/sm %d: %.1f GB/s\n", bpsm, 5 * 2.0 * bytes / ms / 1e6);
    }
  }
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) CK(cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice));
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  printf("cudaMemcpy D2D: %.1f GB/s\n", 5 * 2.0 * bytes / ms / 1e6);
  size_t fr, tot; cudaMemGetInfo(&fr, &tot); printf("free %.1f GB total %.1f GB\n", fr / 1e9, tot / 1e9);
  return 0;
}
