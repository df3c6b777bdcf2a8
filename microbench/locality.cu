// DRAM locality microbenchmark for the tuple-tile access pattern of the K2 / K3 kernels.
//
// A tile = T tuples x 2^MB members (512 double2, MB = 9 - log2 T).  Member bits sit at the
// given physical positions, tuple bits fill the remaining positions from the bottom (the
// kernels' insert_zeros layout).  One warp reads its tile (16 independent 16 B loads per lane,
// lanes on the 5 lowest of the 9 tile bits) and writes it back in place: pure memory traffic
// with exactly the kernels' address pattern.  Prints GB/s (2 x 16 B per amplitude).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o locality locality.cu
//   ./locality [L=32]
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

struct Pat {
  uint64_t lane_off[32];
  uint64_t it_off[16];
  uint64_t lo_mask[9];  // member positions sorted (for zero insertion)
  int mb;
  int tb;
  uint64_t n_tiles;
  int order;  // 0: tile = warp-global index (adjacent warps adjacent tuples); 1: member-major
};

__device__ __forceinline__ uint64_t insert_zeros(uint64_t t, const uint64_t* pos, int m) {
  for (int j = 0; j < m; ++j) {
    const uint64_t p = pos[j];
    t = ((t >> p) << (p + 1)) | (t & ((1ull << p) - 1));
  }
  return t;
}

__global__ void __launch_bounds__(512, 1) tile_rw(double2* a, const __grid_constant__ Pat p, double s) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
  const uint64_t stride = (uint64_t)gridDim.x * W;
  for (uint64_t tl = (uint64_t)blockIdx.x * W + warp; tl < p.n_tiles; tl += stride) {
    double2* base = a + insert_zeros(tl << p.tb, p.lo_mask, p.mb) + p.lane_off[lane];
    double2 x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = base[p.it_off[i]];
#pragma unroll
    for (int i = 0; i < 16; ++i) base[p.it_off[i]] = make_double2(x[i].x * s, x[i].y * s);
  }
}

static Pat make_pat(const std::vector<int>& mpos, int L) {
  Pat p{};
  const int MB = (int)mpos.size(), TB = 9 - MB;
  p.mb = MB;
  p.tb = TB;
  std::vector<int> sorted = mpos;
  std::sort(sorted.begin(), sorted.end());
  for (int j = 0; j < MB; ++j) p.lo_mask[j] = sorted[j];
  // tile bit list: TB tuple bits at the lowest free positions + member bits, sorted by position
  std::vector<int> bits;
  for (int f = 0, nf = 0; f < L && nf < TB; ++f)
    if (std::find(mpos.begin(), mpos.end(), f) == mpos.end()) { bits.push_back(f); ++nf; }
  for (int m : mpos) bits.push_back(m);
  std::sort(bits.begin(), bits.end());
  for (int l = 0; l < 32; ++l) {
    uint64_t o = 0;
    for (int b = 0; b < 5; ++b) if ((l >> b) & 1) o += 1ull << bits[b];
    p.lane_off[l] = o;
  }
  for (int i = 0; i < 16; ++i) {
    uint64_t o = 0;
    for (int b = 0; b < 4; ++b) if ((i >> b) & 1) o += 1ull << bits[5 + b];
    p.it_off[i] = o;
  }
  p.n_tiles = (1ull << (L - MB)) >> TB;
  return p;
}

int main(int argc, char** argv) {
  const int L = argc > 1 ? atoi(argv[1]) : 32;
  const uint64_t N = 1ull << L;
  double2* a;
  CK(cudaMalloc(&a, N * sizeof(double2)));
  CK(cudaMemset(a, 0, N * sizeof(double2)));
  std::vector<std::vector<int>> cases = {
      {0, 1, 2, 3, 4, 5}, {6, 7, 8, 9, 10, 11}, {26, 27, 28, 29, 30, 31}, {0, 1, 28, 29, 30, 31},
      {2, 3, 28, 29, 30, 31}, {4, 5, 28, 29, 30, 31}, {6, 7, 28, 29, 30, 31}, {8, 9, 28, 29, 30, 31},
      {10, 11, 28, 29, 30, 31}, {14, 15, 28, 29, 30, 31}, {18, 19, 28, 29, 30, 31},
      {22, 23, 28, 29, 30, 31}, {10, 11, 20, 21, 30, 31}, {10, 11, 12, 13, 14, 15},
      {16, 17, 18, 19, 20, 21}, {20, 21, 22, 23, 24, 25},
      // K2-shaped tiles (32 tuples x 16 members)
      {0, 1, 30, 31}, {4, 5, 30, 31}, {6, 7, 30, 31}, {8, 9, 30, 31}, {10, 11, 30, 31},
      {14, 15, 30, 31}, {20, 21, 30, 31}, {28, 29, 30, 31}, {10, 11, 12, 13},
      // one tuple bit below the members: 8 tuples, 2^? contiguous
  };
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int warps : {16, 8}) {
    for (auto& c : cases) {
      bool ok = true;
      for (int m : c) ok &= m < L;
      if (!ok) continue;
      Pat p = make_pat(c, L);
      const int grid = 148;
      for (int w = 0; w < 2; ++w) tile_rw<<<grid, warps * 32>>>(a, p, 1.0);
      CK(cudaEventRecord(e0));
      const int reps = 3;
      for (int r = 0; r < reps; ++r) tile_rw<<<grid, warps * 32>>>(a, p, 1.0);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      ms /= reps;
      printf("warps %2d  members", warps);
      for (int m : c) printf(" %2d", m);
      printf("%*s  %8.3f ms  %7.1f GB/s\n", (int)(6 - c.size()) * 3, "", ms,
             2.0 * 16 * N / (ms * 1e-3) / 1e9);
    }
  }
  CK(cudaFree(a));
  return 0;
}
