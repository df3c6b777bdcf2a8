// sm_100a kernels of the TANQ hot path.
//
//   K1/K2  gate_kernel<K>   FMA register stream: 4^K-member tuple gathered with 16 B (or,
//                           when physical bit 0 is a target bit, 32 B) loads, y = S x with S
//                           read from the kernel-parameter constant bank, written in place.
//   K3     gate3_kernel     fused 3-qubit ops: 64x64 complex superoperator on the FP64
//                           tensor pipe (mma.sync m8n8k4 f64 -> DMMA.8x8x4), tuples staged
//                           through shared memory with cp.async, 3-real-multiply complex GEMM.
//   remap  swap/pack/unpack, vec<->physical gather/scatter, diagonal, readout, Pauli
//          expectation, CDF + Philox sampling.
//
// Paper: each op performs 4^{n-k} independent [4^k x 4^k] x [4^k] complex mat-vecs on the
// tuples of Eq. 4; the tuple base s_i is the tuple index with zero bits inserted
// at the target positions (generalised to arbitrary physical bit positions here).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>

#include "tanq_internal.h"

namespace tanq {

static constexpr int kThreads = 256;

// cudaFuncSetAttribute applies to the current device only: raise the dynamic shared-memory
// limit once per (kernel, device) -- a handle may spread shards over several devices.
template <typename Kern>
static cudaError_t ensure_smem_attr(Kern kern, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = (uint64_t)1 << (dev & 63);
  if (done.load(std::memory_order_relaxed) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e == cudaSuccess) done.fetch_or(bit);
  return e;
}

// Debug / test knob (env TANQ_GRID_CAP=N, default off): cap the grid of the persistent group,
// tile and DMMA k=2 kernels at N CTAs so that small registers still run many tiles per warp
// (the loop paths a full-size launch takes).  Never set in production.
static unsigned grid_cap() {
  static int cap = -1;
  if (cap < 0) {
    const char* e = getenv("TANQ_GRID_CAP");
    cap = e ? atoi(e) : 0;
    if (cap < 0) cap = 0;
  }
  return (unsigned)cap;
}
static inline unsigned capped(unsigned g) {
  const unsigned c = grid_cap();
  return (c && g > c) ? c : g;
}

static inline unsigned grid_for(uint64_t work, int threads, uint64_t cap = 148ull * 64) {
  uint64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

__device__ __forceinline__ uint64_t insert_zeros(uint64_t t, const uint64_t* lo, int cnt) {
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (j < cnt) t = ((t & ~lo[j]) << 1) | (t & lo[j]);
  return t;
}

// Hermitian mirror (DESIGN.md §5 "mirror mode"): with the interleaved single-shard layout
// the row / column bits of every qubit are adjacent, so the transpose position of a tuple
// index (or of a member index) swaps each adjacent bit pair.  rho' Hermitian gives
// rho'[mirror] = conj(rho'[element]).
__device__ __forceinline__ uint64_t pair_swap(uint64_t x) {
  return ((x & 0x5555555555555555ull) << 1) | ((x >> 1) & 0x5555555555555555ull);
}
__device__ __forceinline__ double2 cj(double2 v) { return make_double2(v.x, -v.y); }
// Transpose of an index from which r low bits (whole pairs below the pair boundary) have been
// removed, under the shard's transpose descriptor (TDesc, tanq_internal.h): pairs below the
// boundary swap, the half-global row bits above it flip by the shard mask.
__device__ __forceinline__ uint64_t tpose(uint64_t x, uint64_t lo, uint64_t m, int r) {
  const uint64_t l = lo >> r;
  return pair_swap(x & l) | ((x & ~l) ^ (m >> r));
}

// Packed Hermitian layout: of each transpose pair {e, pair_swap(e)} only the
// element with e <= pair_swap(e) is kept up to date (diagonal-type elements e = pair_swap(e)
// always); the other is recovered as conj of its transpose.  Kernels in packed mode read and
// write one element per pair: 16 B per amplitude per pass instead of 32.  The kernels process
// the tuple / tile t <= pair_swap(t) of each transpose pair, whose elements are then mostly
// stored in place (no conjugation, no transposed addresses) -- the same orientation.
__device__ __forceinline__ bool packed_stored(uint64_t e, uint64_t e_mirror) { return e <= e_mirror; }
__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
// A tile whose base index has a differing (row, col) pair above every in-tile position `hi`
// orders all its elements against their transposes the same way: when that pair makes the
// base the stored one, every element is read and written in place (the common case for the
// canonical tiles the kernels visit) and the per-element test is skipped.
// (A differing pair counts at its lower position; a flipped half-global row bit at its own.)
__device__ __forceinline__ bool packed_tile_direct(uint64_t base, int hi, uint64_t lo, uint64_t m) {
  const uint64_t bt = tpose(base, lo, m, 0);
  const uint64_t d = (base ^ bt) & (0x5555555555555555ull | ~lo);
  if (!d) return false;
  const int hb = 63 - __clzll(d);
  return hb > hi && packed_stored(base, bt);
}

__device__ __forceinline__ void ld32(const double2* p, double2& a, double2& b) {
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
               : "l"(p));
}
__device__ __forceinline__ void st32(double2* p, const double2& a, const double2& b) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x),
               "d"(b.y)
               : "memory");
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__host__ __device__ constexpr int pswap_c(int i) {
  return ((i & 0x55) << 1) | ((i >> 1) & 0x55);
}

// ------------------------------------------------------------------------------------
// K1 / K2: FMA register stream
// ------------------------------------------------------------------------------------
template <int K, bool PAIR>
__global__ void __launch_bounds__(kThreads, K == 2 ? 2 : 1)
    gate_kernel(double2* __restrict__ a, const __grid_constant__ GateParams<K> p) {
  constexpr int M = 1 << (2 * K);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < p.n_tuples; t += stride) {
    uint64_t tm = t;
    if (p.mirror) {  // packed mode: only the canonical tuple of each transpose pair
      tm = tpose(t, p.tp_lo, p.tp_m, 2 * K);
      if (tm < t) continue;
    }
    uint64_t base = t, basem = tm;
#pragma unroll
    for (int j = 0; j < 2 * K; ++j) {
      base = ((base & ~p.lo_mask[j]) << 1) | (base & p.lo_mask[j]);
      basem = ((basem & ~p.lo_mask[j]) << 1) | (basem & p.lo_mask[j]);
    }
    double2* ptr = a + base;
    uint64_t off[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      uint64_t o = 0;
#pragma unroll
      for (int j = 0; j < 2 * K; ++j)
        if ((i >> j) & 1) o += (uint64_t)1 << p.pos[j];
      off[i] = o;
    }
    double2 x[M];
    if (p.mirror) {  // member i lives at its own address if stored there, else at its transpose
#pragma unroll
      for (int i = 0; i < M; ++i) {  // one load per element: select the address first
        const uint64_t e = base + off[i], em = basem + off[pswap_c(i)];
        const bool in_place = packed_stored(e, em);
        const double2 v = a[in_place ? e : em];
        x[i] = in_place ? v : cj(v);
      }
    } else if constexpr (PAIR) {
#pragma unroll
      for (int i = 0; i < M; i += 2) ld32(ptr + off[i], x[i], x[i + 1]);
    } else {
#pragma unroll
      for (int i = 0; i < M; ++i) x[i] = ptr[off[i]];
    }
#pragma unroll
    for (int l = 0; l < M; l += 2) {
      double2 y[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        double yr = 0.0, yi = 0.0;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const double2 s = p.S[(l + u) * M + m];
          yr = fma(s.x, x[m].x, yr);
          yr = fma(-s.y, x[m].y, yr);
          yi = fma(s.x, x[m].y, yi);
          yi = fma(s.y, x[m].x, yi);
        }
        y[u] = make_double2(yr, yi);
      }
      if (p.mirror) {  // store each result where the packed layout keeps it
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint64_t e = base + off[l + u], em = basem + off[pswap_c(l + u)];
          if (packed_stored(e, em)) a[e] = y[u];
          else if (tm != t) a[em] = cj(y[u]);  // self tuple: the transpose is stored above
        }
      } else if constexpr (PAIR) {
        st32(ptr + off[l], y[0], y[1]);
      } else {
        ptr[off[l]] = y[0];
        ptr[off[l + 1]] = y[1];
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// K2 on the FP64 tensor pipe: one warp = 8 tuples per tile, Y[16x8] = S[16x16] X[16x8]
// as three real m8n8k4 GEMMs (P1 = Sr Xr, P2 = Si Xi, P3 = (Sr+Si)(Xr+Xi);
// Yr = P1 - P2, Yi = P3 - P1 - P2), operands straight from registers:
//   A fragments (S, constant for the launch) live in registers for the whole kernel,
//   B fragment of k-step ks = member 4ks + (lane&3) of tuple lane>>2 -> one 16 B load,
//   D fragment = member 8mt + (lane>>2) of tuples 2(lane&3), 2(lane&3)+1 -> one 32 B store
//   when consecutive tuples are adjacent in memory (physical bit 0 not a target).
// The next tile's loads are issued before the current tile's DMMAs (register prefetch).
// Packed Hermitian mode: canonical 16-tuple blocks only; each element is read from / written
// to where the packed layout keeps it (self-transposed blocks: named barrier, in-place only).
template <bool ADJ>
__global__ void __launch_bounds__(256, 2)
    gate2_mma_kernel(double2* __restrict__ a, const __grid_constant__ GateParams<2> p) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t n_tiles = (p.n_tuples + 7) >> 3;
  const int r4 = lane >> 2, c4 = lane & 3;

  // S staged in shared memory: if register pressure makes the compiler re-load a fragment
  // inside the loop it is a conflict-free LDS, not a lane-indexed (serialised) constant load
  __shared__ double2 sS[256];
  for (int e = threadIdx.x; e < 256; e += blockDim.x) sS[e] = p.S[e];
  __syncthreads();
  double sr[2][4], si[2][4], ss[2][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const double2 v = sS[(8 * mt + r4) * 16 + 4 * ks + c4];
      sr[mt][ks] = v.x;
      si[mt][ks] = v.y;
      ss[mt][ks] = v.x + v.y;
    }
  auto member_off = [&](int m) {
    uint64_t o = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if ((m >> j) & 1) o += (uint64_t)1 << p.pos[j];
    return o;
  };
  uint64_t offB[4], offD[2];  // (transposed offsets are formed on the packed slow path only,
#pragma unroll                // keeping the S fragments resident in registers)
  for (int ks = 0; ks < 4; ++ks) offB[ks] = member_off(4 * ks + c4);
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) offD[mt] = member_off(8 * mt + r4);
  auto base_of = [&](uint64_t t) {
    uint64_t b = t;
#pragma unroll
    for (int j = 0; j < 4; ++j) b = ((b & ~p.lo_mask[j]) << 1) | (b & p.lo_mask[j]);
    return b;
  };
  // highest in-tile position: the 3 tuple bits of a tile sit at the lowest free positions
  int hi_tile = (int)p.pos[3];
  for (int f = 0, nf = 0; f < 64 && nf < 3; ++f)
    if (f != (int)p.pos[0] && f != (int)p.pos[1] && f != (int)p.pos[2] && f != (int)p.pos[3]) {
      hi_tile = max(hi_tile, f);
      ++nf;
    }
  // packed mode: the transpose of (tuple t, member m) is (pair_swap(t), pswap_c(m)); tiles
  // whose elements are all stored in place (packed_tile_direct) skip the per-element test
  auto tile_packed = [&](uint64_t tl) {
    return p.mirror && !packed_tile_direct(base_of(tl * 8), hi_tile, p.tp_lo, p.tp_m);
  };
  auto load_tile = [&](uint64_t tl, double2* x, bool packed) {
    const uint64_t t = tl * 8 + r4;
    if (tl < n_tiles && t < p.n_tuples) {
      const uint64_t b = base_of(t);
      if (packed) {
        const uint64_t bm = base_of(tpose(t, p.tp_lo, p.tp_m, 4));
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {  // one load per element: select the address first
          const uint64_t e = b + offB[ks], em = bm + member_off(pswap_c(4 * ks + c4));
          const bool in_place = packed_stored(e, em);
          const double2 v = a[in_place ? e : em];
          x[ks] = in_place ? v : cj(v);
        }
      } else {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) x[ks] = a[b + offB[ks]];
      }
    } else {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) x[ks] = make_double2(0.0, 0.0);
    }
  };
  // packed mode: only tiles of canonical 16-tuple blocks (block b <= its transpose block);
  // the two tiles of a block belong to warps 2j, 2j+1 of one CTA
  auto next_tile = [&](uint64_t tl) {
    if (p.mirror)
      while (tl < n_tiles && (tl >> 1) > tpose(tl >> 1, p.tp_lo, p.tp_m, 8)) tl += nwarps;
    return tl;
  };

  double2 xb_cur[4], xb_nxt[4];
  uint64_t tile = next_tile(warp);
  bool pk_cur = tile < n_tiles && tile_packed(tile);
  load_tile(tile, xb_cur, pk_cur);
  while (tile < n_tiles) {
    const uint64_t nxt = next_tile(tile + nwarps);
    const bool pk_nxt = nxt < n_tiles && tile_packed(nxt);
    load_tile(nxt, xb_nxt, pk_nxt);  // register prefetch of the next tile
    double p1[2][2], p2[2][2], p3[2][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
      p1[mt][0] = p1[mt][1] = p2[mt][0] = p2[mt][1] = p3[mt][0] = p3[mt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const double2 xb = xb_cur[ks];
      const double xs = xb.x + xb.y;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        dmma(p1[mt][0], p1[mt][1], sr[mt][ks], xb.x);
        dmma(p2[mt][0], p2[mt][1], si[mt][ks], xb.y);
        dmma(p3[mt][0], p3[mt][1], ss[mt][ks], xs);
      }
    }
    const uint64_t t0 = tile * 8 + 2 * c4;
    const bool self = p.mirror && (tile >> 1) == tpose(tile >> 1, p.tp_lo, p.tp_m, 8);
    if (self) named_bar(1 + ((threadIdx.x >> 5) >> 1), 64);  // both tiles' loads are done
    const uint64_t b0 = base_of(t0), b1 = base_of(t0 + 1);
    uint64_t bm0 = 0, bm1 = 0;
    if (pk_cur) {
      bm0 = base_of(tpose(t0, p.tp_lo, p.tp_m, 4));
      bm1 = base_of(tpose(t0 + 1, p.tp_lo, p.tp_m, 4));
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const double2 y0 = make_double2(p1[mt][0] - p2[mt][0], p3[mt][0] - p1[mt][0] - p2[mt][0]);
      const double2 y1 = make_double2(p1[mt][1] - p2[mt][1], p3[mt][1] - p1[mt][1] - p2[mt][1]);
      const uint64_t e0 = b0 + offD[mt], e1 = b1 + offD[mt];
      if (!pk_cur) {
        if (ADJ && t0 + 1 < p.n_tuples) {
          st32(a + e0, y0, y1);
        } else {
          if (t0 < p.n_tuples) a[e0] = y0;
          if (t0 + 1 < p.n_tuples) a[e1] = y1;
        }
      } else {  // slow path: per-element placement
        const uint64_t om = member_off(pswap_c(8 * mt + r4));
        if (t0 < p.n_tuples) {
          if (packed_stored(e0, bm0 + om)) a[e0] = y0;
          else if (!self) a[bm0 + om] = cj(y0);
        }
        if (t0 + 1 < p.n_tuples) {
          if (packed_stored(e1, bm1 + om)) a[e1] = y1;
          else if (!self) a[bm1 + om] = cj(y1);
        }
      }
    }
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) xb_cur[ks] = xb_nxt[ks];
    pk_cur = pk_nxt;
    tile = nxt;
  }
}

template <int K>
static cudaError_t launch_gate_impl(double2* a, const GateParams<K>& p, cudaStream_t st) {
  // grid-stride: up to 32 resident 256-thread waves per SM-count multiple
  unsigned grid = grid_for(p.n_tuples, kThreads, 148ull * 256);
  if (p.pos[0] == 0)
    gate_kernel<K, true><<<grid, kThreads, 0, st>>>(a, p);
  else
    gate_kernel<K, false><<<grid, kThreads, 0, st>>>(a, p);
  return cudaGetLastError();
}

cudaError_t launch_gate1(double2* a, const GateParams<1>& p, cudaStream_t st) {
  return launch_gate_impl<1>(a, p, st);
}
static int g_k2_variant = -1;  // 0 = FMA stream, 1 = DMMA (default); env TANQ_K2=fma|mma

cudaError_t launch_gate2(double2* a, const GateParams<2>& p, cudaStream_t st) {
  if (g_k2_variant < 0) {
    const char* e = getenv("TANQ_K2");
    g_k2_variant = (e && e[0] == 'f') ? 0 : 1;
  }
  if (g_k2_variant == 0) return launch_gate_impl<2>(a, p, st);
  const uint64_t tiles = (p.n_tuples + 7) / 8;
  uint64_t warps = tiles;
  const uint64_t cap = 148ull * 16;  // one wave: 2 CTAs x 8 warps per SM, persistent
  if (warps > cap) warps = cap;
  unsigned grid = capped((unsigned)((warps + 7) / 8));
  if (p.pos[0] == 0)
    gate2_mma_kernel<false><<<grid, 256, 0, st>>>(a, p);
  else
    gate2_mma_kernel<true><<<grid, 256, 0, st>>>(a, p);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// K3: 3- and 4-qubit groups on DMMA.8x8x4 (mma.sync.m8n8k4 f64).
//
// One HBM round trip per group: a warp stages a tile of 512 amplitudes -- T tuples x 4^NQ
// members, the group's 2*NQ physical bits (NQ = 3: 8 x 64, NQ = 4: 2 x 256) -- in shared
// memory with cp.async, runs the group's program of sub-ops on the tile, and writes the tile
// back.  Sub-ops:
//   k=3  dense 64x64 superoperator (NQ = 3 only; the fused k=3 op of SURVEY A-5): Y = S X.
//   k=2  16x16 superoperator on the 4^(NQ-2) sub-tuples of each tuple: Y[16x32] = S X[16x32].
//   k=1  4x4 superoperator on the 4^(NQ-1) sub-tuples (FMA).
// Complex products use three real GEMMs: P1 = Sr Xr, P2 = Si Xi, P3 = (Sr+Si)(Xr+Xi);
// Yr = P1 - P2, Yi = P3 - P1 - P2 (25% fewer FP64 ops than the paper's 4-MMA scheme).
// Fragments (PTX m8n8k4 .row.col f64): A[8x4] lane -> (lane>>2, lane&3);
// B[4x8] lane -> (k = lane&3, n = lane>>2); D[8x8] lane -> (lane>>2, 2*(lane&3)+{0,1}).
// The 32 columns of a k=2 sub-op are (sub-tuple u, tuple t): col = u*T + t.
// Sub-op matrices are stored in A-fragment order by the host (group_make_*).
// ------------------------------------------------------------------------------------

// Tile element (member m, tuple t), linear e = m*T + t, lives at e ^ ((e >> 3) & 7) (XOR
// swizzle; for NQ = 3 this is m*8 + (t ^ (m & 7))): conflict-free tuple-major fragment reads
// and address-ordered global<->shared copies.
template <int T>
__device__ __forceinline__ int xs_idx(int m, int t) {
  const int e = m * T + t;
  if constexpr (T == 32)  // 2-qubit tiles (32 tuples x 16 members): slot t ^ f(m), f = 0,3,4,7
    return e ^ (((m & 3) << 1) | (m & 1));
  else
    return e ^ ((e >> 3) & 7);
}

size_t group_frag_elems(int k) { return k == 3 ? 4096 : (k == 2 ? 256 : 16); }

void group_make_frags(int k, const double2* S, double2* frag) {
  if (k == 1) {
    for (int i = 0; i < 16; ++i) frag[i] = S[i];
    return;
  }
  const int M = k == 3 ? 64 : 16, KS = M / 4, MT = M / 8;
  for (int mt = 0; mt < MT; ++mt)
    for (int ks = 0; ks < KS; ++ks)
      for (int lane = 0; lane < 32; ++lane) {
        const int row = mt * 8 + (lane >> 2), col = ks * 4 + (lane & 3);
        frag[((size_t)mt * KS + ks) * 32 + lane] = S[row * M + col];
      }
}

__device__ __forceinline__ void group_sub_k3(double2* X, const double2* F, int lane) {
  // NQ = 3 only (T = 8): tile members are the sub-op members
  const int r4 = lane >> 2, c4 = lane & 3;
  double p1[8][2], p2[8][2], p3[8][2];
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) p1[mt][0] = p1[mt][1] = p2[mt][0] = p2[mt][1] = p3[mt][0] = p3[mt][1] = 0.0;
#pragma unroll 4
  for (int ks = 0; ks < 16; ++ks) {
    const double2 xb = X[xs_idx<8>(ks * 4 + c4, r4)];
    const double xs = xb.x + xb.y;
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      const double2 sv = F[(mt * 16 + ks) * 32 + lane];
      dmma(p1[mt][0], p1[mt][1], sv.x, xb.x);
      dmma(p2[mt][0], p2[mt][1], sv.y, xb.y);
      dmma(p3[mt][0], p3[mt][1], sv.x + sv.y, xs);
    }
  }
  __syncwarp();
#pragma unroll
  for (int mt = 0; mt < 8; ++mt)
#pragma unroll
    for (int c = 0; c < 2; ++c)
      X[xs_idx<8>(mt * 8 + r4, 2 * c4 + c)] =
          make_double2(p1[mt][c] - p2[mt][c], p3[mt][c] - p1[mt][c] - p2[mt][c]);
}

template <int T, int UI>  // T tuples per tile; UI n-tiles (of 8 columns) processed at once
__device__ __forceinline__ void group_sub_k2(double2* X, const double2* F, const uint8_t* mi,
                                             const uint8_t* mu, int lane) {
  constexpr int TB = T == 32 ? 5 : (T == 8 ? 3 : 1);
  const int r4 = lane >> 2, c4 = lane & 3;
  double sr[2][4], si[2][4], ss[2][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const double2 v = F[(mt * 4 + ks) * 32 + lane];
      sr[mt][ks] = v.x;
      si[mt][ks] = v.y;
      ss[mt][ks] = v.x + v.y;
    }
  int mb[4], md[2];
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) mb[ks] = mi[4 * ks + c4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) md[mt] = mi[8 * mt + r4];
  // B column of this lane in n-tile j: (sub-tuple member offset, tuple) = (col >> TB, col % T)
  int mob[4], tb[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if constexpr (T == 8) {  // col >> 3 = n-tile, col & 7 = r4
      mob[j] = mu[j];
      tb[j] = r4;
    } else {
      const int col = j * 8 + r4;
      mob[j] = mu[col >> TB];
      tb[j] = col & (T - 1);
    }
  }
  // The n-tile passes touch disjoint columns (tile elements), and every mma.sync converges the
  // warp after its B loads, so passes need no __syncwarp between them: the first k-step of
  // the next pass is loaded before this pass's epilogue, overlapping it with the DMMA tail.
  double2 xn[UI];
#pragma unroll
  for (int u = 0; u < UI; ++u) xn[u] = X[xs_idx<T>(mb[0] | mob[u], tb[u])];
#pragma unroll
  for (int n0 = 0; n0 < 4; n0 += UI) {
    double p1[UI][2][2], p2[UI][2][2], p3[UI][2][2];
#pragma unroll
    for (int u = 0; u < UI; ++u)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
        p1[u][mt][0] = p1[u][mt][1] = p2[u][mt][0] = p2[u][mt][1] = p3[u][mt][0] = p3[u][mt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      double2 xb[UI];
#pragma unroll
      for (int u = 0; u < UI; ++u)
        xb[u] = ks == 0 ? xn[u] : X[xs_idx<T>(mb[ks] | mob[n0 + u], tb[n0 + u])];
      if (ks == 3 && n0 + UI < 4) {
#pragma unroll
        for (int u = 0; u < UI; ++u) xn[u] = X[xs_idx<T>(mb[0] | mob[n0 + UI + u], tb[n0 + UI + u])];
      }
#pragma unroll
      for (int u = 0; u < UI; ++u) {
        const double xs = xb[u].x + xb[u].y;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          dmma(p1[u][mt][0], p1[u][mt][1], sr[mt][ks], xb[u].x);
          dmma(p2[u][mt][0], p2[u][mt][1], si[mt][ks], xb[u].y);
          dmma(p3[u][mt][0], p3[u][mt][1], ss[mt][ks], xs);
        }
      }
    }
    __syncwarp();  // every lane's B loads of this pass precede any lane's D stores
#pragma unroll
    for (int u = 0; u < UI; ++u)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int col = (n0 + u) * 8 + 2 * c4 + c;
        const int mo = T == 8 ? mob[n0 + u] : mu[col >> TB], t = col & (T - 1);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
          X[xs_idx<T>(md[mt] | mo, t)] = make_double2(
              p1[u][mt][c] - p2[u][mt][c], p3[u][mt][c] - p1[u][mt][c] - p2[u][mt][c]);
      }
  }
  __syncwarp();
}

template <int T>
__device__ __forceinline__ void group_sub_k1(double2* X, const double2* F, const uint8_t* mi,
                                             const uint8_t* mu, int lane) {
  constexpr int TB = T == 32 ? 5 : (T == 8 ? 3 : 1);
  double2 S[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) S[i] = F[i];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int col = lane + 32 * j, mo = mu[col >> TB], t = col & (T - 1);
    double2 x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = X[xs_idx<T>(mi[i] | mo, t)];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      double yr = 0.0, yi = 0.0;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        yr = fma(S[l * 4 + m].x, x[m].x, yr);
        yr = fma(-S[l * 4 + m].y, x[m].y, yr);
        yi = fma(S[l * 4 + m].x, x[m].y, yi);
        yi = fma(S[l * 4 + m].y, x[m].x, yi);
      }
      X[xs_idx<T>(mi[l] | mo, t)] = make_double2(yr, yi);
    }
  }
}

// Packed-mode copy helpers shared by the group and tile kernels.  An element at tile-relative
// offset off has its transpose at pair_swap(off) relative to pair_swap(base) (pair_swap is a
// bit permutation, so it distributes over the disjoint base / offset bits).

// NQ group qubits, WARPS warps per CTA (one CTA per SM), NBUF tile buffers per warp
// (2 = cp.async double buffering), HAS3: the program may contain a dense k=3 sub-op (needs
// the register budget of 8 warps), UI: n-tiles per k=2 pass.
// Packed mode (p.mirror): only tiles of canonical 16-tuple blocks are processed; every element
// is read from, and written to, the one of {itself, its transpose} the packed layout keeps.
// A self-transposed block spans 16 / T warp tiles that read each other's elements: those warps
// meet at a named barrier between their loads and their stores.
template <int NQ, int WARPS, int NBUF, bool HAS3, int UI>
__global__ void __launch_bounds__(WARPS * 32, 1)
    group_kernel(double2* __restrict__ a, const __grid_constant__ GroupParams p) {
  constexpr int MB = 2 * NQ, TB = 9 - MB, T = 1 << TB;
  constexpr int WPB = 16 / T;  // warp tiles per 16-tuple block
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // shared: program | X tiles WARPS x NBUF x 512 double2 |
  //         copy tables | sub-op headers
  double2* sProg = reinterpret_cast<double2*>(smem_raw);
  double2* sX = sProg + ((p.prog_elems + 7) & ~7);
  // copy tables: iteration i (16) -> offset [i], transpose offset [16 + i], tuple/member bits
  uint64_t* sIterOff = reinterpret_cast<uint64_t*>(sX + WARPS * NBUF * 512);  // [2][16]
  int* sIterTM = reinterpret_cast<int*>(sIterOff + 32);                          // [16]
  GroupSub* sSub = reinterpret_cast<GroupSub*>(sIterTM + 32);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // The 9 index bits of a tile element (TB tuple bits at the lowest free physical positions,
  // MB member bits at pos[]) sorted by physical position: lanes take the 5 lowest, the copy
  // iterations the next 4, so every copy instruction covers the most contiguous addresses.
  int freep[4];
  {
    int nf = 0;
    for (int f = 0; f < 64 && nf < 4; ++f) {
      bool tgt = false;
      for (int j = 0; j < MB; ++j) tgt |= (int)p.pos[j] == f;
      if (!tgt) freep[nf++] = f;
    }
  }
  int lane_tm;
  uint64_t lane_off;
  {
    int bit_pos[9], bit_id[9];  // id < TB: tuple bit, else member bit id-TB
    for (int j = 0; j < TB; ++j) {
      bit_pos[j] = freep[j];
      bit_id[j] = j;
    }
    for (int j = 0; j < MB; ++j) {
      bit_pos[TB + j] = (int)p.pos[j];
      bit_id[TB + j] = TB + j;
    }
    for (int x = 1; x < 9; ++x)  // insertion sort by position
      for (int y = x; y > 0 && bit_pos[y] < bit_pos[y - 1]; --y) {
        int tp = bit_pos[y]; bit_pos[y] = bit_pos[y - 1]; bit_pos[y - 1] = tp;
        int ti = bit_id[y]; bit_id[y] = bit_id[y - 1]; bit_id[y - 1] = ti;
      }
    auto tm_of = [&](int bits, int first, int cnt, uint64_t& off) {
      int t = 0, m = 0;
      off = 0;
      for (int b = 0; b < cnt; ++b)
        if ((bits >> b) & 1) {
          const int id = bit_id[first + b];
          if (id < TB) t |= 1 << id; else m |= 1 << (id - TB);
          off += (uint64_t)1 << bit_pos[first + b];
        }
      return t | (m << TB);
    };
    lane_tm = tm_of(lane, 0, 5, lane_off);
    if (threadIdx.x < 16) {
      sIterTM[threadIdx.x] = tm_of(threadIdx.x, 5, 4, sIterOff[threadIdx.x]);
      sIterOff[16 + threadIdx.x] = pair_swap(sIterOff[threadIdx.x]);
    }
  }
  const uint64_t lane_poff = pair_swap(lane_off);
  const int hi_tile = max(freep[TB - 1], (int)p.pos[MB - 1]);  // highest in-tile position
  for (int e = threadIdx.x; e < p.prog_elems; e += blockDim.x) sProg[e] = p.prog[e];
  for (int e = threadIdx.x; e < p.n_sub; e += blockDim.x) sSub[e] = p.sub[e];
  __syncthreads();

  const uint64_t n_tiles = (p.n_tuples + T - 1) >> TB;
  const uint64_t tile_stride = (uint64_t)gridDim.x * WARPS;
  // packed mode: only tiles of canonical 16-tuple blocks (block b <= its transpose block)
  auto block_of = [&](uint64_t tl) { return (tl << TB) >> 4; };
  auto next_tile = [&](uint64_t tl) {
    if (p.mirror)
      while (tl < n_tiles && block_of(tl) > tpose(block_of(tl), p.tp_lo, p.tp_m, MB + 4))
        tl += tile_stride;
    return tl;
  };
  uint64_t tile = next_tile((uint64_t)blockIdx.x * WARPS + warp);
  double2* const wbuf = sX + warp * NBUF * 512;  // NBUF 512-double2 tiles (no indexed array:
                                                  // a dynamically indexed pointer array spills)
  // issue the tile's copies; returns the mask of elements copied from transpose positions
  auto issue_load = [&](uint64_t tl, double2* buf) {
    const uint64_t tb0 = insert_zeros(tl << TB, p.lo_mask, MB);
    const uint64_t base = tb0 + lane_off, pbase = tpose(tb0, p.tp_lo, p.tp_m, 0) + lane_poff;
    const bool packed = p.mirror && !packed_tile_direct(tb0, hi_tile, p.tp_lo, p.tp_m);
    unsigned mask = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int tm = lane_tm | sIterTM[i];
      const int t = tm & (T - 1), m = tm >> TB;
      const bool ok = (tl << TB) + t < p.n_tuples;
      uint64_t src = base + sIterOff[i];
      if (packed) {
        const uint64_t srcm = pbase + sIterOff[16 + i];
        if (!packed_stored(src, srcm)) {
          src = srcm;
          mask |= 1u << i;
        }
      }
      cp_async16(buf + xs_idx<T>(m, t), ok ? a + src : a, ok);
    }
    cp_async_commit();
    return mask;
  };
  auto fixup = [&](double2* buf, unsigned mask) {
    for (; mask; mask &= mask - 1) {
      const int tm = lane_tm | sIterTM[__ffs(mask) - 1];
      double* im = &buf[xs_idx<T>(tm >> TB, tm & (T - 1))].y;
      *im = -*im;
    }
  };

  unsigned mask_next = 0;
  if (NBUF == 2 && tile < n_tiles) mask_next = issue_load(tile, wbuf);
  int cur = 0;
  for (; tile < n_tiles; tile = next_tile(tile + tile_stride)) {
    unsigned mask;
    if constexpr (NBUF == 2) {
      mask = mask_next;
      const uint64_t next = next_tile(tile + tile_stride);
      if (next < n_tiles) {
        mask_next = issue_load(next, wbuf + ((cur ^ 1) << 9));
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
    } else {
      mask = (p.dbg & 2) ? 0u : issue_load(tile, wbuf);
      cp_async_wait<0>();
    }
    double2* X = wbuf + (NBUF == 2 ? (cur << 9) : 0);
    fixup(X, mask);
    __syncwarp();
    for (int s = 0; s < (p.dbg & 1 ? 0 : p.n_sub); ++s) {
      const GroupSub& g = sSub[s];
      const double2* F = sProg + g.s_off;
      if (g.k == 2) {
        group_sub_k2<T, UI>(X, F, g.mi, g.mu, lane);
      } else if (g.k == 3) {
        if constexpr (HAS3 && NQ == 3) group_sub_k3(X, F, lane);
      } else {
        group_sub_k1<T>(X, F, g.mi, g.mu, lane);
      }
      __syncwarp();
    }
    const bool self =
        p.mirror && block_of(tile) == tpose(block_of(tile), p.tp_lo, p.tp_m, MB + 4);
    if (self) named_bar(1 + warp / WPB, 32 * WPB);  // the block's loads are all done
    if (!(p.dbg & 2)) {
      const uint64_t tb0 = insert_zeros(tile << TB, p.lo_mask, MB);
      const uint64_t base = tb0 + lane_off, pbase = tpose(tb0, p.tp_lo, p.tp_m, 0) + lane_poff;
      const bool packed = p.mirror && !packed_tile_direct(tb0, hi_tile, p.tp_lo, p.tp_m);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int tm = lane_tm | sIterTM[i];
        const int t = tm & (T - 1), m = tm >> TB;
        if ((tile << TB) + t >= p.n_tuples) continue;
        const uint64_t dst = base + sIterOff[i];
        const double2 v = X[xs_idx<T>(m, t)];
        if (!packed) {
          a[dst] = v;
        } else {
          const uint64_t dstm = pbase + sIterOff[16 + i];
          if (packed_stored(dst, dstm)) a[dst] = v;
          else if (!self) a[dstm] = cj(v);  // self block: the transpose is stored directly
        }
      }
    }
    __syncwarp();
    cur ^= 1;
  }
}

template <int NQ, int WARPS, int NBUF, bool HAS3, int UI>
static size_t group_smem(const GroupParams& p) {
  return (size_t)((p.prog_elems + 7) & ~7) * sizeof(double2) +
         (size_t)WARPS * NBUF * 512 * sizeof(double2) + 32 * 8 + 32 * 4 +
         (size_t)p.n_sub * sizeof(GroupSub);
}

template <int NQ, int WARPS, int NBUF, bool HAS3, int UI>
static cudaError_t launch_group_cfg(double2* a, const GroupParams& p, cudaStream_t st) {
  static std::atomic<uint64_t> attr_done{0};
  constexpr int T = 1 << (9 - 2 * NQ);
  const size_t smem = group_smem<NQ, WARPS, NBUF, HAS3, UI>(p);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  auto kern = group_kernel<NQ, WARPS, NBUF, HAS3, UI>;
  cudaError_t ea = ensure_smem_attr(kern, attr_done);
  if (ea != cudaSuccess) return ea;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t tiles = (p.n_tuples + T - 1) / T;
  const uint64_t ctas = (tiles + WARPS - 1) / WARPS;
  unsigned grid = capped((unsigned)(ctas < (uint64_t)sms ? ctas : (uint64_t)sms));
  if (grid < 1) grid = 1;
  kern<<<grid, WARPS * 32, smem, st>>>(a, p);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// Cooperative tiles: one CTA (WARPS warps) owns a tile of WARPS x 512 amplitudes = TT tuples x
// 4^NQ members (TT = WARPS x T; 4 warps: 128 tuples for NQ = 2, 32 for NQ = 3, 8 for NQ = 4).
// The tile's index bits -- the TTB lowest free physical positions (tuple bits) and the 2 NQ
// member positions -- include physical positions 0..4 whenever TTB >= 5, so every warp-wide
// copy instruction moves one contiguous 512 B run (microbench/locality.cu: 5.9-6.1 TB/s for
// any member positions, against 4.1-4.9 TB/s for 8-tuple warp tiles whose members sit at
// position >= 6).  Warp w computes on tuples [wT, (w+1)T) of the tile with the sub-op code
// above; only the copies are shared.
// Packed mode needs TTB even (8 warps: 256 / 64 / 16 tuples): a tile is then a whole
// transpose block -- processed when tile <= pair_swap(tile), self-transposed tiles entirely
// inside one CTA, so its loads finish (barrier) before any of its stores.
// ------------------------------------------------------------------------------------
template <int NQ, int WARPS, int NBUF, int UI>
__global__ void __launch_bounds__(WARPS * 32, (NBUF == 2 ? 12 : 16) / WARPS)
    tile_kernel(double2* __restrict__ a, const __grid_constant__ GroupParams p) {
  constexpr int MB = 2 * NQ, TB = 9 - MB, T = 1 << TB;
  constexpr int WB = WARPS == 16 ? 4 : (WARPS == 8 ? 3 : (WARPS == 4 ? 2 : 1));
  constexpr int TTB = TB + WB, TT = 1 << TTB;
  constexpr int HB = 5 + WB, NBITS = HB + 4, ELEMS = WARPS * 512;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // shared: program | NBUF tiles | copy tables (offset [16], transpose offset [16], bits) | subs
  const int prog_cap = (p.prog_elems + 7) & ~7;
  double2* sProg = reinterpret_cast<double2*>(smem_raw);
  double2* sX = sProg + prog_cap;
  uint64_t* sIterOff = reinterpret_cast<uint64_t*>(sX + NBUF * ELEMS);
  int* sIterTM = reinterpret_cast<int*>(sIterOff + 32);
  GroupSub* sSub = reinterpret_cast<GroupSub*>(sIterTM + 32);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if constexpr (TTB & 1) {
    if (p.mirror) __trap();  // the host never launches packed mode with odd TTB
  }

  int freep[TTB];
  {
    int nf = 0;
    for (int f = 0; f < 64 && nf < TTB; ++f) {
      bool tgt = false;
      for (int j = 0; j < MB; ++j) tgt |= (int)p.pos[j] == f;
      if (!tgt) freep[nf++] = f;
    }
  }
  // NBITS tile bits sorted by physical position: threads take the HB lowest, iterations the
  // next 4.
  int thr_tm;
  uint64_t thr_off;
  {
    int bit_pos[NBITS], bit_id[NBITS];  // id < TTB: tuple bit, else member bit id-TTB
    for (int j = 0; j < TTB; ++j) {
      bit_pos[j] = freep[j];
      bit_id[j] = j;
    }
    for (int j = 0; j < MB; ++j) {
      bit_pos[TTB + j] = (int)p.pos[j];
      bit_id[TTB + j] = TTB + j;
    }
    for (int x = 1; x < NBITS; ++x)
      for (int y = x; y > 0 && bit_pos[y] < bit_pos[y - 1]; --y) {
        int tp = bit_pos[y]; bit_pos[y] = bit_pos[y - 1]; bit_pos[y - 1] = tp;
        int ti = bit_id[y]; bit_id[y] = bit_id[y - 1]; bit_id[y - 1] = ti;
      }
    auto tm_of = [&](int bits, int first, int cnt, uint64_t& off) {
      int t = 0, m = 0;
      off = 0;
      for (int b = 0; b < cnt; ++b)
        if ((bits >> b) & 1) {
          const int id = bit_id[first + b];
          if (id < TTB) t |= 1 << id; else m |= 1 << (id - TTB);
          off += (uint64_t)1 << bit_pos[first + b];
        }
      return t | (m << TTB);
    };
    thr_tm = tm_of(threadIdx.x, 0, HB, thr_off);
    if (threadIdx.x < 16) {
      sIterTM[threadIdx.x] = tm_of(threadIdx.x, HB, 4, sIterOff[threadIdx.x]);
      sIterOff[16 + threadIdx.x] = pair_swap(sIterOff[threadIdx.x]);
    }
  }
  const uint64_t thr_poff = pair_swap(thr_off);
  const int hi_tile = max(freep[TTB - 1], (int)p.pos[MB - 1]);  // highest in-tile position
  for (int e = threadIdx.x; e < p.prog_elems; e += blockDim.x) sProg[e] = p.prog[e];
  for (int e = threadIdx.x; e < p.n_sub; e += blockDim.x) sSub[e] = p.sub[e];
  __syncthreads();

  const uint64_t n_tiles = (p.n_tuples + TT - 1) >> TTB;
  auto next_tile = [&](uint64_t tl) {
    if (p.mirror)
      while (tl < n_tiles && tl > tpose(tl, p.tp_lo, p.tp_m, MB + TTB)) tl += gridDim.x;
    return tl;
  };
  // shared index of tile element (tuple t, member m): warp sub-tile t / T, swizzled inside
  auto sidx = [](int tm) {
    const int t = tm & (TT - 1), m = tm >> TTB;
    return ((t >> TB) << 9) + xs_idx<T>(m, t & (T - 1));
  };
  auto issue_load = [&](uint64_t tl, double2* buf) {
    const uint64_t tb0 = insert_zeros(tl << TTB, p.lo_mask, MB);
    const uint64_t base = tb0 + thr_off, pbase = tpose(tb0, p.tp_lo, p.tp_m, 0) + thr_poff;
    const bool packed = p.mirror && !packed_tile_direct(tb0, hi_tile, p.tp_lo, p.tp_m);
    unsigned mask = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int tm = thr_tm | sIterTM[i];
      const bool ok = (tl << TTB) + (tm & (TT - 1)) < p.n_tuples;
      uint64_t src = base + sIterOff[i];
      if (packed) {
        const uint64_t srcm = pbase + sIterOff[16 + i];
        if (!packed_stored(src, srcm)) {
          src = srcm;
          mask |= 1u << i;
        }
      }
      cp_async16(buf + sidx(tm), ok ? a + src : a, ok);
    }
    cp_async_commit();
    return mask;
  };
  auto fixup = [&](double2* buf, unsigned mask) {  // conj of the transposed copies
    for (; mask; mask &= mask - 1) {
      double* im = &buf[sidx(thr_tm | sIterTM[__ffs(mask) - 1])].y;
      *im = -*im;
    }
  };

  // NBUF = 2: the next tile's copies are issued right after the barrier that makes the current
  // tile visible, so they overlap the compute and the stores (2 barriers per tile).
  uint64_t tile = next_tile(blockIdx.x);
  unsigned mask_next = 0;
  if (NBUF == 2 && tile < n_tiles) mask_next = issue_load(tile, sX);
  int cur = 0;
  while (tile < n_tiles) {
    const uint64_t next = next_tile(tile + gridDim.x);
    double2* buf = sX + (NBUF == 2 ? cur * ELEMS : 0);
    unsigned mask = mask_next;
    if constexpr (NBUF == 1) mask = (p.dbg & 2) ? 0u : issue_load(tile, sX);
    cp_async_wait<0>();
    fixup(buf, mask);
    __syncthreads();  // current tile visible; the other buffer's stores are done
    if constexpr (NBUF == 2)
      if (next < n_tiles) mask_next = issue_load(next, sX + (cur ^ 1) * ELEMS);
    double2* X = buf + (warp << 9);
    for (int s = 0; s < (p.dbg & 1 ? 0 : p.n_sub); ++s) {
      const GroupSub& g = sSub[s];
      const double2* F = sProg + g.s_off;
      if (g.k == 2)
        group_sub_k2<T, UI>(X, F, g.mi, g.mu, lane);
      else
        group_sub_k1<T>(X, F, g.mi, g.mu, lane);
      __syncwarp();
    }
    __syncthreads();
    if (!(p.dbg & 2)) {
      const uint64_t tb0 = insert_zeros(tile << TTB, p.lo_mask, MB);
      const uint64_t base = tb0 + thr_off, pbase = tpose(tb0, p.tp_lo, p.tp_m, 0) + thr_poff;
      const bool self = tpose(tile, p.tp_lo, p.tp_m, MB + TTB) == tile;
      const bool packed = p.mirror && !packed_tile_direct(tb0, hi_tile, p.tp_lo, p.tp_m);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int tm = thr_tm | sIterTM[i];
        if ((tile << TTB) + (tm & (TT - 1)) >= p.n_tuples) continue;
        const uint64_t dst = base + sIterOff[i];
        const double2 v = buf[sidx(tm)];
        if (!packed) {
          a[dst] = v;
        } else {
          const uint64_t dstm = pbase + sIterOff[16 + i];
          if (packed_stored(dst, dstm)) a[dst] = v;
          else if (!self) a[dstm] = cj(v);  // self tile: the transpose is stored directly
        }
      }
    }
    if constexpr (NBUF == 1) __syncthreads();  // the buffer is reloaded next
    tile = next;
    cur ^= 1;
  }
}

template <int NQ, int WARPS, int NBUF, int UI>
static cudaError_t launch_tile_cfg(double2* a, const GroupParams& p, cudaStream_t st) {
  static std::atomic<uint64_t> attr_done{0};
  constexpr int TT = WARPS << (9 - 2 * NQ);
  const size_t smem = (size_t)((p.prog_elems + 7) & ~7) * sizeof(double2) +
                      (size_t)NBUF * WARPS * 512 * sizeof(double2) + 32 * 8 + 32 * 4 +
                      (size_t)p.n_sub * sizeof(GroupSub);
  auto kern = tile_kernel<NQ, WARPS, NBUF, UI>;
  cudaError_t ea = ensure_smem_attr(kern, attr_done);
  if (ea != cudaSuccess) return ea;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const uint64_t tiles = (p.n_tuples + TT - 1) / TT;
  const uint64_t cap = (uint64_t)sms * per_sm;
  const unsigned grid = capped((unsigned)(tiles < cap ? tiles : cap));
  kern<<<grid, WARPS * 32, smem, st>>>(a, p);
  return cudaGetLastError();
}

static int g_tile_mode = -1;  // env TANQ_GROUP = auto | warp | q1 | o1 (experiments)

cudaError_t launch_group3(double2* a, const GroupParams& p, cudaStream_t st) {
  if (g_tile_mode < 0) {
    const char* e = getenv("TANQ_GROUP");
    g_tile_mode = !e ? 9 : !strcmp(e, "warp") ? 0 : !strcmp(e, "q1") ? 1 : !strcmp(e, "o1") ? 2 : 9;
  }
  bool has3 = false;
  int n2 = 0;
  uint32_t lo = 64;
  for (int i = 0; i < p.n_sub; ++i) {
    has3 |= p.sub[i].k == 3;
    n2 += p.sub[i].k == 2;
  }
  for (int j = 0; j < 2 * p.nq; ++j) lo = p.pos[j] < lo ? p.pos[j] : lo;
  // dense 64x64 sub-ops are DMMA-bound: per-warp tiles, 2 buffers, 8 independent warps
  if (has3 && p.nq != 3) return cudaErrorInvalidValue;  // the planner never emits this
  if (has3) return launch_group_cfg<3, 8, 2, true, 4>(a, p, st);
  int mode = g_tile_mode;
  if (mode == 9) {
    // auto (measured at n = 16, scripts/kbench.py).  Full layout: cooperative tiles while the
    // group is memory-bound (<= 2 k=2 sub-ops) and its lowest member position is >= 6
    // (per-warp tiles then read 128 B runs, microbench/locality.cu); heavier programs are
    // DMMA-bound and run best on 16 independent warps.  Packed layout (half the traffic):
    // 3-qubit groups are DMMA-bound -> 16 independent warps; 4-qubit groups need the 8-warp
    // tile for contiguous copies (per-warp tiles hold 2 tuples).
    if (p.mirror)
      mode = p.nq == 3 ? 0 : 2;
    else
      mode = (p.nq == 2 || (lo > 5 && n2 <= 2)) ? 1 : 0;
  }
  if (p.nq == 2 && mode == 0) mode = 1;
  if (p.mirror && mode == 1) mode = 2;  // packed mode needs whole transpose blocks per tile
  // packed k=2 tiles: 2-warp CTAs (64 tuples, an even number of tuple bits) -- many small
  // independent CTAs per SM hide the copy latency best (14.6-15.0 vs 16.8-17.3 ms for 8-warp
  // tiles at n = 16)
  if (p.nq == 2 && p.mirror) return launch_tile_cfg<2, 2, 1, 2>(a, p, st);
  switch (mode) {
    case 0:
      if (p.nq == 4) return launch_group_cfg<4, 16, 1, false, 1>(a, p, st);
      return launch_group_cfg<3, 16, 1, false, 2>(a, p, st);
    case 2:
      if (p.nq == 2) return launch_tile_cfg<2, 8, 1, 2>(a, p, st);
      if (p.nq == 4) return launch_tile_cfg<4, 8, 1, 1>(a, p, st);
      return launch_tile_cfg<3, 8, 1, 2>(a, p, st);
    default:
      if (p.nq == 2) return launch_tile_cfg<2, 4, 1, 2>(a, p, st);
      if (p.nq == 4) return launch_tile_cfg<4, 4, 1, 1>(a, p, st);
      return launch_tile_cfg<3, 4, 1, 2>(a, p, st);
  }
}

// Packed -> full layout: every element the packed layout does not keep gets conj(transpose).
__global__ void unpack_kernel(double2* __restrict__ a, uint64_t n, uint64_t lo, uint64_t m) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n; e += stride) {
    const uint64_t em = tpose(e, lo, m, 0);
    if (!packed_stored(e, em)) a[e] = cj(a[em]);
  }
}

cudaError_t launch_unpack(double2* a, int L, TDesc td, cudaStream_t st) {
  const uint64_t n = (uint64_t)1 << L;
  unpack_kernel<<<grid_for(n, kThreads, 148ull * 16), kThreads, 0, st>>>(a, n, td.lo, td.m);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// state init, remap
// ------------------------------------------------------------------------------------
__global__ void set_one_kernel(double2* a) { a[0] = make_double2(1.0, 0.0); }

cudaError_t launch_init(double2* a, uint64_t elems, bool one_at_zero, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(a, 0, elems * sizeof(double2), st);
  if (e != cudaSuccess) return e;
  if (one_at_zero) set_one_kernel<<<1, 1, 0, st>>>(a);
  return cudaGetLastError();
}

__global__ void swap_halves_kernel(double2* __restrict__ A, double2* __restrict__ B, uint64_t half,
                                   int b, int va, int vb) {
  const uint64_t lowmask = ((uint64_t)1 << b) - 1;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < half; e += stride) {
    uint64_t hi = (e >> b) << (b + 1), lo = e & lowmask;
    uint64_t oa = hi | ((uint64_t)va << b) | lo;
    uint64_t ob = hi | ((uint64_t)vb << b) | lo;
    double2 x = A[oa], y = B[ob];
    A[oa] = y;
    B[ob] = x;
  }
}

cudaError_t launch_swap_halves(double2* A, double2* B, int L, int b, int va, int vb,
                               cudaStream_t st) {
  uint64_t half = (uint64_t)1 << (L - 1);
  swap_halves_kernel<<<grid_for(half, kThreads, 148ull * 32), kThreads, 0, st>>>(A, B, half, b, va,
                                                                               vb);
  return cudaGetLastError();
}

// ---- parity-layout remap (tanq_internal.h) ----
struct Oct {
  uint64_t lo0, lo1, lo2;  // (1 << p) - 1 of the sorted positions of x, y, z
  uint64_t bx, by, bz;
  __device__ uint64_t base(uint64_t o) const {
    o = ((o & ~lo0) << 1) | (o & lo0);
    o = ((o & ~lo1) << 1) | (o & lo1);
    return ((o & ~lo2) << 1) | (o & lo2);
  }
  __device__ uint64_t off(int i) const {  // i: bit 0 = x, bit 1 = y, bit 2 = z
    return ((i & 1) ? bx : 0) | ((i & 2) ? by : 0) | ((i & 4) ? bz : 0);
  }
};
static Oct make_oct(int x, int y, int z) {
  int p[3] = {x, y, z};
  std::sort(p, p + 3);
  Oct o;
  o.lo0 = ((uint64_t)1 << p[0]) - 1;
  o.lo1 = ((uint64_t)1 << p[1]) - 1;
  o.lo2 = ((uint64_t)1 << p[2]) - 1;
  o.bx = (uint64_t)1 << x;
  o.by = (uint64_t)1 << y;
  o.bz = (uint64_t)1 << z;
  return o;
}
// destination octet slot of slot i (ex, ey, ez) from a shard with parity bit s
__device__ __forceinline__ int par_dst(int i, int s) {
  const int ex = i & 1, ey = (i >> 1) & 1;
  return ey | (ex << 1) | ((ex ^ s) << 2);
}
__device__ __forceinline__ int par_leaves(int i, int s) { return (((i >> 1) ^ (i >> 2)) & 1) != s; }

__global__ void parity_swap_kernel(double2* __restrict__ A, double2* __restrict__ B, uint64_t noct,
                                   Oct oc) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t o = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; o < noct; o += stride) {
    const uint64_t b = oc.base(o);
    double2 va[8], vb[8], oa[8], ob[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      va[i] = A[b + oc.off(i)];
      vb[i] = B[b + oc.off(i)];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {  // A has parity bit 0, B 1; an element lands on shard ey ^ ez
      if (par_leaves(i, 0)) ob[par_dst(i, 0)] = va[i]; else oa[par_dst(i, 0)] = va[i];
      if (par_leaves(i, 1)) oa[par_dst(i, 1)] = vb[i]; else ob[par_dst(i, 1)] = vb[i];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i != 0 && i != 7) A[b + oc.off(i)] = oa[i];  // slots 000 / 111 of A keep their element
      if (i != 4 && i != 3) B[b + oc.off(i)] = ob[i];  // (ex, ey, ez) = 001 / 110 of B too
    }
  }
}

cudaError_t launch_parity_swap(double2* A, double2* B, int L, int x, int y, int z,
                               cudaStream_t st) {
  const uint64_t noct = (uint64_t)1 << (L - 3);
  parity_swap_kernel<<<grid_for(noct, kThreads, 148ull * 16), kThreads, 0, st>>>(A, B, noct,
                                                                                make_oct(x, y, z));
  return cudaGetLastError();
}

__global__ void parity_stay_kernel(double2* __restrict__ a, uint64_t noct, Oct oc, int s) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t o = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; o < noct; o += stride) {
    const uint64_t b = oc.base(o);
    double2 v[8], w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (!par_leaves(i, s) && par_dst(i, s) != i) v[i] = a[b + oc.off(i)];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (!par_leaves(i, s) && par_dst(i, s) != i) w[par_dst(i, s)] = v[i];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (!par_leaves(i, s) && par_dst(i, s) != i) a[b + oc.off(par_dst(i, s))] = w[par_dst(i, s)];
  }
}

// leaving slot j (0..3) of a shard with parity bit s: ex = j >> 1, ey = j & 1, ez = ey ^ 1 ^ s
__device__ __forceinline__ int par_slot(int j, int s) {
  const int ex = j >> 1, ey = j & 1;
  return ex | (ey << 1) | ((ey ^ 1 ^ s) << 2);
}

__global__ void parity_pack_kernel(const double2* __restrict__ a, double2* __restrict__ buf,
                                   Oct oc, int s, uint64_t first, uint64_t count, int dir) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += stride) {
    const uint64_t e = first + i;
    const uint64_t b = oc.base(e >> 2);
    const int j = (int)(e & 3);
    if (dir == 0) {
      buf[i] = a[b + oc.off(par_slot(j, s))];
    } else {  // received slot j of the partner (parity bit s ^ 1)
      const_cast<double2*>(a)[b + oc.off(par_dst(par_slot(j, s ^ 1), s ^ 1))] = buf[i];
    }
  }
}

cudaError_t launch_parity_stay(double2* a, int L, int x, int y, int z, int s, cudaStream_t st) {
  const uint64_t noct = (uint64_t)1 << (L - 3);
  parity_stay_kernel<<<grid_for(noct, kThreads, 148ull * 16), kThreads, 0, st>>>(
      a, noct, make_oct(x, y, z), s);
  return cudaGetLastError();
}
cudaError_t launch_parity_pack(const double2* a, double2* buf, int L, int x, int y, int z, int s,
                               uint64_t first, uint64_t count, cudaStream_t st) {
  (void)L;
  parity_pack_kernel<<<grid_for(count, kThreads, 148ull * 32), kThreads, 0, st>>>(
      a, buf, make_oct(x, y, z), s, first, count, 0);
  return cudaGetLastError();
}
cudaError_t launch_parity_unpack(double2* a, const double2* buf, int L, int x, int y, int z,
                                 int s, uint64_t first, uint64_t count, cudaStream_t st) {
  (void)L;
  parity_pack_kernel<<<grid_for(count, kThreads, 148ull * 32), kThreads, 0, st>>>(
      a, const_cast<double2*>(buf), make_oct(x, y, z), s, first, count, 1);
  return cudaGetLastError();
}

__global__ void pack_kernel(const double2* __restrict__ a, double2* __restrict__ buf, int b, int v,
                            uint64_t first, uint64_t count, int dir) {
  const uint64_t lowmask = ((uint64_t)1 << b) - 1;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += stride) {
    uint64_t e = first + i;
    uint64_t o = ((e >> b) << (b + 1)) | ((uint64_t)v << b) | (e & lowmask);
    if (dir == 0)
      buf[i] = a[o];
    else
      const_cast<double2*>(a)[o] = buf[i];
  }
}

cudaError_t launch_pack_half(const double2* a, double2* buf, int b, int v, uint64_t first,
                             uint64_t count, cudaStream_t st) {
  pack_kernel<<<grid_for(count, kThreads, 148ull * 32), kThreads, 0, st>>>(a, buf, b, v, first,
                                                                          count, 0);
  return cudaGetLastError();
}
cudaError_t launch_unpack_half(double2* a, const double2* buf, int b, int v, uint64_t first,
                               uint64_t count, cudaStream_t st) {
  pack_kernel<<<grid_for(count, kThreads, 148ull * 32), kThreads, 0, st>>>(
      a, const_cast<double2*>(buf), b, v, first, count, 1);
  return cudaGetLastError();
}

// Quarter {o : bit_b0(o) == v0, bit_b1(o) == v1} (b0 < b1) of a shard to / from a contiguous
// buffer, elements [first, first + count) of the quarter in run order (batched 2-bit remap).
__global__ void pack_quarter_kernel(double2* __restrict__ a, double2* __restrict__ buf, int b0,
                                    int v0, int b1, int v1, uint64_t first, uint64_t count,
                                    int dir) {
  const uint64_t m0 = ((uint64_t)1 << b0) - 1, m1 = ((uint64_t)1 << b1) - 1;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += stride) {
    uint64_t o = first + i;
    o = ((o & ~m0) << 1) | ((uint64_t)v0 << b0) | (o & m0);
    o = ((o & ~m1) << 1) | ((uint64_t)v1 << b1) | (o & m1);
    if (dir == 0)
      buf[i] = a[o];
    else
      a[o] = buf[i];
  }
}

cudaError_t launch_pack_quarter(const double2* a, double2* buf, int b0, int v0, int b1, int v1,
                                uint64_t first, uint64_t count, cudaStream_t st) {
  pack_quarter_kernel<<<grid_for(count, kThreads, 148ull * 32), kThreads, 0, st>>>(
      const_cast<double2*>(a), buf, b0, v0, b1, v1, first, count, 0);
  return cudaGetLastError();
}
cudaError_t launch_unpack_quarter(double2* a, const double2* buf, int b0, int v0, int b1, int v1,
                                  uint64_t first, uint64_t count, cudaStream_t st) {
  pack_quarter_kernel<<<grid_for(count, kThreads, 148ull * 32), kThreads, 0, st>>>(
      a, const_cast<double2*>(buf), b0, v0, b1, v1, first, count, 1);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// vec(rho) order <-> physical order
// ------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t vec_to_phys(uint64_t v, const BitMap& bm, int n) {
  // v = r + c 2^n; logical bit 2q = r_q, 2q+1 = c_q
  uint64_t P = 0;
  for (int q = 0; q < n; ++q) {
    P |= ((v >> q) & 1ull) << bm.phys[2 * q];
    P |= ((v >> (n + q)) & 1ull) << bm.phys[2 * q + 1];
  }
  for (uint64_t h = bm.par; h; h &= h - 1) {  // parity layout: the col slot holds r XOR c
    const int q = __ffsll((long long)h) - 1;
    P ^= ((v >> q) & 1ull) << bm.phys[2 * q + 1];
  }
  return P;
}

__global__ void gather_vec_kernel(const double2* __restrict__ a, double2* __restrict__ out,
                                  const __grid_constant__ BitMap bm, int n, int L, uint64_t shard,
                                  uint64_t first, uint64_t count, int zero_unowned) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t lmask = ((uint64_t)1 << L) - 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += stride) {
    uint64_t P = vec_to_phys(first + i, bm, n);
    if ((P >> L) == shard)
      out[i] = a[P & lmask];
    else if (zero_unowned)
      out[i] = make_double2(0.0, 0.0);
  }
}

__global__ void scatter_vec_kernel(double2* __restrict__ a, const double2* __restrict__ in,
                                   const __grid_constant__ BitMap bm, int n, int L, uint64_t shard,
                                   uint64_t first, uint64_t count) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t lmask = ((uint64_t)1 << L) - 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += stride) {
    uint64_t P = vec_to_phys(first + i, bm, n);
    if ((P >> L) == shard) a[P & lmask] = in[i];
  }
}

cudaError_t launch_gather_vec(const double2* a, double2* out, const BitMap& bm, int n, int L,
                              uint64_t shard, uint64_t first, uint64_t count, bool zero_unowned,
                              cudaStream_t st) {
  gather_vec_kernel<<<grid_for(count, kThreads, 148ull * 32), kThreads, 0, st>>>(
      a, out, bm, n, L, shard, first, count, zero_unowned ? 1 : 0);
  return cudaGetLastError();
}
cudaError_t launch_scatter_vec(double2* a, const double2* in, const BitMap& bm, int n, int L,
                               uint64_t shard, uint64_t first, uint64_t count, cudaStream_t st) {
  scatter_vec_kernel<<<grid_for(count, kThreads, 148ull * 32), kThreads, 0, st>>>(
      a, in, bm, n, L, shard, first, count);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// diagonal reductions (A-7)
// ------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t diag_phys(uint64_t x, const BitMap& bm, int n) {
  uint64_t P = 0;
  for (int q = 0; q < n; ++q) {
    uint64_t b = (x >> q) & 1ull;
    P |= b << bm.phys[2 * q];
    if (!((bm.par >> q) & 1ull)) P |= b << bm.phys[2 * q + 1];  // parity r XOR c = 0
  }
  return P;
}

__global__ void diag_kernel(const double2* __restrict__ a, double* __restrict__ probs,
                            unsigned long long* imax, const __grid_constant__ BitMap bm, int n,
                            int L, uint64_t shard) {
  const uint64_t N = (uint64_t)1 << n;
  const uint64_t lmask = ((uint64_t)1 << L) - 1;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  double mi = 0.0;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < N; x += stride) {
    uint64_t P = diag_phys(x, bm, n);
    if ((P >> L) != shard) continue;
    double2 v = a[P & lmask];
    probs[x] = v.x;
    mi = fmax(mi, fabs(v.y));
  }
  if (mi > 0.0) atomicMax(imax, (unsigned long long)__double_as_longlong(mi));
}

cudaError_t launch_diag(const double2* a, double* probs, unsigned long long* imax,
                        const BitMap& bm, int n, int L, uint64_t shard, cudaStream_t st) {
  uint64_t N = (uint64_t)1 << n;
  diag_kernel<<<grid_for(N, kThreads, 148ull * 8), kThreads, 0, st>>>(a, probs, imax, bm, n, L,
                                                                     shard);
  return cudaGetLastError();
}

__global__ void readout_kernel(double* p, uint64_t half, int q, double p10, double p01) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t lo = ((uint64_t)1 << q) - 1;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < half; e += stride) {
    uint64_t x0 = ((e & ~lo) << 1) | (e & lo), x1 = x0 | ((uint64_t)1 << q);
    double a0 = p[x0], a1 = p[x1];
    p[x0] = (1.0 - p10) * a0 + p01 * a1;
    p[x1] = p10 * a0 + (1.0 - p01) * a1;
  }
}

cudaError_t launch_readout(double* p, int n, const double* p10, const double* p01,
                           cudaStream_t st) {
  uint64_t half = (uint64_t)1 << (n - 1);
  for (int q = 0; q < n; ++q) {
    double a = p10 ? p10[q] : 0.0, b = p01 ? p01[q] : 0.0;
    if (a == 0.0 && b == 0.0) continue;
    readout_kernel<<<grid_for(half, kThreads, 148ull * 8), kThreads, 0, st>>>(p, half, q, a, b);
  }
  return cudaGetLastError();
}

int expect_blocks(int n) {
  uint64_t N = (uint64_t)1 << n;
  uint64_t b = (N + kThreads * 8 - 1) / (kThreads * 8);
  if (b > 148 * 4) b = 148 * 4;
  if (b < 1) b = 1;
  return (int)b;
}

__device__ __forceinline__ double2 block_sum2(double2 v) {
  __shared__ double2 red[kThreads / 32];
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  double2 s = make_double2(0.0, 0.0);
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      s.x += red[i].x;
      s.y += red[i].y;
    }
  return s;
}

// tr(P rho) = (-i)^{popc(x&z)} sum_a (-1)^{popc(a&z)} rho[a^x][a]   (A-7)
__global__ void expect_kernel(const double2* __restrict__ a, double2* partial,
                              const __grid_constant__ BitMap bm, int n, int L, uint64_t shard,
                              uint64_t xm, uint64_t zm) {
  const uint64_t N = (uint64_t)1 << n;
  const uint64_t lmask = ((uint64_t)1 << L) - 1;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  double2 acc = make_double2(0.0, 0.0);
  for (uint64_t col = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; col < N; col += stride) {
    uint64_t row = col ^ xm;
    uint64_t P = 0;
    for (int q = 0; q < n; ++q) {
      P |= ((row >> q) & 1ull) << bm.phys[2 * q];
      P |= ((col >> q) & 1ull) << bm.phys[2 * q + 1];
    }
    for (uint64_t h = bm.par; h; h &= h - 1) {
      const int q = __ffsll((long long)h) - 1;
      P ^= ((row >> q) & 1ull) << bm.phys[2 * q + 1];
    }
    if ((P >> L) != shard) continue;
    double2 v = a[P & lmask];
    double sgn = (__popcll(col & zm) & 1) ? -1.0 : 1.0;
    acc.x += sgn * v.x;
    acc.y += sgn * v.y;
  }
  double2 s = block_sum2(acc);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

cudaError_t launch_expect(const double2* a, double2* partial, int nblocks, const BitMap& bm,
                          int n, int L, uint64_t shard, uint64_t xm, uint64_t zm,
                          cudaStream_t st) {
  expect_kernel<<<nblocks, kThreads, 0, st>>>(a, partial, bm, n, L, shard, xm, zm);
  return cudaGetLastError();
}

__global__ void reduce_partials_kernel(const double2* partial, int nb, double2* out) {
  double2 acc = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    acc.x += partial[i].x;
    acc.y += partial[i].y;
  }
  double2 s = block_sum2(acc);
  if (threadIdx.x == 0) *out = s;
}

cudaError_t launch_reduce_partials(const double2* partial, int nblocks, double2* out,
                                   cudaStream_t st) {
  reduce_partials_kernel<<<1, kThreads, 0, st>>>(partial, nblocks, out);
  return cudaGetLastError();
}

__global__ void add_kernel(double* dst, const double* src, uint64_t count) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += stride)
    dst[i] += src[i];
}
__global__ void herm_check_kernel(const double2* __restrict__ a, uint64_t N, uint64_t tlo,
                                  uint64_t tm, unsigned long long* res) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  double d = 0.0, m = 0.0;
  for (uint64_t P = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; P < N; P += stride) {
    const double2 x = a[P], y = a[tpose(P, tlo, tm, 0)];
    d = fmax(d, fmax(fabs(x.x - y.x), fabs(x.y + y.y)));
    m = fmax(m, fmax(fabs(x.x), fabs(x.y)));
  }
  for (int o = 16; o > 0; o >>= 1) {
    d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(res, (unsigned long long)__double_as_longlong(d));
    atomicMax(res + 1, (unsigned long long)__double_as_longlong(m));
  }
}

cudaError_t launch_herm_check(const double2* a, int L, TDesc td, unsigned long long* res,
                              cudaStream_t st) {
  const uint64_t N = (uint64_t)1 << L;
  herm_check_kernel<<<grid_for(N, kThreads, 148ull * 8), kThreads, 0, st>>>(a, N, td.lo, td.m,
                                                                           res);
  return cudaGetLastError();
}

cudaError_t launch_add(double* dst, const double* src, uint64_t count, cudaStream_t st) {
  add_kernel<<<grid_for(count, kThreads, 148ull * 8), kThreads, 0, st>>>(dst, src, count);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// sampling: clamp + scan (one CTA), Philox4x32-10 + binary search
// ------------------------------------------------------------------------------------
__global__ void cdf_kernel(const double* __restrict__ p, double* __restrict__ cdf, uint64_t N) {
  __shared__ double part[1024];
  const uint64_t per = (N + blockDim.x - 1) / blockDim.x;
  const uint64_t b0 = threadIdx.x * per, b1 = min(N, b0 + per);
  double s = 0.0;
  for (uint64_t i = b0; i < b1; ++i) s += fmax(p[i], 0.0);
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double run = 0.0;
    for (unsigned i = 0; i < blockDim.x; ++i) {
      double v = part[i];
      part[i] = run;
      run += v;
    }
  }
  __syncthreads();
  double run = part[threadIdx.x];
  for (uint64_t i = b0; i < b1; ++i) {
    run += fmax(p[i], 0.0);
    cdf[i] = run;
  }
}

cudaError_t launch_cdf(const double* p, double* cdf, int n, cudaStream_t st) {
  cdf_kernel<<<1, 1024, 0, st>>>(p, cdf, (uint64_t)1 << n);
  return cudaGetLastError();
}

__device__ __forceinline__ void philox_round(uint32_t c[4], const uint32_t k[2]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
  uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
  uint32_t n0 = hi1 ^ c[1] ^ k[0], n1 = lo1, n2 = hi0 ^ c[3] ^ k[1], n3 = lo0;
  c[0] = n0;
  c[1] = n1;
  c[2] = n2;
  c[3] = n3;
}

__device__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  uint32_t k[2] = {k0, k1};
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    philox_round(c, k);
    k[0] += 0x9E3779B9u;
    k[1] += 0xBB67AE85u;
  }
}

__global__ void sample_kernel(const double* __restrict__ cdf, uint64_t N, uint64_t seed,
                              uint64_t shots, unsigned long long* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const double total = cdf[N - 1];
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < shots; s += stride) {
    uint32_t c[4] = {(uint32_t)s, (uint32_t)(s >> 32), 0u, 0u};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    uint64_t bits = ((uint64_t)c[0] << 21) ^ ((uint64_t)c[1] >> 11);  // 53 random bits
    double u = (double)(bits & ((1ull << 53) - 1)) * (1.0 / 9007199254740992.0);
    double target = u * total;
    uint64_t lo = 0, hi = N - 1;  // first index with cdf > target
    while (lo < hi) {
      uint64_t mid = (lo + hi) >> 1;
      if (cdf[mid] > target)
        hi = mid;
      else
        lo = mid + 1;
    }
    out[s] = lo;
  }
}

cudaError_t launch_sample(const double* cdf, int n, uint64_t seed, uint64_t shots,
                          unsigned long long* out, cudaStream_t st) {
  sample_kernel<<<grid_for(shots, kThreads, 148ull * 8), kThreads, 0, st>>>(
      cdf, (uint64_t)1 << n, seed, shots, out);
  return cudaGetLastError();
}

}  // namespace tanq
