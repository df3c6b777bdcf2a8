// K3 "block pipeline" kernel (round 2): a fused group of k <= 2 sub-ops on 2 or
// 3 qubits applied to the state in one HBM round trip, with the HBM traffic moved by the
// asynchronous bulk-copy engine so that it overlaps the FP64 tensor work.
//
// Data unit: a block = 5 whole qubits -- the group's qubits plus the lowest free qubits --
// i.e. 10 physical index bits, 1024 amplitudes, 16 KB.  Its lowest 4 bits are always physical
// bits 0..3 (qubits 0 and 1 are in every block), so a block is 64 contiguous 256 B pieces.
// Each pair of warps owns two block stages in shared memory:
//
//   load     every pair thread issues one cp.async.bulk (global -> shared) of its piece,
//            signalling the stage's mbarrier (arrive.expect_tx 256 B each, 64 arrivals);
//   wait     both warps wait on the mbarrier (phase parity);
//   fixup    packed layout only: pieces read from the transposed position are permuted
//            (swap of each qubit's row/col bit inside the piece) and conjugated in place;
//            self-transposed blocks are symmetrised (non-canonical <- conj(canonical));
//   compute  each warp applies the group's sub-ops to its half of the block (8 tuples x 64
//            members for 3-qubit groups): k=2 sub-ops on the FP64 tensor pipe
//            (mma.sync.m8n8k4.f64 -> DMMA.8x8x4), k=1 sub-ops as DFMA streams;
//   store    unfixup, fence.proxy.async, one cp.async.bulk (shared -> global) per piece back
//            to where the piece came from; the stage is refilled with the pair's next block
//            after cp.async.bulk.wait_group.read -- one iteration later, so the copy of block
//            i+1 runs during the compute of block i and the stores drain behind it.
//
// Pieces are placed in shared memory at 16 * rank + G(piece) units (16 B), G a per-launch
// linear bank rotation chosen by the host so that the DMMA B-fragment loads and D-fragment
// stores of every sub-op are (near) bank-conflict free; every lane's shared-memory offsets
// come from per-sub-op tables built by the host (tanq_host.cpp: build_block).
//
// Complex arithmetic, per k=2 sub-op (S = a + ib, x = c + id), three real products with no
// epilogue additions:  k1 = a(c+d);  Re y = k1 - (a+b) d;  Im y = k1 + (b-a) c, where the
// second and third products accumulate onto k1 (DMMA with C = k1).  a, -(a+b) and (b-a) are
// precomputed fragments, so the only FP64 adds left are the c+d of each B element.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <atomic>

#include "tanq_internal.h"

namespace tanq {

namespace {

__device__ __forceinline__ uint64_t pair_swap64(uint64_t x) {
  return ((x & 0x5555555555555555ull) << 1) | ((x >> 1) & 0x5555555555555555ull);
}
// transpose of an index with r low bits removed under the shard's descriptor (TDesc)
__device__ __forceinline__ uint64_t tpose64(uint64_t x, uint64_t lo, uint64_t m, int r) {
  const uint64_t l = lo >> r;
  return pair_swap64(x & l) | ((x & ~l) ^ (m >> r));
}
// MODE bit 1: the shard's transpose descriptor (several shards, parity layout); without it
// the single-shard pair_swap (the same map for tp_lo = ~0, tp_m = 0).
template <int MODE>
__device__ __forceinline__ uint64_t tpb(uint64_t x, const BlockParams& p, int r) {
  if constexpr ((MODE & 2) != 0) return tpose64(x, p.tp_lo, p.tp_m, r);
  else return pair_swap64(x);
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async16_cg(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
// arrive on the mbarrier once all of this thread's prior cp.async copies have landed
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, const int* c,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]),
      "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_5d(const CUtensorMap* map, const int* c, const void* src) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(src))
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void pair_bar(int pair) {
  asm volatile("bar.sync %0, 64;" ::"r"(1 + pair) : "memory");
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
// D = A B + C with C and D distinct
__device__ __forceinline__ void dmma_c(double& d0, double& d1, double a, double b, double c0,
                                       double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}
__device__ __forceinline__ uint64_t insert_zeros10(uint64_t t, const uint64_t* lo) {
#pragma unroll
  for (int j = 0; j < 10; ++j) t = ((t & ~lo[j]) << 1) | (t & lo[j]);
  return t;
}

// 16-element piece, in-piece index t = (r0 c0 r1 c1): transpose swaps each row/col bit pair.
__device__ __forceinline__ int pswap4(int t) { return ((t & 5) << 1) | ((t >> 1) & 5); }

// In-place (permute + conjugate) of one piece: X[pswap4(t)] <- conj(X[t]).  Involution.  Lane
// j of a quarter warp visits t = i ^ rot(j), rot = {0,1,2,3,12,13,14,15}[j]: both t and
// pswap4(t) = pswap4(i) ^ pswap4(rot) then cover all 8 banks, so loads and stores are
// conflict-free (for pieces with the same bank rotation).
__device__ __forceinline__ int piece_rot(int j) { return (j & 4) ? 8 + j : j & 3; }
__device__ __forceinline__ void piece_transpose(double2* P, int rot) {
  double2 v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = P[i ^ rot];
#pragma unroll
  for (int i = 0; i < 16; ++i) P[pswap4(i ^ rot)] = make_double2(v[i].x, -v[i].y);
}

// k = 2 sub-op on one warp's half block.  F: fragments [3][4 ks][32 lanes][2 mt] doubles
// (a, -(a+b), b-a); T: this lane's 32 offsets (16 B-fragment [ks][j], 16 D-fragment [mt][j][c]).
template <int UI, int ACC>
__device__ __forceinline__ void blk_sub_k2(double2* X, const double* F, const uint16_t* T,
                                           int lane, int trow, int rows) {
  double a1[2][4], a2[2][4], a3[2][4];
  const double2* F2 = reinterpret_cast<const double2*>(F);  // [mat][ks][lane] = (mt 0, mt 1)
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const double2 v1 = F2[(0 * 4 + ks) * 32 + lane], v2 = F2[(1 * 4 + ks) * 32 + lane],
                  v3 = F2[(2 * 4 + ks) * 32 + lane];
    a1[0][ks] = v1.x; a1[1][ks] = v1.y;
    a2[0][ks] = v2.x; a2[1][ks] = v2.y;
    a3[0][ks] = v3.x; a3[1][ks] = v3.y;
  }
  uint32_t ob[8], od[8];  // packed uint16 pairs
  {  // table [4 chunks][rows][8 uint16]: a quarter warp reads 8 consecutive 16 B chunks
    const uint4* t4 = reinterpret_cast<const uint4*>(T);
    const uint4 b0 = t4[trow], b1 = t4[rows + trow], d0 = t4[2 * rows + trow],
                d1 = t4[3 * rows + trow];
    ob[0] = b0.x; ob[1] = b0.y; ob[2] = b0.z; ob[3] = b0.w;
    ob[4] = b1.x; ob[5] = b1.y; ob[6] = b1.z; ob[7] = b1.w;
    od[0] = d0.x; od[1] = d0.y; od[2] = d0.z; od[3] = d0.w;
    od[4] = d1.x; od[5] = d1.y; od[6] = d1.z; od[7] = d1.w;
  }
  auto boff = [&](int ks, int j) {
    const int e = ks * 4 + j;
    return (int)((ob[e >> 1] >> ((e & 1) * 16)) & 0xffffu);
  };
  auto doff = [&](int mt, int j, int c) {
    const int e = (mt * 4 + j) * 2 + c;
    return (int)((od[e >> 1] >> ((e & 1) * 16)) & 0xffffu);
  };
  if constexpr (ACC == 2) {
    // all four n-tiles at once in two phases: k1 for 8 independent (n-tile, m-tile) chains,
    // then the Re/Im chains seeded from k1 (16 chains), re-reading the B fragments from
    // shared memory instead of keeping 32 of them in registers
    double k1[4][2][2];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) k1[u][mt][0] = k1[u][mt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 xb = X[boff(ks, u)];
        const double sx = xb.x + xb.y;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) dmma(k1[u][mt][0], k1[u][mt][1], a1[mt][ks], sx);
      }
    double yr[4][2][2], yi[4][2][2];
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 xb = X[boff(ks, u)];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          if (ks == 0) {
            dmma_c(yr[u][mt][0], yr[u][mt][1], a2[mt][0], xb.y, k1[u][mt][0], k1[u][mt][1]);
            dmma_c(yi[u][mt][0], yi[u][mt][1], a3[mt][0], xb.x, k1[u][mt][0], k1[u][mt][1]);
          } else {
            dmma(yr[u][mt][0], yr[u][mt][1], a2[mt][ks], xb.y);
            dmma(yi[u][mt][0], yi[u][mt][1], a3[mt][ks], xb.x);
          }
        }
      }
    __syncwarp();  // every lane's B loads precede any lane's D stores
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int c = 0; c < 2; ++c)
          X[doff(mt, u, c)] = make_double2(yr[u][mt][c], yi[u][mt][c]);
    return;
  }
#pragma unroll
  for (int n0 = 0; n0 < 4; n0 += UI) {
    double2 xb[UI][4];
#pragma unroll
    for (int u = 0; u < UI; ++u)
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) xb[u][ks] = X[boff(ks, n0 + u)];
    double k1[UI][2][2];
#pragma unroll
    for (int u = 0; u < UI; ++u)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) k1[u][mt][0] = k1[u][mt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
#pragma unroll
      for (int u = 0; u < UI; ++u) {
        const double sx = xb[u][ks].x + xb[u][ks].y;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) dmma(k1[u][mt][0], k1[u][mt][1], a1[mt][ks], sx);
      }
    double yr[UI][2][2], yi[UI][2][2];
    if constexpr (ACC == 0) {  // seeded: Re/Im chains start from k1 (no epilogue adds)
#pragma unroll
      for (int u = 0; u < UI; ++u)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          dmma_c(yr[u][mt][0], yr[u][mt][1], a2[mt][0], xb[u][0].y, k1[u][mt][0], k1[u][mt][1]);
          dmma_c(yi[u][mt][0], yi[u][mt][1], a3[mt][0], xb[u][0].x, k1[u][mt][0], k1[u][mt][1]);
        }
#pragma unroll
      for (int ks = 1; ks < 4; ++ks)
#pragma unroll
        for (int u = 0; u < UI; ++u)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            dmma(yr[u][mt][0], yr[u][mt][1], a2[mt][ks], xb[u][ks].y);
            dmma(yi[u][mt][0], yi[u][mt][1], a3[mt][ks], xb[u][ks].x);
          }
    } else {  // three independent chains (critical path 4 DMMA), 2 DADD per output
#pragma unroll
      for (int u = 0; u < UI; ++u)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) yr[u][mt][0] = yr[u][mt][1] = yi[u][mt][0] = yi[u][mt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
#pragma unroll
        for (int u = 0; u < UI; ++u)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            dmma(yr[u][mt][0], yr[u][mt][1], a2[mt][ks], xb[u][ks].y);
            dmma(yi[u][mt][0], yi[u][mt][1], a3[mt][ks], xb[u][ks].x);
          }
#pragma unroll
      for (int u = 0; u < UI; ++u)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            yr[u][mt][c] += k1[u][mt][c];
            yi[u][mt][c] += k1[u][mt][c];
          }
    }
    __syncwarp();  // every lane's B loads of this pass precede any lane's D stores
#pragma unroll
    for (int u = 0; u < UI; ++u)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int c = 0; c < 2; ++c)
          X[doff(mt, n0 + u, c)] = make_double2(yr[u][mt][c], yi[u][mt][c]);
  }
}

// Sparse k = 2 sub-op (DFMA, one 16-member tuple per lane): the noisy superoperators of
// Pauli-frame gates (CX, CP, RZ, X with depolarizing / thermal noise) keep 36-40 of their 256
// entries, where the dense DMMA form spends 768 multiply-adds per tuple.  F: the nonzeros
// (double2, row by row) then the uint16 row starts [17]; T[e * rows + trow]: this lane's
// shared-memory slot of entry e's input member, T[(nnz + i) * rows + trow]: of output member i.
// Each lane reads and writes only its own tuple, so no lane waits for another.
__device__ __forceinline__ void blk_sub_k2s(double2* X, const double* F, const uint16_t* T,
                                            int trow, int rows, int nnz) {
  const double2* sv = reinterpret_cast<const double2*>(F);
  const uint16_t* rs = reinterpret_cast<const uint16_t*>(sv + nnz);
  double2 y[16];
  int e = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    double yr = 0.0, yi = 0.0;
    const int end = rs[i + 1];
    for (; e < end; ++e) {
      const double2 sc = sv[e];
      const double2 x = X[T[e * rows + trow]];
      yr = fma(sc.x, x.x, yr);
      yr = fma(-sc.y, x.y, yr);
      yi = fma(sc.x, x.y, yi);
      yi = fma(sc.y, x.x, yi);
    }
    y[i] = make_double2(yr, yi);
  }
  const uint16_t* To = T + nnz * rows + trow;
#pragma unroll
  for (int i = 0; i < 16; ++i) X[To[i * rows]] = y[i];
}

// Real-basis transform (BlockParams::rb_nq): per group qubit, every (x1, x2) = (row 1 col 0,
// row 0 col 1) element pair of the block -> (x1 + x2, i (x2 - x1)) (forward) or back,
// x1 = (u1 + i u2) / 2, x2 = (u1 - i u2) / 2.  Each pair thread owns 4 pairs per qubit
// (table T: [nq][64][4][2] slots); the pair meets at a barrier before every qubit's pass
// (and, forward, after the last) because the pairs of one qubit span both warp halves.
__device__ __forceinline__ void blk_rbasis(double2* X, const uint16_t* T, int nq, int pt, int pair,
                                           bool fwd) {
  for (int t = 0; t < nq; ++t) {
    pair_bar(pair);
    const uint4 e = reinterpret_cast<const uint4*>(T)[t * 64 + pt];
    const uint32_t w[4] = {e.x, e.y, e.z, e.w};
    double2 u[4], v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      u[j] = X[w[j] & 0xffffu];
      v[j] = X[w[j] >> 16];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double2 a = u[j], b = v[j];
      if (fwd) {
        X[w[j] & 0xffffu] = make_double2(a.x + b.x, a.y + b.y);
        X[w[j] >> 16] = make_double2(a.y - b.y, b.x - a.x);
      } else {
        X[w[j] & 0xffffu] = make_double2(0.5 * (a.x - b.y), 0.5 * (a.y + b.x));
        X[w[j] >> 16] = make_double2(0.5 * (a.x + b.y), 0.5 * (a.y - b.x));
      }
    }
  }
  if (fwd && nq) pair_bar(pair);
}

// k = 2 sub-op in the real basis: Y = R X with R real, i.e. two real products per n-tile
// (Re y = R Re x, Im y = R Im x) -- 2/3 of the DMMAs of the complex form and no B-side adds.
// F: [4 ks][32 lanes][2 mt] doubles; T: the same offset tables as blk_sub_k2.
__device__ __forceinline__ void blk_sub_k2r(double2* X, const double* F, const uint16_t* T,
                                            int lane, int trow, int rows) {
  double ar[2][4];
  const double2* F2 = reinterpret_cast<const double2*>(F);
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const double2 v = F2[ks * 32 + lane];
    ar[0][ks] = v.x;
    ar[1][ks] = v.y;
  }
  uint32_t ob[8], od[8];
  {
    const uint4* t4 = reinterpret_cast<const uint4*>(T);
    const uint4 b0 = t4[trow], b1 = t4[rows + trow], d0 = t4[2 * rows + trow],
                d1 = t4[3 * rows + trow];
    ob[0] = b0.x; ob[1] = b0.y; ob[2] = b0.z; ob[3] = b0.w;
    ob[4] = b1.x; ob[5] = b1.y; ob[6] = b1.z; ob[7] = b1.w;
    od[0] = d0.x; od[1] = d0.y; od[2] = d0.z; od[3] = d0.w;
    od[4] = d1.x; od[5] = d1.y; od[6] = d1.z; od[7] = d1.w;
  }
  auto boff = [&](int ks, int j) {
    const int e = ks * 4 + j;
    return (int)((ob[e >> 1] >> ((e & 1) * 16)) & 0xffffu);
  };
  auto doff = [&](int mt, int j, int c) {
    const int e = (mt * 4 + j) * 2 + c;
    return (int)((od[e >> 1] >> ((e & 1) * 16)) & 0xffffu);
  };
  double yr[4][2][2], yi[4][2][2];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) yr[u][mt][0] = yr[u][mt][1] = yi[u][mt][0] = yi[u][mt][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double2 xb = X[boff(ks, u)];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        dmma(yr[u][mt][0], yr[u][mt][1], ar[mt][ks], xb.x);
        dmma(yi[u][mt][0], yi[u][mt][1], ar[mt][ks], xb.y);
      }
    }
  __syncwarp();  // every lane's B loads precede any lane's D stores
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int c = 0; c < 2; ++c) X[doff(mt, u, c)] = make_double2(yr[u][mt][c], yi[u][mt][c]);
}

// k = 1 sub-op (4x4 complex, DFMA): T = this lane's 16 offsets [j column][i member].
__device__ __forceinline__ void blk_sub_k1(double2* X, const double* F, const uint16_t* T,
                                           int trow, int rows) {
  const double2* S = reinterpret_cast<const double2*>(F);
  uint32_t o[8];
  {  // table [2 chunks][rows][8 uint16]
    const uint4* t4 = reinterpret_cast<const uint4*>(T);
    const uint4 a = t4[trow], b = t4[rows + trow];
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
    o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
  }
  auto off = [&](int j, int i) {
    const int e = j * 4 + i;
    return (int)((o[e >> 1] >> ((e & 1) * 16)) & 0xffffu);
  };
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double2 x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = X[off(j, i)];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      double yr = 0.0, yi = 0.0;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const double2 s = S[l * 4 + m];
        yr = fma(s.x, x[m].x, yr);
        yr = fma(-s.y, x[m].y, yr);
        yi = fma(s.x, x[m].y, yi);
        yi = fma(s.y, x[m].x, yi);
      }
      X[off(j, l)] = make_double2(yr, yi);
    }
  }
}

}  // namespace

constexpr int kStageUnits = 1032;  // 16 x 64 + rotation slack (<= 7), rounded to 8 units
// shared header: mbarriers [2 * kBlockMaxPairs], piece offsets [64] (u64), starts [64] (u16)
constexpr int kBlockHdrBytes = 896;
constexpr int kBlockHdrBytesWs = 896;  // full + done mbarriers, piece tables
static_assert(32 * kBlockMaxPairs + 64 * 8 + 64 * 2 <= kBlockHdrBytesWs, "block header (ws)");
static_assert(16 * kBlockMaxPairs + 64 * 8 + 64 * 2 <= kBlockHdrBytes, "block header");

// COPY = 0: every pair thread moves one 256 B piece with cp.async.bulk (G2S with mbarrier
// complete_tx, S2G bulk_group).  COPY = 1: the pair's 64 threads move the block as 16 B
// cp.async.cg copies (16 per thread, 16 lanes per piece: every warp instruction reads two
// contiguous 256 B runs), signalled with cp.async.mbarrier.arrive, and store it back with
// coalesced LDS + STG.128 -- no per-lane serialised bulk-copy issue.
template <int UI, int COPY, int ACC, int MODE>
__global__ void __launch_bounds__(384, 1)
    block_kernel(double2* __restrict__ a, const __grid_constant__ BlockParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem_raw);  // [2 * kMaxPairs]
  uint64_t* sGoff = mbar + 2 * kBlockMaxPairs;              // [64] piece offsets by rank
  uint16_t* sStart = reinterpret_cast<uint16_t*>(sGoff + 64);  // [64] piece starts by rank
  unsigned char* sBlob = smem_raw + kBlockHdrBytes;
  double2* sStage = reinterpret_cast<double2*>(sBlob + p.blob_bytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, half = warp & 1, pt = threadIdx.x & 63;

  {  // blob (sub-op fragments + offset tables) -> shared; piece tables; mbarrier init
    const uint4* src = reinterpret_cast<const uint4*>(p.blob);
    uint4* dst = reinterpret_cast<uint4*>(sBlob);
    for (int i = threadIdx.x; i < p.blob_bytes / 16; i += blockDim.x) dst[i] = src[i];
    if (threadIdx.x < 64) {
      sGoff[threadIdx.x] = p.piece_goff[threadIdx.x];
      sStart[threadIdx.x] = p.piece_start[threadIdx.x];
    }
    if (threadIdx.x < 2 * p.pairs) mbar_init(&mbar[threadIdx.x], 64);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (pair >= p.pairs) return;

  double2* stage0 = sStage + (size_t)pair * 2 * kStageUnits;
  const uint64_t goff = sGoff[pt];
  const int sstart = sStart[pt];
  const int rot = piece_rot(pt & 7);
  const uint64_t nb = p.n_blocks;
  const uint64_t npairs = (uint64_t)gridDim.x * p.pairs;
  const bool mirror = p.mirror != 0;
  auto next_block = [&](uint64_t i) {
    if (mirror)
      while (i < nb && i > tpb<MODE>(i, p, 10)) i += npairs;
    return i;
  };
  // where piece (offset go) of the block at `base` lives: in place, or (packed layout,
  // non-canonical piece of a block that is not self-transposed) at the transposed position
  auto piece_src = [&](uint64_t base, bool self, uint64_t go, bool& tr) {
    const uint64_t e0 = base + go;
    const uint64_t em = tpb<MODE>(e0, p, 0);
    tr = mirror && !self && e0 > em;
    return tr ? em : e0;
  };
  auto is_self = [&](uint64_t base) {
    return mirror && tpb<MODE>(base, p, 0) == base;
  };
  auto issue = [&](uint64_t i, int s) {
    uint64_t* bar = &mbar[pair * 2 + s];
    double2* st = stage0 + s * kStageUnits;
    if (p.dbg & 2) {
      mbar_arrive(bar);
      return;
    }
    const uint64_t base = insert_zeros10(i, p.lo_mask);
    const bool self = is_self(base);
    if constexpr (COPY == 0 || COPY == 2) {
      bool tr;
      const uint64_t src = piece_src(base, self, goff, tr);
      mbar_arrive_tx(bar, 256);
      bulk_g2s(st + sstart, a + src, 256, bar);
    } else {
      const int u = pt & 15, qb = pt >> 4;
#pragma unroll 4
      for (int it = 0; it < 16; ++it) {
        const int q = it * 4 + qb;
        bool tr;
        const uint64_t src = piece_src(base, self, sGoff[q], tr);
        cp_async16_cg(st + sStart[q] + u, a + src + u);
      }
      cp_async_mbar_arrive(bar);
    }
  };

  // this pair's blocks b0, b1, ...: b_k is computed in iteration k from stage k % 2; stages
  // start with b0 and b1; from iteration 1 on, iteration k refills the stage stored in
  // iteration k-1 with b_{k+1}
  uint64_t cur = next_block((uint64_t)blockIdx.x * p.pairs + pair);
  uint64_t nxt = cur < nb ? next_block(cur + npairs) : nb;
  if (cur < nb) issue(cur, 0);
  if (nxt < nb) issue(nxt, 1);
  uint32_t parity[2] = {0u, 0u};
  bool first = true;
  int s = 0;
  while (cur < nb) {
    double2* X = stage0 + s * kStageUnits;
    mbar_wait(&mbar[pair * 2 + s], parity[s]);
    parity[s] ^= 1u;
    if constexpr (COPY == 0) {
      if (!first) {  // refill the other stage (its bulk stores have read it out)
        bulk_wait_read0();
        if (nxt < nb) issue(nxt, s ^ 1);
      }
    }
    const uint64_t base = insert_zeros10(cur, p.lo_mask);
    const bool self = is_self(base);
    bool trp;
    piece_src(base, self, goff, trp);  // this thread's piece came from the transpose?
    if (trp) piece_transpose(X + sstart, rot);
    if (self) {  // non-canonical element <- conj(its transpose, canonical, same block)
      for (int k = 0; k < 16; ++k) {
        const int idx = pt * 16 + ((k + pt) & 15);
        const int idm = ((idx & 0x155) << 1) | ((idx >> 1) & 0x155);
        if (idx > idm) {
          const double2 v = X[p.start_by_pidx[idm >> 4] + (idm & 15)];
          X[p.start_by_pidx[idx >> 4] + (idx & 15)] = make_double2(v.x, -v.y);
        }
      }
    }
    pair_bar(pair);
    if constexpr (COPY == 1 || COPY == 2) {
      // the other stage was read out (LDS for the stores) before the barrier above
      if (!first && nxt < nb) issue(nxt, s ^ 1);
    }
    if (!(p.dbg & 1)) {
      if constexpr ((MODE & 1) != 0) {  // sparse / real-basis / per-sub-op split programs
        const uint16_t* RB = reinterpret_cast<const uint16_t*>(sBlob) + p.rb_off;
        blk_rbasis(X, RB, p.rb_nq, pt, pair, true);
        for (int q = 0; q < p.n_sub; ++q) {
          const BlockSub& g = p.sub[q];
          if (g.sync) pair_bar(pair);  // the other warp's half of the last sub-op is done
          const bool shared_tab = g.hadd >= 0;
          double2* Xh = X + (shared_tab ? half * g.hadd : 0);
          const int trow = shared_tab ? lane : half * 32 + lane, trows = shared_tab ? 32 : 64;
          const double* F = reinterpret_cast<const double*>(sBlob) + g.a_off;
          const uint16_t* T = reinterpret_cast<const uint16_t*>(sBlob) + g.t_off;
          if (g.k == 2 && g.nnz)
            blk_sub_k2s(Xh, F, T, trow, trows, g.nnz);
          else if (g.k == 2 && p.rb_nq)
            blk_sub_k2r(Xh, F, T, lane, trow, trows);
          else if (g.k == 2)
            blk_sub_k2<UI, ACC>(Xh, F, T, lane, trow, trows);
          else
            blk_sub_k1(Xh, F, T, trow, trows);
          __syncwarp();
        }
        blk_rbasis(X, RB, p.rb_nq, pt, pair, false);
      } else {
        const bool shared_tab = p.half_add >= 0;
        double2* Xh = X + (shared_tab ? half * p.half_add : 0);
        const int trow = shared_tab ? lane : half * 32 + lane, trows = shared_tab ? 32 : 64;
        for (int q = 0; q < p.n_sub; ++q) {
          const BlockSub& g = p.sub[q];
          const double* F = reinterpret_cast<const double*>(sBlob) + g.a_off;
          const uint16_t* T = reinterpret_cast<const uint16_t*>(sBlob) + g.t_off;
          if (g.k == 2)
            blk_sub_k2<UI, ACC>(Xh, F, T, lane, trow, trows);
          else
            blk_sub_k1(Xh, F, T, trow, trows);
          __syncwarp();
        }
      }
    }
    pair_bar(pair);
    if (trp) piece_transpose(X + sstart, rot);
    if constexpr (COPY == 0) fence_async_smem();
    pair_bar(pair);
    if (!(p.dbg & 2)) {
      if constexpr (COPY == 0) {
        bool t2;
        const uint64_t dst = piece_src(base, self, goff, t2);
        bulk_s2g(a + dst, X + sstart, 256);
        bulk_commit();
      } else {
        const int u = pt & 15, qb = pt >> 4;
#pragma unroll 4
        for (int it = 0; it < 16; ++it) {
          const int q = it * 4 + qb;
          bool tr;
          const uint64_t dst = piece_src(base, self, sGoff[q], tr);
          a[dst + u] = X[sStart[q] + u];
        }
      }
    }
    first = false;
    cur = nxt;
    nxt = cur < nb ? next_block(cur + npairs) : nb;
    s ^= 1;
  }
  if constexpr (COPY == 0) bulk_wait0();
}

// TMA layout kernel (BlockParams::tma = 1).  Shared memory: mbarriers | blob (fragments,
// tables, slot table) | 1024 B-aligned stages of 16 KB (box order, 128 B swizzle).  Per block:
//   direct (every element stored in place: the base differs at a pair above hi_blk, or the
//   full layout) -- pair thread 0 issues one TMA box load (arrive.expect_tx 16 KB, the other 63
//   threads plain arrivals) and, after the sub-ops, one TMA box store;
//   otherwise -- every pair thread issues 16 cp.async 16 B copies (16 lanes per 256 B piece)
//   straight to each element's final slot (pieces read from the transposed position land
//   already permuted), conjugates them after the wait, and stores them back with STG.
template <int UI, int ACC, int MODE>
__global__ void __launch_bounds__(384, 1)
    block_kernel_tma(double2* __restrict__ a, const __grid_constant__ BlockParams p,
                     const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem_raw);
  unsigned char* sBlob = smem_raw + kBlockHdrBytes;
  const size_t stage_off = (kBlockHdrBytes + (size_t)p.blob_bytes + 1023) & ~(size_t)1023;
  double2* sStage = reinterpret_cast<double2*>(smem_raw + stage_off);
  const uint16_t* sSlot = reinterpret_cast<const uint16_t*>(sBlob) + p.slot_off;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, half = warp & 1, pt = threadIdx.x & 63;
  {
    const uint4* src = reinterpret_cast<const uint4*>(p.blob);
    uint4* dst = reinterpret_cast<uint4*>(sBlob);
    for (int i = threadIdx.x; i < p.blob_bytes / 16; i += blockDim.x) dst[i] = src[i];
    if (threadIdx.x < 2 * p.pairs) mbar_init(&mbar[threadIdx.x], 64);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (pair >= p.pairs) return;
  double2* stage0 = sStage + (size_t)pair * 2 * 1024;
  const uint64_t nb = p.n_blocks;
  const uint64_t npairs = (uint64_t)gridDim.x * p.pairs;
  const bool mirror = p.mirror != 0;
  auto next_block = [&](uint64_t i) {
    if (mirror)
      while (i < nb && i > tpb<MODE>(i, p, 10)) i += npairs;
    return i;
  };
  // block classification: 0 direct (TMA), 1 cp.async with transposed pieces, 2 self-transposed
  auto kind_of = [&](uint64_t base) {
    if (!mirror) return 0;
    const uint64_t d = (base ^ tpb<MODE>(base, p, 0)) &
                       (0x5555555555555555ull | ((MODE & 2) != 0 ? ~p.tp_lo : 0ull));
    if (!d) return 2;
    return (63 - __clzll(d)) > p.hi_blk ? 0 : 1;
  };
  auto coords = [&](uint64_t base, int* c) {
#pragma unroll
    for (int d = 0; d < 5; ++d)
      c[d] = d < p.tdims ? (int)((base >> p.tlo[d]) & (((uint64_t)1 << p.tbits[d]) - 1)) : 0;
    c[0] *= 2;  // dim 0 counts doubles
  };
  auto issue = [&](uint64_t i, int s) {
    uint64_t* bar = &mbar[pair * 2 + s];
    double2* st = stage0 + s * 1024;
    if (p.dbg & 2) {
      mbar_arrive(bar);
      return;
    }
    const uint64_t base = insert_zeros10(i, p.lo_mask);
    const int kd = kind_of(base);
    if (kd == 0) {
      if (pt == 0) {
        mbar_arrive_tx(bar, 16384);
        int c[5];
        coords(base, c);
        tma_load_5d(st, &tmap, c, bar);
      } else {
        mbar_arrive(bar);
      }
    } else {
      const int u = pt & 15, qb = pt >> 4;
#pragma unroll 4
      for (int it = 0; it < 16; ++it) {
        const int q = it * 4 + qb;
        const uint64_t e0 = base + p.piece_goff[q];
        const uint64_t em = tpb<MODE>(e0, p, 0);
        const bool tr = kd == 1 && e0 > em;
        cp_async16_cg(st + sSlot[q * 16 + (tr ? pswap4(u) : u)], a + (tr ? em : e0) + u);
      }
      cp_async_mbar_arrive(bar);
    }
  };

  uint64_t cur = next_block((uint64_t)blockIdx.x * p.pairs + pair);
  uint64_t nxt = cur < nb ? next_block(cur + npairs) : nb;
  if (cur < nb) issue(cur, 0);
  if (nxt < nb) issue(nxt, 1);
  uint32_t parity[2] = {0u, 0u};
  bool first = true;
  int s = 0;
  while (cur < nb) {
    double2* X = stage0 + s * 1024;
    // this thread's cp.async copies of the block have landed (the mbarrier below covers the
    // other threads'; the explicit wait also lets compute-sanitizer's racecheck see it)
    asm volatile("cp.async.wait_all;" ::: "memory");
    mbar_wait(&mbar[pair * 2 + s], parity[s]);
    parity[s] ^= 1u;
    if (pt == 0 && !first) bulk_wait_read0();  // last iteration's TMA store has read its stage
    const uint64_t base = insert_zeros10(cur, p.lo_mask);
    const int kd = (p.dbg & 2) ? 0 : kind_of(base);
    if (kd == 1) {  // conjugate the pieces that came from the transposed position
      const uint64_t e0 = base + p.piece_goff[pt];
      if (e0 > tpb<MODE>(e0, p, 0)) {
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          double* im = &X[sSlot[pt * 16 + ((t + pt) & 15)]].y;
          *im = -*im;
        }
      }
    } else if (kd == 2) {  // self-transposed: non-canonical <- conj(canonical)
      for (int k = 0; k < 16; ++k) {
        const int idx = pt * 16 + ((k + pt) & 15);
        const int idm = ((idx & 0x155) << 1) | ((idx >> 1) & 0x155);
        if (idx > idm) {
          const double2 v = X[sSlot[idm]];
          X[sSlot[idx]] = make_double2(v.x, -v.y);
        }
      }
    }
    pair_bar(pair);
    if (!first && nxt < nb) issue(nxt, s ^ 1);
    if (!(p.dbg & 1)) {
      if constexpr ((MODE & 1) != 0) {  // sparse / real-basis / per-sub-op split programs
        double2* Xh = X;
        const int trow = half * 32 + lane;
        const uint16_t* RB = reinterpret_cast<const uint16_t*>(sBlob) + p.rb_off;
        blk_rbasis(X, RB, p.rb_nq, pt, pair, true);
        for (int q = 0; q < p.n_sub; ++q) {
          const BlockSub& g = p.sub[q];
          if (g.sync) pair_bar(pair);  // the other warp's half of the last sub-op is done
          const double* F = reinterpret_cast<const double*>(sBlob) + g.a_off;
          const uint16_t* T = reinterpret_cast<const uint16_t*>(sBlob) + g.t_off;
          if (g.k == 2 && g.nnz)
            blk_sub_k2s(Xh, F, T, trow, 64, g.nnz);
          else if (g.k == 2 && p.rb_nq)
            blk_sub_k2r(Xh, F, T, lane, trow, 64);
          else if (g.k == 2)
            blk_sub_k2<UI, ACC>(Xh, F, T, lane, trow, 64);
          else
            blk_sub_k1(Xh, F, T, trow, 64);
          __syncwarp();
        }
        blk_rbasis(X, RB, p.rb_nq, pt, pair, false);
      } else {
        const int trow = half * 32 + lane;
        for (int q = 0; q < p.n_sub; ++q) {
          const BlockSub& g = p.sub[q];
          const double* F = reinterpret_cast<const double*>(sBlob) + g.a_off;
          const uint16_t* T = reinterpret_cast<const uint16_t*>(sBlob) + g.t_off;
          if (g.k == 2)
            blk_sub_k2<UI, ACC>(X, F, T, lane, trow, 64);
          else
            blk_sub_k1(X, F, T, trow, 64);
          __syncwarp();
        }
      }
    }
    if (kd == 0) fence_async_smem();
    pair_bar(pair);
    if (!(p.dbg & 2)) {
      if (kd == 0) {
        if (pt == 0) {
          int c[5];
          coords(base, c);
          tma_store_5d(&tmap, c, X);
          bulk_commit();
        }
      } else {
        const int u = pt & 15, qb = pt >> 4;
#pragma unroll 4
        for (int it = 0; it < 16; ++it) {
          const int q = it * 4 + qb;
          const uint64_t e0 = base + p.piece_goff[q];
          const uint64_t em = tpb<MODE>(e0, p, 0);
          const bool tr = kd == 1 && e0 > em;
          double2 v = X[sSlot[q * 16 + (tr ? pswap4(u) : u)]];
          if (tr) v.y = -v.y;
          a[(tr ? em : e0) + u] = v;
        }
      }
    }
    first = false;
    cur = nxt;
    nxt = cur < nb ? next_block(cur + npairs) : nb;
    s ^= 1;
  }
  if (pt == 0) bulk_wait0();
}

size_t block_smem_bytes_tma(int pairs, int blob_bytes) {
  return ((kBlockHdrBytes + (size_t)blob_bytes + 1023) & ~(size_t)1023) + (size_t)pairs * 2 * 16384;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link dependency)
static cudaError_t encode_block_tmap(CUtensorMap* map, double2* a, const BlockParams& p) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !f) return cudaErrorNotSupported;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  cuuint64_t gdim[5], gstride[4];
  cuuint32_t box[5], estride[5] = {1, 1, 1, 1, 1};
  const int top = p.tlo[p.tdims - 1] + p.tbits[p.tdims - 1];  // = local bits L
  for (int d = 0; d < 5; ++d) {
    if (d < p.tdims) {
      gdim[d] = (cuuint64_t)1 << p.tbits[d];
      box[d] = 1u << p.tbox[d];
    } else {  // unit padding dims beyond the whole shard
      gdim[d] = 1;
      box[d] = 1;
    }
    if (d >= 1) gstride[d - 1] = (cuuint64_t)16 << (d < p.tdims ? p.tlo[d] : top);
  }
  gdim[0] *= 2;  // doubles
  box[0] *= 2;
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, a, gdim, gstride, box, estride,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int ACC, int MODE>
static cudaError_t launch_block_tma(double2* a, const BlockParams& p, cudaStream_t st) {
  static std::atomic<uint64_t> attr_done{0};
  auto kern = block_kernel_tma<2, ACC, MODE>;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = (uint64_t)1 << (dev & 63);
  if (!(attr_done.load() & bit)) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr_done.fetch_or(bit);
  }
  CUtensorMap map;
  e = encode_block_tmap(&map, a, p);
  if (e != cudaSuccess) {
    set_error("cuTensorMapEncodeTiled rejected the block box");
    return e;
  }
  const size_t smem = block_smem_bytes_tma(p.pairs, p.blob_bytes);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t want = (p.n_blocks + p.pairs - 1) / p.pairs;
  unsigned grid = (unsigned)(want < (uint64_t)sms ? want : (uint64_t)sms);
  const char* cap = getenv("TANQ_GRID_CAP");
  if (cap && atoi(cap) > 0 && grid > (unsigned)atoi(cap)) grid = (unsigned)atoi(cap);
  if (grid < 1) grid = 1;
  kern<<<grid, 64 * p.pairs, smem, st>>>(a, p, map);
  return cudaGetLastError();
}

template <int UI, int COPY, int ACC, int MODE>
static cudaError_t launch_block_cfg(double2* a, const BlockParams& p, size_t smem,
                                    cudaStream_t st) {
  static std::atomic<uint64_t> attr_done{0};
  auto kern = block_kernel<UI, COPY, ACC, MODE>;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = (uint64_t)1 << (dev & 63);
  if (!(attr_done.load() & bit)) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr_done.fetch_or(bit);
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t want = (p.n_blocks + p.pairs - 1) / p.pairs;
  unsigned grid = (unsigned)(want < (uint64_t)sms ? want : (uint64_t)sms);
  const char* cap = getenv("TANQ_GRID_CAP");
  if (cap && atoi(cap) > 0 && grid > (unsigned)atoi(cap)) grid = (unsigned)atoi(cap);
  if (grid < 1) grid = 1;
  kern<<<grid, 64 * p.pairs, smem, st>>>(a, p);
  return cudaGetLastError();
}

size_t block_smem_bytes(int pairs, int blob_bytes) {
  return kBlockHdrBytes + (size_t)blob_bytes + (size_t)pairs * 2 * kStageUnits * 16;
}

// env TANQ_BLOCK_COPY = bulk (default) | ldg | bs: how blocks move between HBM and shared
// memory -- bulk: cp.async.bulk pieces both ways; ldg: 16 B cp.async loads + coalesced STG
// stores; bs: bulk loads + STG stores.  A warp-specialised producer variant (2 producer warps
// issuing every piece) and a single-elected-thread issue loop were measured slower and removed
// (profiles/r02_block_copy_variants.txt).  TANQ_BLOCK_ACC = 1: three independent DMMA
// accumulators + 2 DADD per output instead of the seeded chain.
cudaError_t launch_block_group(double2* a, const BlockParams& p, int L, cudaStream_t st) {
  (void)L;
  static int copy = -1, acc = -1;
  if (copy < 0) {
    const char* e = getenv("TANQ_BLOCK_COPY");
    copy = !e ? 0 : (e[0] == 'l' ? 1 : (!strcmp(e, "bs") ? 2 : 0));
    const char* f = getenv("TANQ_BLOCK_ACC");
    acc = (f && f[0] == '1') ? 1 : ((f && f[0] == '2') ? 2 : 0);
  }
  // MODE: bit 0 = the program uses sparse / real-basis / per-sub-op-split sub-ops, bit 1 = a
  // non-trivial shard transpose descriptor; the plain single-shard programs of the bench run
  // the instantiation without either (their extra code measurably slowed the hot loop)
  bool ext = p.rb_nq > 0;
  for (int q = 0; q < p.n_sub; ++q)
    ext = ext || p.sub[q].nnz > 0 || p.sub[q].sync != 0 || p.sub[q].hadd != p.half_add;
  const int mode = (ext ? 1 : 0) | ((p.tp_lo != ~0ull || p.tp_m != 0) ? 2 : 0);
  if (p.tma) {
    if (acc == 2) return launch_block_tma<2, 3>(a, p, st);
    switch (mode) {
      case 0: return launch_block_tma<0, 0>(a, p, st);
      case 1: return launch_block_tma<0, 1>(a, p, st);
      case 2: return launch_block_tma<0, 2>(a, p, st);
      default: return launch_block_tma<0, 3>(a, p, st);
    }
  }
  const size_t smem = block_smem_bytes(p.pairs, p.blob_bytes);
  if (smem > 227 * 1024 || p.pairs < 1 || p.pairs > kBlockMaxPairs) return cudaErrorInvalidValue;
  if (acc == 1) {  // experiment variants: the generic instantiation
    if (copy == 1) return launch_block_cfg<2, 1, 1, 3>(a, p, smem, st);
    if (copy == 2) return launch_block_cfg<2, 2, 1, 3>(a, p, smem, st);
    return launch_block_cfg<2, 0, 1, 3>(a, p, smem, st);
  }
  if (acc == 2) return launch_block_cfg<2, 0, 2, 3>(a, p, smem, st);
  if (copy == 1) return launch_block_cfg<2, 1, 0, 3>(a, p, smem, st);
  if (copy == 2) return launch_block_cfg<2, 2, 0, 3>(a, p, smem, st);
  switch (mode) {
    case 0: return launch_block_cfg<2, 0, 0, 0>(a, p, smem, st);
    case 1: return launch_block_cfg<2, 0, 0, 1>(a, p, smem, st);
    case 2: return launch_block_cfg<2, 0, 0, 2>(a, p, smem, st);
    default: return launch_block_cfg<2, 0, 0, 3>(a, p, smem, st);
  }
}

}  // namespace tanq
