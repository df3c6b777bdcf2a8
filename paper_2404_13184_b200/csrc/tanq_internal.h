// Internal interface between the host planner (tanq_host.cpp) and the sm_100a kernels
// (tanq_kernels.cu).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tanq {

void set_error(const char* msg);  // message returned by tanq_last_error() (thread-local)

// A gate launch: apply a dense 4^K x 4^K complex matrix to every tuple of one shard.
// Member i of a tuple sits at physical offset base + sum_j bit_j(i) << pos[j], where
// pos[0] < pos[1] < ... < pos[2K-1] are the op's physical target bits (all local);
// base is the tuple index with zero bits inserted at pos[] (Eq. 4's s_i generalised,
// P:82-98).  S is stored in member order (the host permutes the paper's r + c 2^k order).
template <int K>
struct GateParams {
  static constexpr int M = 1 << (2 * K);
  double2 S[M * M];
  uint64_t lo_mask[2 * K];   // (1 << pos[j]) - 1
  uint64_t n_tuples;         // 2^(L - 2K)
  uint32_t pos[2 * K];
  uint32_t mirror;           // 1: packed Hermitian mode
  uint64_t tp_lo, tp_m;      // packed mode: transpose descriptor of the shard (TDesc below)
};

// K3 groups: a program of sub-ops (k = 1, 2 or 3) applied to 4^nq-member tuples (2 nq
// physical bits pos[], all local, nq = 3 or 4) in one HBM round trip.  Sub-op matrices live in `prog` in A-fragment
// order (group_make_frags); mi[i] / mu[u] map sub-op member i / sub-tuple u to tile members.
static constexpr int kMaxSub = 40;
static constexpr int kGroupProgMax = 5632;  // double2 (88 KiB): one dense k=3 + 6 k=2, or 22 k=2
struct GroupSub {
  int32_t k;
  int32_t s_off;     // offset of the sub-op matrix in prog (double2 units)
  uint8_t mi[16];    // tile member of sub-op member i
  uint8_t mu[64];    // tile member offset of sub-tuple u (4^(NQ-k) sub-tuples)
};
struct GroupParams {
  const double2* prog;
  int32_t prog_elems;
  int32_t n_sub;
  int32_t nq;                // group qubits: 3 (64-member tuples) or 4 (256-member tuples)
  uint64_t lo_mask[8];
  uint64_t n_tuples;
  uint32_t pos[8];
  uint32_t mirror;           // 1: packed Hermitian mode
  uint64_t tp_lo, tp_m;      // packed mode: transpose descriptor of the shard
  uint32_t dbg;              // profiling experiments only (env TANQ_DBG): 1 skip sub-ops,
                             // 2 skip HBM copies; 0 in production
  GroupSub sub[kMaxSub];
};

// Block-pipeline group kernel (tanq_block.cu).  A block = 10 physical bits (5 whole qubits in
// the packed layout: the group's plus the lowest free ones), 64 pieces of 16 contiguous
// amplitudes; a pair of warps streams blocks through two shared-memory stages.
static constexpr int kBlockMaxPairs = 6;
static constexpr int kBlockMaxSub = 12;
struct BlockSub {
  int32_t k;       // 1 or 2
  int32_t a_off;   // doubles: k=2 fragments [3][4 ks][32 lanes][2 mt] (a, -(a+b), b-a);
                   // k=1: 16 double2; sparse k=2: nnz double2 values (row-major) + uint16
                   // row starts [17]
  int32_t t_off;   // uint16: per-lane shared-memory offset tables [1|2 halves][32][32|16];
                   // sparse k=2: [nnz + 16][rows] (entry inputs, then the 16 outputs)
  int32_t tmask;   // k=2: nonzero 8x4 A tiles, bit mt * 4 + ks (zero tiles are skipped)
  int32_t nnz;     // k=2: > 0 -> sparse DFMA sub-op (one tuple per lane), 0 -> DMMA
  int32_t hadd;    // >= 0: one table for both warp halves, the second adding hadd units;
                   // -1: a table per half (the warp-half bit of this sub-op)
  int32_t sync;    // 1: the warp-half bit differs from the previous sub-op's (5-qubit block
                   // groups): the pair meets at a barrier first
};
struct BlockParams {
  const void* blob;          // sub-op fragments + offset tables (device), copied to shared
  int32_t blob_bytes;        // multiple of 16
  int32_t n_sub;
  int32_t pairs;             // warp pairs per CTA (smem-limited, <= kBlockMaxPairs)
  uint32_t mirror;           // packed Hermitian layout
  uint64_t tp_lo, tp_m;      // packed mode: transpose descriptor of the shard
  uint32_t dbg;              // experiments only: 1 skip sub-ops, 2 skip HBM copies
  int32_t half_add;          // >= 0: one offset table for both warp halves, the second half
                             // adding half_add units; -1: a table per half
  uint64_t n_blocks;         // 2^(L - 10)
  uint64_t lo_mask[10];      // (1 << pos) - 1 of the 10 block positions, ascending
  uint64_t piece_goff[64];   // element offset of the piece handled by pair thread j
  uint16_t piece_start[64];  // its shared-memory start (16 B units) in a stage
  uint16_t start_by_pidx[64];// shared-memory start of piece index (block bits 4..9)
  BlockSub sub[kBlockMaxSub];
  // TMA layout (tma = 1): the block is described as a <= 5-D box of the shard -- dim d covers
  // physical bits [tlo[d], tlo[d] + tbits[d]), its lowest tbox[d] bits vary inside the block --
  // and lands in shared memory in box order with the 128 B swizzle: element idx (block order)
  // at 16 B unit idx ^ ((idx >> 3) & 7).  Blocks whose elements are all stored in place (no
  // pair above hi_blk needed to decide, not self-transposed) move with one TMA load / store;
  // the others with 16 B cp.async copies placed through the slot table.
  uint32_t tma;
  int32_t tdims;
  int32_t tlo[5];
  int32_t tbits[5];
  int32_t tbox[5];
  int32_t hi_blk;            // highest block bit position
  int32_t slot_off;          // uint16 offset of the 1024-entry slot table in the blob
  // Real basis (rb_nq > 0): after the load the block is transformed on rb_nq
  // group qubits -- each qubit's (row 1 col 0, row 0 col 1) element pair (x1, x2) becomes
  // (x1 + x2, i (x2 - x1)) -- where every Hermiticity-preserving sub-op is a REAL matrix R:
  // k=2 sub-ops run as 2 real DMMA products (R Re x, R Im x; fragments [4 ks][32][2 mt])
  // instead of 3; the inverse transform runs before the store.  Tables at rb_off (uint16):
  // [rb_nq][64 pair threads][4 pairs][2 slots].
  int32_t rb_nq;
  int32_t rb_off;
};

// Transpose descriptor of a shard in the packed Hermitian layout.  The
// transpose of a local element index e is  pair_swap(e & lo) | ((e & ~lo) ^ m):  the fully
// local qubits occupy aligned (row, col) pairs below the boundary lo = 2^(2F) - 1, and above it
// sit the row bits of the half-global qubits of the shard-local parity layout, whose global bit
// holds r XOR c -- the transpose keeps the shard and flips the row bit where the shard's parity
// bit is 1 (m).  One shard: lo = ~0, m = 0 (plain pair_swap).
struct TDesc {
  uint64_t lo = ~0ull;
  uint64_t m = 0;
};

struct BitMap {               // physical bit of each logical bit (row q -> 2q, col q -> 2q+1)
  uint32_t phys[64];
  int nbits;                 // 2n
  uint64_t par;              // qubits h whose col slot phys[2h+1] holds r_h XOR c_h (parity
                             // layout: every global bit is such a parity bit)
};

// kernel launchers (all asynchronous on `st`)
cudaError_t launch_gate1(double2* a, const GateParams<1>& p, cudaStream_t st);
cudaError_t launch_gate2(double2* a, const GateParams<2>& p, cudaStream_t st);
cudaError_t launch_group3(double2* a, const GroupParams& p, cudaStream_t st);
cudaError_t launch_block_group(double2* a, const BlockParams& p, int L, cudaStream_t st);
size_t block_smem_bytes(int pairs, int blob_bytes);
// packed Hermitian layout -> full layout (single shard, interleaved identity bit map)
cudaError_t launch_unpack(double2* a, int L, TDesc td, cudaStream_t st);
size_t group_frag_elems(int k);                               // double2 per sub-op matrix
void group_make_frags(int k, const double2* S_member_order, double2* frag /*host*/);

cudaError_t launch_init(double2* a, uint64_t elems, bool one_at_zero, cudaStream_t st);
// In-place swap of the halves two shards exchange when global bit g swaps with local bit b:
// element e in [0, 2^(L-1)): j = e >> b, low = e & (2^b - 1);
//   A[(j << (b+1)) | (va << b) | low]  <->  B[(j << (b+1)) | (vb << b) | low]
cudaError_t launch_swap_halves(double2* A, double2* B, int L, int b, int va, int vb,
                               cudaStream_t st);
// pack / unpack the half {o : bit_b(o) == v} of a shard to / from a contiguous buffer,
// elements [first, first + count) of the half in run order.
cudaError_t launch_pack_half(const double2* a, double2* buf, int b, int v, uint64_t first,
                             uint64_t count, cudaStream_t st);
cudaError_t launch_unpack_half(double2* a, const double2* buf, int b, int v, uint64_t first,
                               uint64_t count, cudaStream_t st);
// the same for the quarter {o : bit_b0(o) == v0, bit_b1(o) == v1}, b0 < b1
cudaError_t launch_pack_quarter(const double2* a, double2* buf, int b0, int v0, int b1, int v1,
                                uint64_t first, uint64_t count, cudaStream_t st);
cudaError_t launch_unpack_quarter(double2* a, const double2* buf, int b0, int v0, int b1, int v1,
                                  uint64_t first, uint64_t count, cudaStream_t st);

// Parity-layout remap: half-global qubit h (local row bit x, global parity bit
// a) trades places with fully local qubit v (row bit y, col bit z).  An element with local
// bits (ex, ey, ez) on the shard whose bit a is s moves to the shard whose bit a is ey ^ ez, at
// local bits (x, y, z) = (ey, ex, ex ^ s).  Octet = the 8 elements differing in x, y, z.
// Single process: both shards of a pair (A: bit a = 0, B: 1) in one in-place kernel.
cudaError_t launch_parity_swap(double2* A, double2* B, int L, int x, int y, int z,
                               cudaStream_t st);
// One process per shard: the staying elements (ey ^ ez == s) are permuted in place; the
// leaving ones are packed as (octet, slot j = 2 ex + ey) and the partner's arrive in the
// slots they vacate (elements [first, first + count) of that order; count, first % 4 == 0).
cudaError_t launch_parity_stay(double2* a, int L, int x, int y, int z, int s, cudaStream_t st);
cudaError_t launch_parity_pack(const double2* a, double2* buf, int L, int x, int y, int z, int s,
                               uint64_t first, uint64_t count, cudaStream_t st);
cudaError_t launch_parity_unpack(double2* a, const double2* buf, int L, int x, int y, int z,
                                 int s, uint64_t first, uint64_t count, cudaStream_t st);

// Paper vec index v = r + c 2^n  <->  physical index; gather / scatter the owned entries
// of a range [first, first+count) of vec(rho) for shard `shard` (local bits L).
cudaError_t launch_gather_vec(const double2* a, double2* out, const BitMap& bm, int n, int L,
                              uint64_t shard, uint64_t first, uint64_t count, bool zero_unowned,
                              cudaStream_t st);
cudaError_t launch_scatter_vec(double2* a, const double2* in, const BitMap& bm, int n, int L,
                               uint64_t shard, uint64_t first, uint64_t count, cudaStream_t st);

// probs[x] = Re rho[x][x] for owned x (others untouched); atomically max |Im| into *imax
// (as the bit pattern of a non-negative double).
cudaError_t launch_diag(const double2* a, double* probs, unsigned long long* imax,
                        const BitMap& bm, int n, int L, uint64_t shard, cudaStream_t st);
cudaError_t launch_readout(double* p, int n, const double* p10, const double* p01,
                           cudaStream_t st);
// Partial sums of (-1)^{popc(a & z)} rho[a ^ x][a] over owned a into partial[blocks] (re, im)
cudaError_t launch_expect(const double2* a, double2* partial, int nblocks, const BitMap& bm,
                          int n, int L, uint64_t shard, uint64_t xm, uint64_t zm,
                          cudaStream_t st);
int expect_blocks(int n);
cudaError_t launch_reduce_partials(const double2* partial, int nblocks, double2* out,
                                   cudaStream_t st);
// sampling: clamp + inclusive scan (single CTA), then Philox draws + binary search
cudaError_t launch_cdf(const double* p, double* cdf, int n, cudaStream_t st);
cudaError_t launch_sample(const double* cdf, int n, uint64_t seed, uint64_t shots,
                          unsigned long long* out, cudaStream_t st);
cudaError_t launch_add(double* dst, const double* src, uint64_t count, cudaStream_t st);
// res[0] = max |a[P] - conj(a[pair_swap(P)])|, res[1] = max |a[P]| (bit patterns of doubles)
cudaError_t launch_herm_check(const double2* a, int L, TDesc td, unsigned long long* res,
                              cudaStream_t st);

}  // namespace tanq
