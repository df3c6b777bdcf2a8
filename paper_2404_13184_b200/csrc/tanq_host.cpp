// libtanq host side: C ABI (include/tanq.h), superoperator builder, noise binding, gate
// fusion, layout / remap planner and device orchestration.  Kernels: tanq_kernels.cu.
//
// Citations: P:n = /root/reference/PAPER.md line n.  DESIGN.md lists the readings R1-R20.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <thread>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "tanq.h"
#include "tanq_internal.h"

using cd = std::complex<double>;

namespace {

thread_local std::string g_err;

tanq_status fail(tanq_status s, const std::string& m) {
  g_err = m;
  return s;
}
}  // namespace

void tanq::set_error(const char* msg) { g_err = msg; }

namespace {

// NCCL is loaded on demand (multi-process mode only) with dlopen: an already-loaded
// libnccl.so.2 (e.g. the one torch brought in) is reused, so the library never pins an
// NCCL version into a process that imports torch afterwards.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;  // optional
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;                        // optional
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  // TANQ_NCCL_LIB names another implementation of the NCCL calls used here (tests: the
  // host-staged transport of tests/nccl_shim.cpp, which lets several ranks share one GPU)
  const char* env = getenv("TANQ_NCCL_LIB");
  void* h = env ? dlopen(env, RTLD_NOW | RTLD_LOCAL) : dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h && !env) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
#define LOAD(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
  LOAD(GetUniqueId);
  LOAD(CommInitRank);
  LOAD(CommDestroy);
  LOAD(GroupStart);
  LOAD(GroupEnd);
  LOAD(Send);
  LOAD(Recv);
  LOAD(AllReduce);
  LOAD(GetErrorString);
  LOAD(CommGetAsyncError);
  LOAD(CommAbort);
#undef LOAD
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart &&
           api.GroupEnd && api.Send && api.Recv && api.AllReduce && api.GetErrorString;
  return api;
}

#define CUDA_TRY(x)                                                                     \
  do {                                                                                  \
    cudaError_t _e = (x);                                                               \
    if (_e != cudaSuccess)                                                              \
      return fail(TANQ_E_CUDA, std::string(#x) + " -> " + cudaGetErrorString(_e));     \
  } while (0)
#define NCCL_TRY(x)                                                                     \
  do {                                                                                  \
    ncclResult_t _r = (x);                                                              \
    if (_r != ncclSuccess)                                                              \
      return fail(TANQ_E_NCCL, std::string(#x) + " -> " + nccl().GetErrorString(_r));    \
  } while (0)
#define TRY(x)                                                                          \
  do {                                                                                  \
    tanq_status _s = (x);                                                               \
    if (_s != TANQ_OK) return _s;                                                       \
  } while (0)

// ------------------------------------------------------------------------------------
// small dense complex matrices (row-major)
// ------------------------------------------------------------------------------------
struct Mat {
  int d = 0;
  std::vector<cd> a;
  Mat() = default;
  explicit Mat(int dim) : d(dim), a((size_t)dim * dim, cd(0.0, 0.0)) {}
  cd& operator()(int i, int j) { return a[(size_t)i * d + j]; }
  const cd& operator()(int i, int j) const { return a[(size_t)i * d + j]; }
};

Mat identity(int d) {
  Mat m(d);
  for (int i = 0; i < d; ++i) m(i, i) = 1.0;
  return m;
}

Mat matmul(const Mat& A, const Mat& B) {
  Mat C(A.d);
  for (int i = 0; i < A.d; ++i)
    for (int l = 0; l < A.d; ++l) {
      const cd x = A(i, l);
      if (x == cd(0.0, 0.0)) continue;
      for (int j = 0; j < A.d; ++j) C(i, j) += x * B(l, j);
    }
  return C;
}

// ------------------------------------------------------------------------------------
// gate unitaries (local index sum_j b(q_j) 2^j; q[0] = control of CX/CZ/CP)
// ------------------------------------------------------------------------------------
int kind_arity(int kind) {
  if (kind >= TANQ_ID && kind <= TANQ_RZ) return 1;
  if (kind == TANQ_RESET) return 1;
  if (kind >= TANQ_CX && kind <= TANQ_SWAP) return 2;
  return 0;  // user matrices: arity from op.k
}

Mat gate_unitary(int kind, double th) {
  const double c = std::cos(th / 2), s = std::sin(th / 2), r2 = 1.0 / std::sqrt(2.0);
  const cd I(0.0, 1.0);
  Mat u(kind_arity(kind) == 2 ? 4 : 2);
  switch (kind) {
    case TANQ_ID: u = identity(2); break;
    case TANQ_X: u(0, 1) = 1; u(1, 0) = 1; break;
    case TANQ_Y: u(0, 1) = -I; u(1, 0) = I; break;
    case TANQ_Z: u(0, 0) = 1; u(1, 1) = -1; break;
    case TANQ_H: u(0, 0) = r2; u(0, 1) = r2; u(1, 0) = r2; u(1, 1) = -r2; break;
    case TANQ_S: u(0, 0) = 1; u(1, 1) = I; break;
    case TANQ_SDG: u(0, 0) = 1; u(1, 1) = -I; break;
    case TANQ_T: u(0, 0) = 1; u(1, 1) = std::polar(1.0, M_PI / 4); break;
    case TANQ_TDG: u(0, 0) = 1; u(1, 1) = std::polar(1.0, -M_PI / 4); break;
    case TANQ_SX:
      u(0, 0) = cd(0.5, 0.5); u(0, 1) = cd(0.5, -0.5);
      u(1, 0) = cd(0.5, -0.5); u(1, 1) = cd(0.5, 0.5);
      break;
    case TANQ_RX: u(0, 0) = c; u(0, 1) = -I * s; u(1, 0) = -I * s; u(1, 1) = c; break;
    case TANQ_RY: u(0, 0) = c; u(0, 1) = -s; u(1, 0) = s; u(1, 1) = c; break;
    case TANQ_RZ: u(0, 0) = std::polar(1.0, -th / 2); u(1, 1) = std::polar(1.0, th / 2); break;
    case TANQ_CX:  // |c=1,t=0> (1) <-> |c=1,t=1> (3)
      u(0, 0) = 1; u(2, 2) = 1; u(3, 1) = 1; u(1, 3) = 1;
      break;
    case TANQ_CZ: u(0, 0) = 1; u(1, 1) = 1; u(2, 2) = 1; u(3, 3) = -1; break;
    case TANQ_CP: u(0, 0) = 1; u(1, 1) = 1; u(2, 2) = 1; u(3, 3) = std::polar(1.0, th); break;
    case TANQ_SWAP: u(0, 0) = 1; u(1, 2) = 1; u(2, 1) = 1; u(3, 3) = 1; break;
  }
  return u;
}

// ------------------------------------------------------------------------------------
// superoperators, local vec index l = r + c d (column stacking)
// ------------------------------------------------------------------------------------
// vec(U X U^dag)[r' + c' d] = sum U[r'][r] X[r][c] conj(U[c'][c])  ->  S = conj(U) (x) U
void add_superop_of(const Mat& K, Mat& S) {
  const int d = K.d;
  for (int c2 = 0; c2 < d; ++c2)
    for (int r2 = 0; r2 < d; ++r2)
      for (int c = 0; c < d; ++c) {
        const cd kc = std::conj(K(c2, c));
        if (kc == cd(0.0, 0.0)) continue;
        for (int r = 0; r < d; ++r) S(r2 + c2 * d, r + c * d) += kc * K(r2, r);
      }
}

Mat superop_from_kraus(const std::vector<Mat>& Ks) {
  Mat S(Ks[0].d * Ks[0].d);
  for (const Mat& K : Ks) add_superop_of(K, S);
  return S;
}

// depolarizing on the k qubits jointly (reading R7): (1-p) X + p tr(X) I/d
Mat superop_depol(int k, double p) {
  const int d = 1 << k, D = d * d;
  Mat S = identity(D);
  for (int i = 0; i < D; ++i) S(i, i) *= (1.0 - p);
  for (int r = 0; r < d; ++r)
    for (int r2 = 0; r2 < d; ++r2) S(r2 + r2 * d, r + r * d) += p / d;
  return S;
}

// thermal relaxation on one qubit (reading R8): populations rho11 -> e^{-t/T1} rho11,
// rho00 -> rho00 + (1 - e^{-t/T1}) rho11, coherences -> e^{-t/T2}.  (AD(gamma) then
// PD(lambda) with gamma = 1 - e^{-t/T1}, lambda = 1 - e^{-2t(1/T2 - 1/(2T1))}.)
Mat superop_thermal(double t1, double t2, double t) {
  Mat S(4);
  const double e1 = std::exp(-t / t1), e2 = std::exp(-t / t2);
  S(0, 0) = 1.0;
  S(0, 3) = 1.0 - e1;
  S(3, 3) = e1;
  S(1, 1) = e2;
  S(2, 2) = e2;
  return S;
}

// coherent over-rotation (reading R10): E = cos(e/2) I - i sin(e/2) A, A^2 = I
Mat overrot_unitary(int k, double eps) {
  const int d = 1 << k;
  Mat A(d);
  if (k == 1) {
    A(0, 1) = 1; A(1, 0) = 1;
  } else {  // Z on local qubit 0 (control), X on local qubit 1 (target)
    for (int i = 0; i < 4; ++i) {
      int j = i ^ 2;
      A(j, i) = (i & 1) ? -1.0 : 1.0;
    }
  }
  Mat E(d);
  const double c = std::cos(eps / 2), s = std::sin(eps / 2);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) E(i, j) = (i == j ? c : 0.0) + cd(0.0, -s) * A(i, j);
  return E;
}

// Embed a superoperator on sub-qubits (positions pos[j] within a k-qubit local space).
Mat embed_superop(const Mat& Ss, const std::vector<int>& pos, int k) {
  const int ks = (int)pos.size(), ds = 1 << ks, d = 1 << k, D = d * d;
  if (ks == k) {
    bool ident = true;
    for (int j = 0; j < k; ++j) ident &= pos[j] == j;
    if (ident) return Ss;
  }
  int mask = 0;
  for (int p : pos) mask |= 1 << p;
  auto sub = [&](int x) {
    int v = 0;
    for (int j = 0; j < ks; ++j) v |= ((x >> pos[j]) & 1) << j;
    return v;
  };
  Mat S(D);
  for (int l2 = 0; l2 < D; ++l2) {
    const int r2 = l2 & (d - 1), c2 = l2 >> k;
    for (int l = 0; l < D; ++l) {
      const int r = l & (d - 1), c = l >> k;
      if ((r2 & ~mask) != (r & ~mask) || (c2 & ~mask) != (c & ~mask)) continue;
      S(l2, l) = Ss(sub(r2) + sub(c2) * ds, sub(r) + sub(c) * ds);
    }
  }
  return S;
}

// Hermiticity preservation of a superoperator in the vec convention l = r + c d: the map
// sends X^dag to E(X)^dag iff S[(r',c'),(r,c)] = conj(S[(c',r'),(c,r)]).  Every Kraus form
// has it; user superoperators are checked.
bool is_herm_preserving(const Mat& S, int k) {
  const int d = 1 << k, D = d * d;
  for (int l2 = 0; l2 < D; ++l2)
    for (int l = 0; l < D; ++l) {
      const int t2 = (l2 % d) * d + l2 / d, t = (l % d) * d + l / d;
      const cd a = S(l2, l), b = std::conj(S(t2, t));
      if (std::abs(a - b) > 1e-14 * (1.0 + std::abs(a))) return false;
    }
  return true;
}

// ------------------------------------------------------------------------------------
// ops, fusion
// ------------------------------------------------------------------------------------
struct FusedOp {
  int k = 0;
  int q[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // k <= 3 for ops; a factored group spans <= 5 qubits
  Mat S;            // 4^k, local index over q[0..k-1] (for a factored group: the dense product)
  int parts = 1;    // number of pre-fusion ops folded in
  bool herm = true;  // Hermiticity-preserving: S[(r',c'),(r,c)] = conj S[(c',r'),(c,r)]
  std::vector<FusedOp> sub;  // k=3 factored group: sub-ops applied in order in one pass
};

// B200 cost model in units of one K1 pass over the state, calibrated with
// scripts/kbench.py at n = 16 on B200 in the packed Hermitian layout (16 B / amplitude per
// pass; profiles/r01_kbench_n16_packed.jsonl): K1 10.6 ms = 1, K2 11.6-12.2 ms (low targets,
// register stream) / 17.4-18.6 ms (a high target), ~1.4 on average; a dense k=3 op on DMMA
// 37-40 ms (3.6, FP64 bound).  A factored group costs 0.55 + 0.62 per k=2 sub-op (2 ops
// 1.70-1.92, 3 ops 2.29-2.43, 4 ops 2.95-3.05): DMMA-bound, the copies overlap.
double sep_cost(int k) { return k == 1 ? 1.0 : (k == 2 ? 1.4 : 3.6); }
double sub_cost(int k) { return k == 1 ? 0.1 : (k == 2 ? 0.62 : 3.6); }
constexpr double kGroupBase = 0.55;
double op_cost(int k) { return k <= 2 ? 1.0 : 3.6; }

bool shares(const FusedOp& a, const int* q, int k) {
  for (int i = 0; i < a.k; ++i)
    for (int j = 0; j < k; ++j)
      if (a.q[i] == q[j]) return true;
  return false;
}

// Fold G into Q (G applied after Q) on the union of their qubits.
FusedOp merge(const FusedOp& Q, const FusedOp& G) {
  FusedOp U;
  U.k = Q.k;
  for (int i = 0; i < Q.k; ++i) U.q[i] = Q.q[i];
  for (int j = 0; j < G.k; ++j) {
    bool found = false;
    for (int i = 0; i < U.k; ++i) found |= U.q[i] == G.q[j];
    if (!found) U.q[U.k++] = G.q[j];
  }
  std::vector<int> pq, pg;
  for (int i = 0; i < Q.k; ++i) pq.push_back(i);
  for (int j = 0; j < G.k; ++j)
    for (int i = 0; i < U.k; ++i)
      if (U.q[i] == G.q[j]) pg.push_back(i);
  U.S = matmul(embed_superop(G.S, pg, U.k), embed_superop(Q.S, pq, U.k));
  U.parts = Q.parts + G.parts;
  U.herm = Q.herm && G.herm;
  return U;
}

// mode 1: paper -- merge into the latest op touching the same qubits only if it
// acts on the identical ordered qubit tuple.  mode 2: greedy union up to k_max (<= 2 first,
// then 3-qubit groups kept only when the cost model says they save passes).
// 4-qubit groups (k_max = 4) run on the block kernel when they contain qubit 0 or 1 (a block
// is the group + the lowest free qubit, and its lowest 4 bits must be qubits 0 and 1 for
// 256 B contiguous pieces); other 4-qubit unions stay 3-qubit groups.  Env TANQ_QUAD_ANY=1
// allows any 4-qubit group (round-1 behaviour: those run on the cooperative tile kernel).
// k_max = 5 ("block groups"): a factored group may span up to 5 qubits when at most 3 of them
// are outside {0, 1} -- the block kernel's 5-qubit block always holds qubits 0 and 1 (its
// contiguous pieces), so sub-ops on any block qubit ride in the same HBM pass.  Members per
// block group are capped (env TANQ_BLOCK_GROUP_MAX, default 6): every k=2 sub-op adds ~10 KB
// of fragments and tables to the shared-memory blob, which costs warp pairs.
int block_group_max() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("TANQ_BLOCK_GROUP_MAX");
    v = e ? std::max(2, std::min(12, std::atoi(e))) : 6;
  }
  return v;
}
bool block_group_fits(const int* q, int k) {
  static int hmax = -1;
  if (hmax < 0) {
    const char* e = std::getenv("TANQ_BLOCK_HIGH_MAX");  // planner experiments only: the
    hmax = e ? std::max(1, std::min(3, std::atoi(e))) : 3;  // block kernel holds 3 + {0, 1}
  }
  if (k > hmax + 2) return false;
  int high = 0;
  for (int i = 0; i < k; ++i) high += q[i] >= 2 ? 1 : 0;
  return high <= hmax;
}

bool quad_ok(const int* q) {
  static int any = -1;
  if (any < 0) {
    const char* e = std::getenv("TANQ_QUAD_ANY");
    any = e && e[0] == '1' ? 1 : 0;
  }
  if (any) return true;
  for (int i = 0; i < 4; ++i)
    if (q[i] == 0 || q[i] == 1) return true;
  return false;
}

std::vector<FusedOp> fuse(const std::vector<FusedOp>& in, int mode, int kmax) {
  if (mode == 0) return in;
  auto pass = [&](const std::vector<FusedOp>& src, int klim, bool paper) {
    std::vector<FusedOp> out;
    out.reserve(src.size());
    for (const FusedOp& G : src) {
      int idx = -1;
      for (int i = (int)out.size() - 1; i >= 0; --i)
        if (shares(out[i], G.q, G.k)) {
          idx = i;
          break;
        }
      if (idx >= 0) {
        FusedOp& Q = out[idx];
        if (paper) {
          bool same = Q.k == G.k;
          for (int i = 0; same && i < G.k; ++i) same = Q.q[i] == G.q[i];
          if (same) {
            Q.S = matmul(G.S, Q.S);
            Q.parts += G.parts;
            Q.herm = Q.herm && G.herm;
            continue;
          }
        } else {
          int uk = Q.k;
          for (int j = 0; j < G.k; ++j) {
            bool f = false;
            for (int i = 0; i < Q.k; ++i) f |= Q.q[i] == G.q[j];
            if (!f) ++uk;
          }
          if (uk <= klim && op_cost(uk) <= op_cost(Q.k) + op_cost(G.k)) {
            Q = merge(Q, G);
            continue;
          }
        }
      }
      out.push_back(G);
    }
    return out;
  };
  if (mode == 1) return pass(in, 2, true);
  std::vector<FusedOp> l1 = pass(in, std::min(kmax, 2), false);
  if (kmax < 3) return l1;
  const int glim = kmax == 5 ? 8 : std::min(kmax, 4);  // group qubits (factored groups only)
  // 3-qubit grouping: greedy groups of <= 3 qubits over the k<=2 ops; a group replaces its
  // members only when their summed pass cost exceeds one dense k=3 pass.
  struct Group {
    FusedOp op;  // qubit union only (S is formed on demand)
    std::vector<int> members;
  };
  std::vector<Group> groups;
  for (int gi = 0; gi < (int)l1.size(); ++gi) {
    const FusedOp& G = l1[gi];
    int idx = -1;
    for (int i = (int)groups.size() - 1; i >= 0; --i)
      if (shares(groups[i].op, G.q, G.k)) {
        idx = i;
        break;
      }
    if (idx >= 0) {
      Group& Q = groups[idx];
      bool has3 = G.k == 3;
      for (int m : Q.members) has3 |= l1[m].k == 3;
      const int lim = has3 ? 3 : glim;  // dense k=3 sub-ops only run on 3-qubit tiles
      int uq[8], uk = Q.op.k;
      for (int i = 0; i < Q.op.k; ++i) uq[i] = Q.op.q[i];
      bool fits = true;
      for (int j = 0; j < G.k && fits; ++j) {
        bool f = false;
        for (int i = 0; i < uk; ++i) f |= uq[i] == G.q[j];
        if (!f) {
          if (uk >= lim) fits = false; else uq[uk++] = G.q[j];
        }
      }
      if (uk > lim) fits = false;  // a dense k=3 op never joins a 4-qubit group
      if (kmax == 5) {
        if (fits && uk >= 4 && (!block_group_fits(uq, uk) ||
                                (int)Q.members.size() + 1 > block_group_max()))
          fits = false;
      } else if (fits && uk == 4 && !quad_ok(uq)) {
        fits = false;
      }
      if (fits) {
        Q.op.k = uk;
        for (int i = 0; i < uk; ++i) Q.op.q[i] = uq[i];
        Q.members.push_back(gi);
        continue;
      }
    }
    Group g;
    g.op.k = G.k;
    for (int i = 0; i < G.k; ++i) g.op.q[i] = G.q[i];
    g.members.push_back(gi);
    groups.push_back(std::move(g));
  }
  // Forward merge (post-pass): a group may move LATER, past groups disjoint from its qubits,
  // into the first later group that shares a qubit with it, when their union still fits a
  // tile.  Its members run first (they precede, or commute with, every member of the target:
  // a member sharing a qubit with the target would have joined the target, the latest sharing
  // group).  A k=2 op left standalone because the group before it was full then rides in the
  // next group's pass instead of costing its own HBM pass.  Env TANQ_FWD_MERGE=0 disables.
  static int fwd = -1;
  if (fwd < 0) {
    const char* e = std::getenv("TANQ_FWD_MERGE");
    fwd = e && e[0] == '0' ? 0 : 1;
  }
  for (size_t i = 0; fwd && i < groups.size(); ++i) {
    Group& A = groups[i];
    if (A.members.empty()) continue;
    for (size_t j = i + 1; j < groups.size(); ++j) {
      Group& B = groups[j];
      if (B.members.empty() || !shares(B.op, A.op.q, A.op.k)) continue;
      bool has3 = false;
      for (int m : A.members) has3 |= l1[m].k == 3;
      for (int m : B.members) has3 |= l1[m].k == 3;
      const int lim = has3 ? 3 : glim;
      int uq[16], uk = B.op.k;
      for (int t = 0; t < B.op.k; ++t) uq[t] = B.op.q[t];
      for (int t = 0; t < A.op.k; ++t) {
        bool f = false;
        for (int u = 0; u < uk; ++u) f |= uq[u] == A.op.q[t];
        if (!f) uq[uk++] = A.op.q[t];
      }
      const bool ok4 = kmax == 5 ? (uk < 4 || (block_group_fits(uq, uk) &&
                                               (int)(A.members.size() + B.members.size()) <=
                                                   block_group_max()))
                                 : (uk < 4 || quad_ok(uq));
      if (uk <= lim && uk >= 3 && ok4) {  // (k <= 2 unions: level 1)
        B.op.k = uk;
        for (int t = 0; t < uk; ++t) B.op.q[t] = uq[t];
        B.members.insert(B.members.begin(), A.members.begin(), A.members.end());
        A.members.clear();
      }
      break;  // only the first later group sharing a qubit may absorb A
    }
  }
  // the dense superoperator of a group on its union (members applied in order)
  auto dense_of = [&](const Group& g) {
    FusedOp acc = l1[g.members[0]];
    for (size_t i = 1; i < g.members.size(); ++i) acc = merge(acc, l1[g.members[i]]);
    // re-express on the group's qubit order
    std::vector<int> pos;
    for (int j = 0; j < acc.k; ++j)
      for (int i = 0; i < g.op.k; ++i)
        if (g.op.q[i] == acc.q[j]) pos.push_back(i);
    FusedOp out = g.op;
    out.S = embed_superop(acc.S, pos, g.op.k);
    out.parts = acc.parts;
    out.herm = acc.herm;
    return out;
  };
  std::vector<FusedOp> out;
  for (Group& g : groups) {
    if (g.members.empty()) continue;  // moved into a later group
    if (g.members.size() == 1 || g.op.k < 3) {  // k<=2 unions were merged by level 1
      for (int m : g.members) out.push_back(l1[m]);
      continue;
    }
    double sep = 0, fact = 0;
    size_t prog = 0;
    for (int m : g.members) {
      sep += sep_cost(l1[m].k);
      fact += sub_cost(l1[m].k);
      prog += l1[m].k == 3 ? 4096 : (l1[m].k == 2 ? 256 : 16);
    }
    fact = std::max(1.0, kGroupBase + fact);
    const double dense = g.op.k == 3 ? sep_cost(3) : 1e30;
    const bool fact_ok = g.members.size() <= (size_t)tanq::kMaxSub &&
                         prog <= (size_t)tanq::kGroupProgMax;
    if (fact_ok && fact <= dense && fact < sep) {
      FusedOp f = g.op;  // factored: S formed only on export (tanq_plan_get_op)
      for (int m : g.members) {
        f.sub.push_back(l1[m]);
        f.herm = f.herm && l1[m].herm;
      }
      out.push_back(std::move(f));
    } else if (dense < sep) {
      out.push_back(dense_of(g));
    } else {
      for (int m : g.members) out.push_back(l1[m]);
    }
  }
  return out;
}

struct Prof {
  int cls;
  cudaEvent_t e0, e1;
  double bytes, flops, hw_flops;
};
constexpr int kProfClasses = 5;
const char* kProfNames[kProfClasses] = {"gate_k1", "gate_k2", "group_dmma", "remap", "unpack"};

}  // namespace

// ------------------------------------------------------------------------------------
// the simulator handle
// ------------------------------------------------------------------------------------
struct Shard {
  int id = 0;          // global shard id
  int device = 0;
  cudaStream_t stream = nullptr;
  double2* data = nullptr;
  bool external = false;  // caller-owned buffer (tanq_create_ex): never freed here
};

struct DevScratch {
  int device = -1;
  double* probs = nullptr;        // 2^n
  double* probs_tmp = nullptr;    // 2^n (multi-device combine)
  double* cdf = nullptr;          // 2^n
  double2* partial = nullptr;     // expect partial sums
  double2* scal = nullptr;        // 2 double2
  unsigned long long* imax = nullptr;
  double2* stage = nullptr;       // get/set_state staging
  size_t stage_elems = 0;
  double2* frag = nullptr;        // k=3 fragment buffer
  size_t frag_elems = 0;
};

struct tanq_plan;
struct PlanCacheEntry {
  std::string key;       // exact serialisation of circuit + noise model + options
  tanq_plan* plan = nullptr;
  uint64_t hits = 0;
  uint64_t last_use = 0;
};

struct tanq_sim {
  int n = 0, L = 0, world = 1, rank0 = 0;
  bool dist = false;
  std::vector<Shard> shards;
  std::vector<DevScratch> scratch;  // per distinct device
  uint32_t phys[64];                // logical bit (2q row, 2q+1 col) -> physical bit
  uint64_t par = 0;                 // parity layout: half-global qubits (phys[2h+1] is a global
                                    // bit holding r_h XOR c_h, phys[2h] the local row bit)
  bool parity = false;              // shard-local parity layout, world > 1
  ncclComm_t comm = nullptr;
  double2* xsend = nullptr;         // 2 staging slots of xchunk elements (send)
  double2* xrecv = nullptr;         // 2 staging slots (receive)
  size_t xchunk = 0;
  cudaStream_t xstream = nullptr;   // NCCL stream of the pipelined exchange
  cudaEvent_t xev_pack[2] = {nullptr, nullptr}, xev_comm[2] = {nullptr, nullptr};
  bool prof_on = false;
  std::vector<Prof> prof;
  std::vector<cudaEvent_t> event_pool;  // recycled timing events (no create per launch)
  bool herm_state = true;   // rho known Hermitian (create / reset; cleared by set_state and
                            // by non-Hermiticity-preserving ops; tanq_check_hermitian sets it)
  bool mirror_allowed = true;  // env TANQ_MIRROR=0 disables the packed Hermitian mode
  bool packed = false;      // packed Hermitian layout: only e >= pair_swap(e) is up to date
  double prof_ms[kProfClasses] = {};
  double prof_bytes[kProfClasses] = {};
  double prof_flops[kProfClasses] = {};
  double prof_hw_flops[kProfClasses] = {};
  uint64_t prof_launches[kProfClasses] = {};
  uint64_t launches = 0;
  uint64_t remap_count = 0, remap_bytes = 0;
  std::vector<std::pair<int, cudaStream_t>> owned;  // library-created stream per device
  double2* frag_host = nullptr;                      // pinned staging of k=3 fragments
  size_t frag_host_elems = 0;
  cudaEvent_t frag_done = nullptr;
  bool frag_done_pending = false;
  std::vector<PlanCacheEntry> plan_cache;  // tanq_run_circuit: recently run circuits
  uint64_t plan_cache_clock = 0;
  cudaStream_t own_streams_of(int dev) const {
    for (auto& p : owned)
      if (p.first == dev) return p.second;
    return nullptr;
  }
};

namespace {

DevScratch& scratch_for(tanq_sim* s, int device) {
  for (auto& d : s->scratch)
    if (d.device == device) return d;
  s->scratch.push_back(DevScratch{});
  s->scratch.back().device = device;
  return s->scratch.back();
}

tanq_status ensure_scratch(tanq_sim* s, DevScratch& d) {
  if (d.probs) return TANQ_OK;
  CUDA_TRY(cudaSetDevice(d.device));
  const size_t N = (size_t)1 << s->n;
  CUDA_TRY(cudaMalloc(&d.probs, N * sizeof(double)));
  CUDA_TRY(cudaMalloc(&d.probs_tmp, N * sizeof(double)));
  CUDA_TRY(cudaMalloc(&d.cdf, N * sizeof(double)));
  CUDA_TRY(cudaMalloc(&d.partial, 148 * 4 * sizeof(double2)));
  CUDA_TRY(cudaMalloc(&d.scal, 2 * sizeof(double2)));
  CUDA_TRY(cudaMalloc(&d.imax, sizeof(unsigned long long)));
  d.stage_elems = (size_t)1 << 21;  // 32 MiB
  CUDA_TRY(cudaMalloc(&d.stage, d.stage_elems * sizeof(double2)));
  return TANQ_OK;
}

int ilog2_(int x) {
  int l = 0;
  while ((1 << l) < x) ++l;
  return l;
}

tanq::BitMap bitmap_of(const tanq_sim* s) {
  tanq::BitMap bm;
  bm.nbits = 2 * s->n;
  for (int i = 0; i < 64; ++i) bm.phys[i] = s->phys[i];
  bm.par = s->par;
  return bm;
}

// Multi-shard layout.  env TANQ_LAYOUT=bits: the round-1 layout (identity bit
// map, the top log2 G physical bits -- row / col bits of the top qubits -- select the shard,
// transpose pairs cross shards, so multi-shard runs cannot use the packed Hermitian layout).
// Default: the shard-local parity layout -- the top g = log2 G qubits are half-global: qubit
// h's global bit holds r_h XOR c_h (invariant under transpose, so every transpose pair stays
// on its shard) and its row bit is local, above the aligned (row, col) pairs of the n - g
// fully local qubits.
// It needs n - g >= 5 fully local qubits (a 4-qubit op on a half-global qubit still finds a
// victim); smaller registers keep the bit layout.
bool parity_layout_for(int n, int world) {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("TANQ_LAYOUT");
    v = e && !std::strcmp(e, "bits") ? 0 : 1;
  }
  int g = 0;
  while ((1 << g) < world) ++g;
  return v == 1 && world > 1 && n - g >= 5;
}

void init_layout(uint32_t* phys, uint64_t& par, int n, int g, bool parity) {
  for (int i = 0; i < 64; ++i) phys[i] = (uint32_t)i;  // rowpos(q)=2q, colpos(q)=2q+1
  par = 0;
  if (!parity || g == 0) return;
  const int F = n - g, L = 2 * n - g;
  for (int i = 0; i < g; ++i) {
    const int h = F + i;
    phys[2 * h] = (uint32_t)(2 * F + i);  // local row bit above the pairs
    phys[2 * h + 1] = (uint32_t)(L + i);  // global parity bit
    par |= 1ull << h;
  }
}

void reset_layout(tanq_sim* s) {
  init_layout(s->phys, s->par, s->n, ilog2_(s->world), s->parity);
}

// Transpose descriptor of shard `id` (tanq::TDesc): pairs below 2 (n - g) in the parity
// layout; the half-global row bits flip where the shard's parity bit is 1.
tanq::TDesc tdesc_of(const tanq_sim* s, int id) {
  tanq::TDesc td;
  if (!s->par) return td;
  const int g = __builtin_popcountll(s->par);
  td.lo = ((uint64_t)1 << (2 * (s->n - g))) - 1;
  for (uint64_t h = s->par; h; h &= h - 1) {
    const int q = __builtin_ctzll(h);
    if ((id >> (s->phys[2 * q + 1] - s->L)) & 1) td.m |= (uint64_t)1 << s->phys[2 * q];
  }
  return td;
}

tanq_status host_wait(tanq_sim* s, cudaStream_t st);

// wait for all shards' streams (cross-stream / cross-device ordering point)
tanq_status join_all(tanq_sim* s) {
  for (auto& sh : s->shards) {
    CUDA_TRY(cudaSetDevice(sh.device));
    TRY(host_wait(s, sh.stream));
  }
  return TANQ_OK;
}

tanq_status stream_wait(const Shard& waiter, const Shard& on) {
  if (waiter.stream == on.stream) return TANQ_OK;
  cudaEvent_t ev;
  CUDA_TRY(cudaSetDevice(on.device));
  CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(ev, on.stream));
  CUDA_TRY(cudaSetDevice(waiter.device));
  CUDA_TRY(cudaStreamWaitEvent(waiter.stream, ev, 0));
  CUDA_TRY(cudaEventDestroy(ev));
  return TANQ_OK;
}

cudaEvent_t pooled_event(tanq_sim* s) {
  if (!s->event_pool.empty()) {
    cudaEvent_t e = s->event_pool.back();
    s->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void prof_begin(tanq_sim* s, Shard& sh, Prof& p) {
  if (!s->prof_on || sh.id != s->rank0) return;
  p.e0 = pooled_event(s);
  p.e1 = pooled_event(s);
  cudaEventRecord(p.e0, sh.stream);
}
void prof_end(tanq_sim* s, Shard& sh, Prof& p) {
  if (!s->prof_on || sh.id != s->rank0) return;
  cudaEventRecord(p.e1, sh.stream);
  s->prof.push_back(p);
}

// Swap physical bit a (global, a >= L) with local bit b (A-6).
tanq_status ensure_unpacked(tanq_sim* s);

// Chunked exchange of `total` elements with `peer` through 2 x 2 staging slots, pipelined
// (SURVEY NEXT-2 overlap): pack / unpack kernels run on the shard's stream, the grouped
// send/recv on s->xstream, so chunk i's transfer overlaps chunk i-1's unpack and chunk i+1's
// pack.  Stream S: pack0 pack1 | unpack0 pack2 | unpack1 pack3 ...; stream X: comm0 comm1 ...
// Ordering: comm(i) waits pack(i) (event xev_pack[j]); unpack(i) waits comm(i) (xev_comm[j]);
// pack(i+2) reuses slot j after unpack(i) on S, so slot reuse is ordered by S itself.
// In place: pack(i) reads chunk i of the outgoing part before unpack(i) overwrites it (S order).
// Host wait for a stream.  Multi-process handles poll instead of blocking: every NCCL call is
// asynchronous, so a peer that died or a broken link shows up only as a stream that never
// completes (the paper saw fine-grained remote access hang the fabric).  The poll
// checks ncclCommGetAsyncError and gives up after TANQ_NCCL_TIMEOUT_S seconds (default 600),
// aborting the communicator and returning TANQ_E_NCCL instead of hanging the process.
tanq_status host_wait(tanq_sim* s, cudaStream_t st) {
  if (!s->comm) {
    CUDA_TRY(cudaStreamSynchronize(st));
    return TANQ_OK;
  }
  static double timeout_s = -1;
  if (timeout_s < 0) {
    const char* e = getenv("TANQ_NCCL_TIMEOUT_S");
    timeout_s = e ? std::atof(e) : 600.0;
    if (timeout_s <= 0) timeout_s = 600.0;
  }
  cudaEvent_t ev;
  CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  cudaError_t ce = cudaEventRecord(ev, st);
  if (ce != cudaSuccess) {
    cudaEventDestroy(ev);
    return fail(TANQ_E_CUDA, std::string("cudaEventRecord -> ") + cudaGetErrorString(ce));
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned it = 0;; ++it) {
    ce = cudaEventQuery(ev);
    if (ce == cudaSuccess) break;
    if (ce != cudaErrorNotReady) {
      cudaEventDestroy(ev);
      return fail(TANQ_E_CUDA, std::string("stream wait -> ") + cudaGetErrorString(ce));
    }
    ncclResult_t ar = ncclSuccess;
    if (nccl().CommGetAsyncError && nccl().CommGetAsyncError(s->comm, &ar) == ncclSuccess &&
        ar != ncclSuccess && ar != ncclInProgress) {
      cudaEventDestroy(ev);
      if (nccl().CommAbort) nccl().CommAbort(s->comm);
      s->comm = nullptr;
      return fail(TANQ_E_NCCL, std::string("NCCL asynchronous error: ") + nccl().GetErrorString(ar));
    }
    const double el =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > timeout_s) {
      cudaEventDestroy(ev);
      if (nccl().CommAbort) nccl().CommAbort(s->comm);
      s->comm = nullptr;
      return fail(TANQ_E_NCCL, "stream did not complete within TANQ_NCCL_TIMEOUT_S (" +
                                   std::to_string(timeout_s) + " s): peer or link failure; "
                                   "communicator aborted");
    }
    if (it > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  cudaEventDestroy(ev);
  return TANQ_OK;
}

template <class Pack, class Unpack>
tanq_status exchange_pipelined(tanq_sim* s, Shard& sh, int peer, uint64_t total, Pack pack,
                               Unpack unpack) {
  const uint64_t C = s->xchunk, nch = (total + C - 1) / C;
  auto cnt_of = [&](uint64_t i) { return std::min<uint64_t>(C, total - i * C); };
  for (uint64_t i = 0; i < std::min<uint64_t>(2, nch); ++i) {
    CUDA_TRY(pack(i * C, cnt_of(i), s->xsend + (i & 1) * C));
    CUDA_TRY(cudaEventRecord(s->xev_pack[i & 1], sh.stream));
    s->launches++;
  }
  for (uint64_t i = 0; i < nch; ++i) {
    const int j = (int)(i & 1);
    const uint64_t cnt = cnt_of(i);
    CUDA_TRY(cudaStreamWaitEvent(s->xstream, s->xev_pack[j], 0));
    NCCL_TRY(nccl().GroupStart());
    NCCL_TRY(nccl().Send(s->xsend + j * C, cnt * 2, ncclDouble, peer, s->comm, s->xstream));
    NCCL_TRY(nccl().Recv(s->xrecv + j * C, cnt * 2, ncclDouble, peer, s->comm, s->xstream));
    NCCL_TRY(nccl().GroupEnd());
    CUDA_TRY(cudaEventRecord(s->xev_comm[j], s->xstream));
    CUDA_TRY(cudaStreamWaitEvent(sh.stream, s->xev_comm[j], 0));
    CUDA_TRY(unpack(i * C, cnt, s->xrecv + j * C));
    s->launches++;
    if (i + 2 < nch) {
      CUDA_TRY(pack((i + 2) * C, cnt_of(i + 2), s->xsend + j * C));
      CUDA_TRY(cudaEventRecord(s->xev_pack[j], sh.stream));
      s->launches++;
    }
    s->remap_bytes += cnt * sizeof(double2);
  }
  return TANQ_OK;
}

tanq_status remap_swap(tanq_sim* s, int a, int b) {
  TRY(ensure_unpacked(s));  // (packed mode is single-shard only; kept for safety)
  const int L = s->L, gb = a - L;
  const uint64_t half = (uint64_t)1 << (L - 1);
  if (!s->dist) {
    for (auto& sh : s->shards) {
      const int g = sh.id;
      if ((g >> gb) & 1) continue;
      const int g2 = g ^ (1 << gb);
      Shard* other = nullptr;
      for (auto& o : s->shards)
        if (o.id == g2) other = &o;
      TRY(stream_wait(sh, *other));
      CUDA_TRY(cudaSetDevice(sh.device));
      const int va = 1 - ((g >> gb) & 1), vb = 1 - ((g2 >> gb) & 1);
      // algorithmic bytes: both exchanged halves read and written once
      Prof pr{3, nullptr, nullptr, 4.0 * half * sizeof(double2), 0.0, 0.0};
      prof_begin(s, sh, pr);
      CUDA_TRY(tanq::launch_swap_halves(sh.data, other->data, L, b, va, vb, sh.stream));
      prof_end(s, sh, pr);
      s->launches++;
      TRY(stream_wait(*other, sh));
      s->remap_bytes += half * sizeof(double2);
    }
  } else {
    Shard& sh = s->shards[0];
    const int g = sh.id, g2 = g ^ (1 << gb);
    const int v = 1 - ((g >> gb) & 1);
    CUDA_TRY(cudaSetDevice(sh.device));
    // bytes = the half sent + the half received over NVLink
    Prof pr{3, nullptr, nullptr, 2.0 * half * sizeof(double2), 0.0, 0.0};
    prof_begin(s, sh, pr);
    TRY(exchange_pipelined(
        s, sh, g2, half,
        [&](uint64_t first, uint64_t cnt, double2* buf) {
          return tanq::launch_pack_half(sh.data, buf, b, v, first, cnt, sh.stream);
        },
        [&](uint64_t first, uint64_t cnt, const double2* buf) {
          return tanq::launch_unpack_half(sh.data, buf, b, v, first, cnt, sh.stream);
        }));
    prof_end(s, sh, pr);
  }
  // bookkeeping: logical bits at a and b exchange positions
  for (int i = 0; i < 2 * s->n; ++i) {
    if (s->phys[i] == (uint32_t)a)
      s->phys[i] = (uint32_t)b;
    else if (s->phys[i] == (uint32_t)b)
      s->phys[i] = (uint32_t)a;
  }
  s->remap_count++;
  return TANQ_OK;
}

bool batch_remaps() {  // env TANQ_REMAP_BATCH=0: two pairwise exchanges instead
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("TANQ_REMAP_BATCH");
    v = e && e[0] == '0' ? 0 : 1;
  }
  return v == 1;
}

// Two swaps (a0 <-> b0, a1 <-> b1; a0 != a1 global, b0 != b1 local) as ONE exchange in the
// multi-process mode: after both swaps an element with local bits (l0, l1) at
// (b0, b1) lives on the shard whose bits (a0, a1) are (l0, l1), at local bits (b0, b1) = this
// shard's (g0, g1).  So the quarter with (l0, l1) = (g0, g1) stays, and for each of the 3
// peers h: this shard's quarter (l0, l1) = (h0, h1) goes to h and h's quarter (g0, g1) lands in
// its place.  3/4 of the shard crosses NVLink instead of 2 x 1/2 for two pairwise swaps; the
// result is identical to the two swaps in sequence (same bit map).
tanq_status remap_swap2(tanq_sim* s, int a0, int b0, int a1, int b1) {
  if (!s->dist || a0 == a1 || b0 == b1) {
    TRY(remap_swap(s, a0, b0));
    return remap_swap(s, a1, b1);
  }
  TRY(ensure_unpacked(s));
  const int L = s->L;
  Shard& sh = s->shards[0];
  const int g = sh.id, ga0 = a0 - L, ga1 = a1 - L;
  // order the local bits for the quarter kernels (values travel with their bits)
  const bool sw = b0 > b1;
  const int lb0 = sw ? b1 : b0, lb1 = sw ? b0 : b1;
  const uint64_t quarter = (uint64_t)1 << (L - 2);
  CUDA_TRY(cudaSetDevice(sh.device));
  Prof pr{3, nullptr, nullptr, 2.0 * 3.0 * quarter * sizeof(double2), 0.0, 0.0};
  prof_begin(s, sh, pr);
  // step d pairs every shard with g ^ (d on bits ga0, ga1): mutual partners at every step, so
  // the grouped send/recv rendezvous cannot form a cycle
  for (int d = 1; d < 4; ++d) {
    const int h0 = ((g >> ga0) & 1) ^ (d & 1), h1 = ((g >> ga1) & 1) ^ (d >> 1);
    const int peer = (g & ~((1 << ga0) | (1 << ga1))) | (h0 << ga0) | (h1 << ga1);
    const int v0 = sw ? h1 : h0, v1 = sw ? h0 : h1;  // bit values at lb0 < lb1
    TRY(exchange_pipelined(
        s, sh, peer, quarter,
        [&](uint64_t first, uint64_t cnt, double2* buf) {
          return tanq::launch_pack_quarter(sh.data, buf, lb0, v0, lb1, v1, first, cnt, sh.stream);
        },
        [&](uint64_t first, uint64_t cnt, const double2* buf) {
          return tanq::launch_unpack_quarter(sh.data, buf, lb0, v0, lb1, v1, first, cnt,
                                             sh.stream);
        }));
  }
  prof_end(s, sh, pr);
  for (auto [a, b] : {std::pair<int, int>{a0, b0}, std::pair<int, int>{a1, b1}}) {
    for (int i = 0; i < 2 * s->n; ++i) {
      if (s->phys[i] == (uint32_t)a)
        s->phys[i] = (uint32_t)b;
      else if (s->phys[i] == (uint32_t)b)
        s->phys[i] = (uint32_t)a;
    }
    s->remap_count++;
  }
  return TANQ_OK;
}

void apply_parity_remap(uint32_t* phys, uint64_t& par, int h, int v);

// Parity-layout remap: half-global qubit h becomes fully local in the pair of
// the fully local qubit v, which becomes half-global.  Half of every shard crosses to the
// partner shard (the one differing in h's global bit); a quarter moves inside the shard.
tanq_status remap_parity(tanq_sim* s, int h, int v) {
  TRY(ensure_unpacked(s));
  const int L = s->L;
  const int x = (int)s->phys[2 * h], a = (int)s->phys[2 * h + 1];
  const int y = (int)s->phys[2 * v], z = (int)s->phys[2 * v + 1], gb = a - L;
  const uint64_t half = (uint64_t)1 << (L - 1);
  if (!s->dist) {
    for (auto& sh : s->shards) {
      const int g = sh.id;
      if ((g >> gb) & 1) continue;
      const int g2 = g ^ (1 << gb);
      Shard* other = nullptr;
      for (auto& o : s->shards)
        if (o.id == g2) other = &o;
      TRY(stream_wait(sh, *other));
      CUDA_TRY(cudaSetDevice(sh.device));
      // both shards read once, 3/4 of them written
      Prof pr{3, nullptr, nullptr, 3.5 * (double)((uint64_t)1 << L) * sizeof(double2), 0.0, 0.0};
      prof_begin(s, sh, pr);
      CUDA_TRY(tanq::launch_parity_swap(sh.data, other->data, L, x, y, z, sh.stream));
      prof_end(s, sh, pr);
      s->launches++;
      TRY(stream_wait(*other, sh));
      s->remap_bytes += half * sizeof(double2);
    }
  } else {
    Shard& sh = s->shards[0];
    const int g = sh.id, g2 = g ^ (1 << gb), sa = (g >> gb) & 1;
    CUDA_TRY(cudaSetDevice(sh.device));
    Prof pr{3, nullptr, nullptr, 2.0 * half * sizeof(double2), 0.0, 0.0};
    prof_begin(s, sh, pr);
    CUDA_TRY(tanq::launch_parity_stay(sh.data, L, x, y, z, sa, sh.stream));
    s->launches++;
    TRY(exchange_pipelined(
        s, sh, g2, half,
        [&](uint64_t first, uint64_t cnt, double2* buf) {
          return tanq::launch_parity_pack(sh.data, buf, L, x, y, z, sa, first, cnt, sh.stream);
        },
        [&](uint64_t first, uint64_t cnt, const double2* buf) {
          return tanq::launch_parity_unpack(sh.data, buf, L, x, y, z, sa, first, cnt, sh.stream);
        }));
    prof_end(s, sh, pr);
  }
  apply_parity_remap(s->phys, s->par, h, v);
  s->remap_count++;
  return TANQ_OK;
}

// Victim for a remap (pure layout logic, shared by execution and tanq_plan_schedule): a local
// bit not targeted by the op whose qubit is used furthest in the future (lookahead 256 ops
// over `next` from `next_from`), ties to the highest position.  -1 if none.
int choose_victim(const uint32_t* phys, int n, int L, const std::vector<int>& tgt,
                  const std::vector<FusedOp>* next, size_t next_from) {
  int best = -1;
  long best_dist = -1;
  for (int b = L - 1; b >= 0; --b) {
    int lid = -1;
    for (int i = 0; i < 2 * n; ++i)
      if (phys[i] == (uint32_t)b) lid = i;
    if (std::find(tgt.begin(), tgt.end(), lid) != tgt.end()) continue;
    const int lq = lid / 2;
    long dist = 1L << 40;
    if (next) {
      for (size_t t = next_from; t < next->size() && t < next_from + 256; ++t) {
        const FusedOp& f = (*next)[t];
        bool uses = false;
        for (int j = 0; j < f.k; ++j) uses |= f.q[j] == lq;
        if (uses) {
          dist = (long)(t - next_from);
          break;
        }
      }
    }
    if (dist > best_dist) {
      best_dist = dist;
      best = b;
    }
  }
  return best;
}

// A remap step.  kind 1 (bit layout): swap global bit a with local bit b.  kind 2 (parity
// layout): half-global qubit a and fully local qubit b trade places.
struct Remap {
  int kind, a, b;
};

// Parity-layout victim: a fully local qubit the op does not target whose next use is furthest
// (lookahead 256 ops), ties to the highest pair.  -1 if none.
int choose_victim_qubit(const uint32_t* phys, uint64_t par, int n, const FusedOp& op,
                        const std::vector<FusedOp>* next, size_t next_from) {
  int best = -1;
  long best_dist = -1;
  uint32_t best_pos = 0;
  for (int q = 0; q < n; ++q) {
    if ((par >> q) & 1) continue;
    bool tgt = false;
    for (int j = 0; j < op.k; ++j) tgt |= op.q[j] == q;
    if (tgt) continue;
    long dist = 1L << 40;
    if (next) {
      for (size_t t = next_from; t < next->size() && t < next_from + 256; ++t) {
        const FusedOp& f = (*next)[t];
        bool uses = false;
        for (int j = 0; j < f.k; ++j) uses |= f.q[j] == q;
        if (uses) {
          dist = (long)(t - next_from);
          break;
        }
      }
    }
    if (dist > best_dist || (dist == best_dist && phys[2 * q] > best_pos)) {
      best_dist = dist;
      best = q;
      best_pos = phys[2 * q];
    }
  }
  return best;
}

// Bookkeeping of a parity remap: qubit h takes v's (row, col) pair, v's row bit goes to h's
// local row slot and its parity to h's global bit.
void apply_parity_remap(uint32_t* phys, uint64_t& par, int h, int v) {
  const uint32_t x = phys[2 * h], a = phys[2 * h + 1], y = phys[2 * v], z = phys[2 * v + 1];
  phys[2 * h] = y;
  phys[2 * h + 1] = z;
  phys[2 * v] = x;
  phys[2 * v + 1] = a;
  par ^= ((uint64_t)1 << h) | ((uint64_t)1 << v);
}

// The remaps that make op `op` local, applied to (phys, par) in order ({-1, ..} on failure).
std::vector<Remap> plan_remaps(uint32_t* phys, uint64_t& par, int n, int L, const FusedOp& op,
                               const std::vector<FusedOp>* next, size_t next_from) {
  std::vector<Remap> out;
  if (par) {
    for (int j = 0; j < op.k; ++j) {
      const int h = op.q[j];
      if (!((par >> h) & 1)) continue;
      const int v = choose_victim_qubit(phys, par, n, op, next, next_from);
      if (v < 0) return {{-1, -1, -1}};
      out.push_back({2, h, v});
      apply_parity_remap(phys, par, h, v);
    }
    return out;
  }
  std::vector<int> tgt;
  for (int j = 0; j < op.k; ++j) {
    tgt.push_back(2 * op.q[j]);
    tgt.push_back(2 * op.q[j] + 1);
  }
  for (int id : tgt) {
    const int a = (int)phys[id];
    if (a < L) continue;
    const int b = choose_victim(phys, n, L, tgt, next, next_from);
    if (b < 0) return {{-1, -1, -1}};
    out.push_back({1, a, b});
    for (int i = 0; i < 2 * n; ++i) {
      if (phys[i] == (uint32_t)a)
        phys[i] = (uint32_t)b;
      else if (phys[i] == (uint32_t)b)
        phys[i] = (uint32_t)a;
    }
  }
  return out;
}

// Make every target bit of `op` local on the device (remap_swap per planned swap).
tanq_status ensure_local(tanq_sim* s, const FusedOp& op, const std::vector<FusedOp>* next,
                         size_t next_from) {
  uint32_t phys[64];
  std::memcpy(phys, s->phys, sizeof(phys));
  uint64_t par = s->par;
  auto swaps = plan_remaps(phys, par, s->n, s->L, op, next, next_from);
  for (auto& r : swaps)
    if (r.kind < 0) return fail(TANQ_E_ARG, "no local qubit available for remap");
  if (s->par) {
    for (auto& r : swaps) TRY(remap_parity(s, r.a, r.b));
    return TANQ_OK;
  }
  // swaps are independent (distinct global and distinct local bits): batch them in pairs
  size_t i = 0;
  if (s->dist && batch_remaps())
    for (; i + 1 < swaps.size(); i += 2)
      TRY(remap_swap2(s, swaps[i].a, swaps[i].b, swaps[i + 1].a, swaps[i + 1].b));
  for (; i < swaps.size(); ++i) TRY(remap_swap(s, swaps[i].a, swaps[i].b));
  return TANQ_OK;
}

tanq_status prof_flush(tanq_sim* s) {
  if (s->prof.empty()) return TANQ_OK;
  TRY(join_all(s));
  for (Prof& p : s->prof) {
    float ms = 0;
    cudaEventElapsedTime(&ms, p.e0, p.e1);
    s->prof_ms[p.cls] += ms;
    s->prof_bytes[p.cls] += p.bytes;
    s->prof_flops[p.cls] += p.flops;
    s->prof_hw_flops[p.cls] += p.hw_flops;
    s->prof_launches[p.cls]++;
    s->event_pool.push_back(p.e0);
    s->event_pool.push_back(p.e1);
  }
  s->prof.clear();
  return TANQ_OK;
}

// Member order of an op on the current layout: member bit t <-> the t-th lowest physical
// target bit; l_of[i] = paper local vec index (r + c 2^k) of member i.
struct MemberMap {
  std::vector<std::pair<int, int>> bits;  // sorted (physical pos, paper-index bit)
  std::vector<int> l_of;
};

MemberMap member_map(const tanq_sim* s, int k, const int* q) {
  MemberMap mm;
  for (int j = 0; j < k; ++j) {
    mm.bits.push_back({(int)s->phys[2 * q[j]], j});
    mm.bits.push_back({(int)s->phys[2 * q[j] + 1], k + j});
  }
  std::sort(mm.bits.begin(), mm.bits.end());
  const int M = 1 << (2 * k);
  mm.l_of.resize(M);
  for (int i = 0; i < M; ++i) {
    int l = 0;
    for (int t = 0; t < 2 * k; ++t)
      if ((i >> t) & 1) l |= 1 << mm.bits[t].second;
    mm.l_of[i] = l;
  }
  return mm;
}

std::vector<double2> member_order_S(const FusedOp& op, const MemberMap& mm) {
  const int M = 1 << (2 * op.k);
  std::vector<double2> out((size_t)M * M);
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < M; ++j) {
      const cd v = op.S(mm.l_of[i], mm.l_of[j]);
      out[(size_t)i * M + j] = make_double2(v.real(), v.imag());
    }
  return out;
}

// Packed Hermitian mode: rho known Hermitian, op Hermiticity-preserving, one
// shard with the initial interleaved layout (row/col bits of every qubit adjacent, so the
// transpose of element e is pair_swap(e)), whole 16-tuple blocks.
// Several shards: the shard-local parity layout, whose transpose pairs never
// leave their shard; every kernel's in-tile bits (targets + lowest free qubits, at most 6
// qubits) must lie below the pair boundary, so at least 6 fully local qubits.
bool use_mirror(const tanq_sim* s, const FusedOp& op) {
  if (!s->mirror_allowed || !s->herm_state || !op.herm) return false;
  if (s->par) {
    if (s->n - __builtin_popcountll(s->par) < 6) return false;
  } else {
    if (s->shards.size() != 1 || s->dist) return false;
    for (int i = 0; i < 2 * s->n; ++i)
      if (s->phys[i] != (uint32_t)i) return false;
  }
  const int tuple_bits = s->L - 2 * op.k;  // groups: op.k = tile qubits (3 or 4)
  return op.k == 1 ? tuple_bits >= 2 : tuple_bits >= 4;
}

// k = 2 ops whose targets all sit at physical position >= 6 run as 2-qubit cooperative tiles
// (tile_kernel<2>: 512 B contiguous copies); the register-streaming gate2_mma_kernel reads
// 8 tuples = 128 B runs per member there (microbench/locality.cu).  Env TANQ_K2PATH =
// direct | tile | auto (default).
bool k2_tiled(const tanq_sim* s, const FusedOp& op) {
  static int mode = -1;
  if (mode < 0) {
    const char* e = std::getenv("TANQ_K2PATH");
    mode = e && !std::strcmp(e, "direct") ? 0 : (e && !std::strcmp(e, "tile") ? 1 : 2);
  }
  if (op.k != 2 || mode == 0) return false;
  if (mode == 1) return true;
  int lo = 64, hi = 0;
  for (int j = 0; j < 2; ++j) {
    lo = std::min(lo, (int)std::min(s->phys[2 * op.q[j]], s->phys[2 * op.q[j] + 1]));
    hi = std::max(hi, (int)std::max(s->phys[2 * op.q[j]], s->phys[2 * op.q[j] + 1]));
  }
  // packed layout: the register stream keeps its in-place fast path only when every target is
  // low (a high target makes every element's placement depend on the member bits)
  if (use_mirror(s, op)) return hi >= 6;
  return lo >= 6;
}

// ops launched through the group / tile program path
bool uses_prog(const tanq_sim* s, const FusedOp& op) { return op.k >= 3 || k2_tiled(s, op); }

size_t group_prog_elems(const FusedOp& op) {
  if (op.sub.empty()) return tanq::group_frag_elems(op.k);
  size_t e = 0;
  for (const auto& sb : op.sub) e += tanq::group_frag_elems(sb.k);
  return e;
}

// Build the K3 group program (sub-op headers + fragment-ordered matrices) for the current
// layout; returns the kernel parameters except `prog`.
void build_group(const tanq_sim* s, const FusedOp& op, tanq::GroupParams& p, double2* prog) {
  const int TBITS = 2 * op.k;  // 4, 6 or 8 (2-, 3- or 4-qubit tile)
  const MemberMap tile = member_map(s, op.k, op.q);
  p.nq = op.k;
  for (int t = 0; t < 8; ++t) {
    p.pos[t] = t < TBITS ? (uint32_t)tile.bits[t].first : 63u;
    p.lo_mask[t] = t < TBITS ? ((uint64_t)1 << tile.bits[t].first) - 1 : 0;
  }
  p.n_tuples = (uint64_t)1 << (s->L - TBITS);
  p.mirror = use_mirror(s, op) ? 1u : 0u;
  {
    const tanq::TDesc td = tdesc_of(s, s->shards.empty() ? 0 : s->shards[0].id);
    p.tp_lo = td.lo;
    p.tp_m = td.m;
  }
  static int dbg = -1;
  if (dbg < 0) {
    const char* e = std::getenv("TANQ_DBG");
    dbg = e ? std::atoi(e) : 0;
  }
  p.dbg = (uint32_t)dbg;
  std::vector<const FusedOp*> subs;
  if (op.sub.empty())
    subs.push_back(&op);
  else
    for (const auto& sb : op.sub) subs.push_back(&sb);
  size_t off = 0;
  p.n_sub = (int)subs.size();
  for (size_t i = 0; i < subs.size(); ++i) {
    const FusedOp& sb = *subs[i];
    const MemberMap mm = member_map(s, sb.k, sb.q);
    tanq::GroupSub& g = p.sub[i];
    std::memset(&g, 0, sizeof(g));
    g.k = sb.k;
    g.s_off = (int)off;
    // tile bit index of each of the sub-op's sorted physical positions
    int tb[8], nb = 0, rb[8], nr = 0;
    for (int t = 0; t < 2 * sb.k; ++t)
      for (int u = 0; u < TBITS; ++u)
        if (tile.bits[u].first == mm.bits[t].first) tb[nb++] = u;
    for (int u = 0; u < TBITS; ++u) {
      bool used = false;
      for (int t = 0; t < nb; ++t) used |= tb[t] == u;
      if (!used) rb[nr++] = u;
    }
    if (sb.k < 3) {
      for (int m = 0; m < (1 << (2 * sb.k)); ++m) {
        int v = 0;
        for (int t = 0; t < nb; ++t)
          if ((m >> t) & 1) v |= 1 << tb[t];
        g.mi[m] = (uint8_t)v;
      }
      for (int u = 0; u < (1 << nr); ++u) {
        int v = 0;
        for (int t = 0; t < nr; ++t)
          if ((u >> t) & 1) v |= 1 << rb[t];
        g.mu[u] = (uint8_t)v;
      }
    }
    const std::vector<double2> Sm = member_order_S(sb, mm);
    tanq::group_make_frags(sb.k, Sm.data(), prog + off);
    off += tanq::group_frag_elems(sb.k);
  }
  p.prog_elems = (int)off;
}

// ------------------------------------------------------------------------------------
// Block-pipeline group programs (tanq_block.cu)
// ------------------------------------------------------------------------------------
// A block = the op's 2 NQ physical target bits + the lowest free physical bits, 10 in all
// (in the packed layout: 5 whole qubits).  Block-order bit j <-> physical position bpos[j]
// (ascending); bits 0..3 are always physical 0..3 (the free bits fill from 0), so a block is 64
// contiguous 16-amplitude pieces.  Shared-memory bank of block element idx (16 B units, 8 banks
// of 16 B): (idx & 7) + G(idx >> 4) mod 8, where the piece placement G is linear in the 6
// piece-index bits with weights w[4..9] chosen here; w[0..2] = 1, 2, 4 and w[3] = 0 follow from
// the contiguous 256 B piece.  For each sub-op the lane -> (member, column) assignment of the
// DMMA fragments is chosen so that the 8 lanes of every quarter-warp hit distinct banks:
//   B fragment (k-step loads): lanes vary the 2 in-index bits k0, k1 and column bit n0;
//   D fragment (stores):      lanes vary out-index bit o0 and column bits n1, n2.
bool block_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("TANQ_BLOCK");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// sparse k = 2 sub-ops (DFMA, tanq_block.cu blk_sub_k2s) take superoperators with at most
// this many nonzeros (env TANQ_SPARSE_MAX, up to 64).  Default 0 = always DMMA: measured on
// QPE-16 (36-40 of 256 entries nonzero in 97 of its 128 updates) the sparse form is slower,
// 24.3 vs 15.8 ms per group pass (profiles/r02_sparse_subop_experiment.txt) -- every nonzero
// costs a dependent table + element load from shared memory, while DMMA reads each element
// once per k-step for 8 output rows.
int sparse_max() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("TANQ_SPARSE_MAX");
    v = e ? std::max(0, std::min(64, std::atoi(e))) : 0;
  }
  return v;
}
size_t sparse_sub_bytes(int nnz) { return (size_t)16 * nnz + 48 + (((size_t)(nnz + 16) * 64 * 2 + 15) & ~(size_t)15); }
size_t block_sub_bytes(int k) {
  return k == 2 ? std::max<size_t>(768 * 8 + 2 * 32 * 32 * 2, sparse_sub_bytes(64))
                : 32 * 8 + 2 * 32 * 16 * 2;
}

size_t block_blob_bytes(const FusedOp& op) {  // upper bound (incl. TMA slot + transform tables)
  size_t b = 2048 + 5 * 1024;
  if (op.sub.empty()) return b + block_sub_bytes(op.k);
  for (const auto& sb : op.sub) b += block_sub_bytes(sb.k);
  return b;
}

int block_pairs_for(size_t blob_bytes) {
  for (int P = tanq::kBlockMaxPairs; P >= 3; --P)
    if (tanq::block_smem_bytes(P, (int)blob_bytes) <= 227 * 1024) return P;
  return 0;
}

// Ops the block kernel runs: 3-qubit groups of k <= 2 sub-ops (not dense k = 3 ops), at least
// 4 blocks, small enough programs.  Env TANQ_BLOCK=0 restores the round-1 group kernels.
// standalone k = 2 ops whose targets sit at physical position >= 6 (the cooperative-tile
// case) also run as one-sub-op blocks (2 group + 3 free qubits): QPE-16 132.1 vs 131.4
// updates/s (profiles/r02_bench_c4_k2blk.json).  Env TANQ_BLOCK_K2=0 restores the tile kernel.
bool block_k2_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("TANQ_BLOCK_K2");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

bool block_ok(const tanq_sim* s, const FusedOp& op) {
  if (!block_enabled() || s->L < 12) return false;
  if (op.k == 2 && op.sub.empty()) return block_k2_enabled() && k2_tiled(s, op);
  if (op.k == 4 || op.k == 5) {  // 4- / 5-qubit groups: the block's lowest 4 bits must be
    if (op.sub.empty()) return false;  // physical 0..3
    std::vector<int> pos;
    for (int j = 0; j < op.k; ++j)
      for (int b = 0; b < 2; ++b) pos.push_back((int)s->phys[2 * op.q[j] + b]);
    for (int f = 0; pos.size() < 10; ++f)
      if (std::find(pos.begin(), pos.end(), f) == pos.end()) pos.push_back(f);
    for (int b = 0; b < 4; ++b)
      if (std::find(pos.begin(), pos.end(), b) == pos.end()) return false;
  } else if (op.k != 3 || op.sub.empty()) {
    return false;
  }
  if ((int)op.sub.size() > tanq::kBlockMaxSub) return false;
  for (const auto& sb : op.sub)
    if (sb.k > 2) return false;
  return block_pairs_for(block_blob_bytes(op)) > 0;
}

size_t prog_capacity(const FusedOp& op) {
  return std::max(group_prog_elems(op), (block_blob_bytes(op) + 15) / 16);
}

// max lanes per bank over the 8 lane combinations of a quarter warp whose 3 varying index bits
// have bank contributions w0, w1, w2: added mod 8 (rotation layout) or XORed (TMA swizzle)
bool g_bank_xor = false;  // set by build_block while it evaluates a layout
int phase_degree(int w0, int w1, int w2) {
  int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, mx = 0;
  for (int c = 0; c < 8; ++c) {
    const int b = g_bank_xor ? ((c & 1 ? w0 : 0) ^ (c & 2 ? w1 : 0) ^ (c & 4 ? w2 : 0))
                             : ((c & 1 ? w0 : 0) + (c & 2 ? w1 : 0) + (c & 4 ? w2 : 0)) & 7;
    mx = std::max(mx, ++cnt[b]);
  }
  return mx;
}

int block_tma_mode() {  // env TANQ_BLOCK_TMA = 0 (never) | 1 (whenever possible) | auto
  static int m = -1;
  if (m < 0) {
    const char* e = std::getenv("TANQ_BLOCK_TMA");
    m = !e ? 2 : (e[0] == '0' ? 0 : (e[0] == '1' ? 1 : 2));
  }
  return m;
}

// Zero-tile skipping (BlockSub::tmask) measured slower on B200 (uniform branches around the
// DMMAs and +16 registers cost more than the 25% of DMMAs QPE's sparse sub-ops save), so the
// kernel issues every tile and the mapping is chosen for bank conflicts only (weight 0).
constexpr int kTileWeight = 0;

struct BlockSubChoice {
  int k0 = 0, k1 = 0, o0 = 0, o3 = 0, n[3] = {0, 0, 0}, cost = 0, tiles = 8;
  uint32_t tmask = 0xffu;  // nonzero 8x4 A tiles (bit mt * 4 + ks)
};

// nonzero 8x4 A tiles of a k=2 sub-op (16x16, sub-op member order, nz[out * 16 + in]) when
// in-index bits (0, 1) = members (i, j), ks = the other two (ascending), and mt = member o3
uint32_t tile_mask(const uint8_t* nz, int i, int j, int o3) {
  int kb[2], nk = 0;
  for (int t = 0; t < 4; ++t)
    if (t != i && t != j) kb[nk++] = t;
  uint32_t m = 0;
  for (int mo = 0; mo < 16; ++mo)
    for (int mi = 0; mi < 16; ++mi)
      if (nz[mo * 16 + mi]) {
        const int mt = (mo >> o3) & 1, ks = ((mi >> kb[0]) & 1) | (((mi >> kb[1]) & 1) << 1);
        m |= 1u << (mt * 4 + ks);
      }
  return m;
}

// best lane mapping of one sub-op (member / column block bits) for bank weights w.  k = 2:
// fewest nonzero A tiles first (every zero 8x4 tile saves 3 DMMA per n-tile pass), then the
// fewest bank conflicts of the B (k0, k1, n0) and D (o0, n1, n2) quarter-warp accesses.
BlockSubChoice best_choice(int k, const std::vector<int>& mem, const std::vector<int>& col,
                           const int* w, const uint8_t* nz = nullptr) {
  BlockSubChoice best;
  best.cost = 1 << 20;
  if (k == 1) {  // lanes vary column bits n0..n2 (col = lane + 32 j)
    for (size_t a = 0; a < col.size(); ++a)
      for (size_t b = 0; b < col.size(); ++b)
        for (size_t c = 0; c < col.size(); ++c) {
          if (a == b || a == c || b == c) continue;
          const int d = phase_degree(w[col[a]], w[col[b]], w[col[c]]);
          if (d < best.cost) {
            best.cost = d;
            best.n[0] = col[a];
            best.n[1] = col[b];
            best.n[2] = col[c];
          }
        }
    return best;
  }
  int dB[4][4][8], dD[4][8][8];  // bank degrees by (i, j, a) and (o, b, c)
  const int nc = (int)col.size();
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j)
      for (int a = 0; a < nc; ++a) dB[i][j][a] = phase_degree(w[mem[i]], w[mem[j]], w[col[a]]);
  for (int o = 0; o < 4; ++o)
    for (int b = 0; b < nc; ++b)
      for (int c = 0; c < nc; ++c) dD[o][b][c] = phase_degree(w[mem[o]], w[col[b]], w[col[c]]);
  for (int i = 0; i < 4; ++i)
    for (int j = i + 1; j < 4; ++j)
      for (int o3 = 0; o3 < 4; ++o3) {
        const uint32_t tm = nz ? tile_mask(nz, i, j, o3) : 0xffu;
        const int tiles = __builtin_popcount(tm);
        for (int o = 0; o < 4; ++o) {
          if (o == o3) continue;
          for (int a = 0; a < nc; ++a)
            for (int b = 0; b < nc; ++b)
              for (int c = b + 1; c < nc; ++c) {
                if (b == a || c == a) continue;
                const int cost = kTileWeight * tiles + dB[i][j][a] + dD[o][b][c];
                if (cost < best.cost) {
                  best.cost = cost;
                  best.tiles = tiles;
                  best.tmask = tm;
                  best.k0 = mem[i];
                  best.k1 = mem[j];
                  best.o0 = mem[o];
                  best.o3 = mem[o3];
                  best.n[0] = col[a];
                  best.n[1] = col[b];
                  best.n[2] = col[c];
                }
              }
        }
      }
  return best;
}

// Build the block-kernel parameters and blob (fragments + offset tables) of a 3-qubit group for
// the current layout.  Returns the blob size in bytes (written to `blob`).
// Real basis for the block kernel (BlockParams::rb_nq).  A Hermiticity-
// preserving superoperator commutes with J: (J x)[(r, c)] = conj x[(c, r)], so in the basis in
// which J-invariant vectors have real coordinates -- per qubit e00, e10 + e01, i (e01 - e10),
// e11 -- it is a real matrix R = F S F^-1.  Groups whose sub-ops are all Hermiticity-preserving
// transform the block once after the load and back before the store; every k=2 sub-op then
// needs 2 real DMMA products instead of 3.  Opt-in (env TANQ_RBASIS=1; TANQ_RBASIS_MIN = the
// fewest k=2 sub-ops a group needs, default 1): measured slower on B200 -- QPE-16 113.4 vs
// 127.1 updates/s, config 3 (k_max 4) 1751 vs 1842 (profiles/r02_rbasis_experiment.txt): the
// per-qubit pair passes over shared memory and their pair barriers cost more than the third
// of the DMMAs they save.
int rbasis_min() {
  static int v = -2;
  if (v == -2) {
    const char* e = std::getenv("TANQ_RBASIS");
    const char* m = std::getenv("TANQ_RBASIS_MIN");
    v = !(e && e[0] == '1') ? -1 : (m ? std::max(1, std::atoi(m)) : 1);
  }
  return v;
}

// F (forward transform) in a sub-op's member order: member bit rbit[j] / cbit[j] = row / col
// bit of sub-op qubit j.  Pair (x1: r=1 c=0, x2: r=0 c=1) -> (u1, u2) = (x1 + x2, i (x2 - x1)).
Mat rbasis_matrix(int k, const int* rbit, const int* cbit, bool inverse) {
  const int M = 1 << (2 * k);
  Mat F = identity(M);
  for (int j = 0; j < k; ++j) {
    Mat Fj = identity(M);
    for (int m = 0; m < M; ++m) {
      const int r = (m >> rbit[j]) & 1, c = (m >> cbit[j]) & 1;
      if (!(r == 1 && c == 0)) continue;
      const int m1 = m, m2 = (m & ~(1 << rbit[j])) | (1 << cbit[j]);
      if (!inverse) {
        Fj(m1, m1) = 1.0; Fj(m1, m2) = 1.0;
        Fj(m2, m1) = cd(0, -1); Fj(m2, m2) = cd(0, 1);
      } else {
        Fj(m1, m1) = 0.5; Fj(m1, m2) = cd(0, 0.5);
        Fj(m2, m1) = 0.5; Fj(m2, m2) = cd(0, -0.5);
      }
    }
    F = matmul(Fj, F);
  }
  return F;
}

size_t build_block(const tanq_sim* s, const FusedOp& op, tanq::BlockParams& p, unsigned char* blob) {
  const int NQ = op.k, MB = 2 * NQ;
  const MemberMap tile = member_map(s, NQ, op.q);  // group member bit u <-> tile.bits[u].first
  std::vector<int> tpos(MB);
  for (int u = 0; u < MB; ++u) tpos[u] = tile.bits[u].first;
  // block positions: targets + lowest free positions
  std::vector<int> bpos(tpos);
  for (int f = 0; (int)bpos.size() < 10; ++f)
    if (std::find(tpos.begin(), tpos.end(), f) == tpos.end()) bpos.push_back(f);
  std::sort(bpos.begin(), bpos.end());
  auto bit_of_pos = [&](int pos) {
    return (int)(std::find(bpos.begin(), bpos.end(), pos) - bpos.begin());
  };
  std::vector<int> is_member(10, -1);  // block bit -> group member bit u, or -1 (tuple bit)
  for (int u = 0; u < MB; ++u) is_member[bit_of_pos(tpos[u])] = u;
  int half = -1;                        // warp-half bit: the highest tuple bit
  for (int j = 9; j >= 0 && half < 0; --j)
    if (is_member[j] < 0) half = j;
  std::vector<const FusedOp*> subs;
  for (const auto& sb : op.sub) subs.push_back(&sb);
  if (subs.empty()) subs.push_back(&op);  // a standalone k = 2 op: one sub-op on 2 qubits
  // member / column block bits of every sub-op
  std::vector<std::vector<int>> smem_bits(subs.size()), scol_bits(subs.size());
  std::vector<MemberMap> smap(subs.size());
  std::vector<std::vector<uint8_t>> snz(subs.size());  // nonzero pattern, sub-op member order
  for (size_t i = 0; i < subs.size(); ++i) {
    smap[i] = member_map(s, subs[i]->k, subs[i]->q);
    if (subs[i]->k == 2) {
      const std::vector<double2> Sm = member_order_S(*subs[i], smap[i]);
      snz[i].resize(256);
      for (int e = 0; e < 256; ++e) snz[i][e] = (Sm[e].x != 0.0 || Sm[e].y != 0.0) ? 1 : 0;
    }
    for (int t = 0; t < 2 * subs[i]->k; ++t) smem_bits[i].push_back(bit_of_pos(smap[i].bits[t].first));
  }
  // warp-half bit of each sub-op: the group's highest tuple bit; a 5-qubit block group has
  // none, so each sub-op splits the block on a bit it does not touch (in-piece bit 3 when
  // possible: one shared table), and the pair meets at a barrier when the split changes
  std::vector<int> shalf(subs.size(), half);
  for (size_t i = 0; i < subs.size(); ++i) {
    auto in_sub = [&](int j) {
      return std::find(smem_bits[i].begin(), smem_bits[i].end(), j) != smem_bits[i].end();
    };
    if (shalf[i] < 0) {
      if (!in_sub(3)) shalf[i] = 3;
      for (int j = 9; j >= 0 && shalf[i] < 0; --j)
        if (!in_sub(j)) shalf[i] = j;
    }
    for (int j = 0; j < 10; ++j)
      if (j != shalf[i] && !in_sub(j)) scol_bits[i].push_back(j);
  }
  // real basis: every sub-op Hermiticity-preserving, enough k=2 sub-ops, R real to rounding
  std::vector<std::vector<double2>> sR(subs.size());  // sub-op matrices in the real basis
  bool rb = false;
  {
    int n2 = 0;
    bool herm = true;
    for (const FusedOp* sb : subs) {
      n2 += sb->k == 2 ? 1 : 0;
      herm = herm && sb->herm;
    }
    rb = rbasis_min() > 0 && herm && n2 >= rbasis_min() && sparse_max() == 0;
    for (size_t i = 0; rb && i < subs.size(); ++i) {
      const int k = subs[i]->k, M = 1 << (2 * k);
      int rbit[2], cbit[2];
      for (int t = 0; t < 2 * k; ++t) {
        const int b = smap[i].bits[t].second;  // paper-index bit: row of qubit b, col of b - k
        if (b < k) rbit[b] = t; else cbit[b - k] = t;
      }
      const std::vector<double2> Sm = member_order_S(*subs[i], smap[i]);
      Mat S(M);
      for (int e = 0; e < M * M; ++e) S.a[e] = cd(Sm[e].x, Sm[e].y);
      const Mat R = matmul(rbasis_matrix(k, rbit, cbit, false),
                           matmul(S, rbasis_matrix(k, rbit, cbit, true)));
      double mx = 0.0, im = 0.0;
      for (const cd& v : R.a) {
        mx = std::max(mx, std::abs(v));
        im = std::max(im, std::abs(v.imag()));
      }
      if (im > 1e-13 * std::max(1.0, mx)) {
        rb = false;
        break;
      }
      sR[i].resize((size_t)M * M);
      for (int e = 0; e < M * M; ++e) sR[i][e] = make_double2(R.a[e].real(), 0.0);
    }
  }
  // piece-placement weights: start from one rotation per qubit pair of piece-index bits,
  // (1,2), (4,1), (2,4) (conflict-free for every pair of 3 group qubits when the group sits
  // above qubit 1), then coordinate descent
  int w[10] = {1, 2, 4, 0, 0, 0, 0, 0, 0, 0};
  {
    static const int init[3][2] = {{1, 2}, {4, 1}, {2, 4}};
    int qi = 0;
    for (int j = 4; j + 1 < 10; j += 2)
      if (is_member[j] >= 0 && is_member[j + 1] >= 0 && qi < 3) {
        w[j] = init[qi][0];
        w[j + 1] = init[qi][1];
        ++qi;
      }
  }
  auto total_cost = [&](const int* ww) {
    int c = 0;
    for (size_t i = 0; i < subs.size(); ++i)
      c += best_choice(subs[i]->k, smem_bits[i], scol_bits[i], ww,
                       snz[i].empty() ? nullptr : snz[i].data()).cost;
    return c;
  };
  int cost = total_cost(w);
  const int ideal = [&] {  // every sub-op at its fewest tiles and conflict-free
    int c = 0;
    for (size_t i = 0; i < subs.size(); ++i) {
      if (subs[i]->k != 2) {
        c += 1;
        continue;
      }
      int tmin = 8;
      for (int a = 0; a < 4; ++a)
        for (int b = a + 1; b < 4; ++b)
          for (int o3 = 0; o3 < 4; ++o3)
            tmin = std::min(tmin, __builtin_popcount(tile_mask(snz[i].data(), a, b, o3)));
      c += kTileWeight * tmin + 2;
    }
    return c;
  }();
  for (int sweep = 0; sweep < 4 && cost > ideal; ++sweep)
    for (int j = 4; j < 10; ++j)
      for (int v = 0; v < 8; ++v) {
        const int old = w[j];
        w[j] = v;
        const int c = total_cost(w);
        if (c < cost) cost = c;
        else w[j] = old;
      }
  // TMA layout: the block as a box of <= 5 dims (runs of block bits + the gap above each run,
  // bits 0-2 as the 128 B inner dim) landing in box order with the 128 B swizzle.  The dims
  // after the inner one may come in any order: their first three box bits are the swizzle's row
  // bits (XORed into the bank), so the order is chosen for the fewest bank conflicts.  Bank
  // contributions XOR: bits 0-2 -> 1, 2, 4; the first three row bits -> 1, 2, 4; others none.
  bool use_tma = false;
  int tdims = 0, tlo[5] = {0, 0, 0, 0, 0}, tbits[5] = {0, 0, 0, 0, 0}, tbox[5] = {0, 0, 0, 0, 0};
  int sbit[10];  // TMA layout: box-linear bit of block bit j
  {
    std::vector<std::pair<int, int>> runs;  // block-bit runs above bit 2: (first block bit, length)
    for (int j = 3; j < 10; ++j) {
      if (!runs.empty() && bpos[runs.back().first] + runs.back().second == bpos[j]) ++runs.back().second;
      else runs.push_back({j, 1});
    }
    // split runs at qubit boundaries while dims remain, so the order search can choose which
    // qubit's bits become the swizzle row bits
    for (bool split = true; split && runs.size() < 4;) {
      split = false;
      for (size_t r = 0; r < runs.size() && !split; ++r)
        for (int b = 1; b < runs[r].second; ++b)
          if ((bpos[runs[r].first + b] & 1) == 0) {  // a qubit's row bit starts here
            runs.insert(runs.begin() + r + 1, {runs[r].first + b, runs[r].second - b});
            runs[r].second = b;
            split = true;
            break;
          }
    }
    if (runs.size() <= 4 && block_tma_mode() != 0) {
      std::vector<int> ord(runs.size());
      for (size_t r = 0; r < ord.size(); ++r) ord[r] = (int)r;
      int best_cost = 1 << 30;
      std::vector<int> best_ord = ord;
      int wx[10];
      do {
        int pos = 3;
        for (int j = 0; j < 3; ++j) wx[j] = 1 << j;
        for (int r : ord)
          for (int b = 0; b < runs[r].second; ++b, ++pos)
            wx[runs[r].first + b] = pos < 6 ? 1 << (pos - 3) : 0;
        g_bank_xor = true;
        const int c = total_cost(wx);
        g_bank_xor = false;
        if (c < best_cost) {
          best_cost = c;
          best_ord = ord;
        }
      } while (std::next_permutation(ord.begin(), ord.end()));
      tdims = 1 + (int)runs.size();
      tlo[0] = 0; tbits[0] = 3; tbox[0] = 3;
      int pos = 3;
      for (int j = 0; j < 3; ++j) sbit[j] = j;
      for (size_t d = 0; d < best_ord.size(); ++d) {
        const int r = best_ord[d];
        const int first = bpos[runs[r].first];
        tlo[d + 1] = first;
        tbox[d + 1] = runs[r].second;
        const int next = (size_t)r + 1 < runs.size() ? bpos[runs[r + 1].first] : s->L;
        tbits[d + 1] = next - first;
        for (int b = 0; b < runs[r].second; ++b, ++pos) {
          sbit[runs[r].first + b] = pos;
          wx[runs[r].first + b] = pos < 6 ? 1 << (pos - 3) : 0;
        }
      }
      for (int j = 0; j < 3; ++j) wx[j] = 1 << j;
      // packed layout: blocks are moved by one TMA only when no member pair decides where an
      // element is stored, i.e. the base differs at a qubit above the group -- require at least
      // two qubits above the group (about 3/4 of the processed blocks or more); the others go
      // through the cp.async path
      const int pair_top = s->par ? 2 * (s->n - __builtin_popcountll(s->par)) : s->L;
      const bool mostly_direct = !use_mirror(s, op) || bpos[9] + 4 < pair_top;
      static int slack = -1;
      if (slack < 0) {
        const char* e = std::getenv("TANQ_BLOCK_TMA_SLACK");
        slack = e ? std::atoi(e) : 1;
      }
      use_tma = block_tma_mode() == 1 || (mostly_direct && best_cost <= cost + slack);
      if (std::getenv("TANQ_BLOCK_DEBUG"))
        std::fprintf(stderr, "block q=%d,%d,%d dims=%d cost rot %d tma %d direct %d -> %s\n",
                     op.q[0], op.q[1], op.k > 2 ? op.q[2] : -1, tdims, cost, best_cost,
                     (int)mostly_direct, use_tma ? "tma" : "rot");
      if (use_tma) {
        for (int j = 0; j < 10; ++j) w[j] = wx[j];
        cost = best_cost;
      }
    }
  }
  if (use_tma) g_bank_xor = true;
  // placement: pieces sorted by G, piece at 16 * rank + G
  int G[64], order[64];
  for (int pi = 0; pi < 64; ++pi) {
    int g = 0;
    for (int b = 0; b < 6; ++b)
      if ((pi >> b) & 1) g += w[4 + b];
    G[pi] = g & 7;
    order[pi] = pi;
  }
  if (!use_tma) std::stable_sort(order, order + 64, [&](int x, int y) { return G[x] < G[y]; });
  int start_by_pidx[64];
  for (int r = 0; r < 64; ++r) {
    const int pi = order[r];
    start_by_pidx[pi] = use_tma ? 16 * pi : 16 * r + G[pi];  // TMA: slot() applies the swizzle
    uint64_t off = 0;
    for (int b = 0; b < 6; ++b)
      if ((pi >> b) & 1) off += (uint64_t)1 << bpos[4 + b];
    p.piece_goff[r] = off;
    p.piece_start[r] = (uint16_t)start_by_pidx[pi];
  }
  for (int pi = 0; pi < 64; ++pi) p.start_by_pidx[pi] = (uint16_t)start_by_pidx[pi];
  auto slot = [&](int idx) {
    if (!use_tma) return start_by_pidx[idx >> 4] + (idx & 15);
    int sidx = 0;  // box-linear index, then the 128 B swizzle
    for (int j = 0; j < 10; ++j)
      if ((idx >> j) & 1) sidx |= 1 << sbit[j];
    return sidx ^ ((sidx >> 3) & 7);
  };
  p.tma = use_tma ? 1u : 0u;
  p.tdims = tdims;
  for (int d = 0; d < 5; ++d) {
    p.tlo[d] = tlo[d];
    p.tbits[d] = tbits[d];
    p.tbox[d] = tbox[d];
  }
  p.hi_blk = bpos[9];
  for (int j = 0; j < 10; ++j) p.lo_mask[j] = ((uint64_t)1 << bpos[j]) - 1;
  p.n_blocks = (uint64_t)1 << (s->L - 10);
  p.mirror = use_mirror(s, op) ? 1u : 0u;
  {
    const tanq::TDesc td = tdesc_of(s, s->shards.empty() ? 0 : s->shards[0].id);
    p.tp_lo = td.lo;
    p.tp_m = td.m;
  }
  static int dbg = -1;
  if (dbg < 0) {
    const char* e = std::getenv("TANQ_DBG");
    dbg = e ? std::atoi(e) : 0;
  }
  p.dbg = (uint32_t)dbg;
  p.n_sub = (int)subs.size();
  // the warp-half bit is in-piece bit 3 (both halves' offsets differ by 8 units): one table
  p.half_add = (shalf[0] == 3 && !use_tma) ? 8 : -1;
  // blob: per sub-op fragments then tables (both 16 B aligned)
  size_t off = 0;
  for (size_t i = 0; i < subs.size(); ++i) {
    const FusedOp& sb = *subs[i];
    tanq::BlockSub& g = p.sub[i];
    g.k = sb.k;
    const int half = shalf[i];
    const bool share = half == 3 && !use_tma;
    const int halves = share ? 1 : 2;
    g.hadd = share ? 8 : -1;
    g.sync = (i > 0 && shalf[i] != shalf[i - 1]) ? 1 : 0;
    const BlockSubChoice ch = best_choice(sb.k, smem_bits[i], scol_bits[i], w,
                                          snz[i].empty() ? nullptr : snz[i].data());
    g.tmask = sb.k == 2 ? (int)ch.tmask : 0xff;
    const std::vector<double2> Sm = rb ? sR[i] : member_order_S(sb, smap[i]);  // member order
    // sub-op member bit t <-> block bit smem_bits[i][t]
    auto sub_member = [&](const int* blkbits, int nb, int v) {  // value over blkbits -> member
      int m = 0;
      for (int b = 0; b < nb; ++b)
        if ((v >> b) & 1) {
          const int t = (int)(std::find(smem_bits[i].begin(), smem_bits[i].end(), blkbits[b]) -
                              smem_bits[i].begin());
          m |= 1 << t;
        }
      return m;
    };
    auto deposit = [&](const int* blkbits, int nb, int v) {
      int idx = 0;
      for (int b = 0; b < nb; ++b)
        if ((v >> b) & 1) idx |= 1 << blkbits[b];
      return idx;
    };
    // column bit order: n[0..2] first, then the rest ascending
    std::vector<int> cols(ch.n, ch.n + 3);
    for (int c : scol_bits[i])
      if (std::find(cols.begin(), cols.end(), c) == cols.end()) cols.push_back(c);
    g.a_off = (int)(off / 8);
    g.nnz = 0;
    uint16_t* T;
    int nnz = 0;
    if (sb.k == 2)
      for (const double2& v : Sm) nnz += (v.x != 0.0 || v.y != 0.0) ? 1 : 0;
    if (sb.k == 2 && nnz > 0 && nnz <= sparse_max()) {
      // sparse DFMA sub-op: lane = tuple (the 5 block bits outside the sub-op and the half
      // bit); the 3 lane bits of a quarter warp are chosen for distinct banks
      g.nnz = nnz;
      double2* sv = reinterpret_cast<double2*>(blob + off);
      uint16_t rs[17];
      std::vector<int> ein;  // input member of entry e
      for (int r = 0, e = 0; r < 16; ++r) {
        rs[r] = (uint16_t)e;
        for (int c = 0; c < 16; ++c) {
          const double2 v = Sm[(size_t)r * 16 + c];
          if (v.x != 0.0 || v.y != 0.0) {
            sv[e++] = v;
            ein.push_back(c);
          }
        }
        rs[16] = (uint16_t)e;
      }
      off += (size_t)16 * nnz;
      std::memcpy(blob + off, rs, sizeof(rs));
      off += 48;
      g.t_off = (int)(off / 2);
      T = reinterpret_cast<uint16_t*>(blob + off);
      std::vector<int> tb(scol_bits[i]);  // 5 tuple bits
      {  // order: the 3 bits that spread a quarter warp over the most banks first
        int best = 1 << 30;
        std::vector<int> best_tb = tb;
        for (int x = 0; x < 5; ++x)
          for (int y = x + 1; y < 5; ++y)
            for (int z = y + 1; z < 5; ++z) {
              std::vector<int> cand{tb[x], tb[y], tb[z]};
              for (int u = 0; u < 5; ++u)
                if (u != x && u != y && u != z) cand.push_back(tb[u]);
              int cost = 0;
              for (int m = 0; m < 16; ++m)
                for (int ph = 0; ph < 4; ++ph) {
                  int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, mx = 0;
                  for (int l = 0; l < 8; ++l) {
                    const int idx = deposit(smem_bits[i].data(), 4, m) |
                                    deposit(cand.data(), 5, l | (ph << 3));
                    mx = std::max(mx, ++cnt[slot(idx) & 7]);
                  }
                  cost += mx;
                }
              if (cost < best) {
                best = cost;
                best_tb = cand;
              }
            }
        tb = best_tb;
      }
      const int rows = halves * 32;
      for (int h = 0; h < halves; ++h)
        for (int lane = 0; lane < 32; ++lane) {
          const int tup = deposit(tb.data(), 5, lane) | (h << half);
          for (int e = 0; e < nnz; ++e)
            T[(size_t)e * rows + h * 32 + lane] =
                (uint16_t)slot(deposit(smem_bits[i].data(), 4, ein[e]) | tup);
          for (int m = 0; m < 16; ++m)
            T[(size_t)(nnz + m) * rows + h * 32 + lane] =
                (uint16_t)slot(deposit(smem_bits[i].data(), 4, m) | tup);
        }
      off += ((size_t)(nnz + 16) * rows * 2 + 15) & ~(size_t)15;
    } else if (sb.k == 2) {
      int in_bits[4] = {ch.k0, ch.k1, 0, 0}, out_bits[4] = {ch.o0, 0, 0, ch.o3};
      for (int t = 0, a = 2, b = 1; t < 4; ++t) {
        const int bb = smem_bits[i][t];
        if (bb != ch.k0 && bb != ch.k1) in_bits[a++] = bb;
        if (bb != ch.o0 && bb != ch.o3) out_bits[b++] = bb;
      }
      double* F = reinterpret_cast<double*>(blob + off);
      for (int mt = 0; mt < 2; ++mt)
        for (int ks = 0; ks < 4; ++ks)
          for (int lane = 0; lane < 32; ++lane) {
            const int row = mt * 8 + (lane >> 2), colk = ks * 4 + (lane & 3);
            const double2 v = Sm[(size_t)sub_member(out_bits, 4, row) * 16 + sub_member(in_bits, 4, colk)];
            const int e = (ks * 32 + lane) * 2 + mt;  // [mat][ks][lane][mt]
            F[0 * 256 + e] = v.x;
            if (!rb) {
              F[1 * 256 + e] = -(v.x + v.y);
              F[2 * 256 + e] = v.y - v.x;
            }
          }
      off += (rb ? 256 : 768) * 8;
      g.t_off = (int)(off / 2);
      T = reinterpret_cast<uint16_t*>(blob + off);
      // layout [4 chunks][rows = halves x 32][8 uint16]: entry e of a row is in chunk e / 8
      const int rows = halves * 32;
      for (int h = 0; h < halves; ++h)
        for (int lane = 0; lane < 32; ++lane) {
          uint16_t t[32];
          const int c4 = lane & 3, r4 = lane >> 2, hb = h << half;
          for (int ks = 0; ks < 4; ++ks)
            for (int j = 0; j < 4; ++j) {
              const int idx = deposit(in_bits, 4, c4 | (ks << 2)) |
                              deposit(cols.data(), (int)cols.size(), 8 * j + r4) | hb;
              t[ks * 4 + j] = (uint16_t)slot(idx);
            }
          for (int mt = 0; mt < 2; ++mt)
            for (int j = 0; j < 4; ++j)
              for (int c = 0; c < 2; ++c) {
                const int idx = deposit(out_bits, 4, r4 | (mt << 3)) |
                                deposit(cols.data(), (int)cols.size(), 8 * j + 2 * c4 + c) | hb;
                t[16 + (mt * 4 + j) * 2 + c] = (uint16_t)slot(idx);
              }
          for (int e = 0; e < 32; ++e) T[((e >> 3) * rows + h * 32 + lane) * 8 + (e & 7)] = t[e];
        }
      off += (size_t)halves * 32 * 32 * 2;
    } else {
      double2* F = reinterpret_cast<double2*>(blob + off);
      for (int e = 0; e < 16; ++e) F[e] = Sm[e];
      off += 32 * 8;
      g.t_off = (int)(off / 2);
      T = reinterpret_cast<uint16_t*>(blob + off);
      const int mbits[2] = {smem_bits[i][0], smem_bits[i][1]};  // member order = sorted position
      const int rows = halves * 32;  // layout [2 chunks][rows][8 uint16]
      for (int h = 0; h < halves; ++h)
        for (int lane = 0; lane < 32; ++lane) {
          uint16_t t[16];
          for (int j = 0; j < 4; ++j)
            for (int m = 0; m < 4; ++m) {
              const int idx = deposit(mbits, 2, m) |
                              deposit(cols.data(), (int)cols.size(), lane + 32 * j) | (h << half);
              t[j * 4 + m] = (uint16_t)slot(idx);
            }
          for (int e = 0; e < 16; ++e) T[((e >> 3) * rows + h * 32 + lane) * 8 + (e & 7)] = t[e];
        }
      off += (size_t)halves * 32 * 16 * 2;
    }
  }
  p.rb_nq = 0;
  p.rb_off = 0;
  if (rb) {  // transform tables: [qubit][64 pair threads][4 pairs][x1 slot, x2 slot]
    p.rb_off = (int)(off / 2);
    uint16_t* RT = reinterpret_cast<uint16_t*>(blob + off);
    for (int j = 0; j < op.k; ++j) {
      const int rbit = bit_of_pos((int)s->phys[2 * op.q[j]]);
      const int cbit = bit_of_pos((int)s->phys[2 * op.q[j] + 1]);
      std::vector<int> ob;
      for (int b = 0; b < 10; ++b)
        if (b != rbit && b != cbit) ob.push_back(b);
      // the 3 lane bits of a quarter warp: the triple spreading x1 and x2 over the most banks
      std::vector<int> best_ob = ob;
      int best = 1 << 30;
      for (int x = 0; x < 8; ++x)
        for (int y = x + 1; y < 8; ++y)
          for (int z = y + 1; z < 8; ++z) {
            std::vector<int> cand{ob[x], ob[y], ob[z]};
            for (int u = 0; u < 8; ++u)
              if (u != x && u != y && u != z) cand.push_back(ob[u]);
            int cost = 0;
            for (int hi = 0; hi < 32; ++hi)
              for (int which = 0; which < 2; ++which) {
                int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, m = 0;
                for (int l = 0; l < 8; ++l) {
                  int idx = 1 << (which ? cbit : rbit);
                  const int o = l | (hi << 3);
                  for (int b = 0; b < 8; ++b)
                    if ((o >> b) & 1) idx |= 1 << cand[b];
                  m = std::max(m, ++cnt[slot(idx) & 7]);
                }
                cost += m;
              }
            if (cost < best) {
              best = cost;
              best_ob = cand;
            }
          }
      for (int o = 0; o < 256; ++o) {
        int base = 0;
        for (int b = 0; b < 8; ++b)
          if ((o >> b) & 1) base |= 1 << best_ob[b];
        const int pt = o & 63, jj = o >> 6;
        RT[((size_t)(j * 64 + pt) * 4 + jj) * 2 + 0] = (uint16_t)slot(base | (1 << rbit));
        RT[((size_t)(j * 64 + pt) * 4 + jj) * 2 + 1] = (uint16_t)slot(base | (1 << cbit));
      }
    }
    p.rb_nq = op.k;
    off += (size_t)op.k * 64 * 8 * 2;
  }
  if (use_tma) {  // slot table for the cp.async path of blocks that are not moved by TMA
    p.slot_off = (int)(off / 2);
    uint16_t* st = reinterpret_cast<uint16_t*>(blob + off);
    for (int idx = 0; idx < 1024; ++idx) st[idx] = (uint16_t)slot(idx);
    off += 2048;
  } else {
    p.slot_off = -1;
  }
  g_bank_xor = false;
  p.blob_bytes = (int)off;
  p.pairs = block_pairs_for(off);
  return off;
}

// Packed -> full layout (one pass), before anything that reads or writes elements the packed
// layout does not keep up to date.
tanq_status ensure_unpacked(tanq_sim* s) {
  if (!s->packed) return TANQ_OK;
  for (auto& sh : s->shards) {
    CUDA_TRY(cudaSetDevice(sh.device));
    Prof pr{4, nullptr, nullptr, 16.0 * (double)((uint64_t)1 << s->L), 0.0, 0.0};
    prof_begin(s, sh, pr);
    CUDA_TRY(tanq::launch_unpack(sh.data, s->L, tdesc_of(s, sh.id), sh.stream));
    prof_end(s, sh, pr);
    s->launches++;
  }
  s->packed = false;
  return TANQ_OK;
}

// Launch one fused op on every shard (targets must be local).  For k >= 3 (groups), `prog`
// holds the group program already copied to each device (indexed like s->scratch).
tanq_status launch_op(tanq_sim* s, const FusedOp& op, const tanq::GroupParams* gp,
                      const std::vector<const double2*>* prog,
                      const tanq::BlockParams* bp = nullptr) {
  const int k = op.k, M = 1 << (2 * k);
  const uint64_t n_tuples = (uint64_t)1 << (s->L - 2 * k);
  const double amps = (double)((uint64_t)1 << s->L);
  // algorithmic: 8 flops per complex MAC; executed: K1 (FMA) 8, K2 / K3 (3-multiply DMMA) 6
  double flops_amp = 8.0 * M, hw_amp = (k == 1 ? 8.0 : 6.0) * M;
  // (real basis: k=2 sub-ops execute 4 -- two real products)
  const double hw2 = (bp && bp->rb_nq) ? 4.0 : 6.0;
  if (bp && op.sub.empty() && k == 2) hw_amp = hw2 * M;
  if ((gp || bp) && !op.sub.empty()) {
    flops_amp = hw_amp = 0;
    for (const auto& sb : op.sub) {
      const int Ms = 1 << (2 * sb.k);
      flops_amp += 8.0 * Ms;
      hw_amp += (sb.k == 1 ? 8.0 : hw2) * Ms;
    }
  }
  const bool mir_op = gp ? gp->mirror != 0 : (bp ? bp->mirror != 0 : use_mirror(s, op));
  if (!mir_op) TRY(ensure_unpacked(s));
  MemberMap mm;
  std::vector<double2> Sm;
  if (!gp && !bp) {
    mm = member_map(s, k, op.q);
    Sm = member_order_S(op, mm);
  }
  for (auto& sh : s->shards) {
    CUDA_TRY(cudaSetDevice(sh.device));
    // packed layout: only the canonical element of each transpose pair is read and written
    // (16 B per amplitude per pass) and half the tuples are computed
    const bool mir = mir_op;
    const double fr = mir ? 0.5 : 1.0;
    Prof pr{std::min(k, 3) - 1, nullptr, nullptr, (mir ? 16.0 : 32.0) * amps,
            fr * flops_amp * amps, fr * hw_amp * amps};
    prof_begin(s, sh, pr);
    const tanq::TDesc td = tdesc_of(s, sh.id);
    if (gp || bp) {
      int di = 0;
      for (size_t i = 0; i < s->scratch.size(); ++i)
        if (s->scratch[i].device == sh.device) di = (int)i;
      if (bp) {
        tanq::BlockParams p = *bp;
        p.blob = (*prog)[di];
        p.tp_lo = td.lo;
        p.tp_m = td.m;
        g_err.clear();
        const cudaError_t be = tanq::launch_block_group(sh.data, p, s->L, sh.stream);
        if (be != cudaSuccess)
          return fail(TANQ_E_CUDA, std::string("launch_block_group -> ") + cudaGetErrorString(be) +
                                       (g_err.empty() ? "" : " [" + g_err + "]"));
      } else {
        tanq::GroupParams p = *gp;
        p.prog = (*prog)[di];
        p.tp_lo = td.lo;
        p.tp_m = td.m;
        CUDA_TRY(tanq::launch_group3(sh.data, p, sh.stream));
      }
    } else if (k == 1) {
      tanq::GateParams<1> p;
      std::memcpy(p.S, Sm.data(), sizeof(p.S));
      for (int t = 0; t < 2; ++t) {
        p.pos[t] = (uint32_t)mm.bits[t].first;
        p.lo_mask[t] = ((uint64_t)1 << mm.bits[t].first) - 1;
      }
      p.n_tuples = n_tuples;
      p.mirror = mir ? 1u : 0u;
      p.tp_lo = td.lo;
      p.tp_m = td.m;
      CUDA_TRY(tanq::launch_gate1(sh.data, p, sh.stream));
    } else if (k == 2) {
      tanq::GateParams<2> p;
      std::memcpy(p.S, Sm.data(), sizeof(p.S));
      for (int t = 0; t < 4; ++t) {
        p.pos[t] = (uint32_t)mm.bits[t].first;
        p.lo_mask[t] = ((uint64_t)1 << mm.bits[t].first) - 1;
      }
      p.n_tuples = n_tuples;
      p.mirror = mir ? 1u : 0u;
      p.tp_lo = td.lo;
      p.tp_m = td.m;
      CUDA_TRY(tanq::launch_gate2(sh.data, p, sh.stream));
    } else {
      return fail(TANQ_E_UNSUPPORTED, "k >= 3 op without a group program");
    }
    s->launches++;
    prof_end(s, sh, pr);
  }
  if (mir_op) s->packed = true;
  if (!op.herm) s->herm_state = false;
  return TANQ_OK;
}

tanq_status ensure_frag_capacity(tanq_sim* s, DevScratch& d, size_t elems) {
  if (d.frag_elems >= elems) return TANQ_OK;
  CUDA_TRY(cudaSetDevice(d.device));
  if (d.frag) CUDA_TRY(cudaFree(d.frag));
  CUDA_TRY(cudaMalloc(&d.frag, elems * sizeof(double2)));
  d.frag_elems = elems;
  return TANQ_OK;
}

// 5-qubit block groups (k_max = 5) run only on the block kernel; where it cannot take one (a
// multi-shard layout, a small register, a group whose qubits do not cover physical bits 0..3)
// the group's sub-ops run as separate ops -- the same product, one pass each.
const std::vector<FusedOp>& runnable_ops(const tanq_sim* s, const std::vector<FusedOp>& ops,
                                         std::vector<FusedOp>& storage) {
  auto needs = [&](const FusedOp& op) {
    return op.k == 5 && (s->shards.size() != 1 || s->par || !block_ok(s, op));
  };
  bool any = false;
  for (const auto& op : ops) any |= needs(op);
  if (!any) return ops;
  storage.clear();
  for (const auto& op : ops) {
    if (needs(op))
      storage.insert(storage.end(), op.sub.begin(), op.sub.end());
    else
      storage.push_back(op);
  }
  return storage;
}

// Execute a list of fused ops in order (remaps inserted as needed).
tanq_status exec_ops(tanq_sim* s, const std::vector<FusedOp>& ops_in) {
  std::vector<FusedOp> expanded;
  const std::vector<FusedOp>& ops = runnable_ops(s, ops_in, expanded);
  // K3 group programs depend on the layout at execution time, so they are built op by op
  // into a persistent pinned host buffer and copied (async) to each device before the launch.
  size_t total = 0;
  for (const auto& op : ops)
    if (op.k >= 2) total += prog_capacity(op);  // k = 2: tiled or not, decided at launch
  if (total) {
    for (auto& sh : s->shards) {
      DevScratch& d = scratch_for(s, sh.device);
      TRY(ensure_scratch(s, d));
      TRY(ensure_frag_capacity(s, d, total));
    }
    if (s->frag_done_pending) {  // previous H2D copies from the pinned buffer must be done
      CUDA_TRY(cudaEventSynchronize(s->frag_done));
      s->frag_done_pending = false;
    }
    if (s->frag_host_elems < total) {
      if (s->frag_host) CUDA_TRY(cudaFreeHost(s->frag_host));
      CUDA_TRY(cudaMallocHost(&s->frag_host, total * sizeof(double2)));
      s->frag_host_elems = total;
    }
  }
  size_t off = 0;
  tanq::GroupParams gp;
  tanq::BlockParams bp;
  for (size_t i = 0; i < ops.size(); ++i) {
    const FusedOp& op = ops[i];
    TRY(ensure_local(s, op, &ops, i + 1));
    const bool blk = block_ok(s, op);
    if (!blk && !uses_prog(s, op)) {
      TRY(launch_op(s, op, nullptr, nullptr));
      continue;
    }
    double2* hp = s->frag_host + off;
    size_t elems;
    if (blk) {
      elems = (build_block(s, op, bp, reinterpret_cast<unsigned char*>(hp)) + 15) / 16;
    } else {
      build_group(s, op, gp, hp);
      elems = gp.prog_elems;
    }
    std::vector<const double2*> ptrs(s->scratch.size(), nullptr);
    for (auto& sh : s->shards) {
      int di = 0;
      for (size_t q = 0; q < s->scratch.size(); ++q)
        if (s->scratch[q].device == sh.device) di = (int)q;
      if (!ptrs[di]) {
        double2* dst = s->scratch[di].frag + off;
        CUDA_TRY(cudaSetDevice(sh.device));
        CUDA_TRY(cudaMemcpyAsync(dst, hp, elems * sizeof(double2), cudaMemcpyHostToDevice,
                                 sh.stream));
        ptrs[di] = dst;
      }
    }
    off += elems;
    if (blk)
      TRY(launch_op(s, op, nullptr, &ptrs, &bp));
    else
      TRY(launch_op(s, op, &gp, &ptrs));
  }
  if (total) {
    Shard& s0 = s->shards[0];
    for (auto& sh : s->shards) TRY(stream_wait(s0, sh));
    CUDA_TRY(cudaSetDevice(s0.device));
    if (!s->frag_done) CUDA_TRY(cudaEventCreateWithFlags(&s->frag_done, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(s->frag_done, s0.stream));
    s->frag_done_pending = true;
  }
  return TANQ_OK;
}

tanq_status check_qubits(const tanq_sim* s, int k, const int* q) {
  if (k < 1 || k > 3) return fail(TANQ_E_ARG, "k must be 1..3");
  if (!q) return fail(TANQ_E_ARG, "qubits is NULL");
  for (int i = 0; i < k; ++i) {
    if (q[i] < 0 || q[i] >= s->n) return fail(TANQ_E_ARG, "qubit out of range");
    for (int j = 0; j < i; ++j)
      if (q[i] == q[j]) return fail(TANQ_E_ARG, "repeated qubit");
  }
  if (2 * k > s->L) return fail(TANQ_E_ARG, "op needs more local bits than a shard holds");
  return TANQ_OK;
}

Mat mat_from(const tanq_c64* m, int d) {
  Mat M(d);
  for (int i = 0; i < d * d; ++i) M.a[i] = cd(m[i].re, m[i].im);
  return M;
}

bool finite_mat(const Mat& M) {
  for (const cd& v : M.a)
    if (!std::isfinite(v.real()) || !std::isfinite(v.imag())) return false;
  return true;
}

// Noise binding (Sec. 3.5; readings R4-R10): one superoperator per circuit op.
tanq_status bind_op(const tanq_sim* s, const tanq_op& op, const tanq_noise_model* nm,
                    const std::map<std::tuple<int, int, int>, const tanq_gate_cal*>& cal,
                    FusedOp& out) {
  const int kind = op.kind;
  if (kind < 0 || kind >= TANQ_N_KINDS) return fail(TANQ_E_ARG, "unknown op kind");
  int k = kind_arity(kind);
  if (k == 0) k = op.k;
  if (kind_arity(kind) && op.k != 0 && op.k != k) return fail(TANQ_E_ARG, "k does not match gate");
  TRY(check_qubits(s, k, op.q));
  out.k = k;
  for (int j = 0; j < k; ++j) out.q[j] = op.q[j];
  const int d = 1 << k;
  if (kind == TANQ_U || kind == TANQ_KRAUS || kind == TANQ_SUPEROP) {
    if (!op.m) return fail(TANQ_E_ARG, "matrix payload is NULL");
    if (kind == TANQ_U) {
      Mat U = mat_from(op.m, d);
      if (!finite_mat(U)) return fail(TANQ_E_ARG, "non-finite matrix");
      out.S = superop_from_kraus({U});
    } else if (kind == TANQ_KRAUS) {
      if (op.n_kraus < 1) return fail(TANQ_E_ARG, "n_kraus < 1");
      std::vector<Mat> Ks;
      for (int i = 0; i < op.n_kraus; ++i) Ks.push_back(mat_from(op.m + (size_t)i * d * d, d));
      out.S = superop_from_kraus(Ks);
    } else {
      out.S = mat_from(op.m, d * d);
      out.herm = is_herm_preserving(out.S, k);
    }
    if (!finite_mat(out.S)) return fail(TANQ_E_ARG, "non-finite matrix");
    return TANQ_OK;
  }
  if (kind == TANQ_RESET) {  // {|0><0|, |0><1|}: noiseless, no calibration (reading R19)
    Mat K0(2), K1(2);
    K0(0, 0) = 1.0;
    K1(0, 1) = 1.0;
    out.S = superop_from_kraus({K0, K1});
    return TANQ_OK;
  }
  if ((kind == TANQ_RX || kind == TANQ_RY || kind == TANQ_RZ || kind == TANQ_CP) &&
      !std::isfinite(op.theta))
    return fail(TANQ_E_ARG, "non-finite theta");
  Mat S = superop_from_kraus({gate_unitary(kind, op.theta)});
  if (!nm || kind == TANQ_RZ) {  // RZ noiseless
    out.S = S;
    return TANQ_OK;
  }
  auto it = cal.find({kind, op.q[0], k == 2 ? op.q[1] : -1});
  if (it == cal.end())
    return fail(TANQ_E_ARG, "missing calibration for kind " + std::to_string(kind) + " on qubit " +
                                std::to_string(op.q[0]));
  const tanq_gate_cal& gc = *it->second;
  if (gc.overrot_rad != 0.0) S = matmul(superop_from_kraus({overrot_unitary(k, gc.overrot_rad)}), S);
  Mat Sth = identity(d * d);
  bool has_th = false;
  const double t_us = gc.duration_ns * 1e-3;
  if (t_us > 0.0) {
    for (int j = 0; j < k; ++j) {
      const tanq_qubit_cal& qc = nm->qubits[op.q[j]];
      if (qc.t1_us <= 0.0) continue;
      Sth = matmul(embed_superop(superop_thermal(qc.t1_us, qc.t2_us, t_us), {j}, k), Sth);
      has_th = true;
    }
  }
  const bool has_dep = gc.depol_p != 0.0;
  const Mat Sdep = has_dep ? superop_depol(k, gc.depol_p) : Mat();
  if (nm->order == 0) {
    if (has_th) S = matmul(Sth, S);
    if (has_dep) S = matmul(Sdep, S);
  } else {
    if (has_dep) S = matmul(Sdep, S);
    if (has_th) S = matmul(Sth, S);
  }
  out.S = S;
  return TANQ_OK;
}

tanq_status validate_noise(const tanq_sim* s, const tanq_noise_model* nm,
                           std::map<std::tuple<int, int, int>, const tanq_gate_cal*>& cal) {
  if (!nm) return TANQ_OK;
  if (nm->n != s->n || !nm->qubits) return fail(TANQ_E_ARG, "noise model size mismatch");
  if (nm->order != 0 && nm->order != 1) return fail(TANQ_E_ARG, "noise order must be 0 or 1");
  for (int q = 0; q < nm->n; ++q) {
    const tanq_qubit_cal& qc = nm->qubits[q];
    if (qc.t1_us > 0.0 && (!(qc.t2_us > 0.0) || qc.t2_us > 2.0 * qc.t1_us))
      return fail(TANQ_E_ARG, "T2 must be in (0, 2 T1] on qubit " + std::to_string(q));
  }
  for (uint64_t i = 0; i < nm->n_gates; ++i) {
    const tanq_gate_cal& g = nm->gates[i];
    if (!(g.depol_p >= 0.0 && g.depol_p <= 1.0))
      return fail(TANQ_E_ARG, "depolarizing p outside [0,1]");
    if (!(g.duration_ns >= 0.0) || !std::isfinite(g.overrot_rad))
      return fail(TANQ_E_ARG, "bad duration / over-rotation");
    int k = kind_arity(g.kind);
    if (k == 0) return fail(TANQ_E_ARG, "calibration for a non-named gate kind");
    cal[{g.kind, g.q[0], k == 2 ? g.q[1] : -1}] = &g;
  }
  return TANQ_OK;
}

tanq_status apply_single(tanq_sim* s, FusedOp op) {
  std::vector<FusedOp> ops{std::move(op)};
  return exec_ops(s, ops);
}

tanq_status combine_probs(tanq_sim* s, DevScratch*& primary) {
  // every shard writes its owned diagonal entries into its device's buffer
  std::vector<DevScratch*> devs;
  for (auto& sh : s->shards) {
    DevScratch& d = scratch_for(s, sh.device);
    TRY(ensure_scratch(s, d));
    if (std::find(devs.begin(), devs.end(), &d) == devs.end()) {
      devs.push_back(&d);
      CUDA_TRY(cudaSetDevice(sh.device));
      CUDA_TRY(cudaMemsetAsync(d.probs, 0, sizeof(double) << s->n, sh.stream));
      CUDA_TRY(cudaMemsetAsync(d.imax, 0, sizeof(unsigned long long), sh.stream));
    }
  }
  tanq::BitMap bm = bitmap_of(s);
  for (auto& sh : s->shards) {
    DevScratch& d = scratch_for(s, sh.device);
    CUDA_TRY(cudaSetDevice(sh.device));
    // shards sharing a device share a stream: order is implied; otherwise wait
    CUDA_TRY(tanq::launch_diag(sh.data, d.probs, d.imax, bm, s->n, s->L, (uint64_t)sh.id,
                               sh.stream));
    s->launches++;
  }
  Shard& s0 = s->shards[0];
  primary = &scratch_for(s, s0.device);
  if (devs.size() > 1) {
    for (auto& sh : s->shards) TRY(stream_wait(s0, sh));
    CUDA_TRY(cudaSetDevice(s0.device));
    for (DevScratch* d : devs) {
      if (d == primary) continue;
      CUDA_TRY(cudaMemcpyPeerAsync(primary->probs_tmp, s0.device, d->probs, d->device,
                                   sizeof(double) << s->n, s0.stream));
      CUDA_TRY(tanq::launch_add(primary->probs, primary->probs_tmp, (uint64_t)1 << s->n,
                                s0.stream));
      s->launches++;
    }
  }
  if (s->dist && s->world > 1) {
    CUDA_TRY(cudaSetDevice(s0.device));
    NCCL_TRY(nccl().AllReduce(primary->probs, primary->probs, (size_t)1 << s->n, ncclDouble, ncclSum,
                           s->comm, s0.stream));
    // every rank must take the same TANQ_E_STATE decision: max of |Im diag| over ranks (the
    // bit patterns of non-negative doubles order like the values)
    NCCL_TRY(nccl().AllReduce(primary->imax, primary->imax, 1, ncclUint64, ncclMax, s->comm,
                              s0.stream));
  }
  // |Im diag| check (stream-ordered read: the library streams are non-blocking)
  double imx = 0.0;
  for (DevScratch* d : devs) {
    unsigned long long bits = 0;
    cudaStream_t st = s0.stream;
    for (auto& sh : s->shards)
      if (sh.device == d->device) st = sh.stream;
    CUDA_TRY(cudaSetDevice(d->device));
    CUDA_TRY(cudaMemcpyAsync(&bits, d->imax, sizeof(bits), cudaMemcpyDeviceToHost, st));
    TRY(host_wait(s, st));
    double v;
    std::memcpy(&v, &bits, sizeof(v));
    imx = std::max(imx, v);
  }
  if (imx >= 1e-6) return fail(TANQ_E_STATE, "|Im diag| = " + std::to_string(imx) + " >= 1e-6");
  return TANQ_OK;
}

}  // namespace

// ======================================================================================
// C ABI
// ======================================================================================
static int ilog2(int x) {
  int l = 0;
  while ((1 << l) < x) ++l;
  return l;
}

extern "C" {

const char* tanq_last_error(void) { return g_err.c_str(); }

static tanq_status create_common(int n, tanq_sim* s) {
  const size_t shard_bytes = sizeof(double2) << s->L;
  for (auto& sh : s->shards) {
    CUDA_TRY(cudaSetDevice(sh.device));
    size_t fr = 0, tot = 0;
    CUDA_TRY(cudaMemGetInfo(&fr, &tot));
    int same = 0;
    for (auto& o : s->shards) same += (o.device == sh.device && o.data == nullptr && !o.external);
    const size_t need = shard_bytes * (size_t)same + ((size_t)64 << 20) +
                        (s->dist ? 4 * s->xchunk * sizeof(double2) : 0) + (sizeof(double) * 3 << n);
    if (need > fr)
      return fail(TANQ_E_NOMEM, "memory guard: need " + std::to_string(need) + " B, free " +
                                    std::to_string(fr) + " B on device " +
                                    std::to_string(sh.device));
    // one stream per device (shards on the same device share it)
    for (auto& o : s->shards)
      if (o.device == sh.device && o.stream && &o != &sh) sh.stream = o.stream;
    if (!sh.stream) {
      CUDA_TRY(cudaStreamCreateWithFlags(&sh.stream, cudaStreamNonBlocking));
      s->owned.push_back({sh.device, sh.stream});
    }
    if (!sh.external) CUDA_TRY(cudaMalloc(&sh.data, shard_bytes));
    CUDA_TRY(tanq::launch_init(sh.data, (uint64_t)1 << s->L, sh.id == 0, sh.stream));
    s->launches++;
  }
  // peer access between distinct devices
  for (auto& a : s->shards)
    for (auto& b : s->shards)
      if (a.device != b.device) {
        int ok = 0;
        cudaDeviceCanAccessPeer(&ok, a.device, b.device);
        if (ok) {
          cudaSetDevice(a.device);
          cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            return fail(TANQ_E_CUDA, "peer access");
          cudaGetLastError();
        }
      }
  reset_layout(s);
  {
    const char* mv = getenv("TANQ_MIRROR");
    s->mirror_allowed = !(mv && mv[0] == '0');
  }
  s->herm_state = true;
  return TANQ_OK;
}

tanq_status tanq_create(int n_qubits, int n_shards, tanq_sim** out) {
  if (!out) return fail(TANQ_E_ARG, "out is NULL");
  *out = nullptr;
  if (n_qubits < 1 || n_qubits > 24) return fail(TANQ_E_ARG, "n_qubits must be in [1, 24]");
  if (n_shards != 1 && n_shards != 2 && n_shards != 4 && n_shards != 8)
    return fail(TANQ_E_ARG, "n_shards must be 1, 2, 4 or 8");
  const int L = 2 * n_qubits - ilog2(n_shards);
  if (L < 2) return fail(TANQ_E_ARG, "too few local bits for this shard count");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
    cudaGetLastError();
    return fail(TANQ_E_UNSUPPORTED, "no CUDA device");
  }
  tanq_sim* s = new tanq_sim();
  s->n = n_qubits;
  s->L = L;
  s->world = n_shards;
  s->rank0 = 0;
  s->parity = parity_layout_for(n_qubits, n_shards);
  for (int g = 0; g < n_shards; ++g) {
    Shard sh;
    sh.id = g;
    sh.device = g % ndev;
    s->shards.push_back(sh);
  }
  tanq_status st = create_common(n_qubits, s);
  if (st != TANQ_OK) {
    tanq_destroy(s);
    return st;
  }
  *out = s;
  return TANQ_OK;
}

tanq_status tanq_create_ex(int n_qubits, int n_shards, void* const* buffers, const int* devices,
                           size_t bytes_each, tanq_sim** out) {
  if (!out || !buffers || !devices) return fail(TANQ_E_ARG, "NULL argument");
  *out = nullptr;
  if (n_qubits < 1 || n_qubits > 24) return fail(TANQ_E_ARG, "n_qubits must be in [1, 24]");
  if (n_shards != 1 && n_shards != 2 && n_shards != 4 && n_shards != 8)
    return fail(TANQ_E_ARG, "n_shards must be 1, 2, 4 or 8");
  const int L = 2 * n_qubits - ilog2(n_shards);
  if (L < 2) return fail(TANQ_E_ARG, "too few local bits for this shard count");
  if (bytes_each < (sizeof(double2) << L))
    return fail(TANQ_E_ARG, "buffer smaller than 16 * 4^n / n_shards bytes");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
    cudaGetLastError();
    return fail(TANQ_E_UNSUPPORTED, "no CUDA device");
  }
  for (int g = 0; g < n_shards; ++g) {
    if (!buffers[g] || (reinterpret_cast<uintptr_t>(buffers[g]) & 15))
      return fail(TANQ_E_ARG, "shard buffer NULL or not 16-byte aligned");
    if (devices[g] < 0 || devices[g] >= ndev) return fail(TANQ_E_ARG, "bad device");
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, buffers[g]) != cudaSuccess || pa.type != cudaMemoryTypeDevice ||
        pa.device != devices[g]) {
      cudaGetLastError();
      return fail(TANQ_E_ARG, "shard buffer is not device memory of the given device");
    }
  }
  tanq_sim* s = new tanq_sim();
  s->n = n_qubits;
  s->L = L;
  s->world = n_shards;
  s->rank0 = 0;
  s->parity = parity_layout_for(n_qubits, n_shards);
  for (int g = 0; g < n_shards; ++g) {
    Shard sh;
    sh.id = g;
    sh.device = devices[g];
    sh.data = static_cast<double2*>(buffers[g]);
    sh.external = true;
    s->shards.push_back(sh);
  }
  tanq_status st = create_common(n_qubits, s);
  if (st != TANQ_OK) {
    tanq_destroy(s);
    return st;
  }
  *out = s;
  return TANQ_OK;
}

tanq_status tanq_nccl_unique_id(void* out, size_t len) {
  if (!out || len < sizeof(ncclUniqueId)) return fail(TANQ_E_ARG, "need 128 bytes");
  ncclUniqueId id;
  if (!nccl().ok) return fail(TANQ_E_UNSUPPORTED, "libnccl.so.2 not loadable");
  NCCL_TRY(nccl().GetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
  return TANQ_OK;
}

tanq_status tanq_create_dist(int n_qubits, int world_size, int rank, int device,
                             const void* nccl_uid, tanq_sim** out) {
  if (!out) return fail(TANQ_E_ARG, "out is NULL");
  *out = nullptr;
  if (n_qubits < 1 || n_qubits > 24) return fail(TANQ_E_ARG, "n_qubits must be in [1, 24]");
  if (world_size != 1 && world_size != 2 && world_size != 4 && world_size != 8)
    return fail(TANQ_E_ARG, "world_size must be 1, 2, 4 or 8");
  if (rank < 0 || rank >= world_size) return fail(TANQ_E_ARG, "rank out of range");
  if (world_size > 1 && !nccl_uid) return fail(TANQ_E_ARG, "nccl_uid required");
  const int L = 2 * n_qubits - ilog2(world_size);
  if (L < 2) return fail(TANQ_E_ARG, "too few local bits for this world size");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
    cudaGetLastError();
    return fail(TANQ_E_UNSUPPORTED, "no CUDA device");
  }
  if (device < 0 || device >= ndev) return fail(TANQ_E_ARG, "device out of range");
  tanq_sim* s = new tanq_sim();
  s->n = n_qubits;
  s->L = L;
  s->world = world_size;
  s->rank0 = rank;
  s->dist = true;
  s->parity = parity_layout_for(n_qubits, world_size);
  Shard sh;
  sh.id = rank;
  sh.device = device;
  s->shards.push_back(sh);
  // 2 x 2 staging slots of 128 MiB (pipelined exchange); env TANQ_XCHUNK_LOG2 (tests) caps
  // a slot at 2^k elements so small states still run several chunks
  int xlog = 23;
  if (const char* e = std::getenv("TANQ_XCHUNK_LOG2")) xlog = std::max(4, std::min(23, std::atoi(e)));
  s->xchunk = std::min<size_t>((size_t)1 << xlog, (size_t)1 << (L > 2 ? L - 2 : 0));
  tanq_status st = create_common(n_qubits, s);
  if (st == TANQ_OK && world_size > 1) {
    cudaSetDevice(device);
    if (cudaMalloc(&s->xsend, 2 * s->xchunk * sizeof(double2)) != cudaSuccess ||
        cudaMalloc(&s->xrecv, 2 * s->xchunk * sizeof(double2)) != cudaSuccess ||
        cudaStreamCreateWithFlags(&s->xstream, cudaStreamNonBlocking) != cudaSuccess)
      st = fail(TANQ_E_NOMEM, "staging");
    for (int j = 0; j < 2 && st == TANQ_OK; ++j)
      if (cudaEventCreateWithFlags(&s->xev_pack[j], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&s->xev_comm[j], cudaEventDisableTiming) != cudaSuccess)
        st = fail(TANQ_E_CUDA, "exchange events");
    ncclUniqueId id;
    std::memcpy(&id, nccl_uid, sizeof(id));
    if (st == TANQ_OK) {
      if (!nccl().ok) {
        st = fail(TANQ_E_UNSUPPORTED, "libnccl.so.2 not loadable");
      } else {
        ncclResult_t r = nccl().CommInitRank(&s->comm, world_size, id, rank);
        if (r != ncclSuccess) st = fail(TANQ_E_NCCL, nccl().GetErrorString(r));
      }
    }
  }
  if (st != TANQ_OK) {
    tanq_destroy(s);
    return st;
  }
  *out = s;
  return TANQ_OK;
}

tanq_status tanq_plan_destroy(tanq_plan* p);

tanq_status tanq_destroy(tanq_sim* s) {
  if (!s) return TANQ_OK;
  for (auto& e : s->plan_cache) tanq_plan_destroy(e.plan);
  s->plan_cache.clear();
  for (auto& p : s->prof) {
    cudaEventDestroy(p.e0);
    cudaEventDestroy(p.e1);
  }
  for (cudaEvent_t e : s->event_pool) cudaEventDestroy(e);
  for (auto& sh : s->shards) {
    cudaSetDevice(sh.device);
    if (sh.stream) cudaStreamSynchronize(sh.stream);
    if (sh.data && !sh.external) cudaFree(sh.data);
  }
  for (auto& p : s->owned) {
    cudaSetDevice(p.first);
    cudaStreamDestroy(p.second);
  }
  for (auto& d : s->scratch) {
    cudaSetDevice(d.device);
    cudaFree(d.probs);
    cudaFree(d.probs_tmp);
    cudaFree(d.cdf);
    cudaFree(d.partial);
    cudaFree(d.scal);
    cudaFree(d.imax);
    cudaFree(d.stage);
    cudaFree(d.frag);
  }
  if (s->frag_host) cudaFreeHost(s->frag_host);
  if (s->frag_done) cudaEventDestroy(s->frag_done);
  if (s->xsend) cudaFree(s->xsend);
  if (s->xrecv) cudaFree(s->xrecv);
  if (s->xstream) cudaStreamDestroy(s->xstream);
  for (int j = 0; j < 2; ++j) {
    if (s->xev_pack[j]) cudaEventDestroy(s->xev_pack[j]);
    if (s->xev_comm[j]) cudaEventDestroy(s->xev_comm[j]);
  }
  if (s->comm) nccl().CommDestroy(s->comm);
  cudaGetLastError();
  delete s;
  return TANQ_OK;
}

tanq_status tanq_reset(tanq_sim* s) {
  if (!s) return fail(TANQ_E_ARG, "NULL handle");
  for (auto& sh : s->shards) {
    CUDA_TRY(cudaSetDevice(sh.device));
    CUDA_TRY(tanq::launch_init(sh.data, (uint64_t)1 << s->L, sh.id == 0, sh.stream));
    s->launches++;
  }
  reset_layout(s);
  s->herm_state = true;
  s->packed = false;
  return TANQ_OK;
}

tanq_status tanq_info_get(tanq_sim* s, tanq_info* o) {
  if (!s || !o) return fail(TANQ_E_ARG, "NULL");
  std::memset(o, 0, sizeof(*o));
  o->n_qubits = s->n;
  o->n_shards = (int)s->shards.size();
  o->world_size = s->world;
  o->rank = s->rank0;
  o->local_bits = s->L;
  for (int q = 0; q < s->n && q < 32; ++q) {
    o->rowpos[q] = (int)s->phys[2 * q];
    o->colpos[q] = (int)s->phys[2 * q + 1];
  }
  o->shard_bytes = sizeof(double2) << s->L;
  o->parity_qubits = s->par;
  return TANQ_OK;
}

tanq_status tanq_set_stream(tanq_sim* s, int shard, void* stream) {
  if (!s || shard < 0 || shard >= (int)s->shards.size()) return fail(TANQ_E_ARG, "bad shard");
  Shard& sh = s->shards[shard];
  CUDA_TRY(cudaSetDevice(sh.device));
  TRY(host_wait(s, sh.stream));
  cudaStream_t ns = stream ? (cudaStream_t)stream : s->own_streams_of(sh.device);
  for (auto& o : s->shards)
    if (o.device == sh.device) o.stream = ns;
  return TANQ_OK;
}

tanq_status tanq_apply_gate(tanq_sim* s, int k, const int* qubits, const tanq_c64* U) {
  if (!s) return fail(TANQ_E_ARG, "NULL handle");
  TRY(check_qubits(s, k, qubits));
  if (!U) return fail(TANQ_E_ARG, "U is NULL");
  FusedOp op;
  op.k = k;
  for (int j = 0; j < k; ++j) op.q[j] = qubits[j];
  Mat G = mat_from(U, 1 << k);
  if (!finite_mat(G)) return fail(TANQ_E_ARG, "non-finite matrix");
  op.S = superop_from_kraus({G});
  return apply_single(s, std::move(op));
}

tanq_status tanq_apply_channel(tanq_sim* s, int k, const int* qubits, int m, const tanq_c64* kraus,
                               int check_cptp) {
  if (!s) return fail(TANQ_E_ARG, "NULL handle");
  TRY(check_qubits(s, k, qubits));
  if (!kraus || m < 1) return fail(TANQ_E_ARG, "empty Kraus list");
  const int d = 1 << k;
  std::vector<Mat> Ks;
  for (int i = 0; i < m; ++i) {
    Ks.push_back(mat_from(kraus + (size_t)i * d * d, d));
    if (!finite_mat(Ks.back())) return fail(TANQ_E_ARG, "non-finite matrix");
  }
  if (check_cptp) {
    Mat sum(d);
    for (const Mat& K : Ks)
      for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j)
          for (int l = 0; l < d; ++l) sum(i, j) += std::conj(K(l, i)) * K(l, j);
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j)
        if (std::abs(sum(i, j) - (i == j ? 1.0 : 0.0)) > 1e-12)
          return fail(TANQ_E_ARG, "channel is not trace preserving (sum K^dag K != I)");
  }
  FusedOp op;
  op.k = k;
  for (int j = 0; j < k; ++j) op.q[j] = qubits[j];
  op.S = superop_from_kraus(Ks);
  return apply_single(s, std::move(op));
}

tanq_status tanq_apply_superop(tanq_sim* s, int k, const int* qubits, const tanq_c64* S) {
  if (!s) return fail(TANQ_E_ARG, "NULL handle");
  TRY(check_qubits(s, k, qubits));
  if (!S) return fail(TANQ_E_ARG, "S is NULL");
  FusedOp op;
  op.k = k;
  for (int j = 0; j < k; ++j) op.q[j] = qubits[j];
  op.S = mat_from(S, 1 << (2 * k));
  if (!finite_mat(op.S)) return fail(TANQ_E_ARG, "non-finite matrix");
  op.herm = is_herm_preserving(op.S, k);
  return apply_single(s, std::move(op));
}

}  // extern "C"

struct tanq_plan {
  int n = 0;
  std::vector<FusedOp> ops;
  uint64_t ops_in = 0;
  double plan_ms = 0;
  int flags = 0;
  // CUDA-graph replay cache (flags bit1, single-shard handles): valid for one handle, one
  // shard buffer and one starting layout; group programs live in a plan-owned device buffer.
  struct GraphCache {
    const tanq_sim* sim = nullptr;
    const double2* data = nullptr;
    uint32_t phys[64];
    bool herm = false, mirror = false, packed = false, packed_end = false;
    cudaGraphExec_t exec = nullptr;
    double2* dprog = nullptr;
    int device = -1;
    uint64_t kernels = 0;
  };
  mutable GraphCache g;
  ~tanq_plan() {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.dprog) {
      cudaSetDevice(g.device);
      cudaFree(g.dprog);
    }
  }
};

namespace {
// Capture the whole plan as one CUDA graph (single shard: the layout never changes, so every
// kernel parameter is known before the first launch), then replay it.
tanq_status exec_graph(tanq_sim* s, const tanq_plan* p) {
  Shard& sh = s->shards[0];
  auto& g = p->g;
  std::vector<FusedOp> expanded;
  const std::vector<FusedOp>& ops = runnable_ops(s, p->ops, expanded);
  const bool hit = g.exec && g.sim == s && g.data == sh.data && g.herm == s->herm_state &&
                   g.mirror == s->mirror_allowed && g.packed == s->packed &&
                   std::memcmp(g.phys, s->phys, sizeof(g.phys)) == 0;
  CUDA_TRY(cudaSetDevice(sh.device));
  if (const char* e = std::getenv("TANQ_GRAPH_DEBUG"); e && e[0] == '1')
    std::fprintf(stderr, "exec_graph: %s (exec %d sim %d data %d herm %d mirror %d packed %d phys %d)\n",
                 hit ? "replay" : "capture", g.exec != nullptr, g.sim == s, g.data == sh.data,
                 g.herm == s->herm_state, g.mirror == s->mirror_allowed, g.packed == s->packed,
                 std::memcmp(g.phys, s->phys, sizeof(g.phys)) == 0);
  if (!hit) {
    if (g.exec) {
      CUDA_TRY(cudaGraphExecDestroy(g.exec));
      g.exec = nullptr;
    }
    if (g.dprog) {
      CUDA_TRY(cudaSetDevice(g.device));
      CUDA_TRY(cudaFree(g.dprog));
      g.dprog = nullptr;
      CUDA_TRY(cudaSetDevice(sh.device));
    }
    size_t total = 0;
    for (const auto& op : ops)
      if (op.k >= 2) total += prog_capacity(op);  // upper bound (k = 2 may run direct)
    std::vector<double2> host(total ? total : 1);
    std::vector<tanq::GroupParams> gps;
    std::vector<tanq::BlockParams> bps;
    std::vector<size_t> elems;
    std::vector<int> kind;  // per op: 0 direct, 1 group, 2 block
    size_t off = 0;
    const bool herm_in = s->herm_state;
    for (const auto& op : ops) {  // the Hermitian flag as it will be when op runs
      if (block_ok(s, op)) {
        bps.emplace_back();
        const size_t e = (build_block(s, op, bps.back(), reinterpret_cast<unsigned char*>(
                                                             host.data() + off)) + 15) / 16;
        elems.push_back(e);
        kind.push_back(2);
        off += e;
      } else if (uses_prog(s, op)) {
        gps.emplace_back();
        build_group(s, op, gps.back(), host.data() + off);
        elems.push_back(gps.back().prog_elems);
        kind.push_back(1);
        off += gps.back().prog_elems;
      } else {
        kind.push_back(0);
        elems.push_back(0);
      }
      if (!op.herm) s->herm_state = false;
    }
    s->herm_state = herm_in;
    if (total) {
      CUDA_TRY(cudaMalloc(&g.dprog, total * sizeof(double2)));
      CUDA_TRY(cudaMemcpy(g.dprog, host.data(), total * sizeof(double2), cudaMemcpyHostToDevice));
    }
    g.device = sh.device;
    std::vector<const double2*> ptr(s->scratch.size() + 1, nullptr);
    int di = 0;
    for (size_t i = 0; i < s->scratch.size(); ++i)
      if (s->scratch[i].device == sh.device) di = (int)i;
    const bool herm0 = s->herm_state, packed0 = s->packed;
    cudaGraph_t graph;
    CUDA_TRY(cudaStreamBeginCapture(sh.stream, cudaStreamCaptureModeThreadLocal));
    const uint64_t l0 = s->launches;
    off = 0;
    size_t gi = 0, bi = 0;
    tanq_status st = TANQ_OK;
    for (size_t oi = 0; oi < ops.size(); ++oi) {
      const FusedOp& op = ops[oi];
      if (kind[oi] == 0) {
        st = launch_op(s, op, nullptr, nullptr);
      } else {
        ptr[di] = g.dprog + off;
        off += elems[oi];
        st = kind[oi] == 2 ? launch_op(s, op, nullptr, &ptr, &bps[bi++])
                           : launch_op(s, op, &gps[gi++], &ptr);
      }
      if (st != TANQ_OK) break;
    }
    cudaError_t ce = cudaStreamEndCapture(sh.stream, &graph);
    if (st != TANQ_OK) {
      if (ce == cudaSuccess) cudaGraphDestroy(graph);
      return st;
    }
    if (ce != cudaSuccess) return fail(TANQ_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    ce = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ce != cudaSuccess) return fail(TANQ_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
    g.kernels = s->launches - l0;
    s->launches = l0;
    g.sim = s;
    g.data = sh.data;
    g.herm = herm0;
    g.packed = packed0;
    g.packed_end = s->packed;
    g.mirror = s->mirror_allowed;
    std::memcpy(g.phys, s->phys, sizeof(g.phys));
  }
  CUDA_TRY(cudaGraphLaunch(g.exec, sh.stream));
  s->launches += g.kernels;
  s->packed = g.packed_end;
  for (const auto& op : ops)
    if (!op.herm) s->herm_state = false;
  return TANQ_OK;
}
}  // namespace

extern "C" {

static tanq_status plan_create(int n, int L, const tanq_circuit* c, const tanq_noise_model* nm,
                               const tanq_run_opts* o, tanq_plan** out) {
  if (!c || !out) return fail(TANQ_E_ARG, "NULL argument");
  *out = nullptr;
  if (c->n_ops && !c->ops) return fail(TANQ_E_ARG, "ops is NULL");
  tanq_run_opts opts{2, 3, 0, 0, 0};
  if (o) opts = *o;
  if (opts.fuse < 0 || opts.fuse > 2) return fail(TANQ_E_ARG, "fuse must be 0, 1 or 2");
  if (opts.k_max < 1 || opts.k_max > 5) return fail(TANQ_E_ARG, "k_max must be 1..5");
  if (opts.k_max == 5 && L < 14) opts.k_max = 4;  // 5-qubit block groups need block tuples
  if (opts.k_max == 4 && L < 10) opts.k_max = 3;  // 4-qubit tiles need 8 member bits + tuples
  if (opts.k_max == 3 && L < 6) opts.k_max = 2;
  const auto t0 = std::chrono::steady_clock::now();
  tanq_sim shape;  // only n and L are read by the validators
  shape.n = n;
  shape.L = L;
  std::map<std::tuple<int, int, int>, const tanq_gate_cal*> cal;
  TRY(validate_noise(&shape, nm, cal));
  std::vector<FusedOp> ops;
  ops.reserve(c->n_ops);
  for (uint64_t i = 0; i < c->n_ops; ++i) {
    FusedOp f;
    TRY(bind_op(&shape, c->ops[i], nm, cal, f));
    ops.push_back(std::move(f));
  }
  tanq_plan* p = new tanq_plan();
  p->n = n;
  p->ops = fuse(ops, opts.fuse, opts.k_max);
  if (const char* e = std::getenv("TANQ_PLAN_DUMP"); e && e[0] == '1') {  // diagnostics
    for (const auto& f : p->ops) {
      std::fprintf(stderr, "op k=%d subs=%zu q=", f.k, f.sub.size());
      for (int j = 0; j < f.k; ++j) std::fprintf(stderr, "%d%s", f.q[j], j + 1 < f.k ? "," : "");
      for (const auto& sb : f.sub) {
        std::fprintf(stderr, " [");
        for (int j = 0; j < sb.k; ++j) std::fprintf(stderr, "%d%s", sb.q[j], j + 1 < sb.k ? "," : "]");
      }
      std::fprintf(stderr, "\n");
    }
  }
  p->ops_in = c->n_ops;
  p->flags = opts.flags;
  p->plan_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  *out = p;
  return TANQ_OK;
}

tanq_status tanq_plan_create(tanq_sim* s, const tanq_circuit* c, const tanq_noise_model* nm,
                             const tanq_run_opts* o, tanq_plan** out) {
  if (!s) return fail(TANQ_E_ARG, "NULL handle");
  return plan_create(s->n, s->L, c, nm, o, out);
}

tanq_status tanq_plan_create_host(int n_qubits, int world_size, const tanq_circuit* c,
                                  const tanq_noise_model* nm, const tanq_run_opts* o,
                                  tanq_plan** out) {
  if (n_qubits < 1 || n_qubits > 24) return fail(TANQ_E_ARG, "n_qubits must be in [1, 24]");
  if (world_size != 1 && world_size != 2 && world_size != 4 && world_size != 8)
    return fail(TANQ_E_ARG, "world_size must be 1, 2, 4 or 8");
  const int L = 2 * n_qubits - ilog2(world_size);
  if (L < 2) return fail(TANQ_E_ARG, "too few local bits");
  return plan_create(n_qubits, L, c, nm, o, out);
}

tanq_status tanq_plan_info(const tanq_plan* p, tanq_run_stats* st) {
  if (!p || !st) return fail(TANQ_E_ARG, "NULL argument");
  std::memset(st, 0, sizeof(*st));
  st->ops_in = p->ops_in;
  st->ops_fused = p->ops.size();
    for (const auto& f : p->ops) st->gate_updates += f.sub.empty() ? 1 : f.sub.size();
  for (const auto& f : p->ops) st->n_k[f.k]++;
  st->plan_ms = p->plan_ms;
  return TANQ_OK;
}

tanq_status tanq_plan_schedule(const tanq_plan* p, int world_size, int32_t* items, uint64_t max,
                               uint64_t* n_items) {
  if (!p || !n_items) return fail(TANQ_E_ARG, "NULL argument");
  if (world_size != 1 && world_size != 2 && world_size != 4 && world_size != 8)
    return fail(TANQ_E_ARG, "world_size must be 1, 2, 4 or 8");
  const int L = 2 * p->n - ilog2(world_size);
  uint32_t phys[64];
  uint64_t par = 0;
  init_layout(phys, par, p->n, ilog2(world_size), parity_layout_for(p->n, world_size));
  uint64_t cnt = 0;
  auto put = [&](int32_t a, int32_t b, int32_t c) {
    if (items && cnt < max) {
      items[3 * cnt] = a;
      items[3 * cnt + 1] = b;
      items[3 * cnt + 2] = c;
    }
    ++cnt;
  };
  for (size_t i = 0; i < p->ops.size(); ++i) {
    if (2 * p->ops[i].k > L) return fail(TANQ_E_ARG, "op needs more local bits than a shard holds");
    for (auto& r : plan_remaps(phys, par, p->n, L, p->ops[i], &p->ops, i + 1)) {
      if (r.kind < 0) return fail(TANQ_E_ARG, "no local qubit available for remap");
      put(r.kind, r.a, r.b);
    }
    put(0, (int32_t)i, 0);
  }
  *n_items = cnt;
  return TANQ_OK;
}

// Instrumentation: the block-pipeline program of plan op i on a single-shard register in the
// initial interleaved layout (packed = 1: the packed Hermitian layout), exactly as the launch
// would build it.  *kind = 2 if the block kernel takes the op (params / blob written), else 0.
tanq_status tanq_plan_block_program(const tanq_plan* p, uint64_t i, int packed, void* params,
                                    size_t params_size, void* blob, size_t blob_cap, int* kind,
                                    size_t* blob_bytes) {
  if (!p || !kind) return fail(TANQ_E_ARG, "NULL argument");
  if (i >= p->ops.size()) return fail(TANQ_E_ARG, "op index out of range");
  tanq_sim shape;
  shape.n = p->n;
  shape.L = 2 * p->n;
  for (int b = 0; b < 64; ++b) shape.phys[b] = (uint32_t)b;
  shape.shards.resize(1);
  shape.herm_state = true;
  shape.mirror_allowed = packed != 0;
  *kind = 0;
  const FusedOp& op = p->ops[i];
  if (!block_ok(&shape, op)) return TANQ_OK;
  if (params_size != sizeof(tanq::BlockParams))
    return fail(TANQ_E_ARG, "params_size mismatch (sizeof BlockParams)");
  std::vector<unsigned char> tmp(block_blob_bytes(op) + 16);
  tanq::BlockParams bp;
  std::memset(&bp, 0, sizeof(bp));
  const size_t bytes = build_block(&shape, op, bp, tmp.data());
  if (blob_bytes) *blob_bytes = bytes;
  if (blob) {
    if (blob_cap < bytes) return fail(TANQ_E_ARG, "blob buffer too small");
    std::memcpy(blob, tmp.data(), bytes);
  }
  if (params) std::memcpy(params, &bp, sizeof(bp));
  *kind = 2;
  return TANQ_OK;
}

tanq_status tanq_plan_get_op(const tanq_plan* p, uint64_t i, int* k, int* qubits, tanq_c64* S) {
  if (!p || !k || !qubits) return fail(TANQ_E_ARG, "NULL argument");
  if (i >= p->ops.size()) return fail(TANQ_E_ARG, "op index out of range");
  const FusedOp& f = p->ops[i];
  *k = f.k;
  for (int j = 0; j < f.k; ++j) qubits[j] = f.q[j];
  if (S) {
    Mat D = f.S;
    if (!f.sub.empty()) {  // factored group: product of the embedded sub-ops, in order
      D = identity(1 << (2 * f.k));
      for (const FusedOp& sb : f.sub) {
        std::vector<int> pos;
        for (int j = 0; j < sb.k; ++j)
          for (int u = 0; u < f.k; ++u)
            if (f.q[u] == sb.q[j]) pos.push_back(u);
        D = matmul(embed_superop(sb.S, pos, f.k), D);
      }
    }
    for (size_t e = 0; e < D.a.size(); ++e) S[e] = tanq_c64{D.a[e].real(), D.a[e].imag()};
  }
  return TANQ_OK;
}

tanq_status tanq_plan_exec(tanq_sim* s, const tanq_plan* p, tanq_run_stats* st) {
  if (!s || !p) return fail(TANQ_E_ARG, "NULL argument");
  if (p->n != s->n) return fail(TANQ_E_ARG, "plan built for a different register size");
  for (const auto& f : p->ops)
    if (2 * f.k > s->L) return fail(TANQ_E_ARG, "op needs more local bits than a shard holds");
  const uint64_t r0 = s->remap_count, b0 = s->remap_bytes;
  const bool mirror_saved = s->mirror_allowed;
  if (p->flags & 4) s->mirror_allowed = false;
  tanq_status r;
  if ((p->flags & 2) && s->shards.size() == 1 && !s->dist && !(p->flags & 1)) {
    r = exec_graph(s, p);
  } else {
    s->prof_on = (p->flags & 1) != 0;
    r = exec_ops(s, p->ops);
    s->prof_on = false;
  }
  s->mirror_allowed = mirror_saved;
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->ops_in = p->ops_in;
    st->ops_fused = p->ops.size();
    for (const auto& f : p->ops) st->gate_updates += f.sub.empty() ? 1 : f.sub.size();
    for (const auto& f : p->ops) st->n_k[f.k]++;
    st->n_remaps = s->remap_count - r0;
    st->remap_bytes = s->remap_bytes - b0;
    st->plan_ms = p->plan_ms;
  }
  return r;
}

tanq_status tanq_plan_destroy(tanq_plan* p) {
  delete p;
  return TANQ_OK;
}

// tanq_run_circuit keeps the plans of the last kPlanCacheSize distinct (circuit, noise model,
// options) it ran, keyed by an exact byte serialisation of everything the plan depends on
// (ops with their matrix payloads, calibrations, fusion options) -- a repeated call skips
// noise binding, superoperator construction and fusion.  From the second run of the same
// single-shard plan on, its launches are replayed as one CUDA graph (flags bit1), unless
// per-kernel profiling (bit0) is requested.  Env TANQ_PLAN_CACHE=0 disables the cache.
namespace {
constexpr size_t kPlanCacheSize = 8;

void key_put(std::string& k, const void* p, size_t n) {
  k.append(reinterpret_cast<const char*>(p), n);
}

bool plan_key(const tanq_sim* s, const tanq_circuit* c, const tanq_noise_model* nm,
              const tanq_run_opts* o, std::string& k) {
  if (!c || (c->n_ops && !c->ops)) return false;
  k.clear();
  k.reserve(64 + c->n_ops * 48);
  key_put(k, &s->n, sizeof(s->n));
  key_put(k, &s->L, sizeof(s->L));
  tanq_run_opts opts{2, 3, 0, 0, 0};
  if (o) opts = *o;
  key_put(k, &opts.fuse, sizeof(opts.fuse));
  key_put(k, &opts.k_max, sizeof(opts.k_max));
  key_put(k, &opts.chunk_bytes, sizeof(opts.chunk_bytes));
  key_put(k, &opts.flags, sizeof(opts.flags));
  key_put(k, &c->n_ops, sizeof(c->n_ops));
  for (uint64_t i = 0; i < c->n_ops; ++i) {
    const tanq_op& op = c->ops[i];
    key_put(k, &op.kind, sizeof(op.kind));
    key_put(k, &op.k, sizeof(op.k));
    key_put(k, op.q, sizeof(op.q));
    key_put(k, &op.n_kraus, sizeof(op.n_kraus));
    key_put(k, &op.theta, sizeof(op.theta));
    if (op.m && op.k >= 1 && op.k <= 3) {
      const size_t d = (size_t)1 << op.k;
      size_t cnt = op.kind == TANQ_SUPEROP ? d * d * d * d
                                           : (op.kind == TANQ_KRAUS ? (size_t)std::max(0, op.n_kraus) * d * d : d * d);
      key_put(k, op.m, cnt * sizeof(tanq_c64));
    }
  }
  const int has_nm = nm != nullptr;
  key_put(k, &has_nm, sizeof(has_nm));
  if (nm) {
    if ((nm->n > 0 && !nm->qubits) || (nm->n_gates && !nm->gates)) return false;
    key_put(k, &nm->n, sizeof(nm->n));
    key_put(k, &nm->order, sizeof(nm->order));
    if (nm->n > 0) key_put(k, nm->qubits, (size_t)nm->n * sizeof(tanq_qubit_cal));
    key_put(k, &nm->n_gates, sizeof(nm->n_gates));
    if (nm->n_gates) key_put(k, nm->gates, nm->n_gates * sizeof(tanq_gate_cal));
  }
  return true;
}

bool plan_cache_on() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("TANQ_PLAN_CACHE");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}
}  // namespace

tanq_status tanq_run_circuit(tanq_sim* s, const tanq_circuit* c, const tanq_noise_model* nm,
                             const tanq_run_opts* o, tanq_run_stats* st) {
  if (!s) return fail(TANQ_E_ARG, "NULL handle");
  std::string key;
  if (!plan_cache_on() || !plan_key(s, c, nm, o, key)) {
    tanq_plan* p = nullptr;
    TRY(tanq_plan_create(s, c, nm, o, &p));
    tanq_status r = tanq_plan_exec(s, p, st);
    tanq_plan_destroy(p);
    return r;
  }
  PlanCacheEntry* hit = nullptr;
  for (auto& e : s->plan_cache)
    if (e.key == key) hit = &e;
  if (!hit) {
    tanq_plan* p = nullptr;
    TRY(tanq_plan_create(s, c, nm, o, &p));
    if (s->plan_cache.size() >= kPlanCacheSize) {  // evict the least recently used
      auto lru = std::min_element(s->plan_cache.begin(), s->plan_cache.end(),
                                  [](const PlanCacheEntry& a, const PlanCacheEntry& b) {
                                    return a.last_use < b.last_use;
                                  });
      tanq_plan_destroy(lru->plan);
      s->plan_cache.erase(lru);
    }
    s->plan_cache.push_back(PlanCacheEntry{std::move(key), p, 0, 0});
    hit = &s->plan_cache.back();
  } else {
    hit->hits++;
    if (hit->hits == 1 && !(hit->plan->flags & 1)) hit->plan->flags |= 2;  // replay as a graph
  }
  hit->last_use = ++s->plan_cache_clock;
  tanq_status r = tanq_plan_exec(s, hit->plan, st);
  if (st && hit->hits) st->plan_ms = 0.0;  // no planning on a cache hit
  return r;
}

tanq_status tanq_probs(tanq_sim* s, const tanq_readout* ro, double* probs) {
  if (!s || !probs) return fail(TANQ_E_ARG, "NULL argument");
  if (ro) {
    for (int q = 0; q < s->n; ++q) {
      double a = ro->p10 ? ro->p10[q] : 0.0, b = ro->p01 ? ro->p01[q] : 0.0;
      if (!(a >= 0.0 && a <= 1.0 && b >= 0.0 && b <= 1.0))
        return fail(TANQ_E_ARG, "readout probability outside [0,1]");
    }
  }
  DevScratch* pd = nullptr;
  TRY(combine_probs(s, pd));
  Shard& s0 = s->shards[0];
  CUDA_TRY(cudaSetDevice(s0.device));
  if (ro) {
    CUDA_TRY(tanq::launch_readout(pd->probs, s->n, ro->p10, ro->p01, s0.stream));
    s->launches += s->n;
  }
  CUDA_TRY(cudaMemcpyAsync(probs, pd->probs, sizeof(double) << s->n, cudaMemcpyDeviceToHost,
                           s0.stream));
  TRY(host_wait(s, s0.stream));
  return TANQ_OK;
}

tanq_status tanq_expect_pauli(tanq_sim* s, uint64_t xm, uint64_t zm, double* out_re,
                              double* out_im) {
  if (!s || !out_re) return fail(TANQ_E_ARG, "NULL argument");
  const uint64_t lim = s->n >= 64 ? ~0ull : ((1ull << s->n) - 1);
  if ((xm & ~lim) || (zm & ~lim)) return fail(TANQ_E_ARG, "Pauli mask outside the register");
  if (xm) TRY(ensure_unpacked(s));  // X / Y factors read off-diagonal elements
  tanq::BitMap bm = bitmap_of(s);
  const int nb = tanq::expect_blocks(s->n);
  double re = 0.0, im = 0.0;
  std::vector<double2> host(s->shards.size());
  for (size_t i = 0; i < s->shards.size(); ++i) {
    Shard& sh = s->shards[i];
    DevScratch& d = scratch_for(s, sh.device);
    TRY(ensure_scratch(s, d));
    CUDA_TRY(cudaSetDevice(sh.device));
    CUDA_TRY(tanq::launch_expect(sh.data, d.partial, nb, bm, s->n, s->L, (uint64_t)sh.id, xm, zm,
                                 sh.stream));
    CUDA_TRY(tanq::launch_reduce_partials(d.partial, nb, d.scal, sh.stream));
    s->launches += 2;
    if (s->dist && s->world > 1)
      NCCL_TRY(nccl().AllReduce(d.scal, d.scal, 2, ncclDouble, ncclSum, s->comm, sh.stream));
    CUDA_TRY(cudaMemcpyAsync(&host[i], d.scal, sizeof(double2), cudaMemcpyDeviceToHost,
                             sh.stream));
    TRY(host_wait(s, sh.stream));
  }
  for (auto& v : host) {
    re += v.x;
    im += v.y;
  }
  // global factor (-i)^{popc(x & z)}
  switch (__builtin_popcountll(xm & zm) & 3) {
    case 0: break;
    case 1: { double t = re; re = im; im = -t; break; }
    case 2: re = -re; im = -im; break;
    case 3: { double t = re; re = -im; im = t; break; }
  }
  *out_re = re;
  if (out_im) *out_im = im;
  return TANQ_OK;
}

tanq_status tanq_sample(tanq_sim* s, const tanq_readout* ro, uint64_t seed, uint64_t shots,
                        uint64_t* outcomes) {
  if (!s || (!outcomes && shots)) return fail(TANQ_E_ARG, "NULL argument");
  if (shots == 0) return TANQ_OK;
  DevScratch* pd = nullptr;
  TRY(combine_probs(s, pd));
  Shard& s0 = s->shards[0];
  CUDA_TRY(cudaSetDevice(s0.device));
  if (ro) {
    CUDA_TRY(tanq::launch_readout(pd->probs, s->n, ro->p10, ro->p01, s0.stream));
    s->launches += s->n;
  }
  CUDA_TRY(tanq::launch_cdf(pd->probs, pd->cdf, s->n, s0.stream));
  unsigned long long* dout = nullptr;
  CUDA_TRY(cudaMallocAsync(&dout, shots * sizeof(unsigned long long), s0.stream));
  CUDA_TRY(tanq::launch_sample(pd->cdf, s->n, seed, shots, dout, s0.stream));
  s->launches += 2;
  CUDA_TRY(cudaMemcpyAsync(outcomes, dout, shots * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                           s0.stream));
  CUDA_TRY(cudaFreeAsync(dout, s0.stream));
  TRY(host_wait(s, s0.stream));
  return TANQ_OK;
}

// Philox4x32-10 (same constants as the sampling kernel), first 53-bit uniform of (seed, 0).
static double philox_uniform(uint64_t seed, uint64_t ctr) {
  uint32_t c[4] = {(uint32_t)ctr, (uint32_t)(ctr >> 32), 0u, 0u};
  uint32_t k[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c[1] ^ k[0], n1 = lo1, n2 = hi0 ^ c[3] ^ k[1], n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    k[0] += 0x9E3779B9u;
    k[1] += 0xBB67AE85u;
  }
  const uint64_t bits = (((uint64_t)c[0] << 21) ^ ((uint64_t)c[1] >> 11)) & ((1ull << 53) - 1);
  return (double)bits * (1.0 / 9007199254740992.0);
}

tanq_status tanq_measure(tanq_sim* s, int qubit, uint64_t seed, int* outcome, double* prob) {
  if (!s) return fail(TANQ_E_ARG, "NULL handle");
  if (qubit < 0 || qubit >= s->n) return fail(TANQ_E_ARG, "qubit out of range");
  double z = 0.0;
  TRY(tanq_expect_pauli(s, 0, 1ull << qubit, &z, nullptr));  // <Z_q> = p0 - p1 (diagonal)
  const double p1 = std::min(1.0, std::max(0.0, 0.5 * (1.0 - z)));
  const int b = philox_uniform(seed, 0) < p1 ? 1 : 0;
  const double pb = b ? p1 : 1.0 - p1;
  if (pb < 1e-300) return fail(TANQ_E_STATE, "measured outcome has zero probability");
  FusedOp op;  // superoperator of rho -> P_b rho P_b / p_b : only the (b,b) block survives
  op.k = 1;
  op.q[0] = qubit;
  op.S = Mat(4);
  op.S(3 * b, 3 * b) = 1.0 / pb;
  TRY(apply_single(s, std::move(op)));
  if (outcome) *outcome = b;
  if (prob) *prob = pb;
  return TANQ_OK;
}

static tanq_status state_io(tanq_sim* s, uint64_t first, uint64_t count, tanq_c64* out,
                            const tanq_c64* in) {
  const uint64_t total = (uint64_t)1 << (2 * s->n);
  if (first > total || count > total - first) return fail(TANQ_E_ARG, "range outside vec(rho)");
  if (!count) return TANQ_OK;
  tanq::BitMap bm = bitmap_of(s);
  bool multi_dev = false;
  for (auto& sh : s->shards) multi_dev |= sh.device != s->shards[0].device;
  std::vector<double2> acc;
  for (auto& sh : s->shards) {
    DevScratch& d = scratch_for(s, sh.device);
    TRY(ensure_scratch(s, d));
  }
  const size_t chunk = scratch_for(s, s->shards[0].device).stage_elems;
  for (uint64_t off = 0; off < count; off += chunk) {
    const uint64_t cnt = std::min<uint64_t>(chunk, count - off);
    if (in) {
      for (auto& sh : s->shards) {
        DevScratch& d = scratch_for(s, sh.device);
        CUDA_TRY(cudaSetDevice(sh.device));
        CUDA_TRY(cudaMemcpyAsync(d.stage, in + off, cnt * sizeof(double2), cudaMemcpyHostToDevice,
                                 sh.stream));
        CUDA_TRY(tanq::launch_scatter_vec(sh.data, d.stage, bm, s->n, s->L, (uint64_t)sh.id,
                                          first + off, cnt, sh.stream));
        s->launches++;
        TRY(host_wait(s, sh.stream));
      }
      continue;
    }
    const bool need_sum = multi_dev || (s->dist && s->world > 1);
    if (need_sum) {
      acc.assign(cnt, make_double2(0.0, 0.0));
      std::vector<double2> tmp(cnt);
      for (auto& sh : s->shards) {
        DevScratch& d = scratch_for(s, sh.device);
        CUDA_TRY(cudaSetDevice(sh.device));
        CUDA_TRY(tanq::launch_gather_vec(sh.data, d.stage, bm, s->n, s->L, (uint64_t)sh.id,
                                         first + off, cnt, true, sh.stream));
        s->launches++;
        if (s->dist)
          NCCL_TRY(nccl().AllReduce(d.stage, d.stage, cnt * 2, ncclDouble, ncclSum, s->comm,
                                 sh.stream));
        CUDA_TRY(cudaMemcpyAsync(tmp.data(), d.stage, cnt * sizeof(double2),
                                 cudaMemcpyDeviceToHost, sh.stream));
        TRY(host_wait(s, sh.stream));
        for (uint64_t i = 0; i < cnt; ++i) {  // exactly one shard owns each entry: x + 0
          acc[i].x += tmp[i].x;
          acc[i].y += tmp[i].y;
        }
      }
      std::memcpy(out + off, acc.data(), cnt * sizeof(double2));
    } else {
      Shard& s0 = s->shards[0];
      DevScratch& d = scratch_for(s, s0.device);
      CUDA_TRY(cudaSetDevice(s0.device));
      for (auto& sh : s->shards) {
        CUDA_TRY(tanq::launch_gather_vec(sh.data, d.stage, bm, s->n, s->L, (uint64_t)sh.id,
                                         first + off, cnt, false, sh.stream));
        s->launches++;
      }
      for (auto& sh : s->shards) TRY(stream_wait(s0, sh));  // every shard's gather lands first
      CUDA_TRY(cudaMemcpyAsync(out + off, d.stage, cnt * sizeof(double2), cudaMemcpyDeviceToHost,
                               s0.stream));
      TRY(host_wait(s, s0.stream));
    }
  }
  return TANQ_OK;
}

tanq_status tanq_get_state(tanq_sim* s, uint64_t first, uint64_t count, tanq_c64* out) {
  if (!s || (!out && count)) return fail(TANQ_E_ARG, "NULL argument");
  TRY(ensure_unpacked(s));
  return state_io(s, first, count, out, nullptr);
}

tanq_status tanq_set_state(tanq_sim* s, uint64_t first, uint64_t count, const tanq_c64* in) {
  if (!s || (!in && count)) return fail(TANQ_E_ARG, "NULL argument");
  TRY(ensure_unpacked(s));  // elements outside [first, first + count) must stay valid
  s->herm_state = false;  // unknown until tanq_check_hermitian
  return state_io(s, first, count, nullptr, in);
}

tanq_status tanq_check_hermitian(tanq_sim* s, double tol, int* is_herm) {
  if (!s || !is_herm) return fail(TANQ_E_ARG, "NULL argument");
  *is_herm = 0;
  if (s->packed) {  // the packed layout stores one element per transpose pair: Hermitian
    *is_herm = 1;
    return TANQ_OK;
  }
  // transpose pairs must stay on their shard: one shard in the identity layout, or the
  // parity layout (single process; a multi-process handle would need a reduction)
  if (s->dist && s->world > 1) return TANQ_OK;
  if (!s->par) {
    if (s->shards.size() != 1) return TANQ_OK;
    for (int i = 0; i < 2 * s->n; ++i)
      if (s->phys[i] != (uint32_t)i) return TANQ_OK;
  }
  double diff = 0.0, mx = 0.0;
  for (auto& sh : s->shards) {
    DevScratch& d = scratch_for(s, sh.device);
    TRY(ensure_scratch(s, d));
    CUDA_TRY(cudaSetDevice(sh.device));
    unsigned long long* res = reinterpret_cast<unsigned long long*>(d.scal);  // [diff, maxabs]
    CUDA_TRY(cudaMemsetAsync(res, 0, 2 * sizeof(unsigned long long), sh.stream));
    CUDA_TRY(tanq::launch_herm_check(sh.data, s->L, tdesc_of(s, sh.id), res, sh.stream));
    s->launches++;
    unsigned long long h[2];
    CUDA_TRY(cudaMemcpyAsync(h, res, sizeof(h), cudaMemcpyDeviceToHost, sh.stream));
    TRY(host_wait(s, sh.stream));
    double dd, mm;
    std::memcpy(&dd, &h[0], sizeof(double));
    std::memcpy(&mm, &h[1], sizeof(double));
    diff = std::max(diff, dd);
    mx = std::max(mx, mm);
  }
  *is_herm = diff <= tol * std::max(1.0, mx) ? 1 : 0;
  s->herm_state = *is_herm != 0;
  return TANQ_OK;
}

tanq_status tanq_sync(tanq_sim* s) {
  if (!s) return fail(TANQ_E_ARG, "NULL handle");
  TRY(join_all(s));
  CUDA_TRY(cudaGetLastError());
  return TANQ_OK;
}

tanq_status tanq_profile_read(tanq_sim* s, tanq_kernel_prof* out, int max, int* n_out) {
  if (!s || !n_out) return fail(TANQ_E_ARG, "NULL argument");
  TRY(prof_flush(s));
  int n = 0;
  for (int c = 0; c < kProfClasses && n < max; ++c) {
    if (!s->prof_launches[c]) continue;
    tanq_kernel_prof& p = out[n++];
    std::memset(&p, 0, sizeof(p));
    std::strncpy(p.name, kProfNames[c], sizeof(p.name) - 1);
    p.launches = s->prof_launches[c];
    p.total_ms = s->prof_ms[c];
    p.bytes = s->prof_bytes[c];
    p.flops = s->prof_flops[c];
    p.hw_flops = s->prof_hw_flops[c];
  }
  *n_out = n;
  return TANQ_OK;
}

tanq_status tanq_profile_reset(tanq_sim* s) {
  if (!s) return fail(TANQ_E_ARG, "NULL handle");
  TRY(prof_flush(s));
  for (int c = 0; c < kProfClasses; ++c) {
    s->prof_ms[c] = s->prof_bytes[c] = s->prof_flops[c] = s->prof_hw_flops[c] = 0;
    s->prof_launches[c] = 0;
  }
  return TANQ_OK;
}

uint64_t tanq_launch_count(tanq_sim* s) { return s ? s->launches : 0; }

}  // extern "C"
