/* TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Dense density-matrix primitives for the CPU oracle.  rho is the full
 * 2^n x 2^n complex matrix, row-major: rho[r * 2^n + c] = rho_{r,c}.
 * Nothing here knows about vec(rho), superoperators, fusion or GPU layouts.
 *
 * Every channel acts block-wise: for every pair (r0, c0) of row/column indices
 * whose bits at the op's qubits are zero, the 2^k x 2^k block
 *     X[i][j] = rho[r0 | bits(i)][c0 | bits(j)],   bits(i) = sum_j b_j(i) 2^{q_j}
 * is replaced by its image.  This is Eq. (onegate) rho <- G rho G^dag with
 * G = I (x) ... (x) G_q (x) ... (x) I, written without the
 * Kronecker expansion.  Blocks are disjoint, so the OpenMP loop over r0 is
 * race-free and bitwise deterministic.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

typedef double complex cplx;

#define MAXD 16 /* 2^k, k <= 4 */

static uint64_t spread_bits(uint64_t i, int k, const int* q) {
  uint64_t v = 0;
  for (int j = 0; j < k; ++j)
    if ((i >> j) & 1u) v |= (uint64_t)1 << q[j];
  return v;
}

/* xi(rho) = sum_m K_m rho K_m^dag.  K: m matrices, each d x d row-major. */
void orc_apply_kraus(cplx* rho, int n, int k, const int* q, int m, const cplx* K) {
  const uint64_t N = (uint64_t)1 << n, d = (uint64_t)1 << k;
  const uint64_t mask = spread_bits(d - 1, k, q);
  uint64_t off[MAXD];
  for (uint64_t i = 0; i < d; ++i) off[i] = spread_bits(i, k, q);
#pragma omp parallel for schedule(static)
  for (uint64_t r0 = 0; r0 < N; ++r0) {
    if (r0 & mask) continue;
    cplx X[MAXD][MAXD], Y[MAXD][MAXD], T[MAXD][MAXD];
    for (uint64_t c0 = 0; c0 < N; ++c0) {
      if (c0 & mask) continue;
      for (uint64_t i = 0; i < d; ++i)
        for (uint64_t j = 0; j < d; ++j) {
          X[i][j] = rho[(r0 | off[i]) * N + (c0 | off[j])];
          Y[i][j] = 0;
        }
      for (int mm = 0; mm < m; ++mm) {
        const cplx* Km = K + (size_t)mm * d * d;
        /* T = K_m X */
        for (uint64_t i = 0; i < d; ++i)
          for (uint64_t j = 0; j < d; ++j) {
            cplx s = 0;
            for (uint64_t l = 0; l < d; ++l) s += Km[i * d + l] * X[l][j];
            T[i][j] = s;
          }
        /* Y += T K_m^dag,  (K^dag)[l][j] = conj(K[j][l]) */
        for (uint64_t i = 0; i < d; ++i)
          for (uint64_t j = 0; j < d; ++j) {
            cplx s = 0;
            for (uint64_t l = 0; l < d; ++l) s += T[i][l] * conj(Km[j * d + l]);
            Y[i][j] += s;
          }
      }
      for (uint64_t i = 0; i < d; ++i)
        for (uint64_t j = 0; j < d; ++j) rho[(r0 | off[i]) * N + (c0 | off[j])] = Y[i][j];
    }
  }
}

/* Depolarizing channel on the k qubits jointly, by its definition (reading R7):
 *   E(rho) = (1-p) rho + p (I_Q / d) (x) Tr_Q(rho).
 * Block (r0,c0) of (I_Q/d) (x) Tr_Q(rho) is (tr X_{r0,c0} / d) I. */
void orc_apply_depolarizing(cplx* rho, int n, int k, const int* q, double p) {
  const uint64_t N = (uint64_t)1 << n, d = (uint64_t)1 << k;
  const uint64_t mask = spread_bits(d - 1, k, q);
  uint64_t off[MAXD];
  for (uint64_t i = 0; i < d; ++i) off[i] = spread_bits(i, k, q);
#pragma omp parallel for schedule(static)
  for (uint64_t r0 = 0; r0 < N; ++r0) {
    if (r0 & mask) continue;
    for (uint64_t c0 = 0; c0 < N; ++c0) {
      if (c0 & mask) continue;
      cplx tr = 0;
      for (uint64_t i = 0; i < d; ++i) tr += rho[(r0 | off[i]) * N + (c0 | off[i])];
      for (uint64_t i = 0; i < d; ++i)
        for (uint64_t j = 0; j < d; ++j) {
          cplx* e = &rho[(r0 | off[i]) * N + (c0 | off[j])];
          *e = (1.0 - p) * (*e) + (i == j ? p * tr / (double)d : 0.0);
        }
    }
  }
}

/* A raw superoperator S (4^k x 4^k, row-major) acting on the column-stacked
 * block: vec(X)[r + c d] = X[r][c] (vec = column stacking),
 * vec(X') = S vec(X). */
void orc_apply_superop(cplx* rho, int n, int k, const int* q, const cplx* S) {
  const uint64_t N = (uint64_t)1 << n, d = (uint64_t)1 << k, D = d * d;
  const uint64_t mask = spread_bits(d - 1, k, q);
  uint64_t off[MAXD];
  for (uint64_t i = 0; i < d; ++i) off[i] = spread_bits(i, k, q);
#pragma omp parallel for schedule(static)
  for (uint64_t r0 = 0; r0 < N; ++r0) {
    if (r0 & mask) continue;
    cplx x[MAXD * MAXD], y[MAXD * MAXD];
    for (uint64_t c0 = 0; c0 < N; ++c0) {
      if (c0 & mask) continue;
      for (uint64_t c = 0; c < d; ++c)
        for (uint64_t r = 0; r < d; ++r) x[r + c * d] = rho[(r0 | off[r]) * N + (c0 | off[c])];
      for (uint64_t a = 0; a < D; ++a) {
        cplx s = 0;
        for (uint64_t b = 0; b < D; ++b) s += S[a * D + b] * x[b];
        y[a] = s;
      }
      for (uint64_t c = 0; c < d; ++c)
        for (uint64_t r = 0; r < d; ++r) rho[(r0 | off[r]) * N + (c0 | off[c])] = y[r + c * d];
    }
  }
}

/* probs[x] = Re rho[x][x]  (the density matrix yields outcome probabilities). */
void orc_diag(const cplx* rho, int n, double* probs) {
  const uint64_t N = (uint64_t)1 << n;
  for (uint64_t x = 0; x < N; ++x) probs[x] = creal(rho[x * N + x]);
}

/* Readout confusion per qubit (reading R11): p' = (M_{n-1} (x) ... (x) M_0) p with
 * M_q = [[1-p10_q, p01_q], [p10_q, 1-p01_q]], applied one qubit at a time. */
void orc_readout(double* p, int n, const double* p10, const double* p01) {
  const uint64_t N = (uint64_t)1 << n;
  for (int q = 0; q < n; ++q) {
    const uint64_t bit = (uint64_t)1 << q;
    for (uint64_t x = 0; x < N; ++x) {
      if (x & bit) continue;
      double a = p[x], b = p[x | bit];
      p[x] = (1.0 - p10[q]) * a + p01[q] * b;
      p[x | bit] = p10[q] * a + (1.0 - p01[q]) * b;
    }
  }
}

/* Single-qubit Pauli entries: s = 0:I 1:X 2:Y 3:Z. */
static cplx pauli_entry(int s, int a, int b) {
  switch (s) {
    case 0: return a == b ? 1.0 : 0.0;
    case 1: return a != b ? 1.0 : 0.0;
    case 2: return a == b ? 0.0 : (a == 0 ? -I : I);
    default: return a == b ? (a == 0 ? 1.0 : -1.0) : 0.0;
  }
}

/* tr(P rho) = sum_{a,b} P[a][b] rho[b][a], P = (x)_q sigma_q with sigma_q chosen by
 * (x_mask, z_mask) bit q: (0,0) I, (1,0) X, (1,1) Y, (0,1) Z.  Full double loop;
 * zero Pauli entries are skipped only after they are computed. */
void orc_expect_pauli(const cplx* rho, int n, uint64_t xm, uint64_t zm, double* out_re,
                      double* out_im) {
  const uint64_t N = (uint64_t)1 << n;
  int sel[64];
  for (int q = 0; q < n; ++q) {
    int xb = (xm >> q) & 1, zb = (zm >> q) & 1;
    sel[q] = xb ? (zb ? 2 : 1) : (zb ? 3 : 0);
  }
  double sre = 0.0, sim = 0.0;
#pragma omp parallel for reduction(+ : sre, sim) schedule(static)
  for (uint64_t a = 0; a < N; ++a) {
    for (uint64_t b = 0; b < N; ++b) {
      cplx pe = 1.0;
      for (int q = 0; q < n && pe != 0.0; ++q)
        pe *= pauli_entry(sel[q], (int)((a >> q) & 1), (int)((b >> q) & 1));
      if (pe == 0.0) continue;
      cplx t = pe * rho[b * N + a];
      sre += creal(t);
      sim += cimag(t);
    }
  }
  *out_re = sre;
  *out_im = sim;
}

/* Invariants: out[0] = Re tr, out[1] = Im tr, out[2] = max |rho - rho^dag|,
 * out[3] = min Re diag, out[4] = max |Im diag|. */
void orc_invariants(const cplx* rho, int n, double* out) {
  const uint64_t N = (uint64_t)1 << n;
  double tre = 0, tim = 0, herm = 0, mind = INFINITY, imd = 0;
  for (uint64_t x = 0; x < N; ++x) {
    cplx v = rho[x * N + x];
    tre += creal(v);
    tim += cimag(v);
    if (creal(v) < mind) mind = creal(v);
    if (fabs(cimag(v)) > imd) imd = fabs(cimag(v));
  }
#pragma omp parallel for reduction(max : herm) schedule(static)
  for (uint64_t r = 0; r < N; ++r)
    for (uint64_t c = r + 1; c < N; ++c) {
      double e = cabs(rho[r * N + c] - conj(rho[c * N + r]));
      if (e > herm) herm = e;
    }
  out[0] = tre;
  out[1] = tim;
  out[2] = herm;
  out[3] = mind;
  out[4] = imd;
}

/* rho <- |0..0><0..0|  (reading R1). */
void orc_init_ground(cplx* rho, int n) {
  const uint64_t N = (uint64_t)1 << n;
  memset(rho, 0, sizeof(cplx) * N * N);
  rho[0] = 1.0;
}
