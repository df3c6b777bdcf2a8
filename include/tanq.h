/*
 * tanq.h -- C ABI of libtanq.so, the B200-native noisy density-matrix gate engine
 * implementing the data-parallel hot path of TANQ-Sim (arXiv 2404.13184).
 *
 * Citations: P:n = /root/reference/PAPER.md line n (LaTeX paragraph, section named).
 *
 * Problem statement (Sec. 2.1, Eq. (dmsim)):
 *   rho_out = G_{m-1} ... (G_1 (G_0 rho_in G_0^dag) G_1^dag) ... G_{m-1}^dag
 * with every noisy gate applied as its Liouville superoperator
 *   S = sum_i conj(K_i) (x) K_i  acting on the column-stacked vec(rho)
 * (Sec. 3.1), i.e. as 4^{n-k} independent [4^k x 4^k] complex
 * mat-vecs over strided tuples of vec(rho) (Eq. 4 and the s_i formula).
 *
 * Conventions
 *   - Amplitudes are IEEE binary64 complex (tanq_c64, layout-compatible with
 *     cuDoubleComplex and std::complex<double>).
 *   - Host-visible order of vec(rho) is the paper's column stacking
 *     v = r + c * 2^n: vec[v] = rho[r][c].
 *   - A k-qubit matrix acting on qubits[0..k-1] uses the local basis index
 *     sum_j b(qubits[j]) 2^j  (qubits[0] is the least significant bit).
 *     Two-qubit named gates take qubits = {control, target}.
 *   - A k-qubit superoperator is 4^k x 4^k, row-major, local vec index
 *     l = r + c * 2^k (the paper's Eq. 4 tuple order).
 *   - Outcome integers: bit q = qubit q.
 *   - Device memory is owned by the library; every pointer argument is
 *     caller-owned, read or written only during the call and never retained.
 *   - Apply/run calls are stream-ordered and may return before the GPU
 *     finishes; calls that write host buffers synchronise first.
 *   - One handle is not thread-safe; distinct handles are independent.
 *   - Every non-OK status leaves a message for tanq_last_error() (thread-local).
 *     TANQ_E_ARG errors are detected before any device work (no partial effect).
 *
 * Internal layout (not visible through the ABI except via tanq_info): the
 * 2n index bits of vec(rho) are permuted so that the row and column bits of
 * each qubit are adjacent (rowpos(q)=2q, colpos(q)=2q+1 initially) and the
 * top log2(n_shards) bits select the shard (P:161 partitions by high bits).
 * With several shards the default is the shard-local parity layout
 * (DESIGN.md §7): the g = log2(world) top qubits are half-global -- the
 * shard bit holds row XOR col of the qubit (invariant under transpose, so a
 * transpose pair never leaves its shard and the packed Hermitian layout
 * runs on every shard), the row bit is local; env TANQ_LAYOUT=bits selects
 * the plain bit layout.
 */
#ifndef TANQ_ABI_H_
#define TANQ_ABI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tanq_sim tanq_sim;
typedef struct { double re, im; } tanq_c64;

typedef enum {
  TANQ_OK = 0,
  TANQ_E_ARG = 1,          /* bad n, shard count, k, qubit out of range / repeated, bad probability,
                              T2 > 2 T1, missing calibration, non-CPTP channel when checked */
  TANQ_E_NOMEM = 2,        /* memory guard: 16*4^n/G bytes + staging exceed free HBM */
  TANQ_E_CUDA = 3,         /* CUDA runtime error (message carries cudaGetErrorString) */
  TANQ_E_NCCL = 4,         /* NCCL error in a multi-process remap or reduction */
  TANQ_E_STATE = 5,        /* state invariant violated: |Im diag| >= 1e-6 or trace drift > 1e-6 */
  TANQ_E_UNSUPPORTED = 6   /* feature not built / not available (e.g. no CUDA device) */
} tanq_status;

/* Gate kinds (Sec. 4 basis gates ID, SX, X, RZ, CX; plus common logical gates). */
typedef enum {
  TANQ_ID = 0, TANQ_X = 1, TANQ_Y = 2, TANQ_Z = 3, TANQ_H = 4, TANQ_S = 5, TANQ_SDG = 6,
  TANQ_T = 7, TANQ_TDG = 8, TANQ_SX = 9,
  TANQ_RX = 10, TANQ_RY = 11, TANQ_RZ = 12,       /* theta; RZ(t) = diag(e^{-it/2}, e^{it/2}) */
  TANQ_CX = 13, TANQ_CZ = 14, TANQ_CP = 15, TANQ_SWAP = 16,   /* q[0] = control for CX/CZ/CP */
  TANQ_U = 17,        /* user matrix m: 2^k x 2^k (need not be unitary) */
  TANQ_KRAUS = 18,    /* user channel: n_kraus matrices 2^k x 2^k contiguous in m */
  TANQ_SUPEROP = 19,  /* user superoperator m: 4^k x 4^k, local vec index r + c 2^k */
  TANQ_RESET = 20,    /* reset q[0] to |0>: channel {|0><0|, |0><1|} (reading R19), noiseless */
  TANQ_N_KINDS = 21
} tanq_kind;

/* One circuit operation.  k = number of qubits (1..3; named gates fix k). */
typedef struct {
  int32_t kind;
  int32_t k;
  int32_t q[3];
  int32_t n_kraus;        /* TANQ_KRAUS only */
  double theta;           /* RX/RY/RZ/CP angle */
  const tanq_c64* m;      /* TANQ_U / TANQ_KRAUS / TANQ_SUPEROP payload, else NULL */
} tanq_op;

typedef struct {
  uint64_t n_ops;
  const tanq_op* ops;
} tanq_circuit;

/* Per-qubit calibration (Sec. 3.5).  t1_us <= 0 disables thermal relaxation. */
typedef struct {
  double t1_us, t2_us;
  double p_meas1_prep0;   /* P(1|0) */
  double p_meas0_prep1;   /* P(0|1) */
} tanq_qubit_cal;

/* Per-(gate kind, qubits) calibration.  depol_p: E(rho) = (1-p) rho + p I/d on the gate's
 * qubits jointly; duration_ns: thermal relaxation time; overrot_rad: coherent over-rotation
 * E = exp(-i eps A/2), A = X (1q) or Z_control (x) X_target (2q).  See DESIGN.md R4-R10. */
typedef struct {
  int32_t kind;
  int32_t k;
  int32_t q[2];
  double depol_p;
  double duration_ns;
  double overrot_rad;
} tanq_gate_cal;

/* Noise model.  Every named gate except RZ (noiseless) must have a gate_cal entry
 * when a model is given (else TANQ_E_ARG).  order 0: U, over-rotation, thermal, depolarizing;
 * order 1: U, over-rotation, depolarizing, thermal. */
typedef struct {
  int32_t n;
  int32_t order;
  const tanq_qubit_cal* qubits;   /* n entries */
  uint64_t n_gates;
  const tanq_gate_cal* gates;
} tanq_noise_model;

/* Readout confusion per qubit: M_q = [[1-p10, p01], [p10, 1-p01]]. NULL arrays = 0. */
typedef struct {
  const double* p10;
  const double* p01;
} tanq_readout;

/* fuse: 0 none, 1 paper (same qubit / same ordered pair), 2 greedy up to k_max
 * with the B200 cost model (default).  k_max in {1,...,5}: fused superoperators never exceed
 * 2 qubits (or a user's 3-qubit op); k_max >= 3 lets the K3 group kernel run several of them
 * in one HBM pass over 3-qubit (k_max = 3, default) or up to 4-qubit tiles (k_max = 4), and
 * k_max = 5 forms "block groups" of up to 5 qubits with at most 3 outside {0, 1} (the block
 * kernel's 5-qubit shared-memory block).  chunk_bytes: reserved, must be 0 (the remap
 * staging is fixed when a multi-process handle is created: 2 x 2 pipelined slots of 128 MiB,
 * DESIGN.md §7).  flags: bit0 = record per-kernel CUDA-event timings; bit1 = plans
 * on single-shard handles capture their launches into a CUDA graph on the first
 * tanq_plan_exec and replay it afterwards (ignored with bit0); bit2 = disable the
 * Hermitian mirror mode for this run. */
typedef struct {
  int32_t fuse;
  int32_t k_max;
  uint64_t chunk_bytes;
  int32_t flags;
  int32_t reserved;
} tanq_run_opts;

typedef struct {
  uint64_t ops_in;         /* circuit ops */
  uint64_t ops_fused;      /* fused ops executed (kernel launches of the plan) */
  uint64_t gate_updates;   /* fused-gate updates: k<=2 fused superoperators applied to the whole
                              state (a K3 group of m sub-ops counts m, a dense k=3 op counts 1) */
  uint64_t n_k[6];         /* kernels by arity k = 1..5 (index k; k >= 3: K3 group kernels) */
  uint64_t n_remaps;       /* global<->local bit swaps */
  uint64_t remap_bytes;    /* bytes sent by this process */
  double plan_ms;          /* host planning time */
} tanq_run_stats;

typedef struct {
  int32_t n_qubits;
  int32_t n_shards;        /* shards in this process */
  int32_t world_size;      /* total shards over all processes */
  int32_t rank;            /* first shard id held by this process */
  int32_t local_bits;      /* log2(amplitudes per shard) */
  int32_t rowpos[32];      /* current physical bit of qubit q's row bit */
  int32_t colpos[32];      /* (parity layout: for a half-global qubit, the global bit that
                              holds row XOR col) */
  uint64_t shard_bytes;
  uint64_t parity_qubits;  /* half-global qubits of the shard-local parity layout (bit q) */
} tanq_info;

/* Per-kernel-class timing accumulated while flags bit0 is set (CUDA events on the
 * launching stream).  bytes / flops are ALGORITHMIC: 32 B per amplitude per
 * gate kernel, 8*4^k flops per amplitude. */
typedef struct {
  char name[32];
  uint64_t launches;
  double total_ms;
  double bytes;      /* algorithmic HBM bytes: 32 per amplitude per launch */
  double flops;      /* algorithmic flops: 8 per complex multiply-add of S x */
  double hw_flops;   /* flops the kernel executes (2 per real FMA; the 3-multiply complex
                        product of the DMMA kernels executes 6 per complex multiply-add) */
} tanq_kernel_prof;

/* ---- lifetime ---------------------------------------------------------------------- */

/* Create rho = |0..0><0..0| (reading R1) over n_shards shards held by this process
 * (n_shards in {1,2,4,8}; shard s on device s % cudaGetDeviceCount).  1 <= n_qubits <= 24
 * and 2n - log2(n_shards) >= 2 (ops on k qubits need 2k local bits).  Errors: TANQ_E_ARG, TANQ_E_NOMEM, TANQ_E_CUDA. */
tanq_status tanq_create(int n_qubits, int n_shards, tanq_sim** out);

/* Like tanq_create, with every shard in a caller-owned device buffer (e.g. a PyTorch tensor;
 * SURVEY §8(b) tanq_create_ex): shard s in buffers[s] on device devices[s], each at least
 * 16 * 4^n / n_shards bytes and 16-byte aligned.  The handle initialises the buffers to
 * |0..0><0..0| and never frees them; the caller keeps them alive until tanq_destroy.  They
 * hold vec(rho) in the library's physical layout (tanq_info_get reports the bit
 * map); in the packed Hermitian layout only the canonical element of each transpose pair is
 * current until tanq_get_state (which unpacks).  Errors: TANQ_E_ARG (size, alignment, not
 * device memory of that device), TANQ_E_NOMEM (scratch), TANQ_E_CUDA. */
tanq_status tanq_create_ex(int n_qubits, int n_shards, void* const* buffers, const int* devices,
                           size_t bytes_each, tanq_sim** out);

/* Multi-process mode (one process per GPU, launched by torchrun): this process holds shard
 * `rank` of `world_size` on `device`; remaps use NCCL point-to-point over NVLink.
 * nccl_uid: NCCL_UNIQUE_ID_BYTES (128) bytes from tanq_nccl_unique_id on rank 0, shared
 * by the caller (e.g. torch.distributed broadcast).  world_size == 1 needs no uid. */
tanq_status tanq_create_dist(int n_qubits, int world_size, int rank, int device,
                             const void* nccl_uid, tanq_sim** out);
tanq_status tanq_nccl_unique_id(void* out, size_t len);
tanq_status tanq_destroy(tanq_sim* s);
tanq_status tanq_reset(tanq_sim* s);                 /* back to |0..0><0..0|, layout reset */
tanq_status tanq_info_get(tanq_sim* s, tanq_info* out);
/* Launch on this CUDA stream (cudaStream_t) for shard `shard` of this process (0 = default). */
tanq_status tanq_set_stream(tanq_sim* s, int shard, void* stream);

/* ---- operations (Sec. 3.1) ----------------------------------------------------------- */

/* rho <- G rho G^dag for a k-qubit matrix G (2^k x 2^k row-major). */
tanq_status tanq_apply_gate(tanq_sim* s, int k, const int* qubits, const tanq_c64* U);
/* rho <- sum_i K_i rho K_i^dag, m Kraus operators contiguous.  check_cptp != 0
 * verifies sum K^dag K = I within 1e-12 (TANQ_E_ARG otherwise). */
tanq_status tanq_apply_channel(tanq_sim* s, int k, const int* qubits, int m, const tanq_c64* kraus,
                               int check_cptp);
/* vec(rho) <- S vec(rho) on the op's tuples (Eq. 4). */
tanq_status tanq_apply_superop(tanq_sim* s, int k, const int* qubits, const tanq_c64* S);
/* Bind noise (Sec. 3.5) -> superoperators -> fuse (Sec. 3.3) -> execute (Eq. dmsim). */
tanq_status tanq_run_circuit(tanq_sim* s, const tanq_circuit* c, const tanq_noise_model* nm,
                             const tanq_run_opts* o, tanq_run_stats* st);

/* Planned execution: bind + fuse once (host steps A-1..A-4), execute many times.  A plan is
 * immutable, owned by the caller, valid for any handle with the same n_qubits. */
typedef struct tanq_plan tanq_plan;
tanq_status tanq_plan_create(tanq_sim* s, const tanq_circuit* c, const tanq_noise_model* nm,
                             const tanq_run_opts* o, tanq_plan** out);
tanq_status tanq_plan_exec(tanq_sim* s, const tanq_plan* p, tanq_run_stats* st);
tanq_status tanq_plan_destroy(tanq_plan* p);
/* Host-only planning (no device needed): same plan as tanq_plan_create on a handle with
 * n_qubits and world_size shards. */
tanq_status tanq_plan_create_host(int n_qubits, int world_size, const tanq_circuit* c,
                                  const tanq_noise_model* nm, const tanq_run_opts* o,
                                  tanq_plan** out);
/* ops_in, ops_fused, n_k[] and plan_ms of a plan (n_remaps / remap_bytes are 0). */
tanq_status tanq_plan_info(const tanq_plan* p, tanq_run_stats* st);
/* Execution schedule of a plan on world_size shards, as the engine runs it: items of three
 * int32 {kind, x, y}; kind 0 = fused op x; kind 1 = remap swapping physical bit x (global)
 * with local bit y (bit layout, A-6); kind 2 = parity-layout remap: half-global
 * qubit x trades places with fully local qubit y.  Pass items = NULL to query
 * the count. */
tanq_status tanq_plan_schedule(const tanq_plan* p, int world_size, int32_t* items, uint64_t max,
                               uint64_t* n_items);
/* Fused op i: arity k (<= 5), qubits (k ints) and, if S != NULL, its 4^k x 4^k superoperator
 * in the paper's vec convention (local index r + c 2^k over qubits[0..k-1]).  For a K3 group
 * this is the product of its sub-ops. */
tanq_status tanq_plan_get_op(const tanq_plan* p, uint64_t i, int* k, int* qubits, tanq_c64* S);
/* Instrumentation (tests): the block-pipeline kernel program of plan op i on a
 * single-shard register in the initial layout, packed = 1 for the packed Hermitian layout.
 * params receives the kernel's parameter struct (params_size must equal its size), blob the
 * fragments + shared-memory offset tables (*blob_bytes).  *kind = 2 if the block kernel would
 * run the op, else 0 (nothing written).  Host only; no device work. */
tanq_status tanq_plan_block_program(const tanq_plan* p, uint64_t i, int packed, void* params,
                                    size_t params_size, void* blob, size_t blob_cap, int* kind,
                                    size_t* blob_bytes);


/* ---- reductions from the diagonal ---------------------------------------------------- */

/* probs[x] = Re rho[x][x] for x in [0, 2^n), then readout confusion (ro may be NULL).
 * Caller buffer of 2^n doubles.  In multi-process mode every rank receives the full vector.
 * TANQ_E_STATE if |Im diag| >= 1e-6. */
tanq_status tanq_probs(tanq_sim* s, const tanq_readout* ro, double* probs);
/* Re tr(P rho), P = (x)_q sigma_q with (x_mask, z_mask) bit q: (0,0) I, (1,0) X, (1,1) Y,
 * (0,1) Z.  Exact expectation, no readout noise (reading R12). out_im may be NULL. */
tanq_status tanq_expect_pauli(tanq_sim* s, uint64_t x_mask, uint64_t z_mask, double* out_re,
                              double* out_im);
/* Draw `shots` outcomes from the readout-noisy distribution with a counter-based Philox
 * generator keyed by seed (shot i uses counter i); negatives > -1e-10 clamped to 0. */
tanq_status tanq_sample(tanq_sim* s, const tanq_readout* ro, uint64_t seed, uint64_t shots,
                        uint64_t* outcomes);

/* Mid-circuit projective measurement of `qubit` in the computational basis (the measurement
 * gate announced at P:45 / P:50, text absent; reading R19): p1 = Tr(|1><1|_q rho) from the
 * diagonal, outcome b = [u < p1] with u the first Philox4x32-10 uniform of (seed, counter 0),
 * then rho <- P_b rho P_b / p_b.  *outcome = b, *prob = p_b (either may be NULL).
 * TANQ_E_STATE if p_b < 1e-300 (cannot happen for the drawn outcome unless rho is invalid). */
tanq_status tanq_measure(tanq_sim* s, int qubit, uint64_t seed, int* outcome, double* prob);

/* ---- state I/O (paper vec order v = r + c 2^n) --------------------------------------- */
tanq_status tanq_get_state(tanq_sim* s, uint64_t first, uint64_t count, tanq_c64* out);
tanq_status tanq_set_state(tanq_sim* s, uint64_t first, uint64_t count, const tanq_c64* in);

tanq_status tanq_sync(tanq_sim* s);
const char* tanq_last_error(void);

/* Packed Hermitian layout: while rho is known to be Hermitian and an op is
 * Hermiticity-preserving (every Kraus-form op; user superoperators are checked), single-shard
 * handles keep only the canonical element of each transpose pair up to date and every kernel
 * reads and writes only those (16 instead of 32 B per amplitude per pass, half the FP64 work);
 * the other half is restored by one unpack pass before anything reads it.  rho is known Hermitian
 * after create / reset; tanq_set_state clears it; this call measures max|rho - rho^dag| and
 * sets it when <= tol * max(1, max|rho|).  Disable with env TANQ_MIRROR=0 or run flag bit2. */
tanq_status tanq_check_hermitian(tanq_sim* s, double tol, int* is_herm);

/* ---- OpenQASM 2.0 front-end (subset: qelib1 gates, qreg/creg, measure, reset, barrier;
 *      no gate definitions / if) -- the paper's circuits arrive as QASM2 among other
 *      front-ends and are transpiled to the device basis ---------------- */
typedef struct tanq_qasm tanq_qasm;
/* Parse; to_basis != 0 lowers every gate to {ID, SX, X, RZ, CX} (+ reset).  TANQ_E_ARG with
 * "line L:C: ..." in tanq_last_error() on a syntax or semantic error. */
tanq_status tanq_qasm_parse(const char* text, int to_basis, tanq_qasm** out);
/* The parsed circuit; ops stay owned by the tanq_qasm and valid until tanq_qasm_free. */
tanq_status tanq_qasm_circuit(const tanq_qasm* q, tanq_circuit* c, int* n_qubits, int* n_clbits);
/* qubit measured into each classical bit (n_clbits entries), -1 if none. */
tanq_status tanq_qasm_measures(const tanq_qasm* q, int32_t* qubit_of_clbit);
tanq_status tanq_qasm_free(tanq_qasm* q);

/* ---- device calibration (NEXT-4; Sec. 3.5; schema SPEC S:365-370) -------
 * { "name", "num_qubits", "qubits": [{"t1_us", "t2_us", "prob_meas0_prep1",
 *   "prob_meas1_prep0", "frequency_ghz"?, "readout_length_ns"?}], "gates": [{"name": id|sx|x|
 *   rz|cx, "qubits": [q] | [c, t], "error", "duration_ns", "overrot_rad"?}], "coupling_map"? }
 * Gate error e -> depolarizing p = e d/(d-1), d = 2^k, clamped to 1 (reading R6); RZ entries
 * ignored (noiseless); T2 > 2 T1 rejected.  TANQ_E_ARG names the JSON path at fault. */
typedef struct tanq_device tanq_device;
tanq_status tanq_device_parse(const char* json, tanq_device** out);
/* The noise model of the device (order 0); its arrays stay owned by the tanq_device and
 * valid until tanq_device_free.  *n_qubits (nullable) = num_qubits. */
tanq_status tanq_device_noise(const tanq_device* d, tanq_noise_model* nm, int* n_qubits);
/* coupling_map pairs (2 int32 each); pairs = NULL queries the count. */
tanq_status tanq_device_coupling(const tanq_device* d, int32_t* pairs, uint64_t max, uint64_t* n);
const char* tanq_device_name(const tanq_device* d);
tanq_status tanq_device_free(tanq_device* d);

/* ---- instrumentation -------------------------------------------------------------- */
/* Copy up to max entries of the per-kernel profile; returns count in *n_out. */
tanq_status tanq_profile_read(tanq_sim* s, tanq_kernel_prof* out, int max, int* n_out);
tanq_status tanq_profile_reset(tanq_sim* s);
/* Kernel launches issued by this handle since creation (all kernel classes). */
uint64_t tanq_launch_count(tanq_sim* s);

#ifdef __cplusplus
}
#endif
#endif /* TANQ_ABI_H_ */
