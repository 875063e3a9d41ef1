/*
 * qva.h -- C ABI of the B200-native QVA state-evolution library (libqva.so).
 *
 * The library computes, on NVIDIA B200 (sm_100a) GPUs, the full-state evolution of a
 * p-layer quantum variational ansatz and its objective (arXiv 2110.03963, PAPER.md):
 *
 *   |psi(theta)> = prod_{k=1..p} U_M(beta_k) U_Q(gamma_k) |psi0>        Eq. 1,
 *                                                                     Eq. qaoa (:185), Eq. qwoa (:298)
 *   f(theta)     = <psi|Q|psi> = sum_x |psi_x|^2 q_x                   Eq. 2
 *
 *   U_Q(gamma) = exp(-i gamma Q), Q = diag(q)                          Eq. 3 / phase_shift_qaoa (:62-69, :152-155)
 *   U_M(beta)  = exp(-i beta W) with W one of
 *     QVA_MIXER_X         W = sum_j X_j (hypercube)                    Eq. mixing_qaoa (:159-171), reading R1
 *     QVA_MIXER_CIRCULANT W circulant, F^-1 diag(e^{-i beta lambda}) F  Sec. 3 (:315-333), readings R3, R4
 *     QVA_MIXER_SPARSE    W real symmetric CSR, truncated Taylor action Sec. 3 (:333), reading R13
 *     QVA_MIXER_PARITY    QAOAz: U = e^{-itB_last} e^{-itB_even} e^{-itB_odd}, B = sum XX+YY over
 *                         qubit pairs of an ordered subsequence   Eqs. parity_terms / qaoaz_mixers
 *                                                                   (:213-248), reading R19
 *
 * Conventions (all calls):
 *  - theta layout [gamma_1, beta_1, ..., gamma_p, beta_p] (reading R7); layer 1 acts first (R6).
 *  - States are complex128 stored as interleaved (re, im) doubles, index x = sum_j bit_j 2^j.
 *  - Every pointer argument is a CALLER-OWNED HOST buffer unless the name ends in _device
 *    (a device pointer on the plan's device).  The library copies in/out and never retains or
 *    frees caller memory.  The plan owns all device memory (state, q, spectrum, CSR, scratch,
 *    receive buffers) and the NCCL communicator, and frees them in qva_plan_destroy
 *    (Table 1 "destroy").
 *  - Every call returns qva_status; no exception or abort crosses the ABI.  On error a
 *    thread-local message is available from qva_last_error().  After a failed evolve the plan
 *    remains valid but the state is unspecified.
 *  - Calls are synchronous with respect to the host: they return after the device work they
 *    enqueue on the plan's stream has completed.
 *  - Multi-process (world > 1): every rank makes the same calls with the same theta (the paper
 *    broadcasts theta from rank 0; here the caller does).  Global offsets are used
 *    for set_xxx and get_xxx ranges; each rank only accepts/returns indices of its own partition
 *    (COMM-psi contiguous blocks, Eqs. local_i / offset).
 *  - A plan is single-threaded; several plans may coexist.
 */
#ifndef QVA_H
#define QVA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default) /* every qva_* symbol is exported from libqva.so */
#endif

typedef struct qva_plan qva_plan; /* opaque */

typedef enum {
    QVA_OK = 0,
    QVA_ERR_INVALID_ARGUMENT = 1, /* structural error: NULL/negative/shape error */
    QVA_ERR_SIZE_MISMATCH = 2,    /* range outside the partition / wrong length */
    QVA_ERR_NOT_READY = 3,        /* evolve/expectation before set_qualities ("required") */
    QVA_ERR_NUMERIC = 4,          /* non-finite q/theta/lambda, Taylor non-convergence */
    QVA_ERR_UNSUPPORTED = 5,      /* e.g. X mixer with dim != 2^n, non-power-of-two world */
    QVA_ERR_OUT_OF_MEMORY = 6,
    QVA_ERR_CUDA = 7,
    QVA_ERR_NCCL = 8
} qva_status;

typedef enum { QVA_MIXER_X = 0, QVA_MIXER_CIRCULANT = 1, QVA_MIXER_SPARSE = 2, QVA_MIXER_PARITY = 3 } qva_mixer;

typedef struct {
    uint64_t dim;            /* N = number of basis states of the (sub)space; X mixer: 2^n_qubits */
    int32_t n_qubits;        /* log2(dim) for QVA_MIXER_X, else -1 (ignored)                      */
    int32_t mixer;           /* qva_mixer                                                         */
    int32_t rank;            /* this process's rank in [0, world)                                 */
    int32_t world;           /* number of processes (one GPU each); 1 = single GPU                */
    const void *nccl_unique_id; /* 128-byte ncclUniqueId (from qva_nccl_unique_id on rank 0) when
                                   world > 1; NULL otherwise                                      */
    int32_t device;          /* CUDA device ordinal                                               */
    int32_t virtual_shards;  /* >1: simulate this many COMM-psi shards on ONE device with a
                                loopback transport (tests the sharded schedule on one GPU); world
                                must be 1.  0 or 1: normal                                        */
    void *stream;            /* cudaStream_t to launch on, or NULL (the plan creates one)         */
    int32_t max_batch;       /* largest B for qva_evolve_batch (0 -> 1)                           */
    int32_t reserved[7];     /* reserved[0]: 1 = replicated mode (every rank holds the whole state;
                                batches shard over ranks).  reserved[1]: 1 = generate weighted MaxCut
                                qualities inside the tile passes at every size (default: from 2^26
                                amplitudes).  reserved[2]: 1 =
                                circulant mixer: three-level FFT split where one exists (tests; used
                                anyway above 8192^2 states).  reserved[3]: 1 = virtual shards run
                                the exchanges through the peer-store paths of real shards (X
                                mixer: global<->local exchange; circulant: row/column transposes
                                fused into the FFT pass stores), each virtual shard's buffer as
                                its "peer"; tests the code multi-GPU plans use.  reserved[4]: 1 =
                                circulant mixer with a spectrum set by
                                qva_set_circulant_eigenvalues_const (lambda_0, c, ..., c): apply it
                                in closed form, U psi = e^{-i beta c} psi + (e^{-i beta lambda_0} -
                                e^{-i beta c}) mean(psi) (one 40-B pass per layer; on a row-
                                sharded state one 16-B all-reduce of sum(psi) per layer, SURVEY
                                C6; an O(N) speed-of-light reference for the FFT path, SURVEY K10;
                                the FFT stays the default).  Others must be 0. */
} qva_plan_desc;

/* ---- lifecycle (Table 1 plan / destroy) ------------------------------------ */

/* Allocates device memory for the state (and the sharding receive buffer / batch states).
 * world > 1 creates the plan's NCCL communicator from desc->nccl_unique_id (collective: every
 * rank calls it) and, for sharded X / circulant plans, exports both state buffers as CUDA IPC
 * handles and maps every peer's (the fused peer-store exchange); if any rank
 * fails to map, all ranks fall back to NCCL send/recv (decided by a min-vote).
 * QVA_ERR_UNSUPPORTED: X mixer with dim != 2^n_qubits, world / shard count not a power of two
 * for the X mixer or a world > 1 parity mixer, fewer than 12 local qubits, virtual shards of a
 * sparse or parity mixer, a sharded circulant dim with no split M1*M2 that the shard count
 * divides.  A world > 1 sparse plan holds a row block of W (qva_set_sparse_mixer_rows); a world > 1
 * parity (QAOAz) plan runs the pair terms that touch a rank qubit as peer passes over the other
 * ranks' IPC-mapped state buffers (QVA_ERR_UNSUPPORTED at evolve if they could not be mapped). */
qva_status qva_plan_create(const qva_plan_desc *desc, qva_plan **out);

/* Host transport of a world > 1 plan: the caller's own process group (e.g. torch.distributed over
 * gloo) carries the plan's collectives instead of NCCL.  Every buffer argument is a host buffer
 * valid for the duration of the call; every rank calls each function in the same order with the
 * same sizes.  Return 0 on success, non-zero on failure (mapped to QVA_ERR_NCCL).
 *   allgather(ctx, in, out, bytes): out[r*bytes .. (r+1)*bytes) = rank r's `in` (rank-major).
 *   allreduce_f64(ctx, vals, n, op): in place element-wise over ranks; op 0 = sum, 1 = max, 2 = min.
 *   alltoall(ctx, send, recv, chunk_bytes): chunk t of `send` (world chunks) goes to rank t; chunk s
 *     of `recv` is the one rank s sent to us.
 * What uses it (COMM-psi; COMM-grad_f, :374-389): the IPC-handle all-gather and
 * min-vote at plan creation, the one-word barrier after a fused peer-store pass (the library
 * synchronises its stream first, so every rank's stores into our buffer have landed when the
 * barrier returns), the <Q> / batch / q-range all-reduces, and the exchange / transpose fallbacks
 * when IPC is unavailable (device data staged through host memory: slow; tests).  The data path
 * of the fused exchange stays device-to-device over IPC-mapped peer memory.  This is how the
 * multi-rank code path runs when several ranks share one GPU (NCCL refuses two ranks per device).
 * The struct is copied; ctx must outlive the plan. */
typedef struct {
    void *ctx;
    int (*allgather)(void *ctx, const void *in, void *out, uint64_t bytes);
    int (*allreduce_f64)(void *ctx, double *vals, uint64_t n, int32_t op);
    int (*alltoall)(void *ctx, const void *send, void *recv, uint64_t chunk_bytes);
} qva_transport;
/* qva_plan_create with an optional host transport (NULL = NCCL as in qva_plan_create; non-NULL:
 * world > 1 and desc->nccl_unique_id is ignored).  QVA_ERR_INVALID_ARGUMENT if a function is NULL. */
qva_status qva_plan_create_ex(const qva_plan_desc *desc, const qva_transport *transport, qva_plan **out);
/* NULL-safe; frees everything the plan owns.  For world > 1 it is collective: every rank unmaps
 * the peers' IPC buffers, then all ranks pass a barrier before any exported buffer is freed. */
qva_status qva_plan_destroy(qva_plan *plan);
/* COMM-psi partition of this rank: local_n = local_i, offset = local_i_offset
 * (Eqs. local_i, offset).  Contiguous equal blocks for power-of-two N
 * (rank = top log2(world) index bits); remainder to the lowest ranks otherwise (R16). */
qva_status qva_plan_get_partition(const qva_plan *plan, uint64_t *local_n, uint64_t *offset);
/* Host-only partition rule (no plan / no GPU needed): same rule as above. */
qva_status qva_partition(uint64_t dim, int32_t world, int32_t rank, uint64_t *local_n, uint64_t *offset);

/* ---- operators (Table 2 observable/operator functions) ---------------------- */

/* q[0..count) -> diag(Q) entries [offset, offset+count) (global indices within this rank's
 * partition).  Chunked uploads allowed.  QVA_ERR_NUMERIC on a non-finite value. */
qva_status qva_set_qualities(qva_plan *plan, const double *q, uint64_t offset, uint64_t count);
/* Same from a device pointer (count doubles on the plan's device). */
qva_status qva_set_qualities_device(qva_plan *plan, const double *q_device, uint64_t offset, uint64_t count);
/* On-device generation of the max-cut qualities q_x = -cut_w(x) = -sum_e w_e [bit_u(x) != bit_v(x)]
 * (Eq. maxcut-cost, cfg sign R10) for the whole partition.  u, v: m vertex
 * indices in [0, n_qubits); w: m weights or NULL for unit weights.  X mixer only. */
qva_status qva_set_qualities_maxcut(qva_plan *plan, int32_t m, const int32_t *u, const int32_t *v,
                                    const double *w);
/* On-device generation of the qualities of a permutation-encoded subspace (QWOA, PAPER.md:98-120,
 * :255-300; readings R23, R24).  Index i of the state holds s_i, the i-th k-permutation of the
 * elements {0..m-1} in lexicographic order (Lehmer code: digit a has radix m-a), so the plan's dim
 * must be m!/(m-k)! (else QVA_ERR_SIZE_MISMATCH); and
 *     q_i = C(s_i) = sum_{a<k} ( lin[a*m + s_a] + sum_{b<k} F[a*k + b] * D[s_a*m + s_b] )
 * (quadratic assignment; TSP: F = directed cycle; summed a-major in this order, F's zero entries
 * skipped).  F: k*k row-major or NULL (no quadratic term), at most 400 nonzeros; D: m*m row-major
 * (required when F is given); lin: k*m or NULL.  1 <= k <= m <= 20, else
 * QVA_ERR_INVALID_ARGUMENT.  Host arrays, copied.  Any mixer; each rank generates its own
 * partition.  QVA_ERR_NUMERIC on a non-finite input or result. */
qva_status qva_set_qualities_permutation(qva_plan *plan, int32_t m, int32_t k, const double *F, const double *D,
                                         const double *lin);

/* Copy diag(Q) entries [offset, offset+count) (global, this rank's partition, layout of the
 * partition) back to q_out[count]. */
qva_status qva_get_qualities(qva_plan *plan, double *q_out, uint64_t offset, uint64_t count);

/* Circulant spectrum lambda[j], j = forward-DFT bin (numpy sign convention, R4), entries
 * [offset, offset+count) of the global length-dim array. */
qva_status qva_set_circulant_eigenvalues(qva_plan *plan, const double *lambda, uint64_t offset, uint64_t count);
/* Spectrum of the form (lambda0, c, c, ..., c): the complete-graph family (adjacency: (N-1, -1);
 * Laplacian: (0, N), cfg3) without storing an N-length array. */
qva_status qva_set_circulant_eigenvalues_const(qva_plan *plan, double lambda0, double c);

/* Real symmetric sparse mixer W in CSR: rows [0, dim), row_ptr[dim+1]
 * (int64, row_ptr[0] = 0), col[nnz] (int32), val[nnz] (fp64; NULL = all ones).  The Taylor
 * action uses s = max(1, ceil(|beta| ||W||_1 / 3)) sub-steps of degree <= 40 (reading R13). */
qva_status qva_set_sparse_mixer(qva_plan *plan, const int64_t *row_ptr, const int32_t *col,
                                const double *val, uint64_t nnz);
/* Row-partitioned W for a world > 1 sparse plan (the paper's distributed SpMV, PAPER.md:333,
 * :1099; COMM-psi partition, Eqs. local_i / offset, :356-366): this rank's rows [row_offset,
 * row_offset + rows), which must be its partition (qva_plan_get_partition); row_ptr[rows + 1]
 * local (row_ptr[0] = 0, row_ptr[rows] = nnz), col[nnz] GLOBAL column indices in [0, dim),
 * val[nnz] or NULL.  Collective: every rank calls it; ||W||_1 is the global maximum row sum, and
 * every rank's Taylor-term buffers are exported as CUDA IPC handles and mapped, so each SpMV reads
 * the entries of remote columns straight from the owning rank's buffer over NVLink (if any rank
 * cannot map them, every term vector is all-gathered instead); the per-term norm maximum is one
 * all-reduce of two doubles, which also orders every rank's term k before any term k + 1.  With
 * world = 1 it equals qva_set_sparse_mixer (row_offset 0, rows = dim).
 * QVA_ERR_SIZE_MISMATCH: rows / row_offset not this rank's partition or row_ptr inconsistent. */
qva_status qva_set_sparse_mixer_rows(qva_plan *plan, const int64_t *row_ptr, const int32_t *col,
                                     const double *val, uint64_t row_offset, uint64_t rows, uint64_t nnz);

/* QAOAz parity mixer (QVA_MIXER_PARITY plans; PAPER.md:213-248 Eqs. parity_terms, qaoaz_mixers):
 * the ordered qubit subsequence s[0..count) the mixing operators act on.
 * B_odd = sum over pairs (s0,s1), (s2,s3), ...; B_even over (s1,s2), (s3,s4), ... (no wrap);
 * B_last = the pair (s_{count-1}, s0) iff count is odd (reading R19).  Default: all qubits
 * 0..n-1 in order.  QVA_ERR_INVALID_ARGUMENT: count < 2, an index outside [0, n) or repeated.
 * The QAOAz initial state (a parity-constrained state) is set with qva_set_initial_state; the
 * default |+> is allowed but not parity-constrained. */
qva_status qva_set_parity_mixer(qva_plan *plan, const int32_t *qubits, int32_t count);

/* Optional initial state psi0 (default |+>, PAPER.md:174-178 / R2): interleaved re,im,
 * entries [offset, offset+count). */
qva_status qva_set_initial_state(qva_plan *plan, const double *re_im, uint64_t offset, uint64_t count);
/* Return to the default |+> initial state. */
qva_status qva_clear_initial_state(qva_plan *plan);

/* ---- evolution (Table 3 evolve_state) --------------------------------------- */

/* psi <- psi0 (current state reset). */
qva_status qva_reset_state(qva_plan *plan);
/* Step-level operations on the current state (for parity tests of each step). */
qva_status qva_apply_phase(qva_plan *plan, double gamma);
qva_status qva_apply_mixer(qva_plan *plan, double beta);
/* psi <- prod_k U_M(beta_k) U_Q(gamma_k) psi0; theta[2p] host array.  Always restarts from psi0. */
qva_status qva_evolve(qva_plan *plan, const double *theta, int32_t p);
/* <psi|Q|psi> of the current state, globally reduced; every rank receives it (Eq. 2). */
qva_status qva_expectation(qva_plan *plan, double *out);
/* sum_x |psi_x|^2 (norm check). */
qva_status qva_norm2(qva_plan *plan, double *out);
/* Copy amplitudes [offset, offset+count) (global, within this rank's partition) to re_im[2*count]. */
qva_status qva_get_state(qva_plan *plan, double *re_im, uint64_t offset, uint64_t count);
/* p_x = |psi_x|^2 for [offset, offset+count) (Table 3 get_probabilities). */
qva_status qva_get_probabilities(qva_plan *plan, double *out, uint64_t offset, uint64_t count);

/* B independent evolutions (e.g. the 2|theta|+1 central-difference sets of the parallel
 * gradient) sharing Q: thetas[B][2p] -> f_out[B] = <psi_b|Q|psi_b>.  With
 * world > 1 the B sets are split across ranks (COMM-grad_f analogue) and every rank receives
 * all B values.  The current state afterwards is unspecified.  B <= desc.max_batch. */
qva_status qva_evolve_batch(qva_plan *plan, const double *thetas, int32_t B, int32_t p, double *f_out);

/* ex-QAOA (Eqs. phase_shift_qaoa_ex and qaoa_ex; reading R25) on a plan whose
 * qualities are a max-cut graph (qva_set_qualities_maxcut, m edges; X or parity mixer):
 * theta[(m+1)*p] = per layer [gamma_{i,1}, ..., gamma_{i,m}, t_i]; layer i applies
 * prod_e exp(-i gamma_{i,e} Sigma_e), Sigma_e(x) = -w_e [bit_u(x) != bit_v(x)] (the edge terms of
 * q = -cut_w, so equal gammas give qva_evolve), then the mixer U(t_i); layer 1 first.  Restarts from
 * psi0; <Q> (the plan's q) as after qva_evolve.  QVA_ERR_NOT_READY without a max-cut graph. */
qva_status qva_evolve_ex(qva_plan *plan, const double *theta, int32_t p);
/* B ex-QAOA parameter sets thetas[B][(m+1)*p] -> f_out[B] (members one after another; with world
 * > 1 in replicated mode the members are split across ranks).  The state afterwards is
 * unspecified. */
qva_status qva_evolve_ex_batch(qva_plan *plan, const double *thetas, int32_t B, int32_t p, double *f_out);

/* ---- NCCL bootstrap (multi-process) ------------------------------------------------------------- */

/* Writes a 128-byte ncclUniqueId into id_out (call on rank 0, broadcast to the other ranks). */
qva_status qva_nccl_unique_id(void *id_out);
/* Host-only: which batch entries [first, first+count) rank `rank` evolves (B split across ranks,
 * remainder to the lowest ranks). */
qva_status qva_batch_partition(int32_t B, int32_t world, int32_t rank, int32_t *first, int32_t *count);
/* Host-only: the global<->local qubit swap of the sharded X mixer (COMM-psi)
 * as a chunk exchange.  Every shard's local array (2^L elements) is G equal chunks, chunk index
 * = the top g = log2 G local bits.  For local chunk t of shard `rank`: peer_of_chunk[t] = the
 * shard it is sent to and received from (t), peer_chunk[t] = the chunk index it occupies there
 * (rank).  Applying it swaps the g global index bits with the top g local bits (a G x G block
 * transpose); it is an involution, so the same plan returns to layout A.  Both arrays hold G
 * entries (caller-owned).  QVA_ERR_INVALID_ARGUMENT unless G is a power of two and
 * 0 <= rank < G. */
qva_status qva_exchange_plan(int32_t G, int32_t rank, int32_t *peer_of_chunk, int32_t *peer_chunk);

/* ---- introspection ---------------------------------------------------------------------------- */

/* Host-only (no GPU): the window passes of the QAOAz parity mixer over `seq` (reading R19,
 * PAPER.md:213-248) for an n-qubit state.  out receives, per window, [w, np, the w physical bits
 * of the window (ascending), then np pairs (a, b) in application order]; *n_windows the count.
 * Entries beyond cap are not written.  Every pair term of B_odd, B_even, B_last appears once, after
 * every earlier-group term it shares a qubit with. */
qva_status qva_parity_schedule(int32_t n, const int32_t *seq, int32_t count, int32_t *out, int32_t cap,
                               int32_t *n_windows);

/* Pass schedule the X-mixer path uses for (n_local, p): writes up to cap entries of
 * (tile_set_index, n_rot_before_phase, has_phase, n_rot_after_phase) as 4 int32 per pass and
 * returns the pass count in *n_passes.  Host-only. */
qva_status qva_x_schedule(int32_t n_local, int32_t p, int32_t *out, int32_t cap, int32_t *n_passes);
/* Host-only: the permuted out-of-place schedule used by qva_evolve on a single shard with
 * n_local >= 21 qubits.  Per pass, 8 int64 in out[8*i ..]:
 * {first bit of the 9-bit read window (3 = contiguous tile), layer of the R1 rotations (-1: none),
 *  layer of the R2 rotations (-1), phase layer (-1), expectation fused (0/1), logical-qubit mask
 *  of R1, logical-qubit mask of R2, TMA dims of the pass}.  cap = passes that fit in out.
 * QVA_ERR_INVALID_ARGUMENT unless 21 <= n_local <= 40 and p >= 1. */
qva_status qva_x_schedule_permuted(int32_t n_local, int32_t p, int64_t *out, int32_t cap, int32_t *n_passes);
/* Host-only: the FFT plan the circulant mixer uses for dimension dim over `shards` COMM-psi shards
 * (1 = single GPU; > 1: direct four-step with shards | M1 and shards | M2) (Sec. 3,
 * PAPER.md:315-333).  flags bit 0: prefer a three-level split (tests; three levels are used
 * anyway above 8192^2).
 * out[9] = {kind (0: one-CTA whole evolution, 1: four-step mixed radix with M = dim, 2: Bluestein
 * with M >= 2 dim - 1, 3: three-level mixed radix M = M1 * Mi1 * Mi2; -1: none), transform length
 * M, M1, M2 (M = M1 * M2), columns per column-pass CTA, rows per row-pass CTA, levels, Mi1, Mi2}.
 * QVA_ERR_UNSUPPORTED when no plan exists. */
qva_status qva_circulant_plan_shape(uint64_t dim, int32_t shards, int32_t flags, int64_t *out);
/* Kernel timing: when enabled, every kernel launch of the plan is bracketed with CUDA events
 * on the plan's stream; qva_kernel_stats returns, for kernel class `which` (0 = X tile pass,
 * 1 = small-state fused evolve, 2 = FFT column pass, 3 = FFT row pass, 4 = sparse SpMV,
 * 5 = reduction, 6 = exchange, 7 = other, 8 = three-level FFT inner passes run in groups on
 * auxiliary streams: launches and bytes counted, not timed -- 0 ms), the summed device
 * milliseconds, launches and algorithmic bytes since the last reset. */
qva_status qva_set_profiling(qva_plan *plan, int32_t enable);
qva_status qva_kernel_stats(qva_plan *plan, int32_t which, double *ms, int64_t *launches, double *bytes);
qva_status qva_reset_kernel_stats(qva_plan *plan);
/* Number of kernel launches issued by the plan since the last reset (all classes). */
qva_status qva_launch_count(qva_plan *plan, int64_t *launches);
/* Plan introspection (host only, no device work): what = 0: 1 if the global<->local exchange and
 * the circulant transposes run fused into the pass stores over IPC-mapped peer memory (world > 1)
 * or over virtual-shard peers, else 0; 1: shard count G (world x virtual shards); 2: 1 if the plan's
 * collectives run over a host transport (qva_plan_create_ex), else 0; 3: world; 4: rank; 5: state
 * bytes one shard has sent to the other shards (global<->local exchanges, circulant transposes:
 * (G-1)/G of a shard's slice each) since the last qva_reset_kernel_stats -- the NVLink traffic of
 * a real shard, the notional one of a virtual shard; 6: 1 if the last QAOAz (parity) evolution ran
 * as TMA tile passes with the pair terms on register groups, 0 if it took the window kernel; 7: 1 if
 * a row-partitioned sparse mixer reads remote columns from the peers' IPC-mapped Taylor buffers,
 * 0 (single shard, or the term-gather fallback).
 * QVA_ERR_INVALID_ARGUMENT for another `what`. */
qva_status qva_plan_query(const qva_plan *plan, int32_t what, int64_t *out);

const char *qva_status_string(qva_status s);
const char *qva_last_error(void);
/* Library version string. */
const char *qva_version(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* QVA_H */
