// qva_internal.h -- internal declarations shared by the libqva translation units.
// Product code only: nothing here is shared with oracle/ (DESIGN.md "Oracle").
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/qva.h"

namespace qva {

// ---------------------------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------------------------
void set_error(const std::string &msg);

#define QVA_CUDA_TRY(expr)                                                                      \
    do {                                                                                        \
        cudaError_t _e = (expr);                                                                \
        if (_e != cudaSuccess) {                                                                \
            ::qva::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));             \
            return QVA_ERR_CUDA;                                                                \
        }                                                                                       \
    } while (0)

#define QVA_NCCL_TRY(expr)                                                                      \
    do {                                                                                        \
        ncclResult_t _r = (expr);                                                               \
        if (_r != ncclSuccess) {                                                                \
            ::qva::set_error(std::string(#expr) + ": " + ncclGetErrorString(_r));             \
            return QVA_ERR_NCCL;                                                                \
        }                                                                                       \
    } while (0)

#define QVA_TRY(expr)                                                                           \
    do {                                                                                        \
        qva_status _s = (expr);                                                                 \
        if (_s != QVA_OK) return _s;                                                            \
    } while (0)

// ---------------------------------------------------------------------------------------------
// X-mixer tile passes (kernels_tile.cu)
// ---------------------------------------------------------------------------------------------
constexpr int kTileBits = 12;                 // 2^12 amplitudes (64 KiB) per tile
constexpr int kGroupBits = 5;                 // 32 amplitudes per consumer thread in registers
constexpr int kCT_BITS = 7;                   // 128 consumer threads
constexpr int kMaxSteps = 16;
constexpr int kMaxGroups = 5;                // X, Y, W (X mixer) + V, Z (QAOAz parity pair terms)
constexpr int kMaxStepPairs = 6;             // parity pair terms per register-group step
constexpr int kSmallMaxQubits = 12;           // whole-state-in-one-CTA path
constexpr int kQGenInt = 3;                   // tile-pass q mode: generated MaxCut q, unit weights
constexpr int kQGenF64 = 9;                   // tile-pass q mode: generated MaxCut q, fp64 weights
constexpr int kMaxPeers = 8;                  // fused peer-store exchange: ranks per plan

// Register group: which tile-local bits the 5 register-index bits (ebit) and the 7 consumer
// thread-index bits (tbit) address.  Chosen on the host so that every 8-lane phase of a
// 16-byte smem access hits 8 distinct bank groups under SWIZZLE_128B.
struct TileGroup {
    int8_t ebit[kGroupBits];
    int8_t tbit[kCT_BITS];
};

struct PassStep {
    int8_t group;      // index into TilePassParams::groups
    int8_t mask;       // 5-bit rotation mask over the group's register bits
    int8_t angle;      // 0: first beta slot (R1), 1: second (R2)
    int8_t phase;      // apply the phase after the rotations of this step (group must be gq)
    // QAOAz parity mixer (R19): pair terms exp(-i t (X_aX_b + Y_aY_b)), in order,
    // on register bits (ja, jb) of this group, encoded ja * 8 + jb (ja < jb); the pass's angle record
    // holds t1 = cos 2t, t2 = sin 2t
    int8_t npair;
    int8_t pair[kMaxStepPairs];
};

// Per-member angle record for one pass (device array [batch]).  Rotations use the factored
// form a' = a - i t b, b' = b - i t a (t = tan beta); the dropped scalar cos beta (per rotation)
// is applied once at the end of the pass as `scale`.  When |cos beta| < 2^-10 the host applies
// two steps of half the angle instead.
struct PassAngles {
    double t1, t2;           // R1 / R2 tan(beta) (of beta/2 when halved)
    double gamma;            // phase angle
    double2 scale;           // product of the dropped rotation factors of this pass
};

// Non-tile physical bits as runs: base(t) = sum_r ((t >> src_r) & (2^w_r - 1)) << dst_r
constexpr int kMaxRuns = 4;
constexpr int kMaxBatchSmem = 64;            // batch members per tile-pass launch (angles live in smem)

struct TilePassParams {
    double2 *psi_out;        // output array (input comes through the tensor map; may alias)
    const void *qt;          // q in consumer order of group gq: [n_tiles][4096] fp64 / int8 / int16
    const double2 *tab;      // integer codes: [batch][ntab] phase factors exp(-i gamma (qmin + j))
    const PassAngles *angles;// [batch]
    double *partials;        // [batch][gridDim.x][4 warps][2] (expectation, norm); zeroed by host
    uint64_t member_stride;  // elements between batch members
    uint64_t n_tiles;        // tiles per member
    int batch;
    int tile_bits[kTileBits];// physical bit of tile-local bit k (ascending)
    int n_runs;
    int run_src[kMaxRuns], run_dst[kMaxRuns], run_w[kMaxRuns];
    uint64_t run_mask[kMaxRuns];  // 2^run_w - 1 (0 for unused runs)
    int log2_tiles;          // n_tiles = 2^log2_tiles
    // TMA coordinates: dim d takes bits [dim_src, dim_src + dim_w) of the tile number
    // (dim_w = 0: a tile dim, coordinate 0); member_dim adds member << dim_w
    int dim_src[5], dim_w[5];
    int member_dim;
    int n_groups;
    TileGroup groups[kMaxGroups];
    int n_steps;
    PassStep steps[kMaxSteps];
    uint64_t st_estr[kGroupBits];  // final group: physical stride of register bit j
    int st_tphys[kCT_BITS];        // final group: physical bit of consumer-thread bit j
    int gq;                  // group in which q is consumed (phase / expectation), -1: no q
    int init;                // 1: first pass, psi = amp0 (no read)
    int expect;              // accumulate partial <Q> and norm in the final group (== gq)
    int qmin, ntab;
    int apply_scale;
    int tail_mode;           // measurement switch QVA_TAIL (bit 0: claim the refill's tile at the start
                             // of a tile; bit 1: defer the store-read wait + refill to the next barrier)
    int fold_scale_gf;       // fp64 factorised generated phase: multiply the per-member G factors by
                             // angles[member].scale instead of every amplitude (apply_scale = 0)
    int tma_store;           // 1: write the tile back with a TMA tensor store (strided tile sets)
    int release_step;        // step after whose smem accesses the stage is released (n_steps: after
                             // the expectation; -1: before any step, i.e. init passes without q)
    double amp0;
    // generated MaxCut qualities (qbytes kQGenInt / kQGenF64): qt points at the per-tile records
    const void *gen_thr;     // [128][8] int / double: per consumer thread {C, beta[5]} of group gq
    const void *gen_G;       // [32] int / double: G(e) over the 5 register bits of group gq
    int gen_m;               // number of edges (integer mode: qmin = -gen_m)
    // global <-> local exchange fused into this pass's stores (world > 1, register-store path):
    // an element whose output local index has chunk t = bits [xshift, xshift + log2 xg) goes to
    // rank t's receive buffer xpeer[t] (peer memory over NVLink, IPC-mapped) at the same index
    // with those bits replaced by xrank -- the all-to-all of COMM-psi done by
    // the stores themselves.  xg = 0: ordinary local stores.
    unsigned long long *work_ctr;  // zeroed per launch: tiles are claimed dynamically (atomicAdd), so
                                   // SMs that stream faster take more tiles (no end-of-pass tail)
    double2 *xpeer[kMaxPeers];
    int xg, xrank, xshift;
    int xvirt;               // virtual shards: the sending shard is physical bits [xshift + log2 xg,
                             // + log2 xg) (stripped from the index) instead of xrank
};

// Compile-time pass programs (kernels_tile.cu): group sequence g[0..n), which steps rotate,
// the step after whose rotations the phase is applied (-1: none) and whether the expectation is
// accumulated.  Program 0 = the generic interpreter of TilePassParams::steps.
struct TileProg {
    int n;
    int g[6];
    bool rot[6];
    int phase_k;
    bool expect;
};
constexpr int kNumTileProgs = 19;
constexpr int kFirstParityProg = 11;  // programs >= this apply the steps' QAOAz pair terms
constexpr TileProg kTileProgs[kNumTileProgs] = {
    {0, {0, 0, 0, 0, 0}, {0, 0, 0, 0, 0}, -1, false},  // 0: generic
    {2, {0, 1, 0, 0, 0}, {1, 1, 0, 0, 0}, -1, false},  // 1: X Y            (B/C pass)
    {3, {0, 2, 1, 0, 0}, {1, 1, 1, 0, 0}, -1, false},  // 2: X W Y          (A pass)
    {4, {0, 1, 1, 0, 0}, {1, 1, 1, 1, 0}, 1, false},   // 3: X Y | P | Y X  (B/C pass across a layer boundary)
    {2, {0, 1, 0, 0, 0}, {1, 1, 0, 0, 0}, -1, true},   // 4: X Y + <Q>      (last pass)
    {4, {0, 0, 2, 1, 0}, {0, 1, 1, 1, 0}, 0, false},   // 5: P | X W Y      (first pass, from |+>)
    {3, {0, 0, 1, 0, 0}, {0, 1, 1, 0, 0}, 0, false},   // 6: P | X Y        (first pass, row bits deferred)
    {6, {0, 1, 2, 2, 0, 1}, {1, 1, 1, 1, 1, 1}, 2, false},  // 7: X Y W | P | W X Y (in-place layer boundary
                                                            //    on the contiguous set: batches, n <= 20)
    {1, {1, 0, 0, 0, 0, 0}, {1, 0, 0, 0, 0, 0}, -1, false}, // 8: Y            (short sets: shards, n < 24)
    {1, {1, 0, 0, 0, 0, 0}, {1, 0, 0, 0, 0, 0}, -1, true},  // 9: Y + <Q>
    {2, {1, 1, 0, 0, 0, 0}, {1, 1, 0, 0, 0, 0}, 0, false},  // 10: Y | P | Y
    // QAOAz parity windows (pair terms in every step, runtime lists; groups V = 3, Z = 4): the shapes
    // the window planner gives the default sequence (contiguous window W Z X V, strided X Y V / Y V)
    {4, {2, 4, 0, 3, 0, 0}, {0, 0, 0, 0, 0, 0}, 0, false},  // 11: P | W Z X V
    {4, {2, 4, 0, 3, 0, 0}, {0, 0, 0, 0, 0, 0}, -1, false}, // 12: W Z X V
    {3, {0, 1, 3, 0, 0, 0}, {0, 0, 0, 0, 0, 0}, -1, false}, // 13: X Y V
    {3, {0, 1, 3, 0, 0, 0}, {0, 0, 0, 0, 0, 0}, 0, false},  // 14: P | X Y V
    {2, {1, 3, 0, 0, 0, 0}, {0, 0, 0, 0, 0, 0}, -1, false}, // 15: Y V
    {2, {1, 3, 0, 0, 0, 0}, {0, 0, 0, 0, 0, 0}, -1, true},  // 16: Y V + <Q>
    {3, {0, 1, 3, 0, 0, 0}, {0, 0, 0, 0, 0, 0}, -1, true},  // 17: X Y V + <Q>
    {2, {1, 3, 0, 0, 0, 0}, {0, 0, 0, 0, 0, 0}, 0, false},  // 18: P | Y V
};

int tile_pass_grid(uint64_t items);
// SM count of the current device (cached; grids are sized in multiples of it)
int num_sms();

// Function attributes (the >48 KiB dynamic shared-memory opt-in) belong to a device context, so
// a kernel's attribute is set once per (kernel, device): a device bit mask under a mutex (plans
// on several devices, or on several threads, may coexist).
struct DeviceOnce {
    std::mutex m;
    uint64_t mask = 0;
};
template <class F>
cudaError_t once_per_device(DeviceOnce &o, F &&f) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(o.m);
    if ((o.mask >> dev) & 1ull) return cudaSuccess;
    e = f();
    if (e == cudaSuccess) o.mask |= 1ull << dev;
    return e;
}
int tile_consumer_warps();
// builds the 5-D load map of psi_in seen through P.tile_bits and the store map of the same box
// into psi_out through the bit permutation obit (nullptr: identity); fills P.dim_*, P.member_dim
// number of TMA dims the maps of (tile_bits, obit) need (must be <= 5; batch 1)
int tile_tma_dims(const int *tile_bits, int L, const int *obit);
qva_status make_tile_tensor_maps(const double2 *psi_in, double2 *psi_out, int L, int batch, TilePassParams &P,
                                 const int *obit, CUtensorMap *map_in, CUtensorMap *map_out);
// qbytes: 0 (no q), 1 (int8 codes), 2 (int16 codes), 8 (fp64)
cudaError_t launch_tile_pass(const CUtensorMap &map, const CUtensorMap &map_out, const TilePassParams &p, int qbytes,
                             int prog, int grid, cudaStream_t s);
// A physical -> logical bit permutation as runs: logical = sum_r ((x >> src_r) & (2^w_r - 1)) << dst_r
// (the identity is one run).  Used where a state is held in a permuted layout (DESIGN.md
// "Permuted layouts").
constexpr int kMaxLayoutRuns = 24;
struct LayoutRuns {
    int n;
    int8_t src[kMaxLayoutRuns], w[kMaxLayoutRuns], dst[kMaxLayoutRuns];
};
cudaError_t launch_qt_gather(void *dst, const void *src, int qbytes, const TilePassParams &p, const TileGroup &g,
                             uint64_t n_tiles, int qmin, const LayoutRuns &lay, cudaStream_t s);
// generated MaxCut qualities: per-tile record inputs (kernels_tile.cu gen_records_kernel)
struct GenPrep {
    LayoutRuns tmap;         // tile-number bits -> logical qubits of the coordinates
    uint64_t const_val;      // logical bits fixed for this shard (rank bits), 0 elsewhere
    int n_tt, n_tb, w_unit;  // edge counts; unit weights
    const int2 *tt_uv;       // [n_tt] logical (u, v): both endpoints outside the tile
    const double *tt_w;
    const int2 *tb_ab;       // [n_tb] (tile-local bit a, logical b outside the tile)
    const double *tb_w;
};
cudaError_t launch_gen_records(void *rec, uint64_t n_tiles, int fp64, const GenPrep &g, cudaStream_t s);
// consumer-order uint8 codes (m - cut) of a unit-weight generated q from its records (gen_codes_kernel)
cudaError_t launch_gen_codes(void *codes, const void *rec, uint64_t n_tiles, const void *thr, const void *G,
                             const TileGroup &g, int m, cudaStream_t s);
// out[logical(x)] = in[x] (restores the natural layout of a permuted state)
cudaError_t launch_permute_copy(double2 *out, const double2 *in, uint64_t n, const LayoutRuns &lay, cudaStream_t s);
// phase tables tab[b][j] = exp(-i gammas[b] (qmin + j)) * mult[b], j < ntab (same fp64 sincos as
// the per-element path; mult = deferred scalar factors of the rotations, nullptr = 1)
cudaError_t launch_phase_table(double2 *tab, const double *gammas, const double2 *mult, int batch, int qmin,
                               int ntab, cudaStream_t s);
// integer-valuedness / range of q: out[0] = all integer (1/0), out[1] = min, out[2] = max
cudaError_t launch_q_range(const double *q, uint64_t n, int *flags, double *minmax_partials, int blocks,
                           cudaStream_t s);
int q_range_blocks(uint64_t n);
cudaError_t launch_q_encode(const double *q, uint64_t n, void *codes, int bytes, cudaStream_t s);

struct SmallEvolveParams {
    double2 *psi;            // [batch][2^n]
    const double2 *psi0;     // optional initial state (nullptr: |+>)
    const double *q;         // [2^n]
    const double *thetas;    // [batch][2p]
    double *out;             // [batch][2] (expectation, norm) or nullptr
    int n, p;
    int mode;                // 0: full evolve; 1: phase only (thetas[0]); 2: mixer only (thetas[0])
};
cudaError_t launch_small_evolve(const SmallEvolveParams &p, int batch, cudaStream_t s);

// qualities generator q_x = -cut_w(x) over [0, count) with global index offset + i
cudaError_t launch_maxcut_q(double *q, uint64_t count, uint64_t offset, int m, const int32_t *u,
                            const int32_t *v, const double *w, cudaStream_t s);
// permutation-subspace qualities (R23, R24) over [0, count) with global rank offset + i;
// dev_pack: cnt[k] u64, D[m*m], Cl[k*m] (linear), fv[nf] f64, frow[k+1], fab[nf] int (a << 8 | b)
constexpr int kKpermMaxMHost = 20, kKpermMaxNfHost = 400;
cudaError_t launch_kperm_q(double *q, uint64_t count, uint64_t offset, int m, int k, const void *dev_pack, int nf,
                           bool linear, cudaStream_t s);
// block transpose of G x G chunks of C elements: out[t][r] = in[r][t]
template <typename T>
cudaError_t launch_chunk_transpose(T *out, const T *in, int G, uint64_t C, cudaStream_t s);
// same for raw bytes (int8/int16 code arrays): elem_bytes in {1, 2}
cudaError_t launch_chunk_transpose_bytes(void *out, const void *in, int G, uint64_t C, int elem_bytes,
                                         cudaStream_t s);
// fixed-order reduction of partials [batch][n][2] -> out [batch][2]
cudaError_t launch_reduce_partials(const double *partials, uint64_t n, int batch, double *out,
                                   cudaStream_t s);
// QAOAz parity-mixer pair term exp(-i t (X_aX_b + Y_aY_b)) on all n_amps amplitudes
cudaError_t launch_parity_pair(double2 *psi, uint64_t n_amps, int a, int b, double t, cudaStream_t s);
// several pair terms over one window of <= 12 physical bits per HBM round trip (parity_window_kernel)
constexpr int kWinMaxBits = 12, kWinMaxPairs = 64, kWinMaxRuns = 12;
struct ParityWindow {
    int n, w;                                 // state bits, window bits
    int n_in, in_src[kWinMaxRuns], in_w[kWinMaxRuns], in_dst[kWinMaxRuns];     // window e -> phys
    int n_out, out_src[kWinMaxRuns + 1], out_w[kWinMaxRuns + 1], out_dst[kWinMaxRuns + 1];  // tile -> phys
    int np;
    int8_t pa[kWinMaxPairs], pb[kWinMaxPairs];  // window-local bits of each pair, in order
    double c, s;                              // cos 2t, sin 2t
    const double *q;                          // phase on load (nullptr: none)
    double gamma;
    const double2 *src;                       // load from here instead of psi (the initial state)
    double init_amp;                          // > 0: the window starts as init_amp (|+>, no load)
};
cudaError_t launch_parity_window(double2 *psi, const ParityWindow &p, cudaStream_t s);
// a pair term with a global (rank) qubit on a sharded state: partner values read from the peers'
// IPC-mapped buffers, out of place (parity_peer_kernel)
struct ParityPeer {
    int L, rank, a, b;                 // local bits; this rank; the pair's (logical = global index) bits
    double c, s;                       // cos 2t, sin 2t
    const double2 *peer[kMaxPeers];    // every rank's current state buffer (this rank's own included)
};
cudaError_t launch_parity_peer(double2 *out, const double2 *in, const ParityPeer &p, cudaStream_t s);
// elementwise phase (generic dims, any mixer): psi *= exp(-i gamma q)
cudaError_t launch_phase(double2 *psi, const double *q, uint64_t n, double gamma, cudaStream_t s);
// psi = 1/sqrt(N)
cudaError_t launch_fill_uniform(double2 *psi, uint64_t n, double amp, cudaStream_t s);
// partial (expectation, norm) over n elements: writes `blocks` partial pairs
cudaError_t launch_expect_partials(const double2 *psi, const double *q, uint64_t n, double *partials,
                                   int blocks, cudaStream_t s);
int expect_partial_blocks(uint64_t n);
cudaError_t launch_probabilities(const double2 *psi, double *out, uint64_t n, cudaStream_t s);
cudaError_t launch_check_finite(const double *x, uint64_t n, int *flag, cudaStream_t s);

// ---------------------------------------------------------------------------------------------
// launch observer: the plan counts launches and (when profiling) brackets them with events
// ---------------------------------------------------------------------------------------------
enum KernelClass { K_TILE = 0, K_SMALL = 1, K_FFT_COL = 2, K_FFT_ROW = 3, K_SPMV = 4, K_REDUCE = 5,
                   K_EXCHANGE = 6, K_OTHER = 7, K_FFT_INNER = 8 };
constexpr int kKernelClasses = 9;
struct LaunchObserver {
    // stream: the stream the launch goes to (nullptr: the plan's stream); the events bracketing
    // the launch are recorded there
    virtual void begin(int cls, double algorithmic_bytes, cudaStream_t stream = nullptr) = 0;
    // a launch counted (launches, bytes) but not bracketed by events (launches that overlap on
    // auxiliary streams, K_FFT_INNER)
    virtual void count(int cls, double algorithmic_bytes) = 0;
    virtual void end() = 0;
    virtual ~LaunchObserver() {}
};

// ---------------------------------------------------------------------------------------------
// circulant (FFT) mixer (kernels_fft.cu)
// ---------------------------------------------------------------------------------------------
struct FftPlan;  // opaque, defined in kernels_fft.cu
struct FftShape {
    bool ok = false, whole = false, bluestein = false;
    uint64_t N = 0, M = 0;   // state length, transform length
    int M1 = 0, M2 = 0, cw = 0, rb = 0;
    int levels = 2, Mi1 = 0, Mi2 = 0, cw2 = 0, rb2 = 0;  // three levels: N = M1 * Mi1 * Mi2
};
// G > 1: sharded (direct four-step, G | M1, M2); force3: three-level split where one exists (tests)
FftShape fft_plan_shape(uint64_t N, int G = 1, bool force3 = false);
qva_status fft_plan_create(uint64_t N, int device, int G, bool force3, FftPlan **out);
void fft_plan_destroy(FftPlan *fp);
// permute lambda (forward-bin order, length N) into the plan's internal spectral order
void fft_permute_spectrum(const FftPlan *fp, const double *lambda, double *lambda_perm);

struct FftRun {
    double2 *psi = nullptr;            // state (in place)
    const double *q = nullptr;         // qualities (phase / expectation)
    const double *lambda_perm = nullptr;  // spectrum in plan order, or nullptr -> (lam0, lamc)
    double lam0 = 0.0, lamc = 0.0;
    const double *theta = nullptr;     // host [2p] (mode 0) or [1] = beta (mode 1)
    int p = 0;
    int mode = 0;                      // 0: p layers of phase + mixer; 1: one mixer only
    int init = 0;                      // 1: first pass writes amp0 instead of reading psi
    double amp0 = 0.0;
    bool expect = false;               // fuse sum |psi|^2 q, sum |psi|^2 into the last pass
    double *red_out = nullptr;         // device [2] receives the reduced pair when expect
};
qva_status fft_run(FftPlan *fp, const FftRun &r, cudaStream_t s, LaunchObserver *obs);
// complete-graph-family spectrum (lambda_0, c, ..., c) in closed form (kernels_complete.cu; opt-in
// ablation, desc.reserved[4]): p + 1 passes of 40 B per amplitude; scratch: complete_scratch_doubles(n)
size_t complete_scratch_doubles(uint64_t n);
// sharded state: in-place sum over ranks of 2 doubles on the device, stream-ordered
struct CompleteComm {
    virtual qva_status sum2_dev(double *dev2) = 0;
    virtual ~CompleteComm() {}
};
qva_status complete_run(const FftRun &r, uint64_t n, uint64_t n_global, double *scratch, cudaStream_t s,
                        LaunchObserver *obs, CompleteComm *comm = nullptr);
// sharded four-step: r.psi is this process's row block(s) in natural order (local * N/G)
struct FftShardIO {
    int G = 1, local = 1, first = 0;  // shards, shards held by this process, global index of local 0
    double2 *col = nullptr;           // column-layout work array (local * N/G)
    const double *q_col = nullptr;    // q in the column layout
    virtual qva_status to_col(const double2 *row, double2 *col) = 0;  // all-to-all transposes
    virtual qva_status to_row(const double2 *col, double2 *row) = 0;
    // transposes fused into the passes' stores: the row pass writes shard s's columns straight
    // into col_dst[s] (its column-layout buffer), the column pass writes shard d's rows into
    // row_dst[d]; peer memory (IPC, NVLink) on real shards, blocks of this process's arrays on
    // virtual ones.  barrier(): every shard's stores into ours are complete.
    bool fused = false;
    double2 *row_dst[kMaxPeers] = {};
    double2 *col_dst[kMaxPeers] = {};
    virtual qva_status barrier() { return QVA_OK; }
    virtual ~FftShardIO() {}
};
bool fft_shardable(const FftPlan *fp, int G);
qva_status fft_run_sharded(FftPlan *fp, const FftRun &r, FftShardIO &io, cudaStream_t s, LaunchObserver *obs);
// out[b][a][c] = in[a][b][c] for an A x B grid of C-element blocks (sharded FFT transposes)
template <typename T>
cudaError_t launch_block_transpose(T *out, const T *in, uint64_t A, uint64_t B, uint64_t C, cudaStream_t s);

// ---------------------------------------------------------------------------------------------
// sparse (CSR truncated Taylor) mixer (kernels_sparse.cu)
// ---------------------------------------------------------------------------------------------
// Where the SpMV finds the entries of the Taylor term vector it multiplies: this process's own
// buffer (one shard), the IPC-mapped buffers of every rank (row-partitioned W over world > 1
// ranks: column c lives on the rank whose partition [off[r], off[r+1]) holds it), or a gathered
// copy of the whole vector (fallback without IPC, rank r's slice at r * stride).
struct SpmvSource {
    int G = 1;                               // 1: local buffer only
    uint64_t off[kMaxPeers + 1] = {};        // partition offsets (COMM-psi, qva_partition)
    const double2 *peer[2][kMaxPeers] = {};  // [Taylor buffer t0 / t1][rank] (IPC-mapped)
    const double2 *gathered = nullptr;       // fallback: all ranks' slices at rank * stride
    uint64_t stride = 0;
};
struct SparseMixer {
    int64_t *row_ptr = nullptr;
    int32_t *col = nullptr;
    double *val = nullptr;   // nullptr: all ones
    uint64_t nnz = 0;
    uint64_t rows = 0;       // rows held here (this rank's partition of a row-partitioned W)
    double norm1 = 0.0;      // ||W||_1 (W symmetric: max row abs sum; global over ranks)
    double2 *t0 = nullptr, *t1 = nullptr;  // Taylor term buffers (rows elements)
    double *scratch = nullptr;             // per-block maxima
    int scratch_blocks = 0;
    SpmvSource src;                        // world > 1: where remote columns are read
    double2 *gather_buf = nullptr;         // fallback gather buffer (G * stride elements)
    bool peer_ok = false;                  // src.peer holds IPC mappings (to close in destroy)
};
// Collectives a row-partitioned mixer needs between Taylor terms (api.cu implements them on the
// plan's transport): the global max of two doubles (which also orders every rank's SpMV before
// any next one) and, without IPC, the all-gather of a term vector.
struct SparseComm {
    virtual qva_status max2(double *v) = 0;
    virtual qva_status gather(const double2 *local, double2 *all, uint64_t stride) = 0;
    virtual ~SparseComm() {}
};
// psi <- exp(-i beta W) psi.  terms_used receives the total number of SpMVs.  comm == nullptr:
// single shard.
qva_status sparse_apply_mixer(SparseMixer &sm, double2 *psi, double beta, cudaStream_t s, LaunchObserver *obs,
                              int *terms_used, SparseComm *comm = nullptr);

}  // namespace qva
