// qva_internal.h -- internal declarations shared by the libqva translation units.
// Product code only: nothing here is shared with oracle/ (DESIGN.md "Oracle").
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

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
// X-mixer tile passes (kernels_x.cu)
// ---------------------------------------------------------------------------------------------
constexpr int kTileBits = 12;                 // 2^12 amplitudes (64 KiB) per CTA tile
constexpr int kTileThreads = 256;             // 16 amplitudes per thread in registers
constexpr int kMaxSteps = 8;
constexpr int kSmallMaxQubits = 12;           // whole-state-in-one-CTA path

// One register-group step of a pass.  Tile-local bits are split in three 4-bit groups:
// group 0 (A) = tile bits 0..3, group 1 (B) = 4..7, group 2 (C) = 8..11.
struct PassStep {
    int8_t group;      // 0 A, 1 B, 2 C
    int8_t mask;       // 4-bit rotation mask inside the group
    int8_t angle;      // 0: first beta slot (R1), 1: second (R2)
    int8_t phase;      // apply the phase after the rotations of this step
};

// Per-member angle record for one pass (device array [batch][kPassAngles]).
struct PassAngles {
    double c1, s1, c2, s2, gamma;
};

struct TilePassParams {
    const double2 *psi_in;   // may alias psi_out
    double2 *psi_out;
    const double *q;         // qualities in the current layout (phase / expectation)
    const PassAngles *angles;// [batch]
    double *partials;        // [batch][n_tiles][2] (expectation, norm) when expect
    uint64_t member_stride;  // elements between batch members
    uint64_t n_tiles;        // tiles per member
    int tile_bits[kTileBits];// physical bit positions of tile-local bits (ascending; 0,1,2 first)
    int n_phys_bits;         // physical index bits of one member's array
    int n_steps;
    PassStep steps[kMaxSteps];
    int init;                // 1: first pass, psi = amp0 (no read); 2: first pass, read psi0 (psi_in)
    int expect;              // accumulate partial <Q> and norm
    double amp0;
};

cudaError_t launch_tile_pass(const TilePassParams &p, int batch, cudaStream_t s);

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
// block transpose of G x G chunks of C elements: out[t][r] = in[r][t]
template <typename T>
cudaError_t launch_chunk_transpose(T *out, const T *in, int G, uint64_t C, cudaStream_t s);
// fixed-order reduction of partials [batch][n][2] -> out [batch][2]
cudaError_t launch_reduce_partials(const double *partials, uint64_t n, int batch, double *out,
                                   cudaStream_t s);
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
                   K_EXCHANGE = 6, K_OTHER = 7 };
struct LaunchObserver {
    virtual void begin(int cls, double algorithmic_bytes) = 0;
    virtual void end() = 0;
    virtual ~LaunchObserver() {}
};

// ---------------------------------------------------------------------------------------------
// circulant (FFT) mixer (kernels_fft.cu)
// ---------------------------------------------------------------------------------------------
struct FftPlan;  // opaque, defined in kernels_fft.cu
qva_status fft_plan_create(uint64_t N, int device, FftPlan **out);
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

// ---------------------------------------------------------------------------------------------
// sparse (CSR truncated Taylor) mixer (kernels_sparse.cu)
// ---------------------------------------------------------------------------------------------
struct SparseMixer {
    int64_t *row_ptr = nullptr;
    int32_t *col = nullptr;
    double *val = nullptr;   // nullptr: all ones
    uint64_t nnz = 0;
    uint64_t rows = 0;
    double norm1 = 0.0;      // ||W||_1 (W symmetric: max row abs sum)
    double2 *t0 = nullptr, *t1 = nullptr;  // Taylor term buffers
    double *scratch = nullptr;             // per-block maxima
    int scratch_blocks = 0;
};
// psi <- exp(-i beta W) psi.  terms_used receives the total number of SpMVs.
qva_status sparse_apply_mixer(SparseMixer &sm, double2 *psi, double beta, cudaStream_t s, LaunchObserver *obs,
                              int *terms_used);

}  // namespace qva
