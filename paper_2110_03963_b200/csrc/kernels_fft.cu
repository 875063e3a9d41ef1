// kernels_fft.cu -- circulant (QWOA) mixer U(beta) = F^-1 diag(exp(-i beta lambda)) F
// (Sec. 3; sign reading R3, spectrum indexing R4) by hand-written fp64
// mixed-radix FFTs on sm_100a, for any N (mixed radix when N splits into two 13-smooth
// factors, Bluestein otherwise).
//
// Convolution engine.  A length-M circulant product F_M^-1 diag(S) F_M v is computed in the
// four-step form M = M1 * M2, index x = x1*M2 + x2:
//   COL pass (one CTA per `cw` adjacent columns x2, 128-B rows):
//       [inverse length-M1 FFTs of the previous product] -> [elementwise ops at natural
//       index x] -> [forward length-M1 FFTs, twiddle w_M^{x2 k1}]
//   ROW pass (one CTA per `rb` rows k1): forward length-M2 FFT -> * S -> inverse length-M2
//       FFT -> twiddle w_M^{-x2 k1}
// so consecutive products share their COL passes and one mixer layer costs two passes
// (plus one final inverse COL pass).  The spectrum S lives in "transposed" order: position
// k1*M2 + k2 holds bin k1 + M1*k2.
//
// Direct path (N = N1*N2 with 13-smooth factors): M = N, S = exp(-i beta lambda)/N, the phase
// exp(-i gamma q) is the elementwise op of the COL pass.
//
// Bluestein path (any N): with chirp c_n = exp(-i pi n^2 / N) (n^2 taken mod 2N in integers),
// nk = (n^2 + k^2 - (k-n)^2)/2 gives  X_k = c_k sum_n (x_n c_n) conj(c_{k-n}),  and the inverse
// x_n = conj(c_n) sum_k (X_k conj(c_k)) c_{n-k}: two linear convolutions, computed as cyclic
// convolutions of length M >= 2N-1 (13-smooth) with the fixed kernel spectra B = F_M b,
// b_m = conj(c_m) (|m| < N, wrapped), and conj(B) (b is even, so F_M conj(b) = conj(B)).
// One mixer:  v = pad(psi * c) -> conv(B) -> * exp(-i beta lambda_k)/N on k < N (the c_k
// factors of X_k and of the inverse's pre-multiply cancel) -> conv(conj B) -> psi = v * conj(c)
// on n < N.  Between layers conj(c) * phase * c = phase, so a layer is four passes over M.
//
// Each length-n sub-FFT runs in shared memory in place: every thread loads the inputs of its
// radix-R butterflies into registers, the block synchronises, then twiddles, transforms and
// stores them in Stockham (autosort) order, so one buffer per transform suffices.
// Direct N <= 4096: the whole p-layer evolution runs in one CTA ("whole" kernel).
//
// For the sub-FFT lengths with a fused-stage codelet (kernels_fft_fs.cu: 768, 4320 rows; 770,
// 810, 840 columns) unsharded direct / three-level plans launch those passes instead (first stage
// from global memory, last stage to global memory, forward / inverse boundary stages fused on the
// registers); three-level plans run each layer's inner passes in groups of top-level rows on two
// auxiliary streams (inner_rows3_grouped).  These kernels stay the path for every other length,
// Bluestein and sharded plans.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "fft_fs.h"
#include "qva_internal.h"

namespace qva {

constexpr int kMaxStages = 24;
constexpr int kFftThreads = 512;
constexpr int kMaxCta = 8192;                     // points per CTA transform set
constexpr int kMaxSub = 8192;                     // longest sub-FFT
constexpr int kColSmemMax = 200 * 1024;
constexpr int kLoadU = 8;                         // independent global loads per thread per batch
// per-CTA twiddle tables: w^{C k} for k < n as
// A[k >> 5] * B[k & 31], i.e. ceil(n/32) + 32 entries per C
// (odd, so that the 8 columns' tables of a column block start in distinct bank groups)
__host__ __device__ constexpr int tw_split_entries(int n) { return (((n + 31) >> 5) + 32) | 1; }
// column passes: forward tables cw * E; three-level inner passes also the outer twiddle
// w^{(x1 M2 + c) K} = A[x1 >> 5] * B[x1 & 31] * C[c]: E + cw entries
__host__ __device__ constexpr int col_tw_entries(int cw, int M1, bool outer) {
    return (outer && tw_split_entries(M1) + cw > cw * tw_split_entries(M1)) ? tw_split_entries(M1) + cw
                                                                             : cw * tw_split_entries(M1);
}
inline size_t col_smem_bytes(int cw, int M1, bool outer = false) {
    return ((size_t)cw * (M1 + (cw > 1 ? 1 : 0)) + (size_t)col_tw_entries(cw, M1, outer)) * 16;
}
inline size_t row_smem_bytes(int rb, int M2) { return ((size_t)rb * M2 + (size_t)rb * tw_split_entries(M2)) * 16; }
constexpr int kRowSmemMax = 200 * 1024;
constexpr size_t kColHalfSmemMax = 110 * 1024;  // two 256-thread column CTAs per SM

struct SubFft {
    int n = 1;
    int ns = 0;
    int r[kMaxStages];
    int m[kMaxStages];
    int twoff[kMaxStages];
    // exact division by multiply-high (divu): magic = ceil(2^32 / d) for d = n / r[s] and m[s]
    uint64_t nbmag[kMaxStages];
    uint64_t mmag[kMaxStages];
};

// x / d for x, d < 2^16 given magic = ceil(2^32 / d): the error magic*d - 2^32 < d keeps
// x * (magic*d - 2^32) < 2^32, so the quotient is exact
__host__ __device__ __forceinline__ uint32_t divu(uint32_t x, uint64_t magic) {
    return (uint32_t)(((uint64_t)x * magic) >> 32);
}
inline uint64_t div_magic(uint32_t d) { return ((1ull << 32) + d - 1) / d; }

struct FftPlan {
    uint64_t N = 0;          // state length
    uint64_t M = 0;          // transform length (N direct, >= 2N-1 Bluestein)
    int device = 0;
    bool whole = false;
    bool bluestein = false;
    int M1 = 1, M2 = 1;          // top-level split N = M1 * M2 (M2 = row length)
    int cw = 8, rb = 1;
    SubFft col, row;             // 2 levels: col = M1, row = M2; 3 levels: col = M1, row = Mi2
    // three levels (N > 8192^2, NEXT-4): each top-level row of length M2 = Mi1 * Mi2 is itself a
    // four-step transform (inner column pass over Mi1, inner row pass over Mi2, both row-local)
    int levels = 2;
    int Mi1 = 0, Mi2 = 0, cw2 = 8, rb2 = 1;
    SubFft col2;
    double2 *d_in_lo = nullptr, *d_in_hi = nullptr;   // inner twiddles w_{M2}
    double2 *d_tw = nullptr;     // stage twiddle tables (col then row)
    double2 *d_big_lo = nullptr, *d_big_hi = nullptr;
    int big_shift = 11;          // w_M^r = hi[r >> s] * lo[r & (2^s - 1)]
    double2 *work = nullptr;     // Bluestein: length-M buffer
    double2 *bhat = nullptr;     // Bluestein: F_M b in transposed order
    double *partials = nullptr;
    int n_partials = 0;
    double *d_theta = nullptr;   // whole-kernel path: angles (host-to-device each evolution)
    int theta_cap = 0;
    // fused-stage passes (kernels_fft_fs.cu) for the compiled lengths of unsharded direct plans:
    // stage tables of the top-level column, inner column (three levels) and row transforms
    double2 *fs_col = nullptr, *fs_col2 = nullptr, *fs_row = nullptr;
    // three-level inner passes in groups of top-level rows on auxiliary streams (L2 reuse between
    // a group's three inner passes, tails of one group's launches under the next group's)
    cudaStream_t aux[4] = {};
    cudaEvent_t ev_fork = nullptr, ev_join[4] = {};
    int n_aux = 0;
};

namespace {

#include "fft_dft.cuh"

// butterflies a thread holds per round of a radix-R stage (register budget: <= 16 inputs plus
// the DFT temporaries at 512 threads x 128 registers)
__host__ __device__ constexpr int nb_of(int R) {
    return R == 2 ? 8 : R == 3 ? 5 : R == 4 ? 4 : R == 5 ? 3 : (R == 6 || R == 7) ? 2 : 1;  // 8..16: 1
}

// Shared-memory addressing of `count` independent transforms (f = transform, i = position):
// AddrLin: f * stride + i (padded column-major / row-major buffers)
struct AddrLin {
    double2 *buf;
    int stride;
    __device__ __forceinline__ double2 *ptr(int f, int i) const { return buf + f * stride + i; }
};
// AddrSw<S>: the same with the low 3 index bits XORed with bits S..S+2 (S = 0: identity).  A
// radix-R first stage (R = 2^S or 2^(S+1)) stores at stride R, which without the swizzle puts 8
// lanes of a 16-B access phase in one bank group; with it they spread over all 8.  Contiguous
// 8-aligned runs map onto themselves, so every other access stays conflict-free.  Needs the
// transform length to be a multiple of 8.
template <int S>
struct AddrSw {
    double2 *buf;
    int stride;
    __device__ __forceinline__ static int sw(int i) { return S ? (i ^ ((i >> S) & 7)) : i; }
    __device__ __forceinline__ double2 *ptr(int f, int i) const { return buf + f * stride + sw(i); }
};

// One Stockham radix-R stage, in place, over `count` independent length-n transforms.  Rounds
// cover whole transforms (a transform's butterflies read and write only its own elements), each
// round loads all its inputs into registers, synchronises, then twiddles, transforms and
// stores.  The host guarantees n / R <= nb_of(R) * blockDim.x.
template <int R, typename Ad>
__device__ __forceinline__ void stage_inplace(const Ad &ad, int n, int count, int m, const double2 *__restrict__ tw,
                                              bool inv, uint64_t nbmag, uint64_t mmag) {
    constexpr int NB = nb_of(R);
    const int nb = n / R;
    const int per_round = max(1, (int)divu(NB * blockDim.x, nbmag));
    for (int f0 = 0; f0 < count; f0 += per_round) {
        const int total = nb * min(per_round, count - f0);
        double2 a[NB][R];
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int J = threadIdx.x + b * blockDim.x;
            if (J < total) {
                const int fq = (int)divu(J, nbmag);
                const int f = f0 + fq, j = J - fq * nb;
#pragma unroll
                for (int t = 0; t < R; ++t) a[b][t] = *ad.ptr(f, j + t * nb);
            }
        }
        __syncthreads();
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int J = threadIdx.x + b * blockDim.x;
            if (J < total) {
                const int fq = (int)divu(J, nbmag);
                const int f = f0 + fq, j = J - fq * nb;
                const int k = j - (int)divu(j, mmag) * m;
                if (m > 1) {
#pragma unroll
                    for (int t = 1; t < R; ++t) a[b][t] = cmul(a[b][t], conj_if(tw[t * k], inv));
                }
                dft<R>(a[b], inv);
                const int o = (j - k) * R + k;
#pragma unroll
                for (int t = 0; t < R; ++t) *ad.ptr(f, o + t * m) = a[b][t];
            }
        }
        __syncthreads();
    }
}

template <typename Ad>
__device__ __forceinline__ void run_fft_ad(const Ad &ad, const SubFft &sf, const double2 *tw, int count, bool inv) {
    // stages are ordered by radix (factor_radices); one loop per radix keeps the live ranges of
    // different radices apart (a switch inside one stage loop made ptxas spill ~10 KB)
    int s = 0;
#define QVA_RADIX_LOOP(R) \
    for (; s < sf.ns && sf.r[s] == R; ++s)                                                            \
        stage_inplace<R>(ad, sf.n, count, sf.m[s], tw + sf.twoff[s], inv, sf.nbmag[s], sf.mmag[s]);
    QVA_RADIX_LOOP(7)
    QVA_RADIX_LOOP(11)
    QVA_RADIX_LOOP(13)
    QVA_RADIX_LOOP(16)
    QVA_RADIX_LOOP(8)
    QVA_RADIX_LOOP(10)
    QVA_RADIX_LOOP(6)
    QVA_RADIX_LOOP(15)
    QVA_RADIX_LOOP(4)
    QVA_RADIX_LOOP(2)
    QVA_RADIX_LOOP(9)
    QVA_RADIX_LOOP(3)
    QVA_RADIX_LOOP(5)
#undef QVA_RADIX_LOOP
}
__device__ __forceinline__ void run_fft(double2 *buf, const SubFft &sf, const double2 *tw, int count, int stride, bool inv) {
    run_fft_ad(AddrLin{buf, stride}, sf, tw, count, inv);
}
// ---- compile-time codelets ----------------------------------------------------------------
// The same Stockham stages with the sub-FFT length, the radix list and hence every stage's m, nb
// and twiddle offset known at compile time: the butterfly index division, the k = j mod m and
// the shared-memory offsets fold into constants (the generic engine spends about half of its
// instructions on that integer work).  The radix order must equal factor_radices'.
template <int R, int N, int M, typename Ad>
__device__ __forceinline__ void stage_ct(const Ad &ad, int count, const double2 *__restrict__ tw, bool inv) {
    constexpr int NB = nb_of(R);
    constexpr int nb = N / R;
    const int per_round = max(1, (int)(NB * blockDim.x) / nb);
    for (int f0 = 0; f0 < count; f0 += per_round) {
        const int total = nb * min(per_round, count - f0);
        double2 a[NB][R];
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int J = threadIdx.x + b * blockDim.x;
            if (J < total) {
                const int f = f0 + J / nb, j = J % nb;
#pragma unroll
                for (int t = 0; t < R; ++t) a[b][t] = *ad.ptr(f, j + t * nb);
            }
        }
        __syncthreads();
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int J = threadIdx.x + b * blockDim.x;
            if (J < total) {
                const int f = f0 + J / nb, j = J % nb;
                const int k = j % M;
                if (M > 1) {
#pragma unroll
                    for (int t = 1; t < R; ++t) a[b][t] = cmul(a[b][t], conj_if(tw[t * k], inv));
                }
                dft<R>(a[b], inv);
                const int o = (j - k) * R + k;
#pragma unroll
                for (int t = 0; t < R; ++t) *ad.ptr(f, o + t * M) = a[b][t];
            }
        }
        __syncthreads();
    }
}
template <int N, int M, int OFF, typename Ad>
__device__ __forceinline__ void stages_ct(const Ad &, const double2 *, int, bool) {}
template <int N, int M, int OFF, typename Ad, int R, int... Rest>
__device__ __forceinline__ void stages_ct(const Ad &ad, const double2 *tw, int count, bool inv) {
    stage_ct<R, N, M>(ad, count, tw + OFF, inv);
    stages_ct<N, M * R, OFF + M * R, Ad, Rest...>(ad, tw, count, inv);
}
template <int R1, int... Rest>
constexpr int first_radix() { return R1; }
template <int N, int... Rs>
struct Codelet {
    static constexpr int n = N;
    static constexpr int kR1 = first_radix<Rs...>();
    static constexpr int kSwz = kR1 == 16 ? 4 : ((kR1 == 8 || kR1 == 4 || kR1 == 2) && N % 8 == 0) ? 3 : 0;
    template <typename Ad>
    __device__ __forceinline__ static void run(const Ad &ad, const SubFft &sf, const double2 *tw, int count, bool inv) {
        stages_ct<N, 1, 0, Ad, Rs...>(ad, tw + sf.twoff[0], count, inv);  // stage tables follow make_sub's
    }
};
// runtime-planned transforms
struct GenericFft {
    static constexpr int n = 0;
    static constexpr int kSwz = 0;
    template <typename Ad>
    __device__ __forceinline__ static void run(const Ad &ad, const SubFft &sf, const double2 *tw, int count, bool inv) {
        run_fft_ad(ad, sf, tw, count, inv);
    }
};

// a call boundary around a whole sub-FFT (used by the small whole-evolution kernel, whose
// layer loop would otherwise spill ~11 KB per thread)
__device__ __noinline__ void run_fft_call(double2 *buf, const SubFft &sf, const double2 *tw, int count, int stride,
                                          bool inv) {
    run_fft(buf, sf, tw, count, stride, inv);
}

__device__ __forceinline__ double2 big_twiddle(const double2 *lo, const double2 *hi, int shift, uint64_t r, bool inv) {
    const uint64_t mask = (1ull << shift) - 1;
    double2 w = cmul(__ldg(hi + (r >> shift)), __ldg(lo + (r & mask)));
    return conj_if(w, inv);
}

__device__ __forceinline__ double2 phase_mul(double2 a, double qv, double gamma) {
    double s, c;
    sincos(gamma * qv, &s, &c);
    return make_double2(fma(c, a.x, s * a.y), fma(c, a.y, -s * a.x));
}

// Bluestein chirp c_x = exp(-i pi x^2 / N), x^2 reduced mod 2N exactly (x < N < 2^31)
__device__ __forceinline__ double2 chirp(uint64_t x, uint64_t N) {
    const uint64_t r = (x * x) % (2 * N);
    double s, c;
    sincospi((double)r / (double)N, &s, &c);
    return make_double2(c, -s);
}

__device__ __forceinline__ void block_reduce2(double &a, double &b, double *red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) {
        red[2 * warp] = a;
        red[2 * warp + 1] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double sa = 0.0, sb = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            sa += red[2 * w];
            sb += red[2 * w + 1];
        }
        a = sa;
        b = sb;
    }
}

// elementwise ops of a COL pass, applied at natural index x in this order
enum : int {
    OP_CHIRP_CONJ = 1,  // v *= conj(c_x)          (end of a Bluestein mixer)
    OP_EXPECT = 2,      // accumulate |v|^2 q_x, |v|^2
    OP_PHASE = 4,       // v *= exp(-i gamma q_x)
    OP_SPEC = 8,        // v *= exp(-i beta lambda_x) / N   (Bluestein middle)
    OP_CHIRP = 16,      // v *= c_x                 (start of a Bluestein mixer)
    OP_MASK = 32,       // v = 0 for x >= N
    OP_OUTER_TW = 64,   // v *= w_N^{-x k1}: top-level inverse twiddle of a three-level transform (x =
                        // position in the top-level row, k1 = its row index = matrix index)
};

struct ColArgs {
    const double2 *in;
    uint64_t in_len;         // elements x >= in_len read as 0
    double2 *out;
    uint64_t out_len;        // elements x >= out_len are not written
    const double *q;
    const double *lam;       // natural-order spectrum for OP_SPEC (nullptr: lam0 / lamc)
    uint64_t N;              // state length (mask, chirp)
    int M1, M2, cw, lcw;     // cw = 2^lcw columns per CTA; M2 = columns held (row stride)
    int col_off, M2g;        // sharded column layout: global index of local column 0, global M2
    uint64_t mat_stride;     // inner (three-level) passes: blockIdx.y selects a matrix at this stride
    int mat_off;             // global top-level row index of matrix 0 (sharded)
    const double2 *otw_lo, *otw_hi;  // OP_OUTER_TW: top-level twiddles w_N
    int otw_shift;
    uint64_t m1mag;          // divu magic of M1
    int init;                // 1: v = amp0 for x < N (no load)
    int do_inv, do_fwd, ops;
    double amp0, gamma, beta, lam0, lamc, invN;
    const double2 *tw;
    const double2 *big_lo, *big_hi;
    int big_shift;
    double *partials;
    int tws, ts_off;         // stage twiddles copied to smem at A + ts_off (tws entries; 0: global)
    int ops_cfast;           // elementwise ops column-fastest with batched q loads (q not L2-resident)
    int xg;                  // > 0: sharded to-row transpose fused into the store (xg shards):
    double2 *xout[kMaxPeers];//   row x1 goes to xout[x1 / (M1 / xg)] at (x1 mod M1/xg) * M2g + column
    SubFft sf;
};

// The arithmetic of one column block (columns c0 .. c0+cwv of matrix mat_y), in shared memory
// through the addressing policy: [inverse column FFTs] -> elementwise ops at the natural index ->
// [forward column FFTs + twiddle w_M^{x2 k1}]; expectation partials to slot pslot.
__device__ __forceinline__ double2 outer_tw(const double2 *Tw, int M1, int x1, int c) {
    const int nh = (M1 + 31) >> 5, E = tw_split_entries(M1);
    return cmul(cmul(Tw[x1 >> 5], Tw[nh + (x1 & 31)]), Tw[E + c]);
}
template <typename F, typename Ad>
__device__ __forceinline__ void col_block(const Ad &ad, const ColArgs &a, int c0, int cwv, int mat_y, int pslot,
                                          double *red, const double2 *Tw, const double2 *twp, int ops_mask) {
    const int M1 = a.M1, M2 = a.M2;
    if (a.do_inv) F::run(ad, a.sf, twp, cwv, true);
    const int ops = a.ops & ops_mask;
    if (ops) {
        double acc = 0.0, nrm = 0.0;
        // one element (c, x1); qv / lv: its q and lambda when loaded ahead (need_q / need_lam)
        const bool need_q = (ops & (OP_EXPECT | OP_PHASE)) != 0, need_lam = (ops & OP_SPEC) && a.lam;
        auto op = [&](int c, int x1, double qv, double lv) {
            const uint64_t x = (uint64_t)x1 * a.M2g + a.col_off + c0 + c;  // natural index
            double2 *slot = ad.ptr(c, x1);
            double2 v = *slot;
            if ((ops & OP_MASK) && x >= a.N) {
                v = make_double2(0.0, 0.0);
            } else {
                if (ops & OP_CHIRP_CONJ) v = cmulc(v, chirp(x, a.N));
                if (ops & OP_EXPECT) {
                    const double pr = v.x * v.x + v.y * v.y;
                    acc = fma(pr, qv, acc);
                    nrm += pr;
                }
                if (ops & OP_PHASE) v = phase_mul(v, qv, a.gamma);
                if (ops & OP_SPEC) {
                    const double lam = a.lam ? lv : (x == 0 ? a.lam0 : a.lamc);
                    double s, cs;
                    sincos(-a.beta * lam, &s, &cs);
                    v = cmul(v, make_double2(cs * a.invN, s * a.invN));
                }
                if (ops & OP_CHIRP) v = cmul(v, chirp(x, a.N));
                if (ops & OP_OUTER_TW) v = cmul(v, outer_tw(Tw, M1, x1, c));  // w_N^{-xl K}, tables
            }
            *slot = v;
        };
        auto live = [&](int c, int x1) {  // element holds data and is not masked off
            return c < cwv && !((ops & OP_MASK) && (uint64_t)x1 * a.M2g + a.col_off + c0 + c >= a.N);
        };
        if (a.ops_cfast) {
            // HBM-resident q (large N): column fastest across the threads, so q arrives in 8-column
            // runs (64 B per row) instead of one 8-B word per M2-strided row, and kLoadU loads per
            // thread are in flight before the first is used
            const int totw = M1 << a.lcw;
            for (int base = threadIdx.x; base < totw; base += kLoadU * blockDim.x) {
                double qv[kLoadU], lv[kLoadU];
#pragma unroll
                for (int u = 0; u < kLoadU; ++u) {
                    const int idx = base + u * blockDim.x, x1 = idx >> a.lcw, c = idx & (a.cw - 1);
                    qv[u] = lv[u] = 0.0;
                    if (idx < totw && live(c, x1)) {
                        if (need_q) qv[u] = __ldg(a.q + (uint64_t)x1 * M2 + c0 + c);
                        if (need_lam) lv[u] = __ldg(a.lam + (uint64_t)x1 * a.M2g + a.col_off + c0 + c);
                    }
                }
#pragma unroll
                for (int u = 0; u < kLoadU; ++u) {
                    const int idx = base + u * blockDim.x, x1 = idx >> a.lcw, c = idx & (a.cw - 1);
                    if (idx < totw && c < cwv) op(c, x1, qv[u], lv[u]);
                }
            }
        } else {
            // L2-resident q: row fastest (measured faster at cfg3)
            const int tot = M1 * cwv;
            for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
                const int c = (int)divu(idx, a.m1mag), x1 = idx - c * M1;
                const uint64_t xl = (uint64_t)x1 * M2 + c0 + c;                  // local (q) index
                const uint64_t x = (uint64_t)x1 * a.M2g + a.col_off + c0 + c;    // natural index
                double2 &slot = *ad.ptr(c, x1);
                double2 v = slot;
                if ((ops & OP_MASK) && x >= a.N) {
                    v = make_double2(0.0, 0.0);
                } else {
                    if (ops & OP_CHIRP_CONJ) v = cmulc(v, chirp(x, a.N));
                    if (ops & OP_EXPECT) {
                        const double pr = v.x * v.x + v.y * v.y;
                        acc = fma(pr, __ldg(a.q + xl), acc);
                        nrm += pr;
                    }
                    if (ops & OP_PHASE) v = phase_mul(v, __ldg(a.q + xl), a.gamma);
                    if (ops & OP_SPEC) {
                        const double lam = a.lam ? __ldg(a.lam + x) : (x == 0 ? a.lam0 : a.lamc);
                        double s, cs;
                        sincos(-a.beta * lam, &s, &cs);
                        v = cmul(v, make_double2(cs * a.invN, s * a.invN));
                    }
                    if (ops & OP_CHIRP) v = cmul(v, chirp(x, a.N));
                    if (ops & OP_OUTER_TW) v = cmul(v, outer_tw(Tw, M1, x1, c));  // w_N^{-xl K}, tables
                }
                slot = v;
            }
        }
        if (ops & OP_EXPECT) {
            block_reduce2(acc, nrm, red);
            if (threadIdx.x == 0) {
                a.partials[2 * pslot] = acc;
                a.partials[2 * pslot + 1] = nrm;
            }
        }
        __syncthreads();
    }
    if (a.do_fwd) F::run(ad, a.sf, twp, cwv, false);  // the twiddle w_M^{x2 k1} is applied by the store
}

// the sub-FFT's stage twiddle tables (tws entries from tw + twoff[0]) into shared memory at Ts;
// returns the base to hand to F::run (its offsets are relative to the global table)
__device__ __forceinline__ const double2 *stage_twiddles(const double2 *tw, const SubFft &sf, int tws, double2 *Ts) {
    if (!tws) return tw;
    const double2 *src = tw + sf.twoff[0];
    for (int i = threadIdx.x; i < tws; i += blockDim.x) Ts[i] = src[i];
    return Ts - sf.twoff[0];  // generic address: only Ts[0..tws) is ever dereferenced
}

template <int NT, typename F = GenericFft>
__global__ void __launch_bounds__(NT, kFftThreads / NT) fft_col_kernel(const ColArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    load_roots();
    __shared__ double red[2 * (kFftThreads / 32)];
    const int M1 = a.M1, M2 = a.M2;
    const int c0 = blockIdx.x * a.cw;
    const int cwv = min(a.cw, M2 - c0);
    const uint64_t mat = (uint64_t)blockIdx.y * a.mat_stride;  // inner passes: matrix = top-level row
    const int stride = cwv > 1 ? M1 + 1 : M1;  // odd padding: column-major stores are conflict-free
    double2 *A = reinterpret_cast<double2 *>(smem_raw);
    const AddrSw<F::kSwz> ad{A, stride};
    const int totw = M1 << a.lcw;  // (x1, c) over the full column width; c >= cwv skipped
    // twiddle tables (their global loads go out with the column block's): forward pass
    // w_M^{C k1} = Tw[c*E + (k1 >> 5)] * Tw[c*E + nh + (k1 & 31)] (C = global column); outer
    // (three-level inverse) w_N^{-xl K} = Tw[x1 >> 5] * Tw[nh + (x1 & 31)] * Tw[E + c]
    // (xl = x1*M2 + c0 + c, K = matrix)
    if (!a.init && fft_async_loads()) {  // the whole column block in flight before the table set-up
        for (int idx = threadIdx.x; idx < totw; idx += blockDim.x) {
            const int x1 = idx >> a.lcw, c = idx & (a.cw - 1);
            if (c >= cwv) continue;
            const uint64_t x = (uint64_t)x1 * M2 + c0 + c;
            if (x < a.in_len) cp_async16(ad.ptr(c, x1), a.in + mat + x);
            else *ad.ptr(c, x1) = make_double2(0.0, 0.0);
        }
    }
    // HBM-resident q of the elementwise phase / <Q>: its rows (cw columns, 64 B) are pulled into L2
    // now, so the batched loads of the ops loop (after the inverse FFT) hit L2 instead of waiting a
    // full DRAM latency per batch (12!: 8.10 -> 7.98 ms per column pass)
    if (a.ops_cfast && (a.ops & (OP_EXPECT | OP_PHASE))) {
        for (int x1 = threadIdx.x; x1 < M1; x1 += blockDim.x)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a.q + (uint64_t)x1 * M2 + c0));
    }
    double2 *Tw = A + (size_t)a.cw * (M1 + (a.cw > 1 ? 1 : 0));
    const int nh = (M1 + 31) >> 5, E = tw_split_entries(M1);
    if (a.do_fwd) {
        for (int i = threadIdx.x; i < cwv * E; i += blockDim.x) {
            const int c = i / E, j = i - c * E;
            const uint64_t C = (uint64_t)(a.col_off + c0 + c);
            const int k = j < nh ? (j << 5) : j - nh;  // every k < M1 (entries past M1 are never read)
            Tw[i] = k < M1 ? big_twiddle(a.big_lo, a.big_hi, a.big_shift, C * (uint64_t)k, false) : make_double2(1.0, 0.0);
        }
    } else if (a.ops & OP_OUTER_TW) {
        const uint64_t K = (uint64_t)(a.mat_off + blockIdx.y);
        for (int i = threadIdx.x; i < E + cwv; i += blockDim.x) {
            const int k = i < nh ? (i << 5) : i - nh;  // x1 split (i < E), then the column (i >= E)
            Tw[i] = (i >= E || k < M1)
                        ? big_twiddle(a.otw_lo, a.otw_hi, a.otw_shift,
                                      i < E ? (uint64_t)k * (uint64_t)M2 * K : (uint64_t)(c0 + i - E) * K, true)
                        : make_double2(1.0, 0.0);
        }
    }
    const double2 *twp = stage_twiddles(a.tw, a.sf, a.tws, A + a.ts_off);
    if (a.init || !fft_async_loads()) {
        // the column block arrives in batches of kLoadU independent loads per thread (one load
        // per iteration would wait a full memory latency for each element before its smem store)
        for (int base = threadIdx.x; base < totw; base += kLoadU * blockDim.x) {
            double2 v[kLoadU];
#pragma unroll
            for (int u = 0; u < kLoadU; ++u) {
                const int idx = base + u * blockDim.x;
                const int x1 = idx >> a.lcw, c = idx & (a.cw - 1);
                const uint64_t x = (uint64_t)x1 * M2 + c0 + c;
                v[u] = make_double2(0.0, 0.0);
                if (idx < totw && c < cwv) {
                    if (a.init) v[u] = make_double2(x < a.N ? a.amp0 : 0.0, 0.0);
                    else if (x < a.in_len) v[u] = a.in[mat + x];
                }
            }
#pragma unroll
            for (int u = 0; u < kLoadU; ++u) {
                const int idx = base + u * blockDim.x;
                const int x1 = idx >> a.lcw, c = idx & (a.cw - 1);
                if (idx < totw && c < cwv) *ad.ptr(c, x1) = v[u];
            }
        }
    } else {
        cp_async_wait_all();
    }
    __syncthreads();
    // an inverse-only pass whose one elementwise op is the outer twiddle (three-level inner inverse
    // column pass) applies it in the store loop instead of a separate shared-memory sweep
    const bool otw_store = a.ops == OP_OUTER_TW && !a.do_fwd;
    col_block<F>(ad, a, c0, cwv, blockIdx.y, blockIdx.x, red, Tw, twp, otw_store ? ~OP_OUTER_TW : ~0);
    for (int idx = threadIdx.x; idx < totw; idx += blockDim.x) {
        const int x1 = idx >> a.lcw, c = idx & (a.cw - 1);
        if (c >= cwv) continue;
        const uint64_t x = (uint64_t)x1 * M2 + c0 + c;
        double2 v = *ad.ptr(c, x1);
        if (a.do_fwd) v = cmul(v, cmul(Tw[c * E + (x1 >> 5)], Tw[c * E + nh + (x1 & 31)]));
        else if (otw_store) v = cmul(v, outer_tw(Tw, M1, x1, c));  // w_N^{-xl K}
        if (a.xg) {  // fused to-row transpose: row x1 belongs to shard d
            const int m1s = M1 / a.xg, d = x1 / m1s;
            a.xout[d][(uint64_t)(x1 - d * m1s) * a.M2g + a.col_off + c0 + c] = v;
        } else if (x < a.out_len) {
            a.out[mat + x] = v;
        }
    }
    if (a.xg) __threadfence_system();  // peer stores visible before the host-side barrier
}

struct RowArgs {
    double2 *buf;
    int M1, M2, rb;
    int row_off;                // sharded row layout: global index of local row 0
    int row_mod;                // three-level inner rows: twiddle row index = row % row_mod (0: none)
    uint64_t m2mag;             // divu magic of M2
    int fwd_only;               // 1: forward FFT only (spectrum out, no twiddle)
    int spec;                   // 0: constant (e0 at bin 0, ec elsewhere); 1: real lambda; 2: complex array
    const double *lam_perm;     // spec 1: transposed order
    const double2 *bhat;        // spec 2: transposed order
    int conj_b;
    double2 e0, ec;             // spec 0 factors (scale included)
    double beta, scale;
    const double2 *tw;
    const double2 *big_lo, *big_hi;
    int big_shift;
    int tws, ts_off;            // stage twiddles copied to smem at A + ts_off (tws entries; 0: global)
    int xg, M2s;                // > 0: sharded to-column transpose fused into the store: column x2
    double2 *xout[kMaxPeers];   //   goes to xout[x2 / M2s] at global row * M2s + (x2 mod M2s)
    SubFft sf;
};

template <int NT = kFftThreads, typename F = GenericFft>
__global__ void __launch_bounds__(NT, kFftThreads / NT) fft_row_kernel(const RowArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    load_roots();
    const int M2 = a.M2;
    const int k1_0 = blockIdx.x * a.rb;  // local row; global row = row_off + local
    double2 *A = reinterpret_cast<double2 *>(smem_raw);
    const AddrSw<F::kSwz> ad{A, M2};
    double2 *rows = a.buf + (uint64_t)k1_0 * M2;
    const int tot = a.rb * M2;
    // (row, column) of the flat index i = threadIdx.x + n * blockDim.x, carried incrementally
    const int r0 = threadIdx.x / M2, x0 = threadIdx.x - r0 * M2;
    const int step_r = blockDim.x / M2, step_x = blockDim.x - step_r * M2;
    auto adv = [&](int &r, int &x) {
        r += step_r;
        x += step_x;
        if (x >= M2) {
            x -= M2;
            ++r;
        }
    };
    if (fft_async_loads()) {  // the whole row block in flight before the stage-table copy
        int r = r0, x = x0;
        for (int i = threadIdx.x; i < tot; i += blockDim.x, adv(r, x)) cp_async16(ad.ptr(r, x), rows + i);
    }
    const double2 *twp = stage_twiddles(a.tw, a.sf, a.tws, A + a.ts_off);
    if (fft_async_loads()) {
        cp_async_wait_all();
    } else {
        int r = r0, x = x0;
        for (int base = threadIdx.x; base < tot; base += kLoadU * blockDim.x) {
            double2 v[kLoadU];
#pragma unroll
            for (int u = 0; u < kLoadU; ++u) {
                const int i = base + u * blockDim.x;
                if (i < tot) v[u] = rows[i];
            }
#pragma unroll
            for (int u = 0; u < kLoadU; ++u) {
                const int i = base + u * blockDim.x;
                if (i < tot) *ad.ptr(r, x) = v[u];
                adv(r, x);
            }
        }
    }
    __syncthreads();
    F::run(ad, a.sf, twp, a.rb, false);
    if (a.fwd_only) {
        int r = r0, x = x0;
        for (int i = threadIdx.x; i < tot; i += blockDim.x, adv(r, x)) rows[i] = *ad.ptr(r, x);
        return;
    }
    // constant spectrum (spec 0: e0 at bin 0, ec elsewhere): F^-1(e X) = ec F^-1 X + (e0 - ec) X_0
    // F^-1 delta_0, and F^-1 delta_0 = 1, so the spectrum is folded into the final store loop (one
    // shared-memory sweep fewer); only the CTA holding global row 0 keeps X_0 for its row 0
    const bool spec_fold = a.spec == 0;
    const bool has0 = spec_fold && a.row_off + k1_0 == 0;
    const double2 x00 = has0 ? *ad.ptr(0, 0) : make_double2(0.0, 0.0);
    const double2 d00 = has0 ? cmul(csub(a.e0, a.ec), x00) : make_double2(0.0, 0.0);
    if (!spec_fold) {
        int r = r0, k2 = x0;
        for (int i = threadIdx.x; i < tot; i += blockDim.x, adv(r, k2)) {
            const int k1 = a.row_off + k1_0 + r;
            const uint64_t pos = (uint64_t)k1 * M2 + k2;
            double2 e;
            if (a.spec == 1) {
                double s, c;
                sincos(-a.beta * __ldg(a.lam_perm + pos), &s, &c);
                e = make_double2(c * a.scale, s * a.scale);
            } else if (a.spec == 2) {
                double2 b = __ldg(a.bhat + pos);
                e = make_double2(b.x * a.scale, (a.conj_b ? -b.y : b.y) * a.scale);
            } else {
                e = (k1 == 0 && k2 == 0) ? a.e0 : a.ec;
            }
            double2 *p = ad.ptr(r, k2);
            *p = cmul(*p, e);
        }
    }
    // final twiddle w^{-x2 kr} = Tr[r*E + (x2 >> 5)] * Tr[r*E + nh + (x2 & 31)] per row r (after
    // the block: its loads overlap the inverse FFT's first stage)
    double2 *Tr = A + tot;
    const int nh = (M2 + 31) >> 5, E = tw_split_entries(M2);
    for (int i = threadIdx.x; i < a.rb * E; i += blockDim.x) {
        const int r = i / E, j = i - r * E;
        const int kr = a.row_off + k1_0 + r;
        const uint64_t K = (uint64_t)(a.row_mod ? kr % a.row_mod : kr);
        const int k = j < nh ? (j << 5) : j - nh;  // every k < M2 (entries past M2 are never read)
        Tr[i] = k < M2 ? big_twiddle(a.big_lo, a.big_hi, a.big_shift, K * (uint64_t)k, true) : make_double2(1.0, 0.0);
    }
    __syncthreads();
    F::run(ad, a.sf, twp, a.rb, true);
    // (a multiply-high divu for (r, x2) here made ptxas emit code that indexed Tr out of range on
    // B200; the incremental form is correct)
    int r = r0, x2 = x0;
    for (int i = threadIdx.x; i < tot; i += blockDim.x, adv(r, x2)) {
        double2 u = *ad.ptr(r, x2);
        if (spec_fold) {
            u = cmul(u, a.ec);
            if (has0 && r == 0) u = cadd(u, d00);
        }
        const double2 v = cmul(u, cmul(Tr[r * E + (x2 >> 5)], Tr[r * E + nh + (x2 & 31)]));
        if (a.xg) {  // fused to-column transpose: column x2 belongs to shard s
            const int sh = x2 / a.M2s;
            a.xout[sh][(uint64_t)(a.row_off + k1_0 + r) * a.M2s + (x2 - sh * a.M2s)] = v;
        } else {
            rows[i] = v;
        }
    }
    if (a.xg) __threadfence_system();  // peer stores visible before the host-side barrier
}

// whole evolution of a (direct, 13-smooth) N <= 4096 state in one CTA
struct WholeArgs {
    double2 *psi;
    const double *q;
    const double *lambda_perm;
    double lam0, lamc, invN;
    const double *theta;  // device [2p] or [1]
    int p, mode, init, do_expect;
    double amp0;
    double *red_out;
    const double2 *tw;
    SubFft sf;
};

__global__ void __launch_bounds__(kFftThreads, 1) fft_whole_kernel(const WholeArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    load_roots();
    __shared__ double red[2 * (kFftThreads / 32)];
    const int N = a.sf.n;
    double2 *A = reinterpret_cast<double2 *>(smem_raw);
    for (int i = threadIdx.x; i < N; i += blockDim.x) A[i] = a.init ? make_double2(a.amp0, 0.0) : a.psi[i];
    __syncthreads();
    const int layers = a.mode == 0 ? a.p : 1;
    for (int k = 0; k < layers; ++k) {
        double beta;
        if (a.mode == 0) {
            const double gamma = a.theta[2 * k];
            beta = a.theta[2 * k + 1];
            for (int i = threadIdx.x; i < N; i += blockDim.x) A[i] = phase_mul(A[i], a.q[i], gamma);
            __syncthreads();
        } else {
            beta = a.theta[0];
        }
        run_fft_call(A, a.sf, a.tw, 1, N, false);
        for (int j = threadIdx.x; j < N; j += blockDim.x) {
            const double lam = a.lambda_perm ? a.lambda_perm[j] : (j == 0 ? a.lam0 : a.lamc);
            double s, c;
            sincos(-beta * lam, &s, &c);
            A[j] = cmul(A[j], make_double2(c * a.invN, s * a.invN));
        }
        __syncthreads();
        run_fft_call(A, a.sf, a.tw, 1, N, true);
    }
    double acc = 0.0, nrm = 0.0;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const double2 v = A[i];
        a.psi[i] = v;
        if (a.do_expect) {
            const double pr = v.x * v.x + v.y * v.y;
            acc = fma(pr, a.q[i], acc);
            nrm += pr;
        }
    }
    if (a.do_expect) {
        block_reduce2(acc, nrm, red);
        if (threadIdx.x == 0) {
            a.red_out[0] = acc;
            a.red_out[1] = nrm;
        }
    }
}

// Codelets compiled in (sizes of the cfg3 / 12! plans and powers of two); the planner prefers
// splits whose sub-FFT lengths have one (kernels_fft.cu "compile-time codelets")
using ColKernelFn = void (*)(ColArgs);
using RowKernelFn = void (*)(RowArgs);
struct CodeletEntry {
    int n;
    ColKernelFn col, col_half;
    RowKernelFn row, row_half;
    int rad[6];  // the codelet's stage order (0-terminated); make_sub builds its tables in it
};
const CodeletEntry kCodelets[] = {
    {768, fft_col_kernel<kFftThreads, Codelet<768, 16, 16, 3>>, fft_col_kernel<kFftThreads / 2, Codelet<768, 16, 16, 3>>, fft_row_kernel<kFftThreads, Codelet<768, 16, 16, 3>>, fft_row_kernel<kFftThreads / 2, Codelet<768, 16, 16, 3>>, {16, 16, 3}},
    {770, fft_col_kernel<kFftThreads, Codelet<770, 7, 11, 10>>, fft_col_kernel<kFftThreads / 2, Codelet<770, 7, 11, 10>>, fft_row_kernel<kFftThreads, Codelet<770, 7, 11, 10>>, fft_row_kernel<kFftThreads / 2, Codelet<770, 7, 11, 10>>, {7, 11, 10}},
    {810, fft_col_kernel<kFftThreads, Codelet<810, 9, 9, 10>>, fft_col_kernel<kFftThreads / 2, Codelet<810, 9, 9, 10>>, fft_row_kernel<kFftThreads, Codelet<810, 9, 9, 10>>, fft_row_kernel<kFftThreads / 2, Codelet<810, 9, 9, 10>>, {9, 9, 10}},
    {840, fft_col_kernel<kFftThreads, Codelet<840, 7, 8, 15>>, fft_col_kernel<kFftThreads / 2, Codelet<840, 7, 8, 15>>, fft_row_kernel<kFftThreads, Codelet<840, 7, 8, 15>>, fft_row_kernel<kFftThreads / 2, Codelet<840, 7, 8, 15>>, {7, 8, 15}},
    {1024, fft_col_kernel<kFftThreads, Codelet<1024, 16, 16, 4>>, fft_col_kernel<kFftThreads / 2, Codelet<1024, 16, 16, 4>>, fft_row_kernel<kFftThreads, Codelet<1024, 16, 16, 4>>, fft_row_kernel<kFftThreads / 2, Codelet<1024, 16, 16, 4>>, {16, 16, 4}},
    {2048, fft_col_kernel<kFftThreads, Codelet<2048, 16, 16, 8>>, fft_col_kernel<kFftThreads / 2, Codelet<2048, 16, 16, 8>>, fft_row_kernel<kFftThreads, Codelet<2048, 16, 16, 8>>, fft_row_kernel<kFftThreads / 2, Codelet<2048, 16, 16, 8>>, {16, 16, 8}},
    {4096, fft_col_kernel<kFftThreads, Codelet<4096, 16, 16, 16>>, fft_col_kernel<kFftThreads / 2, Codelet<4096, 16, 16, 16>>, fft_row_kernel<kFftThreads, Codelet<4096, 16, 16, 16>>, fft_row_kernel<kFftThreads / 2, Codelet<4096, 16, 16, 16>>, {16, 16, 16}},
    {4320, fft_col_kernel<kFftThreads, Codelet<4320, 9, 3, 16, 10>>, fft_col_kernel<kFftThreads / 2, Codelet<4320, 9, 3, 16, 10>>, fft_row_kernel<kFftThreads, Codelet<4320, 9, 3, 16, 10>>, fft_row_kernel<kFftThreads / 2, Codelet<4320, 9, 3, 16, 10>>, {9, 3, 16, 10}},
};
const CodeletEntry *codelet_for(int n) {
    static int env = [] {
        const char *e = getenv("QVA_FFT_CODELETS");
        return e ? atoi(e) : 1;
    }();
    if (!env) return nullptr;
    for (const auto &c : kCodelets)
        if (c.n == n) return &c;
    return nullptr;
}
ColKernelFn col_kernel_for(int n, bool half) {
    const CodeletEntry *c = codelet_for(n);
    if (c) return half ? c->col_half : c->col;
    return half ? fft_col_kernel<kFftThreads / 2> : fft_col_kernel<kFftThreads>;
}
RowKernelFn row_kernel_for(int n, bool half = false) {
    const CodeletEntry *c = codelet_for(n);
    if (c) return half ? c->row_half : c->row;
    return half ? fft_row_kernel<kFftThreads / 2> : fft_row_kernel<>;
}

// ------------------------------------------------------------------------------------------
// host-side planning
// ------------------------------------------------------------------------------------------
const long double kPiL = 3.141592653589793238462643383279502884L;

const CodeletEntry *codelet_for(int n);
bool factor_radices(int n, std::vector<int> &rs, bool codelet_order = true) {
    rs.clear();
    // a compiled codelet fixes its own stage order (chosen per size: a conflict-free first stage);
    // the runtime engine (codelet_order = false: the single-CTA kernel) needs the loops' order
    if (const CodeletEntry *c = codelet_order ? codelet_for(n) : nullptr) {
        int prod = 1;
        for (int i = 0; i < 6 && c->rad[i]; ++i) rs.push_back(c->rad[i]), prod *= c->rad[i];
        if (prod == n) return true;
        rs.clear();
    }
    // order must match run_fft's radix loops: 16, 8, 10, 6, 15, 4, 2, 9, 3, 5, 7, 11, 13 (a 2 goes
    // into a radix-10 or radix-6 stage, a 3 with a 5 into radix 15, where they can: fewer stages)
    int x = n;
    for (int p : {16, 8, 10, 6, 15, 4, 2, 9, 3, 5, 7, 11, 13})
        while (x % p == 0) { rs.push_back(p); x /= p; }
    // execution order: the large odd primes first (their stride-7/11/13 first-stage stores are
    // bank-conflict free), then the rest in extraction order
    std::stable_partition(rs.begin(), rs.end(), [](int r) { return r == 7 || r == 11 || r == 13; });
    return x == 1;
}

// a length-n sub-FFT is plannable: 13-smooth, <= kMaxSub, and every stage's butterflies of one
// transform fit one register round (n / r <= nb_of(r) * threads)
bool sub_ok(int n) {
    std::vector<int> rs;
    if (n < 1 || n > kMaxSub || !factor_radices(n, rs) || (int)rs.size() > kMaxStages) return false;
    for (int r : rs)
        if (n / r > nb_of(r) * kFftThreads) return false;
    return true;
}

bool make_sub(int n, SubFft &sf, std::vector<double2> &tw, bool codelet_order = true) {
    std::vector<int> rs;
    if (n < 1 || n > kMaxSub || !factor_radices(n, rs, codelet_order) || (int)rs.size() > kMaxStages) return false;
    for (int r : rs)
        if (n / r > nb_of(r) * kFftThreads) return false;  // one transform per stage round
    sf.n = n;
    sf.ns = (int)rs.size();
    int m = 1;
    for (int s = 0; s < sf.ns; ++s) {
        sf.r[s] = rs[s];
        sf.m[s] = m;
        sf.nbmag[s] = div_magic(n / rs[s]);
        sf.mmag[s] = div_magic(m);
        const int L = m * rs[s];
        sf.twoff[s] = (int)tw.size();
        for (int j = 0; j < L; ++j) {
            const long double ang = -2.0L * kPiL * (long double)j / (long double)L;
            tw.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
        }
        m = L;
    }
    return true;
}

bool smooth(uint64_t n) {
    if (n == 0) return false;
    for (uint64_t p : {2, 3, 5, 7, 11, 13})
        while (n % p == 0) n /= p;
    return n == 1;
}

struct Split {
    int M1 = 0, M2 = 0, cw = 0, rb = 1;
};

// four-step split M = M1 * M2: both 13-smooth, M2 <= kMaxSub, cw * M1 <= kMaxCta and the
// padded column block fits shared memory; widest column block first (cw = 8: 128-B rows),
// then the most balanced split
Split choose_split(uint64_t M, int G = 1) {
    Split best;
    double best_score = -1e300;
    static const char *force2 = getenv("QVA_FFT2");  // measurement override "M1" (column length)
    for (uint64_t m1 = 2; m1 <= (uint64_t)kMaxSub && m1 <= M; ++m1) {
        if (M % m1) continue;
        const uint64_t m2 = M / m1;
        if (m2 < 2 || m2 > (uint64_t)kMaxSub || !sub_ok((int)m1) || !sub_ok((int)m2)) continue;
        if (m1 % G || m2 % G) continue;  // sharded: whole row / column blocks per shard
        if (force2 && (uint64_t)atoi(force2) != m1) continue;
        int cw = 0;
        for (int c : {8, 4, 2, 1})
            if ((uint64_t)c * m1 <= (uint64_t)kMaxCta && col_smem_bytes(c, (int)m1) <= (size_t)kColSmemMax) {
                cw = c;
                break;
            }
        if (!cw) continue;
        // wave quantisation on the SMs (one 512-thread CTA per SM): fraction of CTA slots used
        auto wave_eff = [](uint64_t blocks) {
            const uint64_t sms = (uint64_t)num_sms();
            const uint64_t w = (blocks + sms - 1) / sms;
            return (double)blocks / (double)(w * sms);
        };
        int rb = 1;
        for (int r = 2; r <= 64; ++r)
            if (m1 % r == 0 && (uint64_t)r * m2 <= (uint64_t)kMaxCta) rb = r;
        const double eff = 0.5 * (wave_eff((m2 + cw - 1) / cw) + wave_eff(m1 / rb));
        const double score = 10.0 * cw + 8.0 * eff - 0.5 * fabs(log((double)m1) - log((double)m2));
        if (score > best_score) {
            best_score = score;
            best.M1 = (int)m1;
            best.M2 = (int)m2;
            best.cw = cw;
        }
    }
    if (best.M1) {
        // several short rows per CTA when rows are short
        best.rb = 1;
        for (int r = 2; r <= 64; ++r)
            if (best.M1 % r == 0 && r * best.M2 <= kMaxCta) best.rb = r;
    }
    return best;
}

// w_M^r = hi[r >> 11] * lo[r & 2047] tables on the device
bool make_big_tables(uint64_t M, double2 **lo_d, double2 **hi_d) {
    const int sft = 11;
    const uint64_t B = 1ull << sft, nhi = (M + B - 1) / B;
    std::vector<double2> lo(B), hi(nhi);
    for (uint64_t j = 0; j < B; ++j) {
        const long double ang = -2.0L * kPiL * (long double)j / (long double)M;
        lo[j] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
    for (uint64_t j = 0; j < nhi; ++j) {
        const long double ang = -2.0L * kPiL * (long double)((j * B) % M) / (long double)M;
        hi[j] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
    if (cudaMalloc(lo_d, B * sizeof(double2)) != cudaSuccess || cudaMalloc(hi_d, nhi * sizeof(double2)) != cudaSuccess)
        return false;
    cudaMemcpy(*lo_d, lo.data(), B * sizeof(double2), cudaMemcpyHostToDevice);
    cudaMemcpy(*hi_d, hi.data(), nhi * sizeof(double2), cudaMemcpyHostToDevice);
    return true;
}

// three-level split N = M1 * (Mi1 * Mi2): column lengths M1, Mi1 <= kMaxCta/8 (128-B column blocks),
// inner row Mi2 <= kMaxSub, every sub-FFT plannable; G | M1 and G | Mi1 * Mi2 when sharded; the
// most balanced triple wins
bool choose_split3(uint64_t N, int G, int &M1, int &Mi1, int &Mi2) {
    double best = -1e300;
    M1 = 0;
    if (const char *e = getenv("QVA_FFT3")) {  // measurement override "a,b,c" (must multiply to N)
        int a = 0, b = 0, c = 0;
        if (sscanf(e, "%d,%d,%d", &a, &b, &c) == 3 && (uint64_t)a * b * c == N && sub_ok(a) && sub_ok(b) && sub_ok(c)) {
            M1 = a;
            Mi1 = b;
            Mi2 = c;
            return true;
        }
    }
    const uint64_t cmax = kMaxCta / 8;
    for (uint64_t a = 2; a <= cmax; ++a) {
        if (N % a || (a % G) || !sub_ok((int)a)) continue;
        const uint64_t R = N / a;
        if (R % G) continue;
        for (uint64_t b = 2; b <= cmax; ++b) {
            if (R % b || !sub_ok((int)b)) continue;
            const uint64_t c = R / b;
            if (c < 2 || c > (uint64_t)kMaxSub || !sub_ok((int)c)) continue;
            // most balanced triple; among equally balanced ones the inner row length with the most
            // factors of 2 (radix-16 codelet stages, swizzled smem: 12! with rows of 768 = 16*16*3
            // measured 143 ms vs 154 ms with rows of 810)
            int twos = 0;
            for (uint64_t x = c; x % 2 == 0; x /= 2) ++twos;
            const double score = std::min(std::min(log((double)a), log((double)b)), log((double)c)) + 1e-3 * twos;
            if (score > best) {
                best = score;
                M1 = (int)a;
                Mi1 = (int)b;
                Mi2 = (int)c;
            }
        }
    }
    return M1 != 0;
}

qva_status upload_roots() {
    std::vector<double2> roots(160, make_double2(0, 0));
    for (int r = 2; r <= 16; ++r)
        for (int j = 0; j < r; ++j) {
            const long double ang = -2.0L * kPiL * j / r;
            roots[root_off(r) + j] = make_double2((double)cosl(ang), (double)sinl(ang));
        }
    QVA_CUDA_TRY(cudaMemcpyToSymbol(c_roots, roots.data(), roots.size() * sizeof(double2)));
    return QVA_OK;
}

size_t col_smem(const FftPlan *fp) { return col_smem_bytes(fp->cw, fp->M1); }
size_t row_smem(const FftPlan *fp) { return row_smem_bytes(fp->rb, fp->M2); }
// stage twiddle entries of a sub-FFT (its tables are contiguous from twoff[0])
int stage_tw_entries(const SubFft &sf) {
    return sf.ns ? sf.twoff[sf.ns - 1] + sf.m[sf.ns - 1] * sf.r[sf.ns - 1] - sf.twoff[0] : 0;
}
// adds the stage tables behind a launch's shared-memory block when they fit under cap and the
// copy is small next to the CTA's elements (a 4320-point row CTA would copy 5504 entries)
template <typename Args>
size_t with_stage_tw(Args &a, size_t base_bytes, size_t cap, int elements) {
    a.ts_off = (int)(base_bytes / sizeof(double2));
    a.tws = stage_tw_entries(a.sf);
    if (4 * a.tws <= elements && base_bytes + (size_t)a.tws * sizeof(double2) <= cap)
        return base_bytes + (size_t)a.tws * sizeof(double2);
    a.tws = 0;
    return base_bytes;
}

// launch helpers shared by planning (Bluestein kernel spectrum) and fft_run
ColArgs col_args(const FftPlan *fp) {
    ColArgs c{};
    c.N = fp->N;
    c.M1 = fp->M1;
    c.M2 = fp->M2;
    c.cw = fp->cw;
    c.lcw = fp->cw == 8 ? 3 : fp->cw == 4 ? 2 : fp->cw == 2 ? 1 : 0;
    c.col_off = 0;
    c.M2g = fp->M2;
    c.mat_stride = 0;
    c.mat_off = 0;
    c.m1mag = div_magic((uint32_t)fp->M1);
    c.invN = 1.0 / (double)fp->N;
    c.tw = fp->d_tw;
    c.big_lo = fp->d_big_lo;
    c.big_hi = fp->d_big_hi;
    c.big_shift = fp->big_shift;
    c.partials = fp->partials;
    c.sf = fp->col;
    static int cfast_env = [] {
        const char *e = getenv("QVA_FFT_CFAST");
        return e ? atoi(e) : -1;
    }();
    c.ops_cfast = cfast_env >= 0 ? cfast_env : (fp->M * 24 > (uint64_t)96 << 20 ? 1 : 0);  // q beyond ~3/4 of L2
    return c;
}
RowArgs row_args(const FftPlan *fp, double2 *buf) {
    RowArgs w{};
    w.buf = buf;
    w.M1 = fp->M1;
    w.M2 = fp->M2;
    w.rb = fp->rb;
    w.m2mag = div_magic((uint32_t)fp->M2);
    w.tw = fp->d_tw;
    w.big_lo = fp->d_big_lo;
    w.big_hi = fp->d_big_hi;
    w.big_shift = fp->big_shift;
    w.sf = fp->row;
    return w;
}
int col_grid(const FftPlan *fp) { return (fp->M2 + fp->cw - 1) / fp->cw; }
int row_grid(const FftPlan *fp) { return fp->M1 / fp->rb; }

}  // namespace

// Pure host planning (no device resources): whole-CTA, direct four-step or Bluestein, and the
// split.  Exposed through qva_circulant_plan_shape for CPU tests.
static FftShape shape3(uint64_t N, int G) {
    FftShape sh;
    sh.N = N;
    int a, b, c;
    if (!smooth(N) || !choose_split3(N, G, a, b, c)) return sh;
    sh.ok = true;
    sh.levels = 3;
    sh.M = N;
    sh.M1 = a;
    sh.M2 = 0;  // top-level row length b * c does not fit an int; see Mi1, Mi2
    sh.Mi1 = b;
    sh.Mi2 = c;
    sh.cw = 8;
    sh.cw2 = 8;
    sh.rb = 1;
    sh.rb2 = 1;
    for (int r = 2; r <= 64; ++r)
        if ((uint64_t)r * c <= (uint64_t)kMaxCta) sh.rb2 = r;
    while (sh.rb2 > 1 && ((uint64_t)a * b) % sh.rb2) --sh.rb2;
    return sh;
}

FftShape fft_plan_shape(uint64_t N, int G, bool force3) {
    if (force3 || (N > (uint64_t)kMaxSub * kMaxSub && smooth(N))) {
        FftShape s3 = shape3(N, G);
        if (s3.ok || N > (uint64_t)kMaxSub * kMaxSub) return s3;
    }
    FftShape sh;
    sh.N = N;
    if (G > 1) {  // sharded: direct four-step with G | M1, G | M2 only
        Split sp = (N >= 4 && smooth(N)) ? choose_split(N, G) : Split();
        if (!sp.M1) return sh;
        sh.ok = true;
        sh.M = N;
        sh.M1 = sp.M1;
        sh.M2 = sp.M2;
        sh.cw = sp.cw;
        sh.rb = sp.rb;
        return sh;
    }
    if (N >= 1 && N <= 4096 && smooth(N) && sub_ok((int)N)) {
        sh.ok = true;
        sh.whole = true;
        sh.M = N;
        sh.M1 = 1;
        sh.M2 = (int)N;
        return sh;
    }
    if (N < 2) return sh;
    Split sp = (N >= 4 && smooth(N)) ? choose_split(N) : Split();
    uint64_t M = N;
    if (!sp.M1) {
        sh.bluestein = true;
        const uint64_t Mmax = (uint64_t)kMaxSub * kMaxSub;
        for (M = 2 * N - 1; M <= Mmax; ++M) {
            if (!smooth(M)) continue;
            sp = choose_split(M);
            if (sp.M1) break;
        }
        if (!sp.M1) return sh;
    }
    sh.ok = true;
    sh.M = M;
    sh.M1 = sp.M1;
    sh.M2 = sp.M2;
    sh.cw = sp.cw;
    sh.rb = sp.rb;
    return sh;
}

qva_status fft_plan_create(uint64_t N, int device, int G, bool force3, FftPlan **out) {
    *out = nullptr;
    FftPlan *fp = new FftPlan();
    fp->N = N;
    fp->device = device;
    auto fail = [&](qva_status s, const std::string &msg) {
        fft_plan_destroy(fp);
        if (!msg.empty()) set_error(msg);
        return s;
    };
    std::vector<double2> tw;
    const FftShape sh = fft_plan_shape(N, G, force3);
    if (!sh.ok)
        return fail(QVA_ERR_UNSUPPORTED,
                    G > 1 ? "sharded circulant mixer: N=" + std::to_string(N) + " has no four-step split M1*M2 (13-smooth, <= 8192) with " +
                                std::to_string(G) + " | M1 and M2"
                          : "circulant mixer: no FFT plan for N=" + std::to_string(N) + " (Bluestein length would exceed 8192^2)");
    fp->whole = sh.whole;
    fp->bluestein = sh.bluestein;
    fp->M = sh.M;
    fp->M1 = sh.M1;
    fp->M2 = sh.M2;
    fp->cw = sh.cw;
    fp->rb = sh.rb;
    if (sh.levels == 3) {
        fp->levels = 3;
        fp->Mi1 = sh.Mi1;
        fp->Mi2 = sh.Mi2;
        fp->cw2 = sh.cw2;
        fp->rb2 = sh.rb2;
        const uint64_t R = (uint64_t)sh.Mi1 * sh.Mi2;
        if (R > (uint64_t)INT32_MAX) return fail(QVA_ERR_UNSUPPORTED, "three-level FFT row too long");
        fp->M2 = (int)R;  // top-level row length (column count of the top-level column pass)
        if (!make_sub(fp->M1, fp->col, tw) || !make_sub(fp->Mi1, fp->col2, tw) || !make_sub(fp->Mi2, fp->row, tw))
            return fail(QVA_ERR_UNSUPPORTED, "FFT planning failed");
        fp->big_shift = 11;
        if (!make_big_tables(N, &fp->d_big_lo, &fp->d_big_hi) || !make_big_tables(R, &fp->d_in_lo, &fp->d_in_hi))
            return fail(QVA_ERR_OUT_OF_MEMORY, "cudaMalloc (FFT twiddles) failed");
        fp->n_partials = std::max(col_grid(fp), fp->M2 / 4);  // fused-stage column blocks may be 4 wide
        if (cudaMalloc(&fp->partials, fp->n_partials * 2 * sizeof(double)) != cudaSuccess)
            return fail(QVA_ERR_OUT_OF_MEMORY, "cudaMalloc (FFT partials) failed");
    } else if (fp->whole) {
        if (!make_sub((int)N, fp->row, tw, false)) return fail(QVA_ERR_UNSUPPORTED, "FFT planning failed");
    } else {
        if (!make_sub(fp->M1, fp->col, tw) || !make_sub(fp->M2, fp->row, tw))
            return fail(QVA_ERR_UNSUPPORTED, "FFT planning failed");
        // four-step twiddles w_M^r = hi[r >> s] * lo[r & (2^s - 1)]
        const int s = 11;
        const uint64_t B = 1ull << s, M = fp->M;
        const uint64_t nhi = (M + B - 1) / B;
        std::vector<double2> lo(B), hi(nhi);
        for (uint64_t j = 0; j < B; ++j) {
            const long double ang = -2.0L * kPiL * (long double)j / (long double)M;
            lo[j] = make_double2((double)cosl(ang), (double)sinl(ang));
        }
        for (uint64_t j = 0; j < nhi; ++j) {
            const long double ang = -2.0L * kPiL * (long double)((j * B) % M) / (long double)M;
            hi[j] = make_double2((double)cosl(ang), (double)sinl(ang));
        }
        fp->big_shift = s;
        if (cudaMalloc(&fp->d_big_lo, B * sizeof(double2)) != cudaSuccess ||
            cudaMalloc(&fp->d_big_hi, nhi * sizeof(double2)) != cudaSuccess)
            return fail(QVA_ERR_OUT_OF_MEMORY, "cudaMalloc (FFT twiddles) failed");
        cudaMemcpy(fp->d_big_lo, lo.data(), B * sizeof(double2), cudaMemcpyHostToDevice);
        cudaMemcpy(fp->d_big_hi, hi.data(), nhi * sizeof(double2), cudaMemcpyHostToDevice);
        fp->n_partials = std::max(col_grid(fp), fp->M2 / 4);  // fused-stage column blocks may be 4 wide
        if (cudaMalloc(&fp->partials, fp->n_partials * 2 * sizeof(double)) != cudaSuccess)
            return fail(QVA_ERR_OUT_OF_MEMORY, "cudaMalloc (FFT partials) failed");
    }
    if (cudaMalloc(&fp->d_tw, std::max<size_t>(tw.size(), 1) * sizeof(double2)) != cudaSuccess)
        return fail(QVA_ERR_OUT_OF_MEMORY, "cudaMalloc (FFT tables) failed");
    cudaMemcpy(fp->d_tw, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice);
    if (!fp->whole && !fp->bluestein && G == 1) {
        auto fs_tab = [&](int n, bool col, double2 **dst) -> bool {
            std::vector<double2> t;
            if (!(col ? fs_col_available(n) : fs_row_available(n)) || !fs_stage_tables(n, col, t)) return true;
            if (cudaMalloc(dst, t.size() * sizeof(double2)) != cudaSuccess) return false;
            cudaMemcpy(*dst, t.data(), t.size() * sizeof(double2), cudaMemcpyHostToDevice);
            return true;
        };
        const int cols = fp->M2, rowlen = fp->levels == 3 ? fp->Mi2 : fp->M2;
        bool ok = true;
        if (fs_col_width(fp->M1) && cols % fs_col_width(fp->M1) == 0) ok = ok && fs_tab(fp->M1, true, &fp->fs_col);
        if (fp->levels == 3 && fs_col_width(fp->Mi1) && fp->Mi2 % fs_col_width(fp->Mi1) == 0)
            ok = ok && fs_tab(fp->Mi1, true, &fp->fs_col2);
        const uint64_t nrows = fp->levels == 3 ? (uint64_t)fp->M1 * fp->Mi1 : (uint64_t)fp->M1;
        const int rbk = fs_row_block(rowlen);
        if (rbk > 0 && nrows % rbk == 0)
            ok = ok && fs_tab(rowlen, false, &fp->fs_row);
        if (!ok) return fail(QVA_ERR_OUT_OF_MEMORY, "cudaMalloc (FFT fused-stage tables) failed");
    }
    qva_status st = upload_roots();
    if (st != QVA_OK) return fail(st, "");
    cudaFuncSetAttribute(fft_col_kernel<kFftThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, kColSmemMax);
    cudaFuncSetAttribute(fft_col_kernel<kFftThreads / 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kColSmemMax);
    cudaFuncSetAttribute(fft_row_kernel<>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRowSmemMax);
    cudaFuncSetAttribute(fft_row_kernel<kFftThreads / 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRowSmemMax);
    for (const auto &cl : kCodelets) {
        cudaFuncSetAttribute(cl.col, cudaFuncAttributeMaxDynamicSharedMemorySize, kColSmemMax);
        cudaFuncSetAttribute(cl.col_half, cudaFuncAttributeMaxDynamicSharedMemorySize, kColSmemMax);
        cudaFuncSetAttribute(cl.row, cudaFuncAttributeMaxDynamicSharedMemorySize, kRowSmemMax);
        cudaFuncSetAttribute(cl.row_half, cudaFuncAttributeMaxDynamicSharedMemorySize, kRowSmemMax);
    }
    cudaFuncSetAttribute(fft_whole_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * (int)sizeof(double2));
    if (fp->bluestein) {
        // kernel b_m = conj(c_m) for |m| < N on the length-M circle (b is even), then B = F_M b
        const uint64_t M = fp->M;
        std::vector<double2> b(M, make_double2(0.0, 0.0));
        for (uint64_t m = 0; m < N; ++m) {
            const uint64_t r = (m * m) % (2 * N);
            const long double ang = kPiL * (long double)r / (long double)N;
            const double2 v = make_double2((double)cosl(ang), (double)sinl(ang));  // conj(exp(-i ang))
            b[m] = v;
            if (m) b[M - m] = v;
        }
        if (cudaMalloc(&fp->bhat, M * sizeof(double2)) != cudaSuccess ||
            cudaMalloc(&fp->work, M * sizeof(double2)) != cudaSuccess)
            return fail(QVA_ERR_OUT_OF_MEMORY, "cudaMalloc (Bluestein buffers) failed");
        cudaMemcpy(fp->bhat, b.data(), M * sizeof(double2), cudaMemcpyHostToDevice);
        ColArgs c = col_args(fp);
        c.in = fp->bhat;
        c.in_len = M;
        c.out = fp->bhat;
        c.out_len = M;
        c.N = M;
        c.do_fwd = 1;
        const size_t sc = with_stage_tw(c, col_smem(fp), kColSmemMax, fp->cw * fp->M1);
        col_kernel_for(fp->M1, false)<<<col_grid(fp), kFftThreads, sc>>>(c);
        RowArgs w = row_args(fp, fp->bhat);
        w.fwd_only = 1;
        const size_t sr = with_stage_tw(w, row_smem(fp), kRowSmemMax, fp->rb * fp->M2);
        row_kernel_for(fp->M2)<<<row_grid(fp), kFftThreads, sr>>>(w);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return fail(QVA_ERR_CUDA, std::string("Bluestein setup: ") + cudaGetErrorString(e));
    }
    *out = fp;
    return QVA_OK;
}

void fft_plan_destroy(FftPlan *fp) {
    if (!fp) return;
    cudaFree(fp->d_tw);
    cudaFree(fp->d_big_lo);
    cudaFree(fp->d_big_hi);
    cudaFree(fp->partials);
    cudaFree(fp->work);
    cudaFree(fp->bhat);
    cudaFree(fp->d_in_lo);
    cudaFree(fp->d_in_hi);
    cudaFree(fp->d_theta);
    cudaFree(fp->fs_col);
    cudaFree(fp->fs_col2);
    cudaFree(fp->fs_row);
    for (int k = 0; k < fp->n_aux; ++k) {
        cudaStreamDestroy(fp->aux[k]);
        cudaEventDestroy(fp->ev_join[k]);
    }
    if (fp->ev_fork) cudaEventDestroy(fp->ev_fork);
    delete fp;
}

void fft_permute_spectrum(const FftPlan *fp, const double *lambda, double *lambda_perm) {
    if (fp->whole || fp->bluestein) {  // consumed in natural order
        memcpy(lambda_perm, lambda, fp->N * sizeof(double));
        return;
    }
    if (fp->levels == 3) {  // position k1*R + k2*Mi2 + k3 holds bin k1 + M1*(k2 + Mi1*k3)
        const uint64_t M1 = fp->M1, A = fp->Mi1, B = fp->Mi2, R = A * B;
        for (uint64_t k1 = 0; k1 < M1; ++k1)
            for (uint64_t k2 = 0; k2 < A; ++k2)
                for (uint64_t k3 = 0; k3 < B; ++k3) lambda_perm[k1 * R + k2 * B + k3] = lambda[k1 + M1 * (k2 + A * k3)];
        return;
    }
    const uint64_t M1 = fp->M1, M2 = fp->M2;
    for (uint64_t k1 = 0; k1 < M1; ++k1)
        for (uint64_t k2 = 0; k2 < M2; ++k2) lambda_perm[k1 * M2 + k2] = lambda[k1 + M1 * k2];
}

// Three-level row transform of `nmat` consecutive top-level rows (matrices Mi1 x Mi2) starting at
// global top-level row mat_off: inner column FFTs (+ w_{M2} twiddle), inner rows (forward FFT,
// spectrum, inverse FFT, inverse w_{M2} twiddle), inner inverse column FFTs + the top-level
// inverse twiddle w_N^{-x k1}.  Row-local: sharded plans run it on their own row blocks.
// fused-stage launch arguments from the engine's (kernels_fft_fs.cu)
static FsColArgs fs_col_args(const FftPlan *fp, const double2 *tab, const ColArgs &c) {
    FsColArgs f{};
    f.in = c.in;
    f.out = c.out;
    f.M2 = c.M2;
    f.col_off = c.col_off;
    f.M2g = c.M2g;
    f.mat_stride = c.mat_stride;
    f.mat_off = c.mat_off;
    f.init = c.init;
    f.ops = c.ops;
    f.q = c.q;
    f.amp0 = c.amp0;
    f.gamma = c.gamma;
    f.partials = fp->partials;
    f.tw = tab;
    f.big_lo = c.big_lo;
    f.big_hi = c.big_hi;
    f.big_shift = c.big_shift;
    f.otw_lo = c.otw_lo;
    f.otw_hi = c.otw_hi;
    f.otw_shift = c.otw_shift;
    return f;
}
static FsRowArgs fs_row_args(const FftPlan *fp, const double2 *tab, const RowArgs &w, const double2 *lo,
                             const double2 *hi) {
    FsRowArgs f{};
    f.buf = w.buf;
    f.row_off = w.row_off;
    f.row_mod = w.row_mod;
    f.spec = w.spec;
    f.lam_perm = w.lam_perm;
    f.beta = w.beta;
    f.scale = w.scale;
    f.ec = w.ec;
    if (w.spec == 0) {
        const double d = w.ec.x * w.ec.x + w.ec.y * w.ec.y;  // e0 / ec
        f.e0_over_ec = make_double2((w.e0.x * w.ec.x + w.e0.y * w.ec.y) / d, (w.e0.y * w.ec.x - w.e0.x * w.ec.y) / d);
    }
    f.tw = tab;
    f.big_lo = lo;
    f.big_hi = hi;
    f.big_shift = fp->big_shift;
    return f;
}

// untimed: the launches overlap with other groups' on auxiliary streams (counted as K_FFT_INNER, no
// event brackets: per-launch events between thousands of short grouped launches cost more than
// the grouping gains)
static qva_status inner_rows3(FftPlan *fp, double2 *psi, int nmat, int mat_off, const FftRun &r, double beta,
                              cudaStream_t s, LaunchObserver *obs, bool untimed = false) {
    const double N = (double)fp->N;
    const uint64_t R = (uint64_t)fp->Mi1 * fp->Mi2;
    ColArgs c = col_args(fp);
    c.M1 = fp->Mi1;
    c.M2 = fp->Mi2;
    c.M2g = fp->Mi2;
    c.cw = fp->cw2;
    c.lcw = fp->cw2 == 8 ? 3 : fp->cw2 == 4 ? 2 : fp->cw2 == 2 ? 1 : 0;
    c.m1mag = div_magic((uint32_t)fp->Mi1);
    c.sf = fp->col2;
    c.big_lo = fp->d_in_lo;
    c.big_hi = fp->d_in_hi;
    c.in = psi;
    c.out = psi;
    c.in_len = R;
    c.out_len = R;
    c.N = R;
    c.mat_stride = R;
    c.mat_off = mat_off;
    c.otw_lo = fp->d_big_lo;
    c.otw_hi = fp->d_big_hi;
    c.otw_shift = fp->big_shift;
    const dim3 gc((fp->Mi2 + c.cw - 1) / c.cw, nmat);
    // 256-thread CTAs, two per SM, when the block fits (as for the top-level column pass)
    bool half = col_smem_bytes(c.cw, fp->Mi1, true) <= kColHalfSmemMax;
    for (int st = 0; st < fp->col2.ns && half; ++st)
        if (fp->col2.n / fp->col2.r[st] > nb_of(fp->col2.r[st]) * (kFftThreads / 2)) half = false;
    static int half_env3 = [] {
        const char *e = getenv("QVA_FFT_COL256");
        return e ? atoi(e) : 1;
    }();
    half = half && half_env3 != 0;
    const size_t smem_c = with_stage_tw(c, col_smem_bytes(c.cw, fp->Mi1, true), half ? kColHalfSmemMax : kColSmemMax,
                                        c.cw * fp->Mi1);
    auto cols = [&](int inv, int ops, int fwd) -> qva_status {
        c.do_inv = inv;
        c.do_fwd = fwd;
        c.ops = ops;
        if (untimed) obs->count(K_FFT_INNER, 32.0 * (double)R * nmat);
        else obs->begin(K_FFT_COL, 32.0 * (double)R * nmat, s);
        cudaError_t e;
        if (fp->fs_col2 && !c.xg) {
            e = fs_col_launch(fp->Mi1, fs_col_args(fp, fp->fs_col2, c), fp->Mi2, nmat, inv != 0, fwd != 0, s);
        } else {
            col_kernel_for(fp->Mi1, half)<<<gc, half ? kFftThreads / 2 : kFftThreads, smem_c, s>>>(c);
            e = cudaGetLastError();
        }
        if (!untimed) obs->end();
        if (e != cudaSuccess) {
            set_error(std::string("fft_col_kernel (inner): ") + cudaGetErrorString(e));
            return QVA_ERR_CUDA;
        }
        return QVA_OK;
    };
    QVA_TRY(cols(0, 0, 1));
    RowArgs w = row_args(fp, psi);
    w.M1 = nmat * fp->Mi1;
    w.M2 = fp->Mi2;
    w.rb = fp->rb2;
    w.m2mag = div_magic((uint32_t)fp->Mi2);
    w.big_lo = fp->d_in_lo;
    w.big_hi = fp->d_in_hi;
    w.row_off = mat_off * fp->Mi1;
    w.row_mod = fp->Mi1;
    if (r.lambda_perm) {
        w.spec = 1;
        w.lam_perm = r.lambda_perm;
        w.beta = beta;
        w.scale = 1.0 / N;
    } else {
        w.spec = 0;
        w.e0 = make_double2(cos(-beta * r.lam0) / N, sin(-beta * r.lam0) / N);
        w.ec = make_double2(cos(-beta * r.lamc) / N, sin(-beta * r.lamc) / N);
    }
    const double row_bytes = 32.0 * (double)R * nmat + (r.lambda_perm ? 8.0 * (double)R * nmat : 0.0);
    if (untimed) obs->count(K_FFT_INNER, row_bytes);
    else obs->begin(K_FFT_ROW, row_bytes, s);
    // 256-thread CTAs over half the rows, two or more per SM, when the stages fit 256 threads
    int rbh = 0;
    for (int x = fp->rb2 / 2; x >= 1 && !rbh; --x)
        if (((uint64_t)nmat * fp->Mi1) % x == 0) rbh = x;
    bool rhalf = half_env3 != 0 && rbh >= 1 && row_smem_bytes(rbh, fp->Mi2) <= kColHalfSmemMax;
    for (int st = 0; st < fp->row.ns && rhalf; ++st)
        if (fp->row.n / fp->row.r[st] > nb_of(fp->row.r[st]) * (kFftThreads / 2)) rhalf = false;
    if (rhalf) w.rb = rbh;
    const size_t smem_r3 = with_stage_tw(w, row_smem_bytes(w.rb, fp->Mi2), rhalf ? kColHalfSmemMax : kRowSmemMax,
                                         w.rb * fp->Mi2);
    cudaError_t e;
    if (fp->fs_row && !w.xg && ((uint64_t)nmat * fp->Mi1) % fs_row_block(fp->Mi2) == 0) {
        e = fs_row_launch(fp->Mi2, fs_row_args(fp, fp->fs_row, w, fp->d_in_lo, fp->d_in_hi), (uint64_t)nmat * fp->Mi1, s);
    } else {
        row_kernel_for(fp->Mi2, rhalf)<<<nmat * fp->Mi1 / w.rb, rhalf ? kFftThreads / 2 : kFftThreads, smem_r3, s>>>(w);
        e = cudaGetLastError();
    }
    if (!untimed) obs->end();
    if (e != cudaSuccess) {
        set_error(std::string("fft_row_kernel (inner): ") + cudaGetErrorString(e));
        return QVA_ERR_CUDA;
    }
    return cols(1, OP_OUTER_TW, 0);
}

// The three inner passes of a three-level layer, optionally in groups of QVA_FFT_GROUP top-level rows
// (matrices) spread round-robin over QVA_FFT_STREAMS auxiliary streams: each group's data (group x
// Mi1 x Mi2 x 16 B) is read from HBM by its inner column pass and stays in L2 for its row and
// inverse column passes, while the groups on the other streams fill the SMs.
static qva_status inner_rows3_grouped(FftPlan *fp, double2 *psi, int nmat, int mat_off, const FftRun &r, double beta,
                                      cudaStream_t s, LaunchObserver *obs) {
    static const int g_env = [] {
        const char *e = getenv("QVA_FFT_GROUP");
        return e ? atoi(e) : -1;
    }();
    static const int k_env = [] {
        const char *e = getenv("QVA_FFT_STREAMS");
        return e ? std::max(1, std::min(4, atoi(e))) : 2;
    }();
    const uint64_t R = (uint64_t)fp->Mi1 * fp->Mi2;
    // default: groups of ~20 MB (two matrices at 12!: 95.6 ms per p=4 evolution against 102.6 ms
    // ungrouped; one matrix 107.4, four 99.2, eight 102.9; two streams beat three or four)
    const int g = g_env >= 0 ? g_env : (int)std::max<uint64_t>(2, std::min<uint64_t>(8, ((20ull << 20) + 8 * R) / (16 * R)));
    if (g <= 0 || 4 * g > nmat) return inner_rows3(fp, psi, nmat, mat_off, r, beta, s, obs);
    if (fp->n_aux < k_env) {
        for (int k = fp->n_aux; k < k_env; ++k) {
            QVA_CUDA_TRY(cudaStreamCreateWithFlags(&fp->aux[k], cudaStreamNonBlocking));
            QVA_CUDA_TRY(cudaEventCreateWithFlags(&fp->ev_join[k], cudaEventDisableTiming));
        }
        if (!fp->ev_fork) QVA_CUDA_TRY(cudaEventCreateWithFlags(&fp->ev_fork, cudaEventDisableTiming));
        fp->n_aux = k_env;
    }
    QVA_CUDA_TRY(cudaEventRecord(fp->ev_fork, s));
    for (int k = 0; k < k_env; ++k) QVA_CUDA_TRY(cudaStreamWaitEvent(fp->aux[k], fp->ev_fork, 0));
    int i = 0;
    for (int m0 = 0; m0 < nmat; m0 += g, ++i) {
        const int gm = std::min(g, nmat - m0);
        QVA_TRY(inner_rows3(fp, psi + (uint64_t)m0 * R, gm, mat_off + m0, r, beta, fp->aux[i % k_env], obs, true));
    }
    for (int k = 0; k < k_env; ++k) {
        QVA_CUDA_TRY(cudaEventRecord(fp->ev_join[k], fp->aux[k]));
        QVA_CUDA_TRY(cudaStreamWaitEvent(s, fp->ev_join[k], 0));
    }
    return QVA_OK;
}

qva_status fft_run(FftPlan *fp, const FftRun &r, cudaStream_t s, LaunchObserver *obs) {
    const double N = (double)fp->N, M = (double)fp->M;
    const double state_bytes = 16.0 * N, q_bytes = 8.0 * N;
    if (fp->whole) {
        WholeArgs a{};
        a.psi = r.psi;
        a.q = r.q;
        a.lambda_perm = r.lambda_perm;
        a.lam0 = r.lam0;
        a.lamc = r.lamc;
        a.invN = 1.0 / N;
        a.p = r.p;
        a.mode = r.mode;
        a.init = r.init;
        a.amp0 = r.amp0;
        a.do_expect = r.expect ? 1 : 0;
        a.red_out = r.red_out;
        a.tw = fp->d_tw;
        a.sf = fp->row;
        const int nth = r.mode == 0 ? 2 * r.p : 1;
        if (fp->theta_cap < nth || !fp->d_theta) {
            cudaFree(fp->d_theta);
            fp->d_theta = nullptr;
            QVA_CUDA_TRY(cudaMalloc(&fp->d_theta, std::max(nth, 1) * sizeof(double)));
            fp->theta_cap = std::max(nth, 1);
        }
        double *dth = fp->d_theta;
        if (nth) QVA_CUDA_TRY(cudaMemcpyAsync(dth, r.theta, nth * sizeof(double), cudaMemcpyHostToDevice, s));
        a.theta = dth;
        obs->begin(K_FFT_ROW, state_bytes * (r.init ? 1 : 2) + q_bytes * (r.mode == 0 ? 1 : 0));
        fft_whole_kernel<<<1, kFftThreads, (size_t)fp->N * sizeof(double2), s>>>(a);
        cudaError_t e = cudaGetLastError();
        obs->end();
        if (e != cudaSuccess) {
            set_error(std::string("fft_whole_kernel: ") + cudaGetErrorString(e));
            return QVA_ERR_CUDA;
        }
        return QVA_OK;
    }
    const bool blu = fp->bluestein;
    double2 *W = blu ? fp->work : r.psi;
    const uint64_t Mi = fp->M;
    ColArgs c = col_args(fp);
    c.q = r.q;
    c.amp0 = r.amp0;
    c.lam0 = r.lam0;
    c.lamc = r.lamc;
    c.lam = blu ? r.lambda_perm : nullptr;
    size_t smem_c = col_smem(fp);
    const int gc = col_grid(fp), gr = row_grid(fp);
    int expect_slots = gc;  // partial slots written by the last column pass
    // column pass with 256-thread CTAs, two per SM (their barrier stalls overlap), when every
    // stage's butterflies of one column fit a 256-thread round and two column blocks fit smem
    static int half_env = [] {
        const char *e = getenv("QVA_FFT_COL256");
        return e ? atoi(e) : 1;
    }();
    bool col_half = half_env != 0 && smem_c <= kColHalfSmemMax;
    for (int st = 0; st < fp->col.ns && col_half; ++st)
        if (fp->col.n / fp->col.r[st] > nb_of(fp->col.r[st]) * (kFftThreads / 2)) col_half = false;
    smem_c = with_stage_tw(c, smem_c, col_half ? kColHalfSmemMax : (size_t)kColSmemMax, fp->cw * fp->M1);

    // in/out: nullptr -> W; the state (r.psi, length N) is named explicitly
    auto launch_col = [&](const double2 *in, uint64_t in_len, double2 *out, uint64_t out_len, int init, int inv,
                          int ops, double gamma, double beta, int fwd) -> qva_status {
        c.in = in;
        c.in_len = in_len;
        c.out = out;
        c.out_len = out_len;
        c.init = init;
        c.do_inv = inv;
        c.do_fwd = fwd;
        c.ops = ops;
        c.gamma = gamma;
        c.beta = beta;
        const double bytes = (init ? 0.0 : 16.0 * (double)std::min<uint64_t>(in_len, Mi)) +
                             16.0 * (double)std::min<uint64_t>(out_len, Mi) +
                             ((ops & (OP_PHASE | OP_EXPECT)) ? q_bytes : 0.0) + ((ops & OP_SPEC) && c.lam ? 8.0 * N : 0.0);
        obs->begin(K_FFT_COL, bytes);
        expect_slots = gc;
        cudaError_t e;
        if (fp->fs_col && !blu && !(ops & ~(OP_PHASE | OP_EXPECT)) && in_len == (uint64_t)fp->N &&
            out_len == (uint64_t)fp->N && (inv || fwd)) {
            FsColArgs f = fs_col_args(fp, fp->fs_col, c);
            expect_slots = fp->M2 / fs_col_width(fp->M1);
            e = fs_col_launch(fp->M1, f, fp->M2, 1, inv != 0, fwd != 0, s);
        } else {
            col_kernel_for(fp->M1, col_half)<<<gc, col_half ? kFftThreads / 2 : kFftThreads, smem_c, s>>>(c);
            e = cudaGetLastError();
        }
        obs->end();
        if (e != cudaSuccess) {
            set_error(std::string("fft_col_kernel: ") + cudaGetErrorString(e));
            return QVA_ERR_CUDA;
        }
        return QVA_OK;
    };
    // direct: spectrum exp(-i beta lambda)/N; Bluestein: kernel spectrum B (or conj B) / M
    auto launch_row = [&](double beta, int bconj) -> qva_status {
        if (fp->levels == 3) return inner_rows3_grouped(fp, W, fp->M1, 0, r, beta, s, obs);
        RowArgs w = row_args(fp, W);
        double extra = 0.0;
        if (blu) {
            w.spec = 2;
            w.bhat = fp->bhat;
            w.conj_b = bconj;
            w.scale = 1.0 / M;
            extra = 16.0 * M;
        } else if (r.lambda_perm) {
            w.spec = 1;
            w.lam_perm = r.lambda_perm;
            w.beta = beta;
            w.scale = 1.0 / N;
            extra = 8.0 * N;
        } else {
            w.spec = 0;
            w.e0 = make_double2(cos(-beta * r.lam0) / N, sin(-beta * r.lam0) / N);
            w.ec = make_double2(cos(-beta * r.lamc) / N, sin(-beta * r.lamc) / N);
        }
        obs->begin(K_FFT_ROW, 32.0 * M + extra);
        cudaError_t e;
        if (fp->fs_row && !blu) {
            e = fs_row_launch(fp->M2, fs_row_args(fp, fp->fs_row, w, fp->d_big_lo, fp->d_big_hi), (uint64_t)fp->M1, s);
        } else {
            const size_t smem_r = with_stage_tw(w, row_smem(fp), kRowSmemMax, fp->rb * fp->M2);
            row_kernel_for(fp->M2)<<<gr, kFftThreads, smem_r, s>>>(w);
            e = cudaGetLastError();
        }
        obs->end();
        if (e != cudaSuccess) {
            set_error(std::string("fft_row_kernel: ") + cudaGetErrorString(e));
            return QVA_ERR_CUDA;
        }
        return QVA_OK;
    };
    auto reduce = [&]() -> qva_status {
        obs->begin(K_REDUCE, 16.0 * expect_slots);
        cudaError_t e = launch_reduce_partials(fp->partials, expect_slots, 1, r.red_out, s);
        obs->end();
        if (e != cudaSuccess) {
            set_error(std::string("reduce: ") + cudaGetErrorString(e));
            return QVA_ERR_CUDA;
        }
        return QVA_OK;
    };
    const uint64_t Nn = fp->N;
    if (!blu) {
        if (r.mode == 1) {
            QVA_TRY(launch_col(r.psi, Nn, r.psi, Nn, 0, 0, 0, 0.0, 0.0, 1));
            QVA_TRY(launch_row(r.theta[0], 0));
            return launch_col(r.psi, Nn, r.psi, Nn, 0, 1, 0, 0.0, 0.0, 0);
        }
        for (int k = 0; k < r.p; ++k) {
            QVA_TRY(launch_col(r.psi, Nn, r.psi, Nn, k == 0 ? r.init : 0, k > 0, OP_PHASE, r.theta[2 * k], 0.0, 1));
            QVA_TRY(launch_row(r.theta[2 * k + 1], 0));
        }
        if (r.p > 0) {
            QVA_TRY(launch_col(r.psi, Nn, r.psi, Nn, 0, 1, r.expect ? OP_EXPECT : 0, 0.0, 0.0, 0));
            if (r.expect) QVA_TRY(reduce());
        }
        return QVA_OK;
    }
    // Bluestein
    if (r.mode == 1) {
        QVA_TRY(launch_col(r.psi, Nn, W, Mi, 0, 0, OP_CHIRP | OP_MASK, 0.0, 0.0, 1));
        QVA_TRY(launch_row(0.0, 0));
        QVA_TRY(launch_col(W, Mi, W, Mi, 0, 1, OP_SPEC | OP_MASK, 0.0, r.theta[0], 1));
        QVA_TRY(launch_row(0.0, 1));
        return launch_col(W, Mi, r.psi, Nn, 0, 1, OP_CHIRP_CONJ | OP_MASK, 0.0, 0.0, 0);
    }
    for (int k = 0; k < r.p; ++k) {
        if (k == 0) {
            QVA_TRY(launch_col(r.psi, Nn, W, Mi, r.init, 0, OP_PHASE | OP_CHIRP | OP_MASK, r.theta[0], 0.0, 1));
        } else {
            // conj(c) * phase * c = phase
            QVA_TRY(launch_col(W, Mi, W, Mi, 0, 1, OP_PHASE | OP_MASK, r.theta[2 * k], 0.0, 1));
        }
        QVA_TRY(launch_row(0.0, 0));
        QVA_TRY(launch_col(W, Mi, W, Mi, 0, 1, OP_SPEC | OP_MASK, 0.0, r.theta[2 * k + 1], 1));
        QVA_TRY(launch_row(0.0, 1));
    }
    if (r.p > 0) {
        QVA_TRY(launch_col(W, Mi, r.psi, Nn, 0, 1, OP_CHIRP_CONJ | OP_MASK | (r.expect ? OP_EXPECT : 0), 0.0, 0.0, 0));
        if (r.expect) QVA_TRY(reduce());
    }
    return QVA_OK;
}

// ------------------------------------------------------------------------------------------
// Sharded four-step (COMM-psi for QWOA): G shards hold contiguous row blocks of
// the natural layout (x = x1*M2 + x2, rows x1 in [s*M1/G, (s+1)*M1/G)); the column pass runs in a
// column layout (shard s: all x1, columns x2 in [s*M2/G, ...)), reached by an all-to-all
// transpose (io.to_col / io.to_row: NCCL, or a block transpose for virtual shards).  Two
// transposes per layer; the row pass runs on the shard's own rows in place.
// ------------------------------------------------------------------------------------------
bool fft_shardable(const FftPlan *fp, int G) {
    return G >= 1 && !fp->whole && !fp->bluestein && fp->M1 % G == 0 && fp->M2 % G == 0;
}

qva_status fft_run_sharded(FftPlan *fp, const FftRun &r, FftShardIO &io, cudaStream_t s, LaunchObserver *obs) {
    const int G = io.G;
    if (!fft_shardable(fp, G)) {
        set_error("circulant mixer: sharding needs a direct four-step plan with G | M1 and G | M2");
        return QVA_ERR_UNSUPPORTED;
    }
    const uint64_t NG = fp->N / G;
    const int M1s = fp->M1 / G, M2s = fp->M2 / G;
    const double N = (double)fp->N;
    ColArgs c = col_args(fp);
    c.M2 = M2s;
    c.M2g = fp->M2;
    c.amp0 = r.amp0;
    c.cw = std::min(fp->cw, 8);
    while (c.cw > 1 && M2s % c.cw) c.cw >>= 1;  // keep whole column blocks inside a shard
    c.lcw = c.cw == 8 ? 3 : c.cw == 4 ? 2 : c.cw == 2 ? 1 : 0;
    const int gc = (M2s + c.cw - 1) / c.cw;
    const size_t smem_c = with_stage_tw(c, col_smem_bytes(c.cw, fp->M1), kColSmemMax, c.cw * fp->M1);
    int rb = 1;
    for (int x = 2; x <= 64; ++x)
        if (M1s % x == 0 && x * fp->M2 <= kMaxCta) rb = x;
    const size_t smem_r = row_smem_bytes(rb, fp->M2);
    if ((size_t)gc * io.local > (size_t)fp->n_partials) {
        cudaFree(fp->partials);
        fp->n_partials = gc * io.local;
        QVA_CUDA_TRY(cudaMalloc(&fp->partials, fp->n_partials * 2 * sizeof(double)));
    }
    // transposes fused into the pass stores (two-level plans; the three-level inner passes keep
    // the separate transposes)
    const bool fused = io.fused && fp->levels == 2 && G <= kMaxPeers;
    auto cols = [&](int init, int inv, int ops, double gamma, int fwd) -> qva_status {
        c.xg = fused ? G : 0;
        for (int t = 0; t < G && fused; ++t) c.xout[t] = io.row_dst[t];
        for (int ls = 0; ls < io.local; ++ls) {
            c.in = io.col + ls * NG;
            c.in_len = NG;
            c.out = io.col + ls * NG;
            c.out_len = NG;
            c.q = io.q_col + ls * NG;
            c.col_off = (io.first + ls) * M2s;
            c.partials = fp->partials + 2 * (size_t)ls * gc;
            c.init = init;
            c.do_inv = inv;
            c.do_fwd = fwd;
            c.ops = ops;
            c.gamma = gamma;
            obs->begin(K_FFT_COL, 16.0 * NG * (init ? 1 : 2) + ((ops & (OP_PHASE | OP_EXPECT)) ? 8.0 * NG : 0.0));
            col_kernel_for(fp->M1, false)<<<gc, kFftThreads, smem_c, s>>>(c);
            cudaError_t e = cudaGetLastError();
            obs->end();
            if (e != cudaSuccess) {
                set_error(std::string("fft_col_kernel: ") + cudaGetErrorString(e));
                return QVA_ERR_CUDA;
            }
        }
        return QVA_OK;
    };
    auto rows = [&](double beta) -> qva_status {
        if (fp->levels == 3) return inner_rows3(fp, r.psi, io.local * M1s, io.first * M1s, r, beta, s, obs);
        RowArgs w = row_args(fp, r.psi);
        w.rb = rb;
        w.row_off = io.first * M1s;
        w.xg = fused ? G : 0;
        w.M2s = M2s;
        for (int t = 0; t < G && fused; ++t) w.xout[t] = io.col_dst[t];
        if (r.lambda_perm) {
            w.spec = 1;
            w.lam_perm = r.lambda_perm;
            w.beta = beta;
            w.scale = 1.0 / N;
        } else {
            w.spec = 0;
            w.e0 = make_double2(cos(-beta * r.lam0) / N, sin(-beta * r.lam0) / N);
            w.ec = make_double2(cos(-beta * r.lamc) / N, sin(-beta * r.lamc) / N);
        }
        obs->begin(K_FFT_ROW, 32.0 * NG * io.local + (r.lambda_perm ? 8.0 * NG * io.local : 0.0));
        const size_t smem_rs = with_stage_tw(w, smem_r, kRowSmemMax, rb * fp->M2);
        row_kernel_for(fp->M2)<<<io.local * M1s / rb, kFftThreads, smem_rs, s>>>(w);
        cudaError_t e = cudaGetLastError();
        obs->end();
        if (e != cudaSuccess) {
            set_error(std::string("fft_row_kernel: ") + cudaGetErrorString(e));
            return QVA_ERR_CUDA;
        }
        return QVA_OK;
    };
    // after a pass: the data is in the other layout already (fused) or gets there by a transpose
    auto after_cols = [&]() { return fused ? io.barrier() : io.to_row(io.col, r.psi); };
    auto after_rows = [&]() { return fused ? io.barrier() : io.to_col(r.psi, io.col); };
    if (r.mode == 1) {
        QVA_TRY(io.to_col(r.psi, io.col));
        QVA_TRY(cols(0, 0, 0, 0.0, 1));
        QVA_TRY(after_cols());
        QVA_TRY(rows(r.theta[0]));
        QVA_TRY(after_rows());
        QVA_TRY(cols(0, 1, 0, 0.0, 0));
        return after_cols();
    }
    if (!r.init) QVA_TRY(io.to_col(r.psi, io.col));
    for (int k = 0; k < r.p; ++k) {
        QVA_TRY(cols(k == 0 ? r.init : 0, k > 0, OP_PHASE, r.theta[2 * k], 1));
        QVA_TRY(after_cols());
        QVA_TRY(rows(r.theta[2 * k + 1]));
        QVA_TRY(after_rows());
    }
    if (r.p > 0) {
        QVA_TRY(cols(0, 1, r.expect ? OP_EXPECT : 0, 0.0, 0));
        if (r.expect) {
            obs->begin(K_REDUCE, 16.0 * gc * io.local);
            cudaError_t e = launch_reduce_partials(fp->partials, (uint64_t)gc * io.local, 1, r.red_out, s);
            obs->end();
            if (e != cudaSuccess) {
                set_error(std::string("reduce: ") + cudaGetErrorString(e));
                return QVA_ERR_CUDA;
            }
        }
    }
    return after_cols();
}

}  // namespace qva
