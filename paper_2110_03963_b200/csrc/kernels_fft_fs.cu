// kernels_fft_fs.cu -- fused-stage FFT passes of the circulant (QWOA) mixer
// U(beta) = F^-1 diag(exp(-i beta lambda)) F (Sec. 3; readings R3, R4) for the
// compiled sub-FFT lengths of the cfg3 / 12! plans.  Same row / column passes, same arithmetic
// order per element and the same twiddle conventions as the shared-memory Stockham engine of
// kernels_fft.cu (whose kernels remain the fallback for every other length and for the Bluestein
// and sharded passes); what changes is where the data lives between stages (fft_fs.h):
//
//   * a transform's first Stockham stage (m = 1, inputs j + t*nb of butterfly j) loads its
//     inputs from global memory straight into registers (no block copy into shared memory);
//   * its last stage (outputs j + t*nb) multiplies the pass's final twiddle in registers and
//     stores straight to global memory;
//   * where one transform follows another in the same pass -- row: forward -> spectrum ->
//     inverse, column: inverse -> <Q> / phase -> forward -- the second runs its radices in
//     reverse order, so its first stage (radix R, m = 1) takes exactly the elements the first
//     transform's last stage (radix R, m = n/R) leaves in the thread's registers: the spectrum /
//     phase is applied there and the pair of stages costs no shared-memory round trip;
//   * final twiddles w^{K x} along a thread's elements x = j + t*nb are one table product for
//     t = 0 and a complex multiply per step (w^{K nb}) after that, instead of per-element tables;
//   * stage twiddles come from a per-codelet table in global memory (L1-resident), entry
//     (t-1)*m + k of stage (m, R) = w_{mR}^{t k}, inverse stages pre-conjugated.
//
// Shared-memory traffic per element of a row pass (768 = 16*16*3, forward + inverse):
// 128 B instead of 224 B, and 7 block barriers instead of 15.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <type_traits>
#include <utility>
#include <vector>

#include "fft_fs.h"
#include "qva_internal.h"

namespace qva {

namespace {

#include "fft_dft.cuh"

template <typename F, int... K>
__device__ __forceinline__ void fs_static_for_impl(F &f, std::integer_sequence<int, K...>) {
    (f(std::integral_constant<int, K>()), ...);
}
template <int N, typename F>
__device__ __forceinline__ void fs_static_for(F &&f) {
    fs_static_for_impl(f, std::make_integer_sequence<int, N>());
}

struct Arr8 {
    int v[8];
};
template <int... Rs>
constexpr Arr8 fs_fwd_arr() {
    Arr8 a{};
    int i = 0;
    ((a.v[i++] = Rs), ...);
    return a;
}
template <int... Rs>
constexpr Arr8 fs_rev_arr() {
    Arr8 a{};
    int i = (int)sizeof...(Rs);
    ((a.v[--i] = Rs), ...);
    return a;
}

// A compiled codelet: forward radix order Rs (direction d = 0), inverse = reversed (d = 1).
template <int... Rs>
struct FsC {
    static constexpr int S = (int)sizeof...(Rs);
    static constexpr int N = (Rs * ... * 1);
    static constexpr Arr8 F = fs_fwd_arr<Rs...>();
    static constexpr Arr8 I = fs_rev_arr<Rs...>();
    __host__ __device__ static constexpr int r(int d, int s) { return d ? I.v[s] : F.v[s]; }
    __host__ __device__ static constexpr int m(int d, int s) {
        int x = 1;
        for (int i = 0; i < s; ++i) x *= r(d, i);
        return x;
    }
    __host__ __device__ static constexpr int tw_dir(int d) {
        int o = 0;
        for (int i = 1; i < S; ++i) o += (r(d, i) - 1) * m(d, i);
        return o;
    }
    // table offset of stage s (s >= 1) of direction d
    __host__ __device__ static constexpr int off(int d, int s) {
        int o = d ? tw_dir(0) : 0;
        for (int i = 1; i < s; ++i) o += (r(d, i) - 1) * m(d, i);
        return o;
    }
    // swizzle for the m = 1 stores (stride R): radix 16 -> 4, radix 8 -> 3, else none
    __host__ __device__ static constexpr int swz() {
        return (r(0, 0) == 16 || r(1, 0) == 16) ? 4 : (r(0, 0) == 8 || r(1, 0) == 8) ? 3 : 0;
    }
};

template <int S>
struct FsAddr {
    double2 *buf;
    int stride;
    __device__ __forceinline__ static int sw(int i) { return S ? (i ^ ((i >> S) & 7)) : i; }
    __device__ __forceinline__ double2 *ptr(int f, int i) const { return buf + f * stride + sw(i); }
};

__device__ __forceinline__ double2 fs_big(const double2 *lo, const double2 *hi, int shift, uint64_t r) {
    const uint64_t mask = (1ull << shift) - 1;
    return cmul(__ldg(hi + (r >> shift)), __ldg(lo + (r & mask)));
}
__device__ __forceinline__ double2 conjd(double2 a) { return make_double2(a.x, -a.y); }

// butterfly J of a stage -> (transform f, butterfly j): rows j-fastest (f = J / nb), column
// blocks column-fastest (f = J % NT, NT a power of two)
template <bool CFAST, int NT, int nb>
__device__ __forceinline__ void fs_map(int J, int &f, int &j) {
    if constexpr (CFAST) {
        f = J & (NT - 1);
        j = J / NT;
    } else {
        f = J / nb;
        j = J - f * nb;
    }
}

// One in-place Stockham stage through shared memory (stage s >= 1 of direction d): inputs
// j + t*nb, twiddle w_{mR}^{t k} (k = j mod m), radix-R DFT, outputs (j - k) R + k + t m.
template <typename C, int D, int s, int T, int NT, bool CFAST, typename Ad>
__device__ __forceinline__ void fs_stage(const Ad &ad, const double2 *__restrict__ tw) {
    constexpr int N = C::N, R = C::r(D, s), M = C::m(D, s), nb = N / R, tot = NT * nb;
    constexpr int NB = (tot + T - 1) / T, OFF = C::off(D, s);
    double2 v[NB][R];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int J = threadIdx.x + b * T;
        if (tot % T == 0 || J < tot) {
            int f, j;
            fs_map<CFAST, NT, nb>(J, f, j);
#pragma unroll
            for (int t = 0; t < R; ++t) v[b][t] = *ad.ptr(f, j + t * nb);
        }
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int J = threadIdx.x + b * T;
        if (tot % T == 0 || J < tot) {
            int f, j;
            fs_map<CFAST, NT, nb>(J, f, j);
            const int k = j % M;
#pragma unroll
            for (int t = 1; t < R; ++t) v[b][t] = cmul(v[b][t], __ldg(tw + OFF + (t - 1) * M + k));
            dft<R>(v[b], D != 0);
            const int o = (j - k) * R + k;
#pragma unroll
            for (int t = 0; t < R; ++t) *ad.ptr(f, o + t * M) = v[b][t];
        }
    }
    __syncthreads();
}

// last stage of direction d from shared memory into registers (outputs j + t*nb, k = j)
template <typename C, int D, int T, int NT, bool CFAST, typename Ad, int NB, int R>
__device__ __forceinline__ void fs_last_stage(const Ad &ad, const double2 *__restrict__ tw, double2 (&v)[NB][R]) {
    constexpr int N = C::N, S = C::S, M = C::m(D, S - 1), nb = N / R, tot = NT * nb, OFF = C::off(D, S - 1);
    static_assert(R == C::r(D, S - 1) && M == nb, "last stage");
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int J = threadIdx.x + b * T;
        if (tot % T == 0 || J < tot) {
            int f, j;
            fs_map<CFAST, NT, nb>(J, f, j);
#pragma unroll
            for (int t = 0; t < R; ++t) v[b][t] = *ad.ptr(f, j + t * nb);
#pragma unroll
            for (int t = 1; t < R; ++t) v[b][t] = cmul(v[b][t], __ldg(tw + OFF + (t - 1) * M + j));
            dft<R>(v[b], D != 0);
        }
    }
}

// first stage (m = 1) of direction d on registers, outputs to shared memory at j*R + t
template <typename C, int D, int T, int NT, bool CFAST, typename Ad, int NB, int R>
__device__ __forceinline__ void fs_first_store(const Ad &ad, double2 (&v)[NB][R]) {
    constexpr int N = C::N, nb = N / R, tot = NT * nb;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int J = threadIdx.x + b * T;
        if (tot % T == 0 || J < tot) {
            int f, j;
            fs_map<CFAST, NT, nb>(J, f, j);
#pragma unroll
            for (int t = 0; t < R; ++t) *ad.ptr(f, j * R + t) = v[b][t];
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Row pass: NT rows of length N per CTA (row r of the block at buf + (blockIdx.x*NT + r) * N):
// forward FFT -> spectrum -> inverse FFT -> final twiddle w_M^{-K x2} (K = global row, mod
// row_mod for three-level inner rows), in place.  As fft_row_kernel with the spectrum folded:
// spec 0 multiplies every bin by ec (carried in the final twiddle) and bin 0 of global row 0 by
// e0 / ec on the registers.
// SM0: the block was copied into shared memory ahead (pipelined kernel) and stage 0 reads it there
template <typename C, int T, int NT, bool SM0>
__device__ __forceinline__ void fs_row_block(const FsRowArgs &a, double2 *A, uint64_t blk) {
    constexpr int N = C::N, S = C::S;
    static_assert(S >= 2 && C::r(0, S - 1) == C::r(1, 0), "reversed inverse order");
    const FsAddr<C::swz()> ad{A, N};
    double2 *rows = a.buf + blk * NT * N;
    const int grow0 = a.row_off + (int)blk * NT;
    // forward stage 0: global (or the prefetched block) -> registers -> DFT -> shared memory
    {
        constexpr int R = C::r(0, 0), nb = N / R, tot = NT * nb, NB = (tot + T - 1) / T;
        double2 v[NB][R];
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int J = threadIdx.x + b * T;
            if (tot % T == 0 || J < tot) {
                int f, j;
                fs_map<false, NT, nb>(J, f, j);
                const double2 *src = rows + f * N + j;
#pragma unroll
                for (int t = 0; t < R; ++t) v[b][t] = SM0 ? *ad.ptr(f, j + t * nb) : src[t * nb];
            }
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int J = threadIdx.x + b * T;
            if (tot % T == 0 || J < tot) dft<R>(v[b], false);
        }
        if constexpr (SM0) __syncthreads();
        fs_first_store<C, 0, T, NT, false>(ad, v);
    }
    __syncthreads();
    fs_static_for<S - 2>([&](auto sc) { fs_stage<C, 0, decltype(sc)::value + 1, T, NT, false>(ad, a.tw); });
    // forward last stage -> spectrum -> inverse stage 0, on the registers
    {
        constexpr int R = C::r(0, S - 1), nb = N / R, tot = NT * nb, NB = (tot + T - 1) / T;
        double2 v[NB][R];
        fs_last_stage<C, 0, T, NT, false>(ad, a.tw, v);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int J = threadIdx.x + b * T;
            if (tot % T == 0 || J < tot) {
                int f, j;
                fs_map<false, NT, nb>(J, f, j);
                if (a.spec == 0) {
                    if (j == 0 && grow0 + f == 0) v[b][0] = cmul(v[b][0], a.e0_over_ec);
                } else {
                    const double *lam = a.lam_perm + (uint64_t)(grow0 + f) * N + j;
#pragma unroll
                    for (int t = 0; t < R; ++t) {
                        double sn, cs;
                        sincos(-a.beta * __ldg(lam + t * nb), &sn, &cs);
                        v[b][t] = cmul(v[b][t], make_double2(cs * a.scale, sn * a.scale));
                    }
                }
                dft<R>(v[b], true);
            }
        }
        __syncthreads();  // every thread has read its last-stage inputs
        fs_first_store<C, 1, T, NT, false>(ad, v);
    }
    __syncthreads();
    fs_static_for<S - 2>([&](auto sc) { fs_stage<C, 1, decltype(sc)::value + 1, T, NT, false>(ad, a.tw); });
    // inverse last stage -> final twiddle -> global
    {
        constexpr int R = C::r(1, S - 1), nb = N / R, tot = NT * nb, NB = (tot + T - 1) / T;
        double2 v[NB][R];
        fs_last_stage<C, 1, T, NT, false>(ad, a.tw, v);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int J = threadIdx.x + b * T;
            if (tot % T == 0 || J < tot) {
                int f, j;
                fs_map<false, NT, nb>(J, f, j);
                const int kr = grow0 + f;
                const uint64_t K = (uint64_t)(a.row_mod ? kr % a.row_mod : kr);
                double2 w = conjd(fs_big(a.big_lo, a.big_hi, a.big_shift, K * (uint64_t)j));
                const double2 st = conjd(fs_big(a.big_lo, a.big_hi, a.big_shift, K * (uint64_t)nb));
                if (a.spec == 0) w = cmul(w, a.ec);
                double2 *dst = rows + f * N + j;
#pragma unroll
                for (int t = 0; t < R; ++t) {
                    dst[t * nb] = cmul(v[b][t], w);
                    if (t + 1 < R) w = cmul(w, st);
                }
            }
        }
    }
}

__device__ __forceinline__ void fs_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void fs_cp_wait_prev() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <typename C, int T, int NT, int MINB>
__global__ void __launch_bounds__(T, MINB) fs_row_kernel(const FsRowArgs a, uint64_t nblk) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    fs_row_block<C, T, NT, false>(a, reinterpret_cast<double2 *>(smem_raw), blockIdx.x);
}
// Persistent pipelined form: CTA b takes blocks b, b + grid, ...; while one block is transformed
// the next one's rows are in flight into the second shared-memory buffer (cp.async), so the
// first stage's loads no longer wait a memory latency per block.
template <typename C, int T, int NT, int MINB>
__global__ void __launch_bounds__(T, MINB) fs_row_pipe_kernel(const FsRowArgs a, uint64_t nblk) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int N = C::N, E = NT * N;
    double2 *A0 = reinterpret_cast<double2 *>(smem_raw);
    auto prefetch = [&](double2 *A, uint64_t blk) {
        const FsAddr<C::swz()> ad{A, N};
        const double2 *src = a.buf + blk * E;
        for (int i = threadIdx.x; i < E; i += T) {
            const int f = i / N;
            cp_async16(ad.ptr(f, i - f * N), src + i);
        }
    };
    uint64_t blk = blockIdx.x;
    int cur = 0;
    if (blk < nblk) prefetch(A0, blk);
    fs_cp_commit();
    for (; blk < nblk; blk += gridDim.x) {
        const uint64_t nxt = blk + gridDim.x;
        if (nxt < nblk) prefetch(A0 + (cur ^ 1) * E, nxt);
        fs_cp_commit();
        fs_cp_wait_prev();
        __syncthreads();
        fs_row_block<C, T, NT, true>(a, A0 + cur * E, blk);
        __syncthreads();
        cur ^= 1;
    }
}

// ---------------------------------------------------------------------------------------------
// Column pass: CW adjacent columns (c0 .. c0+CW) of a matrix with row stride M2, column length
// N, column-fastest over the threads (CW * 16 B = 128-B rows per global access):
// [inverse FFT] -> <Q> partials, phase exp(-i gamma q), outer twiddle (three-level) on the
// registers -> [forward FFT -> twiddle w_M^{C k1}] -> global.  As fft_col_kernel.
template <int N>
constexpr int fs_col_stride() { return (N % 2 == 0) ? N + 1 : N; }  // odd: 8 columns, 8 bank groups
template <typename C, int T, int CW, bool INV, bool FWD>
__device__ __forceinline__ void fs_col_block(const FsColArgs &a, double2 *A, int bx, int by, double *red) {
    constexpr int N = C::N, S = C::S;
    constexpr int CS = fs_col_stride<N>();
    static_assert(S >= 2 && C::r(0, 0) == C::r(1, S - 1), "reversed inverse order");
    const FsAddr<0> ad{A, CS};
    const int c0 = bx * CW;
    const uint64_t mat = (uint64_t)by * a.mat_stride;
    const uint64_t M2 = (uint64_t)a.M2;
    const double2 *in = a.in + mat + c0;
    double2 *out = a.out + mat + c0;
    constexpr int OP_EXP = 2, OP_PH = 4, OP_OTW = 64;
    const bool need_q = (a.ops & (OP_EXP | OP_PH)) != 0;
    if (need_q)  // the block's q rows (CW * 8 B) into L2 while the inverse transform runs
        for (int x1 = threadIdx.x; x1 < N; x1 += T)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a.q + (uint64_t)x1 * M2 + c0));

    // middle element set: x1 = j + t*nbm of column c, radix Rm
    constexpr int Rm = C::r(0, 0), nbm = N / Rm, totm = CW * nbm, NBm = (totm + T - 1) / T;
    double2 v[NBm][Rm];
    if constexpr (INV) {
        {  // inverse stage 0: global -> registers -> DFT -> shared memory
            constexpr int R = C::r(1, 0), nb = N / R, tot = CW * nb, NB = (tot + T - 1) / T;
            double2 u[NB][R];
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                const int J = threadIdx.x + b * T;
                if (tot % T == 0 || J < tot) {
                    int c, j;
                    fs_map<true, CW, nb>(J, c, j);
                    const double2 *src = in + (uint64_t)j * M2 + c;
#pragma unroll
                    for (int t = 0; t < R; ++t) u[b][t] = src[(uint64_t)(t * nb) * M2];
                }
            }
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                const int J = threadIdx.x + b * T;
                if (tot % T == 0 || J < tot) dft<R>(u[b], true);
            }
            fs_first_store<C, 1, T, CW, true>(ad, u);
        }
        __syncthreads();
        fs_static_for<S - 2>([&](auto sc) { fs_stage<C, 1, decltype(sc)::value + 1, T, CW, true>(ad, a.tw); });
        fs_last_stage<C, 1, T, CW, true>(ad, a.tw, v);
    } else {
#pragma unroll
        for (int b = 0; b < NBm; ++b) {
            const int J = threadIdx.x + b * T;
            if (totm % T == 0 || J < totm) {
                int c, j;
                fs_map<true, CW, nbm>(J, c, j);
                const double2 *src = in + (uint64_t)j * M2 + c;
#pragma unroll
                for (int t = 0; t < Rm; ++t)
                    v[b][t] = a.init ? make_double2(a.amp0, 0.0) : src[(uint64_t)(t * nbm) * M2];
            }
        }
    }
    // elementwise ops at (c, x1): <Q> partials of the inverse result, then the phase; the
    // three-level outer twiddle w_N^{-xl K}, xl = x1*M2 + c0 + c, K = matrix
    double acc = 0.0, nrm = 0.0;
    if (a.ops) {
#pragma unroll
        for (int b = 0; b < NBm; ++b) {
            const int J = threadIdx.x + b * T;
            if (totm % T == 0 || J < totm) {
                int c, j;
                fs_map<true, CW, nbm>(J, c, j);
                if (need_q) {
                    const double *qp = a.q + (uint64_t)j * M2 + c0 + c;
                    double qv[Rm];
#pragma unroll
                    for (int t = 0; t < Rm; ++t) qv[t] = __ldg(qp + (uint64_t)(t * nbm) * M2);
#pragma unroll
                    for (int t = 0; t < Rm; ++t) {
                        if (a.ops & OP_EXP) {
                            const double pr = v[b][t].x * v[b][t].x + v[b][t].y * v[b][t].y;
                            acc = fma(pr, qv[t], acc);
                            nrm += pr;
                        }
                        if (a.ops & OP_PH) {
                            double sn, cs;
                            sincos(a.gamma * qv[t], &sn, &cs);
                            v[b][t] = make_double2(fma(cs, v[b][t].x, sn * v[b][t].y), fma(cs, v[b][t].y, -sn * v[b][t].x));
                        }
                    }
                }
                if (a.ops & OP_OTW) {
                    const uint64_t K = (uint64_t)(a.mat_off + by);
                    const uint64_t xl0 = (uint64_t)j * M2 + (uint64_t)(c0 + c);
                    double2 w = conjd(fs_big(a.otw_lo, a.otw_hi, a.otw_shift, K * xl0));
                    const double2 st = conjd(fs_big(a.otw_lo, a.otw_hi, a.otw_shift, K * (uint64_t)nbm * M2));
#pragma unroll
                    for (int t = 0; t < Rm; ++t) {
                        v[b][t] = cmul(v[b][t], w);
                        if (t + 1 < Rm) w = cmul(w, st);
                    }
                }
            }
        }
    }
    if constexpr (FWD) {
#pragma unroll
        for (int b = 0; b < NBm; ++b) {
            const int J = threadIdx.x + b * T;
            if (totm % T == 0 || J < totm) dft<Rm>(v[b], false);
        }
        if constexpr (INV) __syncthreads();  // the inverse last stage's reads are done
        fs_first_store<C, 0, T, CW, true>(ad, v);
        __syncthreads();
        fs_static_for<S - 2>([&](auto sc) { fs_stage<C, 0, decltype(sc)::value + 1, T, CW, true>(ad, a.tw); });
        constexpr int R = C::r(0, S - 1), nb = N / R, tot = CW * nb, NB = (tot + T - 1) / T;
        double2 u[NB][R];
        fs_last_stage<C, 0, T, CW, true>(ad, a.tw, u);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int J = threadIdx.x + b * T;
            if (tot % T == 0 || J < tot) {
                int c, j;
                fs_map<true, CW, nb>(J, c, j);
                const uint64_t Cg = (uint64_t)(a.col_off + c0 + c);
                double2 w = fs_big(a.big_lo, a.big_hi, a.big_shift, Cg * (uint64_t)j);
                const double2 st = fs_big(a.big_lo, a.big_hi, a.big_shift, Cg * (uint64_t)nb);
                double2 *dst = out + (uint64_t)j * M2 + c;
#pragma unroll
                for (int t = 0; t < R; ++t) {
                    dst[(uint64_t)(t * nb) * M2] = cmul(u[b][t], w);
                    if (t + 1 < R) w = cmul(w, st);
                }
            }
        }
    } else {
#pragma unroll
        for (int b = 0; b < NBm; ++b) {
            const int J = threadIdx.x + b * T;
            if (totm % T == 0 || J < totm) {
                int c, j;
                fs_map<true, CW, nbm>(J, c, j);
                double2 *dst = out + (uint64_t)j * M2 + c;
#pragma unroll
                for (int t = 0; t < Rm; ++t) dst[(uint64_t)(t * nbm) * M2] = v[b][t];
            }
        }
    }
    if (a.ops & OP_EXP) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            acc += __shfl_xor_sync(0xffffffffu, acc, o);
            nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
        }
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (lane == 0) {
            red[2 * warp] = acc;
            red[2 * warp + 1] = nrm;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double sa = 0.0, sb = 0.0;
            for (int w = 0; w < (T + 31) / 32; ++w) {
                sa += red[2 * w];
                sb += red[2 * w + 1];
            }
            a.partials[2 * bx] = sa;
            a.partials[2 * bx + 1] = sb;
        }
    }
}

template <typename C, int T, int CW, int MINB, bool INV, bool FWD>
__global__ void __launch_bounds__(T, MINB) fs_col_kernel(const FsColArgs a, int nbx, uint64_t nblk) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double red[2 * (T / 32 + 1)];
    fs_col_block<C, T, CW, INV, FWD>(a, reinterpret_cast<double2 *>(smem_raw), blockIdx.x, blockIdx.y, red);
}
// ---------------------------------------------------------------------------------------------
// Ping-pong column pass: the same transforms with out-of-place stages between two shared-memory
// buffers, so a stage needs one barrier and no thread has to hold all of its butterflies at once
// (butterflies in rounds of T): 768 threads on eight-column blocks (two ~100 KB buffers, one CTA
// per SM) at 80 registers and no spills, where the in-place block needs NB butterflies per thread.
template <typename C, int D, int s, int T, int CW, typename Ad, bool CFAST = true>
__device__ __forceinline__ void fs_stage_pp(const Ad &src, const Ad &dst, const double2 *__restrict__ tw) {
    constexpr int N = C::N, R = C::r(D, s), M = C::m(D, s), nb = N / R, tot = CW * nb, OFF = C::off(D, s);
#pragma unroll
    for (int J = threadIdx.x; J < tot; J += T) {
        int c, j;
        fs_map<CFAST, CW, nb>(J, c, j);
        double2 v[R];
#pragma unroll
        for (int t = 0; t < R; ++t) v[t] = *src.ptr(c, j + t * nb);
        const int k = j % M;
#pragma unroll
        for (int t = 1; t < R; ++t) v[t] = cmul(v[t], __ldg(tw + OFF + (t - 1) * M + k));
        dft<R>(v, D != 0);
        const int o = (j - k) * R + k;
#pragma unroll
        for (int t = 0; t < R; ++t) *dst.ptr(c, o + t * M) = v[t];
    }
    __syncthreads();
}

// Ping-pong row pass: fs_row_block's transforms with out-of-place stages between two buffers
// (rows j-fastest, butterflies in rounds of T), so more, lighter threads fit per SM.
template <typename C, int T, int NT, int MINB>
__global__ void __launch_bounds__(T, MINB) fs_rowpp_kernel(const FsRowArgs a, uint64_t nblk) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int N = C::N, S = C::S;
    static_assert(S >= 2 && C::r(0, S - 1) == C::r(1, 0), "reversed inverse order");
    double2 *A0 = reinterpret_cast<double2 *>(smem_raw);
    using Ad = FsAddr<C::swz()>;
    const Ad b0{A0, N}, b1{A0 + NT * N, N};
    const uint64_t blk = blockIdx.x;
    double2 *rows = a.buf + blk * NT * N;
    const int grow0 = a.row_off + (int)blk * NT;
    {  // forward stage 0: global -> DFT -> b0
        constexpr int R = C::r(0, 0), nb = N / R, tot = NT * nb;
#pragma unroll
        for (int J = threadIdx.x; J < tot; J += T) {
            int f, j;
            fs_map<false, NT, nb>(J, f, j);
            const double2 *src = rows + f * N + j;
            double2 v[R];
#pragma unroll
            for (int t = 0; t < R; ++t) v[t] = src[t * nb];
            dft<R>(v, false);
#pragma unroll
            for (int t = 0; t < R; ++t) *b0.ptr(f, j * R + t) = v[t];
        }
        __syncthreads();
    }
    const Ad *bufs[2] = {&b0, &b1};
    int cur = 0;
    fs_static_for<S - 2>([&](auto sc) {
        fs_stage_pp<C, 0, decltype(sc)::value + 1, T, NT, Ad, false>(*bufs[cur], *bufs[cur ^ 1], a.tw);
        cur ^= 1;
    });
    {  // forward last stage -> spectrum -> inverse stage 0
        constexpr int R = C::r(0, S - 1), M = C::m(0, S - 1), nb = N / R, tot = NT * nb, OFF = C::off(0, S - 1);
        const Ad &src = *bufs[cur], &dst = *bufs[cur ^ 1];
#pragma unroll
        for (int J = threadIdx.x; J < tot; J += T) {
            int f, j;
            fs_map<false, NT, nb>(J, f, j);
            double2 v[R];
#pragma unroll
            for (int t = 0; t < R; ++t) v[t] = *src.ptr(f, j + t * nb);
#pragma unroll
            for (int t = 1; t < R; ++t) v[t] = cmul(v[t], __ldg(a.tw + OFF + (t - 1) * M + j));
            dft<R>(v, false);
            if (a.spec == 0) {
                if (j == 0 && grow0 + f == 0) v[0] = cmul(v[0], a.e0_over_ec);
            } else {
                const double *lam = a.lam_perm + (uint64_t)(grow0 + f) * N + j;
#pragma unroll
                for (int t = 0; t < R; ++t) {
                    double sn, cs;
                    sincos(-a.beta * __ldg(lam + t * nb), &sn, &cs);
                    v[t] = cmul(v[t], make_double2(cs * a.scale, sn * a.scale));
                }
            }
            dft<R>(v, true);
#pragma unroll
            for (int t = 0; t < R; ++t) *dst.ptr(f, j * R + t) = v[t];
        }
        __syncthreads();
        cur ^= 1;
    }
    fs_static_for<S - 2>([&](auto sc) {
        fs_stage_pp<C, 1, decltype(sc)::value + 1, T, NT, Ad, false>(*bufs[cur], *bufs[cur ^ 1], a.tw);
        cur ^= 1;
    });
    {  // inverse last stage -> final twiddle -> global
        constexpr int R = C::r(1, S - 1), M = C::m(1, S - 1), nb = N / R, tot = NT * nb, OFF = C::off(1, S - 1);
        const Ad &src = *bufs[cur];
#pragma unroll
        for (int J = threadIdx.x; J < tot; J += T) {
            int f, j;
            fs_map<false, NT, nb>(J, f, j);
            double2 v[R];
#pragma unroll
            for (int t = 0; t < R; ++t) v[t] = *src.ptr(f, j + t * nb);
#pragma unroll
            for (int t = 1; t < R; ++t) v[t] = cmul(v[t], __ldg(a.tw + OFF + (t - 1) * M + j));
            dft<R>(v, true);
            const int kr = grow0 + f;
            const uint64_t K = (uint64_t)(a.row_mod ? kr % a.row_mod : kr);
            double2 w = conjd(fs_big(a.big_lo, a.big_hi, a.big_shift, K * (uint64_t)j));
            const double2 st = conjd(fs_big(a.big_lo, a.big_hi, a.big_shift, K * (uint64_t)nb));
            if (a.spec == 0) w = cmul(w, a.ec);
            double2 *dd = rows + f * N + j;
#pragma unroll
            for (int t = 0; t < R; ++t) {
                dd[t * nb] = cmul(v[t], w);
                if (t + 1 < R) w = cmul(w, st);
            }
        }
    }
}

template <typename C, int T, int CW, int MINB, bool INV, bool FWD>
__global__ void __launch_bounds__(T, MINB) fs_colpp_kernel(const FsColArgs a, int nbx, uint64_t nblk) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double red[2 * (T / 32 + 1)];
    constexpr int N = C::N, S = C::S, CS = fs_col_stride<N>();
    static_assert(S >= 2 && C::r(0, 0) == C::r(1, S - 1), "reversed inverse order");
    double2 *A0 = reinterpret_cast<double2 *>(smem_raw);
    const FsAddr<0> b0{A0, CS}, b1{A0 + CW * CS, CS};
    const int c0 = (int)blockIdx.x * CW;
    const uint64_t mat = (uint64_t)blockIdx.y * a.mat_stride;
    const uint64_t M2 = (uint64_t)a.M2;
    const double2 *in = a.in + mat + c0;
    double2 *out = a.out + mat + c0;
    constexpr int OP_EXP = 2, OP_PH = 4, OP_OTW = 64;
    const bool need_q = (a.ops & (OP_EXP | OP_PH)) != 0;
    if (need_q)
        for (int x1 = threadIdx.x; x1 < N; x1 += T)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a.q + (uint64_t)x1 * M2 + c0));
    double acc = 0.0, nrm = 0.0;
    // ops on one butterfly's middle elements (c, x1 = j + t*nbm)
    constexpr int Rm = C::r(0, 0), nbm = N / Rm, totm = CW * nbm;
    auto ops = [&](double2 (&v)[Rm], int c, int j) {
        if (need_q) {
            const double *qp = a.q + (uint64_t)j * M2 + c0 + c;
            double qv[Rm];
#pragma unroll
            for (int t = 0; t < Rm; ++t) qv[t] = __ldg(qp + (uint64_t)(t * nbm) * M2);
#pragma unroll
            for (int t = 0; t < Rm; ++t) {
                if (a.ops & OP_EXP) {
                    const double pr = v[t].x * v[t].x + v[t].y * v[t].y;
                    acc = fma(pr, qv[t], acc);
                    nrm += pr;
                }
                if (a.ops & OP_PH) {
                    double sn, cs;
                    sincos(a.gamma * qv[t], &sn, &cs);
                    v[t] = make_double2(fma(cs, v[t].x, sn * v[t].y), fma(cs, v[t].y, -sn * v[t].x));
                }
            }
        }
        if (a.ops & OP_OTW) {
            const uint64_t K = (uint64_t)(a.mat_off + (int)blockIdx.y);
            const uint64_t xl0 = (uint64_t)j * M2 + (uint64_t)(c0 + c);
            double2 w = conjd(fs_big(a.otw_lo, a.otw_hi, a.otw_shift, K * xl0));
            const double2 st = conjd(fs_big(a.otw_lo, a.otw_hi, a.otw_shift, K * (uint64_t)nbm * M2));
#pragma unroll
            for (int t = 0; t < Rm; ++t) {
                v[t] = cmul(v[t], w);
                if (t + 1 < Rm) w = cmul(w, st);
            }
        }
    };
    // after the middle: forward stage 0 to buffer `dst`, or the result straight to global
    auto middle_out = [&](double2 (&v)[Rm], int c, int j, const FsAddr<0> &dst) {
        if constexpr (FWD) {
            dft<Rm>(v, false);
#pragma unroll
            for (int t = 0; t < Rm; ++t) *dst.ptr(c, j * Rm + t) = v[t];
        } else {
            double2 *o = out + (uint64_t)j * M2 + c;
#pragma unroll
            for (int t = 0; t < Rm; ++t) o[(uint64_t)(t * nbm) * M2] = v[t];
        }
    };
    // the forward transform's stages after stage 0 (which wrote buffer `first`) and its store
    auto forward_rest = [&](bool first_is_b0) {
        const FsAddr<0> *bufs[2] = {first_is_b0 ? &b0 : &b1, first_is_b0 ? &b1 : &b0};
        int cur = 0;
        fs_static_for<S - 2>([&](auto sc) {
            fs_stage_pp<C, 0, decltype(sc)::value + 1, T, CW>(*bufs[cur], *bufs[cur ^ 1], a.tw);
            cur ^= 1;
        });
        constexpr int R = C::r(0, S - 1), M = C::m(0, S - 1), nb = N / R, tot = CW * nb, OFF = C::off(0, S - 1);
        const FsAddr<0> &src = *bufs[cur];
#pragma unroll
        for (int J = threadIdx.x; J < tot; J += T) {
            int c, j;
            fs_map<true, CW, nb>(J, c, j);
            double2 v[R];
#pragma unroll
            for (int t = 0; t < R; ++t) v[t] = *src.ptr(c, j + t * nb);
#pragma unroll
            for (int t = 1; t < R; ++t) v[t] = cmul(v[t], __ldg(a.tw + OFF + (t - 1) * M + j));
            dft<R>(v, false);
            const uint64_t Cg = (uint64_t)(a.col_off + c0 + c);
            double2 w = fs_big(a.big_lo, a.big_hi, a.big_shift, Cg * (uint64_t)j);
            const double2 st = fs_big(a.big_lo, a.big_hi, a.big_shift, Cg * (uint64_t)nb);
            double2 *dd = out + (uint64_t)j * M2 + c;
#pragma unroll
            for (int t = 0; t < R; ++t) {
                dd[(uint64_t)(t * nb) * M2] = cmul(v[t], w);
                if (t + 1 < R) w = cmul(w, st);
            }
        }
    };
    if constexpr (INV) {
        {  // inverse stage 0 from global into b0
            constexpr int R = C::r(1, 0), nb = N / R, tot = CW * nb;
#pragma unroll
            for (int J = threadIdx.x; J < tot; J += T) {
                int c, j;
                fs_map<true, CW, nb>(J, c, j);
                const double2 *src = in + (uint64_t)j * M2 + c;
                double2 v[R];
#pragma unroll
                for (int t = 0; t < R; ++t) v[t] = src[(uint64_t)(t * nb) * M2];
                dft<R>(v, true);
#pragma unroll
                for (int t = 0; t < R; ++t) *b0.ptr(c, j * R + t) = v[t];
            }
            __syncthreads();
        }
        const FsAddr<0> *bufs[2] = {&b0, &b1};
        int cur = 0;
        fs_static_for<S - 2>([&](auto sc) {
            fs_stage_pp<C, 1, decltype(sc)::value + 1, T, CW>(*bufs[cur], *bufs[cur ^ 1], a.tw);
            cur ^= 1;
        });
        {  // inverse last stage -> ops -> forward stage 0 (or global)
            constexpr int R = C::r(1, S - 1), M = C::m(1, S - 1), nb = N / R, tot = CW * nb, OFF = C::off(1, S - 1);
            static_assert(R == Rm && nb == nbm, "boundary");
            const FsAddr<0> &src = *bufs[cur], &dst = *bufs[cur ^ 1];
#pragma unroll
            for (int J = threadIdx.x; J < tot; J += T) {
                int c, j;
                fs_map<true, CW, nb>(J, c, j);
                double2 v[R];
#pragma unroll
                for (int t = 0; t < R; ++t) v[t] = *src.ptr(c, j + t * nb);
#pragma unroll
                for (int t = 1; t < R; ++t) v[t] = cmul(v[t], __ldg(a.tw + OFF + (t - 1) * M + j));
                dft<R>(v, true);
                if (a.ops) ops(v, c, j);
                middle_out(v, c, j, dst);
            }
            if constexpr (FWD) {
                __syncthreads();
                forward_rest(cur == 1);
            }
        }
    } else {
#pragma unroll
        for (int J = threadIdx.x; J < totm; J += T) {
            int c, j;
            fs_map<true, CW, nbm>(J, c, j);
            const double2 *src = in + (uint64_t)j * M2 + c;
            double2 v[Rm];
#pragma unroll
            for (int t = 0; t < Rm; ++t) v[t] = a.init ? make_double2(a.amp0, 0.0) : src[(uint64_t)(t * nbm) * M2];
            if (a.ops) ops(v, c, j);
            middle_out(v, c, j, b0);
        }
        if constexpr (FWD) {
            __syncthreads();
            forward_rest(true);
        }
    }
    if (a.ops & OP_EXP) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            acc += __shfl_xor_sync(0xffffffffu, acc, o);
            nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
        }
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (lane == 0) {
            red[2 * warp] = acc;
            red[2 * warp + 1] = nrm;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double sa = 0.0, sb = 0.0;
            for (int w = 0; w < (T + 31) / 32; ++w) {
                sa += red[2 * w];
                sb += red[2 * w + 1];
            }
            a.partials[2 * blockIdx.x] = sa;
            a.partials[2 * blockIdx.x + 1] = sb;
        }
    }
}

// ---------------------------------------------------------------------------------------------
// compiled codelets and their launch shapes (several per length for measurement: QVA_FS_ROWV /
// QVA_FS_COLV select the variant index, default 0)
using FsRowFn = void (*)(FsRowArgs, uint64_t);
using FsColFn = void (*)(FsColArgs, int, uint64_t);

struct FsRowEntry {
    int n, threads, rows, pipe;  // pipe: 1 persistent pipelined, 2 ping-pong (two block buffers each)
    FsRowFn fn;
    Arr8 rad;                    // forward radix order (the stage tables follow it)
};
struct FsColEntry {
    int n, threads, cw, pipe;  // pipe: 0 in place (one block buffer), 2 ping-pong (two buffers)
    FsColFn inv_fwd, fwd, inv;
    Arr8 rad;
};

using C768 = FsC<16, 16, 3>;
using C4320 = FsC<9, 3, 16, 10>;
using C770 = FsC<7, 11, 10>;
using C810 = FsC<10, 9, 9>;
using C840 = FsC<8, 15, 7>;

#define QVA_FS_ROW(C, T, NT, MB) {C::N, T, NT, 0, fs_row_kernel<C, T, NT, MB>, C::F}
#define QVA_FS_ROWP(C, T, NT, MB) {C::N, T, NT, 1, fs_row_pipe_kernel<C, T, NT, MB>, C::F}
#define QVA_FS_ROWPP(C, T, NT, MB) {C::N, T, NT, 2, fs_rowpp_kernel<C, T, NT, MB>, C::F}
// index 0 of each length is the default (measured on one B200, tools/ab_fs.sh, p=4 evolutions
// with the grouped inner passes and 896-thread columns): 12! 768-point rows ping-pong 256 threads x
// 4 rows (two CTAs per SM) 90.7 ms, pipelined persistent 192 x 4 91.4, ping-pong 384 x 4 91.8,
// pipelined 96 x 2 92.1, ping-pong 192 x 2 92.4, one-shot 96 x 2 93.7 ms; cfg3 4320-point rows
// one-shot two CTAs per SM 0.609 ms, ping-pong 512 / 448 threads 0.622 / 0.652, one-shot one CTA
// per SM 0.72, pipelined 0.97 ms
const FsRowEntry kFsRows[] = {
    QVA_FS_ROWPP(C768, 256, 4, 2),
    QVA_FS_ROWP(C768, 192, 4, 2),
    QVA_FS_ROWPP(C768, 384, 4, 2),
    QVA_FS_ROWP(C768, 96, 2, 4),
    QVA_FS_ROW(C768, 192, 4, 3),
    QVA_FS_ROW(C4320, 288, 1, 2),
    QVA_FS_ROWPP(C4320, 512, 1, 1),
    QVA_FS_ROW(C4320, 288, 1, 1),
};
#undef QVA_FS_ROW
#undef QVA_FS_ROWP
#undef QVA_FS_ROWPP
#define QVA_FS_COL(K, C, T, CW, MB, P)                                                      \
    {C::N, T, CW, P, K<C, T, CW, MB, true, true>, K<C, T, CW, MB, false, true>, K<C, T, CW, MB, true, false>, C::F}
// column codelets (index 0 = default; measured on one B200, tools/ab_fs.sh, p=4 evolutions with
// the grouped three-level inner passes): 770 / 810 (12!): ping-pong 896 threads x 8 columns
// 92.1 ms, 1024 x 8 92.4 ms (small spills), 768 x 8 95.6 ms, 512 x 8 102.0 ms, one-shot in place
// 640 / 512 x 8 98.4 ms, ping-pong four wide 384 x 4 111 ms (a pipelined persistent form, removed,
// spilled in its block loop and doubled the DRAM write traffic: 162-205 ms); 840 (cfg3): ping-pong
// 896 x 8 0.609 ms, 1024 x 8 0.619, one-shot 256 x 4 two CTAs per SM 0.622, 480 x 8 0.653.  More
// warps per SM win as long as ptxas keeps the butterflies in registers.  Other radix orders of the
// same lengths (each entry carries its order; the stage tables follow it): 770 as 10*11*7 / 11*7*10
// with 810 as 9*10*9 / 9*9*10: 92.1 / 93.0 ms against 90.9 ms for 7*11*10 with 10*9*9.
const FsColEntry kFsCols[] = {
    QVA_FS_COL(fs_colpp_kernel, C770, 896, 8, 1, 2),
    QVA_FS_COL(fs_colpp_kernel, C770, 1024, 8, 1, 2),
    QVA_FS_COL(fs_colpp_kernel, C770, 768, 8, 1, 2),
    QVA_FS_COL(fs_col_kernel, C770, 640, 8, 1, 0),
    QVA_FS_COL(fs_colpp_kernel, C810, 896, 8, 1, 2),
    QVA_FS_COL(fs_colpp_kernel, C810, 1024, 8, 1, 2),
    QVA_FS_COL(fs_colpp_kernel, C810, 768, 8, 1, 2),
    QVA_FS_COL(fs_col_kernel, C810, 512, 8, 1, 0),
    QVA_FS_COL(fs_colpp_kernel, C840, 896, 8, 1, 2),
    QVA_FS_COL(fs_colpp_kernel, C840, 1024, 8, 1, 2),
    QVA_FS_COL(fs_col_kernel, C840, 256, 4, 2, 0),
    QVA_FS_COL(fs_col_kernel, C840, 480, 8, 1, 0),
};
#undef QVA_FS_COL

int fs_env(const char *name) {
    const char *e = getenv(name);
    return e ? atoi(e) : 0;
}
const FsRowEntry *fs_row_entry(int n) {
    static const int v = fs_env("QVA_FS_ROWV");
    int k = 0;
    for (const auto &e : kFsRows)
        if (e.n == n && k++ == v) return &e;
    for (const auto &e : kFsRows)
        if (e.n == n) return &e;
    return nullptr;
}
const FsColEntry *fs_col_entry(int n) {
    static const int v = fs_env("QVA_FS_COLV");
    int k = 0;
    for (const auto &e : kFsCols)
        if (e.n == n && k++ == v) return &e;
    for (const auto &e : kFsCols)
        if (e.n == n) return &e;
    return nullptr;
}
size_t fs_col_smem(const FsColEntry &e) {
    return (size_t)(e.pipe ? 2 : 1) * e.cw * ((e.n % 2 == 0) ? e.n + 1 : e.n) * sizeof(double2);
}
size_t fs_row_smem(const FsRowEntry &e) { return (size_t)(e.pipe ? 2 : 1) * e.rows * e.n * sizeof(double2); }

DeviceOnce g_fs_attr;

cudaError_t fs_set_attrs() {
    return once_per_device(g_fs_attr, [] {
        for (const auto &e : kFsRows) {
            cudaError_t r = cudaFuncSetAttribute(e.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fs_row_smem(e));
            if (r != cudaSuccess) return r;
        }
        for (const auto &e : kFsCols) {
            for (FsColFn f : {e.inv_fwd, e.fwd, e.inv}) {
                cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fs_col_smem(e));
                if (r != cudaSuccess) return r;
            }
        }
        return cudaSuccess;
    });
}

}  // namespace

bool fs_row_available(int n) {
    const char *e = getenv("QVA_FFT_FS");
    return (!e || atoi(e) != 0) && fs_row_entry(n) != nullptr;
}
bool fs_col_available(int n) {
    const char *e = getenv("QVA_FFT_FS");
    return (!e || atoi(e) != 0) && fs_col_entry(n) != nullptr;
}
int fs_row_block(int n) {
    const FsRowEntry *e = fs_row_entry(n);
    return e ? e->rows : 0;
}
int fs_col_width(int n) {
    const FsColEntry *e = fs_col_entry(n);
    return e ? e->cw : 0;
}

bool fs_stage_tables(int n, bool col, std::vector<double2> &tab) {
    const FsRowEntry *re = col ? nullptr : fs_row_entry(n);
    const FsColEntry *ce = col ? fs_col_entry(n) : nullptr;
    if (!re && !ce) return false;
    const int *rad = re ? re->rad.v : ce->rad.v;
    int S = 0;
    while (S < 8 && rad[S]) ++S;
    tab.clear();
    const long double kPi = 3.141592653589793238462643383279502884L;
    for (int d = 0; d < 2; ++d) {
        int m = 1;
        for (int s = 0; s < S; ++s) {
            const int R = d ? rad[S - 1 - s] : rad[s];
            if (s >= 1)
                for (int t = 1; t < R; ++t)
                    for (int k = 0; k < m; ++k) {
                        const long double ang = (d ? 2.0L : -2.0L) * kPi * (long double)(t * k) / (long double)(m * R);
                        tab.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
                    }
            m *= R;
        }
    }
    return true;
}

// persistent grid of the pipelined kernels: resident CTAs per SM x SMs
template <typename Fn>
static unsigned fs_pipe_grid(Fn f, int threads, size_t smem, uint64_t nblk) {
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, f, threads, smem) != cudaSuccess || per < 1) per = 1;
    return (unsigned)std::min<uint64_t>(nblk, (uint64_t)per * (uint64_t)num_sms());
}

cudaError_t fs_row_launch(int n, const FsRowArgs &a, uint64_t n_rows, cudaStream_t s) {
    const FsRowEntry *e = fs_row_entry(n);
    if (!e || n_rows % e->rows) return cudaErrorInvalidValue;
    cudaError_t r = fs_set_attrs();
    if (r != cudaSuccess) return r;
    if (n_rows == 0) return cudaSuccess;
    const uint64_t nblk = n_rows / e->rows;
    const size_t smem = fs_row_smem(*e);
    const unsigned grid = e->pipe == 1 ? fs_pipe_grid(e->fn, e->threads, smem, nblk) : (unsigned)nblk;
    e->fn<<<grid, e->threads, smem, s>>>(a, nblk);
    return cudaGetLastError();
}

cudaError_t fs_col_launch(int n, const FsColArgs &a, int cols, int nmat, bool inv, bool fwd, cudaStream_t s) {
    const FsColEntry *e = fs_col_entry(n);
    if (!e || cols % e->cw || (!inv && !fwd)) return cudaErrorInvalidValue;
    cudaError_t r = fs_set_attrs();
    if (r != cudaSuccess) return r;
    if (cols == 0 || nmat == 0) return cudaSuccess;
    FsColFn f = inv ? (fwd ? e->inv_fwd : e->inv) : e->fwd;
    const int nbx = cols / e->cw;
    const uint64_t nblk = (uint64_t)nbx * nmat;
    const size_t smem = fs_col_smem(*e);
    f<<<dim3(nbx, nmat), e->threads, smem, s>>>(a, nbx, nblk);
    return cudaGetLastError();
}

}  // namespace qva
