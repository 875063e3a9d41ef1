// kernels_fft.cu -- circulant (QWOA) mixer U(beta) = F^-1 diag(exp(-i beta lambda)) F
// (Sec. 3; sign reading R3, spectrum indexing R4) by hand-written fp64
// mixed-radix FFTs on sm_100a.
//
// Layout: N = N1 * N2 four-step decomposition, index x = x1*N2 + x2.
//   COL pass  (one CTA per `cw` adjacent columns x2): [inverse length-N1 FFTs of the previous
//             layer] -> [phase exp(-i gamma q)] -> [forward length-N1 FFTs, twiddle w_N^{x2 k1}]
//   ROW pass  (one CTA per row k1): forward length-N2 FFT -> * exp(-i beta lambda)/N ->
//             inverse length-N2 FFT -> twiddle w_N^{-x2 k1}
// so one layer costs two passes over the state (plus one final inverse COL pass) and the
// spectrum lives in "transposed" order: position k1*N2 + k2 holds bin k1 + N1*k2.
// Each length-n sub-FFT is a Stockham autosort FFT in shared memory with radix 2/3/4/5/7/8/11/13
// stages (ping-pong buffers), twiddles read from small precomputed tables.
// N <= 4096: the whole p-layer evolution runs in one CTA ("whole" kernel).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "qva_internal.h"

namespace qva {

constexpr int kMaxSub = 4096;     // largest in-CTA sub-FFT
constexpr int kMaxStages = 24;
constexpr int kFftThreads = 256;
constexpr int kWholeThreads = 512;

struct SubFft {
    int n = 1;
    int ns = 0;
    int r[kMaxStages];
    int m[kMaxStages];
    int twoff[kMaxStages];
};

struct FftPlan {
    uint64_t N = 0;
    int device = 0;
    bool whole = false;
    int N1 = 1, N2 = 1;
    int cw = 2;
    SubFft col, row;
    double2 *d_tw = nullptr;     // stage twiddle tables (col then row)
    double2 *d_big_lo = nullptr, *d_big_hi = nullptr;
    int big_shift = 11;          // B = 2^big_shift
    double *partials = nullptr;
    int n_partials = 0;
};

namespace {

// roots of unity exp(-2 pi i j / r) for r = 2..16, offset r*(r-1)/2 - 1
__constant__ double2 c_roots[160];

__host__ __device__ constexpr int root_off(int r) { return r * (r - 1) / 2 - 1; }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 conj_if(double2 a, bool inv) { return inv ? make_double2(a.x, -a.y) : a; }

template <int R>
__device__ __forceinline__ void dft(double2 (&a)[R], bool inv) {
    if constexpr (R == 2) {
        double2 t = a[0];
        a[0] = cadd(t, a[1]);
        a[1] = csub(t, a[1]);
    } else if constexpr (R == 4) {
        double2 s02 = cadd(a[0], a[2]), d02 = csub(a[0], a[2]);
        double2 s13 = cadd(a[1], a[3]), d13 = csub(a[1], a[3]);
        // w = -i (forward) or +i (inverse) times d13
        double2 wd = inv ? make_double2(-d13.y, d13.x) : make_double2(d13.y, -d13.x);
        a[0] = cadd(s02, s13);
        a[2] = csub(s02, s13);
        a[1] = cadd(d02, wd);
        a[3] = csub(d02, wd);
    } else {
        double2 y[R];
#pragma unroll
        for (int t = 0; t < R; ++t) {
            double2 acc = a[0];
#pragma unroll
            for (int u = 1; u < R; ++u) {
                double2 w = conj_if(c_roots[root_off(R) + (t * u) % R], inv);
                acc = cadd(acc, cmul(a[u], w));
            }
            y[t] = acc;
        }
#pragma unroll
        for (int t = 0; t < R; ++t) a[t] = y[t];
    }
}

// One Stockham radix-R stage over `count` independent length-n transforms stored contiguously.
template <int R>
__device__ __forceinline__ void fft_stage(const double2 *__restrict__ in, double2 *__restrict__ out, int n, int count,
                                          int m, const double2 *__restrict__ tw, bool inv) {
    const int nb = n / R;
    const int total = nb * count;
    for (int J = threadIdx.x; J < total; J += blockDim.x) {
        int f = J / nb;
        int j = J - f * nb;
        const double2 *x = in + f * n;
        double2 *y = out + f * n;
        int k = j % m;
        double2 a[R];
#pragma unroll
        for (int t = 0; t < R; ++t) a[t] = x[j + t * nb];
        if (m > 1) {
#pragma unroll
            for (int t = 1; t < R; ++t) a[t] = cmul(a[t], conj_if(__ldg(tw + t * k), inv));
        }
        dft<R>(a, inv);
        int o = (j - k) * R + k;
#pragma unroll
        for (int t = 0; t < R; ++t) y[o + t * m] = a[t];
    }
}

// runs all stages; data starts in A; returns the buffer holding the result
__device__ double2 *run_fft(double2 *A, double2 *B, const SubFft &sf, const double2 *tw, int count, bool inv) {
    double2 *src = A, *dst = B;
    for (int s = 0; s < sf.ns; ++s) {
        const double2 *t = tw + sf.twoff[s];
        switch (sf.r[s]) {
            case 2: fft_stage<2>(src, dst, sf.n, count, sf.m[s], t, inv); break;
            case 3: fft_stage<3>(src, dst, sf.n, count, sf.m[s], t, inv); break;
            case 4: fft_stage<4>(src, dst, sf.n, count, sf.m[s], t, inv); break;
            case 5: fft_stage<5>(src, dst, sf.n, count, sf.m[s], t, inv); break;
            case 7: fft_stage<7>(src, dst, sf.n, count, sf.m[s], t, inv); break;
            case 8: fft_stage<8>(src, dst, sf.n, count, sf.m[s], t, inv); break;
            case 11: fft_stage<11>(src, dst, sf.n, count, sf.m[s], t, inv); break;
            case 13: fft_stage<13>(src, dst, sf.n, count, sf.m[s], t, inv); break;
            default: break;
        }
        __syncthreads();
        double2 *tmp = src;
        src = dst;
        dst = tmp;
    }
    return src;
}

__device__ __forceinline__ double2 big_twiddle(const double2 *lo, const double2 *hi, int shift, uint64_t r, bool inv) {
    uint64_t mask = (1ull << shift) - 1;
    double2 w = cmul(__ldg(hi + (r >> shift)), __ldg(lo + (r & mask)));
    return conj_if(w, inv);
}

__device__ __forceinline__ double2 phase_mul(double2 a, double qv, double gamma) {
    double s, c;
    sincos(gamma * qv, &s, &c);
    return make_double2(fma(c, a.x, s * a.y), fma(c, a.y, -s * a.x));
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

struct ColArgs {
    double2 *psi;
    const double *q;
    int N1, N2, cw;
    int init, do_inv, do_phase, do_fwd, do_expect;
    double amp0, gamma;
    const double2 *tw;
    const double2 *big_lo, *big_hi;
    int big_shift;
    double *partials;
    SubFft sf;
};

__global__ void __launch_bounds__(kFftThreads) fft_col_kernel(const ColArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double red[2 * (kFftThreads / 32)];
    const int N1 = a.N1, N2 = a.N2;
    const int c0 = blockIdx.x * a.cw;
    const int cwv = min(a.cw, N2 - c0);
    double2 *A = reinterpret_cast<double2 *>(smem_raw);
    double2 *B = A + a.cw * N1;
    const int tot = N1 * cwv;
    for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
        int x1 = idx / cwv, c = idx - x1 * cwv;
        A[c * N1 + x1] = a.init ? make_double2(a.amp0, 0.0) : a.psi[(uint64_t)x1 * N2 + c0 + c];
    }
    __syncthreads();
    double2 *cur = A, *oth = B;
    if (a.do_inv) {
        cur = run_fft(A, B, a.sf, a.tw, cwv, true);
        oth = (cur == A) ? B : A;
    }
    if (a.do_phase || a.do_expect) {
        double acc = 0.0, nrm = 0.0;
        for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
            int c = idx / N1, x1 = idx - c * N1;
            uint64_t g = (uint64_t)x1 * N2 + c0 + c;
            double2 v = cur[idx];
            if (a.do_expect) {
                double pr = v.x * v.x + v.y * v.y;
                acc = fma(pr, __ldg(a.q + g), acc);
                nrm += pr;
            }
            if (a.do_phase) cur[idx] = phase_mul(v, __ldg(a.q + g), a.gamma);
        }
        if (a.do_expect) {
            block_reduce2(acc, nrm, red);
            if (threadIdx.x == 0) {
                a.partials[2 * blockIdx.x] = acc;
                a.partials[2 * blockIdx.x + 1] = nrm;
            }
        }
        __syncthreads();
    }
    if (a.do_fwd) {
        double2 *res = run_fft(cur, oth, a.sf, a.tw, cwv, false);
        cur = res;
        for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
            int c = idx / N1, k1 = idx - c * N1;
            uint64_t r = ((uint64_t)(c0 + c) * (uint64_t)k1) % ((uint64_t)N1 * N2);
            cur[idx] = cmul(cur[idx], big_twiddle(a.big_lo, a.big_hi, a.big_shift, r, false));
        }
        __syncthreads();
    }
    for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
        int x1 = idx / cwv, c = idx - x1 * cwv;
        a.psi[(uint64_t)x1 * N2 + c0 + c] = cur[c * N1 + x1];
    }
}

struct RowArgs {
    double2 *psi;
    int N1, N2;
    const double *lambda_perm;  // nullptr -> constant spectrum
    double2 e0, ec;             // exp(-i beta lam0)/N, exp(-i beta c)/N
    double beta, invN;
    const double2 *tw;
    const double2 *big_lo, *big_hi;
    int big_shift;
    SubFft sf;
};

__global__ void __launch_bounds__(kFftThreads) fft_row_kernel(const RowArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N1 = a.N1, N2 = a.N2;
    const int k1 = blockIdx.x;
    double2 *A = reinterpret_cast<double2 *>(smem_raw);
    double2 *B = A + N2;
    double2 *row = a.psi + (uint64_t)k1 * N2;
    for (int i = threadIdx.x; i < N2; i += blockDim.x) A[i] = row[i];
    __syncthreads();
    double2 *cur = run_fft(A, B, a.sf, a.tw, 1, false);
    double2 *oth = (cur == A) ? B : A;
    for (int k2 = threadIdx.x; k2 < N2; k2 += blockDim.x) {
        double2 e;
        if (a.lambda_perm) {
            double s, c;
            sincos(-a.beta * a.lambda_perm[(uint64_t)k1 * N2 + k2], &s, &c);
            e = make_double2(c * a.invN, s * a.invN);
        } else {
            e = (k1 == 0 && k2 == 0) ? a.e0 : a.ec;
        }
        cur[k2] = cmul(cur[k2], e);
    }
    __syncthreads();
    cur = run_fft(cur, oth, a.sf, a.tw, 1, true);
    for (int x2 = threadIdx.x; x2 < N2; x2 += blockDim.x) {
        uint64_t r = ((uint64_t)x2 * (uint64_t)k1) % ((uint64_t)N1 * N2);
        row[x2] = cmul(cur[x2], big_twiddle(a.big_lo, a.big_hi, a.big_shift, r, true));
    }
}

// whole evolution of an N <= 4096 state in one CTA
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

__global__ void __launch_bounds__(kWholeThreads) fft_whole_kernel(const WholeArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double red[2 * (kWholeThreads / 32)];
    const int N = a.sf.n;
    double2 *A = reinterpret_cast<double2 *>(smem_raw);
    double2 *B = A + N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) A[i] = a.init ? make_double2(a.amp0, 0.0) : a.psi[i];
    __syncthreads();
    double2 *cur = A, *oth = B;
    const int layers = a.mode == 0 ? a.p : 1;
    for (int k = 0; k < layers; ++k) {
        double beta;
        if (a.mode == 0) {
            double gamma = a.theta[2 * k];
            beta = a.theta[2 * k + 1];
            for (int i = threadIdx.x; i < N; i += blockDim.x) cur[i] = phase_mul(cur[i], a.q[i], gamma);
            __syncthreads();
        } else {
            beta = a.theta[0];
        }
        cur = run_fft(cur, oth, a.sf, a.tw, 1, false);
        oth = (cur == A) ? B : A;
        for (int j = threadIdx.x; j < N; j += blockDim.x) {
            double lam = a.lambda_perm ? a.lambda_perm[j] : (j == 0 ? a.lam0 : a.lamc);
            double s, c;
            sincos(-beta * lam, &s, &c);
            cur[j] = cmul(cur[j], make_double2(c * a.invN, s * a.invN));
        }
        __syncthreads();
        cur = run_fft(cur, oth, a.sf, a.tw, 1, true);
        oth = (cur == A) ? B : A;
    }
    double acc = 0.0, nrm = 0.0;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        double2 v = cur[i];
        a.psi[i] = v;
        if (a.do_expect) {
            double pr = v.x * v.x + v.y * v.y;
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

// ------------------------------------------------------------------------------------------
// host-side planning
// ------------------------------------------------------------------------------------------
bool factor_radices(int n, std::vector<int> &rs) {
    rs.clear();
    int x = n;
    while (x % 8 == 0) { rs.push_back(8); x /= 8; }
    while (x % 4 == 0) { rs.push_back(4); x /= 4; }
    while (x % 2 == 0) { rs.push_back(2); x /= 2; }
    for (int p : {3, 5, 7, 11, 13})
        while (x % p == 0) { rs.push_back(p); x /= p; }
    return x == 1;
}

bool make_sub(int n, SubFft &sf, std::vector<double2> &tw) {
    std::vector<int> rs;
    if (n < 1 || n > kMaxSub || !factor_radices(n, rs) || (int)rs.size() > kMaxStages) return false;
    sf.n = n;
    sf.ns = (int)rs.size();
    int m = 1;
    for (int s = 0; s < sf.ns; ++s) {
        sf.r[s] = rs[s];
        sf.m[s] = m;
        int L = m * rs[s];
        sf.twoff[s] = (int)tw.size();
        for (int j = 0; j < L; ++j) {
            long double ang = -2.0L * 3.141592653589793238462643383279502884L * (long double)j / (long double)L;
            tw.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
        }
        m = L;
    }
    return true;
}

bool smooth(uint64_t n) {
    for (uint64_t p : {2, 3, 5, 7, 11, 13})
        while (n % p == 0) n /= p;
    return n == 1;
}

qva_status upload_roots() {
    std::vector<double2> roots(160, make_double2(0, 0));
    for (int r = 2; r <= 16; ++r)
        for (int j = 0; j < r; ++j) {
            long double ang = -2.0L * 3.141592653589793238462643383279502884L * j / r;
            roots[root_off(r) + j] = make_double2((double)cosl(ang), (double)sinl(ang));
        }
    QVA_CUDA_TRY(cudaMemcpyToSymbol(c_roots, roots.data(), roots.size() * sizeof(double2)));
    return QVA_OK;
}

}  // namespace

qva_status fft_plan_create(uint64_t N, int device, FftPlan **out) {
    *out = nullptr;
    FftPlan *fp = new FftPlan();
    fp->N = N;
    fp->device = device;
    std::vector<double2> tw;
    if (N <= (uint64_t)kMaxSub && smooth(N)) {
        fp->whole = true;
        fp->N1 = 1;
        fp->N2 = (int)N;
        if (!make_sub((int)N, fp->row, tw)) {
            delete fp;
            set_error("FFT planning failed");
            return QVA_ERR_UNSUPPORTED;
        }
    } else {
        // pick N1 <= N2, both <= kMaxSub and 13-smooth, N1 as large as possible (balanced)
        int best1 = 0;
        for (uint64_t n1 = 2; n1 <= (uint64_t)kMaxSub && n1 * n1 <= N; ++n1) {
            if (N % n1) continue;
            uint64_t n2 = N / n1;
            if (n2 > (uint64_t)kMaxSub || !smooth(n1) || !smooth(n2)) continue;
            if (n1 * 2 * 2 * sizeof(double2) > 200 * 1024) continue;  // col smem (cw=2, ping-pong)
            best1 = (int)n1;
        }
        if (!best1) {
            delete fp;
            set_error("circulant mixer: N=" + std::to_string(N) +
                      " is not a product N1*N2 of two 13-smooth factors <= 4096 (Bluestein path not built yet)");
            return QVA_ERR_UNSUPPORTED;
        }
        fp->N1 = best1;
        fp->N2 = (int)(N / best1);
        fp->cw = 2;
        if (!make_sub(fp->N1, fp->col, tw) || !make_sub(fp->N2, fp->row, tw)) {
            delete fp;
            set_error("FFT planning failed");
            return QVA_ERR_UNSUPPORTED;
        }
        // four-step twiddles w_N^r = hi[r >> s] * lo[r & (2^s - 1)]
        int s = 11;
        uint64_t B = 1ull << s;
        uint64_t nhi = (N + B - 1) / B;
        std::vector<double2> lo(B), hi(nhi);
        for (uint64_t j = 0; j < B; ++j) {
            long double ang = -2.0L * 3.141592653589793238462643383279502884L * (long double)j / (long double)N;
            lo[j] = make_double2((double)cosl(ang), (double)sinl(ang));
        }
        for (uint64_t j = 0; j < nhi; ++j) {
            long double ang = -2.0L * 3.141592653589793238462643383279502884L * (long double)((j * B) % N) / (long double)N;
            hi[j] = make_double2((double)cosl(ang), (double)sinl(ang));
        }
        fp->big_shift = s;
        if (cudaMalloc(&fp->d_big_lo, B * sizeof(double2)) != cudaSuccess ||
            cudaMalloc(&fp->d_big_hi, nhi * sizeof(double2)) != cudaSuccess) {
            fft_plan_destroy(fp);
            set_error("cudaMalloc (FFT twiddles) failed");
            return QVA_ERR_OUT_OF_MEMORY;
        }
        cudaMemcpy(fp->d_big_lo, lo.data(), B * sizeof(double2), cudaMemcpyHostToDevice);
        cudaMemcpy(fp->d_big_hi, hi.data(), nhi * sizeof(double2), cudaMemcpyHostToDevice);
        fp->n_partials = (fp->N2 + fp->cw - 1) / fp->cw;
        if (cudaMalloc(&fp->partials, fp->n_partials * 2 * sizeof(double)) != cudaSuccess) {
            fft_plan_destroy(fp);
            set_error("cudaMalloc (FFT partials) failed");
            return QVA_ERR_OUT_OF_MEMORY;
        }
    }
    if (cudaMalloc(&fp->d_tw, std::max<size_t>(tw.size(), 1) * sizeof(double2)) != cudaSuccess) {
        fft_plan_destroy(fp);
        set_error("cudaMalloc (FFT tables) failed");
        return QVA_ERR_OUT_OF_MEMORY;
    }
    cudaMemcpy(fp->d_tw, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice);
    qva_status st = upload_roots();
    if (st != QVA_OK) {
        fft_plan_destroy(fp);
        return st;
    }
    size_t smem_col = (size_t)2 * fp->cw * fp->N1 * sizeof(double2);
    size_t smem_row = (size_t)2 * fp->N2 * sizeof(double2);
    cudaFuncSetAttribute(fft_col_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem_col, 1));
    cudaFuncSetAttribute(fft_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_row);
    cudaFuncSetAttribute(fft_whole_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_row);
    *out = fp;
    return QVA_OK;
}

void fft_plan_destroy(FftPlan *fp) {
    if (!fp) return;
    cudaFree(fp->d_tw);
    cudaFree(fp->d_big_lo);
    cudaFree(fp->d_big_hi);
    cudaFree(fp->partials);
    delete fp;
}

void fft_permute_spectrum(const FftPlan *fp, const double *lambda, double *lambda_perm) {
    if (fp->whole) {
        memcpy(lambda_perm, lambda, fp->N * sizeof(double));
        return;
    }
    const uint64_t N1 = fp->N1, N2 = fp->N2;
    for (uint64_t k1 = 0; k1 < N1; ++k1)
        for (uint64_t k2 = 0; k2 < N2; ++k2) lambda_perm[k1 * N2 + k2] = lambda[k1 + N1 * k2];
}

qva_status fft_run(FftPlan *fp, const FftRun &r, cudaStream_t s, LaunchObserver *obs) {
    const double N = (double)fp->N;
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
        int nth = r.mode == 0 ? 2 * r.p : 1;
        double *dth = nullptr;
        QVA_CUDA_TRY(cudaMallocAsync((void **)&dth, std::max(nth, 1) * sizeof(double), s));
        if (nth) QVA_CUDA_TRY(cudaMemcpyAsync(dth, r.theta, nth * sizeof(double), cudaMemcpyHostToDevice, s));
        a.theta = dth;
        size_t smem = (size_t)2 * fp->N2 * sizeof(double2);
        obs->begin(K_FFT_ROW, state_bytes * (r.init ? 1 : 2) + q_bytes * (r.mode == 0 ? 1 : 0));
        fft_whole_kernel<<<1, kWholeThreads, smem, s>>>(a);
        cudaError_t e = cudaGetLastError();
        obs->end();
        cudaFreeAsync(dth, s);
        if (e != cudaSuccess) {
            set_error(std::string("fft_whole_kernel: ") + cudaGetErrorString(e));
            return QVA_ERR_CUDA;
        }
        return QVA_OK;
    }
    ColArgs c{};
    c.psi = r.psi;
    c.q = r.q;
    c.N1 = fp->N1;
    c.N2 = fp->N2;
    c.cw = fp->cw;
    c.amp0 = r.amp0;
    c.tw = fp->d_tw;
    c.big_lo = fp->d_big_lo;
    c.big_hi = fp->d_big_hi;
    c.big_shift = fp->big_shift;
    c.partials = fp->partials;
    c.sf = fp->col;
    RowArgs w{};
    w.psi = r.psi;
    w.N1 = fp->N1;
    w.N2 = fp->N2;
    w.lambda_perm = r.lambda_perm;
    w.invN = 1.0 / N;
    w.tw = fp->d_tw;
    w.big_lo = fp->d_big_lo;
    w.big_hi = fp->d_big_hi;
    w.big_shift = fp->big_shift;
    w.sf = fp->row;
    const size_t smem_col = (size_t)2 * fp->cw * fp->N1 * sizeof(double2);
    const size_t smem_row = (size_t)2 * fp->N2 * sizeof(double2);
    const int col_grid = (fp->N2 + fp->cw - 1) / fp->cw;

    auto launch_col = [&](int init, int inv, int phase, double gamma, int fwd, int expect) -> qva_status {
        c.init = init;
        c.do_inv = inv;
        c.do_phase = phase;
        c.gamma = gamma;
        c.do_fwd = fwd;
        c.do_expect = expect;
        double bytes = state_bytes * (init ? 1 : 2) + q_bytes * ((phase || expect) ? 1 : 0);
        obs->begin(K_FFT_COL, bytes);
        fft_col_kernel<<<col_grid, kFftThreads, smem_col, s>>>(c);
        cudaError_t e = cudaGetLastError();
        obs->end();
        if (e != cudaSuccess) {
            set_error(std::string("fft_col_kernel: ") + cudaGetErrorString(e));
            return QVA_ERR_CUDA;
        }
        return QVA_OK;
    };
    auto launch_row = [&](double beta) -> qva_status {
        w.beta = beta;
        double s0, c0, s1, c1;
        s0 = sin(-beta * r.lam0);
        c0 = cos(-beta * r.lam0);
        s1 = sin(-beta * r.lamc);
        c1 = cos(-beta * r.lamc);
        w.e0 = make_double2(c0 / N, s0 / N);
        w.ec = make_double2(c1 / N, s1 / N);
        obs->begin(K_FFT_ROW, state_bytes * 2 + (r.lambda_perm ? 8.0 * N : 0.0));
        fft_row_kernel<<<fp->N1, kFftThreads, smem_row, s>>>(w);
        cudaError_t e = cudaGetLastError();
        obs->end();
        if (e != cudaSuccess) {
            set_error(std::string("fft_row_kernel: ") + cudaGetErrorString(e));
            return QVA_ERR_CUDA;
        }
        return QVA_OK;
    };
    if (r.mode == 1) {
        QVA_TRY(launch_col(0, 0, 0, 0.0, 1, 0));
        QVA_TRY(launch_row(r.theta[0]));
        QVA_TRY(launch_col(0, 1, 0, 0.0, 0, 0));
        return QVA_OK;
    }
    for (int k = 0; k < r.p; ++k) {
        QVA_TRY(launch_col(k == 0 ? r.init : 0, k > 0, 1, r.theta[2 * k], 1, 0));
        QVA_TRY(launch_row(r.theta[2 * k + 1]));
    }
    if (r.p > 0) {
        QVA_TRY(launch_col(0, 1, 0, 0.0, 0, r.expect ? 1 : 0));
        if (r.expect) {
            obs->begin(K_REDUCE, 16.0 * fp->n_partials);
            cudaError_t e = launch_reduce_partials(fp->partials, fp->n_partials, 1, r.red_out, s);
            obs->end();
            if (e != cudaSuccess) {
                set_error(std::string("reduce: ") + cudaGetErrorString(e));
                return QVA_ERR_CUDA;
            }
        }
    }
    return QVA_OK;
}

}  // namespace qva
