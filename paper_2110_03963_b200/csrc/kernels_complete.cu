// kernels_complete.cu -- the circulant mixer with a complete-graph-family spectrum
// lambda = (lambda_0, c, c, ..., c) (cfg3: the K_N Laplacian, lambda_0 = 0, c = N; PAPER.md:293
// Eq. qwoa / :315-333 Sec. 3, readings R3-R5) applied in closed form instead of by FFT
// (SURVEY §2 K10, §8(d) "K_N closed form: 2 passes"): the circulant with that spectrum is
//     U(beta) = F^-1 diag(e^{-i beta lambda}) F = e^{-i beta c} I + (e^{-i beta lambda_0} - e^{-i beta c}) J / N
// (J = all ones: the j = 0 Fourier mode is the uniform vector), so
//     U psi = a psi + d 1,   a = e^{-i beta c},   d = (e^{-i beta lambda_0} - a) mean(psi).
// An O(N) speed-of-light reference for the FFT path (opt-in per plan, desc.reserved[4]).
//
// Schedule of a p-layer evolution: the mixer of layer k is kept as a pending affine map (a_k, d_k)
// and applied by the pass of layer k+1 as it loads: one pass per layer (load, affine map,
// phase, store, per-block sum of the phased state) plus one final pass (affine map, <Q> partials),
// each followed by a one-block kernel that reduces the sums in fixed order and forms (a, d) on the
// device.  40 B per amplitude-layer (read psi 16 + q 8, write psi 16).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "qva_internal.h"

namespace qva {
namespace {

constexpr int kCThreads = 256;

__device__ __forceinline__ void creduce2(double &a, double &b, double *red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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

// One pass: v = init ? amp0 : psi[x]; v = a v + d (pending mixer, ad != nullptr); v *= exp(-i gamma
// q_x) (do_phase); psi[x] = v.  Per block: sum of v (mode 0) or (sum |v|^2 q_x, sum |v|^2) (mode 1).
__global__ void __launch_bounds__(kCThreads) complete_pass_kernel(double2 *psi, const double *q, uint64_t n, int init,
                                                                  double amp0, const double2 *ad, int do_phase,
                                                                  double gamma, int mode, double *partials) {
    __shared__ double red[2 * (kCThreads / 32)];
    double2 a = make_double2(1.0, 0.0), d = make_double2(0.0, 0.0);
    if (ad) {
        a = ad[0];
        d = ad[1];
    }
    double s0 = 0.0, s1 = 0.0;
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) {
        double2 v = init ? make_double2(amp0, 0.0) : psi[x];
        if (ad) v = make_double2(fma(a.x, v.x, fma(-a.y, v.y, d.x)), fma(a.x, v.y, fma(a.y, v.x, d.y)));
        double qv = 0.0;
        if (do_phase || mode == 1) qv = __ldg(q + x);
        if (do_phase) {
            double sn, cs;
            sincos(gamma * qv, &sn, &cs);
            v = make_double2(fma(cs, v.x, sn * v.y), fma(cs, v.y, -sn * v.x));
        }
        psi[x] = v;
        if (mode == 0) {
            s0 += v.x;
            s1 += v.y;
        } else {
            const double pr = v.x * v.x + v.y * v.y;
            s0 = fma(pr, qv, s0);
            s1 += pr;
        }
    }
    creduce2(s0, s1, red);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = s0;
        partials[2 * blockIdx.x + 1] = s1;
    }
}

// (a, d) of U(beta) from the per-block sums of the state it acts on: a = e^{-i beta c},
// d = (e^{-i beta lambda_0} - a) * sum / N.  One block, fixed summation order.  mode 1: only the
// sum, into ad[2] (sharded: reduced over ranks before mode 2); mode 2: (a, d) from ad[2].
__global__ void complete_coef_kernel(const double *partials, int nblocks, double beta, double lam0, double lamc,
                                     double invN, double2 *ad, int mode) {
    __shared__ double red[2 * 32];
    double s0 = 0.0, s1 = 0.0;
    if (mode == 2) {
        s0 = ad[2].x;
        s1 = ad[2].y;
    } else {
        for (int i = threadIdx.x; i < nblocks; i += blockDim.x) {
            s0 += partials[2 * i];
            s1 += partials[2 * i + 1];
        }
        creduce2(s0, s1, red);
    }
    if (threadIdx.x == 0 && mode == 1) ad[2] = make_double2(s0, s1);
    if (threadIdx.x == 0 && mode != 1) {
        double sc, cc, s0l, c0l;
        sincos(-beta * lamc, &sc, &cc);
        sincos(-beta * lam0, &s0l, &c0l);
        const double2 a = make_double2(cc, sc);
        const double2 e = make_double2(c0l - cc, s0l - sc);
        const double mr = s0 * invN, mi = s1 * invN;
        ad[0] = a;
        ad[1] = make_double2(e.x * mr - e.y * mi, e.x * mi + e.y * mr);
    }
}

int complete_grid(uint64_t n) {
    const uint64_t want = (n + kCThreads - 1) / kCThreads;
    const uint64_t cap = (uint64_t)num_sms() * 8;
    return (int)std::max<uint64_t>(1, std::min(want, cap));
}

}  // namespace

size_t complete_scratch_doubles(uint64_t n) { return 2 * (size_t)complete_grid(n) + 6; }

qva_status complete_run(const FftRun &r, uint64_t n, uint64_t n_global, double *scratch, cudaStream_t s,
                        LaunchObserver *obs, CompleteComm *comm) {
    const int grid = complete_grid(n);
    double *partials = scratch;
    double2 *ad = reinterpret_cast<double2 *>(scratch + 2 * (size_t)grid);
    const double invN = 1.0 / (double)n_global;
    auto pass = [&](int init, const double2 *pend, int do_phase, double gamma, int mode) -> qva_status {
        const double bytes = (init ? 0.0 : 16.0 * n) + 16.0 * n + ((do_phase || mode == 1) ? 8.0 * n : 0.0);
        obs->begin(K_OTHER, bytes);
        complete_pass_kernel<<<grid, kCThreads, 0, s>>>(r.psi, r.q, n, init, r.amp0, pend, do_phase, gamma, mode,
                                                        partials);
        cudaError_t e = cudaGetLastError();
        obs->end();
        if (e != cudaSuccess) {
            set_error(std::string("complete_pass_kernel: ") + cudaGetErrorString(e));
            return QVA_ERR_CUDA;
        }
        return QVA_OK;
    };
    auto coef = [&](double beta) -> qva_status {
        obs->begin(K_REDUCE, 16.0 * grid);
        if (!comm) {
            complete_coef_kernel<<<1, 1024, 0, s>>>(partials, grid, beta, r.lam0, r.lamc, invN, ad, 0);
        } else {  // row-sharded state: the sum of psi over every rank (16 B all-reduce)
            complete_coef_kernel<<<1, 1024, 0, s>>>(partials, grid, beta, r.lam0, r.lamc, invN, ad, 1);
            qva_status st = comm->sum2_dev(reinterpret_cast<double *>(ad + 2));
            if (st != QVA_OK) {
                obs->end();
                return st;
            }
            complete_coef_kernel<<<1, 32, 0, s>>>(partials, grid, beta, r.lam0, r.lamc, invN, ad, 2);
        }
        cudaError_t e = cudaGetLastError();
        obs->end();
        if (e != cudaSuccess) {
            set_error(std::string("complete_coef_kernel: ") + cudaGetErrorString(e));
            return QVA_ERR_CUDA;
        }
        return QVA_OK;
    };
    if (r.mode == 1) {  // one mixer on the current state: sum pass, then the affine map
        QVA_TRY(pass(0, nullptr, 0, 0.0, 0));
        QVA_TRY(coef(r.theta[0]));
        return pass(0, ad, 0, 0.0, 0);
    }
    for (int k = 0; k < r.p; ++k) {
        QVA_TRY(pass(k == 0 ? r.init : 0, k == 0 ? nullptr : ad, 1, r.theta[2 * k], 0));
        QVA_TRY(coef(r.theta[2 * k + 1]));
    }
    if (r.p > 0) {
        QVA_TRY(pass(0, ad, 0, 0.0, r.expect ? 1 : 0));
        if (r.expect) {
            obs->begin(K_REDUCE, 16.0 * grid);
            cudaError_t e = launch_reduce_partials(partials, grid, 1, r.red_out, s);
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
