// kernels_x.cu -- sm_100a kernels of the X-mixer (QAOA) path and the shared elementwise /
// reduction kernels.
//
//  (the tile pass of the X mixer lives in kernels_tile.cu)
//  * small_evolve_kernel: whole p-layer evolution of a <= 2^12-amplitude state in one CTA.
//  * maxcut_q_kernel: q_x = -cut_w(x) (Eq. maxcut-cost, reading R10).
//  * fixed-order fp64 reductions (deterministic), elementwise phase, transpose for the
//    global<->local qubit exchange (COMM-psi).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "qva_internal.h"

namespace qva {

namespace {

// a' = c a - i s b ; b' = -i s a + c b   (exp(-i beta X) on the pair; small-state kernel)
__device__ __forceinline__ void butterfly(double2 &a, double2 &b, double c, double s) {
    double ar = a.x, ai = a.y, br = b.x, bi = b.y;
    a.x = fma(c, ar, s * bi);
    a.y = fma(c, ai, -s * br);
    b.x = fma(c, br, s * ai);
    b.y = fma(c, bi, -s * ar);
}

__device__ __forceinline__ void apply_phase(double2 &a, double qv, double gamma) {
    double sn, cs;
    sincos(gamma * qv, &sn, &cs);
    double re = a.x, im = a.y;
    a.x = fma(cs, re, sn * im);
    a.y = fma(cs, im, -sn * re);
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
        int nw = blockDim.x >> 5;
        for (int w = 0; w < nw; ++w) {
            sa += red[2 * w];
            sb += red[2 * w + 1];
        }
        a = sa;
        b = sb;
    }
}

// tab[b][j] = exp(-i gamma_b (qmin + j)) * mult_b (mult: the scalar factors the passes defer to
// the phase, see run_passes; nullptr = 1)
__global__ void phase_table_kernel(double2 *tab, const double *gammas, const double2 *mult, int batch, int qmin,
                                   int ntab) {
    int total = batch * ntab;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
        int b = k / ntab, j = k - b * ntab;
        double sn, cs;
        sincos(gammas[b] * (double)(qmin + j), &sn, &cs);
        double2 f = make_double2(cs, -sn);
        if (mult) {
            const double2 m = mult[b];
            f = make_double2(f.x * m.x - f.y * m.y, f.x * m.y + f.y * m.x);
        }
        tab[k] = f;
    }
}

// flags[0] |= non-integer seen; partial min/max per block
__global__ void q_range_kernel(const double *q, uint64_t n, int *flags, double *mm) {
    __shared__ double smin[256], smax[256];
    double lo = INFINITY, hi = -INFINITY;
    int nonint = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        double x = q[i];
        lo = fmin(lo, x);
        hi = fmax(hi, x);
        if (x != rint(x)) nonint = 1;
    }
    if (nonint) atomicOr(flags, 1);
    smin[threadIdx.x] = lo;
    smax[threadIdx.x] = hi;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + s]);
            smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + s]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        mm[2 * blockIdx.x] = smin[0];
        mm[2 * blockIdx.x + 1] = smax[0];
    }
}

__global__ void q_encode_kernel(const double *q, uint64_t n, void *codes, int bytes) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        int c = (int)q[i];
        if (bytes == 1) reinterpret_cast<int8_t *>(codes)[i] = (int8_t)c;
        else reinterpret_cast<int16_t *>(codes)[i] = (int16_t)c;
    }
}

// ---------------------------------------------------------------------------------------------
// whole-state-in-one-CTA evolution for n <= 12 (cfg1 and small batches)
// ---------------------------------------------------------------------------------------------
constexpr int kSmallThreads = 512;

__global__ void __launch_bounds__(kSmallThreads)
small_evolve_kernel(const SmallEvolveParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *st = reinterpret_cast<double2 *>(smem_raw);
    __shared__ double red[2 * (kSmallThreads / 32)];
    const int N = 1 << P.n;
    const int b = blockIdx.x;
    const int tid = threadIdx.x;
    double2 *gpsi = P.psi + (uint64_t)b * N;
    const double *th = P.thetas + (uint64_t)b * 2 * (P.mode == 0 ? P.p : 1);

    if (P.mode == 0) {
        if (P.psi0) {
            for (int i = tid; i < N; i += blockDim.x) st[i] = P.psi0[i];
        } else {
            double a = 1.0 / sqrt((double)N);
            for (int i = tid; i < N; i += blockDim.x) st[i] = make_double2(a, 0.0);
        }
    } else {
        for (int i = tid; i < N; i += blockDim.x) st[i] = gpsi[i];
    }
    __syncthreads();

    const int layers = (P.mode == 0) ? P.p : 1;
    for (int k = 0; k < layers; ++k) {
        if (P.mode != 2) {
            double gamma = th[2 * k];
            for (int i = tid; i < N; i += blockDim.x) apply_phase(st[i], P.q[i], gamma);
            __syncthreads();
        }
        if (P.mode != 1) {
            double beta = (P.mode == 0) ? th[2 * k + 1] : th[0];
            double s, c;
            sincos(beta, &s, &c);
            for (int j = 0; j < P.n; ++j) {
                for (int pidx = tid; pidx < (N >> 1); pidx += blockDim.x) {
                    int lo = pidx & ((1 << j) - 1);
                    int x = ((pidx >> j) << (j + 1)) | lo;
                    butterfly(st[x], st[x | (1 << j)], c, s);
                }
                __syncthreads();
            }
        }
    }
    double acc = 0.0, nrm = 0.0;
    for (int i = tid; i < N; i += blockDim.x) {
        double2 a = st[i];
        gpsi[i] = a;
        double pr = a.x * a.x + a.y * a.y;
        acc = fma(pr, P.q[i], acc);
        nrm += pr;
    }
    if (P.out) {
        block_reduce2(acc, nrm, red);
        if (tid == 0) {
            P.out[2 * b] = acc;
            P.out[2 * b + 1] = nrm;
        }
    }
}

// ---------------------------------------------------------------------------------------------
constexpr int kEdgeChunk = 1024;

__global__ void maxcut_q_kernel(double *q, uint64_t count, uint64_t offset, int m, const int32_t *u,
                                const int32_t *v, const double *w) {
    __shared__ int su[kEdgeChunk], sv[kEdgeChunk];
    __shared__ double sw[kEdgeChunk];
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < count;
         base += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t i = base + threadIdx.x;
        uint64_t x = offset + i;
        double cut = 0.0;
        for (int e0 = 0; e0 < m; e0 += kEdgeChunk) {
            int ne = min(kEdgeChunk, m - e0);
            __syncthreads();
            for (int k = threadIdx.x; k < ne; k += blockDim.x) {
                su[k] = u[e0 + k];
                sv[k] = v[e0 + k];
                sw[k] = w ? w[e0 + k] : 1.0;
            }
            __syncthreads();
            for (int k = 0; k < ne; ++k) {
                // sequential in edge order: identical rounding to a plain loop
                if (((x >> su[k]) ^ (x >> sv[k])) & 1) cut += sw[k];
            }
        }
        if (i < count) q[i] = -cut;
    }
}

// Permutation-subspace qualities (readings R23, R24): rank r -> the r-th
// k-permutation s of {0..m-1} in lexicographic order (Lehmer digits d_a = r / cnt[a] with
// cnt[a] = (m-a-1)!/(m-k)!, each picking the d_a-th smallest unused element), then
// q_r = sum_a ( Cl[a][s_a] + sum_b F[a][b] D[s_a][s_b] ) in that order (zero F terms skipped:
// adding +0.0 is exact).  s lives in two 64-bit words, 5 bits per slot (k <= 24), so the thread
// stays in registers.  A one-off setup kernel: integer-division bound, not on the step path.
struct KpermArgs {
    int m, k, nf;            // elements, slots, nonzero F entries
    const uint64_t *cnt;     // [k]
    const double *D;         // [m][m]
    const double *Cl;        // [k][m] or nullptr
    const int *fab;          // [nf] (a << 8 | b), a-major
    const double *fv;        // [nf]
    const int *frow;         // [k + 1] start of row a in (fab, fv)
};
constexpr int kKpermMaxM = 20, kKpermMaxNf = 400;
__global__ void kperm_q_kernel(double *q, uint64_t count, uint64_t offset, KpermArgs a) {
    __shared__ double sD[kKpermMaxM * kKpermMaxM], sC[kKpermMaxM * kKpermMaxM], sF[kKpermMaxNf];
    __shared__ unsigned short sFab[kKpermMaxNf];
    __shared__ uint64_t sCnt[kKpermMaxM];
    __shared__ int sRow[kKpermMaxM + 1];
    for (int i = threadIdx.x; i < a.m * a.m; i += blockDim.x) sD[i] = a.D[i];
    for (int i = threadIdx.x; i < a.k * a.m; i += blockDim.x) sC[i] = a.Cl ? a.Cl[i] : 0.0;
    for (int i = threadIdx.x; i < a.nf; i += blockDim.x) {
        sF[i] = a.fv[i];
        sFab[i] = (unsigned short)a.fab[i];
    }
    for (int i = threadIdx.x; i < a.k; i += blockDim.x) sCnt[i] = a.cnt[i];
    for (int i = threadIdx.x; i <= a.k; i += blockDim.x) sRow[i] = a.frow[i];
    __syncthreads();
    const bool lin = a.Cl != nullptr;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t r = offset + i;
        uint32_t used = 0;
        uint64_t w0 = 0, w1 = 0;  // slot a < 12 in w0, else w1 (5 bits each)
        for (int s = 0; s < a.k; ++s) {
            const uint64_t c = sCnt[s];
            const uint64_t d = r / c;
            r -= d * c;
            // the d-th (0-based) element of {0..m-1} not yet used
            uint32_t free = ~used & ((1u << a.m) - 1u);
            for (uint64_t t = 0; t < d; ++t) free &= free - 1u;
            const int e = __ffs(free) - 1;
            used |= 1u << e;
            if (s < 12) w0 |= (uint64_t)e << (5 * s);
            else w1 |= (uint64_t)e << (5 * (s - 12));
        }
        auto slot = [&](int s) -> int {
            return (int)(((s < 12 ? w0 >> (5 * s) : w1 >> (5 * (s - 12)))) & 31u);
        };
        double acc = 0.0;
        for (int s = 0; s < a.k; ++s) {
            const int ea = slot(s);
            if (lin) acc += sC[s * a.m + ea];
            for (int f = sRow[s]; f < sRow[s + 1]; ++f) {
                const int b = sFab[f] & 255;
                acc += sF[f] * sD[ea * a.m + slot(b)];
            }
        }
        q[i] = acc;
    }
}

template <typename T>
__global__ void chunk_transpose_kernel(T *out, const T *in, int G, uint64_t C) {
    uint64_t total = (uint64_t)G * G * C;
    for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t c = idx % C;
        uint64_t rt = idx / C;           // destination chunk index (t*G + r)
        uint64_t tdst = rt / G, r = rt % G;
        out[idx] = in[(r * G + tdst) * C + c];
    }
}

__global__ void reduce_partials_kernel(const double *partials, uint64_t n, double *out) {
    __shared__ double red[64];
    const double *pp = partials + 2 * n * blockIdx.x;
    double a = 0.0, b = 0.0;
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
        a += pp[2 * i];
        b += pp[2 * i + 1];
    }
    block_reduce2(a, b, red);
    if (threadIdx.x == 0) {
        out[2 * blockIdx.x] = a;
        out[2 * blockIdx.x + 1] = b;
    }
}

__global__ void phase_kernel(double2 *psi, const double *q, uint64_t n, double gamma) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double2 a = psi[i];
        apply_phase(a, q[i], gamma);
        psi[i] = a;
    }
}

__global__ void fill_uniform_kernel(double2 *psi, uint64_t n, double amp) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        psi[i] = make_double2(amp, 0.0);
}

__global__ void expect_partials_kernel(const double2 *psi, const double *q, uint64_t n, double *partials) {
    __shared__ double red[64];
    double a = 0.0, b = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double2 v = psi[i];
        double pr = v.x * v.x + v.y * v.y;
        a = fma(pr, q[i], a);
        b += pr;
    }
    block_reduce2(a, b, red);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = a;
        partials[2 * blockIdx.x + 1] = b;
    }
}

__global__ void probabilities_kernel(const double2 *psi, double *out, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double2 v = psi[i];
        out[i] = v.x * v.x + v.y * v.y;
    }
}

__global__ void check_finite_kernel(const double *x, uint64_t n, int *flag) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (!isfinite(x[i])) *flag = 1;
}

inline int grid_for(uint64_t n, int threads) {
    uint64_t b = (n + threads - 1) / threads;
    uint64_t cap = (uint64_t)num_sms() * 16;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

}  // namespace

cudaError_t launch_phase_table(double2 *tab, const double *gammas, const double2 *mult, int batch, int qmin,
                               int ntab, cudaStream_t s) {
    int total = batch * ntab;
    phase_table_kernel<<<(total + 255) / 256, 256, 0, s>>>(tab, gammas, mult, batch, qmin, ntab);
    return cudaGetLastError();
}

int q_range_blocks(uint64_t n) { return grid_for(n, 256); }

cudaError_t launch_q_range(const double *q, uint64_t n, int *flags, double *mm, int blocks, cudaStream_t s) {
    q_range_kernel<<<blocks, 256, 0, s>>>(q, n, flags, mm);
    return cudaGetLastError();
}

cudaError_t launch_q_encode(const double *q, uint64_t n, void *codes, int bytes, cudaStream_t s) {
    q_encode_kernel<<<grid_for(n, 256), 256, 0, s>>>(q, n, codes, bytes);
    return cudaGetLastError();
}

cudaError_t launch_small_evolve(const SmallEvolveParams &p, int batch, cudaStream_t s) {
    static DeviceOnce configured;
    size_t smem = ((size_t)1 << p.n) * sizeof(double2);
    cudaError_t e = once_per_device(configured, [] {
        return cudaFuncSetAttribute(small_evolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(((size_t)1 << kSmallMaxQubits) * sizeof(double2)));
    });
    if (e != cudaSuccess) return e;
    small_evolve_kernel<<<batch, kSmallThreads, smem, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_maxcut_q(double *q, uint64_t count, uint64_t offset, int m, const int32_t *u,
                            const int32_t *v, const double *w, cudaStream_t s) {
    maxcut_q_kernel<<<grid_for(count, 256), 256, 0, s>>>(q, count, offset, m, u, v, w);
    return cudaGetLastError();
}

cudaError_t launch_kperm_q(double *q, uint64_t count, uint64_t offset, int m, int k, const void *dev_pack, int nf,
                           bool linear, cudaStream_t s) {
    // dev_pack layout (packed by qva_set_qualities_permutation): cnt[k] u64, D[m*m], Cl[k*m] (if
    // linear), fv[nf] doubles, then frow[k+1], fab[nf] ints
    if (m < 1 || m > kKpermMaxM || k < 1 || k > m || nf > kKpermMaxNf) return cudaErrorInvalidValue;
    const unsigned char *b = (const unsigned char *)dev_pack;
    KpermArgs a;
    a.m = m;
    a.k = k;
    a.nf = nf;
    a.cnt = (const uint64_t *)b;
    const double *d = (const double *)(b + sizeof(uint64_t) * k);
    a.D = d;
    d += m * m;
    a.Cl = linear ? d : nullptr;
    if (linear) d += k * m;
    a.fv = d;
    d += nf;
    a.frow = (const int *)d;
    a.fab = a.frow + k + 1;
    if (count == 0) return cudaSuccess;
    kperm_q_kernel<<<grid_for(count, 256), 256, 0, s>>>(q, count, offset, a);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_chunk_transpose(T *out, const T *in, int G, uint64_t C, cudaStream_t s) {
    chunk_transpose_kernel<T><<<grid_for((uint64_t)G * G * C, 256), 256, 0, s>>>(out, in, G, C);
    return cudaGetLastError();
}
template cudaError_t launch_chunk_transpose<double2>(double2 *, const double2 *, int, uint64_t, cudaStream_t);
template cudaError_t launch_chunk_transpose<double>(double *, const double *, int, uint64_t, cudaStream_t);

template <typename T>
__global__ void block_transpose_kernel(T *__restrict__ out, const T *__restrict__ in, uint64_t A, uint64_t B,
                                       uint64_t C) {
    const uint64_t total = A * B * C;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t c = k % C, ab = k / C;
        const uint64_t b = ab % B, a = ab / B;  // in[a][b][c] (coalesced reads)
        out[(b * A + a) * C + c] = in[k];
    }
}

template <typename T>
cudaError_t launch_block_transpose(T *out, const T *in, uint64_t A, uint64_t B, uint64_t C, cudaStream_t s) {
    block_transpose_kernel<T><<<grid_for(A * B * C, 256), 256, 0, s>>>(out, in, A, B, C);
    return cudaGetLastError();
}
template cudaError_t launch_block_transpose<double2>(double2 *, const double2 *, uint64_t, uint64_t, uint64_t,
                                                     cudaStream_t);
template cudaError_t launch_block_transpose<double>(double *, const double *, uint64_t, uint64_t, uint64_t,
                                                    cudaStream_t);

// QAOAz parity mixer pair term exp(-i t (X_aX_b + Y_aY_b)) (PAPER.md Eq. parity_terms): a Givens
// rotation by 2t on the {|..1_a..0_b..>, |..0_a..1_b..>} pairs; |00>, |11> untouched.  Thread k
// of N/4 addresses the pair with bit a = 1, bit b = 0 (bits inserted into k at their positions).
__global__ void parity_pair_kernel(double2 *__restrict__ psi, uint64_t quarter, int a, int b, double c, double s) {
    const int lo = min(a, b), hi = max(a, b);
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < quarter;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t x = ((k >> lo) << (lo + 1)) | (k & ((1ull << lo) - 1));
        x = ((x >> hi) << (hi + 1)) | (x & ((1ull << hi) - 1));
        x |= 1ull << a;
        const uint64_t y = (x ^ (1ull << a)) | (1ull << b);
        const double2 u = psi[x], v = psi[y];
        // u' = c u - i s v, v' = -i s u + c v
        psi[x] = make_double2(fma(c, u.x, s * v.y), fma(c, u.y, -s * v.x));
        psi[y] = make_double2(fma(c, v.x, s * u.y), fma(c, v.y, -s * u.x));
    }
}

// A parity pair term exp(-i t (X_a X_b + Y_a Y_b)) whose qubits are not both local to the shard
// (COMM-psi: rank = the top g index bits): element x of this rank pairs with
// y = x ^ 2^a ^ 2^b when bits a and b of x differ, and y lives on rank y >> L.  Out of place (the
// partner reads our old values too): out = c u - i s v with u = psi[x], v = the partner's value,
// read straight from the owning rank's IPC-mapped buffer (NVLink) -- the pairwise half-slice
// exchange of the paper done by the loads of the kernel itself.  00 / 11 elements copy through.
__global__ void parity_peer_kernel(double2 *__restrict__ out, const double2 *__restrict__ in,
                                   const __grid_constant__ ParityPeer P) {
    const uint64_t nl = 1ull << P.L;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t x = ((uint64_t)P.rank << P.L) | i;
        const double2 u = in[i];
        if ((((x >> P.a) ^ (x >> P.b)) & 1) == 0) {
            out[i] = u;
            continue;
        }
        const uint64_t y = x ^ (1ull << P.a) ^ (1ull << P.b);
        const int ry = (int)(y >> P.L);
        const uint64_t j = y & (nl - 1);
        const double2 v = ry == P.rank ? in[j] : P.peer[ry][j];
        out[i] = make_double2(fma(P.c, u.x, P.s * v.y), fma(P.c, u.y, -P.s * v.x));
    }
}

cudaError_t launch_parity_peer(double2 *out, const double2 *in, const ParityPeer &p, cudaStream_t s) {
    const uint64_t nl = 1ull << p.L;
    parity_peer_kernel<<<grid_for(nl, 256), 256, 0, s>>>(out, in, p);
    return cudaGetLastError();
}

// Several parity pair terms in one HBM round trip: each CTA stages a window of 2^w amplitudes (the
// physical bits P.bits, given as runs; bits 0..2 lead, so loads and stores move 128-B rows),
// optionally applies the phase exp(-i gamma q_x) as it loads, then the listed pair rotations in
// order (each a Givens rotation by 2t on the window's 01/10 pairs, a barrier between pairs),
// and writes the window back.  The host orders the pairs so that every term that shares a qubit
// with an earlier-group term comes after it (reading R19).
__global__ void __launch_bounds__(256) parity_window_kernel(double2 *__restrict__ psi, const __grid_constant__ ParityWindow P) {
    extern __shared__ double2 win[];
    const int W = 1 << P.w;
    const uint64_t n_tiles = 1ull << (P.n - P.w);
    for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        // tile number -> the non-window bits (as runs)
        uint64_t base = 0;
        for (int r = 0; r < P.n_out; ++r) base |= ((t >> P.out_src[r]) & ((1ull << P.out_w[r]) - 1)) << P.out_dst[r];
        __syncthreads();  // the previous tile's stores have read the window
        // batches of kWinU independent loads per thread before any is used (one load per
        // iteration would expose a full memory latency per element)
        constexpr int kWinU = 8;
        for (int e0 = threadIdx.x; e0 < W; e0 += kWinU * blockDim.x) {
            double2 v[kWinU];
            double qv[kWinU];
            uint64_t offs[kWinU];
#pragma unroll
            for (int u = 0; u < kWinU; ++u) {
                const int e = e0 + u * blockDim.x;
                uint64_t off = 0;
                for (int r = 0; r < P.n_in; ++r) off |= (uint64_t)((e >> P.in_src[r]) & ((1 << P.in_w[r]) - 1)) << P.in_dst[r];
                offs[u] = off;
                if (e < W) {
                    v[u] = P.init_amp > 0.0 ? make_double2(P.init_amp, 0.0) : (P.src ? P.src : psi)[base + off];
                    qv[u] = P.q ? P.q[base + off] : 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < kWinU; ++u) {
                const int e = e0 + u * blockDim.x;
                if (e >= W) break;
                double2 x = v[u];
                if (P.q) {
                    double sn, cs;
                    sincos(P.gamma * qv[u], &sn, &cs);
                    x = make_double2(fma(cs, x.x, sn * x.y), fma(cs, x.y, -sn * x.x));
                }
                win[e] = x;
            }
        }
        __syncthreads();
        for (int k = 0; k < P.np; ++k) {
            const int a = P.pa[k], b = P.pb[k];
            const int lo = min(a, b), hi = max(a, b);
            for (int m = threadIdx.x; m < W / 4; m += blockDim.x) {
                int x = ((m >> lo) << (lo + 1)) | (m & ((1 << lo) - 1));
                x = ((x >> hi) << (hi + 1)) | (x & ((1 << hi) - 1));
                x |= 1 << a;
                const int y = (x ^ (1 << a)) | (1 << b);
                const double2 u = win[x], v = win[y];
                win[x] = make_double2(fma(P.c, u.x, P.s * v.y), fma(P.c, u.y, -P.s * v.x));
                win[y] = make_double2(fma(P.c, v.x, P.s * u.y), fma(P.c, v.y, -P.s * u.x));
            }
            __syncthreads();
        }
        for (int e = threadIdx.x; e < W; e += blockDim.x) {
            uint64_t off = 0;
            for (int r = 0; r < P.n_in; ++r) off |= (uint64_t)((e >> P.in_src[r]) & ((1 << P.in_w[r]) - 1)) << P.in_dst[r];
            psi[base + off] = win[e];
        }
    }
}

cudaError_t launch_parity_window(double2 *psi, const ParityWindow &p, cudaStream_t s) {
    static DeviceOnce configured;
    const size_t smem = ((size_t)1 << p.w) * sizeof(double2);
    cudaError_t e = once_per_device(configured, [] {
        return cudaFuncSetAttribute(parity_window_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    });
    if (e != cudaSuccess) return e;
    const uint64_t tiles = 1ull << (p.n - p.w);
    const int grid = (int)std::min<uint64_t>(tiles, (uint64_t)num_sms() * 3);
    parity_window_kernel<<<grid, 256, smem, s>>>(psi, p);
    return cudaGetLastError();
}

cudaError_t launch_parity_pair(double2 *psi, uint64_t n_amps, int a, int b, double t, cudaStream_t s) {
    const uint64_t quarter = n_amps / 4;
    parity_pair_kernel<<<grid_for(quarter, 256), 256, 0, s>>>(psi, quarter, a, b, cos(2.0 * t), sin(2.0 * t));
    return cudaGetLastError();
}

cudaError_t launch_chunk_transpose_bytes(void *out, const void *in, int G, uint64_t C, int elem_bytes, cudaStream_t s) {
    uint64_t total = (uint64_t)G * G * C;
    if (elem_bytes == 1)
        chunk_transpose_kernel<int8_t><<<grid_for(total, 256), 256, 0, s>>>((int8_t *)out, (const int8_t *)in, G, C);
    else
        chunk_transpose_kernel<int16_t><<<grid_for(total, 256), 256, 0, s>>>((int16_t *)out, (const int16_t *)in, G, C);
    return cudaGetLastError();
}

cudaError_t launch_reduce_partials(const double *partials, uint64_t n, int batch, double *out, cudaStream_t s) {
    reduce_partials_kernel<<<batch, 1024, 0, s>>>(partials, n, out);
    return cudaGetLastError();
}

cudaError_t launch_phase(double2 *psi, const double *q, uint64_t n, double gamma, cudaStream_t s) {
    phase_kernel<<<grid_for(n, 256), 256, 0, s>>>(psi, q, n, gamma);
    return cudaGetLastError();
}

cudaError_t launch_fill_uniform(double2 *psi, uint64_t n, double amp, cudaStream_t s) {
    fill_uniform_kernel<<<grid_for(n, 256), 256, 0, s>>>(psi, n, amp);
    return cudaGetLastError();
}

int expect_partial_blocks(uint64_t n) { return grid_for(n, 256); }

cudaError_t launch_expect_partials(const double2 *psi, const double *q, uint64_t n, double *partials,
                                   int blocks, cudaStream_t s) {
    expect_partials_kernel<<<blocks, 256, 0, s>>>(psi, q, n, partials);
    return cudaGetLastError();
}

cudaError_t launch_probabilities(const double2 *psi, double *out, uint64_t n, cudaStream_t s) {
    probabilities_kernel<<<grid_for(n, 256), 256, 0, s>>>(psi, out, n);
    return cudaGetLastError();
}

cudaError_t launch_check_finite(const double *x, uint64_t n, int *flag, cudaStream_t s) {
    check_finite_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, n, flag);
    return cudaGetLastError();
}

}  // namespace qva
