// kernels_x.cu -- sm_100a kernels of the X-mixer (QAOA) path and the shared elementwise /
// reduction kernels.
//
//  * tile_pass_kernel: one HBM round trip over the state.  A CTA owns a tile of 2^12
//    amplitudes whose tile-local bits map to 12 physical index bits (the three lowest
//    physical bits are always included so every warp access is >= 128 B contiguous).
//    Inside the tile it applies, in registers, any subset of the single-qubit rotations
//    exp(-i beta X_j) (reading R1), optionally the phase exp(-i gamma q)
//     between two rotation sets, and optionally accumulates
//    sum |psi|^2 q and sum |psi|^2 (Eq. 2).  Register groups of 4 tile bits
//    are exchanged through a swizzled shared-memory tile (conflict-free 16-B accesses).
//  * small_evolve_kernel: whole p-layer evolution of a <= 2^12-amplitude state in one CTA.
//  * maxcut_q_kernel: q_x = -cut_w(x) (Eq. maxcut-cost, reading R10).
//  * fixed-order fp64 reductions (deterministic), elementwise phase, transpose for the
//    global<->local qubit exchange (COMM-psi).
#include <cuda_runtime.h>
#include <stdint.h>

#include "qva_internal.h"

namespace qva {

namespace {

constexpr int kTile = 1 << kTileBits;          // 4096 amplitudes
constexpr int kPerThread = kTile / kTileThreads;  // 16

__device__ __forceinline__ int smem_slot(int i) { return i ^ ((i >> 4) & 7); }

// tile-local index held by (tid, e) in register group g
__device__ __forceinline__ int map_index(int g, int tid, int e) {
    if (g == 0) return (tid << 4) | e;                              // A: register bits = tile bits 0..3
    if (g == 1) return ((tid >> 4) << 8) | (e << 4) | (tid & 15);   // B: tile bits 4..7
    return (e << 8) | tid;                                          // C: tile bits 8..11
}

// a' = c a - i s b ; b' = -i s a + c b   (exp(-i beta X) on the pair)
__device__ __forceinline__ void butterfly(double2 &a, double2 &b, double c, double s) {
    double ar = a.x, ai = a.y, br = b.x, bi = b.y;
    a.x = fma(c, ar, s * bi);
    a.y = fma(c, ai, -s * br);
    b.x = fma(c, br, s * ai);
    b.y = fma(c, bi, -s * ar);
}

template <int B>
__device__ __forceinline__ void rot_bit(double2 (&v)[kPerThread], double c, double s) {
#pragma unroll
    for (int e = 0; e < kPerThread; ++e)
        if (!(e & (1 << B))) butterfly(v[e], v[e | (1 << B)], c, s);
}

__device__ __forceinline__ void rotate_mask(double2 (&v)[kPerThread], int mask, double c, double s) {
    if (mask & 1) rot_bit<0>(v, c, s);
    if (mask & 2) rot_bit<1>(v, c, s);
    if (mask & 4) rot_bit<2>(v, c, s);
    if (mask & 8) rot_bit<3>(v, c, s);
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

__global__ void __launch_bounds__(kTileThreads, 2)
tile_pass_kernel(const TilePassParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *tile = reinterpret_cast<double2 *>(smem_raw);
    uint64_t *off_lo = reinterpret_cast<uint64_t *>(smem_raw + kTile * sizeof(double2));
    uint64_t *off_hi = off_lo + 64;
    __shared__ double red[2 * (kTileThreads / 32)];

    const int tid = threadIdx.x;
    const uint64_t t = blockIdx.x;
    const int member = blockIdx.y;

    // physical offset tables of the tile-local index (bits 0..5 and 6..11)
    if (tid < 128) {
        int j = tid & 63, hi = tid >> 6;
        uint64_t o = 0;
#pragma unroll
        for (int k = 0; k < 6; ++k)
            if ((j >> k) & 1) o |= (uint64_t)1 << P.tile_bits[k + 6 * hi];
        (hi ? off_hi : off_lo)[j] = o;
    }
    // base: deposit the tile number into the non-tile physical bits
    uint64_t tmask = 0;
#pragma unroll
    for (int k = 0; k < kTileBits; ++k) tmask |= (uint64_t)1 << P.tile_bits[k];
    uint64_t base = 0, tt = t;
    for (int b = 0; b < P.n_phys_bits; ++b) {
        if (!((tmask >> b) & 1)) {
            base |= (tt & 1) << b;
            tt >>= 1;
        }
    }
    __syncthreads();

    const PassAngles ang = P.angles[member];
    const double2 *src = P.psi_in + (uint64_t)member * P.member_stride;
    double2 *dst = P.psi_out + (uint64_t)member * P.member_stride;

    double2 v[kPerThread];
    int g = P.steps[0].group;
    if (P.init == 1) {
#pragma unroll
        for (int e = 0; e < kPerThread; ++e) v[e] = make_double2(P.amp0, 0.0);
    } else {
#pragma unroll
        for (int e = 0; e < kPerThread; ++e) {
            int i = map_index(g, tid, e);
            v[e] = src[base + off_lo[i & 63] + off_hi[i >> 6]];
        }
    }

    for (int k = 0; k < P.n_steps; ++k) {
        const PassStep st = P.steps[k];
        if (st.group != g) {
#pragma unroll
            for (int e = 0; e < kPerThread; ++e) tile[smem_slot(map_index(g, tid, e))] = v[e];
            __syncthreads();
            g = st.group;
#pragma unroll
            for (int e = 0; e < kPerThread; ++e) v[e] = tile[smem_slot(map_index(g, tid, e))];
            __syncthreads();
        }
        if (st.mask) {
            double c = st.angle ? ang.c2 : ang.c1;
            double s = st.angle ? ang.s2 : ang.s1;
            rotate_mask(v, st.mask, c, s);
        }
        if (st.phase) {
#pragma unroll
            for (int e = 0; e < kPerThread; ++e) {
                int i = map_index(g, tid, e);
                apply_phase(v[e], __ldg(P.q + base + off_lo[i & 63] + off_hi[i >> 6]), ang.gamma);
            }
        }
    }

    double acc = 0.0, nrm = 0.0;
#pragma unroll
    for (int e = 0; e < kPerThread; ++e) {
        int i = map_index(g, tid, e);
        uint64_t o = base + off_lo[i & 63] + off_hi[i >> 6];
        dst[o] = v[e];
        if (P.expect) {
            double pr = v[e].x * v[e].x + v[e].y * v[e].y;
            acc = fma(pr, __ldg(P.q + o), acc);
            nrm += pr;
        }
    }
    if (P.expect) {
        block_reduce2(acc, nrm, red);
        if (tid == 0) {
            double *pp = P.partials + 2 * ((uint64_t)member * P.n_tiles + t);
            pp[0] = acc;
            pp[1] = nrm;
        }
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
    uint64_t cap = 148ull * 16;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

}  // namespace

cudaError_t launch_tile_pass(const TilePassParams &p, int batch, cudaStream_t s) {
    static bool configured = false;
    size_t smem = kTile * sizeof(double2) + 128 * sizeof(uint64_t);
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(tile_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    dim3 grid((unsigned)p.n_tiles, (unsigned)batch);
    tile_pass_kernel<<<grid, kTileThreads, smem, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_small_evolve(const SmallEvolveParams &p, int batch, cudaStream_t s) {
    static bool configured = false;
    size_t smem = ((size_t)1 << p.n) * sizeof(double2);
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(small_evolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(((size_t)1 << kSmallMaxQubits) * sizeof(double2)));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    small_evolve_kernel<<<batch, kSmallThreads, smem, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_maxcut_q(double *q, uint64_t count, uint64_t offset, int m, const int32_t *u,
                            const int32_t *v, const double *w, cudaStream_t s) {
    maxcut_q_kernel<<<grid_for(count, 256), 256, 0, s>>>(q, count, offset, m, u, v, w);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_chunk_transpose(T *out, const T *in, int G, uint64_t C, cudaStream_t s) {
    chunk_transpose_kernel<T><<<grid_for((uint64_t)G * G * C, 256), 256, 0, s>>>(out, in, G, C);
    return cudaGetLastError();
}
template cudaError_t launch_chunk_transpose<double2>(double2 *, const double2 *, int, uint64_t, cudaStream_t);
template cudaError_t launch_chunk_transpose<double>(double *, const double *, int, uint64_t, cudaStream_t);

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
