// kernels_sparse.cu -- generic sparse mixer exp(-i beta W) psi for a real symmetric CSR W
// (PAPER.md:72-77 Eq. 4; Sec. 3 "a variant of the scaling and squaring algorithm", :333),
// applied as s sub-steps of a truncated Taylor series (reading R13):
//   s = max(1, ceil(|beta| ||W||_1 / 3)),  h = beta / s,
//   per sub-step: F = v; T_0 = v; T_k = (-i h / k) W T_{k-1}; F += T_k
//   stop when ||T_k||_inf + ||T_{k-1}||_inf <= 2^-53 ||F||_inf (at most 40 terms).
// The SpMV, the Taylor-term scaling, the accumulation into F and the inf-norms are one kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "qva_internal.h"

namespace qva {

namespace {

constexpr int kSpmvThreads = 256;
constexpr int kMaxTerms = 40;

__device__ __forceinline__ void block_max2(double &a, double &b, double *red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
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
            sa = fmax(sa, red[2 * w]);
            sb = fmax(sb, red[2 * w + 1]);
        }
        a = sa;
        b = sb;
    }
}

// entry c of the term vector: local (one shard), a peer's IPC-mapped slice, or the gathered copy
__device__ __forceinline__ double2 term_entry(const double2 *__restrict__ t_in, const SpmvSource &S, int which,
                                              uint64_t c) {
    if (S.G == 1) return __ldg(t_in + c);
    int r = 0;
#pragma unroll
    for (int k = 1; k < kMaxPeers; ++k) r += (k < S.G && c >= S.off[k]) ? 1 : 0;
    const uint64_t l = c - S.off[r];
    if (S.gathered) return __ldg(S.gathered + (uint64_t)r * S.stride + l);
    return S.peer[which][r][l];  // NVLink / same-device peer read (not through the read-only path)
}

// t_out = (-i h/k) W t_in ; F += t_out ; per-block (|t_out|_inf, |F|_inf).  Rows are this rank's
// rows; columns are global indices (row-partitioned W: remote entries read from the peers).
__global__ void __launch_bounds__(kSpmvThreads)
spmv_taylor_kernel(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                   const double *__restrict__ val, const double2 *__restrict__ t_in, double2 *__restrict__ t_out,
                   double2 *__restrict__ F, uint64_t rows, double coef, double *__restrict__ scratch,
                   const __grid_constant__ SpmvSource S, int which) {
    __shared__ double red[2 * (kSpmvThreads / 32)];
    double mt = 0.0, mf = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double ar = 0.0, ai = 0.0;
        const int64_t e = row_ptr[i + 1];
        for (int64_t k = row_ptr[i]; k < e; ++k) {
            double w = val ? __ldg(val + k) : 1.0;
            double2 x = term_entry(t_in, S, which, (uint64_t)__ldg(col + k));
            ar = fma(w, x.x, ar);
            ai = fma(w, x.y, ai);
        }
        // -i coef (ar + i ai) = coef*ai - i coef*ar
        double2 t = make_double2(coef * ai, -coef * ar);
        t_out[i] = t;
        double2 f = F[i];
        f.x += t.x;
        f.y += t.y;
        F[i] = f;
        mt = fmax(mt, fmax(fabs(t.x), fabs(t.y)));
        mf = fmax(mf, fmax(fabs(f.x), fabs(f.y)));
    }
    block_max2(mt, mf, red);
    if (threadIdx.x == 0) {
        scratch[2 * blockIdx.x] = mt;
        scratch[2 * blockIdx.x + 1] = mf;
    }
}

__global__ void max_reduce_kernel(const double *scratch, int n, double *out) {
    __shared__ double red[64];
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        a = fmax(a, scratch[2 * i]);
        b = fmax(b, scratch[2 * i + 1]);
    }
    block_max2(a, b, red);
    if (threadIdx.x == 0) {
        out[0] = a;
        out[1] = b;
    }
}

__global__ void inf_norm_kernel(const double2 *v, uint64_t n, double *scratch) {
    __shared__ double red[2 * (kSpmvThreads / 32)];
    double m = 0.0, dummy = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        m = fmax(m, fmax(fabs(v[i].x), fabs(v[i].y)));
    block_max2(m, dummy, red);
    if (threadIdx.x == 0) {
        scratch[2 * blockIdx.x] = m;
        scratch[2 * blockIdx.x + 1] = m;
    }
}

}  // namespace

qva_status sparse_apply_mixer(SparseMixer &sm, double2 *psi, double beta, cudaStream_t s, LaunchObserver *obs,
                              int *terms_used, SparseComm *comm) {
    *terms_used = 0;
    if (beta == 0.0 || (sm.rows == 0 && !comm)) return QVA_OK;
    const uint64_t rows = sm.rows;
    int blocks = (int)std::min<uint64_t>((rows + kSpmvThreads - 1) / kSpmvThreads, (uint64_t)num_sms() * 8);
    if (blocks < 1) blocks = 1;
    if (sm.scratch_blocks < blocks) {
        cudaFree(sm.scratch);
        sm.scratch = nullptr;
        QVA_CUDA_TRY(cudaMalloc(&sm.scratch, (blocks * 2 + 2) * sizeof(double)));
        sm.scratch_blocks = blocks;
    }
    double *d_out = sm.scratch + 2 * blocks;
    const double bnorm = fabs(beta) * sm.norm1;
    const int nsub = std::max(1, (int)std::ceil(bnorm / 3.0));
    const double h = beta / nsub;
    const double eps = std::ldexp(1.0, -53);
    const double bytes_per_spmv =
        (double)sm.nnz * (4.0 + (sm.val ? 8.0 : 0.0) + 16.0) + (double)rows * (8.0 + 16.0 + 32.0);
    for (int sub = 0; sub < nsub; ++sub) {
        // T_0 = v
        QVA_CUDA_TRY(cudaMemcpyAsync(sm.t0, psi, rows * sizeof(double2), cudaMemcpyDeviceToDevice, s));
        obs->begin(K_OTHER, 16.0 * rows);
        inf_norm_kernel<<<blocks, kSpmvThreads, 0, s>>>(psi, rows, sm.scratch);
        max_reduce_kernel<<<1, 1024, 0, s>>>(sm.scratch, blocks, d_out);
        obs->end();
        double host[2];
        QVA_CUDA_TRY(cudaMemcpyAsync(host, d_out, sizeof(host), cudaMemcpyDeviceToHost, s));
        QVA_CUDA_TRY(cudaStreamSynchronize(s));
        // row-partitioned W: the global maxima; the collective also orders every rank's T_0 copy
        // before any rank's first SpMV reads it (and, below, term k's writes before term k+1's reads)
        if (comm) QVA_TRY(comm->max2(host));
        double prev = host[0];
        bool converged = false;
        double2 *tin = sm.t0, *tout = sm.t1;
        int which = 0;  // tin is buffer t0 (0) or t1 (1) on every rank
        for (int k = 1; k <= kMaxTerms; ++k) {
            if (comm && sm.src.gathered) QVA_TRY(comm->gather(tin, sm.gather_buf, sm.src.stride));
            obs->begin(K_SPMV, bytes_per_spmv);
            spmv_taylor_kernel<<<blocks, kSpmvThreads, 0, s>>>(sm.row_ptr, sm.col, sm.val, tin, tout, psi, rows,
                                                               h / k, sm.scratch, sm.src, which);
            max_reduce_kernel<<<1, 1024, 0, s>>>(sm.scratch, blocks, d_out);
            obs->end();
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) {
                set_error(std::string("spmv_taylor_kernel: ") + cudaGetErrorString(e));
                return QVA_ERR_CUDA;
            }
            QVA_CUDA_TRY(cudaMemcpyAsync(host, d_out, sizeof(host), cudaMemcpyDeviceToHost, s));
            QVA_CUDA_TRY(cudaStreamSynchronize(s));
            if (comm) QVA_TRY(comm->max2(host));
            ++*terms_used;
            if (!std::isfinite(host[0]) || !std::isfinite(host[1])) {
                set_error("Taylor action produced non-finite values");
                return QVA_ERR_NUMERIC;
            }
            if (host[0] + prev <= eps * host[1]) {
                converged = true;
                break;
            }
            prev = host[0];
            std::swap(tin, tout);
            which ^= 1;
        }
        if (!converged) {
            set_error("truncated Taylor action did not converge in 40 terms");
            return QVA_ERR_NUMERIC;
        }
    }
    return QVA_OK;
}

}  // namespace qva
