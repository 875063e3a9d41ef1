// Micro-benchmark: TMA tile round trip (load box -> smem -> store box, no compute) over a 2^n
// complex128 array for the three tile shapes of the X-mixer passes.  Isolates the memory-system
// cost of strided 128-B-row tiles.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(32, 1) rt(const __grid_constant__ CUtensorMap m, int dims_w0, int dims_w1, int d0, int d1,
                                              uint64_t n_tiles, int mode, double2 *out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar[4];
    if (threadIdx.x) return;
    for (int s = 0; s < 4; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    uint32_t it = 0;
    auto coords = [&](uint64_t t, int (&c)[5]) {
        for (int d = 0; d < 5; ++d) c[d] = 0;
        c[d0] = (int)(t & ((1ull << dims_w0) - 1));
        c[d1] = (int)(t >> dims_w0);
    };
    auto load = [&](uint64_t t, int s) {
        int c[5];
        coords(t, c);
        uint32_t b = su(&bar[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(65536));
        asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     ::"r"(su(sm + s * 65536)), "l"((uint64_t)&m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(b) : "memory");
    };
    const int S = 3;
    uint64_t t0 = blockIdx.x;
    for (int k = 0; k < S; ++k)
        if (t0 + (uint64_t)k * gridDim.x < n_tiles) load(t0 + (uint64_t)k * gridDim.x, k);
    for (uint64_t t = t0; t < n_tiles; t += gridDim.x, ++it) {
        int s = it % S;
        uint32_t b = su(&bar[s]), ok = 0, par = (it / S) & 1;
        while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(b), "r"(par) : "memory");
        if (mode == 2) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 65536;" ::"l"(out + t * 4096),
                         "r"(su(sm + s * 65536)) : "memory");
            asm volatile("cp.async.bulk.commit_group;");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        if (mode == 1) {
            int c[5];
            coords(t, c);
            asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"((uint64_t)&m),
                         "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(su(sm + s * 65536)) : "memory");
            asm volatile("cp.async.bulk.commit_group;");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        uint64_t nt = t + (uint64_t)S * gridDim.x;
        if (nt < n_tiles) load(nt, s);
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
int main() {
    const int n = 30;
    double2 *psi, *out;
    cudaMalloc(&psi, (1ull << n) * 16);
    cudaMalloc(&out, (1ull << n) * 16);
    cudaMemset(out, 0, (1ull << n) * 16);
    cudaMemset(psi, 0, (1ull << n) * 16);
    cudaFuncSetAttribute(rt, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536);
    // shapes: tile bits {0,1,2} + hi run [a, a+9) (a = 3 -> contiguous 12-bit tile)
    int as[4] = {3, 12, 21, 16};
    for (int mode = 0; mode < 3; ++mode)
        for (int k = 0; k < 4; ++k) {
            int a = as[k];
            // dims: [0-2] 16 dbl, [3, a) nontile (if a>3), [a, a+8) tile, [a+8] tile, [a+9, n) nontile
            cuuint64_t gd[5]; cuuint64_t gs[4]; cuuint32_t bx[5], es[5] = {1, 1, 1, 1, 1};
            int d = 0, w0 = 0, w1 = 0, d0 = 0, d1 = 0;
            gd[0] = 16; bx[0] = 16; d = 1;
            if (a > 3) { gd[d] = 1ull << (a - 3); bx[d] = 1; gs[d - 1] = 128; d0 = d; w0 = a - 3; ++d; }
            gd[d] = 256; bx[d] = 256; gs[d - 1] = (1ull << a) * 16; ++d;
            gd[d] = 2; bx[d] = 2; gs[d - 1] = (1ull << (a + 8)) * 16; ++d;
            int top = n - a - 9;
            gd[d] = 1ull << top; bx[d] = 1; gs[d - 1] = (1ull << (a + 9)) * 16;
            if (a > 3) { d1 = d; } else { d0 = d; w0 = top; d1 = 0; }
            ++d;
            while (d < 5) { gd[d] = 1; bx[d] = 1; gs[d - 1] = 16; ++d; }
            CUtensorMap m;
            CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, psi, gd, gs, bx, es,
                                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r) { printf("encode failed %d\n", r); return 1; }
            uint64_t nt = 1ull << (n - 12);
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(e0);
                rt<<<148, 32, 3 * 65536>>>(m, w0, w1, d0, d1, nt, mode, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double bytes = (double)(1ull << n) * 16 * (mode ? 2 : 1);
            printf("%s hi-run at bit %2d: %.3f ms  %.0f GB/s  (%s)\n",
                   mode == 2 ? "load+contig out-of-place store" : (mode ? "load+in-place store" : "load only "), a, ms, bytes / ms / 1e6,
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
