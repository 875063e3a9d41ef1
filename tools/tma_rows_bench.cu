// Micro-benchmark: TMA tile round trip (load box -> smem -> contiguous out-of-place store) over a
// 2^30 complex128 array, tile = 4096 amplitudes = rows of 2^r amplitudes (bits 0..r-1) plus a run
// of 12-r window bits starting at bit 12.  Measures how the DRAM efficiency of the strided
// window read depends on the row length (r = 3: 128-B rows as in the X-mixer window passes).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_rows tools/tma_rows_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(32, 1) rt(const __grid_constant__ CUtensorMap m, int wlo, uint64_t n_tiles,
                                            double2 *out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar[4];
    if (threadIdx.x) return;
    for (int s = 0; s < 4; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    const int S = 3;
    // coordinates: dim1 = bits [r, 12) (low coordinate run, wlo bits), dim4 = bits [12 + (12 - r), 30)
    auto load = [&](uint64_t t, int s) {
        int c1 = (int)(t & ((1ull << wlo) - 1)), c4 = (int)(t >> wlo);
        uint32_t b = su(&bar[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(65536));
        asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     ::"r"(su(sm + s * 65536)), "l"((uint64_t)&m), "r"(0), "r"(c1), "r"(0), "r"(0), "r"(c4), "r"(b) : "memory");
    };
    uint32_t it = 0;
    for (int k = 0; k < S; ++k)
        if (blockIdx.x + (uint64_t)k * gridDim.x < n_tiles) load(blockIdx.x + (uint64_t)k * gridDim.x, k);
    for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
        int s = it % S;
        uint32_t b = su(&bar[s]), ok = 0, par = (it / S) & 1;
        while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(b), "r"(par) : "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 65536;" ::"l"(out + t * 4096),
                     "r"(su(sm + s * 65536)) : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
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
    cudaMemset(psi, 0, (1ull << n) * 16);
    cudaFuncSetAttribute(rt, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536);
    for (int rep = 0; rep < 2; ++rep)
        for (int r = 3; r <= 7; ++r) {
            // dims: d0 = 2^r amps (row, as doubles, split: d0 16 doubles max for swizzle none -> use no swizzle)
            // d0: row of 2^r amplitudes = 2^(r+1) doubles (box <= 256), d1: coordinate bits [r, 12) (box 1),
            // d2: window bits [12, 12 + min(8, 12-r)) , d3: remaining window bits, d4: coordinate bits above
            int wb = 12 - r, w2 = wb > 8 ? 8 : wb, w3 = wb - w2;
            cuuint64_t gd[5] = {(cuuint64_t)2 << r, 1ull << (12 - r), 1ull << w2, 1ull << w3, 1ull << (n - 12 - wb)};
            cuuint64_t gs[4] = {(cuuint64_t)16 << r, (cuuint64_t)16 << 12, (cuuint64_t)16 << (12 + w2),
                                (cuuint64_t)16 << (12 + wb)};
            cuuint32_t bx[5] = {(cuuint32_t)(2 << r), 1, (cuuint32_t)(1 << w2), (cuuint32_t)(1 << w3), 1};
            cuuint32_t es[5] = {1, 1, 1, 1, 1};
            CUtensorMap m;
            CUresult res = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, psi, gd, gs, bx, es,
                                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (res) { printf("encode failed %d (r=%d)\n", res, r); continue; }
            uint64_t nt = 1ull << (n - 12);
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            rt<<<148, 32, 3 * 65536>>>(m, 12 - r, nt, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("rows of %4d B (r=%d), window at bit 12: %.3f ms  %.0f GB/s  %s\n", 16 << r, r, ms,
                   (double)(1ull << n) * 32 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
