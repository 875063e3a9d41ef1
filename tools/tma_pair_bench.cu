// Micro-benchmark: do two CTAs of a cluster whose TMA tile loads are issued together (by the
// leader, into both CTAs' shared memory) read 128-B-row strided tiles as efficiently as one CTA
// reading 256-B rows?  Tile = bits 0..2 (128-B rows) + window bits 12..20; CTA pair = adjacent
// tiles (bit 3).  Mode 0: each CTA issues its own loads; mode 1: leader issues both.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_pair_bench tools/tma_pair_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.aligned;\n barrier.cluster.wait.aligned;" ::: "memory");
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32, 1)
rt(const __grid_constant__ CUtensorMap m, uint64_t n_tiles, double2 *out, int mode) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t full[3], empty[3];
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int S = 3;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    cluster_sync();
    if (threadIdx.x == 0) {
    const uint64_t cl = blockIdx.x / 2, ncl = gridDim.x / 2;
    const uint64_t n_pairs = n_tiles / 2;
    // CTA `rank` of cluster cl handles tile 2p + rank of pairs p = cl, cl + ncl, ...
    auto load_into = [&](uint64_t t, int s, uint32_t dst_rank) {
        int c1 = (int)(t & 511), c4 = (int)(t >> 9);
        uint32_t dst = su(sm + s * 65536), bar = su(&full[s]);
        if (dst_rank != rank) { dst = mapa(dst, dst_rank); bar = mapa(bar, dst_rank); }
        asm volatile("mbarrier.expect_tx.relaxed.cluster.shared::cluster.b64 [%0], %1;" ::"r"(bar), "r"(65536) : "memory");
        asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     ::"r"(dst), "l"((uint64_t)&m), "r"(0), "r"(c1), "r"(0), "r"(0), "r"(c4), "r"(bar) : "memory");
    };
    auto arrive_full_self = [&](int s) {  // the expect_tx above is not an arrival: add the one arrival
        (void)s;
    };
    (void)arrive_full_self;
    uint32_t it = 0;
    uint64_t n_it = (cl < n_pairs) ? (n_pairs - cl + ncl - 1) / ncl : 0;
    auto issue = [&](uint64_t j) {
        uint64_t p = cl + j * ncl;
        int s = j % S;
        if (mode == 0) {
            load_into(2 * p + rank, s, rank);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&full[s])) : "memory");
        } else if (rank == 0) {
            load_into(2 * p, s, 0);
            load_into(2 * p + 1, s, 1);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&full[s])) : "memory");
            uint32_t rb = mapa(su(&full[s]), 1);
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
        }
    };
    for (uint64_t j = 0; j < (uint64_t)S && j < n_it; ++j) issue(j);
    for (uint64_t j = 0; j < n_it; ++j, ++it) {
        int s = j % S;
        uint32_t b = su(&full[s]), ok = 0, par = (j / S) & 1;
        while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(b), "r"(par) : "memory");
        uint64_t t = 2 * (cl + j * ncl) + rank;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 65536;" ::"l"(out + t * 4096),
                     "r"(su(sm + s * 65536)) : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        if (j + S < n_it) {
            if (mode == 0) {
                issue(j + S);
            } else {
                // stage s free here: tell the leader (empty[s] on rank 0), leader waits for both
                uint32_t eb = mapa(su(&empty[s]), 0);
                if (rank == 1) asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(eb) : "memory");
                if (rank == 0) {
                    uint32_t ok2 = 0, par2 = (j / S) & 1;
                    uint32_t e0 = su(&empty[s]);
                    while (!ok2) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok2) : "r"(e0), "r"(par2) : "memory");
                    issue(j + S);
                }
            }
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    cluster_sync();
}
int main() {
    const int n = 30;
    double2 *psi, *out;
    cudaMalloc(&psi, (1ull << n) * 16);
    cudaMalloc(&out, (1ull << n) * 16);
    cudaMemset(psi, 0, (1ull << n) * 16);
    cudaFuncSetAttribute(rt, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536);
    // tile: d0 = bits 0..2 (16 doubles), d1 = bits 3..11 (coordinate, box 1), d2 = bits 12..19, d3 = bit 20,
    // d4 = bits 21..29 (coordinate)
    cuuint64_t gd[5] = {16, 512, 256, 2, 512};
    cuuint64_t gs[4] = {128, 16ull << 12, 16ull << 20, 16ull << 21};
    cuuint32_t bx[5] = {16, 1, 256, 2, 1}, es[5] = {1, 1, 1, 1, 1};
    CUtensorMap m;
    CUresult res = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, psi, gd, gs, bx, es,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res) { printf("encode failed %d\n", res); return 1; }
    for (int rep = 0; rep < 3; ++rep)
        for (int mode = 0; mode < 2; ++mode) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            rt<<<148, 32, 3 * 65536>>>(m, 1ull << 18, out, mode);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("mode %d (%s): %.3f ms  %.0f GB/s  %s\n", mode, mode ? "leader issues the pair" : "independent", ms,
                   (double)(1ull << n) * 32 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
