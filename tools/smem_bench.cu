// Micro-benchmark: shared-memory transpose cost per register group (X, Y, W) of the tile pass.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/smem_bench tools/smem_bench.cu && /tmp/smem_bench
#include <cstdio>
#include <cstdint>
template <int G>
__device__ __forceinline__ uint32_t gbase(uint32_t buf, int c) {
    const uint32_t l = c & 7, h = c >> 3;
    uint32_t a;
    if (G == 0) a = buf + (l << 4) + (h << 12);
    else if (G == 1) a = buf + ((l ^ ((h & 3) << 1)) << 4) + (h << 8);
    else a = buf + (l << 4) + (l << 7) + (h << 12);
    asm volatile("mov.b32 %0, %0;" : "+r"(a));
    return a;
}
template <int G>
__device__ __forceinline__ uint32_t gaddr(uint32_t A, int e) {
    if (G == 0) return (A ^ ((e & 7) << 4)) + (e << 7);
    if (G == 1) return (A ^ ((e >> 4) << 4)) + ((e >> 4) << 7) + ((e & 15) << 12);
    return (A ^ ((e & 7) << 4)) + ((e >> 3) << 10);
}
template <int G>
__global__ void bench(long long *out, int iters, double *sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint32_t buf = (uint32_t)__cvta_generic_to_shared(sm) + (threadIdx.x >> 7) * 65536;
    int c = threadIdx.x & 127;
    double2 v[32];
    for (int e = 0; e < 32; ++e) v[e] = make_double2(e, c);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t A = gbase<G>(buf, c);
#pragma unroll
        for (int e = 0; e < 32; ++e)
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(gaddr<G>(A, e)), "d"(v[e].x), "d"(v[e].y) : "memory");
        asm volatile("bar.sync %0, 128;" ::"r"(1 + (int)(threadIdx.x >> 7)) : "memory");
#pragma unroll
        for (int e = 0; e < 32; ++e)
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[e].x), "=d"(v[e].y) : "r"(gaddr<G>(A, e)) : "memory");
        asm volatile("bar.sync %0, 128;" ::"r"(1 + (int)(threadIdx.x >> 7)) : "memory");
    }
    long long t1 = clock64();
    double s = 0;
    for (int e = 0; e < 32; ++e) s += v[e].x + v[e].y;
    if (s == 12345.678) sink[0] = s;
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
int main() {
    long long *d; double *sink;
    cudaMalloc(&d, 1024 * 8); cudaMalloc(&sink, 8);
    int iters = 2000;
    for (int wgs = 1; wgs <= 2; ++wgs) {
        void (*ks[3])(long long *, int, double *) = {bench<0>, bench<1>, bench<2>};
        for (int g = 0; g < 3; ++g) {
            cudaFuncSetAttribute(ks[g], cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
            ks[g]<<<148, 128 * wgs, 131072>>>(d, iters, sink);
            cudaDeviceSynchronize();
            long long h;
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            // per iteration per warpgroup: 64 KB written + 64 KB read = 1024 wavefronts ideal
            printf("WGs %d group %c: %.0f cycles per (write+read) of a 64 KiB tile per WG (ideal %d)  err=%s\n", wgs,
                   "XYW"[g], (double)h / iters, 1024 * wgs, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
