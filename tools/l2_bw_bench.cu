// L2-resident vs HBM-resident streaming bandwidth (read + write bytes / time) on one B200.
// Question it answers: can an in-L2 sub-pass (block of the state kept in L2 between two
// rotation sub-passes) run faster than an HBM pass?  Copy src -> dst of `bytes` each, repeated;
// L2 regime when 2*bytes fits the 126 MB L2.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void copy_kernel(const double4 *__restrict__ a, double4 *__restrict__ b, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i < n; i += stride) {
        double4 v = a[i];
        v.x += 1.0;
        b[i] = v;
    }
}
// in place (read-modify-write the same buffer), the in-L2 sub-pass pattern
__global__ void rmw_kernel(double4 *__restrict__ a, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i < n; i += stride) {
        double4 v = a[i];
        v.x += 1.0;
        a[i] = v;
    }
}
int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int l2;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
    printf("SMs %d L2 %d bytes\n", sms, l2);
    size_t maxb = (size_t)4 << 30;
    char *A, *B;
    cudaMalloc(&A, maxb);
    cudaMalloc(&B, maxb);
    cudaMemset(A, 0, maxb);
    cudaMemset(B, 0, maxb);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    size_t sizes[] = {4u << 20, 8u << 20, 16u << 20, 24u << 20, 32u << 20, 48u << 20, 64u << 20, 96u << 20,
                      128u << 20, 256u << 20, (size_t)1 << 30, (size_t)4 << 30};
    for (int mode = 0; mode < 2; ++mode)
        for (size_t bytes : sizes) {
            size_t n = bytes / sizeof(double4);
            int grid = sms * 8;
            int reps = (int)(((size_t)32 << 30) / bytes);
            if (reps < 3) reps = 3;
            if (reps > 2000) reps = 2000;
            for (int w = 0; w < 3; ++w) {
                if (mode == 0) copy_kernel<<<grid, 512>>>((double4 *)A, (double4 *)B, n);
                else rmw_kernel<<<grid, 512>>>((double4 *)A, n);
            }
            cudaEventRecord(e0);
            for (int r = 0; r < reps; ++r) {
                if (mode == 0) copy_kernel<<<grid, 512>>>((double4 *)A, (double4 *)B, n);
                else rmw_kernel<<<grid, 512>>>((double4 *)A, n);
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double gbs = 2.0 * bytes * reps / (ms * 1e-3) / 1e9;
            printf("%s %8.1f MB  reps %5d  %.3f ms/rep  %.1f GB/s\n", mode == 0 ? "copy" : "rmw ", bytes / 1048576.0,
                   reps, ms / reps, gbs);
        }
    return 0;
}
