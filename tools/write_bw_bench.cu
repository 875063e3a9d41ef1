// Write-only HBM bandwidth on one B200 (the ceiling of the write-only init tile pass): 16 GiB
// written with 16-B stores (grid-stride), and with cudaMemsetAsync, vs read-only and copy.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void write_kernel(double2 *__restrict__ a, size_t n, double v) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
    for (; i < n; i += stride) a[i] = make_double2(v, (double)i);
}
__global__ void read_kernel(const double2 *__restrict__ a, size_t n, double *out) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
    double s = 0.0;
    for (; i < n; i += stride) s += a[i].x;
    if (s == 12345.678) *out = s;
}
int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    size_t bytes = (size_t)16 << 30, n = bytes / 16;
    double2 *a;
    double *o;
    cudaMalloc(&a, bytes);
    cudaMalloc(&o, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; ++mode)
        for (int blocksPerSm : {4, 8, 16}) {
            for (int r = 0; r < 4; ++r) {
                if (r == 1) cudaEventRecord(e0);
                if (mode == 0) write_kernel<<<sms * blocksPerSm, 512>>>(a, n, 1.0);
                else if (mode == 1) read_kernel<<<sms * blocksPerSm, 512>>>(a, n, o);
                else cudaMemsetAsync(a, 0, bytes);
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            ms /= 3;
            printf("%s blocks/SM %2d: %.3f ms  %.1f GB/s\n", mode == 0 ? "write " : mode == 1 ? "read  " : "memset", blocksPerSm,
                   ms, bytes / (ms * 1e-3) / 1e9);
            if (mode == 2) break;
        }
    return 0;
}
