// Write-only and read-only HBM bandwidth on all SMs (the field kernel writes
// 8 bytes per output and reads almost nothing; the copy figure in
// MEASURED_PEAKS.json is read + write). 16 GiB buffer, best of 5.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void write_kernel(double2* p, size_t n2, double v) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n2; i += size_t(gridDim.x) * blockDim.x)
        __stcs(p + i, make_double2(v, v));
}
__global__ void read_kernel(const double2* p, size_t n2, double* sink) {
    double acc = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n2; i += size_t(gridDim.x) * blockDim.x) {
        const double2 v = __ldcs(p + i);
        acc += v.x + v.y;
    }
    if (acc == 12345.0) *sink = acc;
}
__global__ void copy_kernel(const double2* a, double2* b, size_t n2) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n2; i += size_t(gridDim.x) * blockDim.x)
        __stcs(b + i, __ldcs(a + i));
}

int main() {
    const size_t bytes = size_t(16) << 30;
    double2* p;
    double* sink;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return 1;
    cudaMalloc(&sink, 8);
    cudaMemset(p, 0, bytes);
    const size_t n2 = bytes / 16;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int blocks_per_sm : {2, 4, 8}) {
        for (int kind = 0; kind < 4; ++kind) {
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(a);
                if (kind == 0) write_kernel<<<sms * blocks_per_sm, 1024>>>(p, n2, 1.0);
                if (kind == 1) read_kernel<<<sms * blocks_per_sm, 1024>>>(p, n2, sink);
                if (kind == 2) copy_kernel<<<sms * blocks_per_sm, 1024>>>(p, p + n2 / 2, n2 / 2);
                if (kind == 3) cudaMemsetAsync(p, 1, bytes);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                best = ms < best ? ms : best;
            }
            const char* name[] = {"write-only", "read-only", "copy (r+w)", "cudaMemset"};
            const double moved = kind == 2 ? double(bytes) : double(bytes);
            printf("%-11s blocks/SM %d: %.1f GB/s\n", name[kind], blocks_per_sm, moved / (best * 1e-3) / 1e9);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
