// Which configurations let a small kernel run beside a persistent
// 544-thread, ~166 KB-smem kernel (the Gram's shape) on every SM?
// Kernel A (148 CTAs) spins until kernel B (launched after it on another
// stream) raises a flag, or gives up after 2 s; prints the outcome.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(544, 1) big_kernel(volatile int* flag, int* timed_out) {
    extern __shared__ double sm[];
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (threadIdx.x == 0) {
        do {
            __nanosleep(1000);
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        } while (*flag == 0 && t - t0 < 2000000000ull);
        if (*flag == 0) atomicAdd(timed_out, 1);
    }
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
}

__global__ void __launch_bounds__(128) small_kernel(int* flag) {
    if (threadIdx.x == 0) atomicAdd(flag, 1);
}

int main() {
    int *flag, *to;
    cudaMallocManaged(&flag, 4);
    cudaMallocManaged(&to, 4);
    cudaStream_t a, b;
    cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    const int smems[] = {165888, 150000, 120000, 100000};
    const int carves[] = {-1, 100};
    for (int smem : smems) {
        for (int ca : carves) {
            for (int cb : carves) {
                *flag = 0;
                *to = 0;
                cudaFuncSetAttribute(big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                if (ca >= 0) cudaFuncSetAttribute(big_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, ca);
                if (cb >= 0) cudaFuncSetAttribute(small_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cb);
                big_kernel<<<148, 544, smem, a>>>(flag, to);
                small_kernel<<<148, 128, 0, b>>>(flag);
                cudaDeviceSynchronize();
                printf("smem %6d carve big %4d small %4d: %s (%d CTAs timed out) err=%s\n", smem, ca, cb,
                       *to ? "NOT co-resident" : "co-resident", *to, cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
    return 0;
}
