// How fast can G dedicated SMs stream an in-place (x - m) / s pass over HBM?
// (Sizing a transform kernel that runs on a few SMs beside a Gram kernel on
// the rest.) One CTA per SM (forced by the shared-memory request); each CTA
// owns a contiguous slice. Variants:
//   ldst-copy / ldst-div / ldst-rcp : 1024 threads, 8 x 16-byte loads in flight
//                                     per thread, then compute + store
//   bulk-div                         : cp.async.bulk 32 KB chunks into a 4-stage
//                                     smem ring (one elected thread), 1024
//                                     threads compute in smem, cp.async.bulk
//                                     store back
// Prints GB/s (read + write bytes) per G.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kThreads = 1024;

template <int MODE>
__device__ __forceinline__ double op(double x, double m, double s, double rs) {
    if (MODE == 0) return x;
    if (MODE == 1) return (x - m) / s;
    return (x - m) * rs;
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) ldst(double* q, size_t n, double m, double s) {
    extern __shared__ double pad[];
    const size_t per = n / gridDim.x;
    double2* p = reinterpret_cast<double2*>(q + per * blockIdx.x);
    const size_t n2 = per / 2;
    const double rs = 1.0 / s;
    constexpr int U = 8;
    for (size_t i = threadIdx.x; i < n2; i += size_t(kThreads) * U) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t k = i + size_t(u) * kThreads;
            if (k < n2) v[u] = __ldcs(p + k);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t k = i + size_t(u) * kThreads;
            if (k < n2) __stcs(p + k, make_double2(op<MODE>(v[u].x, m, s, rs), op<MODE>(v[u].y, m, s, rs)));
        }
    }
    if (threadIdx.x == 0 && per == 0) pad[0] = 0;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

constexpr int kStages = 4;
constexpr int kChunk = 32768;  // bytes

__global__ void __launch_bounds__(kThreads, 1) bulk(double* q, size_t n, double m, double s) {
    extern __shared__ __align__(128) unsigned char raw[];
    double* buf = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
    __shared__ __align__(8) uint64_t full[kStages];
    const size_t per = n / gridDim.x;
    double* base = q + per * blockIdx.x;
    const size_t nch = per * 8 / kChunk;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i)
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&full[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    auto issue = [&](size_t c) {
        const int st = c % kStages;
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(kChunk));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(buf + st * (kChunk / 8))),
            "l"(base + c * (kChunk / 8)), "r"(kChunk), "r"(su32(&full[st]))
            : "memory");
    };
    if (threadIdx.x == 0)
        for (size_t c = 0; c < kStages - 1 && c < nch; ++c) issue(c);
    const double rs = 1.0 / s;
    for (size_t c = 0; c < nch; ++c) {
        const int st = c % kStages;
        const uint32_t par = (c / kStages) & 1;
        asm volatile(
            "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(
                su32(&full[st])),
            "r"(par)
            : "memory");
        double* b = buf + st * (kChunk / 8);
        for (int i = threadIdx.x; i < kChunk / 8; i += kThreads) b[i] = (b[i] - m) / s;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(base + c * (kChunk / 8)),
                         "r"(su32(b)), "r"(kChunk)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;");
            // the stage refilled next (c + kStages - 1) was stored at c - 1: wait for that store's smem read
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            if (c + kStages - 1 < nch) issue(c + kStages - 1);
        }
        (void)rs;
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const size_t n = size_t(1) << 29;  // 4 GiB of doubles
    double* q;
    if (cudaMalloc(&q, n * 8) != cudaSuccess) return 1;
    cudaMemset(q, 0, n * 8);
    const int smem = 150 * 1024;
    cudaFuncSetAttribute(ldst<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(ldst<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(ldst<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int gs[] = {1, 2, 4, 8, 16, 32, 148};
    const char* names[] = {"ldst-copy", "ldst-div", "ldst-rcp", "bulk-div"};
    for (int v = 0; v < 4; ++v) {
        for (int g : gs) {
            // bytes: a slice per CTA, capped so one run stays short
            const size_t elems = std::min<size_t>(n, size_t(g) * (size_t(1) << 25));
            float best = 1e30f;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(a);
                if (v == 0) ldst<0><<<g, kThreads, smem>>>(q, elems, 1.5, 3.0);
                if (v == 1) ldst<1><<<g, kThreads, smem>>>(q, elems, 1.5, 3.0);
                if (v == 2) ldst<2><<<g, kThreads, smem>>>(q, elems, 1.5, 3.0);
                if (v == 3) bulk<<<g, kThreads, smem>>>(q, elems, 1.5, 3.0);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            const cudaError_t e = cudaGetLastError();
            printf("%-10s G=%3d  %8.1f GB/s total  %6.1f GB/s per SM  (%s)\n", names[v], g,
                   2.0 * elems * 8 / (best * 1e-3) / 1e9, 2.0 * elems * 8 / (best * 1e-3) / 1e9 / g,
                   cudaGetErrorString(e));
        }
    }
    return 0;
}
