// Per-SM streaming rate of an in-place (x - m) / s pass with deep TMA bulk
// rings (follow-up to sm_stream.cu): one CTA per SM, NS stages of CH bytes in
// shared memory, cp.async.bulk loads completing on an mbarrier per stage,
// compute in shared memory (exact IEEE quotient via fl(1/s) + Markstein
// correction, or the division itself), cp.async.bulk stores; a stage is
// refilled once its store has read it. Prints GB/s (read + write) for G SMs.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int NS, int CH, int THREADS, bool DIV>
__global__ void __launch_bounds__(THREADS, 1) bulk(double* q, size_t n, double m, double s) {
    extern __shared__ __align__(128) unsigned char raw[];
    double* buf = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
    __shared__ __align__(8) uint64_t full[NS];
    const size_t per = n / gridDim.x;
    double* base = q + per * blockIdx.x;
    const size_t nch = per * 8 / CH;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&full[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    auto issue = [&](size_t c) {
        const int st = c % NS;
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(CH));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(buf + st * (CH / 8))),
                     "l"(base + c * (CH / 8)), "r"(CH), "r"(su32(&full[st]))
                     : "memory");
    };
    if (threadIdx.x == 0)
        for (size_t c = 0; c < NS - 1 && c < nch; ++c) issue(c);
    const double rs = 1.0 / s, nm = -m;
    for (size_t c = 0; c < nch; ++c) {
        const int st = c % NS;
        const uint32_t par = (c / NS) & 1;
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(
                         su32(&full[st])),
                     "r"(par)
                     : "memory");
        double2* b = reinterpret_cast<double2*>(buf + st * (CH / 8));
        for (int i = threadIdx.x; i < CH / 16; i += THREADS) {
            double2 v = b[i];
            double x0 = v.x + nm, x1 = v.y + nm;
            if (DIV) {
                v.x = x0 / s;
                v.y = x1 / s;
            } else {
                double q0 = x0 * rs, q1 = x1 * rs;
                q0 = fma(fma(-q0, s, x0), rs, q0);
                q1 = fma(fma(-q1, s, x1), rs, q1);
                v.x = q0;
                v.y = q1;
            }
            b[i] = v;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(base + c * (CH / 8)),
                         "r"(su32(b)), "r"(CH)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;");
            // refill the stage stored at c - 1 (= (c + NS - 1) % NS): wait until that store read its smem
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            if (c + NS - 1 < nch) issue(c + NS - 1);
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int U, int THREADS>
__global__ void __launch_bounds__(THREADS) ldst(double* q, size_t n, double m, double s) {
    const size_t per = n / gridDim.x;
    double2* p = reinterpret_cast<double2*>(q + per * blockIdx.x);
    const size_t n2 = per / 2;
    const double rs = 1.0 / s, nm = -m;
    for (size_t i = threadIdx.x; i < n2; i += size_t(THREADS) * U) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t k = i + size_t(u) * THREADS;
            if (k < n2) v[u] = __ldcs(p + k);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t k = i + size_t(u) * THREADS;
            double x0 = v[u].x + nm, x1 = v[u].y + nm;
            double q0 = x0 * rs, q1 = x1 * rs;
            q0 = fma(fma(-q0, s, x0), rs, q0);
            q1 = fma(fma(-q1, s, x1), rs, q1);
            if (k < n2) __stcs(p + k, make_double2(q0, q1));
        }
    }
}

template <class F>
void run(const char* name, F launch, double* q, int smem_per_sm_blocks) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int g : {4, 8}) {
        const size_t elems = size_t(g) * (size_t(1) << 25);  // 256 MiB per SM
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            launch(g * smem_per_sm_blocks, elems);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        printf("%-28s G=%d  %7.1f GB/s per SM  (%s)\n", name, g, 2.0 * elems * 8 / (best * 1e-3) / 1e9 / g,
               cudaGetErrorString(cudaGetLastError()));
    }
}

template <int NS, int CH, int T, bool DIV>
void bulk_case(const char* name, double* q) {
    const int smem = NS * CH + 256;
    cudaFuncSetAttribute(bulk<NS, CH, T, DIV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    run(name, [&](int blocks, size_t e) { bulk<NS, CH, T, DIV><<<blocks, T, smem>>>(q, e, 1.5, 3.0); }, q, 1);
}

int main() {
    const size_t n = size_t(1) << 28;  // 2 GiB
    double* q;
    if (cudaMalloc(&q, n * 8) != cudaSuccess) return 1;
    cudaMemset(q, 0, n * 8);
    bulk_case<4, 32768, 512, false>("bulk 4x32K markstein", q);
    bulk_case<6, 32768, 512, false>("bulk 6x32K markstein", q);
    bulk_case<4, 49152, 512, false>("bulk 4x48K markstein", q);
    bulk_case<8, 24576, 512, false>("bulk 8x24K markstein", q);
    bulk_case<6, 32768, 1024, false>("bulk 6x32K markstein T1024", q);
    bulk_case<6, 32768, 512, true>("bulk 6x32K ieee-div", q);
    run("ldst U8 T1024 x1", [&](int blocks, size_t e) { ldst<8, 1024><<<blocks, 1024>>>(q, e, 1.5, 3.0); }, q, 1);
    run("ldst U8 T512 x2", [&](int blocks, size_t e) { ldst<8, 512><<<blocks, 512>>>(q, e, 1.5, 3.0); }, q, 2);
    run("ldst U4 T1024 x2", [&](int blocks, size_t e) { ldst<4, 1024><<<blocks, 1024>>>(q, e, 1.5, 3.0); }, q, 2);
    return 0;
}
