// eig.cu — §8(f) next-row 1: the eigensolve after the Gram, on the device.
//
// pod::eig_sym_desc (reference proj/src/pod.cpp:20-65) calls LAPACK dsyev on
// the host and then (a) reorders to descending, (b) clamps negatives within
// −1e-10·λ1 to zero (NotPsdError below that), (c) flips each eigenvector so
// its largest-magnitude entry — lowest index on ties — is positive.
// pod::reduced_map (pod.cpp:84-101) then forms T_r = U_r·(1/√λ_r).
// Here: cuSOLVER dsyevd (divide and conquer) on the context's device D, then
// one kernel for (a)+(c) (row-major output, as dopinf::Matrix) and one for
// T_r in the reference's arithmetic (inv = 1/sqrt(λ); t = u·inv). The clamp
// (b) is a host check on the n eigenvalues, as in the reference.
//
// cuSOLVER is loaded lazily with dlopen so that the snapshot pass itself does
// not depend on it; when it is absent the call fails (no CPU fallback).
#include <cusolverDn.h>
#include <dlfcn.h>

#include <algorithm>
#include <mutex>
#include <string>

#include "common.cuh"
#include "eig.h"

namespace dopinf_b200 {
namespace eig {

namespace {

using CreateFn = cusolverStatus_t (*)(cusolverDnHandle_t*);
using DestroyFn = cusolverStatus_t (*)(cusolverDnHandle_t);
using SetStreamFn = cusolverStatus_t (*)(cusolverDnHandle_t, cudaStream_t);
using BufFn = cusolverStatus_t (*)(cusolverDnHandle_t, cusolverEigMode_t, cublasFillMode_t, int, const double*, int,
                                   const double*, int*);
using SyevdFn = cusolverStatus_t (*)(cusolverDnHandle_t, cusolverEigMode_t, cublasFillMode_t, int, double*, int,
                                     double*, double*, int, int*);
using PotrfBufFn = cusolverStatus_t (*)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, int*);
using PotrfFn = cusolverStatus_t (*)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, double*, int, int*);
using PotrsFn = cusolverStatus_t (*)(cusolverDnHandle_t, cublasFillMode_t, int, int, const double*, int, double*, int,
                                     int*);

struct Api {
    void* dl = nullptr;
    CreateFn create = nullptr;
    DestroyFn destroy = nullptr;
    SetStreamFn set_stream = nullptr;
    BufFn buffer_size = nullptr;
    SyevdFn syevd = nullptr;
    PotrfBufFn potrf_buffer_size = nullptr;
    PotrfFn potrf = nullptr;
    PotrsFn potrs = nullptr;
    std::string error;
};

const Api& api() {
    static Api a;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libcusolver.so.11", "/usr/local/cuda/lib64/libcusolver.so.11", "libcusolver.so"};
        for (const char* n : names) {
            a.dl = dlopen(n, RTLD_NOW | RTLD_LOCAL);
            if (a.dl) break;
        }
        if (!a.dl) {
            a.error = std::string("cuSOLVER not found: ") + dlerror();
            return;
        }
        a.create = reinterpret_cast<CreateFn>(dlsym(a.dl, "cusolverDnCreate"));
        a.destroy = reinterpret_cast<DestroyFn>(dlsym(a.dl, "cusolverDnDestroy"));
        a.set_stream = reinterpret_cast<SetStreamFn>(dlsym(a.dl, "cusolverDnSetStream"));
        a.buffer_size = reinterpret_cast<BufFn>(dlsym(a.dl, "cusolverDnDsyevd_bufferSize"));
        a.syevd = reinterpret_cast<SyevdFn>(dlsym(a.dl, "cusolverDnDsyevd"));
        a.potrf_buffer_size = reinterpret_cast<PotrfBufFn>(dlsym(a.dl, "cusolverDnDpotrf_bufferSize"));
        a.potrf = reinterpret_cast<PotrfFn>(dlsym(a.dl, "cusolverDnDpotrf"));
        a.potrs = reinterpret_cast<PotrsFn>(dlsym(a.dl, "cusolverDnDpotrs"));
        if (!a.create || !a.destroy || !a.set_stream || !a.buffer_size || !a.syevd || !a.potrf_buffer_size ||
            !a.potrf || !a.potrs) {
            a.error = "cuSOLVER is missing dsyevd / dpotrf / dpotrs entry points";
        }
    });
    return a;
}

// Column k' of the descending, sign-normalised, row-major result from column
// n-1-k' of dsyevd's column-major output. One block per column.
__global__ void __launch_bounds__(256)
    desc_sign_kernel(const double* __restrict__ a, const double* __restrict__ w, int n, double* __restrict__ v,
                     double* __restrict__ lambda) {
    const int k = blockIdx.x;
    const int src = n - 1 - k;
    const double* col = a + static_cast<size_t>(src) * n;
    // argmax |col[i]|, lowest index on ties (pod.cpp:50-63: strict '>' from best = 0)
    double best = 0.0;
    int pivot = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double m = fabs(col[i]);
        if (m > best) {
            best = m;
            pivot = i;
        }
    }
    __shared__ double sb[256];
    __shared__ int sp[256];
    sb[threadIdx.x] = best;
    sp[threadIdx.x] = pivot;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            const double ob = sb[threadIdx.x + s];
            const int op = sp[threadIdx.x + s];
            if (ob > sb[threadIdx.x] || (ob == sb[threadIdx.x] && op < sp[threadIdx.x])) {
                sb[threadIdx.x] = ob;
                sp[threadIdx.x] = op;
            }
        }
        __syncthreads();
    }
    const bool flip = col[sp[0]] < 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        v[static_cast<size_t>(i) * n + k] = flip ? -col[i] : col[i];
    }
    if (threadIdx.x == 0) lambda[k] = w[src];
}

// pod.cpp:84-101: tr(i, k) = V(i, k) * (1 / sqrt(lambda_k)), k < r.
__global__ void reduced_map_kernel(const double* __restrict__ v, const double* __restrict__ lambda, int n, int r,
                                   double* __restrict__ tr) {
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= static_cast<long long>(n) * r) return;
    const int i = static_cast<int>(e / r), k = static_cast<int>(e % r);
    const double inv_sqrt = 1.0 / sqrt(lambda[k]);
    tr[e] = v[static_cast<size_t>(i) * n + k] * inv_sqrt;
}

// T_rᵀ, zero padded to r_pad rows, pitch ld (the Φ_r kernel's B operand).
__global__ void transpose_pad_kernel(const double* __restrict__ tr, int n, int r, int r_pad, size_t ld,
                                     double* __restrict__ trt) {
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= static_cast<long long>(r_pad) * ld) return;
    const int j = static_cast<int>(e / ld), k = static_cast<int>(e % ld);
    trt[e] = (j < r && k < n) ? tr[static_cast<size_t>(k) * r + j] : 0.0;
}

}  // namespace

const char* unavailable_reason() {
    const Api& a = api();
    return a.error.empty() ? nullptr : a.error.c_str();
}

Solver::~Solver() {
    if (handle_) api().destroy(static_cast<cusolverDnHandle_t>(handle_));
    if (start_) cudaEventDestroy(start_);
}

cudaError_t Solver::run(const double* d, int n, double* a_scratch, double* w, double* work_dev, size_t work_doubles,
                        int* info_dev, double* v_out, double* lambda_out, cudaStream_t stream, std::string* err) {
    const Api& x = api();
    if (!x.error.empty()) {
        *err = x.error;
        return cudaErrorNotSupported;
    }
    if (!handle_) {
        cusolverDnHandle_t h;
        if (x.create(&h) != CUSOLVER_STATUS_SUCCESS) {
            *err = "cusolverDnCreate failed";
            return cudaErrorUnknown;
        }
        handle_ = h;
    }
    auto h = static_cast<cusolverDnHandle_t>(handle_);
    x.set_stream(h, stream);
    cudaError_t e = cudaMemcpyAsync(a_scratch, d, static_cast<size_t>(n) * n * sizeof(double),
                                    cudaMemcpyDeviceToDevice, stream);
    if (e != cudaSuccess) return e;
    // D is symmetric: its row-major storage is its column-major storage.
    if (x.syevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n, a_scratch, n, w, work_dev,
                static_cast<int>(work_doubles), info_dev) != CUSOLVER_STATUS_SUCCESS) {
        *err = "cusolverDnDsyevd failed";
        return cudaErrorUnknown;
    }
    desc_sign_kernel<<<n, 256, 0, stream>>>(a_scratch, w, n, v_out, lambda_out);
    note_launch();
    return cudaGetLastError();
}

size_t Solver::workspace_doubles(int n, std::string* err) {
    const Api& x = api();
    if (!x.error.empty()) {
        *err = x.error;
        return 0;
    }
    if (!handle_) {
        cusolverDnHandle_t h;
        if (x.create(&h) != CUSOLVER_STATUS_SUCCESS) {
            *err = "cusolverDnCreate failed";
            return 0;
        }
        handle_ = h;
    }
    int lwork = 0;
    if (x.buffer_size(static_cast<cusolverDnHandle_t>(handle_), CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n,
                      nullptr, n, nullptr, &lwork) != CUSOLVER_STATUS_SUCCESS) {
        *err = "cusolverDnDsyevd_bufferSize failed";
        return 0;
    }
    return static_cast<size_t>(lwork);
}

bool Solver::ensure_handle(std::string* err) {
    const Api& x = api();
    if (!x.error.empty()) {
        *err = x.error;
        return false;
    }
    if (!handle_) {
        cusolverDnHandle_t h;
        if (x.create(&h) != CUSOLVER_STATUS_SUCCESS) {
            *err = "cusolverDnCreate failed";
            return false;
        }
        handle_ = h;
    }
    return true;
}

// Cholesky lanes: the pairs' factorisations are small (n ≈ 10²–10³), so a
// few run concurrently, each lane with its own handle, stream and workspace.
Solver::CholLane::~CholLane() {
    if (handle) api().destroy(static_cast<cusolverDnHandle_t>(handle));
    if (stream) cudaStreamDestroy(stream);
    if (done) cudaEventDestroy(done);
    if (work) cudaFree(work);
}

cudaError_t Solver::chol_lanes(double* a, int n, int batch, double* b, int nrhs, int* info_dev, cudaStream_t stream,
                               std::string* err) {
    if (!ensure_handle(err)) return cudaErrorNotSupported;
    const Api& x = api();
    const int lanes = std::min(kCholLanes, std::max(batch, 1));
    cudaError_t e = cudaSuccess;
    if (!start_ && (e = cudaEventCreateWithFlags(&start_, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(start_, stream)) != cudaSuccess) return e;
    for (int l = 0; l < lanes; ++l) {
        CholLane& ln = lanes_[l];
        if (!ln.handle) {
            cusolverDnHandle_t h;
            if (x.create(&h) != CUSOLVER_STATUS_SUCCESS) {
                *err = "cusolverDnCreate failed";
                return cudaErrorUnknown;
            }
            ln.handle = h;
            if ((e = cudaStreamCreateWithFlags(&ln.stream, cudaStreamNonBlocking)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&ln.done, cudaEventDisableTiming)) != cudaSuccess) return e;
            x.set_stream(static_cast<cusolverDnHandle_t>(ln.handle), ln.stream);
        }
        int lwork = 0;
        if (x.potrf_buffer_size(static_cast<cusolverDnHandle_t>(ln.handle), CUBLAS_FILL_MODE_LOWER, n, a, n,
                                &lwork) != CUSOLVER_STATUS_SUCCESS) {
            *err = "cusolverDnDpotrf_bufferSize failed";
            return cudaErrorUnknown;
        }
        if (static_cast<size_t>(lwork) > ln.work_doubles) {
            if (ln.work) cudaFree(ln.work);
            ln.work = nullptr;
            ln.work_doubles = 0;
            if ((e = cudaMalloc(&ln.work, static_cast<size_t>(lwork) * sizeof(double))) != cudaSuccess) return e;
            ln.work_doubles = static_cast<size_t>(lwork);
        }
        if ((e = cudaStreamWaitEvent(ln.stream, start_, 0)) != cudaSuccess) return e;
    }
    for (int i = 0; i < batch; ++i) {
        CholLane& ln = lanes_[i % lanes];
        auto h = static_cast<cusolverDnHandle_t>(ln.handle);
        double* ai = a + static_cast<size_t>(i) * n * n;
        double* bi = b ? b + static_cast<size_t>(i) * n * nrhs : nullptr;
        if (x.potrf(h, CUBLAS_FILL_MODE_LOWER, n, ai, n, static_cast<double*>(ln.work),
                    static_cast<int>(ln.work_doubles), info_dev + i) != CUSOLVER_STATUS_SUCCESS) {
            *err = "cusolverDnDpotrf failed";
            return cudaErrorUnknown;
        }
        if (b && x.potrs(h, CUBLAS_FILL_MODE_LOWER, n, nrhs, ai, n, bi, n, info_dev + batch + i) !=
                     CUSOLVER_STATUS_SUCCESS) {
            *err = "cusolverDnDpotrs failed";
            return cudaErrorUnknown;
        }
    }
    for (int l = 0; l < lanes; ++l) {
        if ((e = cudaEventRecord(lanes_[l].done, lanes_[l].stream)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(stream, lanes_[l].done, 0)) != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

cudaError_t Solver::spd_solve(double* a, int n, int batch, double* b, int nrhs, int* info_dev, cudaStream_t stream,
                              std::string* err) {
    return chol_lanes(a, n, batch, b, nrhs, info_dev, stream, err);
}

cudaError_t Solver::cholesky(double* a, int n, int batch, int* info_dev, cudaStream_t stream, std::string* err) {
    return chol_lanes(a, n, batch, nullptr, 0, info_dev, stream, err);
}

cudaError_t launch_reduced_map(const double* v, const double* lambda, int n, int r, double* tr, cudaStream_t stream) {
    const long long total = static_cast<long long>(n) * r;
    reduced_map_kernel<<<static_cast<int>((total + 255) / 256), 256, 0, stream>>>(v, lambda, n, r, tr);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_transpose_pad(const double* tr, int n, int r, int r_pad, size_t ld, double* trt,
                                 cudaStream_t stream) {
    const long long total = static_cast<long long>(r_pad) * ld;
    transpose_pad_kernel<<<static_cast<int>((total + 255) / 256), 256, 0, stream>>>(tr, n, r, r_pad, ld, trt);
    note_launch();
    return cudaGetLastError();
}

}  // namespace eig
}  // namespace dopinf_b200
