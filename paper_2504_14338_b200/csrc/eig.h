// eig.h — device eigensolve of the Gram (eig.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include <string>

namespace dopinf_b200 {
namespace eig {

// nullptr when cuSOLVER can be loaded, else why not.
const char* unavailable_reason();

class Solver {
public:
    ~Solver();
    size_t workspace_doubles(int n, std::string* err);
    // v_out (n×n row-major, column k ↔ lambda_out[k]) and lambda_out (n,
    // descending, unclamped) from the symmetric n×n d; a_scratch n×n, w n.
    cudaError_t run(const double* d, int n, double* a_scratch, double* w, double* work_dev, size_t work_doubles,
                    int* info_dev, double* v_out, double* lambda_out, cudaStream_t stream, std::string* err);

    // Cholesky solves of `batch` SPD n×n systems a_i (column-major, lda n;
    // factored in place) with nrhs right-hand sides b_i (column-major, ldb n;
    // overwritten by the solutions), spread over kCholLanes concurrent
    // cuSOLVER streams and joined back into `stream`. info_dev[2·batch]:
    // potrf infos, then potrs.
    cudaError_t spd_solve(double* a, int n, int batch, double* b, int nrhs, int* info_dev, cudaStream_t stream,
                          std::string* err);
    // Only the factorisations (lower Cholesky in place), info_dev[batch].
    cudaError_t cholesky(double* a, int n, int batch, int* info_dev, cudaStream_t stream, std::string* err);

private:
    static constexpr int kCholLanes = 8;
    struct CholLane {
        void* handle = nullptr;
        cudaStream_t stream = nullptr;
        cudaEvent_t done = nullptr;
        void* work = nullptr;
        size_t work_doubles = 0;
        ~CholLane();
    };
    bool ensure_handle(std::string* err);
    cudaError_t chol_lanes(double* a, int n, int batch, double* b, int nrhs, int* info_dev, cudaStream_t stream,
                           std::string* err);
    void* handle_ = nullptr;
    cudaEvent_t start_ = nullptr;
    CholLane lanes_[kCholLanes];
};

cudaError_t launch_reduced_map(const double* v, const double* lambda, int n, int r, double* tr, cudaStream_t stream);
cudaError_t launch_transpose_pad(const double* tr, int n, int r, int r_pad, size_t ld, double* trt,
                                 cudaStream_t stream);

}  // namespace eig
}  // namespace dopinf_b200
