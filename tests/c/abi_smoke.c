/* abi_smoke.c — the C ABI from plain C11 (no C++, no torch): one context, one
 * block, the fused Steps II–III, the projection and the SNP1 header parser,
 * checked against a naive C restatement on the same bytes. TEST
 * INFRASTRUCTURE (tests/test_gpu_cpp_dropin.py runs it on the B200).
 * Exit status 0 iff every check passes. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "dopinf_b200.h"

#define CHECK(call)                                                                      \
    do {                                                                                 \
        int rc_ = (call);                                                                \
        if (rc_ != DOPINF_B200_OK) {                                                     \
            fprintf(stderr, "%s failed: %s (%s)\n", #call, dopinf_b200_status_string(rc_), \
                    dopinf_b200_last_error(ctx));                                        \
            return 1;                                                                    \
        }                                                                                \
    } while (0)

static uint64_t lcg(uint64_t* s) {
    *s = *s * 6364136223846793005ULL + 1442695040888963407ULL;
    return *s >> 11;
}

int main(void) {
    enum { NV = 2, NX = 500, NT = 24, R = 3 };
    const size_t rows = NV * NX;
    double* q = malloc(sizeof(double) * rows * NT);
    double* means = malloc(sizeof(double) * rows);
    double scales[NV], d[NT * NT], tr[NT * R], qhat[R * NT];
    uint64_t seed = 42;
    for (size_t i = 0; i < rows * NT; ++i) q[i] = (double)(lcg(&seed) % 2000001) / 1e6 - 1.0 + (i / NT < NX ? 3.0 : -7.0);

    dopinf_b200_ctx* ctx = NULL;
    if (dopinf_b200_abi_version() != DOPINF_B200_ABI_VERSION) return 1;
    CHECK(dopinf_b200_ctx_create(0, 0, 1, NULL, &ctx));
    dopinf_b200_block* blk = NULL;
    CHECK(dopinf_b200_block_create(ctx, NV, NX, 0, NT, &blk));
    CHECK(dopinf_b200_block_upload(blk, q, NT));
    CHECK(dopinf_b200_snapshot_pass(blk, 1, means, scales, d));

    /* naive restatement: center, max-abs scale per variable, full Gram */
    double* c = malloc(sizeof(double) * rows * NT);
    for (size_t i = 0; i < rows; ++i) {
        double m = 0.0;
        for (int t = 0; t < NT; ++t) m += q[i * NT + t];
        m /= NT;
        if (fabs(m - means[i]) > 1e-13 * (1.0 + fabs(m))) {
            fprintf(stderr, "mean %zu: %g vs %g\n", i, means[i], m);
            return 1;
        }
        for (int t = 0; t < NT; ++t) c[i * NT + t] = q[i * NT + t] - means[i];
    }
    for (int v = 0; v < NV; ++v) {
        double s = 0.0;
        for (size_t i = (size_t)v * NX; i < (size_t)(v + 1) * NX; ++i)
            for (int t = 0; t < NT; ++t) s = fmax(s, fabs(c[i * NT + t]));
        if (fabs(s - scales[v]) > 1e-14 * s) {
            fprintf(stderr, "scale %d: %g vs %g\n", v, scales[v], s);
            return 1;
        }
        for (size_t i = (size_t)v * NX; i < (size_t)(v + 1) * NX; ++i)
            for (int t = 0; t < NT; ++t) c[i * NT + t] /= scales[v];
    }
    double num = 0.0, den = 0.0;
    for (int a = 0; a < NT; ++a)
        for (int b = 0; b < NT; ++b) {
            double g = 0.0;
            for (size_t i = 0; i < rows; ++i) g += c[i * NT + a] * c[i * NT + b];
            num += (d[a * NT + b] - g) * (d[a * NT + b] - g);
            den += g * g;
            if (d[a * NT + b] != d[b * NT + a]) {
                fprintf(stderr, "D not bitwise symmetric at (%d, %d)\n", a, b);
                return 1;
            }
        }
    if (sqrt(num / den) > 1e-12) {
        fprintf(stderr, "Gram rel. Frobenius error %g > 1e-12\n", sqrt(num / den));
        return 1;
    }

    /* projection Q̂ = T_rᵀ D with an arbitrary T_r */
    for (int i = 0; i < NT * R; ++i) tr[i] = (double)(lcg(&seed) % 1000) / 1000.0;
    CHECK(dopinf_b200_project(ctx, tr, NT, R, qhat));
    for (int i = 0; i < R; ++i)
        for (int j = 0; j < NT; ++j) {
            double acc = 0.0;
            for (int l = 0; l < NT; ++l) acc = fma(tr[l * R + i], d[l * NT + j], acc);
            if (acc != qhat[i * NT + j]) {
                fprintf(stderr, "qhat (%d, %d) not bit-identical\n", i, j);
                return 1;
            }
        }

    /* a context-free call reports through last_error(NULL) */
    uint64_t dims[4];
    if (dopinf_b200_snp1_header("/nonexistent.snp1", dims, NULL, 0, NULL) != DOPINF_B200_ERR_DATA_FORMAT ||
        strncmp(dopinf_b200_last_error(NULL), "cannot open snapshot file", 25) != 0) {
        fprintf(stderr, "snp1_header error path\n");
        return 1;
    }

    dopinf_b200_block_destroy(blk);
    dopinf_b200_ctx_destroy(ctx);
    free(q);
    free(c);
    free(means);
    printf("abi_smoke (C11): all checks passed, %llu kernel launches\n",
           (unsigned long long)dopinf_b200_kernel_launches());
    return 0;
}
