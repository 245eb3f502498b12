/*
 * dopinf_oracle.c — CPU restatement of the reference dOpInf snapshot-pass
 * arithmetic. TEST INFRASTRUCTURE ONLY: this file is the checker that tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg compare the CUDA
 * path against. Nothing in paper_2504_14338_b200/ links or calls it.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/proj) in the exact floating-point order the reference
 * executes on an x86-64 host with AVX2+FMA, which is the kernel table the
 * reference selects at run time (src/kernels_dispatch.cpp:13-20, 42-47).
 * Pinned bit-for-bit against the compiled reference (oracle/_ref) by
 * tests/test_oracle_pins.py and against the reference's own known-answer
 * tests (test_transform.cpp, test_linalg.cpp, test_pod.cpp, test_data.cpp).
 *
 * Build: oracle/Makefile -> oracle/_build/libdopinf_oracle.so, compiled with
 * -ffp-contract=off so that every fused multiply-add below is an explicit
 * fma() call and no other contraction happens.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Seeded RNG: std::mt19937_64 (the C++ standard's parameters) + the
 * reference's hand Box-Muller. Restates src/synth.cpp:15-34 and
 * include/dopinf/synth.hpp:20-33. */

#define MT_N 312
#define MT_M 156

typedef struct {
    uint64_t mt[MT_N];
    int idx;
    int have_spare;
    double spare;
} oracle_rng;

static void mt_seed(oracle_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i) {
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    }
    r->idx = MT_N;
}

static uint64_t mt_next(oracle_rng* r) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    const uint64_t matrix_a = 0xB5026F5AA96619E9ULL;
    if (r->idx >= MT_N) {
        for (int i = 0; i < MT_N; ++i) {
            const uint64_t x = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= matrix_a;
            r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

oracle_rng* oracle_rng_new(uint64_t seed) {
    oracle_rng* r = (oracle_rng*)calloc(1, sizeof(oracle_rng));
    if (r) mt_seed(r, seed);
    return r;
}

void oracle_rng_free(oracle_rng* r) { free(r); }

uint64_t oracle_rng_raw(oracle_rng* r) { return mt_next(r); }

/* synth.cpp:15-18: 53 high bits -> [0, 1). */
double oracle_rng_uniform(oracle_rng* r) { return (double)(mt_next(r) >> 11) * 0x1.0p-53; }

/* synth.cpp:22-34: Box-Muller with a cached spare. */
double oracle_rng_normal(oracle_rng* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    const double u1 = 1.0 - oracle_rng_uniform(r);
    const double u2 = oracle_rng_uniform(r);
    const double radius = sqrt(-2.0 * log(u1));
    const double angle = 2.0 * 3.141592653589793115997963468544185161590576171875 * u2;
    r->spare = radius * sin(angle);
    r->have_spare = 1;
    return radius * cos(angle);
}

/* tests/helpers.hpp:14-18 random_matrix: row-major fill with rng.normal(). */
void oracle_rng_fill_normal(oracle_rng* r, double* out, size_t count) {
    for (size_t i = 0; i < count; ++i) out[i] = oracle_rng_normal(r);
}

/* ------------------------------------------------------------------------ */
/* Vector kernels: the AVX2+FMA table (src/kernels_avx2.cpp), 4 f64 lanes. */

/* kernels_avx2.cpp:48-55 sum_avx2 + hsum (:16-22). */
double oracle_k_sum(const double* x, size_t n) {
    double l0 = 0.0, l1 = 0.0, l2 = 0.0, l3 = 0.0;
    size_t i = 0;
    for (; i + 4 <= n; i += 4) {
        l0 += x[i];
        l1 += x[i + 1];
        l2 += x[i + 2];
        l3 += x[i + 3];
    }
    double s = (l0 + l2) + (l1 + l3);
    for (; i < n; ++i) s += x[i];
    return s;
}

/* kernels_avx2.cpp:57-67 max_abs_avx2 (max is order independent). */
double oracle_k_max_abs(const double* x, size_t n) {
    double m = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double a = fabs(x[i]);
        if (a > m) m = a;
    }
    return m;
}

/* kernels_avx2.cpp:69-78 axpy_avx2: y = fma(a, x, y) lane-wise; the scalar
 * tail `y[i] += a * x[i]` is compiled with -mfma and GCC's default
 * -ffp-contract=fast, so it is an FMA as well (pinned in
 * tests/test_oracle_pins.py for odd column counts). */
void oracle_k_axpy(double a, const double* x, double* y, size_t n) {
    for (size_t i = 0; i < n; ++i) y[i] = fma(a, x[i], y[i]);
}

/* kernels_avx2.cpp:32-46 dot_avx2: two 4-lane FMA accumulators over blocks
 * of 8, one over a trailing block of 4, hsum(acc0 + acc1), scalar tail. The
 * tail `acc += a[i] * b[i]` is NOT contracted by the reference's compiler
 * (vmulsd + vaddsd in the compiled kernels_avx2.o, unlike the axpy and
 * scale_shift tails): rounded product, then the add. */
double oracle_k_dot(const double* a, const double* b, size_t n) {
    double c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0};
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
        for (int l = 0; l < 4; ++l) {
            c0[l] = fma(a[i + l], b[i + l], c0[l]);
            c1[l] = fma(a[i + 4 + l], b[i + 4 + l], c1[l]);
        }
    }
    for (; i + 4 <= n; i += 4) {
        for (int l = 0; l < 4; ++l) c0[l] = fma(a[i + l], b[i + l], c0[l]);
    }
    double v[4];
    for (int l = 0; l < 4; ++l) v[l] = c0[l] + c1[l];
    double acc = (v[0] + v[2]) + (v[1] + v[3]);
    for (; i < n; ++i) acc = acc + a[i] * b[i];
    return acc;
}

/* ------------------------------------------------------------------------ */
/* Step II transform (src/transform.cpp). */

/* transform.cpp:10-20 center_in_place: mean = sum(row)/nt; row += -mean. */
void oracle_center_in_place(double* q, size_t rows, size_t cols, double* means) {
    for (size_t i = 0; i < rows; ++i) {
        double* row = q + i * cols;
        const double mean = oracle_k_sum(row, cols) / (double)cols;
        const double neg = -mean;
        for (size_t t = 0; t < cols; ++t) row[t] += neg;
        means[i] = mean;
    }
}

/* center_in_place's mean (transform.cpp:14-15) and the max-abs that
 * compute_global_scales then takes of the centered row (transform.cpp:29-31),
 * without writing the centered values: max over t of |fl(x_t + (-mean))|,
 * the same numbers center_in_place stores. Rows at pitch ld. */
void oracle_row_stats(const double* q, size_t ld, size_t rows, size_t cols, double* means,
                      double* maxabs) {
    for (size_t i = 0; i < rows; ++i) {
        const double* row = q + i * ld;
        const double mean = oracle_k_sum(row, cols) / (double)cols;
        const double neg = -mean;
        double m = 0.0;
        for (size_t t = 0; t < cols; ++t) {
            const double a = fabs(row[t] + neg);
            if (a > m) m = a;
        }
        means[i] = mean;
        maxabs[i] = m;
    }
}

/* transform.cpp:29-31: per-variable max-abs over the contiguous
 * nx_i * nt segment of variable j (before the MAX all-reduce). */
void oracle_local_maxabs(const double* q, size_t n_vars, size_t nx_i, size_t cols,
                         double* out) {
    for (size_t j = 0; j < n_vars; ++j) {
        out[j] = oracle_k_max_abs(q + j * nx_i * cols, nx_i * cols);
    }
}

/* transform.cpp:32-39 + comm_inprocess.cpp:101-112: MAX across ranks in
 * ascending rank order; returns the first degenerate variable index, or -1. */
long oracle_reduce_scales(const double* per_rank, int p, size_t n_vars, double* out) {
    for (size_t j = 0; j < n_vars; ++j) out[j] = per_rank[j];
    for (int r = 1; r < p; ++r) {
        for (size_t j = 0; j < n_vars; ++j) {
            const double v = per_rank[(size_t)r * n_vars + j];
            out[j] = out[j] < v ? v : out[j];
        }
    }
    for (size_t j = 0; j < n_vars; ++j) {
        if (out[j] == 0.0) return (long)j;
    }
    return -1;
}

/* transform.cpp:43-49 scale_in_place: true IEEE division per variable. */
void oracle_scale_in_place(double* q, size_t n_vars, size_t nx_i, size_t cols,
                           const double* scales) {
    for (size_t j = 0; j < n_vars; ++j) {
        double* seg = q + j * nx_i * cols;
        const size_t count = nx_i * cols;
        for (size_t i = 0; i < count; ++i) seg[i] /= scales[j];
    }
}

/* transform.cpp:51-72 inverse transform: x = scale * x + mean (FMA lanes). */
void oracle_inverse_transform_block(double* values, size_t rows, size_t cols, size_t nx_i,
                                    const double* means, const double* scales,
                                    int scaling_enabled) {
    for (size_t i = 0; i < rows; ++i) {
        const double s = scaling_enabled ? scales[i / nx_i] : 1.0;
        for (size_t t = 0; t < cols; ++t) {
            values[i * cols + t] = fma(s, values[i * cols + t], means[i]);
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Step III Gram and projection (src/linalg.cpp, src/pod.cpp). */

/* linalg.cpp:50-58 gram (called by pod::local_gram, pod.cpp:11-13): the full
 * square, rows outer, c.row(i) += q(l, i) * q.row(l) via axpy. */
void oracle_gram(const double* q, size_t rows, size_t cols, double* d) {
    memset(d, 0, cols * cols * sizeof(double));
    for (size_t l = 0; l < rows; ++l) {
        const double* ql = q + l * cols;
        for (size_t i = 0; i < cols; ++i) oracle_k_axpy(ql[i], ql, d + i * cols, cols);
    }
}

/* linalg.cpp:50-58 gram restricted to the entries (ii[p], jj[p]) and
 * continued over a further slice of rows (pitch ld): entry (i, j) of the
 * reference's Gram only ever receives axpy's fma(q(l, i), q(l, j), c(i, j)),
 * rows ascending, so acc[p] carried across consecutive row slices ends as the
 * reference's value bit for bit (for a slice sequence in block-row order). */
void oracle_gram_entries(const double* q, size_t ld, size_t rows, const size_t* ii, const size_t* jj,
                         size_t npairs, double* acc) {
    for (size_t l = 0; l < rows; ++l) {
        const double* ql = q + l * ld;
        for (size_t p = 0; p < npairs; ++p) acc[p] = fma(ql[ii[p]], ql[jj[p]], acc[p]);
    }
}

/* linalg.cpp:50-58 gram over one tile of entries, rows [i0, i0+ni) × columns
 * [j0, j0+nj) of D, all rows of q (pitch ld) in order: out (ni × nj) receives
 * the reference's FMA chains bit for bit (each entry only ever receives
 * fma(q(l, i), q(l, j), c), rows ascending). The j loop is the reference's
 * axpy (element-wise FMAs, vectorisable without changing any result); tiles
 * are independent, so a full D is computed tile by tile on several threads. */
__attribute__((optimize("O3"))) void oracle_gram_tile(const double* q, size_t ld, size_t rows, size_t i0,
                                                      size_t ni, size_t j0, size_t nj, double* out) {
    memset(out, 0, ni * nj * sizeof(double));
    for (size_t l = 0; l < rows; ++l) {
        const double* ql = q + l * ld;
        for (size_t i = 0; i < ni; ++i) {
            const double a = ql[i0 + i];
            double* o = out + i * nj;
            const double* x = ql + j0;
            for (size_t j = 0; j < nj; ++j) o[j] = fma(a, x[j], o[j]);
        }
    }
}

/* comm_inprocess.cpp:101-112: SUM all-reduce, ascending rank order
 * (pod::global_gram, pod.cpp:15-18). parts is p x count. */
void oracle_allreduce_sum(const double* parts, int p, size_t count, double* out) {
    memcpy(out, parts, count * sizeof(double));
    for (int r = 1; r < p; ++r) {
        const double* s = parts + (size_t)r * count;
        for (size_t i = 0; i < count; ++i) out[i] += s[i];
    }
}

/* linalg.cpp:28-37 matmul_tn (pod::project, pod.cpp:103-105):
 * c = a^T b, a is m x ka, b is m x nb, c is ka x nb. */
void oracle_matmul_tn(const double* a, size_t m, size_t ka, const double* b, size_t nb,
                      double* c) {
    memset(c, 0, ka * nb * sizeof(double));
    for (size_t l = 0; l < m; ++l) {
        for (size_t i = 0; i < ka; ++i) oracle_k_axpy(a[l * ka + i], b + l * nb, c + i * nb, nb);
    }
}

/* linalg.cpp:17-26 matmul (postprocess::reconstruct_field, postprocess.cpp:66):
 * c = a b, a is m x k, b is k x nb. */
void oracle_matmul(const double* a, size_t m, size_t k, const double* b, size_t nb,
                   double* c) {
    memset(c, 0, m * nb * sizeof(double));
    for (size_t i = 0; i < m; ++i) {
        for (size_t l = 0; l < k; ++l) oracle_k_axpy(a[i * k + l], b + l * nb, c + i * nb, nb);
    }
}

/* linalg.cpp:39-48 matmul_nt (postprocess::reconstruct_field, postprocess.cpp:67):
 * c(i, j) = kernels::dot(a.row(i), b.row(j)); a is m x k, b is n x k. */
void oracle_matmul_nt(const double* a, size_t m, size_t k, const double* b, size_t n, double* c) {
    for (size_t i = 0; i < m; ++i) {
        for (size_t j = 0; j < n; ++j) c[i * n + j] = oracle_k_dot(a + i * k, b + j * k, k);
    }
}

/* postprocess.cpp:12-34 basis_rows: naive triple loop, acc += q * tr with a
 * rounded product (postprocess.cpp is compiled without -mfma). Returns the
 * index of the first bad row (>= rows) or -1. */
long oracle_basis_rows(const double* q, size_t rows, size_t cols, const double* tr,
                       size_t r, const size_t* local_rows, size_t nsel, double* out) {
    for (size_t k = 0; k < nsel; ++k) {
        const size_t row = local_rows[k];
        if (row >= rows) return (long)k;
        for (size_t j = 0; j < r; ++j) {
            double acc = 0.0;
            for (size_t t = 0; t < cols; ++t) {
                const double prod = q[row * cols + t] * tr[t * r + j];
                acc = acc + prod;
            }
            out[k * r + j] = acc;
        }
    }
    return -1;
}

/* ------------------------------------------------------------------------ */
/* Row sharding (src/data.cpp:86-103 partition_rows). Returns 0 on success,
 * 1 when p < 1, 2 when p > nx (PartitionError in the reference). */
int oracle_partition_rows(size_t nx, int p, size_t* begin, size_t* end) {
    if (p < 1) return 1;
    if ((size_t)p > nx) return 2;
    const size_t ranks = (size_t)p;
    const size_t base = nx / ranks;
    for (size_t r = 0; r < ranks; ++r) {
        begin[r] = r * base;
        end[r] = (r + 1 == ranks) ? nx : (r + 1) * base;
    }
    return 0;
}
