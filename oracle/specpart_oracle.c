/* oracle/specpart_oracle.c — TEST INFRASTRUCTURE ONLY (see specpart_oracle.h).
 *
 * A plain-C restatement of the reference's hot path, written for checking, not
 * speed: sequential loops, the reference's reduction orders (4096-row chunks for
 * dot/gram, kernels.cpp:12-15), column-major dense blocks (dense.hpp:10-39),
 * compiled with -ffp-contract=off like the reference's x86-64 baseline build.
 * Section comments cite the reference lines each function restates.
 */
#include "specpart_oracle.h"

#include <math.h>
#include <setjmp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ errors */
static char g_err[512];
static jmp_buf g_jmp;
static int g_jmp_armed;

static void fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    if (g_jmp_armed) longjmp(g_jmp, code);
    abort();
}

const char* ref_last_error(void) { return g_err; }

#define GUARD_BEGIN                    \
    int _code = setjmp(g_jmp);         \
    if (_code) {                       \
        g_jmp_armed = 0;               \
        return _code;                  \
    }                                  \
    g_jmp_armed = 1;
#define GUARD_END      \
    g_jmp_armed = 0;   \
    return SP_OK;

static void* xcalloc(size_t n, size_t s) {
    void* p = calloc(n ? n : 1, s ? s : 1);
    if (!p) fail(SP_ERROR, "out of memory");
    return p;
}

/* ---------------------------------------------------------- sparse / dense */
typedef struct {
    int64_t n;
    int64_t* offs;
    int32_t* cols;
    double* vals;
    double* diag;
    double bound;
    int is_diag;
} Op;

static void op_free(Op* o) {
    free(o->offs);
    free(o->cols);
    free(o->vals);
    free(o->diag);
    memset(o, 0, sizeof *o);
}

static double value_at(const sp_graph* g, int64_t k) { return g->values ? g->values[k] : 1.0; }

/* Graph::weighted_degree, graph.cpp:15-20 */
static double wdeg(const sp_graph* g, int64_t v) {
    double s = 0.0;
    for (int64_t k = g->row_offsets[v]; k < g->row_offsets[v + 1]; ++k) s += value_at(g, k);
    return s;
}

/* make_operator / gershgorin_bound / extract_diag, laplacian.cpp:14-51 */
static void finish_op(Op* o) {
    o->bound = 0.0;
    o->diag = xcalloc((size_t)o->n, sizeof(double));
    for (int64_t i = 0; i < o->n; ++i) {
        double d = 0.0, off = 0.0;
        for (int64_t k = o->offs[i]; k < o->offs[i + 1]; ++k) {
            if (o->cols[k] == i) {
                d += o->vals[k];
                o->diag[i] = o->vals[k];
            } else {
                off += fabs(o->vals[k]);
            }
        }
        if (d + off > o->bound) o->bound = d + off;
    }
    o->is_diag = o->offs[o->n] == o->n;
    for (int64_t k = 0; k < o->offs[o->n] && o->is_diag; ++k)
        if (o->cols[k] != k) o->is_diag = 0;
}

/* build_combinatorial (laplacian.cpp:53-83) / build_normalized (:85-127) */
static Op build_lap(const sp_graph* g, int normalized) {
    const int64_t n = g->n;
    if (n == 0) fail(SP_INVALID, normalized ? "build_normalized: empty graph" : "build_combinatorial: empty graph");
    double* isd = NULL;
    if (normalized) {
        isd = xcalloc((size_t)n, sizeof(double));
        for (int64_t i = 0; i < n; ++i) {
            const double d = wdeg(g, i);
            if (d <= 0.0) {
                free(isd);
                char m[160];
                snprintf(m, sizeof m, "normalized Laplacian requires degree >= 1 at vertex %lld", (long long)i);
                fail(SP_DEGENERATE, m);
            }
            isd[i] = 1.0 / sqrt(d);
        }
    }
    const int64_t nnz = g->row_offsets[n] + n;
    Op o = {0};
    o.n = n;
    o.offs = xcalloc((size_t)n + 1, sizeof(int64_t));
    o.cols = xcalloc((size_t)nnz, sizeof(int32_t));
    o.vals = xcalloc((size_t)nnz, sizeof(double));
    int64_t w = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double dv = normalized ? 1.0 : wdeg(g, i);
        int placed = 0;
        for (int64_t k = g->row_offsets[i]; k < g->row_offsets[i + 1]; ++k) {
            const int32_t j = g->col_indices[k];
            if (!placed && j > i) {
                o.cols[w] = (int32_t)i;
                o.vals[w++] = dv;
                placed = 1;
            }
            o.cols[w] = j;
            o.vals[w++] = normalized ? (-value_at(g, k) * isd[i]) * isd[j] : -value_at(g, k);
        }
        if (!placed) {
            o.cols[w] = (int32_t)i;
            o.vals[w++] = dv;
        }
        o.offs[i + 1] = w;
    }
    free(isd);
    finish_op(&o);
    if (normalized && o.bound > 2.0) o.bound = 2.0;
    return o;
}

/* build_degree, laplacian.cpp:129-144 */
static Op build_deg(const sp_graph* g) {
    const int64_t n = g->n;
    if (n == 0) fail(SP_INVALID, "build_degree: empty graph");
    Op o = {0};
    o.n = n;
    o.offs = xcalloc((size_t)n + 1, sizeof(int64_t));
    o.cols = xcalloc((size_t)n, sizeof(int32_t));
    o.vals = xcalloc((size_t)n, sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        o.offs[i] = i;
        o.cols[i] = (int32_t)i;
        o.vals[i] = wdeg(g, i);
    }
    o.offs[n] = n;
    finish_op(&o);
    return o;
}

static Op build_kind(int kind, const sp_graph* g) {
    if (kind == SP_LAP_COMBINATORIAL) return build_lap(g, 0);
    if (kind == SP_LAP_NORMALIZED) return build_lap(g, 1);
    if (kind == SP_LAP_DEGREE) return build_deg(g);
    fail(SP_INVALID, "unknown operator kind");
    return (Op){0};
}

/* spmv_block (kernels.cpp:36-62) / diag_scale (:187-197) via apply_block (laplacian.cpp:146-153) */
static void apply(const Op* o, const double* X, int m, double* Y) {
    const int64_t n = o->n;
    if (o->is_diag) {
        for (int64_t i = 0; i < n; ++i)
            for (int c = 0; c < m; ++c) Y[(size_t)c * n + i] = o->diag[i] * X[(size_t)c * n + i];
        return;
    }
    for (int64_t i = 0; i < n; ++i)
        for (int c = 0; c < m; ++c) {
            const double* xc = X + (size_t)c * n;
            double acc = 0.0;
            for (int64_t k = o->offs[i]; k < o->offs[i + 1]; ++k) acc += o->vals[k] * xc[o->cols[k]];
            Y[(size_t)c * n + i] = acc;
        }
}

#define CHUNK 4096

/* kernels::dot (kernels.cpp:159-178) */
static double dot(const double* u, const double* v, int64_t n) {
    const int64_t nch = (n + CHUNK - 1) / CHUNK;
    double s = 0.0;
    if (nch <= 1) {
        for (int64_t i = 0; i < n; ++i) s += u[i] * v[i];
        return s;
    }
    for (int64_t ch = 0; ch < nch; ++ch) {
        const int64_t lo = ch * CHUNK, hi = lo + CHUNK < n ? lo + CHUNK : n;
        double p = 0.0;
        for (int64_t i = lo; i < hi; ++i) p += u[i] * v[i];
        s += p;
    }
    return s;
}

/* kernels::gram (kernels.cpp:79-110): G (mu x mv, column-major) = U^T V */
static void gram(const double* U, int mu, const double* V, int mv, int64_t n, double* G) {
    const int64_t nch = (n + CHUNK - 1) / CHUNK;
    memset(G, 0, sizeof(double) * (size_t)mu * mv);
    if (nch <= 1) {
        for (int j = 0; j < mv; ++j)
            for (int i = 0; i < mu; ++i) {
                double s = 0.0;
                for (int64_t r = 0; r < n; ++r) s += U[(size_t)i * n + r] * V[(size_t)j * n + r];
                G[(size_t)j * mu + i] = s;
            }
        return;
    }
    for (int64_t ch = 0; ch < nch; ++ch) {
        const int64_t lo = ch * CHUNK, hi = lo + CHUNK < n ? lo + CHUNK : n;
        for (int j = 0; j < mv; ++j)
            for (int i = 0; i < mu; ++i) {
                double s = 0.0;
                for (int64_t r = lo; r < hi; ++r) s += U[(size_t)i * n + r] * V[(size_t)j * n + r];
                G[(size_t)j * mu + i] += s;  /* partial[ch] = 0 + s, then summed in chunk order */
            }
    }
}

/* kernels::mult (kernels.cpp:127-142): Y (n x mc) = X (n x mx) * C (mx x mc) */
static void mult(const double* X, int mx, const double* C, int mc, int64_t n, double* Y) {
    for (int64_t i = 0; i < n; ++i)
        for (int j = 0; j < mc; ++j) {
            double s = 0.0;
            for (int k = 0; k < mx; ++k) s += X[(size_t)k * n + i] * C[(size_t)j * mx + k];
            Y[(size_t)j * n + i] = s;
        }
}

/* ------------------------------------------------------------ mt19937_64 */
typedef struct {
    uint64_t mt[312];
    int mti;
} Mt64;

static void mt_seed(Mt64* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i) r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = 312;
}

static uint64_t mt_next(Mt64* r) {
    static const uint64_t MAG[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    if (r->mti >= 312) {
        int i;
        uint64_t x;
        for (i = 0; i < 312 - 156; ++i) {
            x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[i + 1] & 0x7FFFFFFFULL);
            r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ MAG[x & 1];
        }
        for (; i < 311; ++i) {
            x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[i + 1] & 0x7FFFFFFFULL);
            r->mt[i] = r->mt[i - 156] ^ (x >> 1) ^ MAG[x & 1];
        }
        x = (r->mt[311] & 0xFFFFFFFF80000000ULL) | (r->mt[0] & 0x7FFFFFFFULL);
        r->mt[311] = r->mt[155] ^ (x >> 1) ^ MAG[x & 1];
        r->mti = 0;
    }
    uint64_t y = r->mt[r->mti++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

static double mt_unit(Mt64* r) { return 2.0 * ((double)(mt_next(r) >> 11) * 0x1.0p-53) - 1.0; }

/* initial_guess_random / _piecewise, eigensolver.cpp:20-51 */
static void init_block(int init, int64_t n, int d, uint64_t seed, double* X) {
    if (d > n) fail(SP_INFEASIBLE, "initial guess: d > n");
    if (d < 1) fail(SP_INFEASIBLE, "initial guess: d < 1");
    if (init == SP_INIT_PIECEWISE) {
        memset(X, 0, sizeof(double) * (size_t)n * d);
        for (int64_t i = 0; i < n; ++i) X[i] = 1.0;
        const int64_t base = n / d, rem = n % d;
        int64_t start = 0;
        for (int b = 0; b + 1 < d; ++b) {
            const int64_t len = base + (b < rem ? 1 : 0);
            for (int64_t i = start; i < start + len; ++i) X[(size_t)(b + 1) * n + i] = 1.0;
            start += len;
        }
        return;
    }
    Mt64 r;
    mt_seed(&r, seed);
    for (int64_t t = 0; t < n * d; ++t) X[t] = mt_unit(&r);
}

/* --------------------------------------------------------- dense (dense.cpp) */
static double offnorm(const double* M, int m) {
    double s = 0.0;
    for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i)
            if (i != j) s += M[j * m + i] * M[j * m + i];
    return sqrt(s);
}

/* sym_eig: cyclic Jacobi, ascending stable order (dense.cpp:29-84) */
static void sym_eig(const double* A, int m, double* vals, double* vecs) {
    double* M = xcalloc((size_t)m * m, sizeof(double));
    double* V = xcalloc((size_t)m * m, sizeof(double));
    memcpy(M, A, sizeof(double) * (size_t)m * m);
    for (int i = 0; i < m; ++i) V[i * m + i] = 1.0;
    double scale = 0.0;
    for (int t = 0; t < m * m; ++t)
        if (fabs(M[t]) > scale) scale = fabs(M[t]);
    const double stop = scale == 0.0 ? 0.0 : 1e-15 * scale * (double)m;
    for (int sweep = 0; sweep < 64; ++sweep) {
        if (offnorm(M, m) <= stop) break;
        for (int p = 0; p < m - 1; ++p)
            for (int q = p + 1; q < m; ++q) {
                const double apq = M[q * m + p];
                if (fabs(apq) <= stop / ((double)m * m + 1.0)) continue;
                const double tau = (M[q * m + q] - M[p * m + p]) / (2.0 * apq);
                const double t = tau >= 0.0 ? 1.0 / (tau + sqrt(1.0 + tau * tau)) : 1.0 / (tau - sqrt(1.0 + tau * tau));
                const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
                for (int k = 0; k < m; ++k) {
                    const double a = M[p * m + k], b = M[q * m + k];
                    M[p * m + k] = c * a - s * b;
                    M[q * m + k] = s * a + c * b;
                }
                for (int k = 0; k < m; ++k) {
                    const double a = M[k * m + p], b = M[k * m + q];
                    M[k * m + p] = c * a - s * b;
                    M[k * m + q] = s * a + c * b;
                }
                for (int k = 0; k < m; ++k) {
                    const double a = V[p * m + k], b = V[q * m + k];
                    V[p * m + k] = c * a - s * b;
                    V[q * m + k] = s * a + c * b;
                }
            }
    }
    int* order = xcalloc((size_t)m, sizeof(int));
    for (int i = 0; i < m; ++i) order[i] = i;
    for (int i = 1; i < m; ++i) { /* stable insertion sort on the diagonal */
        const int o = order[i];
        int j = i - 1;
        while (j >= 0 && M[o * m + o] < M[order[j] * m + order[j]]) {
            order[j + 1] = order[j];
            --j;
        }
        order[j + 1] = o;
    }
    for (int j = 0; j < m; ++j) {
        vals[j] = M[order[j] * m + order[j]];
        for (int i = 0; i < m; ++i) vecs[j * m + i] = V[order[j] * m + i];
    }
    free(order);
    free(M);
    free(V);
}

static int cholesky(double* A, int n) { /* dense.cpp:86-104 */
    for (int j = 0; j < n; ++j) {
        double d = A[j * n + j];
        for (int k = 0; k < j; ++k) d -= A[k * n + j] * A[k * n + j];
        if (!(d > 0.0)) return 0;
        const double l = sqrt(d);
        A[j * n + j] = l;
        for (int i = j + 1; i < n; ++i) {
            double s = A[j * n + i];
            for (int k = 0; k < j; ++k) s -= A[k * n + i] * A[k * n + j];
            A[j * n + i] = s / l;
        }
        for (int i = 0; i < j; ++i) A[j * n + i] = 0.0;
    }
    return 1;
}

static void solve_lower(const double* L, int n, double* b) { /* dense.cpp:106-113 */
    for (int i = 0; i < n; ++i) {
        double s = b[i];
        for (int k = 0; k < i; ++k) s -= L[k * n + i] * b[k];
        b[i] = s / L[i * n + i];
    }
}

/* ------------------------------------------------- preconditioners (Jacobi, GMRES) */
typedef struct {
    int kind; /* 0 none, 1 jacobi, 2 poly */
    double* inv;
    double* roots;
    int k;
    const Op* A;
} Prec;

/* harmonic_ritz_values, preconditioners.cpp:232-273 */
static void harmonic_ritz(const double* Hk, int k, double beta, double* out) {
    double* C = xcalloc((size_t)k * k, sizeof(double));
    double* T = xcalloc((size_t)k * k, sizeof(double));
    double* L = xcalloc((size_t)k * k, sizeof(double));
    double* row = xcalloc((size_t)k, sizeof(double));
    double* vecs = xcalloc((size_t)k * k, sizeof(double));
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) {
            double s = 0.0;
            for (int l = 0; l < k; ++l) s += Hk[i * k + l] * Hk[j * k + l];
            C[j * k + i] = s;
        }
    C[(k - 1) * k + k - 1] += beta * beta;
    double trace = 0.0;
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) T[j * k + i] = 0.5 * (Hk[j * k + i] + Hk[i * k + j]);
    for (int i = 0; i < k; ++i) trace += T[i * k + i];
    memcpy(L, T, sizeof(double) * (size_t)k * k);
    double shift = 0.0;
    while (!cholesky(L, k)) {
        shift = shift == 0.0 ? 1e-14 * (trace > 1.0 ? trace : 1.0) : shift * 100.0;
        memcpy(L, T, sizeof(double) * (size_t)k * k);
        for (int i = 0; i < k; ++i) L[i * k + i] += shift;
        if (shift > 1.0) fail(SP_ERROR, "harmonic Ritz reduction failed");
    }
    for (int j = 0; j < k; ++j) solve_lower(L, k, C + (size_t)j * k);
    for (int i = 0; i < k; ++i) {
        for (int j = 0; j < k; ++j) row[j] = C[j * k + i];
        solve_lower(L, k, row);
        for (int j = 0; j < k; ++j) C[j * k + i] = row[j];
    }
    sym_eig(C, k, out, vecs);
    free(C);
    free(T);
    free(L);
    free(row);
    free(vecs);
}

/* leja_order, preconditioners.cpp:278-307 */
static void leja(double* r, int k) {
    double* out = xcalloc((size_t)k, sizeof(double));
    char* used = xcalloc((size_t)k, 1);
    int first = 0;
    for (int i = 1; i < k; ++i)
        if (fabs(r[i]) > fabs(r[first])) first = i;
    out[0] = r[first];
    used[first] = 1;
    for (int c = 1; c < k; ++c) {
        int best = k;
        double bs = -INFINITY;
        for (int i = 0; i < k; ++i) {
            if (used[i]) continue;
            double sc = 0.0;
            for (int t = 0; t < c; ++t) {
                const double d = fabs(r[i] - out[t]);
                sc += log(d > 1e-300 ? d : 1e-300);
            }
            if (sc > bs) {
                bs = sc;
                best = i;
            }
        }
        out[c] = r[best];
        used[best] = 1;
    }
    memcpy(r, out, sizeof(double) * (size_t)k);
    free(out);
    free(used);
}

/* polynomial_build, preconditioners.cpp:315-382 (GMRES roots) */
static Prec poly_build(const Op* A, uint64_t seed, int degree) {
    if (degree < 1) fail(SP_INFEASIBLE, "polynomial_build: degree < 1");
    const int64_t n = A->n;
    const int kr = (int)(degree < n ? degree : n);
    double* V = xcalloc((size_t)n * (kr + 1), sizeof(double));
    double* Hs = xcalloc((size_t)(kr + 1) * kr, sizeof(double));
    double* w = xcalloc((size_t)n, sizeof(double));
    Mt64 r;
    mt_seed(&r, seed);
    for (int64_t i = 0; i < n; ++i) V[i] = mt_unit(&r);
    double mean = 0.0;
    for (int64_t i = 0; i < n; ++i) mean += V[i];
    mean /= (double)n;
    for (int64_t i = 0; i < n; ++i) V[i] -= mean;
    const double nrm0 = sqrt(dot(V, V, n));
    if (nrm0 > 0.0)
        for (int64_t i = 0; i < n; ++i) V[i] /= nrm0;
    else {
        memset(V, 0, sizeof(double) * (size_t)n);
        V[0] = 1.0;
    }
    int kg = 0;
    double beta = 0.0;
    const double tiny = 1e-13 * (A->bound > 0.0 ? A->bound : 1.0);
    const int ld = kr + 1;
    for (int j = 0; j < kr; ++j) {
        apply(A, V + (size_t)j * n, 1, w);
        for (int pass = 0; pass < 2; ++pass)
            for (int i = 0; i <= j; ++i) {
                const double h = dot(V + (size_t)i * n, w, n);
                for (int64_t t = 0; t < n; ++t) w[t] += -h * V[(size_t)i * n + t];
                Hs[j * ld + i] += h;
            }
        const double nrm = sqrt(dot(w, w, n));
        kg = j + 1;
        if (nrm <= tiny) {
            beta = 0.0;
            break;
        }
        Hs[j * ld + j + 1] = nrm;
        beta = nrm;
        for (int64_t t = 0; t < n; ++t) V[(size_t)(j + 1) * n + t] = w[t] / nrm;
    }
    double* Hk = xcalloc((size_t)kg * kg, sizeof(double));
    for (int i = 0; i < kg; ++i)
        for (int j = 0; j < kg; ++j) Hk[j * kg + i] = Hs[j * ld + i];
    Prec p = {0};
    p.kind = 2;
    p.A = A;
    p.k = kg;
    p.roots = xcalloc((size_t)kg, sizeof(double));
    harmonic_ritz(Hk, kg, kg == kr ? beta : 0.0, p.roots);
    leja(p.roots, kg);
    free(Hk);
    free(V);
    free(Hs);
    free(w);
    return p;
}

/* Preconditioner::apply: Jacobi (preconditioners.cpp:54-68), GMRES product form (:171-193) */
static void prec_apply(const Prec* M, const double* R, int m, int64_t n, double* H) {
    if (M->kind == 1) {
        for (int64_t i = 0; i < n; ++i)
            for (int c = 0; c < m; ++c) H[(size_t)c * n + i] = M->inv[i] * R[(size_t)c * n + i];
        return;
    }
    if (M->kind == 0) {
        memcpy(H, R, sizeof(double) * (size_t)n * m);
        return;
    }
    const size_t sz = (size_t)n * m;
    double* prod = xcalloc(sz, sizeof(double));
    double* AP = xcalloc(sz, sizeof(double));
    memcpy(prod, R, sizeof(double) * sz);
    memset(H, 0, sizeof(double) * sz);
    for (int i = 0; i < M->k; ++i) {
        const double inv = 1.0 / M->roots[i];
        for (size_t t = 0; t < sz; ++t) H[t] += inv * prod[t];
        if (i + 1 < M->k) {
            apply(M->A, prod, m, AP);
            for (size_t t = 0; t < sz; ++t) prod[t] -= inv * AP[t];
        }
    }
    free(prod);
    free(AP);
}

/* --------------------------------------------------------------- LOBPCG */
typedef struct {
    const Op* A;
    const double* bd; /* B diagonal or NULL */
    int64_t n;
} Prob;

/* b_orthonormalize (eigensolver.cpp:88-129); returns the kept count, V compacted */
static int b_orth(const Prob* P, double* V, int cols, const double* against, int acols) {
    const int64_t n = P->n;
    double* s = xcalloc((size_t)n, sizeof(double));
#define BV(v) (P->bd ? (({ for (int64_t _i = 0; _i < n; ++_i) s[_i] = P->bd[_i] * (v)[_i]; }), s) : (v))
    int out = 0;
    for (int j = 0; j < cols; ++j) {
        double* vj = V + (size_t)j * n;
        double o = dot(vj, BV(vj), n);
        const double orig = sqrt(o > 0.0 ? o : 0.0);
        if (orig == 0.0) continue;
        for (int pass = 0; pass < 2; ++pass) {
            for (int q = 0; q < acols; ++q) {
                const double* aq = against + (size_t)q * n;
                const double c = dot(aq, BV(vj), n);
                for (int64_t t = 0; t < n; ++t) vj[t] += -c * aq[t];
            }
            for (int q = 0; q < out; ++q) {
                const double* vq = V + (size_t)q * n;
                const double c = dot(vq, BV(vj), n);
                for (int64_t t = 0; t < n; ++t) vj[t] += -c * vq[t];
            }
        }
        double nn = dot(vj, BV(vj), n);
        const double nrm = sqrt(nn > 0.0 ? nn : 0.0);
        if (nrm < 1e-10 * orig) continue;
        const double inv = 1.0 / nrm;
        double* dst = V + (size_t)out * n;
        if (dst != vj) memcpy(dst, vj, sizeof(double) * (size_t)n);
        for (int64_t t = 0; t < n; ++t) dst[t] *= inv;
        ++out;
    }
#undef BV
    free(s);
    return out;
}

/* projected_eig (eigensolver.cpp:138-155) */
static void projected_eig(const Prob* P, const double* Q, int m, int nev, double* theta, double* Y) {
    const int64_t n = P->n;
    double* AQ = xcalloc((size_t)n * m, sizeof(double));
    double* H = xcalloc((size_t)m * m, sizeof(double));
    double* vals = xcalloc((size_t)m, sizeof(double));
    double* vecs = xcalloc((size_t)m * m, sizeof(double));
    apply(P->A, Q, m, AQ);
    gram(Q, m, AQ, m, n, H);
    for (int j = 0; j < m; ++j)
        for (int i = 0; i < j; ++i) {
            const double sv = 0.5 * (H[j * m + i] + H[i * m + j]);
            H[j * m + i] = H[i * m + j] = sv;
        }
    sym_eig(H, m, vals, vecs);
    memcpy(theta, vals, sizeof(double) * (size_t)nev);
    memcpy(Y, vecs, sizeof(double) * (size_t)m * nev);
    free(AQ);
    free(H);
    free(vals);
    free(vecs);
}

typedef struct {
    int iterations, retries;
    double theta[SP_MAX_EIG], res[SP_MAX_EIG];
    uint8_t conv[SP_MAX_EIG];
} Eig;

static int all_conv(const Eig* e, int nev) {
    for (int j = 0; j < nev; ++j)
        if (!e->conv[j]) return 0;
    return nev > 0;
}

/* lobpcg (eigensolver.cpp:177-337); X (n x nev) in: X0, out: eigenvectors */
static void lobpcg(const Prob* P, const Prec* M, double* X, int nev, double tol, int max_iters, int locking, Eig* E) {
    const int64_t n = P->n;
    if (nev < 1) fail(SP_INFEASIBLE, "lobpcg: nev < 1");
    if (nev > n) fail(SP_INFEASIBLE, "lobpcg: nev > n");
    if (!(tol > 0.0)) fail(SP_INFEASIBLE, "lobpcg: tol must be positive");
    if (max_iters < 1) fail(SP_INFEASIBLE, "lobpcg: max_iters < 1");
    const double cs = P->A->bound > 0.0 ? (P->A->bound < 1.0 ? P->A->bound : 1.0) : 1.0;
    memset(E, 0, sizeof *E);
    const size_t blk = (size_t)n * nev;
    double* R = xcalloc(blk, sizeof(double));
    double* BX = xcalloc(blk, sizeof(double));
    double* Pd = xcalloc(blk, sizeof(double));
    double* S = xcalloc(blk * 3, sizeof(double));
    double* Xo = xcalloc(blk, sizeof(double));
    double* RI = xcalloc(blk, sizeof(double));
    double* HI = xcalloc(blk, sizeof(double));
    double* Y = xcalloc((size_t)3 * nev * nev, sizeof(double));
    double* Yhp = xcalloc((size_t)3 * nev * nev, sizeof(double));
    int pcols = 0, iter = 0, retried = 0;
    double theta[SP_MAX_EIG];
    int active[SP_MAX_EIG];

#define UPDATE_RES()                                                                              \
    do {                                                                                          \
        apply(P->A, X, nev, R);                                                                   \
        for (size_t t = 0; t < blk; ++t) BX[t] = P->bd ? P->bd[t % n] * X[t] : X[t];              \
        for (int j = 0; j < nev; ++j) {                                                           \
            double* rj = R + (size_t)j * n;                                                       \
            const double* bx = BX + (size_t)j * n;                                                \
            for (int64_t i = 0; i < n; ++i) rj[i] -= theta[j] * bx[i];                            \
            E->res[j] = sqrt(dot(rj, rj, n));                                                     \
            E->conv[j] = E->res[j] <= tol * cs ? 1 : 0;                                           \
        }                                                                                         \
    } while (0)

    for (;;) {
        memcpy(Xo, X, sizeof(double) * blk);
        const int kept = b_orth(P, Xo, nev, NULL, 0);
        if (kept < nev) {
            if (retried) {
                snprintf(g_err, sizeof g_err, "eigensolver breakdown at iteration %d (after retry without search directions)", iter);
                fail(SP_BREAKDOWN, g_err);
            }
            retried = 1;
            ++E->retries;
            continue;
        }
        projected_eig(P, Xo, nev, nev, theta, Y);
        mult(Xo, nev, Y, nev, n, X);
        break;
    }
    UPDATE_RES();
    while (iter < max_iters && !all_conv(E, nev)) {
        ++iter;
        int na = 0;
        for (int j = 0; j < nev; ++j)
            if (!locking || !E->conv[j]) active[na++] = j;
        for (int a = 0; a < na; ++a) memcpy(RI + (size_t)a * n, R + (size_t)active[a] * n, sizeof(double) * (size_t)n);
        prec_apply(M, RI, na, n, HI);
        int m = 0, hp = 0;
        for (;;) {
            memcpy(S, X, sizeof(double) * blk);
            const int kx = b_orth(P, S, nev, NULL, 0);
            if (kx < nev) {
                if (retried) {
                    snprintf(g_err, sizeof g_err, "eigensolver breakdown at iteration %d (after retry without search directions)", iter);
                    fail(SP_BREAKDOWN, g_err);
                }
                retried = 1;
                ++E->retries;
                pcols = 0;
                continue;
            }
            memcpy(S + (size_t)kx * n, HI, sizeof(double) * (size_t)n * na);
            const int kh = b_orth(P, S + (size_t)kx * n, na, S, kx);
            int kp = 0;
            if (pcols > 0) {
                memcpy(S + (size_t)(kx + kh) * n, Pd, sizeof(double) * (size_t)n * pcols);
                kp = b_orth(P, S + (size_t)(kx + kh) * n, pcols, S, kx + kh);
            }
            m = kx + kh + kp;
            hp = kx;
            break;
        }
        projected_eig(P, S, m, nev, theta, Y);
        mult(S, m, Y, nev, n, X);
        UPDATE_RES();
        int nn = 0;
        for (int j = 0; j < nev; ++j)
            if (!locking || !E->conv[j]) active[nn++] = j;
        const int hpc = m - hp;
        if (hpc > 0 && nn > 0) {
            for (int a = 0; a < nn; ++a)
                for (int r = 0; r < hpc; ++r) Yhp[a * hpc + r] = Y[(size_t)active[a] * m + hp + r];
            mult(S + (size_t)hp * n, hpc, Yhp, nn, n, Pd);
            pcols = nn;
        } else {
            pcols = 0;
        }
    }
#undef UPDATE_RES
    E->iterations = iter;
    memcpy(E->theta, theta, sizeof(double) * (size_t)nev);
    free(R);
    free(BX);
    free(Pd);
    free(S);
    free(Xo);
    free(RI);
    free(HI);
    free(Y);
    free(Yhp);
}

/* --------------------------------------------------------------- MJ (partitioner.cpp) */
typedef struct Node {
    int64_t leaves;
    int dim, nk;
    struct Node* kids;
} Node;

static void plan(Node* nd, int64_t target, int dim, int rem) { /* build_plan :43-61 */
    nd->leaves = target;
    nd->dim = -1;
    nd->nk = 0;
    nd->kids = NULL;
    if (target <= 1 || rem <= 0) return;
    int64_t m = (int64_t)ceil(pow((double)target, 1.0 / rem) - 1e-12);
    if (m < 2) m = 2;
    if (m > target) m = target;
    nd->dim = dim;
    nd->nk = (int)m;
    nd->kids = xcalloc((size_t)m, sizeof(Node));
    for (int64_t s = 0; s < m; ++s) plan(&nd->kids[s], target / m + (s < target % m ? 1 : 0), dim + 1, rem - 1);
}

static int64_t leaf_count(const Node* nd) {
    if (!nd->nk) return 1;
    int64_t t = 0;
    for (int s = 0; s < nd->nk; ++s) t += leaf_count(&nd->kids[s]);
    return t;
}

static void plan_free(Node* nd) {
    for (int s = 0; s < nd->nk; ++s) plan_free(&nd->kids[s]);
    free(nd->kids);
}

typedef struct {
    const double* coords;
    int64_t n;
    int dims;
    const double* w;
    int32_t* asg;
    int32_t next;
} MjSt;

static const double* g_sortcol;
static int cmp_ids(const void* pa, const void* pb) {
    const int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
    const double ca = g_sortcol[a], cb = g_sortcol[b];
    if (ca != cb) return ca < cb ? -1 : 1;
    return a < b ? -1 : (a > b);
}

static void mj_rec(MjSt* st, const Node* nd, int64_t* ids, int64_t cnt) { /* mj_recurse :86-136 */
    if (!nd->nk) {
        const int32_t part = st->next++;
        for (int64_t t = 0; t < cnt; ++t) st->asg[ids[t]] = part;
        return;
    }
    g_sortcol = st->coords + (size_t)(nd->dim % st->dims) * st->n;
    qsort(ids, (size_t)cnt, sizeof(int64_t), cmp_ids);
    double tw = 0.0;
    for (int64_t t = 0; t < cnt; ++t) tw += st->w ? st->w[ids[t]] : 1.0;
    int64_t pos = 0, done = 0;
    double consumed = 0.0;
    for (int s = 0; s < nd->nk; ++s) {
        const Node* ch = &nd->kids[s];
        done += leaf_count(ch);
        const int64_t begin = pos;
        if (s + 1 == nd->nk) {
            pos = cnt;
        } else {
            const double target = tw * (double)done / (double)nd->leaves;
            const int64_t max_take = cnt - pos - (nd->leaves - done), min_take = leaf_count(ch);
            int64_t taken = 0;
            while (pos < cnt && taken < max_take && (taken < min_take || consumed < target)) {
                consumed += st->w ? st->w[ids[pos]] : 1.0;
                ++pos;
                ++taken;
            }
        }
        int64_t* sub = xcalloc((size_t)(pos - begin), sizeof(int64_t));
        memcpy(sub, ids + begin, sizeof(int64_t) * (size_t)(pos - begin));
        mj_rec(st, ch, sub, pos - begin);
        free(sub);
    }
}

static void mj(const double* coords, int64_t n, int dims, const double* w, int64_t K, int32_t* asg) {
    if (K < 1) fail(SP_INFEASIBLE, "mj_partition: K < 1");
    if (n < K) fail(SP_INFEASIBLE, "mj_partition: fewer points than parts");
    if (w)
        for (int64_t i = 0; i < n; ++i)
            if (!(w[i] > 0.0)) fail(SP_INFEASIBLE, "mj_partition: weights must be positive");
    Node root;
    plan(&root, K, 0, dims);
    int64_t* ids = xcalloc((size_t)n, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) ids[i] = i;
    MjSt st = {coords, n, dims, w, asg, 0};
    mj_rec(&st, &root, ids, n);
    free(ids);
    plan_free(&root);
}

/* make_partition / cutsize / imbalance (graph.cpp:184-230) */
static void metrics(const sp_graph* g, const int32_t* a, int64_t K, int doubled, double* cut, double* imb, double* pw) {
    for (int64_t k = 0; k < K; ++k) pw[k] = 0.0;
    for (int64_t v = 0; v < g->n; ++v) {
        if (a[v] < 0 || a[v] >= K) fail(SP_INVALID, "make_partition: part id out of range");
        pw[a[v]] += g->vertex_weights ? g->vertex_weights[v] : 1.0;
    }
    for (int64_t k = 0; k < K; ++k)
        if (pw[k] <= 0.0) fail(SP_INVALID, "make_partition: empty part");
    double c = 0.0;
    for (int64_t i = 0; i < g->n; ++i)
        for (int64_t k = g->row_offsets[i]; k < g->row_offsets[i + 1]; ++k) {
            const int32_t j = g->col_indices[k];
            if (j > i && a[i] != a[j]) c += value_at(g, k);
        }
    *cut = doubled ? 2.0 * c : c;
    double tot = 0.0, mx = 0.0;
    for (int64_t k = 0; k < K; ++k) {
        tot += pw[k];
        if (pw[k] > mx) mx = pw[k];
    }
    *imb = mx / (tot / (double)K);
}

/* ---------------------------------------------------------------- exports */
int ref_build_laplacian(int32_t kind, const sp_graph* g, int64_t* offs, int32_t* cols, double* vals, double* diag,
                        double* bound, int32_t* isdiag) {
    GUARD_BEGIN
    Op o = build_kind(kind, g);
    const int64_t nnz = o.offs[o.n];
    if (offs) memcpy(offs, o.offs, sizeof(int64_t) * (size_t)(o.n + 1));
    if (cols) memcpy(cols, o.cols, sizeof(int32_t) * (size_t)nnz);
    if (vals) memcpy(vals, o.vals, sizeof(double) * (size_t)nnz);
    if (diag) memcpy(diag, o.diag, sizeof(double) * (size_t)o.n);
    if (bound) *bound = o.bound;
    if (isdiag) *isdiag = o.is_diag;
    op_free(&o);
    GUARD_END
}

int ref_spmm(int32_t kind, const sp_graph* g, const double* X, int32_t m, double* Y) {
    GUARD_BEGIN
    Op o = build_kind(kind, g);
    apply(&o, X, m, Y);
    op_free(&o);
    GUARD_END
}

int ref_spmm_csr(int64_t nrows, int64_t ncols, const int64_t* offs, const int32_t* cols, const double* vals,
                 const double* X, int32_t m, double* Y) {
    GUARD_BEGIN
    (void)ncols;
    for (int64_t i = 0; i < nrows; ++i)
        for (int c = 0; c < m; ++c) {
            double acc = 0.0;
            for (int64_t k = offs[i]; k < offs[i + 1]; ++k) acc += (vals ? vals[k] : 1.0) * X[(size_t)c * ncols + cols[k]];
            Y[(size_t)c * nrows + i] = acc;
        }
    GUARD_END
}

int ref_gram(int64_t n, const double* U, int32_t mu, const double* V, int32_t mv, const double* b, double* G) {
    GUARD_BEGIN
    double* BV = NULL;
    if (b) {
        BV = xcalloc((size_t)n * mv, sizeof(double));
        for (int j = 0; j < mv; ++j)
            for (int64_t i = 0; i < n; ++i) BV[(size_t)j * n + i] = b[i] * V[(size_t)j * n + i];
    }
    gram(U, mu, b ? BV : V, mv, n, G);
    free(BV);
    GUARD_END
}

int ref_initial_guess(int32_t init, int64_t n, int32_t d, uint64_t seed, double* X) {
    GUARD_BEGIN
    init_block(init, n, d, seed, X);
    GUARD_END
}

int ref_sym_eig(int32_t m, const double* A, double* vals, double* vecs) {
    GUARD_BEGIN
    sym_eig(A, m, vals, vecs);
    GUARD_END
}

int ref_mj_partition(int64_t n, int32_t dims, const double* coords, const double* w, int64_t K, int32_t* asg,
                     double* pw, double* imb) {
    GUARD_BEGIN
    mj(coords, n, dims, w, K, asg);
    double* p = xcalloc((size_t)K, sizeof(double));
    for (int64_t v = 0; v < n; ++v) p[asg[v]] += w ? w[v] : 1.0;
    double tot = 0.0, mx = 0.0;
    for (int64_t k = 0; k < K; ++k) {
        tot += p[k];
        if (p[k] > mx) mx = p[k];
    }
    if (pw) memcpy(pw, p, sizeof(double) * (size_t)K);
    if (imb) *imb = mx / (tot / (double)K);
    free(p);
    GUARD_END
}

int ref_cut_imbalance(const sp_graph* g, const int32_t* a, int64_t K, int32_t doubled, double* cut, double* imb,
                      double* pw) {
    GUARD_BEGIN
    double* p = xcalloc((size_t)K, sizeof(double));
    double c = 0.0, im = 0.0;
    metrics(g, a, K, doubled, &c, &im, p);
    if (cut) *cut = c;
    if (imb) *imb = im;
    if (pw) memcpy(pw, p, sizeof(double) * (size_t)K);
    free(p);
    GUARD_END
}

static Prob make_prob(const sp_graph* g, int problem, Op* A, Op* D) {
    Prob P = {0};
    memset(D, 0, sizeof *D);
    *A = build_kind(problem == SP_PROBLEM_NORMALIZED ? SP_LAP_NORMALIZED : SP_LAP_COMBINATORIAL, g);
    P.A = A;
    P.n = g->n;
    if (problem == SP_PROBLEM_GENERALIZED) {
        *D = build_deg(g);
        for (int64_t i = 0; i < g->n; ++i)
            if (!(D->diag[i] > 0.0)) fail(SP_DEGENERATE, "generalized problem requires positive degrees");
        P.bd = D->diag;
    }
    return P;
}

static Prec make_prec(const Op* A, int precond, uint64_t pseed, int pdeg) {
    Prec M = {0};
    if (precond == SP_PRECOND_JACOBI) {
        M.kind = 1;
        M.inv = xcalloc((size_t)A->n, sizeof(double));
        for (int64_t i = 0; i < A->n; ++i) M.inv[i] = fabs(A->diag[i]) < 1e-300 ? 1.0 : 1.0 / A->diag[i];
    } else if (precond == SP_PRECOND_POLYNOMIAL) {
        M = poly_build(A, pseed, pdeg > 0 ? pdeg : 25);
    }
    return M;
}

int ref_lobpcg(const sp_graph* g, int32_t problem, int32_t precond, uint64_t pseed, int32_t pdeg, const double* X0,
               int32_t nev, double tol, int32_t max_iters, int32_t locking, double* theta, double* X, double* res,
               uint8_t* conv, int32_t* iters, int32_t* retries) {
    GUARD_BEGIN
    Op A, D;
    Prob P = make_prob(g, problem, &A, &D);
    Prec M = make_prec(&A, precond, pseed, pdeg);
    double* Xw = xcalloc((size_t)g->n * nev, sizeof(double));
    memcpy(Xw, X0, sizeof(double) * (size_t)g->n * nev);
    Eig E;
    lobpcg(&P, &M, Xw, nev, tol, max_iters, locking, &E);
    for (int j = 0; j < nev; ++j) {
        theta[j] = E.theta[j];
        if (res) res[j] = E.res[j];
        if (conv) conv[j] = E.conv[j];
    }
    if (X) memcpy(X, Xw, sizeof(double) * (size_t)g->n * nev);
    if (iters) *iters = E.iterations;
    if (retries) *retries = E.retries;
    free(Xw);
    free(M.inv);
    free(M.roots);
    op_free(&A);
    op_free(&D);
    GUARD_END
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* partition_graph (pipeline.cpp:47-167) */
int ref_partition(const sp_graph* g, const sp_config* c, int32_t* asg, sp_report* rep, const double* x0) {
    GUARD_BEGIN
    if (x0) fail(SP_INVALID, "ref_partition: explicit X0 not supported");
    const int64_t n = g->n, K = c->num_parts;
    if (K < 2) fail(SP_INFEASIBLE, "partition_graph: K must be >= 2");
    if (K > n) fail(SP_INFEASIBLE, "partition_graph: K exceeds vertex count");
    if (c->epsilon < 0.0) fail(SP_INFEASIBLE, "partition_graph: epsilon < 0");
    const double t0 = now_s();
    int64_t maxd = 0;
    for (int64_t v = 0; v < n; ++v)
        if (g->row_offsets[v + 1] - g->row_offsets[v] > maxd) maxd = g->row_offsets[v + 1] - g->row_offsets[v];
    const double avg = (double)g->row_offsets[n] / (double)n;
    const double ratio = avg > 0.0 ? (double)maxd / avg : (maxd > 0 ? INFINITY : 0.0);
    const int regular = ratio <= 10.0;
    int precond = c->precond == SP_PRECOND_AUTO ? (regular ? SP_PRECOND_AMG : SP_PRECOND_POLYNOMIAL) : c->precond;
    if (precond == SP_PRECOND_AMG) fail(SP_ERROR, "AMG is not restated by the C oracle");
    int aprob;
    double atol;
    if (precond == SP_PRECOND_POLYNOMIAL) {
        aprob = regular ? SP_PROBLEM_COMBINATORIAL : SP_PROBLEM_NORMALIZED;
        atol = regular ? 1e-3 : 1e-2;
    } else {
        aprob = regular ? SP_PROBLEM_COMBINATORIAL : SP_PROBLEM_GENERALIZED;
        atol = regular ? 1e-3 : 1e-2;
    }
    const int problem = c->problem == SP_PROBLEM_AUTO ? aprob : c->problem;
    const double tol = c->tol > 0.0 ? c->tol : atol;
    const int init = c->init == SP_INIT_AUTO ? (regular ? SP_INIT_RANDOM : SP_INIT_PIECEWISE) : c->init;
    int d = 0;
    for (uint64_t k = (uint64_t)K; k; k >>= 1) ++d; /* bit_width */
    if (d > n) fail(SP_INFEASIBLE, "partition_graph: d > n");
    const double tl = now_s();
    Op A, D;
    Prob P = make_prob(g, problem, &A, &D);
    const double te = now_s();
    Prec M = make_prec(&A, precond, c->seed ^ 0x706f6c79ULL, 25);
    double* X = xcalloc((size_t)n * d, sizeof(double));
    init_block(init, n, d, c->seed, X);
    Eig E;
    lobpcg(&P, &M, X, d, tol, c->max_iters, 1, &E);
    const double tm = now_s();
    mj(X + (size_t)n, n, d - 1, g->vertex_weights, K, asg);
    const double tp = now_s();
    double* pw = xcalloc((size_t)K, sizeof(double));
    double cut = 0.0, imb = 0.0;
    metrics(g, asg, K, c->doubled_cut, &cut, &imb, pw);
    if (rep) {
        double* keep_pw = rep->part_weights;
        sp_trace_record* keep_tr = rep->trace;
        const int32_t cap = rep->trace_capacity;
        memset(rep, 0, sizeof *rep);
        rep->part_weights = keep_pw;
        rep->trace = keep_tr;
        rep->trace_capacity = cap;
        rep->n = n;
        rep->edges = g->row_offsets[n] / 2;
        rep->graph_regular = regular;
        rep->max_degree = maxd;
        rep->avg_degree = avg;
        rep->degree_ratio = ratio;
        rep->num_parts = K;
        rep->problem = problem;
        rep->precond = precond;
        rep->tol = tol;
        rep->init = init;
        rep->eigenvectors = d;
        rep->seed = c->seed;
        rep->max_iters = c->max_iters;
        rep->doubled_cut = c->doubled_cut;
        rep->epsilon = c->epsilon;
        rep->iterations = E.iterations;
        rep->breakdown_retries = E.retries;
        for (int j = 0; j < d; ++j) {
            rep->theta[j] = E.theta[j];
            rep->residual_norms[j] = E.res[j];
            rep->converged[j] = E.conv[j];
        }
        rep->poly_degree = M.kind == 2 ? M.k : 0;
        if (E.retries) rep->warnings |= SP_WARN_BREAKDOWN_RECOVERED;
        if (!all_conv(&E, d)) rep->warnings |= SP_WARN_UNCONVERGED;
        if (imb > 1.0 + c->epsilon) rep->warnings |= SP_WARN_IMBALANCE;
        rep->laplacian_s = te - tl;
        rep->eigensolve_s = tm - te;
        rep->partition_s = tp - tm;
        rep->total_s = now_s() - t0;
        rep->cutsize = cut;
        rep->imbalance = imb;
        if (keep_pw) memcpy(keep_pw, pw, sizeof(double) * (size_t)K);
    }
    free(pw);
    free(X);
    free(M.inv);
    free(M.roots);
    op_free(&A);
    op_free(&D);
    GUARD_END
}
