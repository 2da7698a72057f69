/*
 * TEST INFRASTRUCTURE — CPU ORACLE, NOT PRODUCT CODE.
 *
 * A plain-C restatement of the BlocKOA reference hot path (arxiv 2510.23221,
 * /root/reference/proj/core), used only by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg as the checker. The GPU product never links or
 * calls this file.
 *
 * Parity pinning: every function here is checked in tests/test_oracle.py against
 * the unmodified reference compiled from source (oracle/_ref, see Makefile) and
 * against the golden fixtures in tests/golden (generated from oracle/_ref by
 * tests/golden/make_golden.py), and against the SPEC.md known-answer examples.
 *
 * Functions and the reference code they restate:
 *   orc_assemble        discretize.cpp:114-237 (7-point FV, harmonic faces,
 *                       Dirichlet half-cell, Robin series h_eff, CSR push order
 *                       z-,y-,x-,diag,x+,y+,z+ skipping zero off-diagonals).
 *                       Extensions: face kind 2 = adiabatic
 *                       (zero flux) and optional per-layer dz (non-uniform z);
 *                       with equal dz the reference expressions are used, so the
 *                       result is bitwise the reference's.
 *   orc_apply_block     CsrMatrix::apply_block discretize.cpp:57-95
 *   orc_block_cg        block_cg solvers.cpp:452-665 with PivotedCholesky
 *                       solvers.cpp:347-426 and jacobi_inverse solvers.cpp:53-66
 *   orc_cg              cg solvers.cpp:82-171
 *   orc_combine_action  combine_from_weights pipeline.cpp:187-225 +
 *                       operator_action pipeline.cpp:242-251 +
 *                       relative_residual discretize.cpp:275-286
 *   orc_rng_*           Rng / derive_seed rng.hpp:14-63, rng.cpp:8-60
 *   orc_field_digest    field_digest discretize.cpp:302-319
 *
 * Floating point: built with -ffp-contract=off; the places where the reference
 * build (g++ -O3, default -ffp-contract=fast) contracts `acc += a*b` are written
 * as explicit fma() so apply_block matches the reference bitwise.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_INVALID_SPEC 1
#define ORC_INVALID_CONFIG 2
#define ORC_DIM 3
#define ORC_NONPOS_K 4
#define ORC_NONPOS_H 5
#define ORC_EMPTY 6
#define ORC_OOM 21

/* ------------------------------------------------------------------------- */
/* RNG: xoshiro256** seeded by splitmix64 (rng.hpp:14-63, rng.cpp:8-60)      */
/* ------------------------------------------------------------------------- */
typedef struct {
    uint64_t s[4];
    double spare;
    int have_spare;
} orc_rng;

static uint64_t sm64_next(uint64_t* st) {
    uint64_t z = (*st += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static void rng_init(orc_rng* r, uint64_t seed) {
    uint64_t st = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = sm64_next(&st);
    r->spare = 0.0;
    r->have_spare = 0;
}

static uint64_t rng_u64(orc_rng* r) {
    uint64_t* s = r->s;
    const uint64_t out = rotl64(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return out;
}

static double rng_u01(orc_rng* r) { return (double)(rng_u64(r) >> 11) * 0x1.0p-53; }

static double rng_normal(orc_rng* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    const double u1 = 1.0 - rng_u01(r);
    const double u2 = rng_u01(r);
    const double rad = sqrt(-2.0 * log(u1));
    const double th = 2.0 * 3.141592653589793 * u2;
    r->spare = rad * sin(th);
    r->have_spare = 1;
    return rad * cos(th);
}

static uint64_t rng_below(orc_rng* r, uint64_t n) {
    const uint64_t lim = n * (~(uint64_t)0 / n);
    uint64_t x;
    do {
        x = rng_u64(r);
    } while (x >= lim);
    return x % n;
}

uint64_t orc_derive_seed(uint64_t seed, const char* tag, uint64_t index) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (const unsigned char* c = (const unsigned char*)tag; *c; ++c) {
        h ^= *c;
        h *= 0x100000001b3ULL;
    }
    uint64_t st = seed;
    const uint64_t mixed = sm64_next(&st) ^ h;
    st = mixed + 0x632be59bd9b4e019ULL * (index + 1);
    return sm64_next(&st);
}

void orc_rng_u64(uint64_t seed, int64_t n, uint64_t* out) {
    orc_rng r;
    rng_init(&r, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng_u64(&r);
}
void orc_rng_uniform(uint64_t seed, double lo, double hi, int64_t n, double* out) {
    orc_rng r;
    rng_init(&r, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = lo + rng_u01(&r) * (hi - lo);
}
void orc_rng_normal(uint64_t seed, int64_t n, double* out) {
    orc_rng r;
    rng_init(&r, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng_normal(&r);
}
void orc_rng_below(uint64_t seed, uint64_t bound, int64_t n, uint64_t* out) {
    orc_rng r;
    rng_init(&r, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng_below(&r, bound);
}

/* ------------------------------------------------------------------------- */
/* Assembly (discretize.cpp:114-237)                                          */
/* ------------------------------------------------------------------------- */
typedef struct {
    int64_t n;
    int64_t nnz;
    int64_t* row_ptr; /* n+1 */
    int32_t* col;     /* nnz */
    double* val;      /* nnz */
    double* g;        /* n */
    double* vol;      /* n */
    double* dinv;     /* n, jacobi_inverse */
} orc_op;

/* Boundary face (discretize.cpp:151-165). kind: 0 Dirichlet(a=u0), 1 Robin(a=h,
 * b=u_inf), 2 adiabatic (no conductance, no lift). */
static void bface(int kind, double a, double b, double kc, double area, double delta,
                  double* diag, double* lift) {
    if (kind == 0) {
        const double gf = (2.0 * kc / delta) * area;
        *diag += gf;
        *lift = fma(gf, a, *lift);
    } else if (kind == 1) {
        const double heff = 1.0 / (delta / (2.0 * kc) + 1.0 / a);
        const double gf = heff * area;
        *diag += gf;
        *lift = fma(gf, b, *lift);
    }
}

static double harm(double ki, double kj, double area, double delta) {
    return (2.0 * ki * kj / (ki + kj)) * (area / delta);
}

/* z-face between layers with thicknesses da (cell a) and db (cell b); equal
 * thicknesses use the reference's harmonic form exactly. */
static double zface(double ka, double kb, double da, double db, double area) {
    if (da == db) return harm(ka, kb, area, da);
    return area / (da / (2.0 * ka) + db / (2.0 * kb));
}

void orc_op_free(orc_op* op) {
    if (!op) return;
    free(op->row_ptr);
    free(op->col);
    free(op->val);
    free(op->g);
    free(op->vol);
    free(op->dinv);
    free(op);
}

/* dz: NULL for the reference's uniform grid (dz = lz/nz), else nz thicknesses. */
int orc_assemble(int nx, int ny, int nz, double lx, double ly, double lz,
                 const double* dzs, const double* k, const int* bk, const double* ba,
                 const double* bb, orc_op** out) {
    if (nx < 1 || ny < 1 || nz < 1 || !(lx > 0) || !(ly > 0) || !(lz > 0))
        return ORC_INVALID_SPEC;
    for (int f = 0; f < 6; ++f)
        if (bk[f] == 1 && !(ba[f] > 0.0)) return ORC_NONPOS_H;
    const int64_t n = (int64_t)nx * ny * nz;
    if (n > 2147483647LL) return ORC_INVALID_SPEC;
    for (int64_t i = 0; i < n; ++i)
        if (!(k[i] > 0.0)) return ORC_NONPOS_K;
    if (dzs)
        for (int z = 0; z < nz; ++z)
            if (!(dzs[z] > 0.0)) return ORC_INVALID_SPEC;

    orc_op* op = (orc_op*)calloc(1, sizeof(orc_op));
    op->n = n;
    op->row_ptr = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    op->col = (int32_t*)malloc((size_t)n * 7 * sizeof(int32_t));
    op->val = (double*)malloc((size_t)n * 7 * sizeof(double));
    op->g = (double*)calloc((size_t)n, sizeof(double));
    op->vol = (double*)malloc((size_t)n * sizeof(double));
    op->dinv = (double*)malloc((size_t)n * sizeof(double));
    if (!op->row_ptr || !op->col || !op->val || !op->g || !op->vol || !op->dinv) {
        orc_op_free(op);
        return ORC_OOM;
    }
    const double dx = lx / nx, dy = ly / ny, dzu = lz / nz;
    int64_t p = 0;
    for (int iz = 0; iz < nz; ++iz) {
        const double dz = dzs ? dzs[iz] : dzu;
        const double ax = dy * dz, ay = dx * dz, az = dx * dy;
        const double vol = dx * dy * dz;
        for (int iy = 0; iy < ny; ++iy) {
            for (int ix = 0; ix < nx; ++ix) {
                const int64_t i = ix + (int64_t)nx * (iy + (int64_t)ny * iz);
                const double kc = k[i];
                double diag = 0.0, lift = 0.0;
                double gzm = 0, gym = 0, gxm = 0, gxp = 0, gyp = 0, gzp = 0;
                if (iz > 0) {
                    const double dzo = dzs ? dzs[iz - 1] : dzu;
                    gzm = zface(kc, k[i - (int64_t)nx * ny], dz, dzo, az);
                } else
                    bface(bk[4], ba[4], bb[4], kc, az, dz, &diag, &lift);
                if (iy > 0)
                    gym = harm(kc, k[i - nx], ay, dy);
                else
                    bface(bk[2], ba[2], bb[2], kc, ay, dy, &diag, &lift);
                if (ix > 0)
                    gxm = harm(kc, k[i - 1], ax, dx);
                else
                    bface(bk[0], ba[0], bb[0], kc, ax, dx, &diag, &lift);
                if (ix < nx - 1)
                    gxp = harm(kc, k[i + 1], ax, dx);
                else
                    bface(bk[1], ba[1], bb[1], kc, ax, dx, &diag, &lift);
                if (iy < ny - 1)
                    gyp = harm(kc, k[i + nx], ay, dy);
                else
                    bface(bk[3], ba[3], bb[3], kc, ay, dy, &diag, &lift);
                if (iz < nz - 1) {
                    const double dzo = dzs ? dzs[iz + 1] : dzu;
                    gzp = zface(kc, k[i + (int64_t)nx * ny], dz, dzo, az);
                } else
                    bface(bk[5], ba[5], bb[5], kc, az, dz, &diag, &lift);
                diag += gzm + gym + gxm + gxp + gyp + gzp;
#define PUSH(j, v)                      \
    do {                                \
        op->col[p] = (int32_t)(j);      \
        op->val[p] = (v);               \
        ++p;                            \
    } while (0)
                if (gzm != 0.0) PUSH(i - (int64_t)nx * ny, -gzm);
                if (gym != 0.0) PUSH(i - nx, -gym);
                if (gxm != 0.0) PUSH(i - 1, -gxm);
                PUSH(i, diag);
                if (gxp != 0.0) PUSH(i + 1, -gxp);
                if (gyp != 0.0) PUSH(i + nx, -gyp);
                if (gzp != 0.0) PUSH(i + (int64_t)nx * ny, -gzp);
#undef PUSH
                op->row_ptr[i + 1] = p;
                op->g[i] = lift;
                op->vol[i] = vol;
                op->dinv[i] = diag != 0.0 ? 1.0 / diag : 1.0;
            }
        }
    }
    op->nnz = p;
    *out = op;
    return ORC_OK;
}

/* Generic CSR operator (g = 0, unit volumes) for the SPEC's matrix-level
 * examples (cg on diag(2,3), random SPD block_cg). */
int orc_op_from_csr(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                    orc_op** out) {
    orc_op* op = (orc_op*)calloc(1, sizeof(orc_op));
    const int64_t nnz = row_ptr[n];
    op->n = n;
    op->nnz = nnz;
    op->row_ptr = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
    op->col = (int32_t*)malloc((size_t)(nnz + 1) * sizeof(int32_t));
    op->val = (double*)malloc((size_t)(nnz + 1) * sizeof(double));
    op->g = (double*)calloc((size_t)n, sizeof(double));
    op->vol = (double*)malloc((size_t)n * sizeof(double));
    op->dinv = (double*)malloc((size_t)n * sizeof(double));
    memcpy(op->row_ptr, row_ptr, (size_t)(n + 1) * sizeof(int64_t));
    memcpy(op->col, col, (size_t)nnz * sizeof(int32_t));
    memcpy(op->val, val, (size_t)nnz * sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        op->vol[i] = 1.0;
        op->dinv[i] = 1.0;
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
            if (col[p] == i) {
                if (val[p] != 0.0) op->dinv[i] = 1.0 / val[p];
                break;
            }
    }
    *out = op;
    return ORC_OK;
}

int64_t orc_op_nnz(const orc_op* op) { return op->nnz; }

void orc_op_export(const orc_op* op, int64_t* row_ptr, int32_t* col, double* val,
                   double* g, double* vol) {
    memcpy(row_ptr, op->row_ptr, (size_t)(op->n + 1) * sizeof(int64_t));
    memcpy(col, op->col, (size_t)op->nnz * sizeof(int32_t));
    memcpy(val, op->val, (size_t)op->nnz * sizeof(double));
    memcpy(g, op->g, (size_t)op->n * sizeof(double));
    memcpy(vol, op->vol, (size_t)op->n * sizeof(double));
}

/* Y = A X, X/Y row-major n x s; per-row CSR-order fused accumulation (the
 * reference's apply_block compiles to FMA chains). The single-vector
 * CsrMatrix::apply (discretize.cpp:39-51) compiles to separate mul+add; the
 * scalar sweeps below (operator action, residuals) restate it that way. The
 * reference build's apply_block_fixed<4> (S = 4 only) is vectorised without
 * contraction (mul + add); that width is restated the same way. */
void orc_apply_block(const orc_op* op, const double* x, int s, double* y) {
    double* acc = (double*)malloc((size_t)s * sizeof(double));
    for (int64_t i = 0; i < op->n; ++i) {
        for (int j = 0; j < s; ++j) acc[j] = 0.0;
        for (int64_t q = op->row_ptr[i]; q < op->row_ptr[i + 1]; ++q) {
            const double a = op->val[q];
            const double* xr = x + (int64_t)op->col[q] * s;
            if (s == 4)
                for (int j = 0; j < s; ++j) acc[j] += a * xr[j];
            else
                for (int j = 0; j < s; ++j) acc[j] = fma(a, xr[j], acc[j]);
        }
        for (int j = 0; j < s; ++j) y[i * s + j] = acc[j];
    }
    free(acc);
}

void orc_rhs_from_power(const orc_op* op, const double* q, double* b) {
    for (int64_t i = 0; i < op->n; ++i) b[i] = fma(op->vol[i], q[i], op->g[i]);
}

void orc_power_from_rhs(const orc_op* op, const double* b, double* q) {
    for (int64_t i = 0; i < op->n; ++i) q[i] = (b[i] - op->g[i]) / op->vol[i];
}

/* field_digest (discretize.cpp:302-319): FNV-1a 64 over nx, ny, nz (8 LE
 * bytes each) then every value's raw bits, low byte first. */
uint64_t orc_field_digest(int nx, int ny, int nz, const double* v) {
    uint64_t h = 0xcbf29ce484222325ULL;
    const uint64_t dims[3] = {(uint64_t)nx, (uint64_t)ny, (uint64_t)nz};
    const int64_t n = (int64_t)nx * ny * nz;
    for (int64_t w = 0; w < n + 3; ++w) {
        uint64_t word;
        if (w < 3)
            word = dims[w];
        else
            memcpy(&word, v + (w - 3), 8);
        for (int b = 0; b < 8; ++b) {
            h ^= (word >> (8 * b)) & 0xffu;
            h *= 0x100000001b3ULL;
        }
    }
    return h;
}

/* ||A u - (V q + g)|| / ||V q + g||  (discretize.cpp:275-286) */
double orc_relative_residual(const orc_op* op, const double* u, const double* q) {
    double nb = 0.0, nr = 0.0;
    for (int64_t i = 0; i < op->n; ++i) {
        double acc = 0.0;
        for (int64_t p = op->row_ptr[i]; p < op->row_ptr[i + 1]; ++p)
            acc += op->val[p] * u[op->col[p]]; /* CsrMatrix::apply: not contracted in the reference build */
        const double b = fma(op->vol[i], q[i], op->g[i]);
        const double r = b - acc;
        nb += b * b; /* norm2, discretize.cpp:269-273 */
        nr += r * r;
    }
    nb = sqrt(nb);
    nr = sqrt(nr);
    if (nb == 0.0) return nr == 0.0 ? 0.0 : INFINITY;
    return nr / nb;
}

/* ------------------------------------------------------------------------- */
/* Solvers                                                                    */
/* ------------------------------------------------------------------------- */

/* Diagonally pivoted Cholesky of an s x s SPSD matrix (solvers.cpp:347-388):
 * rank cutoff max(max_diag * s * eps, DBL_MIN); L row-major in pivot order. */
typedef struct {
    int s, rank;
    double* l;
    int* perm;
} pchol;

static void pchol_factor(pchol* c, const double* g, int s) {
    c->s = s;
    c->l = (double*)calloc((size_t)s * s, sizeof(double));
    c->perm = (int*)malloc((size_t)s * sizeof(int));
    double* d = (double*)malloc((size_t)s * sizeof(double));
    double maxd = 0.0;
    for (int i = 0; i < s; ++i) {
        c->perm[i] = i;
        d[i] = g[(size_t)i * s + i];
        if (d[i] > maxd) maxd = d[i];
    }
    double cutoff = maxd * s * 2.220446049250313e-16;
    if (cutoff < 2.2250738585072014e-308) cutoff = 2.2250738585072014e-308;
    c->rank = s;
    for (int k = 0; k < s; ++k) {
        int piv = k;
        for (int i = k + 1; i < s; ++i)
            if (d[c->perm[i]] > d[c->perm[piv]]) piv = i;
        if (!(d[c->perm[piv]] > cutoff)) {
            c->rank = k;
            break;
        }
        int tp = c->perm[k];
        c->perm[k] = c->perm[piv];
        c->perm[piv] = tp;
        for (int t = 0; t < k; ++t) {
            double tv = c->l[(size_t)k * s + t];
            c->l[(size_t)k * s + t] = c->l[(size_t)piv * s + t];
            c->l[(size_t)piv * s + t] = tv;
        }
        const int pk = c->perm[k];
        const double lkk = sqrt(d[pk]);
        c->l[(size_t)k * s + k] = lkk;
        for (int i = k + 1; i < s; ++i) {
            const int pi = c->perm[i];
            double v = g[(size_t)pi * s + pk];
            for (int t = 0; t < k; ++t) v -= c->l[(size_t)i * s + t] * c->l[(size_t)k * s + t];
            const double lik = v / lkk;
            c->l[(size_t)i * s + k] = lik;
            d[pi] -= lik * lik;
        }
    }
    free(d);
}

/* x = G^+ rhs for s x m rhs (solvers.cpp:392-414). */
static void pchol_solve(const pchol* c, const double* rhs, int m, double* x) {
    const int s = c->s;
    double* y = (double*)calloc((size_t)s * m, sizeof(double));
    for (int k = 0; k < c->rank; ++k) {
        const int pk = c->perm[k];
        for (int j = 0; j < m; ++j) {
            double v = rhs[(size_t)pk * m + j];
            for (int t = 0; t < k; ++t) v -= c->l[(size_t)k * s + t] * y[(size_t)t * m + j];
            y[(size_t)k * m + j] = v / c->l[(size_t)k * s + k];
        }
    }
    memset(x, 0, (size_t)s * m * sizeof(double));
    for (int k = c->rank - 1; k >= 0; --k) {
        const int pk = c->perm[k];
        for (int j = 0; j < m; ++j) {
            double v = y[(size_t)k * m + j];
            for (int t = k + 1; t < c->rank; ++t)
                v -= c->l[(size_t)t * s + k] * x[(size_t)c->perm[t] * m + j];
            x[(size_t)pk * m + j] = v / c->l[(size_t)k * s + k];
        }
    }
    free(y);
}

static void pchol_free(pchol* c) {
    free(c->l);
    free(c->perm);
}

/* out = lhs^T rhs over n rows (s x s). */
static void gram(const double* lhs, const double* rhs, int64_t n, int s, double* out) {
    memset(out, 0, (size_t)s * s * sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        const double* li = lhs + i * s;
        const double* ri = rhs + i * s;
        for (int a = 0; a < s; ++a) {
            const double la = li[a];
            double* oa = out + (size_t)a * s;
            for (int b = 0; b < s; ++b) oa[b] = fma(la, ri[b], oa[b]);
        }
    }
}

/* dst += sign * src * m  (n x s by s x s) */
static void add_product(double* dst, const double* src, const double* m, int64_t n, int s,
                        double sign) {
    for (int64_t i = 0; i < n; ++i) {
        const double* si = src + i * s;
        double* di = dst + i * s;
        for (int t = 0; t < s; ++t) {
            const double f = sign * si[t];
            const double* mt = m + (size_t)t * s;
            for (int j = 0; j < s; ++j) di[j] = fma(f, mt[j], di[j]);
        }
    }
}

static double true_rel_residual_col(const orc_op* op, const double* b, int bs, int bj,
                                    const double* x, int xs, int xj, double bnorm) {
    double acc2 = 0.0;
    for (int64_t i = 0; i < op->n; ++i) {
        double acc = 0.0;
        for (int64_t p = op->row_ptr[i]; p < op->row_ptr[i + 1]; ++p)
            acc += op->val[p] * x[(int64_t)op->col[p] * xs + xj];
        const double r = b[i * bs + bj] - acc;
        acc2 += r * r;
    }
    return sqrt(acc2) / bnorm;
}

static void compact_cols(double* blk, int64_t n, int s_old, const int* keep, int s_new) {
    for (int64_t i = 0; i < n; ++i)
        for (int j = 0; j < s_new; ++j) blk[i * s_new + j] = blk[i * s_old + keep[j]];
}

static void compact_sq(double* m, int s_old, const int* keep, int s_new) {
    double* t = (double*)malloc((size_t)s_new * s_new * sizeof(double) + 8);
    for (int a = 0; a < s_new; ++a)
        for (int b = 0; b < s_new; ++b) t[a * s_new + b] = m[keep[a] * s_old + keep[b]];
    memcpy(m, t, (size_t)s_new * s_new * sizeof(double));
    free(t);
}

/* Block CG (solvers.cpp:452-665). b, x row-major n x s. */
int orc_block_cg(const orc_op* op, const double* b, int s, double tol, int max_iter,
                 int precond, double* x, int* iterations, int64_t* matvecs,
                 double* final_res, char* converged) {
    if (!(tol > 0.0) || !(tol < 1.0) || max_iter < 1) return ORC_INVALID_CONFIG;
    if (s < 1) return ORC_DIM;
    const int64_t n = op->n;
    const size_t ns = (size_t)n * s;
    memset(x, 0, ns * sizeof(double));
    *iterations = 0;
    *matvecs = 0;
    double* bnorm = (double*)calloc((size_t)s, sizeof(double));
    int* active = (int*)malloc((size_t)s * sizeof(int));
    int sa = 0;
    for (int j = 0; j < s; ++j) {
        double acc = 0.0;
        for (int64_t i = 0; i < n; ++i) acc += b[i * s + j] * b[i * s + j];
        bnorm[j] = sqrt(acc);
        final_res[j] = 0.0;
        converged[j] = 0;
        if (bnorm[j] == 0.0)
            converged[j] = 1;
        else
            active[sa++] = j;
    }
    const double* dinv = op->dinv;
    double *r = malloc(ns * 8 + 8), *z = malloc(ns * 8 + 8), *p = malloc(ns * 8 + 8),
           *w = malloc(ns * 8 + 8), *xa = calloc(ns + 1, 8);
    size_t ss = (size_t)s * s;
    double *s_old = calloc(ss + 1, 8), *s_new = calloc(ss + 1, 8), *g = calloc(ss + 1, 8),
           *alpha = calloc(ss + 1, 8), *beta = calloc(ss + 1, 8), *rr = calloc((size_t)s + 1, 8);
    int* keep = (int*)malloc((size_t)s * sizeof(int) + 4);
    for (int64_t i = 0; i < n; ++i)
        for (int j = 0; j < sa; ++j) r[i * sa + j] = b[i * s + active[j]];
#define PRECOND(src, dst, width)                                                 \
    for (int64_t i_ = 0; i_ < n; ++i_)                                           \
        for (int j_ = 0; j_ < (width); ++j_)                                     \
            (dst)[i_ * (width) + j_] = precond ? dinv[i_] * (src)[i_ * (width) + j_] \
                                               : (src)[i_ * (width) + j_];
    PRECOND(r, z, sa);
    memcpy(p, z, (size_t)n * sa * 8);
    if (sa > 0) gram(r, z, n, sa, s_old);

    for (int m = 1; m <= max_iter && sa > 0; ++m) {
        orc_apply_block(op, p, sa, w);
        gram(p, w, n, sa, g);
        *matvecs += sa;
        pchol c;
        pchol_factor(&c, g, sa);
        pchol_solve(&c, s_old, sa, alpha);
        pchol_free(&c);
        add_product(xa, p, alpha, n, sa, 1.0);
        add_product(r, w, alpha, n, sa, -1.0);
        for (int j = 0; j < sa; ++j) {
            double acc = 0.0;
            for (int64_t i = 0; i < n; ++i) acc += r[i * sa + j] * r[i * sa + j];
            rr[j] = acc;
        }
        *iterations = m;
        int nk = 0, need_restart = 0;
        for (int j = 0; j < sa; ++j) {
            const int orig = active[j];
            const double rel = sqrt(rr[j]) / bnorm[orig];
            if (rel <= tol) {
                *matvecs += 1;
                const double rt = true_rel_residual_col(op, b, s, orig, xa, sa, j, bnorm[orig]);
                if (rt <= tol) {
                    for (int64_t i = 0; i < n; ++i) x[i * s + orig] = xa[i * sa + j];
                    final_res[orig] = rt;
                    converged[orig] = 1;
                    continue;
                }
                need_restart = 1;
            }
            keep[nk++] = j;
        }
        if (nk != sa) {
            for (int j = 0; j < nk; ++j) active[j] = active[keep[j]];
            compact_cols(r, n, sa, keep, nk);
            compact_cols(p, n, sa, keep, nk);
            compact_cols(xa, n, sa, keep, nk);
            compact_sq(s_old, sa, keep, nk);
            sa = nk;
            if (sa == 0) break;
        }
        if (need_restart) {
            orc_apply_block(op, xa, sa, w);
            *matvecs += sa;
            for (int64_t i = 0; i < n; ++i)
                for (int j = 0; j < sa; ++j) r[i * sa + j] = b[i * s + active[j]] - w[i * sa + j];
            PRECOND(r, z, sa);
            memcpy(p, z, (size_t)n * sa * 8);
            gram(r, z, n, sa, s_old);
            continue;
        }
        PRECOND(r, z, sa);
        gram(r, z, n, sa, s_new);
        pchol_factor(&c, s_old, sa);
        pchol_solve(&c, s_new, sa, beta);
        pchol_free(&c);
        /* P = Z + P beta */
        add_product(z, p, beta, n, sa, 1.0);
        double* tmp = p;
        p = z;
        z = tmp;
        memcpy(s_old, s_new, (size_t)sa * sa * 8);
    }
    for (int j = 0; j < sa; ++j) {
        const int orig = active[j];
        *matvecs += 1;
        const double rt = true_rel_residual_col(op, b, s, orig, xa, sa, j, bnorm[orig]);
        for (int64_t i = 0; i < n; ++i) x[i * s + orig] = xa[i * sa + j];
        final_res[orig] = rt;
        converged[orig] = rt <= tol;
    }
#undef PRECOND
    free(bnorm); free(active); free(r); free(z); free(p); free(w); free(xa);
    free(s_old); free(s_new); free(g); free(alpha); free(beta); free(rr); free(keep);
    return ORC_OK;
}

/* Single-RHS CG (solvers.cpp:82-171). */
int orc_cg(const orc_op* op, const double* b, double tol, int max_iter, int precond,
           double* x, int* iterations, int64_t* matvecs, double* final_res, char* conv) {
    if (!(tol > 0.0) || !(tol < 1.0) || max_iter < 1) return ORC_INVALID_CONFIG;
    const int64_t n = op->n;
    memset(x, 0, (size_t)n * 8);
    *iterations = 0;
    *matvecs = 0;
    *final_res = 0.0;
    *conv = 1;
    double bn = 0.0;
    for (int64_t i = 0; i < n; ++i) bn += b[i] * b[i];
    bn = sqrt(bn);
    if (bn == 0.0) return ORC_OK;
    double *r = malloc(n * 8), *z = malloc(n * 8), *p = malloc(n * 8), *w = malloc(n * 8);
    memcpy(r, b, n * 8);
    for (int64_t i = 0; i < n; ++i) z[i] = precond ? op->dinv[i] * r[i] : r[i];
    memcpy(p, z, n * 8);
    double rho = 0.0;
    for (int64_t i = 0; i < n; ++i) rho += r[i] * z[i];
    int done = 0;
    for (int m = 1; m <= max_iter; ++m) {
        orc_apply_block(op, p, 1, w);
        *matvecs += 1;
        double pw = 0.0;
        for (int64_t i = 0; i < n; ++i) pw += p[i] * w[i];
        if (!(pw > 0.0)) {
            *iterations = m - 1;
            break;
        }
        const double al = rho / pw;
        for (int64_t i = 0; i < n; ++i) x[i] = fma(al, p[i], x[i]);
        for (int64_t i = 0; i < n; ++i) r[i] = fma(-al, w[i], r[i]);
        *iterations = m;
        double rn = 0.0;
        for (int64_t i = 0; i < n; ++i) rn += r[i] * r[i];
        if (sqrt(rn) / bn <= tol) {
            const double rt = true_rel_residual_col(op, b, 1, 0, x, 1, 0, bn);
            *matvecs += 1;
            if (rt <= tol) {
                *final_res = rt;
                done = 1;
                break;
            }
            orc_apply_block(op, x, 1, w);
            for (int64_t i = 0; i < n; ++i) r[i] = b[i] - w[i];
            for (int64_t i = 0; i < n; ++i) z[i] = precond ? op->dinv[i] * r[i] : r[i];
            memcpy(p, z, n * 8);
            rho = 0.0;
            for (int64_t i = 0; i < n; ++i) rho += r[i] * z[i];
            continue;
        }
        for (int64_t i = 0; i < n; ++i) z[i] = precond ? op->dinv[i] * r[i] : r[i];
        double rn2 = 0.0;
        for (int64_t i = 0; i < n; ++i) rn2 += r[i] * z[i];
        const double be = rn2 / rho;
        for (int64_t i = 0; i < n; ++i) p[i] = fma(be, p[i], z[i]);
        rho = rn2;
    }
    if (!done) {
        *final_res = true_rel_residual_col(op, b, 1, 0, x, 1, 0, bn);
        *matvecs += 1;
        *conv = *final_res <= tol;
    }
    free(r); free(z); free(p); free(w);
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Combination + operator action (pipeline.cpp:187-251, 548-571)              */
/* ------------------------------------------------------------------------- */
/* X row-major n x s; C row-major s x N; T, Q sample-major N x n; resid[N] is
 * relative_residual(op, T_j, Q_j). Samples [j0, j1). */
int orc_combine_action(const orc_op* op, const double* x, int s, const double* c,
                       int64_t n_samples, int64_t j0, int64_t j1, double* t_out,
                       double* q_out, double* resid) {
    if (s < 1) return ORC_EMPTY;
    const int64_t n = op->n;
    for (int64_t j = j0; j < j1; ++j) {
        double* t = t_out + (j - j0) * n;
        double* q = q_out + (j - j0) * n;
        int first = 1;
        for (int64_t i = 0; i < n; ++i) t[i] = 0.0;
        for (int tt = 0; tt < s; ++tt) {
            const double w = c[(int64_t)tt * n_samples + j];
            if (w == 0.0) continue;
            if (first) {
                for (int64_t i = 0; i < n; ++i) t[i] = w * x[i * s + tt];
                first = 0;
            } else {
                for (int64_t i = 0; i < n; ++i) t[i] = fma(w, x[i * s + tt], t[i]);
            }
        }
        for (int64_t i = 0; i < n; ++i) {
            double acc = 0.0;
            for (int64_t p = op->row_ptr[i]; p < op->row_ptr[i + 1]; ++p)
                acc += op->val[p] * t[op->col[p]];
            q[i] = (acc - op->g[i]) / op->vol[i];
        }
        if (resid) resid[j - j0] = orc_relative_residual(op, t, q);
    }
    return ORC_OK;
}

double orc_cg_error_bound(double kappa, int m, double e0, int* status) {
    *status = 0;
    if (!(kappa >= 1.0)) {
        *status = 8;
        return 0.0;
    }
    if (m < 0 || !(e0 >= 0.0)) {
        *status = ORC_INVALID_CONFIG;
        return 0.0;
    }
    const double rk = sqrt(kappa);
    return 2.0 * pow((rk - 1.0) / (rk + 1.0), m) * e0;
}

/* ------------------------------------------------------------------------- */
/* Seeded BASELINE-config inputs (DESIGN.md §3 pins)       */
/* ------------------------------------------------------------------------- */
/* Test infrastructure, like everything in this file: the reference arm of
 * bench.py and the CPU tests draw the chips' inputs here so the checker side
 * never loads the product library. The pins are the ones DESIGN.md §3 states
 * (the reference has no generator for the BASELINE configs); every draw goes
 * through the Rng restatement above (rng.hpp:14-63), in this order per chip
 * seed derive_seed(master, "chip", chip_id):
 *   configs 1/2: "k" stream, one U[10,150] per 16x16-cell tile, tile-row-major;
 *   configs 3/5: "layers" stream, bulk k ~ U[1,3]; "lognormal" stream, one
 *                normal per cell (flat order) for k *= exp(ln(1.2) Z);
 *   config 4:    "layers" stream, dz_l ~ U[50,500] um for every layer, then
 *                k_l ~ U[1,400] for every layer, then h_top, h_bot ~ U[1e2,1e4];
 *   per basis map t, stream ("basis", t): for each blob cx ~ U[0,nx),
 *                cy ~ U[0,ny), sigma ~ U[2,8] * scale, amp ~ U[0,1e6]; for each
 *                rectangle x0 = below(nx), y0 = below(ny), w, h = wmin +
 *                below(wmax - wmin + 1), power ~ U[0,2e6];
 *   stream ("coef", 0): C[t][j] ~ U[0,1) row-major.
 * tests/test_oracle.py pins this function bitwise against the product's host
 * generator (bk_synth_chip) for every config. */
typedef struct {
    int nx, ny, nz;
    double lx, ly, lz;
    int has_dz;
    int bc_kind[6]; /* 0 Dirichlet, 1 Robin, 2 adiabatic */
    double bc_a[6], bc_b[6];
} orc_chip_meta;

static double urand(orc_rng* r, double lo, double hi) { return lo + rng_u01(r) * (hi - lo); }

int orc_synth_chip(int config, int nx, int ny, int nz, int s, int64_t N, uint64_t master_seed,
                   uint64_t chip_id, orc_chip_meta* meta, double* dz, double* k, double* Q,
                   double* C) {
    if (nx < 1 || ny < 1 || nz < 1 || s < 1 || N < 0) return ORC_INVALID_SPEC;
    const int64_t plane = (int64_t)nx * ny, n = plane * nz;
    const uint64_t chip = orc_derive_seed(master_seed, "chip", chip_id);
    memset(meta, 0, sizeof(*meta));
    meta->nx = nx;
    meta->ny = ny;
    meta->nz = nz;
    meta->lx = 10e-3;
    meta->ly = 10e-3;
    for (int f = 0; f < 6; ++f) meta->bc_kind[f] = 2;
    int nblobs = 0, nrects = 0, z0 = 0, z1 = nz, cpl = 1, tile = 16, tx = 1;
    double scale = 1.0, kl[16] = {0};
    orc_rng r;
    if (config == 1 || config == 2) {
        meta->lz = 0.15e-3 * nz;
        meta->bc_kind[5] = 1;
        meta->bc_a[5] = 1e3;
        tx = (nx + tile - 1) / tile;
        const int ty = (ny + tile - 1) / tile;
        double* tk = (double*)malloc(sizeof(double) * (size_t)tx * ty);
        if (!tk) return ORC_OOM;
        rng_init(&r, orc_derive_seed(chip, "k", 0));
        for (int i = 0; i < tx * ty; ++i) tk[i] = urand(&r, 10.0, 150.0);
        if (k)
            for (int64_t i = 0; i < n; ++i) {
                const int ix = (int)(i % nx), iy = (int)((i / nx) % ny);
                k[i] = tk[(iy / tile) * tx + ix / tile];
            }
        free(tk);
        nblobs = config == 1 ? 3 : 5;
    } else if (config == 3 || config == 5) {
        if (nz % 8) return ORC_INVALID_SPEC;
        cpl = nz / 8;
        meta->lz = 0.8e-3;
        meta->bc_kind[4] = 1;
        meta->bc_a[4] = 1e2;
        meta->bc_kind[5] = 1;
        meta->bc_a[5] = 1e4;
        rng_init(&r, orc_derive_seed(chip, "layers", 0));
        const double stack[8] = {urand(&r, 1.0, 3.0), 150.0, 5.0, 150.0, 5.0, 150.0, 5.0, 400.0};
        if (k) {
            const double ls = log(1.2);
            rng_init(&r, orc_derive_seed(chip, "lognormal", 0));
            for (int64_t i = 0; i < n; ++i) {
                const double z = rng_normal(&r);
                k[i] = stack[(i / plane) / cpl] * exp(ls * z);
            }
        }
        z0 = cpl;
        z1 = 2 * cpl;
        nblobs = 3;
        nrects = 4;
        scale = nx / 128.0;
    } else if (config == 4) {
        if (nz > 16) return ORC_INVALID_SPEC;
        rng_init(&r, orc_derive_seed(chip, "layers", 0));
        double lz = 0.0;
        for (int l = 0; l < nz; ++l) {
            dz[l] = urand(&r, 50e-6, 500e-6);
            lz += dz[l];
        }
        for (int l = 0; l < nz; ++l) kl[l] = urand(&r, 1.0, 400.0);
        const double h_top = urand(&r, 1e2, 1e4), h_bot = urand(&r, 1e2, 1e4);
        meta->lz = lz;
        meta->has_dz = 1;
        meta->bc_kind[4] = 1;
        meta->bc_a[4] = h_bot;
        meta->bc_kind[5] = 1;
        meta->bc_a[5] = h_top;
        if (k)
            for (int64_t i = 0; i < n; ++i) k[i] = kl[i / plane];
        z0 = nz > 1 ? 1 : 0;
        z1 = z0 + 1;
        nblobs = 5;
        scale = nx / 128.0;
    } else {
        return ORC_INVALID_CONFIG;
    }
    if (Q) {
        memset(Q, 0, sizeof(double) * (size_t)n * s);
        double* pl = (double*)malloc(sizeof(double) * (size_t)plane);
        if (!pl) return ORC_OOM;
        int wmin = (int)(4 * scale);
        if (wmin < 1) wmin = 1;
        int wmax = (int)(32 * scale);
        if (wmax < wmin) wmax = wmin;
        for (int t = 0; t < s; ++t) {
            rng_init(&r, orc_derive_seed(chip, "basis", (uint64_t)t));
            for (int64_t c = 0; c < plane; ++c) pl[c] = 0.0;
            /* blobs: parameters first, then the plane sum in blob order */
            double bp[8][4];
            for (int b = 0; b < nblobs; ++b) {
                bp[b][0] = urand(&r, 0.0, nx);
                bp[b][1] = urand(&r, 0.0, ny);
                const double sig = urand(&r, 2.0, 8.0) * scale;
                bp[b][3] = urand(&r, 0.0, 1e6);
                bp[b][2] = 1.0 / (2.0 * sig * sig);
            }
            double rp[8][5];
            for (int q = 0; q < nrects; ++q) {
                rp[q][0] = (double)rng_below(&r, (uint64_t)nx);
                rp[q][1] = (double)rng_below(&r, (uint64_t)ny);
                rp[q][2] = wmin + (double)rng_below(&r, (uint64_t)(wmax - wmin + 1));
                rp[q][3] = wmin + (double)rng_below(&r, (uint64_t)(wmax - wmin + 1));
                rp[q][4] = urand(&r, 0.0, 2e6);
            }
            for (int b = 0; b < nblobs; ++b)
                for (int iy = 0; iy < ny; ++iy) {
                    const double dy = iy + 0.5 - bp[b][1];
                    for (int ix = 0; ix < nx; ++ix) {
                        const double dx = ix + 0.5 - bp[b][0];
                        pl[(int64_t)iy * nx + ix] += bp[b][3] * exp(-(dx * dx + dy * dy) * bp[b][2]);
                    }
                }
            for (int q = 0; q < nrects; ++q) {
                const int x0 = (int)rp[q][0], y0 = (int)rp[q][1];
                const int w = (int)rp[q][2], h = (int)rp[q][3];
                for (int iy = y0; iy < ny && iy < y0 + h; ++iy)
                    for (int ix = x0; ix < nx && ix < x0 + w; ++ix) pl[(int64_t)iy * nx + ix] += rp[q][4];
            }
            for (int iz = z0; iz < z1; ++iz)
                for (int64_t c = 0; c < plane; ++c) Q[(iz * plane + c) * s + t] = pl[c];
        }
        free(pl);
    }
    if (C) {
        rng_init(&r, orc_derive_seed(chip, "coef", 0));
        for (int64_t i = 0; i < (int64_t)s * N; ++i) C[i] = rng_u01(&r);
    }
    return ORC_OK;
}
