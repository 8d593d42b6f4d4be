/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference
 * algorithm for the Ewald hot path, used as the parity checker by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg.  It is never linked into, called by, or a fallback of the product
 * (paper_1708_01135_b200/), which fails loudly without its CUDA library.
 *
 * Parity pinned: tests/test_oracle_golden.py checks every function here
 * against golden vectors produced by the real reference package
 * (tests/golden/make_golden.py runs /root/reference's ewaldmd).
 *
 * Each function follows the reference file:line it cites
 * (/root/reference/pkg/src/ewaldmd/...).  Worker partitioning follows
 * engine.py:75-91: contiguous particle blocks per thread, private
 * accumulators for incremented globals, reduced in worker-index order.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ECOINCIDENT 2
#define ORC_ECUTOFF 3
#define ORC_EUNWRAPPED 4
#define ORC_ENOMEM 9

/* block_bounds (engine.py:75-82) */
static void block_bounds(int64_t n, int workers, int64_t *bounds) {
    int64_t base = n / workers, rem = n % workers;
    bounds[0] = 0;
    for (int w = 0; w < workers; ++w) bounds[w + 1] = bounds[w] + base + (w < rem ? 1 : 0);
}

static int clamp_workers(int nthreads, int64_t n) {
    if (nthreads < 1) nthreads = 1;
    if (n > 0 && nthreads > n) nthreads = (int)n;
    return nthreads;
}

/* _phase_tables (ewald.py:262-278): cos/sin of m*step*r_a by recurrence */
static void phase_tables(const double *pos, int64_t i, double step, int mmax, double *ct, double *st) {
    for (int a = 0; a < 3; ++a) {
        double th = step * pos[3 * i + a];
        double cb = cos(th), sb = sin(th);
        double *c = ct + a * (mmax + 1), *s = st + a * (mmax + 1);
        c[0] = 1.0;
        s[0] = 0.0;
        for (int m = 1; m <= mmax; ++m) {
            double cp = c[m - 1], sp = s[m - 1];
            c[m] = cp * cb - sp * sb;
            s[m] = sp * cb + cp * sb;
        }
    }
}

static int table_mmax(const int64_t *m, int64_t K) {
    int64_t mm = 0;
    for (int64_t i = 0; i < 3 * K; ++i) {
        int64_t a = m[i] < 0 ? -m[i] : m[i];
        if (a > mm) mm = a;
    }
    return (int)mm;
}

/* compute_rho_hat / _rho_body (ewald.py:281-305, 457-464) */
int orc_rho_hat(const double *pos, const double *q, int64_t n, double L, const int64_t *m,
                int64_t K, int nthreads, double *rho_out) {
    if (n < 0 || K < 1 || !(L > 0.0)) return ORC_EINVAL;
    const double step = 2.0 * M_PI / L;
    const int mmax = table_mmax(m, K);
    int workers = clamp_workers(nthreads, n);
    int64_t *bounds = (int64_t *)malloc(sizeof(int64_t) * (workers + 1));
    double *stack = (double *)calloc((size_t)workers * 2 * K, sizeof(double));
    if (!bounds || !stack) { free(bounds); free(stack); return ORC_ENOMEM; }
    block_bounds(n, workers, bounds);
#pragma omp parallel for num_threads(workers) schedule(static, 1)
    for (int w = 0; w < workers; ++w) {
        double *rho = stack + (size_t)w * 2 * K;
        double *ct = (double *)malloc(sizeof(double) * 3 * (mmax + 1));
        double *st = (double *)malloc(sizeof(double) * 3 * (mmax + 1));
        for (int64_t i = bounds[w]; i < bounds[w + 1]; ++i) {
            const double qi = q[i];
            phase_tables(pos, i, step, mmax, ct, st);
            for (int64_t kk = 0; kk < K; ++kk) {
                const int64_t ax = m[3 * kk], ay = m[3 * kk + 1], az = m[3 * kk + 2];
                const int64_t bx = ax < 0 ? -ax : ax, by = ay < 0 ? -ay : ay, bz = az < 0 ? -az : az;
                const double cx = ct[bx], sx = (ax < 0 ? -1.0 : 1.0) * st[bx];
                const double cy = ct[(mmax + 1) + by], sy = (ay < 0 ? -1.0 : 1.0) * st[(mmax + 1) + by];
                const double cz = ct[2 * (mmax + 1) + bz], sz = (az < 0 ? -1.0 : 1.0) * st[2 * (mmax + 1) + bz];
                const double cxy = cx * cy - sx * sy;
                const double sxy = sx * cy + cx * sy;
                const double cre = cxy * cz - sxy * sz;
                const double sim = sxy * cz + cxy * sz;
                rho[kk] += qi * cre;
                rho[K + kk] -= qi * sim;
            }
        }
        free(ct);
        free(st);
    }
    /* reduce_global in worker order, INC_ZERO overwrite (engine.py:85-91, 247-254) */
    for (int64_t k = 0; k < 2 * K; ++k) {
        double s = 0.0;
        for (int w = 0; w < workers; ++w) s += stack[(size_t)w * 2 * K + k];
        rho_out[k] = s;
    }
    free(bounds);
    free(stack);
    return ORC_OK;
}

/* long_range_energy_forces / _lr_body (ewald.py:308-349, 467-479); force += */
int orc_long_range(const double *pos, const double *q, int64_t n, double L, const int64_t *m,
                   int64_t K, const double *coeff, const double *rho, int nthreads,
                   double *force_inout, double *u_out) {
    if (n < 0 || K < 1 || !(L > 0.0)) return ORC_EINVAL;
    const double step = 2.0 * M_PI / L;
    const int mmax = table_mmax(m, K);
    int workers = clamp_workers(nthreads, n);
    int64_t *bounds = (int64_t *)malloc(sizeof(int64_t) * (workers + 1));
    double *ups = (double *)calloc((size_t)workers, sizeof(double));
    if (!bounds || !ups) { free(bounds); free(ups); return ORC_ENOMEM; }
    block_bounds(n, workers, bounds);
#pragma omp parallel for num_threads(workers) schedule(static, 1)
    for (int w = 0; w < workers; ++w) {
        double *ct = (double *)malloc(sizeof(double) * 3 * (mmax + 1));
        double *st = (double *)malloc(sizeof(double) * 3 * (mmax + 1));
        double uw = 0.0;
        for (int64_t i = bounds[w]; i < bounds[w + 1]; ++i) {
            const double qi = q[i];
            phase_tables(pos, i, step, mmax, ct, st);
            double u = 0.0, fx = 0.0, fy = 0.0, fz = 0.0;
            for (int64_t kk = 0; kk < K; ++kk) {
                const int64_t ax = m[3 * kk], ay = m[3 * kk + 1], az = m[3 * kk + 2];
                const int64_t bx = ax < 0 ? -ax : ax, by = ay < 0 ? -ay : ay, bz = az < 0 ? -az : az;
                const double cx = ct[bx], sx = (ax < 0 ? -1.0 : 1.0) * st[bx];
                const double cy = ct[(mmax + 1) + by], sy = (ay < 0 ? -1.0 : 1.0) * st[(mmax + 1) + by];
                const double cz = ct[2 * (mmax + 1) + bz], sz = (az < 0 ? -1.0 : 1.0) * st[2 * (mmax + 1) + bz];
                const double cxy = cx * cy - sx * sy;
                const double sxy = sx * cy + cx * sy;
                const double cre = cxy * cz - sxy * sz;
                const double sim = sxy * cz + cxy * sz;
                const double rr = rho[kk], ri = rho[K + kk];
                const double re_arho = cre * rr - sim * ri;
                const double im_arho = cre * ri + sim * rr;
                u += coeff[kk] * re_arho;
                const double wgt = 2.0 * coeff[kk] * im_arho;
                fx += wgt * (step * (double)ax);
                fy += wgt * (step * (double)ay);
                fz += wgt * (step * (double)az);
            }
            uw += qi * u;
            force_inout[3 * i] += qi * fx;
            force_inout[3 * i + 1] += qi * fy;
            force_inout[3 * i + 2] += qi * fz;
        }
        ups[w] = uw;
        free(ct);
        free(st);
    }
    double u = 0.0;
    for (int w = 0; w < workers; ++w) u += ups[w];
    *u_out = u;
    free(bounds);
    free(ups);
    return ORC_OK;
}

/* _build_stencil (celllist.py:48-72): distinct periodic 27-stencil ids */
static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* PairLoop over build_cell_list with the screened Coulomb body
 * (celllist.py:75-108, engine.py:102-159, ewald.py:208-221).  Centres are
 * all particles, or the nsel indices in sel (sampled checks).  force += */
int orc_short_range(const double *pos, const double *q, int64_t n, double L, double rc,
                    double alpha, int nthreads, const int64_t *sel, int64_t nsel,
                    double *force_inout, double *u_out) {
    if (!(rc > 0.0)) return ORC_EINVAL;
    if (rc > 0.5 * L) return ORC_ECUTOFF;
    for (int64_t i = 0; i < 3 * n; ++i)
        if (pos[i] < 0.0 || pos[i] >= L) return ORC_EUNWRAPPED;
    const int64_t cpd = (int64_t)floor(L / rc);
    const double edge = L / (double)cpd;
    const int64_t n_cells = cpd * cpd * cpd;
    int64_t *cell_of = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    int64_t *cell_start = (int64_t *)calloc((size_t)n_cells + 1, sizeof(int64_t));
    int64_t *stencil = (int64_t *)malloc(sizeof(int64_t) * 27 * n_cells);
    int64_t *scount = (int64_t *)malloc(sizeof(int64_t) * n_cells);
    if (!cell_of || !order || !cell_start || !stencil || !scount) {
        free(cell_of); free(order); free(cell_start); free(stencil); free(scount);
        return ORC_ENOMEM;
    }
    for (int64_t i = 0; i < n; ++i) {
        int64_t id[3];
        for (int a = 0; a < 3; ++a) {
            int64_t k = (int64_t)floor(pos[3 * i + a] / edge);
            if (k < 0) k = 0;
            if (k > cpd - 1) k = cpd - 1;
            id[a] = k;
        }
        cell_of[i] = id[0] + cpd * (id[1] + cpd * id[2]);
        cell_start[cell_of[i] + 1]++;
    }
    for (int64_t c = 0; c < n_cells; ++c) cell_start[c + 1] += cell_start[c];
    {   /* stable argsort by cell (counting sort keeps index order) */
        int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * n_cells);
        memcpy(cursor, cell_start, sizeof(int64_t) * n_cells);
        for (int64_t i = 0; i < n; ++i) order[cursor[cell_of[i]]++] = i;
        free(cursor);
    }
    for (int64_t c = 0; c < n_cells; ++c) {
        int64_t cx = c % cpd, cy = (c / cpd) % cpd, cz = c / (cpd * cpd);
        int64_t ids[27];
        int t = 0;
        for (int oz = -1; oz <= 1; ++oz)
            for (int oy = -1; oy <= 1; ++oy)
                for (int ox = -1; ox <= 1; ++ox) {
                    int64_t nx = ((cx + ox) % cpd + cpd) % cpd, ny = ((cy + oy) % cpd + cpd) % cpd,
                            nz = ((cz + oz) % cpd + cpd) % cpd;
                    ids[t++] = nx + cpd * (ny + cpd * nz);
                }
        qsort(ids, 27, sizeof(int64_t), cmp_i64);
        int cnt = 0;
        for (int k = 0; k < 27; ++k)
            if (k == 0 || ids[k] != ids[k - 1]) stencil[27 * c + cnt++] = ids[k];
        scount[c] = cnt;
    }
    const double rc2 = rc * rc;
    const double hl = 0.5 * L;
    const double c0 = sqrt(alpha), c1 = alpha, c2 = 2.0 * sqrt(alpha / M_PI);
    const int64_t ncent = sel ? nsel : n;
    int workers = clamp_workers(nthreads, ncent);
    int64_t *bounds = (int64_t *)malloc(sizeof(int64_t) * (workers + 1));
    double *ups = (double *)calloc((size_t)workers, sizeof(double));
    int *errs = (int *)calloc((size_t)workers, sizeof(int));
    block_bounds(ncent, workers, bounds);
#pragma omp parallel for num_threads(workers) schedule(static, 1)
    for (int w = 0; w < workers; ++w) {
        double uw = 0.0;
        for (int64_t ii = bounds[w]; ii < bounds[w + 1] && !errs[w]; ++ii) {
            const int64_t i = sel ? sel[ii] : ii;
            const double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2];
            const int64_t ci = cell_of[i];
            const int scan_all = scount[ci] == n_cells;
            const int64_t ns = scan_all ? 1 : scount[ci];
            for (int64_t s = 0; s < ns; ++s) {
                int64_t pb, pe;
                if (scan_all) { pb = 0; pe = n; }
                else { int64_t c = stencil[27 * ci + s]; pb = cell_start[c]; pe = cell_start[c + 1]; }
                for (int64_t p = pb; p < pe; ++p) {
                    const int64_t j = scan_all ? p : order[p];
                    if (j == i) continue;
                    double dx = xi - pos[3 * j];
                    if (dx >= hl) dx -= L; else if (dx < -hl) dx += L;
                    double dy = yi - pos[3 * j + 1];
                    if (dy >= hl) dy -= L; else if (dy < -hl) dy += L;
                    double dz = zi - pos[3 * j + 2];
                    if (dz >= hl) dz -= L; else if (dz < -hl) dz += L;
                    volatile double t1 = dx * dx; /* no contraction: r2 as the reference */
                    volatile double t2 = dy * dy;
                    volatile double t3 = dz * dz;
                    const double r2 = (t1 + t2) + t3;
                    if (!(r2 < rc2)) continue;
                    if (r2 == 0.0) { errs[w] = 1; break; }
                    const double qq = q[i] * q[j];
                    const double r = sqrt(r2);
                    const double sc = erfc(c0 * r) / r;
                    uw += 0.5 * qq * sc;
                    const double g = qq * (sc + c2 * exp(-c1 * r2)) / r2;
                    force_inout[3 * i] += g * dx;
                    force_inout[3 * i + 1] += g * dy;
                    force_inout[3 * i + 2] += g * dz;
                }
                if (errs[w]) break;
            }
        }
        ups[w] = uw;
    }
    int err = 0;
    double u = 0.0;
    for (int w = 0; w < workers; ++w) { u += ups[w]; err |= errs[w]; }
    *u_out = u;
    free(bounds); free(ups); free(errs);
    free(cell_of); free(order); free(cell_start); free(stencil); free(scount);
    return err ? ORC_ECOINCIDENT : ORC_OK;
}

/* short_range_wide_cutoff / _sr_wide_jit (ewald.py:490-576): every j != i
 * over the 27 nearest images, no fold; for r_c in (L/2, L], N <= 4096. */
int orc_short_range_wide(const double *pos, const double *q, int64_t n, double L, double rc,
                         double alpha, int nthreads, double *force_inout, double *u_out) {
    if (!(rc > 0.0)) return ORC_EINVAL;
    if (rc > L) return 6;      /* BoxTooSmallError */
    if (n > 4096) return 7;    /* OracleSizeError */
    const double rc2 = rc * rc;
    const double c0 = sqrt(alpha), c1 = alpha, c2 = 2.0 * sqrt(alpha / M_PI);
    int workers = clamp_workers(nthreads, n);
    int64_t *bounds = (int64_t *)malloc(sizeof(int64_t) * (workers + 1));
    double *ups = (double *)calloc((size_t)workers, sizeof(double));
    int *errs = (int *)calloc((size_t)workers, sizeof(int));
    block_bounds(n, workers, bounds);
#pragma omp parallel for num_threads(workers) schedule(static, 1)
    for (int w = 0; w < workers; ++w) {
        double uw = 0.0;
        for (int64_t i = bounds[w]; i < bounds[w + 1]; ++i)
            for (int64_t j = 0; j < n; ++j) {
                if (j == i) continue;
                for (int nx = -1; nx <= 1; ++nx)
                    for (int ny = -1; ny <= 1; ++ny)
                        for (int nz = -1; nz <= 1; ++nz) {
                            const double dx = pos[3 * i] - pos[3 * j] + L * nx;
                            const double dy = pos[3 * i + 1] - pos[3 * j + 1] + L * ny;
                            const double dz = pos[3 * i + 2] - pos[3 * j + 2] + L * nz;
                            volatile double t1 = dx * dx;
                            volatile double t2 = dy * dy;
                            volatile double t3 = dz * dz;
                            const double r2 = (t1 + t2) + t3;
                            if (r2 >= rc2) continue;
                            if (r2 == 0.0) { errs[w] = 1; continue; }
                            const double qq = q[i] * q[j];
                            const double r = sqrt(r2);
                            const double sc = erfc(c0 * r) / r;
                            uw += 0.5 * qq * sc;
                            const double g = qq * (sc + c2 * exp(-c1 * r2)) / r2;
                            force_inout[3 * i] += g * dx;
                            force_inout[3 * i + 1] += g * dy;
                            force_inout[3 * i + 2] += g * dz;
                        }
            }
        ups[w] = uw;
    }
    int err = 0;
    double u = 0.0;
    for (int w = 0; w < workers; ++w) { u += ups[w]; err |= errs[w]; }
    *u_out = u;
    free(bounds); free(ups); free(errs);
    return err ? ORC_ECOINCIDENT : ORC_OK;
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
