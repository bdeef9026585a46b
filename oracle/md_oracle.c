/*
 * md_oracle.c -- CPU restatement of the reference MD hot path (TEST INFRASTRUCTURE).
 *
 * This file is the parity checker for the B200 kernels.  It is NOT part of the
 * product: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product path never routes through it.
 *
 * It restates, in plain C with IEEE fp64 and no FMA contraction (compile with
 * -ffp-contract=off, no -ffast-math), the arithmetic of the reference package
 * `mdbench` 0.1.0 (arXiv 2406.04210 artifact):
 *
 *   orc_list_cells      <- pkg/src/mdbench/neighbor.py:112-152  (_list_cells_chunk)
 *   orc_list_brute      <- pkg/src/mdbench/neighbor.py:155-182  (_list_brute_chunk)
 *   orc_force_truncated <- pkg/src/mdbench/forces.py:72-110     (_truncated_chunk)
 *   orc_force_all_pairs <- pkg/src/mdbench/forces.py:29-69      (_all_to_all_chunk)
 *   orc_tree_sum        <- pkg/src/mdbench/observables.py:31-74 (_tree_sum / reduce_sum)
 *   orc_vv_kick / orc_vv_drift_wrap <- pkg/src/mdbench/integrate.py:58-79, core.py:72-93
 *   orc_max_disp2       <- pkg/src/mdbench/neighbor.py:243-254  (needs_rebuild)
 *
 * Extensions the reference does not have ("parity unpinned"
 * by the reference's own tests, pinned only by construction and by property
 * tests): per-particle virial (w_i = 1/2 sum_j fr*r2) and per-pair-type
 * parameter tables (eps, sigma^2, rc^2, shift indexed by species pair).  With
 * ntypes == 1 the table variant performs exactly the reference's operations in
 * the reference's order, so forces/energies stay bit-identical to it.
 *
 * Pinned against golden vectors produced by the real reference
 * (tests/golden/make_golden.py -> tests/golden/ npz files), see tests/test_oracle_golden.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_API __attribute__((visibility("default")))

ORC_API int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Nearest-image reduction of one displacement component, written the way every
 * reference kernel writes it: d - L * rint(d * (1/L)), ties to even.
 * (neighbor.py:140-142, forces.py:88-90, core.py:69) */
static inline double nearest_image(double d, double edge, double inv_edge) {
    return d - edge * rint(d * inv_edge);
}

static inline int64_t wrap_index(int64_t c, int64_t nc) {
    int64_t m = c % nc;
    return m < 0 ? m + nc : m;
}

static void sort_i32(int32_t *row, int64_t len) {
    /* rows come out of the cell scan almost sorted; insertion sort is enough */
    for (int64_t a = 1; a < len; ++a) {
        int32_t v = row[a];
        int64_t b = a - 1;
        while (b >= 0 && row[b] > v) { row[b + 1] = row[b]; --b; }
        row[b + 1] = v;
    }
}

/* 27-cell scan.  pos: (n,3) C-order.  nbr: (n,stride) row-major int32.
 * Scan order = x-offset outermost, z innermost, each wrapped with a true
 * modulo; entries past `stride` are dropped but counted, which raises the
 * per-row overflow byte; the kept prefix is then sorted ascending. */
ORC_API void orc_list_cells(int64_t n, const double *pos, const double *edges,
                            const int64_t *ncell, const int64_t *cell_of,
                            const int64_t *cell_start,
                            const int64_t *cell_particles, double rl2,
                            int64_t stride, int32_t *nbr, int32_t *counts,
                            uint8_t *overflow, int nthreads) {
    const double lx = edges[0], ly = edges[1], lz = edges[2];
    const double ilx = 1.0 / lx, ily = 1.0 / ly, ilz = 1.0 / lz;
    const int64_t ncx = ncell[0], ncy = ncell[1], ncz = ncell[2];
    (void)nthreads;
#pragma omp parallel for schedule(dynamic, 256) num_threads(nthreads)
    for (int64_t i = 0; i < n; ++i) {
        const double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2];
        const int64_t ci = cell_of[i];
        const int64_t cz = ci % ncz;
        const int64_t cy = (ci / ncz) % ncy;
        const int64_t cx = ci / (ncz * ncy);
        int32_t *row = nbr + i * stride;
        int64_t found = 0;
        for (int ox = -1; ox <= 1; ++ox) {
            const int64_t jx = wrap_index(cx + ox, ncx);
            for (int oy = -1; oy <= 1; ++oy) {
                const int64_t jy = wrap_index(cy + oy, ncy);
                for (int oz = -1; oz <= 1; ++oz) {
                    const int64_t jz = wrap_index(cz + oz, ncz);
                    const int64_t cj = (jx * ncy + jy) * ncz + jz;
                    for (int64_t p = cell_start[cj]; p < cell_start[cj + 1]; ++p) {
                        const int64_t j = cell_particles[p];
                        if (j == i) continue;
                        double dx = xi - pos[3 * j];
                        double dy = yi - pos[3 * j + 1];
                        double dz = zi - pos[3 * j + 2];
                        dx = nearest_image(dx, lx, ilx);
                        dy = nearest_image(dy, ly, ily);
                        dz = nearest_image(dz, lz, ilz);
                        const double r2 = dx * dx + dy * dy + dz * dz;
                        if (r2 < rl2) {
                            if (found < stride) row[found] = (int32_t)j;
                            else overflow[i] = 1;
                            ++found;
                        }
                    }
                }
            }
        }
        const int64_t kept = found < stride ? found : stride;
        counts[i] = (int32_t)kept;
        sort_i32(row, kept);
    }
}

/* All-pairs scan used when some axis has fewer than three cells. */
ORC_API void orc_list_brute(int64_t n, const double *pos, const double *edges,
                            double rl2, int64_t stride, int32_t *nbr,
                            int32_t *counts, uint8_t *overflow, int nthreads) {
    const double lx = edges[0], ly = edges[1], lz = edges[2];
    const double ilx = 1.0 / lx, ily = 1.0 / ly, ilz = 1.0 / lz;
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (int64_t i = 0; i < n; ++i) {
        const double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2];
        int32_t *row = nbr + i * stride;
        int64_t found = 0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double dx = nearest_image(xi - pos[3 * j], lx, ilx);
            double dy = nearest_image(yi - pos[3 * j + 1], ly, ily);
            double dz = nearest_image(zi - pos[3 * j + 2], lz, ilz);
            const double r2 = dx * dx + dy * dy + dz * dz;
            if (r2 < rl2) {
                if (found < stride) row[found] = (int32_t)j;
                else overflow[i] = 1;
                ++found;
            }
        }
        counts[i] = (int32_t)(found < stride ? found : stride);
    }
}

/* One LJ pair term in the reference's operation order (forces.py:98-106).
 * tab = {eps, sig2, rc2, shift}.  Returns 0 when the pair is outside the
 * cutoff (r2 >= rc2) or singular (r2 == 0, recorded by the caller). */
typedef struct { double fx, fy, fz, u, w; } pair_acc;

static inline void lj_accumulate(pair_acc *a, const double *tab, double dx,
                                 double dy, double dz, double r2) {
    const double eps = tab[0], sig2 = tab[1], shift = tab[3];
    const double ir2 = 1.0 / r2;
    const double s2 = sig2 * ir2;
    const double s6 = s2 * s2 * s2;
    const double s12 = s6 * s6;
    const double fr = 24.0 * eps * (2.0 * s12 - s6) * ir2;
    a->u += 0.5 * (4.0 * eps * (s12 - s6) + shift);
    a->fx += fr * dx;
    a->fy += fr * dy;
    a->fz += fr * dz;
    a->w += 0.5 * (fr * r2); /* extension: half-share of the pair virial r.f */
}

/* Listed-neighbour LJ forces.  species may be NULL (single type);
 * table: (ntypes*ntypes, 4) = eps, sig2, rc2, shift per (type_i, type_j).
 * virial may be NULL.  bad_j[i] = first coincident partner or -1. */
ORC_API void orc_force_truncated(int64_t n, const double *pos,
                                 const double *edges, const int32_t *species,
                                 int ntypes, const double *table,
                                 int64_t stride, const int32_t *nbr,
                                 const int32_t *counts, double *forces,
                                 double *pe, double *virial, int64_t *bad_j,
                                 int nthreads) {
    const double lx = edges[0], ly = edges[1], lz = edges[2];
    const double ilx = 1.0 / lx, ily = 1.0 / ly, ilz = 1.0 / lz;
    (void)nthreads;
#pragma omp parallel for schedule(static, 256) num_threads(nthreads)
    for (int64_t i = 0; i < n; ++i) {
        const double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2];
        const int ti = species ? species[i] : 0;
        const int32_t *row = nbr + i * stride;
        pair_acc a = {0.0, 0.0, 0.0, 0.0, 0.0};
        bad_j[i] = -1;
        for (int32_t k = 0; k < counts[i]; ++k) {
            const int64_t j = row[k];
            double dx = nearest_image(xi - pos[3 * j], lx, ilx);
            double dy = nearest_image(yi - pos[3 * j + 1], ly, ily);
            double dz = nearest_image(zi - pos[3 * j + 2], lz, ilz);
            const double r2 = dx * dx + dy * dy + dz * dz;
            const int tj = species ? species[j] : 0;
            const double *tab = table + 4 * (ti * ntypes + tj);
            if (r2 >= tab[2]) continue;
            if (r2 == 0.0) {
                if (bad_j[i] < 0) bad_j[i] = j;
                continue;
            }
            lj_accumulate(&a, tab, dx, dy, dz, r2);
        }
        forces[3 * i] = a.fx;
        forces[3 * i + 1] = a.fy;
        forces[3 * i + 2] = a.fz;
        pe[i] = a.u;
        if (virial) virial[i] = a.w;
    }
}

/* Every-pair LJ forces (rc2 may be +inf). */
ORC_API void orc_force_all_pairs(int64_t n, const double *pos,
                                 const double *edges, const int32_t *species,
                                 int ntypes, const double *table,
                                 double *forces, double *pe, double *virial,
                                 int64_t *bad_j, int nthreads) {
    const double lx = edges[0], ly = edges[1], lz = edges[2];
    const double ilx = 1.0 / lx, ily = 1.0 / ly, ilz = 1.0 / lz;
    (void)nthreads;
#pragma omp parallel for schedule(static, 64) num_threads(nthreads)
    for (int64_t i = 0; i < n; ++i) {
        const double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2];
        const int ti = species ? species[i] : 0;
        pair_acc a = {0.0, 0.0, 0.0, 0.0, 0.0};
        bad_j[i] = -1;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double dx = nearest_image(xi - pos[3 * j], lx, ilx);
            double dy = nearest_image(yi - pos[3 * j + 1], ly, ily);
            double dz = nearest_image(zi - pos[3 * j + 2], lz, ilz);
            const double r2 = dx * dx + dy * dy + dz * dz;
            const int tj = species ? species[j] : 0;
            const double *tab = table + 4 * (ti * ntypes + tj);
            if (r2 >= tab[2]) continue;
            if (r2 == 0.0) {
                if (bad_j[i] < 0) bad_j[i] = j;
                continue;
            }
            lj_accumulate(&a, tab, dx, dy, dz, r2);
        }
        forces[3 * i] = a.fx;
        forces[3 * i + 1] = a.fy;
        forces[3 * i + 2] = a.fz;
        pe[i] = a.u;
        if (virial) virial[i] = a.w;
    }
}

/* Fixed-shape adjacent-pair tree over `len` values, odd leftover carried
 * unchanged to the next level (observables.py:31-40).  scratch: len doubles. */
static double pair_tree(const double *v, int64_t len, double *scratch) {
    if (len == 0) return 0.0;
    memcpy(scratch, v, (size_t)len * sizeof(double));
    while (len > 1) {
        const int64_t half = len / 2;
        for (int64_t k = 0; k < half; ++k)
            scratch[k] = scratch[2 * k] + scratch[2 * k + 1];
        if (len & 1) { scratch[half] = scratch[len - 1]; len = half + 1; }
        else len = half;
    }
    return scratch[0];
}

/* Deterministic sum: 4096-value blocks, each by pair_tree, then pair_tree over
 * the block partials (observables.py:57-74).  Empty input sums to 0.0. */
ORC_API double orc_tree_sum(const double *v, int64_t n) {
    enum { BLOCK = 4096 };
    if (n <= 0) return 0.0;
    double *scratch = (double *)malloc(sizeof(double) * (size_t)(n < BLOCK ? BLOCK : n));
    double out;
    if (n <= BLOCK) {
        out = pair_tree(v, n, scratch);
    } else {
        const int64_t nb = (n + BLOCK - 1) / BLOCK;
        double *partials = (double *)malloc(sizeof(double) * (size_t)nb);
        for (int64_t b = 0; b < nb; ++b) {
            const int64_t lo = b * BLOCK;
            const int64_t len = (n - lo) < BLOCK ? (n - lo) : BLOCK;
            partials[b] = pair_tree(v + lo, len, scratch);
        }
        out = pair_tree(partials, nb, scratch);
        free(partials);
    }
    free(scratch);
    return out;
}

/* Half-kick v += (f/m) * (0.5*dt): divide first, then multiply by the
 * pre-multiplied half step (integrate.py:64,79). */
ORC_API void orc_vv_kick(int64_t n, double *vel, const double *forces,
                         const double *masses, double dt, int nthreads) {
    const double half = 0.5 * dt;
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (int64_t i = 0; i < n; ++i) {
        const double m = masses[i];
        for (int c = 0; c < 3; ++c)
            vel[3 * i + c] += (forces[3 * i + c] / m) * half;
    }
}

/* Drift r += v*dt then wrap into [0,L) absorbing the shift into the image
 * counters (integrate.py:67-70, core.py:81-93). */
ORC_API void orc_vv_drift_wrap(int64_t n, double *pos, int64_t *img,
                               const double *vel, const double *edges,
                               double dt, int nthreads) {
    double inv[3] = {1.0 / edges[0], 1.0 / edges[1], 1.0 / edges[2]};
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (int64_t i = 0; i < n; ++i) {
        for (int c = 0; c < 3; ++c) {
            const double L = edges[c];
            double r = pos[3 * i + c] + vel[3 * i + c] * dt;
            double k = floor(r * inv[c]);
            double w = r - k * L;
            if (w < 0.0) { w += L; k -= 1.0; }
            if (w >= L) { w -= L; k += 1.0; }
            pos[3 * i + c] = w;
            img[3 * i + c] += (int64_t)k;
        }
    }
}

/* max_i |(pos + img*L) - at_build|^2 (neighbor.py:251-253); the einsum row
 * product is summed left to right. */
ORC_API double orc_max_disp2(int64_t n, const double *pos, const int64_t *img,
                             const double *edges, const double *at_build) {
    double best = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int c = 0; c < 3; ++c) {
            const double u = pos[3 * i + c] + (double)img[3 * i + c] * edges[c];
            const double d = u - at_build[3 * i + c];
            s += d * d;
        }
        if (s > best) best = s;
    }
    return best;
}

/* Error-scale helper for the fp32 parity metrics (not part of the reference):
 * per particle, the sums of ABSOLUTE pair contributions over the listed,
 * in-range neighbours: sum |f_ij| (force magnitude), sum |u_ij|/2, sum |fr*r2|/2.
 * Dividing an absolute error by these gives a backward-error style relative
 * error that is insensitive to cancellation between neighbours. */
ORC_API void orc_pair_scales(int64_t n, const double *pos, const double *edges,
                             const int32_t *species, int ntypes, const double *table,
                             int64_t stride, const int32_t *nbr, const int32_t *counts,
                             double *f_scale, double *u_scale, double *w_scale,
                             int nthreads) {
    const double lx = edges[0], ly = edges[1], lz = edges[2];
    const double ilx = 1.0 / lx, ily = 1.0 / ly, ilz = 1.0 / lz;
    (void)nthreads;
#pragma omp parallel for schedule(static, 256) num_threads(nthreads)
    for (int64_t i = 0; i < n; ++i) {
        const double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2];
        const int ti = species ? species[i] : 0;
        const int32_t *row = nbr + i * stride;
        double fs = 0.0, us = 0.0, ws = 0.0;
        for (int32_t k = 0; k < counts[i]; ++k) {
            const int64_t j = row[k];
            double dx = nearest_image(xi - pos[3 * j], lx, ilx);
            double dy = nearest_image(yi - pos[3 * j + 1], ly, ily);
            double dz = nearest_image(zi - pos[3 * j + 2], lz, ilz);
            const double r2 = dx * dx + dy * dy + dz * dz;
            const int tj = species ? species[j] : 0;
            const double *tab = table + 4 * (ti * ntypes + tj);
            if (r2 >= tab[2] || r2 == 0.0) continue;
            const double ir2 = 1.0 / r2;
            const double s6 = (tab[1] * ir2) * (tab[1] * ir2) * (tab[1] * ir2);
            const double s12 = s6 * s6;
            const double fr = 24.0 * tab[0] * (2.0 * s12 + s6) * ir2;   /* |repulsive| + |attractive| */
            fs += fr * sqrt(r2);
            us += 0.5 * (4.0 * tab[0] * (s12 + s6) + fabs(tab[3]));
            ws += 0.5 * fr * r2;
        }
        f_scale[i] = fs;
        u_scale[i] = us;
        w_scale[i] = ws;
    }
}
