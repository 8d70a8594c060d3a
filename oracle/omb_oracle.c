/*
 * omb_oracle.c -- CPU restatement of the reference hydro step kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.  The product (paper_2107_10987_b200)
 * never links or calls it.
 *
 * It restates, operation for operation, the reference's compiled backend
 * (/root/reference/pkg/src/octomini/_kernels/_core.pyx) and the numpy parts
 * of the step (hydro/step.py, hydro/eos.py, hydro/sources.py,
 * _kernels/reference.py), with every association kept so that, compiled
 * with -ffp-contract=off (no FMA contraction) and linked against glibc's
 * pow, it reproduces the reference bit for bit.  Pinned against goldens
 * produced by the reference itself (tests/golden/make_golden.py).
 *
 * Layouts are the reference's: a padded sub-grid is (6, m, m, m) float64,
 * z fastest, m = n + 6; lo/hi are (13, 6, m, m, m); FX is (6, n+1, n, n),
 * FY (6, n, n+1, n), FZ (6, n, n, n+1).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stdint.h>
#include <pthread.h>
#include <unistd.h>

#define NF 6
#define NL 13
#define G 3

/* geometry.py:24-41 */
static const int DIRS[NL][3] = {
    {1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 0}, {1, -1, 0}, {1, 0, 1}, {1, 0, -1},
    {0, 1, 1}, {0, 1, -1}, {1, 1, 1}, {1, 1, -1}, {1, -1, 1}, {1, -1, -1}};

/* Face tables (geometry.py:51-123, flattened as flat_face_table). Filled by
 * orc_set_face_table from Python so the oracle consumes the reference's own
 * generator output rather than a hand-typed copy. */
static int FT_KIND[3][9], FT_NROW[3][9], FT_LINE[3][25], FT_DP[3][25][3], FT_FLIP[3][25];
static int FT_READY = 0;

int orc_set_face_table(int axis, const int *kind, const int *nrow, const int *line,
                       const int *dp, const int *flip) {
    if (axis < 0 || axis > 2) return -1;
    for (int i = 0; i < 9; i++) { FT_KIND[axis][i] = kind[i]; FT_NROW[axis][i] = nrow[i]; }
    for (int r = 0; r < 25; r++) {
        FT_LINE[axis][r] = line[r];
        FT_FLIP[axis][r] = flip[r];
        for (int c = 0; c < 3; c++) FT_DP[axis][r][c] = dp[3 * r + c];
    }
    FT_READY |= 1 << axis;
    return 0;
}

#define IDX4(v, i, j, k, m) ((((size_t)(v) * (m) + (i)) * (m) + (j)) * (m) + (k))

/* reference.py:30-45 (numpy primitives, used by both backends) */
void orc_primitives(const double *u, int m, double gamma, double eta, double *prim) {
    size_t nc = (size_t)m * m * m;
    for (size_t c = 0; c < nc; c++) {
        double rho = u[c], s1 = u[nc + c], s2 = u[2 * nc + c], s3 = u[3 * nc + c];
        double eg = u[4 * nc + c], tau = u[5 * nc + c];
        double inv = 1.0 / rho;
        double vx = s1 * inv, vy = s2 * inv, vz = s3 * inv;
        double kin = 0.5 * ((s1 * vx + s2 * vy) + s3 * vz);
        double e1 = eg - kin;
        double eint = (e1 >= eta * eg) ? e1 : pow(tau, gamma);
        double p = (gamma - 1.0) * eint;
        prim[c] = rho; prim[nc + c] = vx; prim[2 * nc + c] = vy; prim[3 * nc + c] = vz;
        prim[4 * nc + c] = p; prim[5 * nc + c] = tau;
    }
}

/* _core.pyx:159-173 */
static double mc_slope_at(const double *prim, int m, int i, int j, int k, int dx, int dy, int dz) {
    double am1 = prim[IDX4(0, i - dx, j - dy, k - dz, m)];
    double ap1 = prim[IDX4(0, i + dx, j + dy, k + dz, m)];
    double a = prim[IDX4(0, i, j, k, m)];
    double dc = 0.5 * (ap1 - am1);
    double dl = 2.0 * (a - am1);
    double dr = 2.0 * (ap1 - a);
    if (dl * dr <= 0.0) return 0.0;
    double mag = fmin(fabs(dc), fmin(fabs(dl), fabs(dr)));
    return dc < 0.0 ? -mag : mag;
}

/* _core.pyx:41-156.  lo/hi must be caller-provided (13,6,m,m,m); only the
 * active lines are written (inactive lines keep whatever the caller put). */
long orc_reconstruct(const double *prim, int m, int new_mode, int contact_on, double gamma,
                     double *lo, double *hi) {
    size_t nc = (size_t)m * m * m;
    double *tmp = (double *)malloc(sizeof(double) * NF * nc);
    int nlines = new_mode ? NL : 3;
    long fallback = 0;
    for (int l = 0; l < nlines; l++) {
        int dx = DIRS[l][0], dy = DIRS[l][1], dz = DIRS[l][2];
        int ilo = dx < 0 ? 2 : 1, ihi = dx < 0 ? m - 1 : m - 2;
        int jlo = dy < 0 ? 2 : 1, jhi = dy < 0 ? m - 1 : m - 2;
        int klo = dz < 0 ? 2 : 1, khi = dz < 0 ? m - 1 : m - 2;
        double *LO = lo + (size_t)l * NF * nc, *HI = hi + (size_t)l * NF * nc;
        for (int v = 0; v < NF; v++)
            for (int i = ilo; i < ihi; i++)
                for (int j = jlo; j < jhi; j++)
                    for (int k = klo; k < khi; k++) {
                        double a = prim[IDX4(v, i, j, k, m)];
                        double ap1 = prim[IDX4(v, i + dx, j + dy, k + dz, m)];
                        double am1 = prim[IDX4(v, i - dx, j - dy, k - dz, m)];
                        double ap2 = prim[IDX4(v, i + 2 * dx, j + 2 * dy, k + 2 * dz, m)];
                        double v7 = (7.0 / 12.0) * (a + ap1) - (1.0 / 12.0) * (am1 + ap2);
                        double mn = fmin(a, ap1), mx = fmax(a, ap1);
                        if (v7 < mn) v7 = mn;
                        if (v7 > mx) v7 = mx;
                        tmp[IDX4(v, i, j, k, m)] = v7;
                    }
        for (int v = 0; v < NF; v++)
            for (int i = 2; i < m - 2; i++)
                for (int j = 2; j < m - 2; j++)
                    for (int k = 2; k < m - 2; k++) {
                        double a = prim[IDX4(v, i, j, k, m)];
                        double hv = tmp[IDX4(v, i, j, k, m)];
                        double lv = tmp[IDX4(v, i - dx, j - dy, k - dz, m)];
                        if ((hv - a) * (a - lv) <= 0.0) {
                            lv = a;
                            hv = a;
                        } else {
                            double diff = hv - lv;
                            double mid = a - 0.5 * (lv + hv);
                            if (diff * mid > diff * diff / 6.0) lv = 3.0 * a - 2.0 * hv;
                            if (-diff * diff / 6.0 > diff * mid) hv = 3.0 * a - 2.0 * lv;
                        }
                        LO[IDX4(v, i, j, k, m)] = lv;
                        HI[IDX4(v, i, j, k, m)] = hv;
                    }
        if (contact_on) {
            for (int i = 2; i < m - 2; i++)
                for (int j = 2; j < m - 2; j++)
                    for (int k = 2; k < m - 2; k++) {
                        double ap1 = prim[IDX4(0, i + dx, j + dy, k + dz, m)];
                        double am1 = prim[IDX4(0, i - dx, j - dy, k - dz, m)];
                        double dr = ap1 - am1;
                        if (fabs(dr) <= 1e-300) continue;
                        double d2m = prim[IDX4(0, i, j, k, m)] - 2.0 * am1 +
                                     prim[IDX4(0, i - 2 * dx, j - 2 * dy, k - 2 * dz, m)];
                        double d2p = prim[IDX4(0, i + 2 * dx, j + 2 * dy, k + 2 * dz, m)] -
                                     2.0 * ap1 + prim[IDX4(0, i, j, k, m)];
                        if (d2m * d2p >= 0.0) continue;
                        if (fabs(dr) - 0.01 * fmin(fabs(ap1), fabs(am1)) <= 0.0) continue;
                        double pp1 = prim[IDX4(4, i + dx, j + dy, k + dz, m)];
                        double pm1 = prim[IDX4(4, i - dx, j - dy, k - dz, m)];
                        double pmin = fmin(pp1, pm1);
                        double rmin = fmin(fabs(ap1), fabs(am1));
                        if (fabs(pp1 - pm1) / pmin >= 0.1 * gamma * fabs(dr) / rmin) continue;
                        double eta_t = (d2m - d2p) / (6.0 * dr);
                        double eta = 20.0 * (eta_t - 0.05);
                        if (eta <= 0.0) continue;
                        if (eta > 1.0) eta = 1.0;
                        double sm = mc_slope_at(prim, m, i - dx, j - dy, k - dz, dx, dy, dz);
                        double sp = mc_slope_at(prim, m, i + dx, j + dy, k + dz, dx, dy, dz);
                        double lv = LO[IDX4(0, i, j, k, m)], hv = HI[IDX4(0, i, j, k, m)];
                        LO[IDX4(0, i, j, k, m)] = lv * (1.0 - eta) + (am1 + 0.5 * sm) * eta;
                        HI[IDX4(0, i, j, k, m)] = hv * (1.0 - eta) + (ap1 - 0.5 * sp) * eta;
                    }
        }
        for (int i = 2; i < m - 2; i++)
            for (int j = 2; j < m - 2; j++)
                for (int k = 2; k < m - 2; k++) {
                    if (LO[IDX4(0, i, j, k, m)] <= 0.0 || LO[IDX4(4, i, j, k, m)] <= 0.0) {
                        fallback++;
                        for (int v = 0; v < NF; v++) LO[IDX4(v, i, j, k, m)] = prim[IDX4(v, i, j, k, m)];
                    }
                    if (HI[IDX4(0, i, j, k, m)] <= 0.0 || HI[IDX4(4, i, j, k, m)] <= 0.0) {
                        fallback++;
                        for (int v = 0; v < NF; v++) HI[IDX4(v, i, j, k, m)] = prim[IDX4(v, i, j, k, m)];
                    }
                }
    }
    free(tmp);
    return fallback;
}

/* _core.pyx:180-220 */
static double kt_point(const double *L, const double *R, int axis, double gamma, double *out) {
    double rl = L[0], vxl = L[1], vyl = L[2], vzl = L[3], pl = L[4], tl = L[5];
    double rr = R[0], vxr = R[1], vyr = R[2], vzr = R[3], pr = R[4], tr = R[5];
    double cl = sqrt(gamma * pl / rl);
    double cr = sqrt(gamma * pr / rr);
    double vnl = axis == 0 ? vxl : (axis == 1 ? vyl : vzl);
    double vnr = axis == 0 ? vxr : (axis == 1 ? vyr : vzr);
    double ap = fmax(0.0, fmax(vnl + cl, vnr + cr));
    double am = fmin(0.0, fmin(vnl - cl, vnr - cr));
    double ul[6], ur[6], fl[6], fr[6];
    double kinl = 0.5 * rl * (vxl * vxl + vyl * vyl + vzl * vzl);
    double kinr = 0.5 * rr * (vxr * vxr + vyr * vyr + vzr * vzr);
    ul[0] = rl; ul[1] = rl * vxl; ul[2] = rl * vyl; ul[3] = rl * vzl;
    ul[4] = pl / (gamma - 1.0) + kinl; ul[5] = tl;
    ur[0] = rr; ur[1] = rr * vxr; ur[2] = rr * vyr; ur[3] = rr * vzr;
    ur[4] = pr / (gamma - 1.0) + kinr; ur[5] = tr;
    for (int v = 0; v < 6; v++) { fl[v] = ul[v] * vnl; fr[v] = ur[v] * vnr; }
    fl[1 + axis] += pl;
    fr[1 + axis] += pr;
    fl[4] += pl * vnl;
    fr[4] += pr * vnr;
    double denom = ap - am;
    if (denom > 0.0) {
        for (int v = 0; v < 6; v++) out[v] = (ap * fl[v] - am * fr[v] + (ap * am) * (ur[v] - ul[v])) / denom;
    } else {
        for (int v = 0; v < 6; v++) out[v] = fl[v];
    }
    return fmax(ap, -am);
}

/* _core.pyx:250-347 */
static double flux_axis(const double *lo, const double *hi, int m, double *F, int axis, int n,
                        double gamma, int new_mode, int override_center) {
    size_t nc = (size_t)m * m * m;
    int n0 = axis == 0 ? n + 1 : n, n1 = axis == 1 ? n + 1 : n, n2 = axis == 2 ? n + 1 : n;
    double amax = 0.0;
    for (int i0 = 0; i0 < n0; i0++)
        for (int i1 = 0; i1 < n1; i1++)
            for (int i2 = 0; i2 < n2; i2++) {
                int low0 = axis == 0 ? G - 1 + i0 : G + i0;
                int low1 = axis == 1 ? G - 1 + i1 : G + i1;
                int low2 = axis == 2 ? G - 1 + i2 : G + i2;
                int rr0 = 0, edge_i = 0, vert_i = 0;
                double Ls[6], Rs[6], fv[6], acc[6], center[6] = {0}, pdev[4][6], edev[6], vdev[6], pair01[6];
                for (int pt = 0; pt < 9; pt++) {
                    int kind = FT_KIND[axis][pt], nrow = FT_NROW[axis][pt];
                    if (kind != 0 && (!new_mode || override_center)) { rr0 += nrow; continue; }
                    for (int v = 0; v < 6; v++) acc[v] = 0.0;
                    for (int r = 0; r < nrow; r++) {
                        int l = FT_LINE[axis][rr0 + r];
                        int px = low0 + FT_DP[axis][rr0 + r][0];
                        int py = low1 + FT_DP[axis][rr0 + r][1];
                        int pz = low2 + FT_DP[axis][rr0 + r][2];
                        int qx = px + DIRS[l][0], qy = py + DIRS[l][1], qz = pz + DIRS[l][2];
                        const double *LOl = lo + (size_t)l * NF * nc, *HIl = hi + (size_t)l * NF * nc;
                        for (int v = 0; v < 6; v++) {
                            if (FT_FLIP[axis][rr0 + r]) {
                                Ls[v] = LOl[IDX4(v, qx, qy, qz, m)];
                                Rs[v] = HIl[IDX4(v, px, py, pz, m)];
                            } else {
                                Ls[v] = HIl[IDX4(v, px, py, pz, m)];
                                Rs[v] = LOl[IDX4(v, qx, qy, qz, m)];
                            }
                        }
                        double sp = kt_point(Ls, Rs, axis, gamma, fv);
                        if (sp > amax) amax = sp;
                        if (nrow == 4) {
                            if (r == 0 || r == 2) {
                                for (int v = 0; v < 6; v++) pair01[v] = fv[v];
                            } else {
                                for (int v = 0; v < 6; v++) acc[v] += pair01[v] + fv[v];
                            }
                        } else {
                            for (int v = 0; v < 6; v++) acc[v] += fv[v];
                        }
                    }
                    rr0 += nrow;
                    if (kind == 0) {
                        for (int v = 0; v < 6; v++) center[v] = acc[v];
                    } else if (kind == 1) {
                        for (int v = 0; v < 6; v++) pdev[edge_i][v] = 0.5 * acc[v] - center[v];
                        if (++edge_i == 4)
                            for (int v = 0; v < 6; v++) edev[v] = (pdev[0][v] + pdev[1][v]) + (pdev[2][v] + pdev[3][v]);
                    } else {
                        for (int v = 0; v < 6; v++) pdev[vert_i][v] = 0.25 * acc[v] - center[v];
                        if (++vert_i == 4)
                            for (int v = 0; v < 6; v++) vdev[v] = (pdev[0][v] + pdev[1][v]) + (pdev[2][v] + pdev[3][v]);
                    }
                }
                size_t s0 = (size_t)n1 * n2, fstride = (size_t)n0 * n1 * n2;
                for (int v = 0; v < 6; v++) {
                    double val = (new_mode && !override_center) ? center[v] + (4.0 * edev[v] + vdev[v]) / 36.0
                                                                : center[v];
                    F[v * fstride + i0 * s0 + (size_t)i1 * n2 + i2] = val;
                }
            }
    return amax;
}

/* _core.pyx:223-247 */
double orc_fluxes(const double *lo, const double *hi, int n, double gamma, int new_mode, int override_center,
                  double *fx, double *fy, double *fz) {
    if (FT_READY != 7) return NAN;
    int m = n + 2 * G;
    double a1 = flux_axis(lo, hi, m, fx, 0, n, gamma, new_mode, override_center);
    double a2 = flux_axis(lo, hi, m, fy, 1, n, gamma, new_mode, override_center);
    double a3 = flux_axis(lo, hi, m, fz, 2, n, gamma, new_mode, override_center);
    return fmax(a1, fmax(a2, a3));
}

/* NaN-propagating max (np.max semantics). */
static double nanmax2(double a, double b) {
    if (a != a || b != b) return NAN;
    return a > b ? a : b;
}

/* step.py:81-92 per leaf: max over cells of max_axis|s|/rho + c (eos.py:28-44). */
double orc_leaf_speed(const double *in, int n, double gamma, double eta) {
    size_t nc = (size_t)n * n * n;
    double best = -INFINITY;
    int first = 1;
    for (size_t c = 0; c < nc; c++) {
        double rho = in[c], sx = in[nc + c], sy = in[2 * nc + c], sz = in[3 * nc + c];
        double eg = in[4 * nc + c], tau = in[5 * nc + c];
        double vm = nanmax2(nanmax2(fabs(sx) / rho, fabs(sy) / rho), fabs(sz) / rho);
        double kin = 0.5 * ((sx * sx + sy * sy) + sz * sz) / rho;
        double e1 = eg - kin;
        double eint = (e1 >= eta * eg) ? e1 : pow(tau, gamma);
        double p = (gamma - 1.0) * eint;
        double cs = sqrt(gamma * p / rho);
        double s = vm + cs;
        best = first ? s : nanmax2(best, s);
        first = 0;
    }
    return best;
}

/* step.py:243-288 + eos.py:50-61 + sources.py:8-35, one leaf.
 * cur/u0/out are interiors (6,n,n,n); out may alias cur.
 * grav: NULL or (4,n,n,n) = gx, gy, gz, dphi_dt. */
void orc_update(const double *cur, const double *u0, const double *fx, const double *fy, const double *fz,
                int n, double dt, double a, double b, double inv_dx, double gamma, double eta,
                double omega, double ox, double oy, double dxl, const double *grav,
                double floor_rho, double floor_tau, double floor_vmax, double *out) {
    size_t nc = (size_t)n * n * n;
    size_t sxf = (size_t)n * n * n;           /* per-field strides of the flux arrays */
    size_t fxs = (size_t)(n + 1) * n * n, fys = (size_t)n * (n + 1) * n, fzs = (size_t)n * n * (n + 1);
    double w2 = omega * omega;
    double inv_gamma = 1.0 / gamma;
    int src = (omega != 0.0) || (grav != NULL);
    (void)sxf;
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++)
            for (int k = 0; k < n; k++) {
                size_t c = ((size_t)i * n + j) * n + k;
                double u[6], r[6], nw[6];
                for (int v = 0; v < 6; v++) u[v] = cur[v * nc + c];
                for (int v = 0; v < 6; v++) {
                    double dfx = fx[v * fxs + ((size_t)(i + 1) * n + j) * n + k] - fx[v * fxs + ((size_t)i * n + j) * n + k];
                    double dfy = fy[v * fys + ((size_t)i * (n + 1) + j + 1) * n + k] - fy[v * fys + ((size_t)i * (n + 1) + j) * n + k];
                    double dfz = fz[v * fzs + ((size_t)i * n + j) * (n + 1) + k + 1] - fz[v * fzs + ((size_t)i * n + j) * (n + 1) + k];
                    double t = 0.0 - dfx * inv_dx;
                    t = t - dfy * inv_dx;
                    t = t - dfz * inv_dx;
                    r[v] = t;
                }
                if (src) {
                    double x = ox + dxl * (double)i;
                    double y = oy + dxl * (double)j;
                    if (omega != 0.0) {
                        double ds[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                        ds[1] = 2.0 * omega * u[2] + u[0] * w2 * x;
                        ds[2] = -2.0 * omega * u[1] + u[0] * w2 * y;
                        ds[4] = w2 * (x * u[1] + y * u[2]);
                        for (int v = 0; v < 6; v++) r[v] = r[v] + ds[v];
                    }
                    if (grav) {
                        double gx = grav[c], gy = grav[nc + c], gz = grav[2 * nc + c], dp = grav[3 * nc + c];
                        double ds[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                        ds[1] = u[0] * gx;
                        ds[2] = u[0] * gy;
                        ds[3] = u[0] * gz;
                        ds[4] = u[1] * gx + u[2] * gy + u[3] * gz + 0.5 * u[0] * dp;
                        for (int v = 0; v < 6; v++) r[v] = r[v] + ds[v];
                    }
                }
                for (int v = 0; v < 6; v++) {
                    double st = u[v] + dt * r[v];
                    nw[v] = (a != 0.0) ? a * u0[v * nc + c] + b * st : st;
                }
                /* dual_energy_sync */
                {
                    double kin = 0.5 * ((nw[1] * nw[1] + nw[2] * nw[2]) + nw[3] * nw[3]) / nw[0];
                    double e1 = nw[4] - kin;
                    if (e1 >= eta * nw[4]) nw[5] = pow(fabs(e1), inv_gamma);
                }
                /* _apply_floors */
                if (floor_rho > 0.0 && nw[0] < floor_rho) nw[0] = floor_rho;
                if (floor_vmax > 0.0 && floor_rho > 0.0) {
                    int thin = nw[0] < 100.0 * floor_rho;
                    double v2 = ((nw[1] * nw[1] + nw[2] * nw[2]) + nw[3] * nw[3]) / (nw[0] * nw[0]);
                    if (thin && v2 > floor_vmax * floor_vmax) {
                        double scale = floor_vmax / sqrt(v2 > 1e-300 ? v2 : 1e-300);
                        double kin_old = 0.5 * ((nw[1] * nw[1] + nw[2] * nw[2]) + nw[3] * nw[3]) / nw[0];
                        nw[1] *= scale; nw[2] *= scale; nw[3] *= scale;
                        double kin_new = 0.5 * ((nw[1] * nw[1] + nw[2] * nw[2]) + nw[3] * nw[3]) / nw[0];
                        nw[4] += kin_new - kin_old;
                    }
                }
                if (floor_tau > 0.0 && nw[5] < floor_tau) nw[5] = floor_tau;
                for (int v = 0; v < 6; v++) out[v * nc + c] = nw[v];
            }
}

/* Batched primitives -> reconstruct -> fluxes over leaves (pthreads, one
 * leaf per work item), the part of one stage the reference runs per leaf
 * through run_kernels (step.py:115-127).  U: (L,6,m,m,m) ghost-filled. */
typedef struct {
    int L, n, new_mode, contact_on, override_center;
    const double *U;
    double gamma, eta;
    double *FX, *FY, *FZ, *amax;
    long *fallback;
    int next;
    pthread_mutex_t mu;
    int err;
} stage_job;

static void *stage_worker(void *arg) {
    stage_job *J = (stage_job *)arg;
    int m = J->n + 2 * G;
    size_t per_u = (size_t)NF * m * m * m, per_f = (size_t)NF * (J->n + 1) * J->n * J->n;
    double *prim = (double *)malloc(sizeof(double) * per_u);
    double *lo = (double *)calloc(NL * per_u, sizeof(double));
    double *hi = (double *)calloc(NL * per_u, sizeof(double));
    if (!prim || !lo || !hi) {
        pthread_mutex_lock(&J->mu); J->err = -1; pthread_mutex_unlock(&J->mu);
    } else {
        for (;;) {
            pthread_mutex_lock(&J->mu);
            int lf = J->next++;
            pthread_mutex_unlock(&J->mu);
            if (lf >= J->L) break;
            orc_primitives(J->U + lf * per_u, m, J->gamma, J->eta, prim);
            J->fallback[lf] = orc_reconstruct(prim, m, J->new_mode, J->contact_on, J->gamma, lo, hi);
            J->amax[lf] = orc_fluxes(lo, hi, J->n, J->gamma, J->new_mode, J->override_center,
                                     J->FX + lf * per_f, J->FY + lf * per_f, J->FZ + lf * per_f);
        }
    }
    free(prim); free(lo); free(hi);
    return NULL;
}

int orc_stage_fluxes(int L, int n, const double *U, double gamma, double eta, int new_mode, int contact_on,
                     int override_center, double *FX, double *FY, double *FZ, double *amax, long *fallback,
                     int nthreads) {
    if (FT_READY != 7) return -2;
    stage_job J = {L, n, new_mode, contact_on, override_center, U, gamma, eta, FX, FY, FZ, amax, fallback,
                   0, PTHREAD_MUTEX_INITIALIZER, 0};
    if (nthreads <= 0) nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (nthreads > L) nthreads = L > 0 ? L : 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    for (int t = 1; t < nthreads; t++) pthread_create(&th[t], NULL, stage_worker, &J);
    stage_worker(&J);
    for (int t = 1; t < nthreads; t++) pthread_join(th[t], NULL);
    free(th);
    return J.err;
}

int orc_max_threads(void) { return (int)sysconf(_SC_NPROCESSORS_ONLN); }

/* libm pow element-wise: the host side of the device pow self-check (tests only) */
void orc_pow_batch(const double *x, const double *y, long n, double *out) {
  for (long i = 0; i < n; i++) out[i] = pow(x[i], y[i]);
}
