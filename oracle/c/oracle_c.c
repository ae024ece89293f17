/* Plain C loops for the oracle at full BASELINE sizes (N up to 1e7).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Nothing here is blocked, fused or
 * reordered beyond the formula it states: these are the same sums as the NumPy functions
 * named below, written as loops so that N = 1e7 finishes in seconds.  Built by
 * __graft_entry__.build() into oracle/lib/liboracle_c.so; shares no code with the CUDA path.
 *
 *   oracle_mid_spread  -- Eq. eq::gridding:
 *                         S[g] += q_j Wx_j(a) Wy_j(b) Wz_j(c) at g = (gx_j[a], gy_j[b], gz_j[c]),
 *                         on the [Ix][Iy][Izs] grid; the stencil indices and weights come from
 *                         oracle/sog.py:stencil (same as oracle.sog.mid_spread, which uses np.add.at)
 *   oracle_ewald2d     -- the textbook Ewald2D sum of oracle/ewald2d.py:ewald2d (SURVEY 8(c),
 *                         Parry 1975 cited at P:991) at sampled targets, one target per thread.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

void oracle_mid_spread(int64_t N, int P, int64_t Ix, int64_t Iy, int64_t Izs, const int64_t* gx, const int64_t* gy,
                       const int64_t* gz, const double* Wx, const double* Wy, const double* Wz, const double* q,
                       double* S) {
    /* threads own disjoint ranges of x planes and each visits every particle in order, so every
     * grid point receives its terms in the serial order (bitwise equal to one thread) */
#pragma omp parallel
    {
        int nt = 1, t = 0;
#ifdef _OPENMP
        nt = omp_get_num_threads();
        t = omp_get_thread_num();
#endif
        const int64_t x0 = Ix * t / nt, x1 = Ix * (t + 1) / nt;
    for (int64_t j = 0; j < N; ++j) {
        for (int a = 0; a < P; ++a) {
            if (gx[j * P + a] < x0 || gx[j * P + a] >= x1) continue;
            for (int b = 0; b < P; ++b) {
                const double qab = q[j] * Wx[j * P + a] * Wy[j * P + b];
                double* col = S + (gx[j * P + a] * Iy + gy[j * P + b]) * Izs;
                for (int c = 0; c < P; ++c) col[gz[j * P + c]] += qab * Wz[j * P + c];
            }
        }
    }
    }
}

/* g(k, z) = exp(k z) erfc(k / (2 alpha) + alpha z).  For x = k/(2 alpha) + alpha z > 26, erfc
 * underflows while the exact value is below exp(-(k/2alpha)^2 - (alpha z)^2) < exp(-169): 0. */
static double g_fn(double k, double z, double alpha) {
    const double x = k / (2.0 * alpha) + alpha * z;
    if (x > 26.0) return 0.0;
    return exp(k * z) * erfc(x);
}

/* phi[t], grad[t][3] at targets tgt[t]; alpha, rcut, kcut as in oracle/ewald2d.py */
void oracle_ewald2d(int64_t N, const double* xyz, const double* q, double Lx, double Ly, int64_t nt,
                    const int64_t* tgt, double alpha, double rcut, double kcut, double* phi, double* grad) {
    const double PI = 3.14159265358979323846, SQPI = 1.77245385090551602730;
    const double A = Lx * Ly;
    const int nx = (int)ceil(rcut / Lx) + 1, ny = (int)ceil(rcut / Ly) + 1;
    const int mx = (int)ceil(kcut * Lx / (2 * PI)), my = (int)ceil(kcut * Ly / (2 * PI));
    /* half plane of kdot != 0 modes (pairs k, -k: factor 2) */
    int nm = 0;
    double* modes = (double*)malloc(sizeof(double) * 3 * (size_t)(mx + 1) * (2 * my + 1));
    for (int a = 0; a <= mx; ++a)
        for (int b = -my; b <= my; ++b) {
            if (a == 0 && b <= 0) continue;
            const double kx = 2 * PI * a / Lx, ky = 2 * PI * b / Ly, k = hypot(kx, ky);
            if (k <= kcut) {
                modes[3 * nm] = kx;
                modes[3 * nm + 1] = ky;
                modes[3 * nm + 2] = k;
                ++nm;
            }
        }
    const double rc2 = rcut * rcut;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t it = 0; it < nt; ++it) {
        const int64_t i = tgt[it];
        const double xi = xyz[3 * i], yi = xyz[3 * i + 1], zi = xyz[3 * i + 2];
        double p = 0, gx = 0, gy = 0, gz = 0;
        /* real space: sum_j sum'_n q_j erfc(alpha |r_ij + n|) / |r_ij + n| */
        for (int n1 = -nx; n1 <= nx; ++n1)
            for (int n2 = -ny; n2 <= ny; ++n2)
                for (int64_t j = 0; j < N; ++j) {
                    if (n1 == 0 && n2 == 0 && j == i) continue;
                    const double X = xi - xyz[3 * j] + n1 * Lx, Y = yi - xyz[3 * j + 1] + n2 * Ly, Z = zi - xyz[3 * j + 2];
                    const double r2 = X * X + Y * Y + Z * Z;
                    if (!(r2 < rc2)) continue;
                    const double r = sqrt(r2), er = erfc(alpha * r);
                    p += q[j] * er / r;
                    const double dfr = -(er / r2 + 2 * alpha / SQPI * exp(-alpha * alpha * r2) / r);
                    const double c = q[j] * dfr / r;
                    gx += c * X;
                    gy += c * Y;
                    gz += c * Z;
                }
        /* kdot != 0: (pi/A) sum_j q_j sum_k cos(k.rho_ij)/k [g(k,z_ij) + g(k,-z_ij)], both half planes */
        for (int m = 0; m < nm; ++m) {
            const double kx = modes[3 * m], ky = modes[3 * m + 1], k = modes[3 * m + 2];
            const double c = 2.0 * (PI / A) / k;
            double sp = 0, sx = 0, sy = 0, sz = 0;
            for (int64_t j = 0; j < N; ++j) {
                const double dx = xi - xyz[3 * j], dy = yi - xyz[3 * j + 1], dz = zi - xyz[3 * j + 2];
                const double ph = kx * dx + ky * dy, cs = cos(ph), sn = sin(ph);
                const double gp = g_fn(k, dz, alpha), gm = g_fn(k, -dz, alpha);
                sp += q[j] * cs * (gp + gm);
                sx += -q[j] * kx * sn * (gp + gm);
                sy += -q[j] * ky * sn * (gp + gm);
                sz += q[j] * cs * k * (gp - gm);
            }
            p += c * sp;
            gx += c * sx;
            gy += c * sy;
            gz += c * sz;
        }
        /* kdot == 0 and self */
        for (int64_t j = 0; j < N; ++j) {
            const double dz = zi - xyz[3 * j + 2];
            p += -(2 * PI / A) * q[j] * (dz * erf(alpha * dz) + exp(-alpha * alpha * dz * dz) / (alpha * SQPI));
            gz += -(2 * PI / A) * q[j] * erf(alpha * dz);
        }
        p += -2.0 * alpha * q[i] / SQPI;
        phi[it] = p;
        grad[3 * it] = gx;
        grad[3 * it + 1] = gy;
        grad[3 * it + 2] = gz;
    }
    free(modes);
}
