// S2: near-field pair sum over the cell list (Eq. eq::phiNDR):
//   Phi^N_i = sum_{j: |r_ij| < r_c} q_j N(r_ij),  N(r) = 1/r - F(r^2),
//   grad_i Phi^N = sum_j q_j (-1/r^3 - 2 F'(u)) r_ij      (u = r^2; R11)
// with F(u) = sum_l w_l exp(-u/s_l^2) from a piecewise Taylor table in u (R16).
#pragma once
#include "kernels_common.cuh"

namespace sog {

struct NearArgs {
    const d4* pos;          // sorted (x,y,z,q)
    const int* start;       // cell start offsets [ncell+1]
    const double* cF;       // table K x (D+1)
    const double* cdF;
    d4* out;                // (phi, gx, gy, gz) per sorted particle
    int N, K;
    double du, inv_du, rc2;
    CellGeo g;
    int ox[3], noffx, oy[3], noffy;   // distinct periodic cell offsets (handles nc < 3)
};

template <int D>
__global__ void __launch_bounds__(256) k_near(NearArgs a) {
    extern __shared__ double tab[];   // [K*(D+1)] F then [K*(D+1)] dF
    const int nt = a.K * (D + 1);
    for (int t = threadIdx.x; t < nt; t += blockDim.x) {
        tab[t] = a.cF[t];
        tab[nt + t] = a.cdF[t];
    }
    __syncthreads();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.N) return;
    const d4 pi = ld_d4(&a.pos[i]);
    const CellGeo& g = a.g;
    int cx = min(g.ncx - 1, max(0, (int)floor((pi.x + 0.5 * g.Lx) * g.sx)));
    int cy = min(g.ncy - 1, max(0, (int)floor((pi.y + 0.5 * g.Ly) * g.sy)));
    int cz = min(g.ncz - 1, max(0, (int)floor((pi.z + 0.5 * g.Lz) * g.sz)));
    double phi = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
    for (int ix = 0; ix < a.noffx; ++ix) {
        int nx = cx + a.ox[ix];
        nx = nx < 0 ? nx + g.ncx : (nx >= g.ncx ? nx - g.ncx : nx);
        for (int iy = 0; iy < a.noffy; ++iy) {
            int ny = cy + a.oy[iy];
            ny = ny < 0 ? ny + g.ncy : (ny >= g.ncy ? ny - g.ncy : ny);
            int z0 = max(0, cz - g.nzr), z1 = min(g.ncz - 1, cz + g.nzr);
            int c0 = (nx * g.ncy + ny) * g.ncz;
            int j0 = a.start[c0 + z0], j1 = a.start[c0 + z1 + 1];   // z-adjacent cells are contiguous
            for (int j = j0; j < j1; ++j) {
                d4 pj = ld_d4(&a.pos[j]);
                double dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
                dx -= g.Lx * rint(dx * g.invLx);       // minimum image in x, y (never z)
                dy -= g.Ly * rint(dy * g.invLy);
                double u = dx * dx + dy * dy + dz * dz;
                if (u < a.rc2 && j != i) {
                    int k = min(a.K - 1, (int)(u * a.inv_du));
                    double d = u - (k + 0.5) * a.du;
                    const double* cf = tab + k * (D + 1);
                    const double* cd = tab + nt + k * (D + 1);
                    double F = cf[D], dF = cd[D - 1];
#pragma unroll
                    for (int n = D - 1; n >= 0; --n) F = fma(F, d, cf[n]);
#pragma unroll
                    for (int n = D - 2; n >= 0; --n) dF = fma(dF, d, cd[n]);
                    double rinv = rsqrt(u);
                    phi = fma(pj.w, rinv - F, phi);
                    double c = pj.w * (-rinv * rinv * rinv - 2.0 * dF);
                    gx = fma(c, dx, gx);
                    gy = fma(c, dy, gy);
                    gz = fma(c, dz, gz);
                }
            }
        }
    }
    st_d4(&a.out[i], d4{phi, gx, gy, gz});
}

}  // namespace sog
