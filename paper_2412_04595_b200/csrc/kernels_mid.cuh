// Mid-range Fourier spectral solver (Algorithm 1).
//   S3 gridding  S[g] = sum_j q_j W(x_g-x_j)_* W(y_g-y_j)_* W(z_g-z_j)   (Eq. eq::gridding)
//   S5 scaling   S_hat <- mult(k) S_hat                                  (Eq. eq::widehat-tilde)
//   S7 gathering phi_i = V_h sum_g W W W Psi[g] (+ gradient with W')     (Eq. eq::Phiconv)
// Grid layout: real [Ix][Iy][Izs] row-major (z fastest); half spectrum [Ix][Iy][Izs/2+1].
#pragma once
#include <cuComplex.h>
#include "kernels_common.cuh"

namespace sog {

struct MidArgs {
    const d4* pos;
    int N;
    int Ix, Iy, Izs;
    double hx, hy, hz;
    double halfx, halfy, halfz;          // I/2 (grid centre offsets)
    double hpx, hpy, hpz;                // I/2 + 1/2 (nearest-point decision constants)
    double invH2Sx, invH2Sy, invH2Sz;    // S / H_d^2
    double Vh;                           // h_x h_y h_z
};

// v1 spread: one thread per particle, separable weights in registers, fp64 RED to global.
template <int P>
__global__ void __launch_bounds__(128) k_mid_spread_atomic(MidArgs a, double* __restrict__ grid) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.N) return;
    constexpr int p = (P - 1) / 2;
    d4 r = ld_d4(&a.pos[i]);
    int gx0 = stencil_g0(r.x, a.hx, a.hpx), gy0 = stencil_g0(r.y, a.hy, a.hpy), gz0 = stencil_g0(r.z, a.hz, a.hpz);
    double wx[P], wy[P], wz[P];
    window_weights<P, false>(r.x, gx0, a.hx, a.halfx, a.invH2Sx, wx, nullptr);
    window_weights<P, false>(r.y, gy0, a.hy, a.halfy, a.invH2Sy, wy, nullptr);
    window_weights<P, false>(r.z, gz0, a.hz, a.halfz, a.invH2Sz, wz, nullptr);
    const size_t zb = (size_t)(gz0 - p);
    for (int u = 0; u < P; ++u) {
        size_t bx = (size_t)wrap(gx0 - p + u, a.Ix) * a.Iy;
        double qx = r.w * wx[u];
        for (int v = 0; v < P; ++v) {
            double* col = grid + ((bx + wrap(gy0 - p + v, a.Iy)) * a.Izs + zb);
            double qxy = qx * wy[v];
#pragma unroll
            for (int c = 0; c < P; ++c) atomicAdd(col + c, qxy * wz[c]);
        }
    }
}

// S5: multiply the half spectrum by mult(k) = sum_{l<=m} A_l Tx[l][ix] Ty[l][iy] Tz[l][iz].
static __global__ void k_mid_scale(cuDoubleComplex* __restrict__ spec, int Ix, int Iy, int nz, int L,
                            const double* __restrict__ A, const double* __restrict__ Tx,
                            const double* __restrict__ Ty, const double* __restrict__ Tz) {
    int iz = blockIdx.x * blockDim.x + threadIdx.x;
    int iy = blockIdx.y, ix = blockIdx.z;
    if (iz >= nz) return;
    double mult = 0.0;
    for (int l = 0; l < L; ++l)
        mult = fma(A[l] * Tx[(size_t)l * Ix + ix] * Ty[(size_t)l * Iy + iy], Tz[(size_t)l * nz + iz], mult);
    size_t idx = ((size_t)ix * Iy + iy) * nz + iz;
    cuDoubleComplex v = spec[idx];
    spec[idx] = make_cuDoubleComplex(v.x * mult, v.y * mult);
}

// v1 gather: one thread per particle, reads the P^3 stencil of Psi (L1/L2 cached).
template <int P>
__global__ void __launch_bounds__(128) k_mid_gather(MidArgs a, const double* __restrict__ psi, d4* __restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.N) return;
    constexpr int p = (P - 1) / 2;
    d4 r = ld_d4(&a.pos[i]);
    int gx0 = stencil_g0(r.x, a.hx, a.hpx), gy0 = stencil_g0(r.y, a.hy, a.hpy), gz0 = stencil_g0(r.z, a.hz, a.hpz);
    double wx[P], wy[P], wz[P], dwx[P], dwy[P], dwz[P];
    window_weights<P, true>(r.x, gx0, a.hx, a.halfx, a.invH2Sx, wx, dwx);
    window_weights<P, true>(r.y, gy0, a.hy, a.halfy, a.invH2Sy, wy, dwy);
    window_weights<P, true>(r.z, gz0, a.hz, a.halfz, a.invH2Sz, wz, dwz);
    const size_t zb = (size_t)(gz0 - p);
    double phi = 0, gx = 0, gy = 0, gz = 0;
    for (int u = 0; u < P; ++u) {
        size_t bx = (size_t)wrap(gx0 - p + u, a.Ix) * a.Iy;
        double px = 0, pdz = 0, pdy = 0;
        for (int v = 0; v < P; ++v) {
            const double* col = psi + ((bx + wrap(gy0 - p + v, a.Iy)) * a.Izs + zb);
            double t0 = 0, t1 = 0;
#pragma unroll
            for (int c = 0; c < P; ++c) {
                double g = __ldg(col + c);
                t0 = fma(wz[c], g, t0);
                t1 = fma(dwz[c], g, t1);
            }
            px = fma(wy[v], t0, px);
            pdy = fma(dwy[v], t0, pdy);
            pdz = fma(wy[v], t1, pdz);
        }
        phi = fma(wx[u], px, phi);
        gx = fma(dwx[u], px, gx);
        gy = fma(wx[u], pdy, gy);
        gz = fma(wx[u], pdz, gz);
    }
    st_d4(&out[i], d4{a.Vh * phi, a.Vh * gx, a.Vh * gy, a.Vh * gz});
}

}  // namespace sog
