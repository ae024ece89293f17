// Long-range Fourier-Chebyshev solver, two-sided proxy form (Algorithm 2; R9):
//   S8  anterpolation  S_b[g] = sum_j q_j L_b(z_j) W(x_g-x_j)_* W(y_g-y_j)_*
//   S10 scaling        S'_a(k) = sum_b K_ab(k) S_b(k)                 (K from P:907/P:533, R10)
//   S12 interpolation  phi_i = h_x h_y sum_g W W sum_a L_a(z_i) Psi_a[g]   (Eq. eq::SOGLong)
// L_b(x) = sum_n C[b][n] T_n(x), x = 2 z / L_z, at first-kind Chebyshev nodes (App. A.2).
// Proxy grids: [Pc][Ilx][Ily] real, spectra [Pc][Ilx][Ily/2+1].
#pragma once
#include <cuComplex.h>
#include "kernels_common.cuh"

namespace sog {

struct LongArgs {
    const d4* pos;
    int N;
    int Ilx, Ily, Pc;
    double hx, hy, halfx, halfy, hpx, hpy, invH2Sx, invH2Sy;
    double two_over_Lz;
    double A;                 // h_x h_y
    const double* C;          // [Pc][Pc] Chebyshev -> Lagrange
};

template <int PCMAX>
__device__ __forceinline__ void cheb_lagrange(double x, int Pc, const double* __restrict__ C, double* L,
                                              double* dL) {
    double T[PCMAX], dT[PCMAX];
    T[0] = 1.0;
    dT[0] = 0.0;
    T[1] = x;
    dT[1] = 1.0;
#pragma unroll
    for (int n = 1; n + 1 < PCMAX; ++n) {
        T[n + 1] = 2.0 * x * T[n] - T[n - 1];
        if (dL) dT[n + 1] = 2.0 * T[n] + 2.0 * x * dT[n] - dT[n - 1];
    }
#pragma unroll
    for (int b = 0; b < PCMAX; ++b) {
        double l = 0.0, dl = 0.0;
        if (b < Pc) {
#pragma unroll
            for (int n = 0; n < PCMAX; ++n)
                if (n < Pc) {
                    double c = __ldg(&C[b * Pc + n]);
                    l = fma(c, T[n], l);
                    if (dL) dl = fma(c, dT[n], dl);
                }
        }
        L[b] = l;
        if (dL) dL[b] = dl;
    }
}

template <int P, int PCMAX>
__global__ void __launch_bounds__(128) k_long_spread_atomic(LongArgs a, double* __restrict__ grid) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.N) return;
    constexpr int p = (P - 1) / 2;
    d4 r = ld_d4(&a.pos[i]);
    int gx0 = stencil_g0(r.x, a.hx, a.hpx), gy0 = stencil_g0(r.y, a.hy, a.hpy);
    double wx[P], wy[P], L[PCMAX];
    window_weights<P, false>(r.x, gx0, a.hx, a.halfx, a.invH2Sx, wx, nullptr);
    window_weights<P, false>(r.y, gy0, a.hy, a.halfy, a.invH2Sy, wy, nullptr);
    cheb_lagrange<PCMAX>(r.z * a.two_over_Lz, a.Pc, a.C, L, nullptr);
    const size_t layer = (size_t)a.Ilx * a.Ily;
    for (int u = 0; u < P; ++u) {
        int gx = wrap(gx0 - p + u, a.Ilx);
        double qx = r.w * wx[u];
        for (int v = 0; v < P; ++v) {
            int gy = wrap(gy0 - p + v, a.Ily);
            double* col = grid + (size_t)gx * a.Ily + gy;
            double qxy = qx * wy[v];
#pragma unroll
            for (int b = 0; b < PCMAX; ++b)
                if (b < a.Pc) atomicAdd(col + b * layer, qxy * L[b]);
        }
    }
}

// S10: one thread per (half mode, a).
static __global__ void k_long_scale(const cuDoubleComplex* __restrict__ in, cuDoubleComplex* __restrict__ out,
                             const double* __restrict__ K, int nmode, int Pc) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nmode * Pc) return;
    int mode = t / Pc, aa = t % Pc;
    const double* Km = K + ((size_t)mode * Pc + aa) * Pc;
    double re = 0, im = 0;
    for (int b = 0; b < Pc; ++b) {
        cuDoubleComplex v = in[(size_t)b * nmode + mode];
        re = fma(Km[b], v.x, re);
        im = fma(Km[b], v.y, im);
    }
    out[(size_t)aa * nmode + mode] = make_cuDoubleComplex(re, im);
}

template <int P, int PCMAX>
__global__ void __launch_bounds__(128) k_long_gather(LongArgs a, const double* __restrict__ psi, d4* __restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.N) return;
    constexpr int p = (P - 1) / 2;
    d4 r = ld_d4(&a.pos[i]);
    int gx0 = stencil_g0(r.x, a.hx, a.hpx), gy0 = stencil_g0(r.y, a.hy, a.hpy);
    double wx[P], wy[P], dwx[P], dwy[P], L[PCMAX], dL[PCMAX];
    window_weights<P, true>(r.x, gx0, a.hx, a.halfx, a.invH2Sx, wx, dwx);
    window_weights<P, true>(r.y, gy0, a.hy, a.halfy, a.invH2Sy, wy, dwy);
    cheb_lagrange<PCMAX>(r.z * a.two_over_Lz, a.Pc, a.C, L, dL);
    const size_t layer = (size_t)a.Ilx * a.Ily;
    double phi = 0, gx = 0, gy = 0, gz = 0;
    for (int u = 0; u < P; ++u) {
        int ix = wrap(gx0 - p + u, a.Ilx);
        double px = 0, pdy = 0, pdz = 0;
        for (int v = 0; v < P; ++v) {
            int iy = wrap(gy0 - p + v, a.Ily);
            const double* col = psi + (size_t)ix * a.Ily + iy;
            double t0 = 0, t1 = 0;
#pragma unroll
            for (int b = 0; b < PCMAX; ++b)
                if (b < a.Pc) {
                    double g = __ldg(col + b * layer);
                    t0 = fma(L[b], g, t0);
                    t1 = fma(dL[b], g, t1);
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
    st_d4(&out[i], d4{a.A * phi, a.A * gx, a.A * gy, a.A * gz * a.two_over_Lz});
}

}  // namespace sog
