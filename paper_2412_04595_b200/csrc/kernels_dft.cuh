// Long range without FFT (Algorithm 3, App. B; R8-D), two-sided Chebyshev
// proxies in the T basis as the FFT path (kernels_long.cuh):
//   S8-D  S~_n(k) = sum_j q_j T_n(2 z_j / Lz) exp(-i k . r_j)          (type-1 sums, Eq. eq::gridnonfft)
//   S10   Psi~_m(k) = sum_n K~_mn(k) S~_n(k)                             (k_long_scale, K~ = C^T K C)
//   S12-D phi_i = sum_m T_m(z_i) Re sum_k c_k Psi~_m(k) exp(i k . r_i)   (type-2 sums, Eq. eq::3.13A)
// over kx = 2 pi n / Lx, |n| <= Kx and ky = 2 pi n / Ly, 0 <= n <= Ky (half plane: c_k = 1 at ky = 0,
// 2 otherwise).  Mode index: mode = ix * nky + iy, ix = n_x + Kx.
#pragma once
#include <type_traits>
#include "kernels_long.cuh"

namespace sog {

struct DftArgs {
    int Kx, Ky, nkx, nky, nmode;
    double kx1, ky1;          // 2 pi / Lx, 2 pi / Ly
};

// exp(-i n k1 x) for n = -K..K (out[2 (n + K)] = re, [.. + 1] = im), scaled by s: recurrence from the
// centre outwards on one sincos
template <typename T>
__device__ __forceinline__ void dft_phases_x(double x, double k1, int K, double s, T* out) {
    double sn, cs;
    sincos(k1 * x, &sn, &cs);                 // e1 = exp(-i k1 x) = (cs, -sn)
    double pr = s, pi = 0.0;                  // n = 0
    out[2 * K] = T(pr);
    out[2 * K + 1] = T(pi);
    for (int n = 1; n <= K; ++n) {
        const double r = pr * cs + pi * sn, i = pi * cs - pr * sn;   // p * e1
        pr = r;
        pi = i;
        out[2 * (K + n)] = T(pr);             // exp(-i n k1 x)
        out[2 * (K + n) + 1] = T(pi);
        out[2 * (K - n)] = T(pr);             // exp(+i n k1 x) = conj
        out[2 * (K - n) + 1] = T(-pi);
    }
}

// S8-D: a block owns a particle range; its rows [ex (2 nkx) | ey (2 NKYP) | T (PCP)] are staged in
// shared memory (double-buffered); thread (ix, iy pair, 6 layers) accumulates 2 x 6 complex sums.
// Partials part[block][n][mode][2] are summed in a fixed order by k_long_sum (deterministic).
constexpr int DFT_KB = 64, DFT_LT = 6;

template <int PCP, int NYT, typename T = double>
__global__ void __launch_bounds__(256, NYT == 2 ? 2 : 1) k_long_dft_spread(LongArgs a, DftArgs d, int per, T* __restrict__ part) {
    constexpr int NLG = PCP / DFT_LT;   // NYT: ky modes per thread (2, or 4 for large mode sets)
    extern __shared__ __align__(16) unsigned char smraw[];
    T* sm = reinterpret_cast<T*>(smraw);
    using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
    const int nky2 = (d.nky + NYT - 1) / NYT;
    const int EX = 2 * d.nkx, EY = 2 * NYT * nky2, RW = ((EX + EY + PCP) + 1) & ~1;
    const int tid = threadIdx.x;
    const int lg = tid % NLG, cg = tid / NLG;
    const int ix = cg / nky2, iy0 = NYT * (cg % nky2);
    const bool own = ix < d.nkx;
    T ar[NYT][DFT_LT], ai[NYT][DFT_LT];
#pragma unroll
    for (int i = 0; i < NYT; ++i)
#pragma unroll
        for (int l = 0; l < DFT_LT; ++l) ar[i][l] = ai[i][l] = T(0);
    const int j0 = blockIdx.x * per, j1 = min(a.N, j0 + per);
    // two threads per staged particle: role 0 -> ex (times q) and T rows, role 1 -> ey row
    auto stage = [&](int base, int buf) {
        const int t = tid >> 1, role = tid & 1;
        if (t >= DFT_KB) return;
        T* row = sm + ((size_t)buf * DFT_KB + t) * RW;
        const int j = base + t;
        if (j >= j1) return;                  // slots >= nb are never read
        const d4 r = ld_d4(&a.pos[j]);
        if (role == 0) {
            dft_phases_x(r.x, d.kx1, d.Kx, r.w, row);
            T* tt = row + EX + EY;            // T_n(2z/Lz), n < PCP (rows n >= Pc are not summed)
            const double x = r.z * a.two_over_Lz;
            double tm = 1.0, tc = x;
            tt[0] = T(1);
            if (PCP > 1) tt[1] = T(x);
            for (int n = 2; n < PCP; ++n) {
                const double tn = 2.0 * x * tc - tm;
                tt[n] = T(tn);
                tm = tc; tc = tn;
            }
        } else {
            T* ey = row + EX;
            double sn, cs;
            sincos(d.ky1 * r.y, &sn, &cs);
            double pr = 1.0, pi = 0.0;
            for (int n = 0; n < NYT * nky2; ++n) {
                ey[2 * n] = T(n < d.nky ? pr : 0.0);
                ey[2 * n + 1] = T(n < d.nky ? pi : 0.0);
                const double rr = pr * cs + pi * sn, ii = pi * cs - pr * sn;
                pr = rr;
                pi = ii;
            }
        }
    };
    if (j0 < j1) stage(j0, 0);
    __syncthreads();
    int buf = 0;
    for (int base = j0; base < j1; base += DFT_KB, buf ^= 1) {
        if (base + DFT_KB < j1) stage(base + DFT_KB, buf ^ 1);
        const int nb = min(DFT_KB, j1 - base);
        if (own) {
            const T* rows = sm + (size_t)buf * DFT_KB * RW;
#pragma unroll 2
            for (int t = 0; t < nb; ++t) {
                const T* row = rows + (size_t)t * RW;
                const V2 ex = *reinterpret_cast<const V2*>(row + 2 * ix);
                T tl[DFT_LT];
#pragma unroll
                for (int l = 0; l < DFT_LT; l += 2) {
                    const V2 v = *reinterpret_cast<const V2*>(row + EX + EY + lg * DFT_LT + l);
                    tl[l] = v.x; tl[l + 1] = v.y;
                }
                T re[NYT], im[NYT];
#pragma unroll
                for (int i = 0; i < NYT; ++i) {
                    const V2 e = *reinterpret_cast<const V2*>(row + EX + 2 * (iy0 + i));
                    re[i] = ex.x * e.x - ex.y * e.y;
                    im[i] = ex.x * e.y + ex.y * e.x;
                }
#pragma unroll
                for (int i = 0; i < NYT; ++i)
#pragma unroll
                    for (int l = 0; l < DFT_LT; ++l) {
                        ar[i][l] = fma(re[i], tl[l], ar[i][l]);
                        ai[i][l] = fma(im[i], tl[l], ai[i][l]);
                    }
            }
        }
        __syncthreads();
    }
    if (own) {
        const size_t G = 2 * (size_t)d.nmode;
        T* o = part + (size_t)blockIdx.x * PCP * G;
#pragma unroll
        for (int i = 0; i < NYT; ++i)
#pragma unroll
            for (int l = 0; l < DFT_LT; ++l) {
                const int iy = iy0 + i, n = lg * DFT_LT + l;
                if (iy < d.nky) {
                    const size_t m = (size_t)ix * d.nky + iy;
                    o[(size_t)n * G + 2 * m] = ar[i][l];
                    o[(size_t)n * G + 2 * m + 1] = ai[i][l];
                }
            }
    }
}

// S12-D: one thread per particle; Psi~ in shared memory as [mode][PCP] complex, walked by every
// thread in the same order (broadcast loads).  Per mode: G = sum_m T_m Psi~_m, G' with T'_m, the
// phase exp(i k . r) by recurrences along kx (outer) and ky (inner).
template <int PCP, typename T = double>
__global__ void __launch_bounds__(128, 4) k_long_dft_gather(LongArgs a, DftArgs d, const T* __restrict__ psi,
                                                          d4* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smraw[];
    T* sPsi = reinterpret_cast<T*>(smraw);                 // [nmode][PCP][2]
    using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
    for (int e = threadIdx.x; e < d.nmode * PCP; e += blockDim.x) {
        const int m = e / PCP, n = e - m * PCP;
        const bool in = n < a.Pc;
        sPsi[2 * e] = in ? psi[2 * ((size_t)n * d.nmode + m)] : T(0);
        sPsi[2 * e + 1] = in ? psi[2 * ((size_t)n * d.nmode + m) + 1] : T(0);
    }
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const bool act = j < a.N;
    const d4 r = act ? ld_d4(&a.pos[j]) : d4{0.0, 0.0, 0.0, 0.0};
    T Tn[PCP], dT[PCP];
    {
        const double x = r.z * a.two_over_Lz;
        double t0 = 1.0, t1 = x, d0v = 0.0, d1v = 1.0;
        Tn[0] = T(t0); dT[0] = T(d0v);
        if (PCP > 1) { Tn[1] = T(t1); dT[1] = T(d1v); }
#pragma unroll
        for (int n = 1; n + 1 < PCP; ++n) {
            const double t2 = 2.0 * x * t1 - t0, d2 = 2.0 * t1 + 2.0 * x * d1v - d0v;
            Tn[n + 1] = T(t2); dT[n + 1] = T(d2);
            t0 = t1; t1 = t2; d0v = d1v; d1v = d2;
        }
    }
    __syncthreads();
    double snx, csx, sny, csy;
    sincos(d.kx1 * r.x, &snx, &csx);
    sincos(d.ky1 * r.y, &sny, &csy);
    // exp(i n_x k1 x) from n_x = -Kx: start at conj(e1)^Kx
    double xr = 1.0, xi = 0.0;
    for (int n = 0; n < d.Kx; ++n) {
        const double rr = xr * csx + xi * snx, ii = xi * csx - xr * snx;
        xr = rr; xi = ii;
    }
    T phi = 0, gx = 0, gy = 0, gz = 0;
    for (int ix = 0; ix < d.nkx; ++ix) {
        const T kx = T(d.kx1 * (ix - d.Kx));
        double pr = xr, pim = xi;                           // exp(i (kx x + ky y)), ky = 0
        T ax = 0, ay = 0;                                   // sum_k c Im(P) weighted for the x, y gradients
        for (int iy = 0; iy < d.nky; ++iy) {
            const V2* c2 = reinterpret_cast<const V2*>(sPsi + 2 * (size_t)(ix * d.nky + iy) * PCP);
            T gr = 0, gi = 0, dr = 0, di = 0;
#pragma unroll
            for (int n = 0; n < PCP; ++n) {
                const V2 ps = c2[n];
                gr = fma(Tn[n], ps.x, gr);
                gi = fma(Tn[n], ps.y, gi);
                dr = fma(dT[n], ps.x, dr);
                di = fma(dT[n], ps.y, di);
            }
            const T c = iy == 0 ? T(1) : T(2);
            const T er = T(pr) * c, ei = T(pim) * c;
            const T Pr = gr * er - gi * ei, Pi = gr * ei + gi * er;
            phi += Pr;
            ax += Pi;
            ay = fma(T(d.ky1 * iy), Pi, ay);
            gz += dr * er - di * ei;
            const double rr = pr * csy - pim * sny, ii = pim * csy + pr * sny;   // times exp(i ky1 y)
            pr = rr; pim = ii;
        }
        gx = fma(-kx, ax, gx);                              // Re(i kx P) = -kx Im(P)
        gy -= ay;
        const double rr = xr * csx - xi * snx, ii = xi * csx + xr * snx;         // times exp(i kx1 x)
        xr = rr; xi = ii;
    }
    if (act) st_d4(&out[j], d4{double(phi), double(gx), double(gy), double(gz) * a.two_over_Lz});
}

}  // namespace sog
