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

}  // namespace sog

namespace sog {

// ---------------------------------------------------------------------------------------
// S8 v2: output-stationary anterpolation.  A CTA owns a tile of TX x TY long-grid columns
// (one thread per column, all Pc layers of its column in registers) and one chunk of the
// particles whose stencils can reach the tile.  Particles are staged in shared memory in
// batches (weights by recurrence, Chebyshev T_n, then L_b = sum_n C[b][n] T_n spread over
// all threads); every column thread adds c = q Wx Wy times L_b(z) to its Pc accumulators.
// Partials go to part[tile][chunk][col][Pc]; k_long_reduce sums chunks in a fixed order, so
// the result is deterministic (no atomics).
struct LongTileArgs {
    LongArgs a;
    int TX, TY, ntx, nty, nchunk;
    int full_range;          // 1: every particle reaches every tile (small periodic grid)
    const int* start;        // cell start offsets (sorted order), for x-slab particle ranges
    int ncx, cells_per_x;    // near-cell grid: ncx slabs of cells_per_x = ncy*ncz cells
    double cell_w;           // Lx / ncx
    double Lx;
    double gamma_x, gamma_y; // window recurrence constants exp(-2 a h^2)
    double* part;
};

constexpr int LB = 64;       // particles per staged batch

template <int P, int PCMAX>
__global__ void __launch_bounds__(256) k_long_spread_tile(LongTileArgs t) {
    extern __shared__ double sm[];
    double* sC = sm;                          // [Pc*Pc]
    double* sW = sC + PCMAX * PCMAX;          // [LB][2P]
    double* sT = sW + LB * 2 * P;             // [LB][PCMAX] Chebyshev T_n, then L_b
    double* sL = sT + LB * PCMAX;             // [LB][PCMAX] L_b(z_j)
    double* sQ = sL + LB * PCMAX;             // [LB]
    int* sG = (int*)(sQ + LB);                // [LB][2]
    const LongArgs& a = t.a;
    constexpr int p = (P - 1) / 2;
    const int Pc = a.Pc;
    const int tile = blockIdx.y, chunk = blockIdx.x;
    const int X0 = (tile / t.nty) * t.TX, Y0 = (tile % t.nty) * t.TY;
    const int tid = threadIdx.x, nthr = blockDim.x;
    for (int k = tid; k < Pc * Pc; k += nthr) sC[k] = a.C[k];
    // particle index ranges reaching this tile (1 or 2 ranges of x-slabs)
    int r0b = 0, r0e = a.N, r1b = 0, r1e = 0;
    if (!t.full_range) {
        // stencil centres gx0 in [X0 - p, X0 + TX - 1 + p] <=> x in [xlo, xhi)
        double xlo = ((X0 - p) - 0.5 - 0.5 * a.Ilx) * a.hx, xhi = ((X0 + t.TX - 1 + p) + 0.5 - 0.5 * a.Ilx) * a.hx;
        int c0 = (int)floor((xlo + 0.5 * t.Lx) / t.cell_w) - 1, c1 = (int)floor((xhi + 0.5 * t.Lx) / t.cell_w) + 1;
        if (c1 - c0 + 1 >= t.ncx) { c0 = 0; c1 = t.ncx - 1; }
        if (c0 < 0) {
            r1b = t.start[(c0 + t.ncx) * t.cells_per_x]; r1e = a.N; c0 = 0;
        } else if (c1 >= t.ncx) {
            r1b = 0; r1e = t.start[(c1 - t.ncx + 1) * t.cells_per_x]; c1 = t.ncx - 1;
        }
        r0b = t.start[c0 * t.cells_per_x];
        r0e = t.start[(c1 + 1) * t.cells_per_x];
    }
    const int n0 = r0e - r0b, ntot = n0 + (r1e - r1b);
    const int per = (ntot + t.nchunk - 1) / t.nchunk;
    const int jb = min(ntot, chunk * per), je = min(ntot, jb + per);
    // my column
    const int cx = X0 + tid / t.TY, cy = Y0 + tid % t.TY;
    const bool own = tid < t.TX * t.TY && cx < a.Ilx && cy < a.Ily;
    double acc[PCMAX];
#pragma unroll
    for (int b = 0; b < PCMAX; ++b) acc[b] = 0.0;
    __syncthreads();
    for (int base = jb; base < je; base += LB) {
        const int nb = min(LB, je - base);
        if (tid < nb) {
            int k = base + tid;
            int j = k < n0 ? r0b + k : r1b + (k - n0);
            d4 r = ld_d4(&a.pos[j]);
            int gx0 = stencil_g0(r.x, a.hx, a.hpx), gy0 = stencil_g0(r.y, a.hy, a.hpy);
            double wx[P], wy[P];
            window_weights_rec<P, false>(r.x, gx0, a.hx, a.halfx, a.invH2Sx, t.gamma_x, wx, nullptr);
            window_weights_rec<P, false>(r.y, gy0, a.hy, a.halfy, a.invH2Sy, t.gamma_y, wy, nullptr);
#pragma unroll
            for (int u = 0; u < P; ++u) { sW[tid * 2 * P + u] = wx[u]; sW[tid * 2 * P + P + u] = wy[u]; }
            sQ[tid] = r.w;
            sG[2 * tid] = gx0 - p;
            sG[2 * tid + 1] = gy0 - p;
            double x = r.z * a.two_over_Lz;
            double tm = 1.0, tc = x;
            sT[tid * PCMAX] = 1.0;
            if (Pc > 1) sT[tid * PCMAX + 1] = x;
            for (int n = 2; n < Pc; ++n) {
                double tn = 2.0 * x * tc - tm;
                sT[tid * PCMAX + n] = tn;
                tm = tc; tc = tn;
            }
        }
        __syncthreads();
        // L_b(z_j) = sum_n C[b][n] T_n(x_j), (j, b) pairs over all threads
        for (int q = tid; q < nb * PCMAX; q += nthr) {
            int j = q / PCMAX, b = q % PCMAX;
            double s = 0.0;
            if (b < Pc)
                for (int n = 0; n < Pc; ++n) s = fma(sC[b * Pc + n], sT[j * PCMAX + n], s);
            sL[q] = s;
        }
        __syncthreads();
        if (own) {
            for (int j = 0; j < nb; ++j) {
                int u = cx - sG[2 * j], v = cy - sG[2 * j + 1];
                u += u < 0 ? a.Ilx : 0; u -= u >= a.Ilx ? a.Ilx : 0;
                v += v < 0 ? a.Ily : 0; v -= v >= a.Ily ? a.Ily : 0;
                if (u < P && v < P) {
                    const double c = sQ[j] * sW[j * 2 * P + u] * sW[j * 2 * P + P + v];
                    const double2* L2 = reinterpret_cast<const double2*>(sL + j * PCMAX);
#pragma unroll
                    for (int b = 0; b < PCMAX; b += 2) {
                        if (b < Pc) {
                            double2 l = L2[b / 2];
                            acc[b] = fma(c, l.x, acc[b]);
                            acc[b + 1] = fma(c, l.y, acc[b + 1]);
                        }
                    }
                }
            }
        }
        __syncthreads();
    }
    if (own) {
        double* o = t.part + (((size_t)tile * t.nchunk + chunk) * (t.TX * t.TY) + tid) * PCMAX;
#pragma unroll
        for (int b = 0; b < PCMAX; ++b) o[b] = acc[b];
    }
}

// grid[b][gx][gy] = sum over chunks (fixed order) of the tile partials.
static __global__ void k_long_reduce(const double* __restrict__ part, double* __restrict__ grid, int Ilx, int Ily,
                                     int Pc, int PCMAX, int TX, int TY, int nty, int nchunk) {
    int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= Ilx * Ily * Pc) return;
    int b = idx / (Ilx * Ily), g = idx % (Ilx * Ily);
    int gx = g / Ily, gy = g % Ily;
    int tile = (gx / TX) * nty + gy / TY, col = (gx % TX) * TY + gy % TY;
    const double* p = part + ((size_t)tile * nchunk * (TX * TY) + col) * PCMAX + b;
    double s = 0.0;
    for (int k = 0; k < nchunk; ++k) s += p[(size_t)k * TX * TY * PCMAX];
    grid[idx] = s;
}

}  // namespace sog

namespace sog {

// Psi [Pc][Ilx][Ily] -> PsiT [Ilx][Ily][PCMAX] (layer fastest, zero padded) for the gather.
static __global__ void k_long_transpose(const double* __restrict__ psi, double* __restrict__ psiT, int Ilx, int Ily,
                                        int Pc, int PCMAX) {
    int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= Ilx * Ily * PCMAX) return;
    int a = idx % PCMAX, g = idx / PCMAX;
    psiT[idx] = a < Pc ? psi[(size_t)a * Ilx * Ily + g] : 0.0;
}

// S12 v2: interpolation back to the particles.  One thread per particle; the (small) proxy
// field is read from shared memory (or L1/L2 for big grids) with all PCMAX layers of a grid
// column contiguous, so a column costs PCMAX/2 128-bit loads for 2*PCMAX FMAs.
template <int P, int PCMAX>
__global__ void __launch_bounds__(128) k_long_gather2(LongArgs a, const double* __restrict__ psiT, d4* __restrict__ out,
                                                      double gamma_x, double gamma_y, int SMEM) {
    extern __shared__ double sm[];
    const int Pc = a.Pc;
    double* sC = sm;                                   // [Pc*Pc]
    double* sP = sm + PCMAX * PCMAX;                   // [Ilx*Ily*PCMAX]
    for (int k = threadIdx.x; k < Pc * Pc; k += blockDim.x) sC[k] = a.C[k];
    if (SMEM) {
        const int n = a.Ilx * a.Ily * PCMAX;
        const double2* s2 = reinterpret_cast<const double2*>(psiT);
        double2* d2 = reinterpret_cast<double2*>(sP);
        for (int k = threadIdx.x; k < n / 2; k += blockDim.x) d2[k] = s2[k];
    }
    __syncthreads();
    const double* P_ = SMEM ? sP : psiT;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.N) return;
    constexpr int p = (P - 1) / 2;
    d4 r = ld_d4(&a.pos[i]);
    const int gx0 = stencil_g0(r.x, a.hx, a.hpx), gy0 = stencil_g0(r.y, a.hy, a.hpy);
    double wx[P], wy[P], dwx[P], dwy[P];
    window_weights_rec<P, true>(r.x, gx0, a.hx, a.halfx, a.invH2Sx, gamma_x, wx, dwx);
    window_weights_rec<P, true>(r.y, gy0, a.hy, a.halfy, a.invH2Sy, gamma_y, wy, dwy);
    // Chebyshev T_n, T_n' at x = 2z/Lz, then L_b, L_b' (zero beyond Pc)
    const double x = r.z * a.two_over_Lz;
    double L[PCMAX], dL[PCMAX];
    {
        double T[PCMAX], dT[PCMAX];
        T[0] = 1.0; dT[0] = 0.0; T[1] = x; dT[1] = 1.0;
#pragma unroll
        for (int n = 1; n + 1 < PCMAX; ++n) {
            T[n + 1] = 2.0 * x * T[n] - T[n - 1];
            dT[n + 1] = 2.0 * T[n] + 2.0 * x * dT[n] - dT[n - 1];
        }
#pragma unroll
        for (int b = 0; b < PCMAX; ++b) {
            double l = 0.0, dl = 0.0;
            if (b < Pc) {
                const double* c = sC + b * Pc;
#pragma unroll
                for (int n = 0; n < PCMAX; ++n)
                    if (n < Pc) { l = fma(c[n], T[n], l); dl = fma(c[n], dT[n], dl); }
            }
            L[b] = l; dL[b] = dl;
        }
    }
    double phi = 0, gx = 0, gy = 0, gz = 0;
#pragma unroll 1
    for (int u = 0; u < P; ++u) {
        int ix = gx0 - p + u;
        ix += ix < 0 ? a.Ilx : 0; ix -= ix >= a.Ilx ? a.Ilx : 0;
        double px = 0, pdy = 0, pdz = 0;
#pragma unroll
        for (int v = 0; v < P; ++v) {
            int iy = gy0 - p + v;
            iy += iy < 0 ? a.Ily : 0; iy -= iy >= a.Ily ? a.Ily : 0;
            const double2* col = reinterpret_cast<const double2*>(P_ + ((size_t)ix * a.Ily + iy) * PCMAX);
            double t0 = 0, t1 = 0;
#pragma unroll
            for (int b = 0; b < PCMAX; b += 2) {
                double2 g = col[b / 2];
                t0 = fma(L[b], g.x, t0); t0 = fma(L[b + 1], g.y, t0);
                t1 = fma(dL[b], g.x, t1); t1 = fma(dL[b + 1], g.y, t1);
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
