// Long-range Fourier-Chebyshev solver, two-sided proxy form (Algorithm 2; R9):
//   S8  anterpolation  S_b[g] = sum_j q_j L_b(z_j) W(x_g-x_j)_* W(y_g-y_j)_*
//   S10 scaling        S'_a(k) = sum_b K_ab(k) S_b(k)                 (K from P:907/P:533, R10)
//   S12 interpolation  phi_i = h_x h_y sum_g W W sum_a L_a(z_i) Psi_a[g]   (Eq. eq::SOGLong)
// L_b(x) = sum_n C[b][n] T_n(x), x = 2 z / L_z, at first-kind Chebyshev nodes (App. A.2).
//
// B200 form: the kernels work in the Chebyshev T basis instead of the Lagrange basis.  The
// spread accumulates S~_n[g] = sum_j q_j T_n(z_j) W W (so S_b = sum_n C[b][n] S~_n), the
// scaling applies K~(k) = C^T K(k) C (plan time, R9), and the gather evaluates
// Psi~_m[g] = sum_a C[a][m] Psi_a[g] as phi = h_x h_y sum_g W W sum_m T_m(z) Psi~_m[g]:
// the same linear maps, no P x P Lagrange evaluation per particle.
// Proxy grids: [Pc][Ilx][Ily] real (T-basis layers), spectra [Pc][Ilx][Ily/2+1].
#pragma once
#include <cuComplex.h>
#include <type_traits>
#include "kernels_common.cuh"

namespace sog {

struct LongArgs {
    const d4* pos;
    int N;
    int Ilx, Ily, Pc, Pl;
    double hx, hy, halfx, halfy, hpx, hpy, invH2Sx, invH2Sy;
    double two_over_Lz;
    double A;                 // h_x h_y
    const double* C;          // [Pc][Pc] Chebyshev -> Lagrange
    int kb;                   // 1: Kaiser-Bessel window (R6-KB), table kt
    KBTab kt;
};

// x or y weights of the long window at the Pl points g0-p..g0+p: Gaussian recurrence or the
// KB polynomials (dW/dx = dW/du / h)
template <int P, bool GRAD>
__device__ __forceinline__ void long_weights(const LongArgs& a, double x, int g0, double h, double half,
                                             double invH2S, double gamma, double* W, double* dW) {
    if (a.kb) {
        if constexpr (P <= KB_PMAX) kb_weights<P, GRAD>(kb_offset(x, h, half, g0), a.kt, W, dW);
        if (GRAD) {
            const double ih = 1.0 / h;
#pragma unroll
            for (int j = 0; j < P; ++j) dW[j] *= ih;
        }
    } else {
        window_weights_rec<P, GRAD>(x, g0, h, half, invH2S, gamma, W, dW);
    }
}

// S10: one thread per (half mode, a).
template <typename C = cuDoubleComplex>
__global__ void k_long_scale(const C* __restrict__ in, C* __restrict__ out, const double* __restrict__ K, int nmode,
                             int Pc) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nmode * Pc) return;
    int mode = t / Pc, aa = t % Pc;
    const double* Km = K + ((size_t)mode * Pc + aa) * Pc;
    double re = 0, im = 0;
    for (int b = 0; b < Pc; ++b) {
        const C v = in[(size_t)b * nmode + mode];
        re = fma(Km[b], (double)v.x, re);
        im = fma(Km[b], (double)v.y, im);
    }
    C o;
    o.x = re;
    o.y = im;
    out[(size_t)aa * nmode + mode] = o;
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
    int ncy, ncz;
    double cell_w, cell_wy;  // Lx / ncx, Ly / ncy
    double Lx, Ly;
    double* grid;            // nchunk == 1: tiles own their columns, written directly (no reduce)
    double gamma_x, gamma_y; // window recurrence constants exp(-2 a h^2)
    double* part;
};

constexpr int LB = 64;       // particles per staged batch

// particle index ranges reaching the tile at (X0, Y0): the near cells whose (x, y) extent overlaps
// the tile's stencil-centre box, one contiguous sorted range per (x column, y run) of cells (all z),
// at most LT_MAXR; beyond that whole x slabs (all y).  One thread; returns the range count.
constexpr int LT_MAXR = 64;
__device__ __forceinline__ int tile_ranges(const LongTileArgs& t, int X0, int Y0, int p, int* sRb, int* sRp) {
    const LongArgs& a = t.a;
    int nr = 0, tot = 0;
    auto add = [&](int b, int e) {
        if (e > b) { sRb[nr] = b; sRp[nr] = tot; tot += e - b; ++nr; }
    };
    if (t.full_range) {
        add(0, a.N);
    } else {
        // stencil centres gx0 in [X0 - p, X0 + TX - 1 + p] <=> x in [xlo, xhi); same in y
        const double xlo = ((X0 - p) - 0.5 - 0.5 * a.Ilx) * a.hx, xhi = ((X0 + t.TX - 1 + p) + 0.5 - 0.5 * a.Ilx) * a.hx;
        const double ylo = ((Y0 - p) - 0.5 - 0.5 * a.Ily) * a.hy, yhi = ((Y0 + t.TY - 1 + p) + 0.5 - 0.5 * a.Ily) * a.hy;
        int c0 = (int)floor((xlo + 0.5 * t.Lx) / t.cell_w) - 1, c1 = (int)floor((xhi + 0.5 * t.Lx) / t.cell_w) + 1;
        const int d0 = (int)floor((ylo + 0.5 * t.Ly) / t.cell_wy) - 1, d1 = (int)floor((yhi + 0.5 * t.Ly) / t.cell_wy) + 1;
        if (c1 - c0 + 1 >= t.ncx) { c0 = 0; c1 = t.ncx - 1; }
        const bool ally = d1 - d0 + 1 >= t.ncy;
        const int nxr = c1 - c0 + 1, nyr = ally ? 1 : (d0 < 0 || d1 >= t.ncy ? 2 : 1);
        if (nxr * nyr > LT_MAXR - 2 || ally) {
            // whole x slabs: [c0, c1] split at the periodic seam
            if (c0 < 0) { add(t.start[(c0 + t.ncx) * t.cells_per_x], a.N); c0 = 0; }
            if (c1 >= t.ncx) { add(0, t.start[(c1 - t.ncx + 1) * t.cells_per_x]); c1 = t.ncx - 1; }
            add(t.start[c0 * t.cells_per_x], t.start[(c1 + 1) * t.cells_per_x]);
        } else {
            for (int c = c0; c <= c1; ++c) {
                const int cc = c < 0 ? c + t.ncx : (c >= t.ncx ? c - t.ncx : c);
                const int base = cc * t.ncy;
                if (d0 < 0) {
                    add(t.start[(base + d0 + t.ncy) * t.ncz], t.start[(base + t.ncy) * t.ncz]);
                    add(t.start[base * t.ncz], t.start[(base + d1 + 1) * t.ncz]);
                } else if (d1 >= t.ncy) {
                    add(t.start[(base + d0) * t.ncz], t.start[(base + t.ncy) * t.ncz]);
                    add(t.start[base * t.ncz], t.start[(base + d1 - t.ncy + 1) * t.ncz]);
                } else {
                    add(t.start[(base + d0) * t.ncz], t.start[(base + d1 + 1) * t.ncz]);
                }
            }
        }
    }
    sRp[nr] = tot;
    return nr;
}

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
    const int tid = threadIdx.x;
    __shared__ int sRb[LT_MAXR], sRp[LT_MAXR + 1], sNR;
    if (tid == 0) sNR = tile_ranges(t, X0, Y0, p, sRb, sRp);
    __syncthreads();
    const int nr = sNR, ntot = sRp[nr];
    const int per = (ntot + t.nchunk - 1) / t.nchunk;
    const int jb = min(ntot, chunk * per), je = min(ntot, jb + per);
    // my column
    const int cx = X0 + tid / t.TY, cy = Y0 + tid % t.TY;
    const bool own = tid < t.TX * t.TY && cx < a.Ilx && cy < a.Ily;
    double acc[PCMAX];
#pragma unroll
    for (int b = 0; b < PCMAX; ++b) acc[b] = 0.0;
    __syncthreads();
    __shared__ int sCnt[2];
    for (int base = jb; base < je; base += LB) {
        const int nbr = min(LB, je - base);
        // stage only the particles whose stencil meets this tile (ballot compaction, stream order)
        bool rel = false;
        d4 r{0.0, 0.0, 0.0, 0.0};
        int gx0 = 0, gy0 = 0;
        if (tid < nbr) {
            const int k = base + tid;
            int e = 0;
            while (e + 1 < nr && sRp[e + 1] <= k) ++e;
            const int j = sRb[e] + (k - sRp[e]);
            r = ld_d4(&a.pos[j]);
            gx0 = stencil_g0(r.x, a.hx, a.hpx);
            gy0 = stencil_g0(r.y, a.hy, a.hpy);
            // stencil [s, s + P) meets tile [X0, X0 + TX) (mod I) <=> d = (X0 - s) mod I < P or > I - TX
            int dx = (X0 - (gx0 - p)) % a.Ilx, dy = (Y0 - (gy0 - p)) % a.Ily;
            dx += dx < 0 ? a.Ilx : 0;
            dy += dy < 0 ? a.Ily : 0;
            rel = (dx < P || dx > a.Ilx - t.TX) && (dy < P || dy > a.Ily - t.TY);
        }
        unsigned bal = 0;
        if (tid < LB) {
            bal = __ballot_sync(0xffffffffu, rel);
            if ((tid & 31) == 0) sCnt[tid >> 5] = __popc(bal);
        }
        __syncthreads();
        const int nb = sCnt[0] + sCnt[1];
        if (rel) {
            const int slot = (tid >= 32 ? sCnt[0] : 0) + __popc(bal & ((1u << (tid & 31)) - 1));
            double wx[P], wy[P];
            long_weights<P, false>(a, r.x, gx0, a.hx, a.halfx, a.invH2Sx, t.gamma_x, wx, nullptr);
            long_weights<P, false>(a, r.y, gy0, a.hy, a.halfy, a.invH2Sy, t.gamma_y, wy, nullptr);
#pragma unroll
            for (int u = 0; u < P; ++u) { sW[slot * 2 * P + u] = wx[u]; sW[slot * 2 * P + P + u] = wy[u]; }
            sQ[slot] = r.w;
            sG[2 * slot] = gx0 - p;
            sG[2 * slot + 1] = gy0 - p;
            // T basis: the layer coefficients are T_n(z_j) (S~_n), zero-padded to PCMAX
            double* L = sL + slot * PCMAX;
            const double x = r.z * a.two_over_Lz;
            double tm = 1.0, tc = x;
            L[0] = 1.0;
            if (Pc > 1) L[1] = x;
            for (int n = 2; n < Pc; ++n) {
                const double tn = 2.0 * x * tc - tm;
                L[n] = tn;
                tm = tc; tc = tn;
            }
            for (int n = Pc; n < PCMAX; ++n) L[n] = 0.0;
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
        if (t.nchunk == 1) {
            const size_t G = (size_t)a.Ilx * a.Ily, g = (size_t)cx * a.Ily + cy;
#pragma unroll
            for (int b = 0; b < PCMAX; ++b)
                if (b < Pc) t.grid[b * G + g] = acc[b];
        } else {
            double* o = t.part + (((size_t)tile * t.nchunk + chunk) * (t.TX * t.TY) + tid) * PCMAX;
#pragma unroll
            for (int b = 0; b < PCMAX; ++b) o[b] = acc[b];
        }
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
    double* sP = sm + PCMAX * PCMAX;                   // [Ilx*Ily*PCMAX]
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
    long_weights<P, true>(a, r.x, gx0, a.hx, a.halfx, a.invH2Sx, gamma_x, wx, dwx);
    long_weights<P, true>(a, r.y, gy0, a.hy, a.halfy, a.invH2Sy, gamma_y, wy, dwy);
    // Chebyshev T_n, T_n' at x = 2z/Lz (zero beyond Pc): the T-basis field Psi~ (see top)
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
            L[b] = b < Pc ? T[b] : 0.0;
            dL[b] = b < Pc ? dT[b] : 0.0;
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


// ---------------------------------------------------------------------------------------
// Small long grids (Ilx <= 32, Ily <= 32, Ilx*Ily <= 256: every particle reaches most of the
// grid).  S8 as a register-tiled product: a CTA keeps a private copy of the whole grid
// S~[n][cx][cy] in registers (thread tile: 1 cx x 4 cy x 6 layers) and streams a slice of the
// particles through shared memory as rotated, zero-padded weight rows
//   Rx_j[cx] = q_j W(x_g - x_j) (stencil points only), Ry_j[cy], T_n(z_j);
// a(cx,cy) = Rx[cx] Ry[cy] and S~ += a T: 24 FMAs per 4 DMULs and 6 shared loads.
// Partials [block][n][cx][cy] are summed in a fixed order by k_long_sum (deterministic).
constexpr int LG_KB = 64, LG_LT = 6, LG_RX = 32, LG_RY = 32;

template <int PCP, typename T = double>
__global__ void __launch_bounds__(256, 2) k_long_spread_gemm(LongArgs a, const int4* __restrict__ g0, double gamma_x,
                                                             double gamma_y, int per, T* __restrict__ part) {
    constexpr int NLG = PCP / LG_LT;
    // double-buffered rows: [2][LG_KB][RXP + RYP + PCP], RXP = Ilx, RYP = Ily rounded up to 4
    extern __shared__ __align__(16) unsigned char smraw[];
    T* sm = reinterpret_cast<T*>(smraw);
    using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
    const int RXP = a.Ilx, RYP = (a.Ily + 3) & ~3, RW = ((RXP + RYP + PCP) + 1) & ~1;
    const int tid = threadIdx.x;
    const int ncy4 = (a.Ily + 3) / 4;
    const int lg = tid % NLG, cg = tid / NLG;
    const int cx = cg / ncy4, cy0 = 4 * (cg % ncy4);
    const bool own = cx < a.Ilx;
    T acc[4][LG_LT];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int l = 0; l < LG_LT; ++l) acc[i][l] = 0.0;
    const int j0 = blockIdx.x * per, j1 = min(a.N, j0 + per);
    const int P = a.Pl;
    // threads per staged particle: 4 with >= 256 threads (Rx row, Ry row, T row, idle), else 2
    // (Rx and T rows, Ry row)
    const bool four = blockDim.x >= 4 * LG_KB;
    auto stage = [&](int base, int buf) {
        const int t = four ? tid >> 2 : tid >> 1, role = four ? tid & 3 : tid & 1;
        if (t >= LG_KB) return;   // blockDim >= 2 * LG_KB = 128
        const bool doX = role == 0, doY = role == 1, doT = four ? role == 2 : role == 0;
        T* row = sm + ((size_t)buf * LG_KB + t) * RW;
        T* rx = row;
        T* ry = row + RXP;
        T* tt = row + RXP + RYP;
        if (doX)
            for (int c = 0; c < RXP; ++c) rx[c] = T(0);
        if (doT)
            for (int n = 0; n < PCP; ++n) tt[n] = T(0);
        if (doY)
            for (int c = 0; c < RYP; ++c) ry[c] = T(0);
        const int j = base + t;
        if (j >= j1 || !(doX || doY || doT)) return;
        const d4 r = ld_d4(&a.pos[j]);
        const unsigned ow = (unsigned)g0[j].w;
        if (doT) {
            const double x = r.z * a.two_over_Lz;
            double tm = 1.0, tc = x;
            tt[0] = T(1);
            if (a.Pc > 1) tt[1] = T(x);
            for (int n = 2; n < a.Pc; ++n) {
                const double tn = 2.0 * x * tc - tm;
                tt[n] = T(tn);
                tm = tc; tc = tn;
            }
        }
        if (doX) {
            const int sx = (int)(ow & 0xffffu) - 32768 - (P - 1) / 2;
            int c = sx < 0 ? sx + a.Ilx : sx;
            if (a.kb) {
                const double qw = r.w;
                const int Il = a.Ilx;
                auto put = [&](int u, double w, double) {
                    const int cc = c + u;
                    rx[cc >= Il ? cc - Il : cc] = T(qw * w);
                };
                kb_emit_rt<false>(P, kb_offset(r.x, a.hx, a.halfx, sx + (P - 1) / 2), a.kt, put);
            } else {
                const double d0 = ((double)sx - a.halfx) * a.hx - r.x;
                double w = exp(-a.invH2Sx * d0 * d0), q = exp(-a.invH2Sx * a.hx * (2.0 * d0 + a.hx));
                for (int u = 0; u < P; ++u) {
                    rx[c] = T(r.w * w);
                    w *= q; q *= gamma_x;
                    c = c + 1 == a.Ilx ? 0 : c + 1;
                }
            }
        } else if (doY) {
            const int sy = (int)(ow >> 16) - 32768 - (P - 1) / 2;
            int c = sy < 0 ? sy + a.Ily : sy;
            if (a.kb) {
                const int Il = a.Ily;
                auto put = [&](int v, double w, double) {
                    const int cc = c + v;
                    ry[cc >= Il ? cc - Il : cc] = T(w);
                };
                kb_emit_rt<false>(P, kb_offset(r.y, a.hy, a.halfy, sy + (P - 1) / 2), a.kt, put);
            } else {
                const double d0 = ((double)sy - a.halfy) * a.hy - r.y;
                double w = exp(-a.invH2Sy * d0 * d0), q = exp(-a.invH2Sy * a.hy * (2.0 * d0 + a.hy));
                for (int v = 0; v < P; ++v) {
                    ry[c] = T(w);
                    w *= q; q *= gamma_y;
                    c = c + 1 == a.Ily ? 0 : c + 1;
                }
            }
        }
    };
    if (j0 < j1) stage(j0, 0);
    __syncthreads();
    int buf = 0;
    for (int base = j0; base < j1; base += LG_KB, buf ^= 1) {
        if (base + LG_KB < j1) stage(base + LG_KB, buf ^ 1);    // next batch while this one computes
        const int nb = min(LG_KB, j1 - base);
        if (own) {
            const T* rows = sm + (size_t)buf * LG_KB * RW;
#pragma unroll 2
            for (int t = 0; t < nb; ++t) {
                const T* row = rows + (size_t)t * RW;
                const T rx = row[cx];
                const V2 y01 = *reinterpret_cast<const V2*>(row + RXP + cy0);
                const V2 y23 = *reinterpret_cast<const V2*>(row + RXP + cy0 + 2);
                T tl[LG_LT];
#pragma unroll
                for (int l = 0; l < LG_LT; l += 2) {
                    const V2 v = *reinterpret_cast<const V2*>(row + RXP + RYP + lg * LG_LT + l);
                    tl[l] = v.x; tl[l + 1] = v.y;
                }
                const T av[4] = {rx * y01.x, rx * y01.y, rx * y23.x, rx * y23.y};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int l = 0; l < LG_LT; ++l) acc[i][l] = fma(av[i], tl[l], acc[i][l]);
            }
        }
        __syncthreads();
    }
    if (own) {
        const size_t G = (size_t)a.Ilx * a.Ily;
        T* o = part + (size_t)blockIdx.x * PCP * G;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int l = 0; l < LG_LT; ++l) {
                const int cy = cy0 + i, n = lg * LG_LT + l;
                if (cy < a.Ily) o[(size_t)n * G + (size_t)cx * a.Ily + cy] = acc[i][l];
            }
    }
}

// S8 on the FP64 tensor path (small long grids, fp64): the anterpolation of a CTA's particle range
// is the product C[n][g] = sum_j T_n(z_j) B_j[g], B_j[g] = q_j Wx_j(cx) Wy_j(cy) (g = cx Ily + cy,
// dense over the Ilx x Ily grid, zero off the stencil) -- a GEMM with K = particles, done with
// mma.sync m8n8k4 f64 (DMMA: the same FP64 pipe as DFMA, 256 FMAs per warp instruction, operands
// straight from registers).  Warp w owns all MT n-tiles (8 layers each) x NTW column tiles (8 columns
// each); per k-step of 4 particles a thread loads one A value per n-tile (T row) and forms one B value
// per column tile from the staged q Wx and Wy rows.  Rows [T (8 MT) | q Wx (Ilx) | Wy (Ily)] of LS_KB
// particles are staged (double-buffered) while the previous batch is multiplied.  Partials
// [block][n][g] as k_long_spread_gemm writes them (summed in a fixed order by k_long_sum).
constexpr int LS_KB = 32;

template <int MT, int NTW>
__global__ void __launch_bounds__(384) k_long_spread_mma(LongArgs a, const int4* __restrict__ g0, double gamma_x,
                                                         double gamma_y, int per, int PCP, double* __restrict__ part) {
    extern __shared__ __align__(16) unsigned char smraw[];
    double* sm = reinterpret_cast<double*>(smraw);
    const int TW = 8 * MT, RW = (TW + a.Ilx + a.Ily + 1) & ~1;
    const int G = a.Ilx * a.Ily, NT = (G + 7) / 8;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const int j0 = blockIdx.x * per, j1 = min(a.N, j0 + per);
    const int P = a.Pl;
    // this thread's B columns (one per column tile): staged row offsets of Wx(cx), Wy(cy)
    int offx[NTW], offy[NTW];
    bool colv[NTW];
#pragma unroll
    for (int t = 0; t < NTW; ++t) {
        const int col = 8 * (warp * NTW + t) + gid;
        colv[t] = col < G;
        const int cx = colv[t] ? col / a.Ily : 0, cy = colv[t] ? col - cx * a.Ily : 0;
        offx[t] = TW + cx;
        offy[t] = TW + a.Ilx + cy;
    }
    double c[MT][NTW][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int t = 0; t < NTW; ++t) c[m][t][0] = c[m][t][1] = 0.0;
    // stage particles [base, base + LS_KB): thread = (particle, role T / X / Y)
    auto stage = [&](int base, int buf) {
        for (int e = tid; e < 3 * LS_KB; e += blockDim.x) {
            const int t = e / 3, role = e - 3 * t;
            double* row = sm + ((size_t)buf * LS_KB + t) * RW;
            const int j = base + t;
            if (role == 0) {
                if (j >= j1) {
                    for (int n = 0; n < TW; ++n) row[n] = 0.0;
                    continue;
                }
                const double x = a.pos[j].z * a.two_over_Lz;
                double tm = 1.0, tc = x;
                row[0] = 1.0;
                for (int n = 1; n < TW; ++n) {
                    row[n] = n < a.Pc ? tc : 0.0;
                    const double tn = 2.0 * x * tc - tm;
                    tm = tc;
                    tc = tn;
                }
            } else {
                const bool X = role == 1;
                double* r = row + TW + (X ? 0 : a.Ilx);
                const int Il = X ? a.Ilx : a.Ily;
                for (int cc = 0; cc < Il; ++cc) r[cc] = 0.0;
                if (j >= j1) continue;
                const d4 pj = ld_d4(&a.pos[j]);
                const unsigned ow = (unsigned)g0[j].w;
                const int s0 = (int)(X ? (ow & 0xffffu) : (ow >> 16)) - 32768 - (P - 1) / 2;
                int cc = s0 < 0 ? s0 + Il : s0;
                const double xx = X ? pj.x : pj.y, hh = X ? a.hx : a.hy, hf = X ? a.halfx : a.halfy;
                const double sc = X ? pj.w : 1.0;
                if (a.kb) {
                    auto put = [&](int u, double w, double) {
                        const int c2 = cc + u;
                        r[c2 >= Il ? c2 - Il : c2] = sc * w;
                    };
                    kb_emit_rt<false>(P, kb_offset(xx, hh, hf, s0 + (P - 1) / 2), a.kt, put);
                } else {
                    const double al = X ? a.invH2Sx : a.invH2Sy, gm = X ? gamma_x : gamma_y;
                    const double d0 = ((double)s0 - hf) * hh - xx;
                    double w = exp(-al * d0 * d0), q = exp(-al * hh * (2.0 * d0 + hh));
                    for (int u = 0; u < P; ++u) {
                        r[cc] = sc * w;
                        w *= q;
                        q *= gm;
                        cc = cc + 1 == Il ? 0 : cc + 1;
                    }
                }
            }
        }
    };
    if (j0 < j1) stage(j0, 0);
    __syncthreads();
    const bool active = warp * NTW < NT;
    int buf = 0;
    for (int base = j0; base < j1; base += LS_KB, buf ^= 1) {
        if (base + LS_KB < j1) stage(base + LS_KB, buf ^ 1);   // next batch while this one multiplies
        if (active) {
            const double* rows = sm + (size_t)buf * LS_KB * RW;
#pragma unroll 2
            for (int kk = 0; kk < LS_KB / 4; ++kk) {
                const double* rw = rows + (size_t)(4 * kk + tig) * RW;   // particle of this thread's k slot
                double av[MT], bv[NTW];
#pragma unroll
                for (int m = 0; m < MT; ++m) av[m] = rw[8 * m + gid];
#pragma unroll
                for (int t = 0; t < NTW; ++t) bv[t] = colv[t] ? rw[offx[t]] * rw[offy[t]] : 0.0;
#pragma unroll
                for (int m = 0; m < MT; ++m)
#pragma unroll
                    for (int t = 0; t < NTW; ++t) dmma_884(c[m][t], av[m], bv[t]);
            }
        }
        __syncthreads();
    }
    if (active) {
        double* o = part + (size_t)blockIdx.x * PCP * G;
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
            for (int t = 0; t < NTW; ++t)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int n = 8 * m + gid, col = 8 * (warp * NTW + t) + 2 * tig + h;
                    if (n < a.Pc && col < G) o[(size_t)n * G + col] = c[m][t][h];
                }
    }
}

// grid[n][g] = sum over blocks (fixed order) of part[block][n][g], n < Pc
template <typename T>
__global__ void k_long_sum(const T* __restrict__ part, T* __restrict__ grid, int G, int Pc, int PCP,
                                  int nblk) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= G * Pc) return;
    const T* p = part + idx;
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += p[(size_t)b * PCP * G];
    grid[idx] = T(s);
}

// S8 v3 for wide long grids: the register-tiled product of k_long_spread_gemm restricted to one
// TX x TY column tile.  The tile's candidates are its near-cell runs (tile_ranges), staged 64 at a
// time as rows [Rx (TX) | Ry (TYP) | T_n (PCP)] holding only the tile's columns (zeros elsewhere)
// plus a relevance flag (rows whose stencil misses the tile are skipped, uniformly per block);
// thread = (1 cx, 4 cy, 6 layers) register accumulators.  Tiles own their columns: one chunk per
// tile writes the grid directly, several write partials summed in a fixed order.
template <int PCP>
__global__ void __launch_bounds__(256, 2) k_long_spread_tgemm(LongTileArgs t) {
    constexpr int NLG = PCP / LG_LT;
    extern __shared__ __align__(16) unsigned char smraw[];
    double* sm = reinterpret_cast<double*>(smraw);
    __shared__ unsigned char sRel[2][LG_KB];
    __shared__ int sRb[LT_MAXR], sRp[LT_MAXR + 1], sNR;
    const LongArgs& a = t.a;
    const int P = a.Pl, p = (P - 1) / 2;
    const int tile = blockIdx.y, chunk = blockIdx.x;
    const int X0 = (tile / t.nty) * t.TX, Y0 = (tile % t.nty) * t.TY;
    const int tid = threadIdx.x;
    const int TYP = (t.TY + 3) & ~3, TYG = TYP / 4, RW = ((t.TX + TYP + PCP) + 1) & ~1;
    const int lg = tid % NLG, cg = tid / NLG;
    const int cx = cg / TYG, cy0 = 4 * (cg % TYG);
    const bool own = cx < t.TX;
    if (tid == 0) sNR = tile_ranges(t, X0, Y0, p, sRb, sRp);
    __syncthreads();
    const int nr = sNR, ntot = sRp[nr];
    const int per = (ntot + t.nchunk - 1) / t.nchunk;
    const int jb = min(ntot, chunk * per), je = min(ntot, jb + per);
    double acc[4][LG_LT];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int l = 0; l < LG_LT; ++l) acc[i][l] = 0.0;
    // staging: (particle, role) work items, role 0 -> Rx row, 1 -> Ry row, 2 -> T row + flag
    auto stage = [&](int base, int buf) {
        const int nb = min(LG_KB, je - base);
        for (int w = tid; w < 3 * nb; w += blockDim.x) {
            const int k = w / 3, role = w - 3 * k;
            const int kk = base + k;
            int e = 0;
            while (e + 1 < nr && sRp[e + 1] <= kk) ++e;
            const int j = sRb[e] + (kk - sRp[e]);
            const d4 r = ld_d4(&a.pos[j]);
            double* row = sm + ((size_t)buf * LG_KB + k) * RW;
            if (role == 2) {
                double* tt = row + t.TX + TYP;
                const double x = r.z * a.two_over_Lz;
                double tm = 1.0, tc = x;
                tt[0] = 1.0;
                if (PCP > 1) tt[1] = x;
                for (int n = 2; n < PCP; ++n) {
                    const double tn = 2.0 * x * tc - tm;
                    tt[n] = tn;
                    tm = tc; tc = tn;
                }
                const int gx0 = stencil_g0(r.x, a.hx, a.hpx), gy0 = stencil_g0(r.y, a.hy, a.hpy);
                int dx = (X0 - (gx0 - p)) % a.Ilx, dy = (Y0 - (gy0 - p)) % a.Ily;
                dx += dx < 0 ? a.Ilx : 0;
                dy += dy < 0 ? a.Ily : 0;
                sRel[buf][k] = (dx < P || dx > a.Ilx - t.TX) && (dy < P || dy > a.Ily - t.TY);
            } else {
                const bool isx = role == 0;
                const int I = isx ? a.Ilx : a.Ily, T0 = isx ? X0 : Y0, TW = isx ? t.TX : TYP;
                const int TV = isx ? t.TX : t.TY;           // valid columns of the row
                const double xc = isx ? r.x : r.y, hh = isx ? a.hx : a.hy, hf = isx ? a.halfx : a.halfy;
                double* rw = isx ? row : row + t.TX;
                for (int c = 0; c < TW; ++c) rw[c] = 0.0;
                const int g0 = stencil_g0(xc, hh, isx ? a.hpx : a.hpy), s0 = g0 - p;
                const double qw = isx ? r.w : 1.0;
                int c = (s0 - T0) % I;
                c += c < 0 ? I : 0;
                auto put = [&](int, double w, double) {
                    if (c < TV) rw[c] = qw * w;
                    c = c + 1 == I ? 0 : c + 1;
                };
                if (a.kb) {
                    kb_emit_rt<false>(P, kb_offset(xc, hh, hf, g0), a.kt, put);
                } else {
                    const double ih = isx ? a.invH2Sx : a.invH2Sy, gam = isx ? t.gamma_x : t.gamma_y;
                    const double d0 = ((double)s0 - hf) * hh - xc;
                    double w = exp(-ih * d0 * d0), q = exp(-ih * hh * (2.0 * d0 + hh));
                    for (int u = 0; u < P; ++u) {
                        put(u, w, 0.0);
                        w *= q; q *= gam;
                    }
                }
            }
        }
    };
    if (jb < je) stage(jb, 0);
    __syncthreads();
    int buf = 0;
    for (int base = jb; base < je; base += LG_KB, buf ^= 1) {
        if (base + LG_KB < je) stage(base + LG_KB, buf ^ 1);
        const int nb = min(LG_KB, je - base);
        if (own) {
            const double* rows = sm + (size_t)buf * LG_KB * RW;
            for (int k = 0; k < nb; ++k) {
                if (!sRel[buf][k]) continue;                   // uniform across the block
                const double* row = rows + (size_t)k * RW;
                const double rx = row[cx];
                const double2 y01 = *reinterpret_cast<const double2*>(row + t.TX + cy0);
                const double2 y23 = *reinterpret_cast<const double2*>(row + t.TX + cy0 + 2);
                double tl[LG_LT];
#pragma unroll
                for (int l = 0; l < LG_LT; l += 2) {
                    const double2 v = *reinterpret_cast<const double2*>(row + t.TX + TYP + lg * LG_LT + l);
                    tl[l] = v.x; tl[l + 1] = v.y;
                }
                const double av[4] = {rx * y01.x, rx * y01.y, rx * y23.x, rx * y23.y};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int l = 0; l < LG_LT; ++l) acc[i][l] = fma(av[i], tl[l], acc[i][l]);
            }
        }
        __syncthreads();
    }
    if (own) {
        const size_t G = (size_t)a.Ilx * a.Ily;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int cy = cy0 + i, gx = X0 + cx, gy = Y0 + cy;
            if (cy >= t.TY || gx >= a.Ilx || gy >= a.Ily) continue;
#pragma unroll
            for (int l = 0; l < LG_LT; ++l) {
                const int n = lg * LG_LT + l;
                if (n >= a.Pc) continue;
                if (t.nchunk == 1)
                    t.grid[n * G + (size_t)gx * a.Ily + gy] = acc[i][l];
                else
                    t.part[(((size_t)tile * t.nchunk + chunk) * PCP + n) * (t.TX * t.TY) + cx * t.TY + cy] = acc[i][l];
            }
        }
    }
}

// grid[n][g] = sum over the chunks of a tile (fixed order) of k_long_spread_tgemm's partials
static __global__ void k_long_treduce(const double* __restrict__ part, double* __restrict__ grid, int Ilx, int Ily,
                                      int Pc, int PCP, int TX, int TY, int nty, int nchunk) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= Ilx * Ily * Pc) return;
    const int n = idx / (Ilx * Ily), g = idx % (Ilx * Ily);
    const int gx = g / Ily, gy = g % Ily;
    const int tile = (gx / TX) * nty + gy / TY, col = (gx % TX) * TY + gy % TY;
    double s = 0.0;
    for (int c = 0; c < nchunk; ++c) s += part[(((size_t)tile * nchunk + c) * PCP + n) * (TX * TY) + col];
    grid[idx] = s;
}

// S12 for small long grids: one thread per particle, the whole T-basis field Psi~ in shared
// memory as [cx][cy][PCP] and read with broadcast 128-bit loads (every thread walks the
// columns in the same order).  Per column: V = sum_m T_m Psi~_m, V' = sum_m T'_m Psi~_m
// (2 PCP FMAs) and 4 products with the rotated weights.  Rx / dRx rows live in shared
// memory (dynamic cx), Ry / dRy in registers (static cy < NCY).
template <int PCP, int NCY, typename T = double>
__global__ void __launch_bounds__(128, 4) k_long_gather_bc(LongArgs a, const int4* __restrict__ g0,
                                                        const T* __restrict__ psi, d4* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smraw[];
    T* sm = reinterpret_cast<T*>(smraw);
    using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
    const int G = a.Ilx * a.Ily;
    T* sPsi = sm;                                  // [G][PCP]
    T* sRx = sm + (size_t)G * PCP;                 // [Ilx][128]
    T* sdRx = sRx + (size_t)a.Ilx * 128;           // [Ilx][128]
    T* sRy = sdRx + (size_t)a.Ilx * 128;           // [NCY][128]
    T* sdRy = sRy + (size_t)NCY * 128;             // [NCY][128]
    for (int e = threadIdx.x; e < G * PCP; e += blockDim.x) {
        const int g = e / PCP, n = e - g * PCP;
        sPsi[e] = n < a.Pc ? psi[(size_t)n * G + g] : T(0);
    }
    const int tid = threadIdx.x;
    const int j = blockIdx.x * blockDim.x + tid;
    const bool act = j < a.N;
    const int P = a.Pl;
    T Tn[PCP], dT[PCP];
    {
        for (int c = 0; c < a.Ilx; ++c) { sRx[c * 128 + tid] = T(0); sdRx[c * 128 + tid] = T(0); }
#pragma unroll
        for (int c = 0; c < NCY; ++c) { sRy[c * 128 + tid] = T(0); sdRy[c * 128 + tid] = T(0); }
        d4 r{0.0, 0.0, 0.0, 0.0};
        int sx = 0, sy = 0;
        if (act) {
            r = ld_d4(&a.pos[j]);
            const unsigned ow = (unsigned)g0[j].w;
            sx = (int)(ow & 0xffffu) - 32768 - (P - 1) / 2;
            sy = (int)(ow >> 16) - 32768 - (P - 1) / 2;
            if (a.kb) {
                const double ux = kb_offset(r.x, a.hx, a.halfx, sx + (P - 1) / 2);
                const double uy = kb_offset(r.y, a.hy, a.halfy, sy + (P - 1) / 2);
                const double ihx = 1.0 / a.hx, ihy = 1.0 / a.hy;
                const int cx0 = sx < 0 ? sx + a.Ilx : sx, cy0 = sy < 0 ? sy + a.Ily : sy;
                const int Ilx = a.Ilx, Ily = a.Ily;
                auto putx = [&](int u, double w, double dw) {
                    const int cc = cx0 + u >= Ilx ? cx0 + u - Ilx : cx0 + u;
                    sRx[cc * 128 + tid] = T(w);
                    sdRx[cc * 128 + tid] = T(dw * ihx);
                };
                auto puty = [&](int v, double w, double dw) {
                    const int cc = cy0 + v >= Ily ? cy0 + v - Ily : cy0 + v;
                    sRy[cc * 128 + tid] = T(w);
                    sdRy[cc * 128 + tid] = T(dw * ihy);
                };
                kb_emit_rt<true>(P, ux, a.kt, putx);
                kb_emit_rt<true>(P, uy, a.kt, puty);
            } else {
            {
                const double d0 = ((double)sx - a.halfx) * a.hx - r.x;
                double w = exp(-a.invH2Sx * d0 * d0), q = exp(-a.invH2Sx * a.hx * (2.0 * d0 + a.hx));
                const double gam = exp(-2.0 * a.invH2Sx * a.hx * a.hx);
                int c = sx < 0 ? sx + a.Ilx : sx;
                for (int u = 0; u < P; ++u) {
                    sRx[c * 128 + tid] = T(w);
                    sdRx[c * 128 + tid] = T(2.0 * a.invH2Sx * (d0 + u * a.hx) * w);
                    w *= q; q *= gam;
                    c = c + 1 == a.Ilx ? 0 : c + 1;
                }
            }
            {
                const double d0 = ((double)sy - a.halfy) * a.hy - r.y;
                double w = exp(-a.invH2Sy * d0 * d0), q = exp(-a.invH2Sy * a.hy * (2.0 * d0 + a.hy));
                const double gam = exp(-2.0 * a.invH2Sy * a.hy * a.hy);
                int c = sy < 0 ? sy + a.Ily : sy;
                for (int v = 0; v < P; ++v) {
                    sRy[c * 128 + tid] = T(w);
                    sdRy[c * 128 + tid] = T(2.0 * a.invH2Sy * (d0 + v * a.hy) * w);
                    w *= q; q *= gam;
                    c = c + 1 == a.Ily ? 0 : c + 1;
                }
            }
            }
        }
        const double x = r.z * a.two_over_Lz;
        double t0 = 1.0, t1 = x, d0v = 0.0, d1v = 1.0;   // Chebyshev T_n, T_n' in fp64, stored as T
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
    T phi = 0, gx = 0, gy = 0, gz = 0;
    for (int cx = 0; cx < a.Ilx; ++cx) {
        const T rx = sRx[cx * 128 + tid], drx = sdRx[cx * 128 + tid];
        const T* col = sPsi + (size_t)cx * a.Ily * PCP;
#pragma unroll
        for (int cy = 0; cy < NCY; ++cy) {
            if (cy < a.Ily) {
                const V2* c2 = reinterpret_cast<const V2*>(col + cy * PCP);
                T v0 = 0, v1 = 0;
#pragma unroll
                for (int n = 0; n < PCP; n += 2) {
                    const V2 ps = c2[n / 2];
                    v0 = fma(Tn[n], ps.x, v0); v0 = fma(Tn[n + 1], ps.y, v0);
                    v1 = fma(dT[n], ps.x, v1); v1 = fma(dT[n + 1], ps.y, v1);
                }
                const T ry = sRy[cy * 128 + tid], dry = sdRy[cy * 128 + tid];
                const T wxy = rx * ry;
                phi = fma(wxy, v0, phi);
                gz = fma(wxy, v1, gz);
                gx = fma(drx * ry, v0, gx);
                gy = fma(rx * dry, v0, gy);
            }
        }
    }
    if (act) st_d4(&out[j], d4{a.A * double(phi), a.A * double(gx), a.A * double(gy), a.A * double(gz) * a.two_over_Lz});
}

// Debug-stage conversions back to the paper's Lagrange (proxy-node) basis:
//   S_b = sum_n C[b][n] S~_n,   Psi_a = sum_m T_m(x_a) Psi~_m  (x_a first-kind nodes).
static __global__ void k_long_to_nodes(const double* __restrict__ in, double* __restrict__ out, int G, int Pc,
                                       const double* __restrict__ M) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= G * Pc) return;
    const int b = idx / G, g = idx - b * G;
    double s = 0.0;
    for (int n = 0; n < Pc; ++n) s = fma(M[b * Pc + n], in[(size_t)n * G + g], s);
    out[idx] = s;
}

}  // namespace sog
