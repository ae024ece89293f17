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

// S7 gather: one thread per particle, separable weights (recurrence) in registers, reads
// the P^3 stencil of Psi through L1 (particles are cell-sorted, so neighbours share lines).
template <int P>
__global__ void __launch_bounds__(128, 4) k_mid_gather(MidArgs a, const double* __restrict__ psi, d4* __restrict__ out,
                                                       double gamma_x, double gamma_y, double gamma_z) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.N) return;
    constexpr int p = (P - 1) / 2;
    d4 r = ld_d4(&a.pos[i]);
    int gx0 = stencil_g0(r.x, a.hx, a.hpx), gy0 = stencil_g0(r.y, a.hy, a.hpy), gz0 = stencil_g0(r.z, a.hz, a.hpz);
    double wx[P], wy[P], wz[P], dwx[P], dwy[P], dwz[P];
    window_weights_rec<P, true>(r.x, gx0, a.hx, a.halfx, a.invH2Sx, gamma_x, wx, dwx);
    window_weights_rec<P, true>(r.y, gy0, a.hy, a.halfy, a.invH2Sy, gamma_y, wy, dwy);
    window_weights_rec<P, true>(r.z, gz0, a.hz, a.halfz, a.invH2Sz, gamma_z, wz, dwz);
    const size_t zb = (size_t)(gz0 - p);
    double phi = 0, gx = 0, gy = 0, gz = 0;
    int ix = gx0 - p;
    ix += ix < 0 ? a.Ix : 0; ix -= ix >= a.Ix ? a.Ix : 0;
    int iy0 = gy0 - p;
    iy0 += iy0 < 0 ? a.Iy : 0; iy0 -= iy0 >= a.Iy ? a.Iy : 0;
#pragma unroll 1
    for (int u = 0; u < P; ++u) {
        const double* plane = psi + (size_t)ix * a.Iy * a.Izs + zb;
        double px = 0, pdz = 0, pdy = 0;
        int iy = iy0;
#pragma unroll
        for (int v = 0; v < P; ++v) {
            const double* col = plane + (size_t)iy * a.Izs;
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
            iy = (iy + 1 == a.Iy) ? 0 : iy + 1;
        }
        phi = fma(wx[u], px, phi);
        gx = fma(dwx[u], px, gx);
        gy = fma(wx[u], pdy, gy);
        gz = fma(wx[u], pdz, gz);
        ix = (ix + 1 == a.Ix) ? 0 : ix + 1;
    }
    st_d4(&out[i], d4{a.Vh * phi, a.Vh * gx, a.Vh * gy, a.Vh * gz});
}

}  // namespace sog

namespace sog {

// ---------------------------------------------------------------------------------------
// S3 v2: output-stationary gridding without atomics.  A CTA owns a 16 x 16 x MT_Z tile of the
// mid grid; its 8 warps each own a 4 (x) x 8 (y) patch of columns, every lane one column
// with MT_Z consecutive z values in registers.  The CTA scans the near-field cells that can
// hold particles whose stencils reach the tile, compacts the hits in cell order (so the
// summation order is fixed -> deterministic), stages their separable weights in shared
// memory, and every warp whose patch a particle touches adds c = q Wx Wy (per lane) times
// Wz (broadcast) into the overlapping z registers, selected by a switch on the z-offset.
// Every grid point is written exactly once (no memset, no atomics).
constexpr int MT_X = 16, MT_Y = 16, MT_Z = 24, MT_B = 256;   // MT_B >= threads per CTA

struct MidTileArgs {
    MidArgs a;
    const int* start;           // cell start offsets
    CellGeo g;
    double gamma_x, gamma_y, gamma_z;
    int ntx, nty, ntz;
    int gz_lo, gz_hi;           // range of stencil centres gz0 any particle can have
    int Y0;                     // tile origin in y (set per CTA)
};

template <int P, int K>
__device__ __forceinline__ void zcase(double (&acc)[MT_Z], double c, const double* wz) {
    constexpr int s = K - (P - 1);     // grid z = Z0 + s + k, k = 0..P-1
#pragma unroll
    for (int k = 0; k < P; ++k) {
        if (s + k >= 0 && s + k < MT_Z) acc[s + k] = fma(c, wz[k], acc[s + k]);
    }
}

// jump table over the particle's z offset (one case per relative stencil position)
template <int P>
__device__ __forceinline__ void zdispatch(int key, double (&acc)[MT_Z], double c, const double* wz) {
#define ZC_(K) \
    case K:    \
        if constexpr (K < MT_Z + P - 1) zcase<P, K>(acc, c, wz); \
        break;
    switch (key) {
        ZC_(0)
        ZC_(1)
        ZC_(2)
        ZC_(3)
        ZC_(4)
        ZC_(5)
        ZC_(6)
        ZC_(7)
        ZC_(8)
        ZC_(9)
        ZC_(10)
        ZC_(11)
        ZC_(12)
        ZC_(13)
        ZC_(14)
        ZC_(15)
        ZC_(16)
        ZC_(17)
        ZC_(18)
        ZC_(19)
        ZC_(20)
        ZC_(21)
        ZC_(22)
        ZC_(23)
        ZC_(24)
        ZC_(25)
        ZC_(26)
        ZC_(27)
        ZC_(28)
        ZC_(29)
        ZC_(30)
        ZC_(31)
        ZC_(32)
        ZC_(33)
        ZC_(34)
        ZC_(35)
        ZC_(36)
        ZC_(37)
        ZC_(38)
        ZC_(39)
        ZC_(40)
        ZC_(41)
        ZC_(42)
        ZC_(43)
        ZC_(44)
        ZC_(45)
        ZC_(46)
        ZC_(47)
        ZC_(48)
        ZC_(49)
        ZC_(50)
        ZC_(51)
        ZC_(52)
        ZC_(53)
        ZC_(54)
        ZC_(55)
        ZC_(56)
        ZC_(57)
        ZC_(58)
        ZC_(59)
        ZC_(60)
        ZC_(61)
        ZC_(62)
        ZC_(63)
        default: break;
    }
#undef ZC_
}

// v mod n for v in (-2n, 2n) without integer division
__device__ __forceinline__ int wrapc(int v, int n) {
    v += v < 0 ? n : 0;
    v += v < 0 ? n : 0;
    v -= v >= n ? n : 0;
    v -= v >= n ? n : 0;
    return v;
}

// Stage weights of sIdx[0..nst) (offsets dxo = (ox - X0) mod Ix etc. precomputed at
// compaction), build each warp's list of particles touching its 4 x 8 column patch, and
// add them into the lanes' z registers.
template <int P>
__device__ __forceinline__ void mid_tile_batch(const MidTileArgs& t, int nst, const int* sIdx, int* sO,
                                               double* sW, unsigned char* sMask, int* sList,
                                               double (&acc)[MT_Z], int X0, int Z0, bool colok) {
    constexpr int p = (P - 1) / 2;
    constexpr int NW = 3 * P + 1;
    const MidArgs& a = t.a;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int s = tid; s < nst; s += blockDim.x) {
        d4 r = ld_d4(&a.pos[sIdx[s]]);
        const int dxo = sO[3 * s], dyo = sO[3 * s + 1];
        // unwrapped stencil centres (the weights need the particle's own periodic image)
        const int gx0 = stencil_g0(r.x, a.hx, a.hpx), gy0 = stencil_g0(r.y, a.hy, a.hpy);
        const int gz0 = stencil_g0(r.z, a.hz, a.hpz);
        double wx[P], wy[P], wz[P];
        window_weights_rec<P, false>(r.x, gx0, a.hx, a.halfx, a.invH2Sx, t.gamma_x, wx, nullptr);
        window_weights_rec<P, false>(r.y, gy0, a.hy, a.halfy, a.invH2Sy, t.gamma_y, wy, nullptr);
        window_weights_rec<P, false>(r.z, gz0, a.hz, a.halfz, a.invH2Sz, t.gamma_z, wz, nullptr);
        double* w = sW + s * NW;
#pragma unroll
        for (int k = 0; k < P; ++k) { w[k] = wx[k]; w[P + k] = wy[k]; w[2 * P + k] = wz[k]; }
        w[3 * P] = r.w;
        // which of the 8 warp patches (4 in x by 2 in y) this stencil touches
        unsigned m = 0;
#pragma unroll
        for (int wq = 0; wq < 8; ++wq) {
            const int u0 = wrapc(4 * (wq & 3) - dxo, a.Ix), v0 = wrapc(8 * (wq >> 2) - dyo, a.Iy);
            if ((u0 < P || u0 > a.Ix - 4) && (v0 < P || v0 > a.Iy - 8)) m |= 1u << wq;
        }
        sMask[s] = (unsigned char)m;
    }
    __syncthreads();
    // per-warp compaction of the particles touching this warp's patch (order preserved)
    int* myl = sList + warp * MT_B;
    int nmy = 0;
    for (int s0 = 0; s0 < nst; s0 += 32) {
        const int s = s0 + lane;
        const bool mine = s < nst && ((sMask[s] >> warp) & 1);
        const unsigned bm = __ballot_sync(0xffffffffu, mine);
        if (mine) myl[nmy + __popc(bm & ((1u << lane) - 1))] = s;
        nmy += __popc(bm);
    }
    __syncwarp();
    const int wofx = 4 * (warp & 3) + (lane & 3), wofy = 8 * (warp >> 2) + (lane >> 2);
    for (int i = 0; i < nmy; ++i) {
        const int s = myl[i];
        const double* w = sW + s * NW;
        const int u = wrapc(wofx - sO[3 * s], a.Ix), v = wrapc(wofy - sO[3 * s + 1], a.Iy);
        const double c = (colok && u < P && v < P) ? w[3 * P] * w[u] * w[P + v] : 0.0;
        zdispatch<P>(sO[3 * s + 2], acc, c, w + 2 * P);
    }
    __syncthreads();
}

template <int P>
__global__ void __launch_bounds__(256, 2) k_mid_spread_tile(MidTileArgs t, double* __restrict__ grid) {
    constexpr int p = (P - 1) / 2;
    extern __shared__ double sW[];                // [MT_B][3P+1] staged weights (dynamic)
    __shared__ int sO[MT_B * 3];                  // (ox - X0) mod Ix, (oy - Y0) mod Iy, z switch key
    __shared__ int sIdx[MT_B];
    __shared__ int sList[8 * MT_B];               // per-warp particle lists
    __shared__ unsigned char sMask[MT_B];
    __shared__ int sWarpCnt[8];
    const MidArgs& a = t.a;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bz = blockIdx.x % t.ntz, rest = blockIdx.x / t.ntz;
    const int by = rest % t.nty, bx = rest / t.nty;
    const int X0 = bx * MT_X, Y0 = by * MT_Y, Z0 = bz * MT_Z;
    t.Y0 = Y0;
    const int wx0 = X0 + 4 * (warp & 3), wy0 = Y0 + 8 * (warp >> 2);
    const int cx = wx0 + (lane & 3), cy = wy0 + (lane >> 2);
    const bool colok = cx < a.Ix && cy < a.Iy;
    double acc[MT_Z];
#pragma unroll
    for (int z = 0; z < MT_Z; ++z) acc[z] = 0.0;

    if ((Z0 + MT_Z - 1 + p >= t.gz_lo) && (Z0 - p <= t.gz_hi)) {
        const CellGeo& g = t.g;
        // candidate cells: stencil centre g0 in [T0 - p, T0 + T - 1 + p]  <=>  x in [lo, hi)
        auto crange = [&](int T0, int T, double h, double half, double L, double sc, int& c0, int& c1) {
            double lo = ((T0 - p) - 0.5 - half) * h, hi = ((T0 + T - 1 + p) + 0.5 - half) * h;
            c0 = (int)floor((lo + 0.5 * L) * sc) - 1;
            c1 = (int)floor((hi + 0.5 * L) * sc) + 1;
        };
        int cx0, cx1, cy0, cy1, cz0, cz1;
        crange(X0, MT_X, a.hx, a.halfx, g.Lx, g.sx, cx0, cx1);
        crange(Y0, MT_Y, a.hy, a.halfy, g.Ly, g.sy, cy0, cy1);
        crange(Z0, MT_Z, a.hz, a.halfz, g.Lz, g.sz, cz0, cz1);
        if (cx1 - cx0 + 1 >= g.ncx) { cx0 = 0; cx1 = g.ncx - 1; }
        if (cy1 - cy0 + 1 >= g.ncy) { cy0 = 0; cy1 = g.ncy - 1; }
        cz0 = max(cz0, 0);
        cz1 = min(cz1, g.ncz - 1);
        const int nyc = cy1 - cy0 + 1, ncol = (cx1 - cx0 + 1) * nyc;
        int nst = 0;                                  // staged count (block-uniform)
        for (int cc = 0; cc < ncol && cz0 <= cz1; ++cc) {
            const int ccx = wrapc(cx0 + cc / nyc, g.ncx), ccy = wrapc(cy0 + cc % nyc, g.ncy);
            const int cbase = (ccx * g.ncy + ccy) * g.ncz;
            const int j0 = t.start[cbase + cz0], j1 = t.start[cbase + cz1 + 1];
            for (int jb = j0; jb < j1; jb += 256) {
                const int j = jb + tid;
                bool hit = false;
                int ox = 0, oy = 0, oz = 0;
                if (j < j1) {
                    d4 r = ld_d4(&a.pos[j]);
                    ox = stencil_g0(r.x, a.hx, a.hpx) - p;
                    oy = stencil_g0(r.y, a.hy, a.hpy) - p;
                    oz = stencil_g0(r.z, a.hz, a.hpz) - p;
                    ox = wrapc(ox - X0, a.Ix);
                    oy = wrapc(oy - Y0, a.Iy);
                    oz = oz - Z0 + (P - 1);                  // z switch key
                    hit = (ox < MT_X || ox > a.Ix - P) && (oy < MT_Y || oy > a.Iy - P) && oz >= 0 && oz < MT_Z + P - 1;
                }
                // deterministic compaction: ballot + prefix over warps in order
                const unsigned m = __ballot_sync(0xffffffffu, hit);
                if (lane == 0) sWarpCnt[warp] = __popc(m);
                __syncthreads();
                int off = 0, tot = 0;
#pragma unroll
                for (int w = 0; w < 8; ++w) { off += w < warp ? sWarpCnt[w] : 0; tot += sWarpCnt[w]; }
                off += __popc(m & ((1u << lane) - 1));
                if (nst + tot > MT_B) {                      // flush before it overflows
                    mid_tile_batch<P>(t, nst, sIdx, sO, sW, sMask, sList, acc, X0, Z0, colok);
                    nst = 0;
                }
                if (hit) {
                    const int q = nst + off;
                    sIdx[q] = j; sO[3 * q] = ox; sO[3 * q + 1] = oy; sO[3 * q + 2] = oz;
                }
                nst += tot;
                __syncthreads();
            }
        }
        if (nst > 0) mid_tile_batch<P>(t, nst, sIdx, sO, sW, sMask, sList, acc, X0, Z0, colok);
    }
    // write my column's MT_Z values: every grid point is written exactly once
    if (colok) {
        const size_t o = ((size_t)cx * a.Iy + cy) * a.Izs + Z0;
        double* col = grid + o;
        const int nz = min(MT_Z, a.Izs - Z0);
        if (nz == MT_Z && (o & 1) == 0) {
            double2* c2 = reinterpret_cast<double2*>(col);
#pragma unroll
            for (int z = 0; z < MT_Z; z += 2) c2[z / 2] = make_double2(acc[z], acc[z + 1]);
        } else {
#pragma unroll
            for (int z = 0; z < MT_Z; ++z)
                if (z < nz) col[z] = acc[z];
        }
    }
}

}  // namespace sog
