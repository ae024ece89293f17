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

// v mod n for v in (-2n, 2n) without integer division
__device__ __forceinline__ int wrapc(int v, int n) {
    v += v < 0 ? n : 0;
    v += v < 0 ? n : 0;
    v -= v >= n ? n : 0;
    v -= v >= n ? n : 0;
    return v;
}

// Stage weights of sIdx[0..nst): Wx[P], Wy[P], q and Wz scattered into the tile's MT_Z
// z slots (zeros elsewhere) with a 2-bit mask of the non-empty 12-slot halves; build each
// warp's list of particles touching its 4 x 8 column patch; then every lane adds
// c = q Wx Wy times the padded Wz into its registers, 12 dense FMAs per touched half
// (no per-particle branching on the z offset).
constexpr int MT_NW(int P) { return (2 * P + 1 + MT_Z + 1) & ~1; }   // [Wz padded | Wx | Wy | q], even

template <int P>
__device__ __forceinline__ void mid_tile_batch(const MidTileArgs& t, const int4* __restrict__ g0, int nst,
                                               const int* sIdx, int* sO, double* sW, unsigned char* sMask,
                                               unsigned short* sList, double (&acc)[MT_Z], bool colok) {
    constexpr int p = (P - 1) / 2;
    constexpr int NW = MT_NW(P);
    const MidArgs& a = t.a;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int s = tid; s < nst; s += blockDim.x) {
        d4 r = ld_d4(&a.pos[sIdx[s]]);
        const int dxo = sO[3 * s], dyo = sO[3 * s + 1], key = sO[3 * s + 2];
        // unwrapped stencil centres (the weights need the particle's own periodic image)
        const int4 o = g0[sIdx[s]];
        const int gx0 = o.x, gy0 = o.y, gz0 = o.z;
        double wx[P], wy[P], wz[P];
        window_weights_rec<P, false>(r.x, gx0, a.hx, a.halfx, a.invH2Sx, t.gamma_x, wx, nullptr);
        window_weights_rec<P, false>(r.y, gy0, a.hy, a.halfy, a.invH2Sy, t.gamma_y, wy, nullptr);
        window_weights_rec<P, false>(r.z, gz0, a.hz, a.halfz, a.invH2Sz, t.gamma_z, wz, nullptr);
        double* wzp = sW + s * NW;                     // 16-byte aligned (NW even)
        double* w = wzp + MT_Z;
#pragma unroll
        for (int k = 0; k < P; ++k) { w[k] = wx[k]; w[P + k] = wy[k]; }
        w[2 * P] = r.w;
        const int zs = key - (P - 1);                  // tile slot of stencil point 0
#pragma unroll
        for (int z = 0; z < MT_Z; ++z) wzp[z] = 0.0;
#pragma unroll
        for (int k = 0; k < P; ++k)
            if (zs + k >= 0 && zs + k < MT_Z) wzp[zs + k] = wz[k];
        unsigned m = 0;
#pragma unroll
        for (int wq = 0; wq < 8; ++wq) {
            const int u0 = wrapc(4 * (wq & 3) - dxo, a.Ix), v0 = wrapc(8 * (wq >> 2) - dyo, a.Iy);
            if ((u0 < P || u0 > a.Ix - 4) && (v0 < P || v0 > a.Iy - 8)) m |= 1u << wq;
        }
        sMask[s] = (unsigned char)m;
        // halves of the z tile that hold stencil points: [zs, zs+P) intersect [0,12) / [12,24)
        sO[3 * s + 2] = (zs < MT_Z / 2 ? 1 : 0) | (zs + P - 1 >= MT_Z / 2 ? 2 : 0);
    }
    __syncthreads();
    // per-warp compaction of the particles touching this warp's patch (order preserved)
    unsigned short* myl = sList + warp * MT_B;
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
        const double* wzp = sW + s * NW;
        const double* w = wzp + MT_Z;
        const int u = wrapc(wofx - sO[3 * s], a.Ix), v = wrapc(wofy - sO[3 * s + 1], a.Iy);
        const double c = (colok && u < P && v < P) ? w[2 * P] * w[u] * w[P + v] : 0.0;
        const int halves = sO[3 * s + 2];
        const double2* wz2 = reinterpret_cast<const double2*>(wzp);
        if (halves & 1) {
#pragma unroll
            for (int z = 0; z < MT_Z / 2; z += 2) {
                const double2 q = wz2[z / 2];
                acc[z] = fma(c, q.x, acc[z]);
                acc[z + 1] = fma(c, q.y, acc[z + 1]);
            }
        }
        if (halves & 2) {
#pragma unroll
            for (int z = MT_Z / 2; z < MT_Z; z += 2) {
                const double2 q = wz2[z / 2];
                acc[z] = fma(c, q.x, acc[z]);
                acc[z + 1] = fma(c, q.y, acc[z + 1]);
            }
        }
    }
    __syncthreads();
}

// Stencil origins (nearest grid points, R6) of every sorted particle, computed once per
// evaluation with the exact-rounding decision of stencil_g0 (shared by spread and gather).
static __global__ void k_stencil_origins(const d4* __restrict__ pos, int N, MidArgs a, int has_mid, double lhx,
                                         double lhy, double lhpx, double lhpy, int4* __restrict__ g0) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const d4 r = ld_d4(&pos[i]);
    int4 o;
    if (has_mid) {
        o.x = stencil_g0(r.x, a.hx, a.hpx);
        o.y = stencil_g0(r.y, a.hy, a.hpy);
        o.z = stencil_g0(r.z, a.hz, a.hpz);
    } else {
        o.x = o.y = o.z = 0;
    }
    const int lx = stencil_g0(r.x, lhx, lhpx), ly = stencil_g0(r.y, lhy, lhpy);
    o.w = (lx + 32768) | ((ly + 32768) << 16);       // long-grid origins, biased 16-bit fields
    g0[i] = o;
}

constexpr int MT_HCAP = 1024;    // hit entries kept per CTA pass

template <int P>
__global__ void __launch_bounds__(256, 2) k_mid_spread_tile(MidTileArgs t, const int4* __restrict__ g0,
                                                            double* __restrict__ grid) {
    constexpr int p = (P - 1) / 2;
    extern __shared__ double sW[];                // [MT_B][MT_NW(P)] staged weights (dynamic)
    __shared__ int sO[MT_B * 3];                  // (ox - X0) mod Ix, (oy - Y0) mod Iy, z key
    __shared__ int sIdx[MT_B];
    __shared__ unsigned short sList[8 * MT_B];    // per-warp particle lists
    __shared__ unsigned char sMask[MT_B];
    __shared__ int sHit[MT_HCAP];                 // hit particle indices (deterministic order)
    __shared__ int sCnt[256];
    const MidArgs& a = t.a;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bz = blockIdx.x % t.ntz, rest = blockIdx.x / t.ntz;
    const int by = rest % t.nty, bx = rest / t.nty;
    const int X0 = bx * MT_X, Y0 = by * MT_Y, Z0 = bz * MT_Z;
    t.Y0 = Y0;
    const int cx = X0 + 4 * (warp & 3) + (lane & 3), cy = Y0 + 8 * (warp >> 2) + (lane >> 2);
    const bool colok = cx < a.Ix && cy < a.Iy;
    double acc[MT_Z];
#pragma unroll
    for (int z = 0; z < MT_Z; ++z) acc[z] = 0.0;

    if ((Z0 + MT_Z - 1 + p >= t.gz_lo) && (Z0 - p <= t.gz_hi)) {
        const CellGeo& g = t.g;
        // candidate cells: stencil origin in [T0 - P + 1, T0 + T - 1]  <=>  coordinate in [lo, hi)
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
        auto is_hit = [&](int j, int& ox, int& oy, int& key) {
            const int4 o = g0[j];
            ox = wrapc(o.x - p - X0, a.Ix);
            oy = wrapc(o.y - p - Y0, a.Iy);
            key = o.z - p - Z0 + (P - 1);
            return (ox < MT_X || ox > a.Ix - P) && (oy < MT_Y || oy > a.Iy - P) && key >= 0 && key < MT_Z + P - 1;
        };
        // Phase A: each thread counts the hits among its candidates (column-major cell order)
        int mycnt = 0;
        if (cz0 <= cz1)
            for (int cc = 0; cc < ncol; ++cc) {
                const int ccx = wrapc(cx0 + cc / nyc, g.ncx), ccy = wrapc(cy0 + cc % nyc, g.ncy);
                const int cbase = (ccx * g.ncy + ccy) * g.ncz;
                const int j0 = t.start[cbase + cz0], j1 = t.start[cbase + cz1 + 1];
                for (int j = j0 + tid; j < j1; j += 256) {
                    int ox, oy, key;
                    mycnt += is_hit(j, ox, oy, key) ? 1 : 0;
                }
            }
        sCnt[tid] = mycnt;
        __syncthreads();
        // exclusive prefix over threads (deterministic order: thread, then candidate)
        for (int o = 1; o < 256; o <<= 1) {
            const int v = tid >= o ? sCnt[tid - o] : 0;
            __syncthreads();
            sCnt[tid] += v;
            __syncthreads();
        }
        const int total = sCnt[255];
        const int myoff = sCnt[tid] - mycnt;
        __syncthreads();
        for (int w0 = 0; w0 < total; w0 += MT_HCAP) {          // usually one window
            // Phase B: write the hits falling in this window
            if (myoff + mycnt > w0 && myoff < w0 + MT_HCAP && cz0 <= cz1) {
                int k = myoff;
                for (int cc = 0; cc < ncol; ++cc) {
                    const int ccx = wrapc(cx0 + cc / nyc, g.ncx), ccy = wrapc(cy0 + cc % nyc, g.ncy);
                    const int cbase = (ccx * g.ncy + ccy) * g.ncz;
                    const int j0 = t.start[cbase + cz0], j1 = t.start[cbase + cz1 + 1];
                    for (int j = j0 + tid; j < j1; j += 256) {
                        int ox, oy, key;
                        if (is_hit(j, ox, oy, key)) {
                            if (k >= w0 && k < w0 + MT_HCAP) sHit[k - w0] = j;
                            ++k;
                        }
                    }
                }
            }
            __syncthreads();
            const int nw = min(MT_HCAP, total - w0);
            // Phase C: stage and apply in batches of MT_B
            for (int b0 = 0; b0 < nw; b0 += MT_B) {
                const int nst = min(MT_B, nw - b0);
                for (int s = tid; s < nst; s += 256) {
                    const int j = sHit[b0 + s];
                    int ox, oy, key;
                    is_hit(j, ox, oy, key);
                    sIdx[s] = j; sO[3 * s] = ox; sO[3 * s + 1] = oy; sO[3 * s + 2] = key;
                }
                __syncthreads();
                mid_tile_batch<P>(t, g0, nst, sIdx, sO, sW, sMask, sList, acc, colok);
            }
        }
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
