// S2 v4: near-field pair sum (Eq. eq::phiNDR), target-stationary.
//
//   phi^N_i = sum_{j: r_ij < r_c} q_j (1/r_ij - F(r_ij^2)),   grad phi^N_i = sum_j q_j (-1/r^3 - 2 F'(u)) r_ij
//
// A CTA owns a chunk of KC consecutive cells of one (x, y) cell column and stages the 3 x 3
// neighbouring columns over the chunk's z range plus one cell on each side (every source within r_c
// of a chunk particle; cells are >= r_c) in shared memory, once: fp32 coordinates relative to the
// chunk corner for the pre-test and the fp64 record (relative x, y, z with the periodic image shift
// applied, q) for the exact evaluation.  Staged columns are z-sorted (cell sort), so a warp whose 32
// lanes own 32 consecutive (z-sorted) targets scans only the z window [z_min - r_c, z_max + r_c] of
// each column.  Every lane tests the same candidate (shared-memory broadcast), in fp32 with a
// conservative threshold; a passing candidate's staged index goes into the lane's own queue.  When a
// queue nears full, the warp runs evaluation rounds: each lane pops one pair and evaluates it
// exactly in fp64 (the r < r_c decision too), so the FP64 work runs with (nearly) all lanes busy.
// F(u) and F'(u) come from ONE polynomial (R16-G) whose coefficients are kernel parameters
// (constant-bank operands shared by all lanes: no per-pair table loads).  Each lane accumulates its
// own target's sums in a fixed order: the result is deterministic.
#pragma once
#include "kernels_common.cuh"
#include "kernels_near3.cuh"

namespace sog {

constexpr int N4_Q = 48;              // queue slots per lane (16-bit staged indices)
constexpr int N4_MAXW = 8;            // warps per CTA (upper bound)

struct Near4Args {
    const d4* pos;          // cell-sorted (x, y, z, q)
    const int* start;       // cell start offsets [ncell + 1]
    d4* out;                // (phi, dphi/dx, dphi/dy, dphi/dz) per sorted particle
    CellGeo g;
    double rc2;             // exact decision r^2 < r_c^2 (fp64)
    float rc2f;             // conservative fp32 pre-test threshold
    float rcz;              // conservative fp32 z-window half width
    int kc;                 // cells per chunk
    int cap;                // staged capacity (records)
};


template <int D>
__global__ void __launch_bounds__(32 * N4_MAXW) k_near4(Near4Args a, NearPolyArg<D> P) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int nw = blockDim.x >> 5;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned short* queue = reinterpret_cast<unsigned short*>(smraw);       // [nw][N4_Q][32]
    __shared__ int colb[9], coln[9];                                        // staged column ranges
    double2* sxy = reinterpret_cast<double2*>(queue + nw * N4_Q * 32);      // [cap] rel x, y (fp64)
    double2* szq = sxy + a.cap;                                             // [cap] rel z (fp64), q
    float* sxf = reinterpret_cast<float*>(szq + a.cap);                     // [cap] rel x, y, z (fp32)
    float* syf = sxf + a.cap;
    float* szf = syf + a.cap;
    const CellGeo& g = a.g;
    const int col = blockIdx.x;                                             // cx * ncy + cy
    const int cx = col / g.ncy, cy = col - cx * g.ncy;
    const int cz0 = blockIdx.y * a.kc, cz1 = min(g.ncz, cz0 + a.kc);        // target cells [cz0, cz1)
    const int cbase = col * g.ncz;
    const int t0 = a.start[cbase + cz0], t1 = a.start[cbase + cz1];
    if (t0 == t1) return;
    const int zl = max(0, cz0 - g.nzr), zh = min(g.ncz - 1, cz1 - 1 + g.nzr);   // staged cells
    const double ox = g.x0 + cx / g.sx, oy = cy / g.sy - 0.5 * g.Ly, oz = cz0 / g.sz - 0.5 * g.Lz;
    // staged column k = 3 (ux - cx + 1) + (uy - cy + 1): global ranges and periodic shifts
    __shared__ int jb[9], jn[9];
    __shared__ double shx[9], shy[9];
    if (threadIdx.x < 9) {
        const int k = threadIdx.x;
        const int ux = cx + k / 3 - 1, uy = cy + k % 3 - 1;
        int b = 0, n = 0;
        double sx = 0.0, sy = 0.0;
        if (g.px || (ux >= 0 && ux < g.ncx)) {                              // x-slab: no x images
            const int nx = ux < 0 ? ux + g.ncx : (ux >= g.ncx ? ux - g.ncx : ux);
            const int ny = uy < 0 ? uy + g.ncy : (uy >= g.ncy ? uy - g.ncy : uy);
            sx = !g.px ? 0.0 : (ux < 0 ? -g.Lx : (ux >= g.ncx ? g.Lx : 0.0));
            sy = uy < 0 ? -g.Ly : (uy >= g.ncy ? g.Ly : 0.0);
            const int cb = (nx * g.ncy + ny) * g.ncz;
            b = a.start[cb + zl];
            n = a.start[cb + zh + 1] - b;
        }
        jb[k] = b;
        jn[k] = n;
        shx[k] = sx;
        shy[k] = sy;
    }
    __syncthreads();
    int ntot = 0;
#pragma unroll
    for (int k = 0; k < 9; ++k) ntot += jn[k];
    const float rc2f = a.rc2f, rcz = a.rcz;
    // the polynomial's coefficients live in registers for the whole kernel (sm_100 DFMA takes no
    // constant-bank operand; occupancy is bounded by shared memory, so the registers are free)
    double cr[D + 1];
#pragma unroll
    for (int n = 0; n <= D; ++n) cr[n] = P.c[n];
    const double inv_h = P.inv_h;
    unsigned short* wq = queue + warp * N4_Q * 32;
    // the neighbourhood in capacity-sized pieces (one piece unless the input is very clustered);
    // piece p covers the concatenated column ranges [pb, pe)
    for (int pb = 0; pb < ntot; pb += a.cap) {
        const int pe = min(ntot, pb + a.cap);
        __syncthreads();
        {
            int base = 0;
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                const int lo = max(pb, base), hi = min(pe, base + jn[k]);
                for (int q = lo + threadIdx.x; q < hi; q += blockDim.x) {
                    const d4 s = ld_d4(&a.pos[jb[k] + (q - base)]);
                    const double rx = (s.x + shx[k]) - ox, ry = (s.y + shy[k]) - oy, rz = s.z - oz;
                    sxy[q - pb] = make_double2(rx, ry);
                    szq[q - pb] = make_double2(rz, s.w);
                    sxf[q - pb] = (float)rx;
                    syf[q - pb] = (float)ry;
                    szf[q - pb] = (float)rz;
                }
                if (threadIdx.x == 0) {
                    colb[k] = max(0, lo - pb);
                    coln[k] = max(0, hi - lo);
                }
                base += jn[k];
            }
        }
        __syncthreads();
        // target groups of 32 consecutive (z-sorted) particles of the chunk
        for (int tg = t0 + 32 * warp; tg < t1; tg += 32 * nw) {
            const int it = tg + lane;
            const bool valid = it < t1;
            double xi = 0.0, yi = 0.0, zi = 0.0;
            if (valid) {
                const d4 p = ld_d4(&a.pos[it]);
                xi = p.x - ox;
                yi = p.y - oy;
                zi = p.z - oz;
            }
            const float xf = (float)xi, yf = (float)yi, zf = (float)zi;
            // z window of the group (lanes past t1 repeat the last valid target)
            float zmn = valid ? zf : 3.0e38f, zmx = valid ? zf : -3.0e38f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                zmn = fminf(zmn, __shfl_xor_sync(0xffffffffu, zmn, o));
                zmx = fmaxf(zmx, __shfl_xor_sync(0xffffffffu, zmx, o));
            }
            // lane k < 9: window [wlo, whi) of staged column k by binary search on the sorted z
            int wlo = 0, whi = 0;
            if (lane < 9) {
                const int b0 = colb[lane], n = coln[lane];
                int lo = 0, hi = n;
                const float zlo = zmn - rcz, zhi = zmx + rcz;
                while (lo < hi) {                                            // first z >= zlo
                    const int m = (lo + hi) >> 1;
                    if (szf[b0 + m] < zlo) lo = m + 1; else hi = m;
                }
                wlo = b0 + lo;
                hi = n;
                while (lo < hi) {                                            // first z > zhi
                    const int m = (lo + hi) >> 1;
                    if (szf[b0 + m] <= zhi) lo = m + 1; else hi = m;
                }
                whi = b0 + lo;
            }
            double phi = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
            int cnt = 0;
            // exact evaluation of one popped pair (R16-G polynomial, joint Horner with constant-bank
            // coefficients); NP pairs per call are independent chains (latency hiding at low occupancy)
            auto eval = [&](int j, double& ph, double& ex, double& ey, double& ez) {
                const double2 sa = sxy[j], sb = szq[j];
                const double dx = xi - sa.x, dy = yi - sa.y, dz = zi - sb.x;
                const double u = fma(dx, dx, fma(dy, dy, dz * dz));
                if (u < a.rc2 && u > 0.0) {
                    const double t = fma(u, inv_h, -1.0);
                    double F = cr[D], dF = 0.0;
#pragma unroll
                    for (int n = D - 1; n >= 0; --n) {
                        dF = fma(dF, t, F);
                        F = fma(F, t, cr[n]);
                    }
                    const double rinv = rsqrt(u);
                    ph = fma(sb.y, rinv - F, ph);
                    const double cc = sb.y * (-rinv * rinv * rinv - 2.0 * inv_h * dF);
                    ex = fma(cc, dx, ex);
                    ey = fma(cc, dy, ey);
                    ez = fma(cc, dz, ez);
                }
            };
            // one round: every lane with a queued pair pops one
            auto round1 = [&]() {
                if (cnt > 0) {
                    --cnt;
                    eval(wq[cnt * 32 + lane], phi, gx, gy, gz);
                }
            };
            // two pops per lane (every valid lane has >= 2 queued): two independent chains
            double p2 = 0.0, x2 = 0.0, y2 = 0.0, z2 = 0.0;
            auto round2 = [&]() {
                if (cnt > 1) {
                    cnt -= 2;
                    const int ja = wq[(cnt + 1) * 32 + lane], jb2 = wq[cnt * 32 + lane];
                    eval(ja, phi, gx, gy, gz);
                    eval(jb2, p2, x2, y2, z2);
                }
            };
#pragma unroll 1
            for (int k = 0; k < 9; ++k) {
                const int lo = __shfl_sync(0xffffffffu, wlo, k), hi = __shfl_sync(0xffffffffu, whi, k);
                for (int j0 = lo; j0 < hi; j0 += 4) {
                    // room for 4 more in every queue (rare: the rounds below run at column ends)
                    while (__any_sync(0xffffffffu, cnt > N4_Q - 4)) round1();
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int j = j0 + r;
                        if (j < hi) {
                            const float dx = xf - sxf[j], dy = yf - syf[j], dz = zf - szf[j];
                            const float u = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                            if (u < rc2f && valid) {
                                wq[cnt * 32 + lane] = (unsigned short)j;
                                ++cnt;
                            }
                        }
                    }
                }
                // rounds while every valid lane has work (full lanes), two pops at a time
                while (__all_sync(0xffffffffu, cnt > 1 || !valid) && __any_sync(0xffffffffu, cnt > 1)) round2();
            }
            while (__all_sync(0xffffffffu, cnt > 1 || !valid) && __any_sync(0xffffffffu, cnt > 1)) round2();
            while (__any_sync(0xffffffffu, cnt > 0)) round1();
            phi += p2;
            gx += x2;
            gy += y2;
            gz += z2;
            if (valid) {
                if (pb == 0) {
                    st_d4(&a.out[it], d4{phi, gx, gy, gz});
                } else {
                    const d4 o = a.out[it];
                    st_d4(&a.out[it], d4{o.x + phi, o.y + gx, o.z + gy, o.w + gz});
                }
            }
        }
    }
}

}  // namespace sog
