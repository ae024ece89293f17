// S2 v3: near-field pair sum (Eq. eq::phiNDR), one CTA per near-field cell.
// The 27 neighbouring cells' particles are staged once per CTA in shared memory (fp64, with
// their periodic image shift applied: cells >= r_c and >= 3 per periodic axis, so each
// neighbour cell has exactly one relevant image).  Each warp owns one target at a time; its
// lanes sweep the staged sources 32 at a time, passing pairs (r < r_c) are compacted by
// ballot into a per-warp list and evaluated 32 at a time with all lanes busy, and the lane
// partials are reduced with shuffles.  F(u), u = r^2, and F'(u) come from one piecewise
// polynomial per piece (joint Horner).
#pragma once
#include "kernels_common.cuh"

namespace sog {

struct Near3Args {
    const d4* pos;          // sorted (x,y,z,q)
    const int* start;       // cell start offsets [ncell+1]
    const double* cF;       // K x (D+1) polynomial coefficients of F on each piece
    d4* out;
    int K;
    double du, inv_du, rc2;
    CellGeo g;
    int cap;                // staged-source capacity (shared memory)
    float rc2f;             // conservative fp32 pre-test threshold
    const int* perm = nullptr;   // x-slab ranks: sorted -> local index; targets are own particles only
    int nown = 0;                //   (local index < nown), halo particles are sources only
};

// x-slab ranks: does cell [t0, t1) hold an own particle (else the CTA has no target)
__device__ __forceinline__ bool near_has_target(const Near3Args& a, int t0, int t1) {
    if (!a.perm) return true;
    int own = 0;
    for (int it = t0 + (int)threadIdx.x; it < t1; it += blockDim.x) own |= a.perm[it] < a.nown;
    return __syncthreads_or(own) != 0;
}

constexpr int NEAR3_WARPS = 4;

// F(u), dF/du from the piecewise table (R16) in shared memory
template <int D>
struct NearTab {
    const double* tab;
    int K;
    double du, inv_du;
    __device__ __forceinline__ void operator()(double u, double& F, double& dF) const {
        const int kk = min(K - 1, (int)(u * inv_du));
        const double d = u - (kk + 0.5) * du;
        const double* cf = tab + kk * (D + 1);
        F = cf[D];
        dF = 0.0;
#pragma unroll
        for (int n = D - 1; n >= 0; --n) {
            dF = fma(dF, d, F);
            F = fma(F, d, cf[n]);
        }
    }
};

// F(u), dF/du from one polynomial in t = u inv_h - 1 (R16-G): the same coefficients for every lane
template <int D>
struct NearPolyArg {
    double c[D + 1];
    double inv_h;
    __device__ __forceinline__ void operator()(double u, double& F, double& dF) const {
        const double t = fma(u, inv_h, -1.0);
        F = c[D];
        double g = 0.0;
#pragma unroll
        for (int n = D - 1; n >= 0; --n) {
            g = fma(g, t, F);
            F = fma(F, t, c[n]);
        }
        dF = g * inv_h;
    }
};

template <class KF>
__device__ __forceinline__ void near_pair(const KF& kf, const Near3Args& a, const d4& pi, int code,
                                          const double2* shift, double& phi, double& gx, double& gy, double& gz) {
    const d4 s = ld_d4(&a.pos[code >> 4]);
    const double2 sh = shift[code & 15];
    const double dx = pi.x - (s.x + sh.x), dy = pi.y - (s.y + sh.y), dz = pi.z - s.z;
    const double u = fma(dx, dx, fma(dy, dy, dz * dz));
    if (!(u < a.rc2 && u > 0.0)) return;        // exact fp64 decision (the fp32 test is a superset)
    double F, dF;
    kf(u, F, dF);
    const double rinv = rsqrt(u);
    phi = fma(s.w, rinv - F, phi);
    const double cc = s.w * (-rinv * rinv * rinv - 2.0 * dF);
    gx = fma(cc, dx, gx);
    gy = fma(cc, dy, gy);
    gz = fma(cc, dz, gz);
}

template <int D, int PD = 0>
__global__ void __launch_bounds__(32 * NEAR3_WARPS) k_near3(Near3Args a, NearPolyArg<PD == 0 ? 1 : PD> poly = {}) {
    extern __shared__ double sm[];
    double* tab = sm;                                                   // [K*(D+1)] (PD == 0)
    double2* shift = reinterpret_cast<double2*>(sm + (PD == 0 ? ((a.K * (D + 1) + 1) & ~1) : 0));   // [9]
    int* lists = reinterpret_cast<int*>(shift + 10);                    // [warps][160]
    // staged sources in 64-wide blocks, candidate q = 64 b + 32 h + l stored as
    //   sxy[b][l] = (x_h0, x_h1, y_h0, y_h1), sz[b][l] = (z_h0, z_h1), sc[b][l] = (code_h0, code_h1)
    // so that one lane tests two candidates with packed fp32x2 arithmetic
    float4* sxy = reinterpret_cast<float4*>(lists + NEAR3_WARPS * 160); // [cap/64][32]
    float2* sz = reinterpret_cast<float2*>(sxy + a.cap / 2);             // [cap/64][32]
    int2* sc = reinterpret_cast<int2*>(sz + a.cap / 2);                  // [cap/64][32]
    const CellGeo& g = a.g;
    const int c = blockIdx.x;
    const int cz = c % g.ncz, cy = (c / g.ncz) % g.ncy, cx = c / (g.ncz * g.ncy);
    const int t0 = a.start[c], t1 = a.start[c + 1];
    if (t0 == t1 || !near_has_target(a, t0, t1)) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (PD == 0)
        for (int t = threadIdx.x; t < a.K * (D + 1); t += blockDim.x) tab[t] = a.cF[t];
    if (threadIdx.x < 9) {
        const int k = threadIdx.x, ux = cx + k / 3 - 1, uy = cy + k % 3 - 1;
        shift[k] = make_double2(!g.px ? 0.0 : (ux < 0 ? -g.Lx : (ux >= g.ncx ? g.Lx : 0.0)),
                                uy < 0 ? -g.Ly : (uy >= g.ncy ? g.Ly : 0.0));
    }
    const double ox = g.x0 + cx / g.sx, oy = cy / g.sy - 0.5 * g.Ly, oz = cz / g.sz - 0.5 * g.Lz;
    const int z0 = max(0, cz - g.nzr), z1 = min(g.ncz - 1, cz + g.nzr);
    int* wl = lists + warp * 160;
    int ns_total = 0;
    for (int k = 0; k < 9; ++k) {
        int nx = cx + k / 3 - 1, ny = cy + k % 3 - 1;
        if (!g.px && (nx < 0 || nx >= g.ncx)) continue;           // x-slab: no x images
        nx += nx < 0 ? g.ncx : 0; nx -= nx >= g.ncx ? g.ncx : 0;
        ny += ny < 0 ? g.ncy : 0; ny -= ny >= g.ncy ? g.ncy : 0;
        const int cb = (nx * g.ncy + ny) * g.ncz;
        ns_total += a.start[cb + z1 + 1] - a.start[cb + z0];
    }
    float* sxyf = reinterpret_cast<float*>(sxy);
    float* szf = reinterpret_cast<float*>(sz);
    int* scf = reinterpret_cast<int*>(sc);
    auto put = [&](int q, float x, float y, float z, int code) {
        const int b = q >> 6, h = (q >> 5) & 1, l = q & 31, e = b * 32 + l;
        sxyf[4 * e + h] = x;
        sxyf[4 * e + 2 + h] = y;
        szf[2 * e + h] = z;
        scf[2 * e + h] = code;
    };
    const float rc2f = a.rc2f;
    // process the neighbourhood in capacity-sized pieces (usually one)
    for (int sbeg = 0; sbeg < ns_total; sbeg += a.cap) {
        const int send = min(ns_total, sbeg + a.cap);
        const int nsrc = send - sbeg, npad = (nsrc + 127) & ~127;
        __syncthreads();
        // stage sources [sbeg, send) of the concatenated 9-column list with image shifts
        {
            int base = 0;
            for (int k = 0; k < 9; ++k) {
                const int ux = cx + k / 3 - 1, uy = cy + k % 3 - 1;
                if (!g.px && (ux < 0 || ux >= g.ncx)) continue;       // x-slab: no x images
                const int nx = ux < 0 ? ux + g.ncx : (ux >= g.ncx ? ux - g.ncx : ux);
                const int ny = uy < 0 ? uy + g.ncy : (uy >= g.ncy ? uy - g.ncy : uy);
                const double sx = !g.px ? 0.0 : (ux < 0 ? -g.Lx : (ux >= g.ncx ? g.Lx : 0.0));
                const double sy = uy < 0 ? -g.Ly : (uy >= g.ncy ? g.Ly : 0.0);
                const int cb = (nx * g.ncy + ny) * g.ncz;
                const int jb = a.start[cb + z0], n = a.start[cb + z1 + 1] - jb;
                const int lo = max(sbeg, base), hi = min(send, base + n);
                for (int q = lo + threadIdx.x; q < hi; q += blockDim.x) {
                    const int j = jb + (q - base);
                    const d4 s = ld_d4(&a.pos[j]);
                    put(q - sbeg, (float)(s.x + sx - ox), (float)(s.y + sy - oy), (float)(s.z - oz), (j << 4) | k);
                }
                base += n;
            }
            for (int q = nsrc + threadIdx.x; q < npad; q += blockDim.x) put(q, 1e18f, 0.f, 0.f, 0);   // sentinels
        }
        __syncthreads();
        for (int it = t0 + warp; it < t1; it += NEAR3_WARPS) {
            if (a.perm && a.perm[it] >= a.nown) continue;      // halo particle: a source only
            const d4 pi = ld_d4(&a.pos[it]);
            const float xi = (float)(pi.x - ox), yi = (float)(pi.y - oy), zi = (float)(pi.z - oz);
            const float2 xi2 = make_float2(xi, xi), yi2 = make_float2(yi, yi), zi2 = make_float2(zi, zi);
            const float2 m1 = make_float2(-1.f, -1.f);
            double phi = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
            int npend = 0;
            for (int q0 = 0; q0 < npad; q0 += 128) {
                // fp32 pre-test of 4 x 32 sources, two per packed fp32x2 operation
                bool pass[4];
                int code[4];
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const int e = (q0 >> 6) * 32 + r * 32 + lane;
                    const float4 xy = sxy[e];
                    const float2 zz = sz[e];
                    const int2 cc = sc[e];
                    const float2 dx = __ffma2_rn(make_float2(xy.x, xy.y), m1, xi2);
                    const float2 dy = __ffma2_rn(make_float2(xy.z, xy.w), m1, yi2);
                    const float2 dz = __ffma2_rn(zz, m1, zi2);
                    const float2 r2 = __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __fmul2_rn(dz, dz)));
                    pass[2 * r] = r2.x < rc2f;
                    pass[2 * r + 1] = r2.y < rc2f;
                    code[2 * r] = cc.x;
                    code[2 * r + 1] = cc.y;
                }
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const unsigned m = __ballot_sync(0xffffffffu, pass[r]);
                    if (pass[r]) wl[npend + __popc(m & ((1u << lane) - 1))] = code[r];
                    npend += __popc(m);
                }
                __syncwarp();
                while (npend >= 32) {                    // evaluate 32 pending pairs, all lanes busy
                    npend -= 32;
                    if constexpr (PD == 0) near_pair(NearTab<D>{tab, a.K, a.du, a.inv_du}, a, pi, wl[npend + lane], shift, phi, gx, gy, gz);
                    else near_pair(poly, a, pi, wl[npend + lane], shift, phi, gx, gy, gz);
                }
                __syncwarp();
            }
            if (lane < npend) {
                if constexpr (PD == 0) near_pair(NearTab<D>{tab, a.K, a.du, a.inv_du}, a, pi, wl[lane], shift, phi, gx, gy, gz);
                else near_pair(poly, a, pi, wl[lane], shift, phi, gx, gy, gz);
            }
            // 4-value butterfly; lanes 0..3 hold phi, gx, gy, gz
            const bool b1 = lane & 1;
            double k0v = b1 ? gx : phi, k1v = b1 ? gz : gy;
            k0v += __shfl_xor_sync(0xffffffffu, b1 ? phi : gx, 1);
            k1v += __shfl_xor_sync(0xffffffffu, b1 ? gy : gz, 1);
            const bool b2 = lane & 2;
            double kk = b2 ? k1v : k0v;
            kk += __shfl_xor_sync(0xffffffffu, b2 ? k0v : k1v, 2);
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) kk += __shfl_xor_sync(0xffffffffu, kk, o);
            if (lane < 4) {
                double* o = reinterpret_cast<double*>(&a.out[it]);
                o[lane] = sbeg == 0 ? kk : o[lane] + kk;
            }
            __syncwarp();
        }
    }
}

}  // namespace sog

namespace sog {

// fp32 mode (c4 at tol 1e-4, parity bar 1e-5): the staged cell-relative fp32 coordinates are
// the evaluation coordinates; F(u) from the same table rounded to fp32, 1/r by rsqrtf, lane
// partial sums in fp32, the warp reduction in fp64.
template <int D>
__global__ void __launch_bounds__(32 * NEAR3_WARPS) k_near3f(Near3Args a) {
    extern __shared__ __align__(16) float smf[];
    float* tab = smf;                                                   // [K*(D+1)]
    int* lists = reinterpret_cast<int*>(smf + ((a.K * (D + 1) + 3) & ~3));   // [warps][160]
    float4* src = reinterpret_cast<float4*>(lists + NEAR3_WARPS * 160);      // [cap]: rel. xyz + q
    const CellGeo& g = a.g;
    const int c = blockIdx.x;
    const int cz = c % g.ncz, cy = (c / g.ncz) % g.ncy, cx = c / (g.ncz * g.ncy);
    const int t0 = a.start[c], t1 = a.start[c + 1];
    if (t0 == t1) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int t = threadIdx.x; t < a.K * (D + 1); t += blockDim.x) tab[t] = (float)a.cF[t];
    const double ox = g.x0 + cx / g.sx, oy = cy / g.sy - 0.5 * g.Ly, oz = cz / g.sz - 0.5 * g.Lz;
    const int z0 = max(0, cz - g.nzr), z1 = min(g.ncz - 1, cz + g.nzr);
    int* wl = lists + warp * 160;
    int ns_total = 0;
    for (int k = 0; k < 9; ++k) {
        int nx = cx + k / 3 - 1, ny = cy + k % 3 - 1;
        if (!g.px && (nx < 0 || nx >= g.ncx)) continue;
        nx += nx < 0 ? g.ncx : 0; nx -= nx >= g.ncx ? g.ncx : 0;
        ny += ny < 0 ? g.ncy : 0; ny -= ny >= g.ncy ? g.ncy : 0;
        const int cb = (nx * g.ncy + ny) * g.ncz;
        ns_total += a.start[cb + z1 + 1] - a.start[cb + z0];
    }
    const float rc2 = (float)a.rc2, du = (float)a.du, inv_du = (float)a.inv_du;
    for (int sbeg = 0; sbeg < ns_total; sbeg += a.cap) {
        const int send = min(ns_total, sbeg + a.cap);
        __syncthreads();
        {
            int base = 0;
            for (int k = 0; k < 9; ++k) {
                const int ux = cx + k / 3 - 1, uy = cy + k % 3 - 1;
                if (!g.px && (ux < 0 || ux >= g.ncx)) continue;
                const int nx = ux < 0 ? ux + g.ncx : (ux >= g.ncx ? ux - g.ncx : ux);
                const int ny = uy < 0 ? uy + g.ncy : (uy >= g.ncy ? uy - g.ncy : uy);
                const double sx = !g.px ? 0.0 : (ux < 0 ? -g.Lx : (ux >= g.ncx ? g.Lx : 0.0));
                const double sy = uy < 0 ? -g.Ly : (uy >= g.ncy ? g.Ly : 0.0);
                const int cb = (nx * g.ncy + ny) * g.ncz;
                const int jb = a.start[cb + z0], n = a.start[cb + z1 + 1] - jb;
                const int lo = max(sbeg, base), hi = min(send, base + n);
                for (int q = lo + threadIdx.x; q < hi; q += blockDim.x) {
                    const d4 s = ld_d4(&a.pos[jb + (q - base)]);
                    src[q - sbeg] = make_float4((float)(s.x + sx - ox), (float)(s.y + sy - oy), (float)(s.z - oz),
                                                (float)s.w);
                }
                base += n;
            }
        }
        __syncthreads();
        const int nsrc = send - sbeg;
        for (int it = t0 + warp; it < t1; it += NEAR3_WARPS) {
            const d4 pi = ld_d4(&a.pos[it]);
            const float xi = (float)(pi.x - ox), yi = (float)(pi.y - oy), zi = (float)(pi.z - oz);
            float phi = 0.f, gx = 0.f, gy = 0.f, gz = 0.f;
            int npend = 0;
            auto pair = [&](int q) {
                const float4 s = src[q];
                const float dx = xi - s.x, dy = yi - s.y, dz = zi - s.z;
                const float u = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                if (!(u < rc2 && u > 0.f)) return;
                const int kk = min(a.K - 1, (int)(u * inv_du));
                const float d = u - (kk + 0.5f) * du;
                const float* cf = tab + kk * (D + 1);
                float F = cf[D], dF = 0.f;
#pragma unroll
                for (int n = D - 1; n >= 0; --n) {
                    dF = fmaf(dF, d, F);
                    F = fmaf(F, d, cf[n]);
                }
                const float rinv = rsqrtf(u);
                phi = fmaf(s.w, rinv - F, phi);
                const float cc = s.w * (-rinv * rinv * rinv - 2.f * dF);
                gx = fmaf(cc, dx, gx);
                gy = fmaf(cc, dy, gy);
                gz = fmaf(cc, dz, gz);
            };
            for (int q0 = 0; q0 < nsrc; q0 += 128) {
                bool pass[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int q = q0 + 32 * r + lane;
                    pass[r] = false;
                    if (q < nsrc) {
                        const float4 s = src[q];
                        const float dx = xi - s.x, dy = yi - s.y, dz = zi - s.z;
                        pass[r] = fmaf(dx, dx, fmaf(dy, dy, dz * dz)) < rc2;
                    }
                }
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const unsigned m = __ballot_sync(0xffffffffu, pass[r]);
                    if (pass[r]) wl[npend + __popc(m & ((1u << lane) - 1))] = q0 + 32 * r + lane;
                    npend += __popc(m);
                }
                __syncwarp();
                while (npend >= 32) {
                    npend -= 32;
                    pair(wl[npend + lane]);
                }
                __syncwarp();
            }
            if (lane < npend) pair(wl[lane]);
            double p = phi, x = gx, y = gy, z = gz;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                p += __shfl_xor_sync(0xffffffffu, p, o);
                x += __shfl_xor_sync(0xffffffffu, x, o);
                y += __shfl_xor_sync(0xffffffffu, y, o);
                z += __shfl_xor_sync(0xffffffffu, z, o);
            }
            if (lane == 0) {
                if (sbeg == 0) st_d4(&a.out[it], d4{p, x, y, z});
                else {
                    d4 o = a.out[it];
                    st_d4(&a.out[it], d4{o.x + p, o.y + x, o.z + y, o.w + z});
                }
            }
            __syncwarp();
        }
    }
}

}  // namespace sog
