// S2 v5: near-field pair sum (Eq. eq::phiNDR) over each pair once (Newton's third law:
// the pair kernel 1/r - F(r^2) is symmetric, so the term q_j G(r_ij) of phi_i and q_i G(r_ij) of
// phi_j share one evaluation of F, F' and 1/r; the gradients are opposite up to the charges).
//
// One CTA per near cell c.  Its sources are the cell itself (pairs i < j only) and the 13 cells of
// the forward half shell (dx, dy, dz) > 0 lexicographically: e = 1..9 are (+1, dy, dz), e = 10..12
// (0, +1, dz), e = 13 (0, 0, +1).  Every unordered pair of near cells within reach is visited by
// exactly one CTA (>= 3 cells per periodic axis, so c + e and c - e are distinct images).
//
// The staged sources are split over the 4 warps in 128-blocks (block b belongs to warp b mod 4), and
// every warp sweeps all targets of the cell against its own blocks: the fp32 pre-test (packed
// fp32x2, as k_near3) compacts passing pairs into the warp's list, 32 pairs are evaluated at a time,
// the target side is reduced over the lanes, and the source side is added to the source's
// accumulator in shared memory (the warp owns the block, and the sources of one batch are distinct,
// so no two lanes or warps ever update one accumulator at the same time).  Every sum runs in a fixed
// order: the result is deterministic.
//
// Outputs, sorted order: out[j] = (self-cell source side) + sum over warps of the target side for the
// particles of c, part[j][e-1] = the source side that the CTA of cell (cell of j) - e computed for j
// (zero where that cell does not exist).  k_near_fold adds the 13 slots to out.
#pragma once
#include "kernels_near3.cuh"

namespace sog {

constexpr int NEAR5_WARPS = 4;
constexpr int NEAR5_TMAX = 64;     // targets per chunk (cells with more run in chunks)
constexpr int NEAR5_LIST = 160;    // pending pairs per warp: < 32 carried + 128 from one block
constexpr int NEAR5_SLOTS = 13;

struct Near5Args {
    const d4* pos;          // sorted (x, y, z, q)
    const int* start;       // cell start offsets [ncell + 1]
    d4* out;                // [N] near (phi, grad) before the fold
    d4* part;               // [N][13] forward-shell source-side partials
    double rc2;
    float rc2f;             // conservative fp32 pre-test threshold
    CellGeo g;
    int cap;                // staged sources per piece (multiple of 128)
};

__host__ __device__ constexpr size_t near5_smem(int cap) {
    return 256 + sizeof(int) * NEAR5_WARPS * NEAR5_LIST + sizeof(double) * NEAR5_WARPS * NEAR5_TMAX * 4 +
           (sizeof(d4) + 16) * (size_t)cap;
}

// (dx, dy, dz) of forward slot e (0 = the cell itself)
__device__ __forceinline__ void near5_offset(int e, int& dx, int& dy, int& dz) {
    if (e == 0) { dx = 0; dy = 0; dz = 0; }
    else if (e <= 9) { dx = 1; dy = (e - 1) / 3 - 1; dz = (e - 1) % 3 - 1; }
    else if (e <= 12) { dx = 0; dy = 1; dz = e - 11; }
    else { dx = 0; dy = 0; dz = 1; }
}

template <int PD>
__global__ void __launch_bounds__(32 * NEAR5_WARPS) k_near5(Near5Args a, NearPolyArg<PD> poly) {
    extern __shared__ __align__(32) unsigned char sm5[];
    double2* shift = reinterpret_cast<double2*>(sm5);                              // [14]
    int* lists = reinterpret_cast<int*>(sm5 + 256);                                 // [warps][LIST]
    double* tacc = reinterpret_cast<double*>(lists + NEAR5_WARPS * NEAR5_LIST);     // [warps][TMAX][4]
    d4* sacc = reinterpret_cast<d4*>(tacc + NEAR5_WARPS * NEAR5_TMAX * 4);          // [cap]
    // staged sources in 64-wide blocks (k_near3's packed layout): candidate q = 64 b + 32 h + l
    float4* sxy = reinterpret_cast<float4*>(sacc + a.cap);                          // [cap/64][32]
    float2* sz = reinterpret_cast<float2*>(sxy + a.cap / 2);
    int2* sc = reinterpret_cast<int2*>(sz + a.cap / 2);
    float* sxyf = reinterpret_cast<float*>(sxy);
    float* szf = reinterpret_cast<float*>(sz);
    int* scf = reinterpret_cast<int*>(sc);
    const CellGeo& g = a.g;
    const int c = blockIdx.x;
    const int cz = c % g.ncz, cy = (c / g.ncz) % g.ncy, cx = c / (g.ncz * g.ncy);
    const int t0 = a.start[c], nself = a.start[c + 1] - t0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 14) {
        int dx, dy, dz;
        near5_offset(tid, dx, dy, dz);
        const int ux = cx + dx, uy = cy + dy;
        shift[tid] = make_double2(ux >= g.ncx ? g.Lx : 0.0, uy < 0 ? -g.Ly : (uy >= g.ncy ? g.Ly : 0.0));
    }
    // own particles' slots whose writer cell (own cell - e) lies outside the z range: zero
    if (cz == 0 || cz == g.ncz - 1) {
        for (int t = tid; t < nself * NEAR5_SLOTS; t += blockDim.x) {
            const int i = t / NEAR5_SLOTS, e = t - i * NEAR5_SLOTS + 1;
            int dx, dy, dz;
            near5_offset(e, dx, dy, dz);
            const int bz = cz - dz;
            if (bz < 0 || bz >= g.ncz) st_d4(&a.part[(size_t)(t0 + i) * NEAR5_SLOTS + e - 1], d4{0.0, 0.0, 0.0, 0.0});
        }
    }
    // the 14 source cells: sorted range [cell start, + n) (n = 0 outside the z range)
    auto src_cell = [&](int e, int& jb) {
        int dx, dy, dz;
        near5_offset(e, dx, dy, dz);
        const int uz = cz + dz;
        if (uz < 0 || uz >= g.ncz) { jb = 0; return 0; }
        int nx = cx + dx, ny = cy + dy;
        nx -= nx >= g.ncx ? g.ncx : 0;
        ny += ny < 0 ? g.ncy : 0;
        ny -= ny >= g.ncy ? g.ncy : 0;
        const int cc = (nx * g.ncy + ny) * g.ncz + uz;
        jb = a.start[cc];
        return a.start[cc + 1] - jb;
    };
    int ns_total = 0;
    for (int e = 0; e < 14; ++e) {
        int jb;
        ns_total += src_cell(e, jb);
    }
    const double ox = g.x0 + cx / g.sx, oy = cy / g.sy - 0.5 * g.Ly, oz = cz / g.sz - 0.5 * g.Lz;
    auto put = [&](int q, float x, float y, float z, int code) {
        const int b = q >> 6, h = (q >> 5) & 1, l = q & 31, e = b * 32 + l;
        sxyf[4 * e + h] = x;
        sxyf[4 * e + 2 + h] = y;
        szf[2 * e + h] = z;
        scf[2 * e + h] = code;
    };
    auto code_of = [&](int q) { return scf[2 * ((q >> 6) * 32 + (q & 31)) + ((q >> 5) & 1)]; };
    const float rc2f = a.rc2f;
    int* wl = lists + warp * NEAR5_LIST;
    double* tw = tacc + warp * NEAR5_TMAX * 4;
    for (int tb = 0; tb == 0 || tb < nself; tb += NEAR5_TMAX) {            // target chunks (usually one)
        const int te = min(nself, tb + NEAR5_TMAX);
        for (int t = tid; t < NEAR5_WARPS * NEAR5_TMAX * 4; t += blockDim.x) tacc[t] = 0.0;
        for (int sbeg = 0; sbeg < ns_total || sbeg == 0; sbeg += a.cap) {  // source pieces (usually one)
            const int send = min(ns_total, sbeg + a.cap);
            const int nsrc = send - sbeg, npad = (nsrc + 127) & ~127;
            __syncthreads();
            {
                int base = 0;
                for (int e = 0; e < 14; ++e) {
                    int jb;
                    const int n = src_cell(e, jb);
                    const double2 sh = shift[e];
                    const int lo = max(sbeg, base), hi = min(send, base + n);
                    for (int q = lo + tid; q < hi; q += blockDim.x) {
                        const int j = jb + (q - base);
                        const d4 s = ld_d4(&a.pos[j]);
                        put(q - sbeg, (float)(s.x + sh.x - ox), (float)(s.y + sh.y - oy), (float)(s.z - oz), (j << 4) | e);
                    }
                    base += n;
                }
                for (int q = nsrc + tid; q < npad; q += blockDim.x) put(q, 1e18f, 0.f, 0.f, 0);   // sentinels
                for (int q = tid; q < nsrc; q += blockDim.x) st_d4(&sacc[q], d4{0.0, 0.0, 0.0, 0.0});
            }
            __syncthreads();
            const int nblk = npad >> 7;
            if (warp < nblk) {
                for (int i = tb; i < te; ++i) {
                    const d4 pi = ld_d4(&a.pos[t0 + i]);
                    const float xi = (float)(pi.x - ox), yi = (float)(pi.y - oy), zi = (float)(pi.z - oz);
                    const float2 xi2 = make_float2(xi, xi), yi2 = make_float2(yi, yi), zi2 = make_float2(zi, zi);
                    const float2 m1 = make_float2(-1.f, -1.f);
                    const int qmin = i - sbeg;        // self cell: sources with staged index > i only
                    double phi = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
                    int npend = 0;
                    // one pair (target i, staged source q): both sides
                    auto pair = [&](int q) {
                        const int code = code_of(q);
                        const d4 s = ld_d4(&a.pos[code >> 4]);
                        const double2 sh = shift[code & 15];
                        const double dx = pi.x - (s.x + sh.x), dy = pi.y - (s.y + sh.y), dz = pi.z - s.z;
                        const double u = fma(dx, dx, fma(dy, dy, dz * dz));
                        if (!(u < a.rc2 && u > 0.0)) return;    // exact fp64 decision
                        double F, dF;
                        poly(u, F, dF);
                        const double rinv = rsqrt(u);
                        const double G = rinv - F;
                        const double cc = -rinv * rinv * rinv - 2.0 * dF;
                        phi = fma(s.w, G, phi);
                        const double ct = s.w * cc;
                        gx = fma(ct, dx, gx);
                        gy = fma(ct, dy, gy);
                        gz = fma(ct, dz, gz);
                        const double cs = -pi.w * cc;
                        double2* sa = reinterpret_cast<double2*>(&sacc[q]);
                        double2 v0 = sa[0], v1 = sa[1];
                        v0.x = fma(pi.w, G, v0.x);
                        v0.y = fma(cs, dx, v0.y);
                        v1.x = fma(cs, dy, v1.x);
                        v1.y = fma(cs, dz, v1.y);
                        sa[0] = v0;
                        sa[1] = v1;
                    };
                    for (int b = warp; b < nblk; b += NEAR5_WARPS) {
                        const int q0 = b << 7;
                        bool pass[4];
                        int qq[4];
#pragma unroll
                        for (int r = 0; r < 2; ++r) {
                            const int e = (q0 >> 6) * 32 + r * 32 + lane;
                            const float4 xy = sxy[e];
                            const float2 zz = sz[e];
                            const float2 dx = __ffma2_rn(make_float2(xy.x, xy.y), m1, xi2);
                            const float2 dy = __ffma2_rn(make_float2(xy.z, xy.w), m1, yi2);
                            const float2 dz = __ffma2_rn(zz, m1, zi2);
                            const float2 r2 = __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __fmul2_rn(dz, dz)));
                            qq[2 * r] = q0 + 64 * r + lane;
                            qq[2 * r + 1] = q0 + 64 * r + 32 + lane;
                            pass[2 * r] = r2.x < rc2f && qq[2 * r] > qmin;
                            pass[2 * r + 1] = r2.y < rc2f && qq[2 * r + 1] > qmin;
                        }
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            const unsigned m = __ballot_sync(0xffffffffu, pass[r]);
                            if (pass[r]) wl[npend + __popc(m & ((1u << lane) - 1))] = qq[r];
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
                    __syncwarp();
                    const bool b1 = lane & 1;
                    double k0v = b1 ? gx : phi, k1v = b1 ? gz : gy;
                    k0v += __shfl_xor_sync(0xffffffffu, b1 ? phi : gx, 1);
                    k1v += __shfl_xor_sync(0xffffffffu, b1 ? gy : gz, 1);
                    const bool b2 = lane & 2;
                    double kk = b2 ? k1v : k0v;
                    kk += __shfl_xor_sync(0xffffffffu, b2 ? k0v : k1v, 2);
#pragma unroll
                    for (int o = 4; o < 32; o <<= 1) kk += __shfl_xor_sync(0xffffffffu, kk, o);
                    if (lane < 4) tw[(i - tb) * 4 + lane] += kk;
                }
            }
            __syncthreads();
            // source side of this piece: self sources into out (first chunk: =), forward ones into part
            for (int t = tid; t < 4 * nsrc; t += blockDim.x) {
                const int q = t >> 2, k = t & 3;
                const int code = code_of(q);
                const int e = code & 15, j = code >> 4;
                const double v = reinterpret_cast<const double*>(&sacc[q])[k];
                double* o = e == 0 ? reinterpret_cast<double*>(&a.out[j]) + k
                                   : reinterpret_cast<double*>(&a.part[(size_t)j * NEAR5_SLOTS + e - 1]) + k;
                *o = tb == 0 ? v : *o + v;
            }
        }
        __syncthreads();
        // target side of the chunk, warps in a fixed order
        for (int t = tid; t < 4 * (te - tb); t += blockDim.x) {
            const int i = t >> 2, k = t & 3;
            double v = tacc[i * 4 + k];
#pragma unroll
            for (int w = 1; w < NEAR5_WARPS; ++w) v += tacc[w * NEAR5_TMAX * 4 + i * 4 + k];
            double* o = reinterpret_cast<double*>(&a.out[t0 + tb + i]) + k;
            *o += v;
        }
        __syncthreads();
    }
}

// out[j] += sum_e part[j][e], e = 0..12 in order (sorted order, one thread per particle component)
template <int S = NEAR5_SLOTS>
__global__ void __launch_bounds__(256) k_near_fold(d4* __restrict__ out, const d4* __restrict__ part, int N) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 4LL * N) return;
    const int j = (int)(t >> 2), k = (int)(t & 3);
    const double* p = reinterpret_cast<const double*>(part + (size_t)j * S) + k;
    double v = reinterpret_cast<const double*>(out + j)[k];
#pragma unroll
    for (int e = 0; e < S; ++e) v += __ldg(p + 4 * e);
    reinterpret_cast<double*>(out + j)[k] = v;
}

}  // namespace sog
