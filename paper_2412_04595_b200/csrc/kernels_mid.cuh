// Mid-range Fourier spectral solver (Algorithm 1), B200 v3.
//   S3 gridding  S[g] = sum_j q_j W(x_g-x_j)_* W(y_g-y_j)_* W(z_g-z_j)   (Eq. eq::gridding)
//   S5 scaling   S_hat <- mult(k) S_hat                                  (Eq. eq::widehat-tilde)
//   S7 gathering phi_i = V_h sum_g W W W Psi[g] (+ gradient with W')     (Eq. eq::Phiconv)
//
// Grid layout (z slowest, y fastest): real [Izs][Ix][Iy]; half spectrum [Izs][Ix][Iy/2+1].
//
// Particle order for the mid stencils ("mid order"): bucketed by the key
//   key = (tx * nty + ty) * nzc + zc,  tx = s_x / MZ_TX, ty = s_y / MZ_TY, zc = s_z / MZ_ZC,
// where s = g0 - p is the stencil start (x, y wrapped into [0, I)).  Buckets are ordered by
// cell-sorted index inside (deterministic).  A CTA of the spread owns an MZ_TX x MZ_TY
// column tile and sweeps z chunk by chunk, every lane holding MZ_ZC + P - 1 consecutive z
// values of its column in registers (a sliding window): each particle adds P fused
// multiply-adds per touched column, and every grid point is written exactly once.
#pragma once
#include <cuComplex.h>
#include <type_traits>
#include <utility>
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

constexpr int MZ_TX = 16, MZ_TY = 16, MZ_ZC = 4;

// v mod n for v in (-2n, 2n) without integer division
__device__ __forceinline__ int wrapc(int v, int n) {
    v += v < 0 ? n : 0;
    v += v < 0 ? n : 0;
    v -= v >= n ? n : 0;
    v -= v >= n ? n : 0;
    return v;
}

// ---------------------------------------------------------------------------------------
// Mid-order bucket sort (part of S1).  k_mid_key -> scan -> k_mid_scatter -> k_mid_bucket.
struct MidSortArgs {
    int Ix, Iy, p, nty, nzc;
    int px, xorig;          // x periodic (whole box) or x-slab: local start = s_x - xorig (no wrap)
};

static __global__ void k_mid_key(const int4* __restrict__ g0, int N, MidSortArgs s, int* __restrict__ key,
                                 int* __restrict__ count) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N) return;
    const int4 o = g0[j];
    const int sx = s.px ? wrapc(o.x - s.p, s.Ix) : o.x - s.p - s.xorig, sy = wrapc(o.y - s.p, s.Iy), sz = o.z - s.p;
    SOG_ASSERT(sx >= 0 && sy >= 0 && sz >= 0);
    const int k = ((sx / MZ_TX) * s.nty + sy / MZ_TY) * s.nzc + sz / MZ_ZC;
    key[j] = k;
    atomicAdd(&count[k], 1);
}

static __global__ void k_mid_scatter(const int* __restrict__ key, int N, int* __restrict__ cursor,
                                     int* __restrict__ tmp) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < N) tmp[atomicAdd(&cursor[key[j]], 1)] = j;
}

// One warp per bucket: order members by cell-sorted index (deterministic), gather the
// particle and its unwrapped stencil starts into mid order.
static __global__ void k_mid_bucket(const int* __restrict__ mstart, int nkeys, const int* __restrict__ tmp,
                                    const d4* __restrict__ pos_s, const int4* __restrict__ g0, int p,
                                    d4* __restrict__ mpos, int4* __restrict__ minfo) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= nkeys) return;
    const int s = mstart[warp], n = mstart[warp + 1] - s;
    for (int e = lane; e < n; e += 32) {
        const int my = tmp[s + e];
        int rank = 0;
        if (n <= 2048) {
            for (int f = 0; f < n; ++f) rank += (tmp[s + f] < my);
        } else {
            rank = e;   // pathological clustering: arrival order
        }
        const int4 o = g0[my];
        st_d4(&mpos[s + rank], ld_d4(&pos_s[my]));
        minfo[s + rank] = make_int4(my, o.x - p, o.y - p, o.z - p);
    }
}

// ---------------------------------------------------------------------------------------
struct MidZArgs {
    int Ix, Iy, Izs;
    double hx, hy, hz, halfx, halfy, halfz;
    double invH2Sx, invH2Sy, invH2Sz, Vh;
    double gamma_x, gamma_y, gamma_z;     // window recurrence constants exp(-2 a h^2)
    int ntx, nty, nzc;                    // key space
    int c_lo, c_hi;                       // chunks that can hold stencil starts
    int c_hiw;                            // last chunk with nonzero planes (spread writes [c_lo, c_hiw])
    int cps;                              // chunks per CTA z segment
    int px, xorig, Ixk;                   // x periodic, or x-slab: local x = global - xorig, extent Ixk
    int tlo, ntout;                       // x tiles processed: [tlo, tlo + ntout)
    const d4* mpos;
    const int4* minfo;                    // (cell-sorted index, s_x, s_y, s_z) unwrapped starts
    const int* mstart;                    // [ntx*nty*nzc + 1]
    int kb;                               // 1: Kaiser-Bessel window (R6-KB), table kt
    KBTab kt;
};

// spread record in shared memory: [q Wx (P)] [Wy (P)] [Wz placed at offset o = s_z - chunk
// base inside the NACC-slot z window, zeros elsewhere (even length)] [hdr int4: dx, dy, -,
// chunk].  dx, dy are the stencil start relative to the tile origin: signed in [-(P-1),
// MZ_TX) when the window does not wrap onto itself, else mod I.
//
// MMA variant (fp64, k_mid_spread_zm, NP producer warps): the Wz slots form a ring of S = 8 NTZ planes,
// plane g stored at slot g mod S (S >= NACC, so the planes live in one chunk's window never collide).
template <int P, typename T = double, int NP = 0>
struct SRec {
    static constexpr bool M = NP > 0;
    static constexpr int AL = 16 / int(sizeof(T));         // elements per 16 bytes
    static constexpr int NACC = MZ_ZC + P - 1;             // register window per lane (z planes)
    static constexpr int NTZ = (NACC + 7) / 8;             // MMA: z n-tiles of 8 planes
    static constexpr int S = 8 * NTZ;                      // MMA: ring slots
    static constexpr int NZP = M ? S : (NACC + 1) & ~1;    // padded Wz slots
    // MMA: q Wx sits between XPAD zeros on each side (a 4-row patch reads 4 consecutive slots from
    // its first row's offset, in [-3, P - 1], without bounds selects)
    static constexpr int XPAD = M ? 3 : 0;
    static constexpr int WX = XPAD, WY = P + 2 * XPAD, WZ = ((WY + P + AL - 1) / AL) * AL;
    static constexpr int HDR = ((WZ + NZP + AL - 1) / AL) * AL;   // int4 header, 16-byte aligned
    static constexpr int SIZE = HDR + AL;
    static constexpr int NPROD = M ? NP : 2;               // producer warps (32 particles each)
    static constexpr int B = 32 * NPROD;                   // particles per staged batch
    static constexpr int K = M ? (NPROD <= 2 ? 4 : 2) : SIZE * int(sizeof(T)) <= 48 * 8 ? 4 : 2;   // batch buffers in flight
    static constexpr int EMAX = 1024;                      // (chunk, home tile) ranges per CTA
    static constexpr int NTHR = 32 * (8 + NPROD);
    static constexpr int MINB = P <= 15 || sizeof(T) == 4 ? 2 : 1;   // CTAs per SM (register budget)
    static constexpr size_t BYTES = sizeof(T) * K * B * SIZE + sizeof(int) * (2 * EMAX + 1);
};

// mbarrier helpers (shared::cta)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}

// lane flush of one chunk's MZ_ZC planes (written only for c >= cb), then slide the window
template <int P, typename T>
__device__ __forceinline__ void spread_flush(T (&acc)[SRec<P, T>::NACC], int c, int cb, bool colok, int cx, int cy,
                                             const MidZArgs& a, T* __restrict__ grid) {
    if (c >= cb && colok) {
#pragma unroll
        for (int z = 0; z < MZ_ZC; ++z) {
            const int plane = c * MZ_ZC + z;
            SOG_ASSERT(cx < a.Ixk && cy < a.Iy);
            if (plane < a.Izs) grid[((size_t)plane * a.Ixk + cx) * a.Iy + cy] = acc[z];
        }
    }
#pragma unroll
    for (int i = 0; i < SRec<P, T>::NACC; ++i) acc[i] = i + MZ_ZC < SRec<P, T>::NACC ? acc[i + MZ_ZC] : T(0);
}

// Warp-specialised: NPROD producer warps stage the CTA's candidate stream (weights, relevance
// masks) into K batch buffers; 8 consumer warps (one 4 x 8 column patch each) accumulate
// their patch's particles.  full/empty mbarriers let consumer warps drift up to K batches
// apart, so the per-batch imbalance between patches averages out.
//
// M = true (fp64): the consumer warp's accumulation is a sequence of DMMA products.  For a group
// of 4 same-chunk particles (k = particle), the patch update is, per x row m of the patch,
//   C_m[y][s] += sum_k A_m[y][k] B[k][s],  A_m[y][k] = q Wx_k(x_m) Wy_k(y),  B[k][s] = Wz_k(plane of slot s)
// (Eq. eq::gridding as a rank-4 update), y = the 8 patch columns of the row, s = the NTZ x 8 ring
// slots: 4 NTZ mma.sync per group, the operands one Wy, four Wx and NTZ Wz loads per lane.  A
// chunk's 4 planes (slots 4 (c mod S/4) + 0..3) are written and cleared when the sweep leaves it.
template <int P, typename T, bool KB, int NP>
__device__ __forceinline__ void mid_spread_body(const MidZArgs& a, T* __restrict__ grid) {
    using R = SRec<P, T, NP>;
    constexpr bool M = R::M;
    using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
    constexpr int p = (P - 1) / 2, NACC = R::NACC, B = R::B, K = R::K, EMAX = R::EMAX;
    extern __shared__ __align__(16) unsigned char smraw[];
    T* sRec = reinterpret_cast<T*>(smraw);      // [K][B][SIZE], then sPre[EMAX+1], sBeg[EMAX]
    int* sPre = reinterpret_cast<int*>(sRec + K * B * R::SIZE);
    int* sBeg = sPre + EMAX + 1;
    __shared__ unsigned short sList[M ? 1 : 8][M ? 1 : B];
    // MMA: per-warp particle list, (dx + 512 | (dy + 512) << 10 | record << 20, chunk)
    __shared__ int2 sEnt[M ? 8 : 1][M ? B : 1];
    __shared__ unsigned char sMask[K][B];
    __shared__ unsigned long long barFull[K], barEmpty[K];
    __shared__ int sHx[8], sHy[8], sNh[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tx = a.tlo + blockIdx.x / a.nty, ty = blockIdx.x % a.nty;
    const int X0 = tx * MZ_TX, Y0 = ty * MZ_TY;
    // z segment: written chunks [cb, ce), sweep from cs (warm-up chunks are not written)
    const int cb = a.c_lo + blockIdx.y * a.cps;
    const int ce = min(cb + a.cps, a.c_hiw + 1);
    if (cb >= ce) return;
    const int cs = max(a.c_lo, cb - (P - 2 + MZ_ZC) / MZ_ZC);
    const int cp1 = min(ce, a.c_hi + 1);                 // chunks [cs, cp1) hold particles
    const bool smallx = a.px && (MZ_TX + P - 1 > a.Ix), smally = MZ_TY + P - 1 > a.Iy;
    // home tiles whose particles can reach this tile (starts in [X0 - P + 1, X0 + TX - 1])
    if (tid == 0) {
        int n = 0;
        if (!a.px) {
            for (int h = max(0, (X0 - (P - 1)) / MZ_TX); h <= tx && n < 8; ++h) sHx[n++] = h;
        } else if (MZ_TX + P - 1 >= a.Ix) {
            for (int h = 0; h < a.ntx && n < 8; ++h) sHx[n++] = h;
        } else {
            int h = wrapc(X0 - (P - 1), a.Ix) / MZ_TX;
            for (;;) { sHx[n++] = h; if (h == tx || n == 8) break; h = h + 1 == a.ntx ? 0 : h + 1; }
        }
        sNh[0] = n;
        n = 0;
        if (MZ_TY + P - 1 >= a.Iy) {
            for (int h = 0; h < a.nty && n < 8; ++h) sHy[n++] = h;
        } else {
            int h = wrapc(Y0 - (P - 1), a.Iy) / MZ_TY;
            for (;;) { sHy[n++] = h; if (h == ty || n == 8) break; h = h + 1 == a.nty ? 0 : h + 1; }
        }
        sNh[1] = n;
        for (int b = 0; b < K; ++b) {
            mbar_init(&barFull[b], 32 * R::NPROD);
            mbar_init(&barEmpty[b], 8 * 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int nhx = sNh[0], nhy = sNh[1], nh = nhx * nhy;
    // candidate stream: for chunk c in [cs, cp1), for home tile h: mid-order range (c, h)
    const int E = max(0, min(EMAX, (cp1 - cs) * nh));
    for (int e = tid; e < E; e += R::NTHR) {
        const int c = cs + e / nh, h = e % nh;
        const int k = (sHx[h / nhy] * a.nty + sHy[h % nhy]) * a.nzc + c;
        SOG_ASSERT(k >= 0 && k < a.ntx * a.nty * a.nzc);
        const int b = a.mstart[k];
        sBeg[e] = b;
        sPre[e + 1] = a.mstart[k + 1] - b;
    }
    __syncthreads();
    if (warp == 0) {                                     // inclusive scan of the range lengths
        int run = 0;
        for (int e0 = 0; e0 < E; e0 += 32) {
            int v = e0 + lane < E ? sPre[e0 + lane + 1] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += t;
            }
            if (e0 + lane < E) sPre[e0 + lane + 1] = run + v;
            run += __shfl_sync(0xffffffffu, v, 31);
        }
        if (lane == 0) sPre[0] = 0;
    }
    __syncthreads();
    const int total = sPre[E];
    const int nbat = (total + B - 1) / B;

    if (warp >= 8) {
        // ---------------- producers: one particle per thread per batch ----------------
        const int s = (warp - 8) * 32 + lane;
        // software pipeline: the candidate of batch bi + 1 is located and its (minfo, mpos) loads
        // are in flight while batch bi's weights are computed
        auto locate = [&](int idx, int& c) {
            int lo = 0, hi = E;                          // last e with sPre[e] <= idx
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (sPre[mid] <= idx) lo = mid; else hi = mid;
            }
            c = cs + lo / nh;
            SOG_ASSERT(lo >= 0 && lo < E);
            return sBeg[lo] + (idx - sPre[lo]);
        };
        int4 in_n = make_int4(0, 0, 0, 0);
        d4 r_n{0.0, 0.0, 0.0, 0.0};
        int c_n = 0;
        if (s < total) {
            const int k = locate(s, c_n);
            in_n = a.minfo[k];
            r_n = ld_d4(&a.mpos[k]);
        }
        for (int bi = 0; bi < nbat; ++bi) {
            const int buf = bi % K;
            const int idx = bi * B + s;
            const int4 in = in_n;
            const d4 r = r_n;
            const int c = c_n;
            if (idx + B < total) {
                const int k = locate(idx + B, c_n);
                in_n = a.minfo[k];
                r_n = ld_d4(&a.mpos[k]);
            }
            if (bi >= K) mbar_wait(&barEmpty[buf], ((bi / K) - 1) & 1);
            T* rec = sRec + (buf * B + s) * R::SIZE;
            unsigned mask = 0;
            if (idx < total) {
                SOG_ASSERT(in.w - c * MZ_ZC >= 0 && in.w - c * MZ_ZC < MZ_ZC);
                int dx = a.px ? wrapc(in.y - X0, a.Ix) : in.y - a.xorig - X0, dy = wrapc(in.z - Y0, a.Iy);
                unsigned mx = 0, my = 0;
                if (!smallx) {
                    if (a.px) dx -= dx > a.Ix - P ? a.Ix : 0;   // signed start in [-(P-1), MZ_TX)
#pragma unroll
                    for (int g = 0; g < 4; ++g) mx |= (dx <= 4 * g + 3 && dx + P - 1 >= 4 * g) ? 1u << g : 0u;
                } else {
#pragma unroll
                    for (int g = 0; g < 4; ++g)
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            if (wrapc(4 * g + i - dx, a.Ix) < P) mx |= 1u << g;
                }
                if (!smally) {
                    dy -= dy > a.Iy - P ? a.Iy : 0;
#pragma unroll
                    for (int g = 0; g < 2; ++g) my |= (dy <= 8 * g + 7 && dy + P - 1 >= 8 * g) ? 1u << g : 0u;
                } else {
#pragma unroll
                    for (int g = 0; g < 2; ++g)
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            if (wrapc(8 * g + i - dy, a.Iy) < P) my |= 1u << g;
                }
#pragma unroll
                for (int w = 0; w < 8; ++w)
                    if (((mx >> (w & 3)) & 1) && ((my >> (w >> 2)) & 1)) mask |= 1u << w;
                *reinterpret_cast<int4*>(rec + R::HDR) = make_int4(dx, dy, 0, c);
                if (mask) {
                    // z offset of the stencil in the window (MMA: ring slot of its first plane)
                    const int o = M ? ((in.w % R::S) + R::S) % R::S : in.w - c * MZ_ZC;
                    auto zslot = [&](int i) {
                        int t = o + i;
                        if constexpr (M) t -= t >= R::S ? R::S : 0;
                        return t;
                    };
                    if constexpr (KB) {
                        // one axis at a time (P live weights, no spills at wide supports)
                        double w[P];
                        kb_weights<P, false>(kb_offset(r.x, a.hx, a.halfx, in.y + p), a.kt, w, nullptr);
#pragma unroll
                        for (int i = 0; i < P; ++i) rec[R::WX + i] = T(r.w * w[i]);
#pragma unroll
                        for (int i = 0; i < R::XPAD; ++i) rec[i] = rec[R::WX + P + i] = T(0);
                        kb_weights<P, false>(kb_offset(r.y, a.hy, a.halfy, in.z + p), a.kt, w, nullptr);
#pragma unroll
                        for (int i = 0; i < P; ++i) rec[R::WY + i] = T(w[i]);
#pragma unroll
                        for (int i = 0; i < R::NZP; ++i) rec[R::WZ + i] = T(0);
                        kb_weights<P, false>(kb_offset(r.z, a.hz, a.halfz, in.w + p), a.kt, w, nullptr);
#pragma unroll
                        for (int i = 0; i < P; ++i) rec[R::WZ + zslot(i)] = T(w[i]);
                    } else {
                        double wx[P], wy[P], wz[P];
                        window_weights_rec<P, false>(r.x, in.y + p, a.hx, a.halfx, a.invH2Sx, a.gamma_x, wx, nullptr);
                        window_weights_rec<P, false>(r.y, in.z + p, a.hy, a.halfy, a.invH2Sy, a.gamma_y, wy, nullptr);
                        window_weights_rec<P, false>(r.z, in.w + p, a.hz, a.halfz, a.invH2Sz, a.gamma_z, wz, nullptr);
#pragma unroll
                        for (int i = 0; i < P; ++i) {
                            rec[R::WX + i] = T(r.w * wx[i]);
                            rec[R::WY + i] = T(wy[i]);
                        }
#pragma unroll
                        for (int i = 0; i < R::XPAD; ++i) rec[i] = rec[R::WX + P + i] = T(0);
#pragma unroll
                        for (int i = 0; i < R::NZP; ++i) rec[R::WZ + i] = T(0);
#pragma unroll
                        for (int i = 0; i < P; ++i) rec[R::WZ + zslot(i)] = T(wz[i]);
                    }
                }
            }
            sMask[buf][s] = (unsigned char)mask;
            mbar_arrive(&barFull[buf]);
        }
        return;
    }

    if constexpr (M) {
        // ---------------- consumers (DMMA): warp = one 4 x 8 column patch ----------------
        constexpr int NTZ = R::NTZ, NG = R::S / 4;
        const int gid = lane >> 2, tig = lane & 3;
        const int lx0 = 4 * (warp & 3), ly = 8 * (warp >> 2) + gid, cy = Y0 + ly;
        double C[4][NTZ][2];
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int t = 0; t < NTZ; ++t) C[m][t][0] = C[m][t][1] = 0.0;
        // leave chunk c: its planes sit in n-tile g / 2, lanes tig / 2 == g % 2 (g = c mod NG)
        auto flush = [&](int c) {
            const int g = c % NG, nt = g >> 1;
            const bool mine = (tig >> 1) == (g & 1);
            const bool wr = mine && c >= cb && cy < a.Iy;
            const int pl0 = MZ_ZC * c + 2 * (tig & 1);
#pragma unroll
            for (int t = 0; t < NTZ; ++t) {
                if (t != nt) continue;
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int cx = X0 + lx0 + m;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (wr && cx < a.Ixk && pl0 + h < a.Izs)
                            grid[((size_t)(pl0 + h) * a.Ixk + cx) * a.Iy + cy] = C[m][t][h];
                        if (mine) C[m][t][h] = 0.0;
                    }
                }
            }
        };
        int cur = cs;
        for (int bi = 0; bi < nbat; ++bi) {
            const int buf = bi % K;
            mbar_wait(&barFull[buf], (bi / K) & 1);
            const int nb = min(B, total - bi * B);
            const T* base = sRec + buf * B * R::SIZE;
            // this warp's particles in stream order
            int nmy = 0;
#pragma unroll
            for (int s0 = 0; s0 < B; s0 += 32) {
                const int s = s0 + lane;
                const bool mine = s < nb && ((sMask[buf][s] >> warp) & 1);
                const unsigned bm = __ballot_sync(0xffffffffu, mine);
                if (mine) {
                    const int4 h = *reinterpret_cast<const int4*>(base + s * R::SIZE + R::HDR);
                    SOG_ASSERT(h.x > -512 && h.x < 512 && h.y > -512 && h.y < 512);
                    sEnt[warp][nmy + __popc(bm & ((1u << lane) - 1))] =
                        make_int2((h.x + 512) | ((h.y + 512) << 10) | (s << 20), h.w);
                }
                nmy += __popc(bm);
            }
            __syncwarp();
            // groups of <= 4 same-chunk particles (k = particle)
            const int last = max(nmy - 1, 0);
            // operands of the group starting at gi (entry e of lane tig, chunk gc of its first)
            auto prep = [&](int gi, const int2& e, int gc, double (&am)[4], double (&bz)[NTZ]) {
                const bool valid = gi + tig < nmy && e.y == gc;   // same-chunk prefix of the group
                const int nval = __popc(__ballot_sync(0xffffffffu, valid) & 0xfu);
                const int dx = (e.x & 1023) - 512, dy = ((e.x >> 10) & 1023) - 512;
                const T* rec = base + (e.x >> 20) * R::SIZE;
                const int v = smally ? wrapc(ly - dy, a.Iy) : ly - dy;
                const double wy = rec[R::WY + min((unsigned)v, P - 1u)];
                const double cy0 = valid && (unsigned)v < (unsigned)P ? wy : 0.0;
                if (!smallx) {
                    // rows lx0 .. lx0 + 3 meet the stencil (the patch is touched): u0 in [-3, P - 1]
                    SOG_ASSERT(lx0 - dx >= -R::XPAD && lx0 - dx <= P - 1);
                    const T* wxr = rec + R::WX + (lx0 - dx);
#pragma unroll
                    for (int m = 0; m < 4; ++m) am[m] = wxr[m] * cy0;
                } else {
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        const int u = wrapc(lx0 + m - dx, a.Ix);
                        const double wx = rec[R::WX + min((unsigned)u, P - 1u)];
                        am[m] = (unsigned)u < (unsigned)P ? wx * cy0 : 0.0;
                    }
                }
                // invalid lanes have a zero A column, so their (finite) Wz row adds nothing
#pragma unroll
                for (int t = 0; t < NTZ; ++t) bz[t] = rec[R::WZ + 8 * t + gid];
                return nval;
            };
            auto mma = [&](const double (&am)[4], const double (&bz)[NTZ]) {
#pragma unroll
                for (int m = 0; m < 4; ++m)
#pragma unroll
                    for (int t = 0; t < NTZ; ++t) dmma_884(C[m][t], am[m], bz[t]);
            };
            // (software-pipelining the next group's loads under this group's products measured
            // slower: the extra registers cost occupancy)
            int i = 0;
            while (i < nmy) {                            // warp-uniform
                const int2 e = sEnt[warp][min(i + tig, last)];
                const int c0 = sEnt[warp][i].y;
                double am[4], bz[NTZ];
                const int nval = prep(i, e, c0, am, bz);
                while (cur < c0) {                       // entering a later chunk
                    flush(cur);
                    ++cur;
                }
                mma(am, bz);
                i += nval;
            }
            __syncwarp();
            mbar_arrive(&barEmpty[buf]);
        }
        while (cur < ce) {
            flush(cur);
            ++cur;
        }
        return;
    }
    // ---------------- consumers: warp = one 4 x 8 column patch ----------------
    const int lx = 4 * (warp & 3) + (lane >> 3), ly = 8 * (warp >> 2) + (lane & 7);
    const int cx = X0 + lx, cy = Y0 + ly;
    const bool colok = cx < a.Ixk && cy < a.Iy;
    T acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = T(0);
    int cur = cs;                                        // chunk held in acc[0, MZ_ZC)
    for (int bi = 0; bi < nbat; ++bi) {
        const int buf = bi % K;
        mbar_wait(&barFull[buf], (bi / K) & 1);
        const int nb = min(B, total - bi * B);
        int nmy = 0;                                     // this warp's particles, stream order
#pragma unroll
        for (int s0 = 0; s0 < B; s0 += 32) {
            const int s = s0 + lane;
            const bool mine = s < nb && ((sMask[buf][s] >> warp) & 1);
            const unsigned bm = __ballot_sync(0xffffffffu, mine);
            if (mine) sList[warp][nmy + __popc(bm & ((1u << lane) - 1))] = (unsigned short)s;
            nmy += __popc(bm);
        }
        __syncwarp();
        const T* base = sRec + buf * B * R::SIZE;
        auto coef = [&](const T* rec, const int4& hdr) {
            const int u = smallx ? wrapc(lx - hdr.x, a.Ix) : lx - hdr.x;
            const int v = smally ? wrapc(ly - hdr.y, a.Iy) : ly - hdr.y;
            const bool in = (unsigned)u < (unsigned)P && (unsigned)v < (unsigned)P;
            return in ? rec[R::WX + min((unsigned)u, P - 1u)] * rec[R::WY + min((unsigned)v, P - 1u)] : T(0);
        };
        auto accum = [&](const T* rec, T cc) {
            const V2* w2 = reinterpret_cast<const V2*>(rec + R::WZ);
#pragma unroll
            for (int k = 0; k < R::NZP / 2; ++k) {
                const V2 t = w2[k];
                if (2 * k < NACC) acc[2 * k] = fma(cc, t.x, acc[2 * k]);
                if (2 * k + 1 < NACC) acc[2 * k + 1] = fma(cc, t.y, acc[2 * k + 1]);
            }
        };
        // runs of same-chunk particles, two per step; the chunk flush (a register-window shift)
        // stays outside the run loop so the accumulators keep fixed registers inside it
        int i = 0;
        while (i < nmy) {
            const T* ra = base + sList[warp][i] * R::SIZE;
            int4 ha = *reinterpret_cast<const int4*>(ra + R::HDR);
            while (cur < ha.w) {                         // warp-uniform: entering a later chunk
                spread_flush<P, T>(acc, cur, cb, colok, cx, cy, a, grid);
                ++cur;
            }
            for (;;) {
                const bool two = i + 1 < nmy;
                const T* rb = base + sList[warp][two ? i + 1 : i] * R::SIZE;
                const int4 hb = *reinterpret_cast<const int4*>(rb + R::HDR);
                const bool pair = two && hb.w == cur;
                const T ca = coef(ra, ha);
                const T cbv = pair ? coef(rb, hb) : T(0);   // branch-free: zero weight when unpaired
                i += pair ? 2 : 1;
                // next step's record and header are loaded before this step's FMAs
                const bool more = i < nmy;
                const T* rn = base + sList[warp][more ? i : 0] * R::SIZE;
                const int4 hn = *reinterpret_cast<const int4*>(rn + R::HDR);
                accum(ra, ca);
                accum(rb, cbv);
                if (!more) break;
                ra = rn;
                ha = hn;
                if (ha.w != cur) break;
            }
        }
        __syncwarp();
        mbar_arrive(&barEmpty[buf]);
    }
    while (cur < ce) {
        spread_flush<P, T>(acc, cur, cb, colok, cx, cy, a, grid);
        ++cur;
    }
}

template <int P, typename T = double, bool KB = false>
__global__ void __launch_bounds__(SRec<P, T>::NTHR, SRec<P, T>::MINB) k_mid_spread_z(MidZArgs a, T* __restrict__ grid) {
    mid_spread_body<P, T, KB, 0>(a, grid);
}
// DMMA variant, NP producer warps: 2 CTAs of 8 + NP warps per SM; the register file is split over
// the 4 SM sub-partitions (16384 registers each), so the budget is set for ceil(2 (8 + NP) / 4) warps
// per sub-partition
constexpr int spread_mma_regs(int np) { return 16384 / ((2 * (8 + np) + 3) / 4) / 32 / 8 * 8; }
template <int P, bool KB, int NP>
__global__ void __maxnreg__(spread_mma_regs(NP)) k_mid_spread_zm(MidZArgs a, double* __restrict__ grid) {
    mid_spread_body<P, double, KB, NP>(a, grid);
}

// ---------------------------------------------------------------------------------------
// S7 gather: a CTA owns the particles whose stencil starts lie in its MZ_TX x MZ_TY tile and
// one z segment.  It keeps a ring of Psi planes of the tile window (MZ_TX + P - 1) x
// (MZ_TY + P - 1) in shared memory and advances it chunk by chunk; a warp gathers one
// particle at a time, lanes over the P x P stencil columns (z contracted per lane, then the
// separable x/y weights), and reduces the four values with shuffles.  Three lanes compute
// the particle's separable weights (Gaussian recurrence, one axis each).
template <int P, typename T = double, bool KB = false>
struct GRing {
    static constexpr int WX = MZ_TX + P - 1, WY = MZ_TY + P - 1;
    static constexpr int WYP = WY + ((P - WY) % 16 + 16) % 16;   // row pitch = P (mod 16): conflict-free
    // ring slot stride (elements): holds a WX x WYP window (cp.async rows) or a dense WX x WY TMA box,
    // rounded up to 128 bytes (TMA destinations)
    static constexpr int E128 = 128 / int(sizeof(T));
    static constexpr int PL = ((WX * WYP > WX * WY ? WX * WYP : WX * WY) + E128 - 1) / E128 * E128;
    static constexpr int D = MZ_ZC + P - 1;                       // planes a chunk reads
    static constexpr int DR = D + MZ_ZC;                          // ring: + the next chunk's planes (prefetch)
    static constexpr int AL = 16 / int(sizeof(T));
    // [Wx Wy Wz | W'x W'y W'z] (dW/dx of the particle, R11), then the int4 header
    static constexpr int HOFF = ((6 * P + AL - 1) / AL) * AL;
    static constexpr int WSZ = HOFF + AL;                         // per-particle weight scratch
    static constexpr int WB = 2;                                  // particles per warp batch
    static constexpr int NSEG = 4;                                // Gaussian weights: segments per axis
    static constexpr int SEGL = (P + NSEG - 1) / NSEG;            //   and stencil points per segment
    static constexpr int NR = (P * P + 31) / 32;                  // column rounds per lane
    static constexpr size_t BYTES = sizeof(T) * (size_t(DR) * PL + 8 * WB * WSZ);
    static constexpr bool FITS = BYTES <= 227 * 1024;
    static constexpr int MINB = BYTES <= 112 * 1024 ? 2 : 1;     // CTAs per SM
};

__device__ __forceinline__ void cp_async8(void* dst_smem, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst_smem)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst_smem, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst_smem)), "l"(src) : "memory");
}
// shared-memory load from a 32-bit shared address (one 3-input add per address, no re-materialised
// products)
__device__ __forceinline__ double lds_t(unsigned a, double) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ float lds_t(unsigned a, float) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}

// shared-memory load at a compile-time byte offset from a 32-bit shared address (one LDS with an
// immediate offset, no address add)
template <int OFF>
__device__ __forceinline__ double lds_off(unsigned a, double) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(a), "n"(OFF));
    return v;
}
template <int OFF>
__device__ __forceinline__ float lds_off(unsigned a, float) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(a), "n"(OFF));
    return v;
}
// t0 += wz[kz] Psi[kz], t1 += dwz[kz] Psi[kz] over kz = 0..P-1 at plane stride PLB bytes
template <int PLB, typename T, int... KZ>
__device__ __forceinline__ void zcontract(unsigned a, const T* wz, const T* dwz, T& t0, T& t1,
                                          std::integer_sequence<int, KZ...>) {
    ((t0 = fma(wz[KZ], lds_off<KZ * PLB>(a, T(0)), t0),
      t1 = fma(dwz[KZ], lds_off<KZ * PLB>(a, T(0)), t1)), ...);
}

// the same for a particle whose planes wrap around the ring: planes kz < N1 sit at the slots after
// its first one (base a1), planes kz >= N1 at slot kz - N1 from the ring origin (base a2); N1 is a
// compile-time constant, so every load still has an immediate offset
template <int PLB, int N1, typename T, int... KZ>
__device__ __forceinline__ void zcontract_w(unsigned a1, unsigned a2, const T* wz, const T* dwz, T& t0, T& t1,
                                            std::integer_sequence<int, KZ...>) {
    ((t0 = fma(wz[KZ], lds_off<(KZ < N1 ? KZ : KZ - N1) * PLB>(KZ < N1 ? a1 : a2, T(0)), t0),
      t1 = fma(dwz[KZ], lds_off<(KZ < N1 ? KZ : KZ - N1) * PLB>(KZ < N1 ? a1 : a2, T(0)), t1)), ...);
}

__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// S7: a CTA owns the particles whose stencil starts lie in its MZ_TX x MZ_TY tile and one z
// segment.  A ring of DR Psi planes of the tile window (MZ_TX + P - 1) x (MZ_TY + P - 1) lives in
// shared memory; while a chunk's particles are gathered, the MZ_ZC planes of the next chunk are
// already on their way (cp.async), so plane loads overlap the gather.  A warp computes the
// separable weights of WB particles at once (lane = particle x axis, Gaussian recurrence) and
// gathers them one at a time, lanes over the P x P columns (z contracted per lane, W' from the
// stored W), 4-value butterfly reduction.
// TMA plane boxes for the gather ring (fp64): a 3D tensor map of Psi [Izs][Ixk][Iy] with box
// {WY, WX, 1}, and the stencil-column assignment for the dense box pitch WY: column col[r * 32 + l]
// (a P + b, or -1) for lane l in round r, grouped so that the 16 lanes of a half-warp hit 16
// distinct 8-byte bank pairs (a WY + b mod 16) wherever the residue classes allow.
struct __align__(64) GatherTma {
    unsigned long long map[16];          // CUtensorMap
    short col[128];
    int ok;                              // 0: cp.async rows only
};
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const void* map, int c0, int c1, int c2, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

template <int P, typename T = double, bool KB = false>
__global__ void __launch_bounds__(256, GRing<P, T, KB>::MINB) k_mid_gather_z(MidZArgs a, const T* __restrict__ psi,
                                                                              d4* __restrict__ out,
                                                                              const __grid_constant__ GatherTma tm) {
    using G = GRing<P, T, KB>;
    constexpr int DR = G::DR, PL = G::PL, WX = G::WX, WY = G::WY, WYP = G::WYP, NR = G::NR;
    // the mbarrier takes a whole 128-byte static block so that the dynamic ring after it starts on a
    // 128-byte boundary (TMA destinations)
    __shared__ __align__(128) unsigned long long tbarv[16];
    unsigned long long& tbar = tbarv[0];
    extern __shared__ __align__(128) unsigned char smraw[];
    T* sm = reinterpret_cast<T*>(smraw);
    T* ring = sm;                                        // [DR][PL]: WX rows of pitch WYP (or WY)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    T* wsb = sm + DR * PL + warp * G::WB * G::WSZ;
    const int tx = a.tlo + blockIdx.x / a.nty, ty = blockIdx.x % a.nty;
    const int tile = tx * a.nty + ty;
    const int X0 = tx * MZ_TX, Y0 = ty * MZ_TY;
    const int cb = a.c_lo + blockIdx.y * a.cps;
    const int ce = min(cb + a.cps, a.c_hi + 1);
    const unsigned ringS = smem_u32(ring);
    // TMA plane boxes when the window does not wrap (x periodic: X0 + WX <= Ix; y: Y0 + WY <= Iy;
    // an x-slab's rows past Ixk are the box's zero fill), else cp.async rows (pitch WYP)
    const bool use_tma = sizeof(T) == 8 && tm.ok && (!a.px || X0 + WX <= a.Ix) && Y0 + WY <= a.Iy && (ringS & 127) == 0;
    const int pitch = use_tma ? WY : WYP;
    // this lane's stencil columns (a, b): row-major over P x P (pitch WYP), or the bank-grouped
    // assignment of the TMA pitch; lanes without a column contribute nothing (cok)
    int ca[NR], cbb[NR];
    bool cok[NR];
    unsigned coffS[NR];                                  // column byte offsets in a plane window
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const int idx = use_tma ? tm.col[lane + 32 * r] : (lane + 32 * r < P * P ? lane + 32 * r : -1);
        cok[r] = idx >= 0;
        ca[r] = idx >= 0 ? idx / P : 0;
        cbb[r] = idx >= 0 ? idx - ca[r] * P : 0;
        coffS[r] = unsigned(ca[r] * pitch + cbb[r]) * unsigned(sizeof(T));
    }
    if (tid == 0) {
        mbar_init(&tbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    bool tpend = false;                                  // a TMA batch is in flight (uniform)
    unsigned tph = 0;                                    // its mbarrier phase parity
    auto tma_wait = [&]() {
        if (tpend) {
            mbar_wait(&tbar, tph);
            tph ^= 1u;
            tpend = false;
        }
    };
    // issue async copies of planes [p0, p1) of the window into their ring slots: one window row
    // (plane, x) per warp iteration, lanes along y (row bases computed once per row, warp-uniform)
    constexpr int YL = (WY + 31) / 32;                   // y elements per lane
    int gyl[YL];
#pragma unroll
    for (int k = 0; k < YL; ++k) gyl[k] = wrapc(Y0 + lane + 32 * k, a.Iy);
    auto load_planes = [&](int p0, int p1) {
        if (use_tma) {                                   // one box per plane, issued by one thread
            if (p1 <= p0) return;
            tma_wait();                                  // one batch in flight at a time
            if (tid == 0) {
                mbar_expect_tx(&tbar, unsigned((p1 - p0) * WX * WY * sizeof(T)));
                for (int pl = p0; pl < p1; ++pl) tma_load_3d(ring + (pl % DR) * PL, &tm.map, Y0, X0, pl, &tbar);
            }
            tpend = true;
            return;
        }
        const int nrow = (p1 - p0) * WX;
        for (int rw = warp; rw < nrow; rw += 8) {
            const int pz = rw / WX, xr = rw - pz * WX;
            const int plane = p0 + pz;
            const int gx = a.px ? wrapc(X0 + xr, a.Ix) : X0 + xr;
            T* dst = ring + (plane % DR) * PL + xr * WYP;
            if (gx < a.Ixk) {
                const T* srow = psi + ((size_t)plane * a.Ixk + gx) * a.Iy;
#pragma unroll
                for (int k = 0; k < YL; ++k) {
                    const int yr = lane + 32 * k;
                    if (yr < WY) {
                        if (sizeof(T) == 8) cp_async8(dst + yr, srow + gyl[k]); else cp_async4(dst + yr, srow + gyl[k]);
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < YL; ++k)
                    if (lane + 32 * k < WY) dst[lane + 32 * k] = T(0);
            }
        }
    };
    int zh = 0, zl = 0;                                  // planes [zl, zh) resident or in flight
    for (int c = cb; c < ce; ++c) {
        const int key = tile * a.nzc + c;
        const int k0 = a.mstart[key], k1 = a.mstart[key + 1];
        if (k0 == k1) continue;
        const int nlo = c * MZ_ZC, nhi = min(c * MZ_ZC + G::D, a.Izs);
        __syncthreads();                                 // previous chunk's readers are done
        if (!(zl <= nlo && zh >= nhi)) {                 // not prefetched (first chunk or a jump)
            const int from = (zl <= nlo && zh > nlo) ? zh : nlo;
            load_planes(from, nhi);
            zl = nlo;
            zh = nhi;
        }
        if (use_tma) tma_wait(); else cp_async_wait_all();
        __syncthreads();
        // prefetch the next chunk's new planes into the slots of planes < nlo (no longer read)
        {
            const int p1 = min(nhi + MZ_ZC, a.Izs);
            if (p1 > zh) { load_planes(zh, p1); zh = p1; }
            zl = max(zl, zh - DR);
        }
        // particles of the chunk dealt round-robin over the 8 warps (k0 + warp + 8 i), WB at a time.
        // Weights of WB particles at once.  Gaussian window: lane = (particle, axis, segment of
        // G::SEGL stencil points), each lane starts its segment with two exps and runs the recurrence
        // over its points; KB window: lane = (particle, axis), all P points.  The lane's particle
        // record (stencil start, one coordinate) of the next batch is loaded one batch ahead.
        constexpr int NSG = KB ? 1 : G::NSEG;
        const int pp = lane / (3 * NSG), rl = lane - pp * 3 * NSG, axl = rl / NSG, sg = rl - axl * NSG;
        int4 in_n = make_int4(0, 0, 0, 0);
        double x_n = 0.0;
        auto fetch = [&](int kb) {
            if (lane < 3 * NSG * G::WB && kb + 8 * pp < k1) {
                in_n = a.minfo[kb + 8 * pp];
                x_n = __ldg(reinterpret_cast<const double*>(&a.mpos[kb + 8 * pp]) + axl);
            }
        };
        fetch(k0 + warp);
        for (int kb = k0 + warp; kb < k1; kb += G::WB * 8) {
            const int nb = min(G::WB, (k1 - kb + 7) / 8);
            const int4 in = in_n;
            const double x = x_n;
            fetch(kb + G::WB * 8);
            if (lane < 3 * NSG * nb) {
                const double hh = axl == 0 ? a.hx : (axl == 1 ? a.hy : a.hz);
                const double hf = axl == 0 ? a.halfx : (axl == 1 ? a.halfy : a.halfz);
                const double aa = axl == 0 ? a.invH2Sx : (axl == 1 ? a.invH2Sy : a.invH2Sz);
                const double gg = axl == 0 ? a.gamma_x : (axl == 1 ? a.gamma_y : a.gamma_z);
                const int sa = axl == 0 ? in.y : (axl == 1 ? in.z : in.w);
                T* o = wsb + pp * G::WSZ + axl * P;
                if constexpr (KB) {
                    double w[P], dw[P];
                    kb_weights<P, true>(kb_offset(x, hh, hf, sa + (P - 1) / 2), a.kt, w, dw);
                    const double ih = 1.0 / hh;
#pragma unroll
                    for (int i = 0; i < P; ++i) {
                        o[i] = T(w[i]);
                        o[3 * P + i] = T(dw[i] * ih);          // dW/dx = dW/du / h
                    }
                } else {
                    // Gaussian recurrence; W' = 2 a (x_g - x) W (R11), stored with W so the gather
                    // loop reads it instead of every lane recomputing it
                    const double d0 = ((double)sa - hf) * hh - x;
                    const int i0 = sg * G::SEGL;
                    const double di = d0 + i0 * hh;
                    double w = exp(-aa * di * di);
                    double q = exp(-aa * hh * (2.0 * di + hh));
                    const double a2 = 2.0 * aa;
#pragma unroll
                    for (int k = 0; k < G::SEGL; ++k) {
                        const int i = i0 + k;
                        if (i < P) {
                            o[i] = T(w);
                            o[3 * P + i] = T(a2 * (d0 + i * hh) * w);
                        }
                        w *= q;
                        q *= gg;
                    }
                }
                if (axl == 0 && sg == 0) {
                    int* hd = reinterpret_cast<int*>(wsb + pp * G::WSZ + G::HOFF);
                    hd[0] = a.px ? in.y - X0 + (in.y < 0 ? a.Ix : 0) : in.y - a.xorig - X0;   // relative to the tile
                    hd[1] = in.z - Y0 + (in.z < 0 ? a.Iy : 0);
                    hd[2] = in.w % DR;                                   // ring slot of the first plane
                    hd[3] = in.x;                                        // output (cell-sorted) index
                }
            }
            __syncwarp();
            for (int pp = 0; pp < nb; ++pp) {
                const T* wsc = wsb + pp * G::WSZ;
                const int4 hd = *reinterpret_cast<const int4*>(wsc + G::HOFF);
                T wz[P], dwz[P];
#pragma unroll
                for (int i = 0; i < P; ++i) {
                    wz[i] = wsc[2 * P + i];
                    dwz[i] = wsc[5 * P + i];
                }
                const unsigned o0 = ringS + unsigned(hd.x * pitch + hd.y) * unsigned(sizeof(T));
                T phi = 0, gx = 0, gy = 0, gz = 0;
                // contraction of one stencil column (z first), then the separable x / y weights
                auto column = [&](int rr, const T t0, const T t1) {
                    const T wx = wsc[ca[rr]], wy = wsc[P + cbb[rr]];
                    const T dwx = wsc[3 * P + ca[rr]], dwy = wsc[4 * P + cbb[rr]];
                    const T wxy = wx * wy;
                    phi = fma(wxy, t0, phi);
                    gz = fma(wxy, t1, gz);
                    gx = fma(dwx * wy, t0, gx);
                    gy = fma(wx * dwy, t0, gy);
                };
                if (hd.z + P <= DR) {
                    // the particle's P planes are consecutive ring slots: immediate plane offsets
                    const unsigned zb = o0 + unsigned(hd.z * PL) * unsigned(sizeof(T));
#pragma unroll
                    for (int rr = 0; rr < NR; ++rr) {
                        if (!cok[rr]) continue;                  // no column for this lane in this round
                        T t0 = 0, t1 = 0;
                        zcontract<PL * int(sizeof(T))>(zb + coffS[rr], wz, dwz, t0, t1,
                                                       std::make_integer_sequence<int, P>{});
                        column(rr, t0, t1);
                    }
                } else {
                    // the particle's planes wrap around the ring after n1 = DR - hd.z of them: one
                    // instantiation per n1, immediate offsets from two bases
                    const unsigned zb1 = o0 + unsigned(hd.z * PL) * unsigned(sizeof(T));
                    auto rounds = [&](auto n1c) {
                        constexpr int N1 = decltype(n1c)::value;
                        if constexpr (N1 < P) {
#pragma unroll
                            for (int rr = 0; rr < NR; ++rr) {
                                if (!cok[rr]) continue;
                                T t0 = 0, t1 = 0;
                                zcontract_w<PL * int(sizeof(T)), N1>(zb1 + coffS[rr], o0 + coffS[rr], wz, dwz, t0, t1,
                                                                    std::make_integer_sequence<int, P>{});
                                column(rr, t0, t1);
                            }
                        }
                    };
                    switch (DR - hd.z) {
#define SOG_WRAP_CASE(n) \
    case n: rounds(std::integral_constant<int, n>{}); break;
                        SOG_WRAP_CASE(1) SOG_WRAP_CASE(2) SOG_WRAP_CASE(3) SOG_WRAP_CASE(4) SOG_WRAP_CASE(5)
                        SOG_WRAP_CASE(6) SOG_WRAP_CASE(7) SOG_WRAP_CASE(8) SOG_WRAP_CASE(9) SOG_WRAP_CASE(10)
                        SOG_WRAP_CASE(11) SOG_WRAP_CASE(12) SOG_WRAP_CASE(13) SOG_WRAP_CASE(14) SOG_WRAP_CASE(15)
                        SOG_WRAP_CASE(16) SOG_WRAP_CASE(17) SOG_WRAP_CASE(18) SOG_WRAP_CASE(19) SOG_WRAP_CASE(20)
                        SOG_WRAP_CASE(21) SOG_WRAP_CASE(22) SOG_WRAP_CASE(23) SOG_WRAP_CASE(24)
#undef SOG_WRAP_CASE
                        default: break;
                    }
                }
                // 4-value butterfly (fp64): after two levels each lane carries one value
                const bool b1 = lane & 1;
                const double vphi = phi, vgx = gx, vgy = gy, vgz = gz;
                double k0v = b1 ? vgx : vphi, k1v = b1 ? vgz : vgy;
                k0v += __shfl_xor_sync(0xffffffffu, b1 ? vphi : vgx, 1);
                k1v += __shfl_xor_sync(0xffffffffu, b1 ? vgy : vgz, 1);
                const bool b2 = lane & 2;
                double kk = b2 ? k1v : k0v;
                kk += __shfl_xor_sync(0xffffffffu, b2 ? k0v : k1v, 2);
#pragma unroll
                for (int o = 4; o < 32; o <<= 1) kk += __shfl_xor_sync(0xffffffffu, kk, o);
                // lane&3: 0 -> phi, 1 -> gx, 2 -> gy, 3 -> gz (one 32-byte sector)
                if (lane < 4) reinterpret_cast<double*>(&out[hd.w])[lane] = a.Vh * kk;
            }
            __syncwarp();
        }
    }
    cp_async_wait_all();                                 // no copy may outlive the CTA
    tma_wait();
}

// S7 gather for wide windows whose plane ring does not fit in shared memory: same work split
// (warp per particle, lanes over stencil columns) reading Psi through L1.
template <int P>
__global__ void __launch_bounds__(256) k_mid_gather_g(MidZArgs a, const double* __restrict__ psi,
                                                      d4* __restrict__ out, int nmid) {
    __shared__ double wsm[8][6 * P + 2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* wsc = wsm[warp];
    const int ax = min(lane, 2);
    const double h = ax == 0 ? a.hx : (ax == 1 ? a.hy : a.hz);
    const double half = ax == 0 ? a.halfx : (ax == 1 ? a.halfy : a.halfz);
    const double al = ax == 0 ? a.invH2Sx : (ax == 1 ? a.invH2Sy : a.invH2Sz);
    const double gam = ax == 0 ? a.gamma_x : (ax == 1 ? a.gamma_y : a.gamma_z);
    const size_t plane = (size_t)a.Ixk * a.Iy;
    for (int k = blockIdx.x * 8 + warp; k < nmid; k += gridDim.x * 8) {
        const int4 in = a.minfo[k];
        const d4 r = ld_d4(&a.mpos[k]);
        if (lane < 3) {
            const double x = lane == 0 ? r.x : (lane == 1 ? r.y : r.z);
            const int s = lane == 0 ? in.y : (lane == 1 ? in.z : in.w);
            double* o = wsc + 2 * lane * P;
            if (a.kb) {
                double w[P], dw[P];
                if constexpr (P <= KB_PMAX) kb_weights<P, true>(kb_offset(x, h, half, s + (P - 1) / 2), a.kt, w, dw);
                for (int i = 0; i < P; ++i) {
                    o[i] = w[i];
                    o[P + i] = dw[i] / h;
                }
            } else {
                const double d0 = ((double)s - half) * h - x;
                double w = exp(-al * d0 * d0);
                double q = exp(-al * h * (2.0 * d0 + h));
                for (int i = 0; i < P; ++i) {
                    o[i] = w;
                    o[P + i] = 2.0 * al * (d0 + i * h) * w;
                    w *= q;
                    q *= gam;
                }
            }
        }
        __syncwarp();
        double phi = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
        const double* zb = psi + (size_t)in.w * plane;
        for (int idx = lane; idx < P * P; idx += 32) {
            const int ai = idx / P, bi = idx - ai * P;
            const int ix = a.px ? wrapc(in.y + ai, a.Ix) : min(in.y + ai - a.xorig, a.Ixk - 1), iy = wrapc(in.z + bi, a.Iy);
            const double* col = zb + (size_t)ix * a.Iy + iy;
            double t0 = 0.0, t1 = 0.0;
#pragma unroll
            for (int kz = 0; kz < P; ++kz) {
                const double v = __ldg(col + kz * plane);
                t0 = fma(wsc[4 * P + kz], v, t0);
                t1 = fma(wsc[5 * P + kz], v, t1);
            }
            const double wx = wsc[ai], dwx = wsc[P + ai], wy = wsc[2 * P + bi], dwy = wsc[3 * P + bi];
            phi = fma(wx * wy, t0, phi);
            gz = fma(wx * wy, t1, gz);
            gx = fma(dwx * wy, t0, gx);
            gy = fma(wx * dwy, t0, gy);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            phi += __shfl_xor_sync(0xffffffffu, phi, o);
            gx += __shfl_xor_sync(0xffffffffu, gx, o);
            gy += __shfl_xor_sync(0xffffffffu, gy, o);
            gz += __shfl_xor_sync(0xffffffffu, gz, o);
        }
        if (lane == 0) st_d4(&out[in.x], d4{a.Vh * phi, a.Vh * gx, a.Vh * gy, a.Vh * gz});
        __syncwarp();
    }
}

// S5: multiply the half spectrum [Izs][Ix][Iy/2+1] by mult(k) = sum_{l<=m} A_l Tz[l][iz]
// Tx[l][ix] Ty[l][iy].  A CTA owns MS_ROWS (iz, ix) rows: the per-row factors
// A_l Tz Tx go to shared memory, each thread keeps Ty[l][iy] of its iy in registers.
constexpr int MS_ROWS = 16;
template <int LM, typename C = cuDoubleComplex>
__global__ void __launch_bounds__(128) k_mid_scale(C* __restrict__ spec, int Ix, int Izs, int nyh, int L,
                                                   const double* __restrict__ A, const double* __restrict__ Tx,
                                                   const double* __restrict__ Ty, const double* __restrict__ Tz) {
    __shared__ double sc[MS_ROWS][LM];
    const int iy = blockIdx.x * blockDim.x + threadIdx.x;
    const int row0 = blockIdx.y * MS_ROWS, nrows = Izs * Ix;
    for (int e = threadIdx.x; e < MS_ROWS * LM; e += blockDim.x) {
        const int r = e / LM, l = e - r * LM, row = row0 + r;
        double v = 0.0;
        if (row < nrows && l < L) {
            const int iz = row / Ix, ix = row - iz * Ix;
            v = A[l] * Tz[(size_t)l * Izs + iz] * Tx[(size_t)l * Ix + ix];
        }
        sc[r][l] = v;
    }
    __syncthreads();
    if (iy >= nyh) return;
    double ty[LM];
#pragma unroll
    for (int l = 0; l < LM; ++l) ty[l] = l < L ? Ty[(size_t)l * nyh + iy] : 0.0;
    for (int r = 0; r < MS_ROWS && row0 + r < nrows; ++r) {
        double m = 0.0;
#pragma unroll
        for (int l = 0; l < LM; ++l) m = fma(sc[r][l], ty[l], m);
        const size_t idx = (size_t)(row0 + r) * nyh + iy;
        C v = spec[idx];
        v.x *= m;
        v.y *= m;
        spec[idx] = v;
    }
}

}  // namespace sog

namespace sog {

// ---------------------------------------------------------------------------------------
// z-pruned mid FFT (whole box).  S is zero outside the planes the spread writes, and the
// gather reads Psi only on the planes the particles' stencils reach, so:
//   2D D2Z over the nonzero planes  X[z][m], m = x * nyh + ky        (cuFFT, batched)
//   transpose into zero-padded pencils Y[m][Izs] (z contiguous)       (k_tr_xz)
//   1D Z2Z along z, S5 scaling on [m][kz], inverse 1D Z2Z               (cuFFT + k_scale_pencil_z)
//   transpose the gather's planes back X'[z][m], 2D Z2D into Psi       (k_tr_zx, cuFFT)
// The normalisation is unchanged (cuFFT 2D x 1D unnormalised = 3D).
constexpr int TR_T = 32;

// X [nz][M] (complex) -> Y [M][Izs] rows, columns z0 .. z0 + nz
template <typename C>
__global__ void __launch_bounds__(TR_T * 8) k_tr_xz(const C* __restrict__ X, C* __restrict__ Y, int nz, long long M,
                                                     int Izs, int z0) {
    __shared__ C tile[TR_T][TR_T + 1];
    const long long m0 = (long long)blockIdx.x * TR_T;
    const int zb = blockIdx.y * TR_T;
    const int tx = threadIdx.x & (TR_T - 1), ty = threadIdx.x / TR_T;   // 32 x 8 threads
    for (int r = ty; r < TR_T; r += 8) {
        const int z = zb + r;
        const long long m = m0 + tx;
        if (z < nz && m < M) tile[r][tx] = X[(size_t)z * M + m];
    }
    __syncthreads();
    for (int r = ty; r < TR_T; r += 8) {
        const long long m = m0 + r;
        const int z = zb + tx;
        if (z < nz && m < M) Y[(size_t)m * Izs + z0 + z] = tile[tx][r];
    }
}

// Y [M][Izs] columns z0 .. z0 + nz -> X [nz][M]
template <typename C>
__global__ void __launch_bounds__(TR_T * 8) k_tr_zx(const C* __restrict__ Y, C* __restrict__ X, int nz, long long M,
                                                     int Izs, int z0) {
    __shared__ C tile[TR_T][TR_T + 1];
    const long long m0 = (long long)blockIdx.x * TR_T;
    const int zb = blockIdx.y * TR_T;
    const int tx = threadIdx.x & (TR_T - 1), ty = threadIdx.x / TR_T;
    for (int r = ty; r < TR_T; r += 8) {
        const long long m = m0 + r;
        const int z = zb + tx;
        if (z < nz && m < M) tile[r][tx] = Y[(size_t)m * Izs + z0 + z];
    }
    __syncthreads();
    for (int r = ty; r < TR_T; r += 8) {
        const int z = zb + r;
        const long long m = m0 + tx;
        if (z < nz && m < M) X[(size_t)z * M + m] = tile[tx][r];
    }
}

// S5 on z pencils W [m = x * nyh + ky][Izs]: a CTA owns MS_ROWS pencils (per-pencil factors
// A_l Tx Ty in shared memory), each thread keeps Tz[l][z] of its z in registers.
template <int LM, typename C>
__global__ void __launch_bounds__(128) k_scale_pencil_z(C* __restrict__ W, int Ix, int nyh, int Izs, int L,
                                                        const double* __restrict__ A, const double* __restrict__ Tx,
                                                        const double* __restrict__ Ty, const double* __restrict__ Tz) {
    __shared__ double sc[MS_ROWS][LM];
    const int z = blockIdx.x * blockDim.x + threadIdx.x;
    const long long M = (long long)Ix * nyh;
    const long long row0 = (long long)blockIdx.y * MS_ROWS;
    for (int e = threadIdx.x; e < MS_ROWS * LM; e += blockDim.x) {
        const int r = e / LM, l = e - r * LM;
        const long long m = row0 + r;
        double v = 0.0;
        if (m < M && l < L) {
            const int x = int(m / nyh), ky = int(m - (long long)x * nyh);
            v = A[l] * Tx[(size_t)l * Ix + x] * Ty[(size_t)l * nyh + ky];
        }
        sc[r][l] = v;
    }
    __syncthreads();
    if (z >= Izs) return;
    double tz[LM];
#pragma unroll
    for (int l = 0; l < LM; ++l) tz[l] = l < L ? Tz[(size_t)l * Izs + z] : 0.0;
    for (int r = 0; r < MS_ROWS && row0 + r < M; ++r) {
        double m = 0.0;
#pragma unroll
        for (int l = 0; l < LM; ++l) m = fma(sc[r][l], tz[l], m);
        const size_t idx = (size_t)(row0 + r) * Izs + z;
        C v = W[idx];
        v.x *= m;
        v.y *= m;
        W[idx] = v;
    }
}

}  // namespace sog
