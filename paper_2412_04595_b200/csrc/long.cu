// Long-range stencil kernels (Algorithm 2, two-sided proxies) and their launchers.
#include <algorithm>
#include <cstdlib>
#include "kernels_long.cuh"
#include "launch.h"

namespace sog {

#define SOG_ODD_P(M) M(5) M(7) M(9) M(11) M(13) M(15) M(17) M(19) M(21) M(23) M(25)

template <int PCMAX>
int long_tile_dispatch(const LongTileArgs& t, int Pl, cudaStream_t st) {
    int nthr = ((t.TX * t.TY + 31) / 32) * 32;
    size_t sh = sizeof(double) * (PCMAX * PCMAX + LB * 2 * Pl + 2 * LB * PCMAX + LB) + sizeof(int) * 2 * LB;
    dim3 grid(t.nchunk, t.ntx * t.nty);
    switch (Pl) {
#define C_(P_)                                                                                         \
    case P_:                                                                                           \
        if (cudaFuncSetAttribute(k_long_spread_tile<P_, PCMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 (int)sh) != cudaSuccess) return 2;                                    \
        k_long_spread_tile<P_, PCMAX><<<grid, nthr, sh, st>>>(t);                                      \
        break;
        SOG_ODD_P(C_)
#undef C_
        default: return 1;
    }
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int launch_long_spread_tile(const LongTileArgs& t, int Pl, double* grid, cudaStream_t st) {
    LongTileArgs tg = t;
    tg.grid = grid;
    int r = t.a.Pc <= 16 ? long_tile_dispatch<16>(tg, Pl, st) : (t.a.Pc <= 32 ? long_tile_dispatch<32>(tg, Pl, st) : 1);
    if (r) return r;
    if (t.nchunk == 1) return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;   // tiles wrote the grid
    int pcmax = t.a.Pc <= 16 ? 16 : 32;
    int n = t.a.Ilx * t.a.Ily * t.a.Pc;
    k_long_reduce<<<(n + 255) / 256, 256, 0, st>>>(t.part, grid, t.a.Ilx, t.a.Ily, t.a.Pc, pcmax, t.TX, t.TY, t.nty,
                                                   t.nchunk);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

template <int PCP>
int tgemm_go(const LongTileArgs& t, double* grid, cudaStream_t st) {
    const int TYP = (t.TY + 3) & ~3;
    const int nthr = ((t.TX * (TYP / 4) * (PCP / LG_LT) + 31) / 32) * 32;
    if (nthr > 256) return 1;
    const int RW = ((t.TX + TYP + PCP) + 1) & ~1;
    const size_t sh = sizeof(double) * 2 * LG_KB * RW;
    if (cudaFuncSetAttribute(k_long_spread_tgemm<PCP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) !=
        cudaSuccess)
        return 2;
    LongTileArgs tg = t;
    tg.grid = grid;
    k_long_spread_tgemm<PCP><<<dim3(t.nchunk, t.ntx * t.nty), nthr, sh, st>>>(tg);
    if (t.nchunk > 1) {
        const int n = t.a.Ilx * t.a.Ily * t.a.Pc;
        k_long_treduce<<<(n + 255) / 256, 256, 0, st>>>(t.part, grid, t.a.Ilx, t.a.Ily, t.a.Pc, PCP, t.TX, t.TY, t.nty,
                                                       t.nchunk);
    }
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int launch_long_spread_tgemm(const LongTileArgs& t, double* grid, cudaStream_t st) {
    switch (long_small_pcp(t.a.Pc)) {
        case 6: return tgemm_go<6>(t, grid, st);
        case 12: return tgemm_go<12>(t, grid, st);
        case 18: return tgemm_go<18>(t, grid, st);
        case 24: return tgemm_go<24>(t, grid, st);
        case 30: return tgemm_go<30>(t, grid, st);
    }
    return 1;
}

#define SOG_PCMAX(M) M(8) M(12) M(16) M(20) M(24) M(28) M(32)

int long_pcmax(int Pc) {
    for (int m : {8, 12, 16, 20, 24, 28, 32})
        if (Pc <= m) return m;
    return 0;
}

template <int P, int PCMAX>
int long_gather2_go(const LongArgs& a, const double* psiT, d4* out, double gx, double gy, cudaStream_t st) {
    const size_t grid_bytes = sizeof(double) * (size_t)a.Ilx * a.Ily * PCMAX;
    const bool smem = grid_bytes <= 96 * 1024;
    const size_t sh = sizeof(double) * PCMAX * PCMAX + (smem ? grid_bytes : 0);
    auto k = k_long_gather2<P, PCMAX>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) != cudaSuccess) return 2;
    k<<<(a.N + 127) / 128, 128, sh, st>>>(a, psiT, out, gx, gy, smem ? 1 : 0);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

template <int PCMAX>
int long_gather2_p(const LongArgs& a, int Pl, const double* psiT, d4* out, double gx, double gy, cudaStream_t st) {
    switch (Pl) {
#define C_(P_) case P_: return long_gather2_go<P_, PCMAX>(a, psiT, out, gx, gy, st);
        SOG_ODD_P(C_)
#undef C_
        default: return 1;
    }
}

int launch_long_gather2(const LongArgs& a, int Pl, const double* psi, double* psiT, d4* out, double gx, double gy,
                        cudaStream_t st) {
    const int pm = long_pcmax(a.Pc);
    if (!pm) return 1;
    const int n = a.Ilx * a.Ily * pm;
    k_long_transpose<<<(n + 255) / 256, 256, 0, st>>>(psi, psiT, a.Ilx, a.Ily, a.Pc, pm);
    switch (pm) {
#define C_(M_) case M_: return long_gather2_p<M_>(a, Pl, psiT, out, gx, gy, st);
        SOG_PCMAX(C_)
#undef C_
    }
    return 1;
}

}  // namespace sog

namespace sog {

// ---- small long grids (T-basis register-tiled spread, broadcast gather) ----
int long_small_pcp(int Pc) { return Pc <= 30 ? ((Pc + LG_LT - 1) / LG_LT) * LG_LT : 0; }

bool long_small_ok(int Ilx, int Ily, int Pc) {
    const int pcp = long_small_pcp(Pc);
    return Ilx <= LG_RX && Ily <= 16 && pcp > 0 && Ilx * ((Ily + 3) / 4) * (pcp / LG_LT) <= 256;
}

template <int PCP, typename T>
int spread_gemm_go(const LongArgs& a, const int4* g0, double gx, double gy, int nblk, T* part, T* grid,
                   cudaStream_t st) {
    int nthr = ((a.Ilx * ((a.Ily + 3) / 4) * (PCP / LG_LT) + 31) / 32) * 32;
    if (nthr > 256) return 1;
    nthr = nthr <= 128 ? 128 : 256;
    const int per = (a.N + nblk - 1) / nblk;
    const int RW = ((a.Ilx + ((a.Ily + 3) & ~3) + PCP) + 1) & ~1;
    const size_t sh = sizeof(T) * 2 * LG_KB * RW;
    if (cudaFuncSetAttribute(k_long_spread_gemm<PCP, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) !=
        cudaSuccess)
        return 2;
    k_long_spread_gemm<PCP, T><<<nblk, nthr, sh, st>>>(a, g0, gx, gy, per, part);
    const int G = a.Ilx * a.Ily;
    k_long_sum<T><<<(G * a.Pc + 255) / 256, 256, 0, st>>>(part, grid, G, a.Pc, PCP, nblk);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

template <typename T>
int spread_gemm_t(const LongArgs& a, const int4* g0, double gx, double gy, int nblk, T* part, T* grid,
                  cudaStream_t st) {
    switch (long_small_pcp(a.Pc)) {
        case 6: return spread_gemm_go<6, T>(a, g0, gx, gy, nblk, part, grid, st);
        case 12: return spread_gemm_go<12, T>(a, g0, gx, gy, nblk, part, grid, st);
        case 18: return spread_gemm_go<18, T>(a, g0, gx, gy, nblk, part, grid, st);
        case 24: return spread_gemm_go<24, T>(a, g0, gx, gy, nblk, part, grid, st);
        case 30: return spread_gemm_go<30, T>(a, g0, gx, gy, nblk, part, grid, st);
    }
    return 1;
}

template <int MT>
int spread_mma_go(const LongArgs& a, const int4* g0, double gx, double gy, int nblk, double* part, double* grid,
                  cudaStream_t st) {
    constexpr int NTW = 3;
    const int G = a.Ilx * a.Ily, NT = (G + 7) / 8, nw = (NT + NTW - 1) / NTW;
    if (nw * 32 > 384) return 1;
    const int per = (a.N + nblk - 1) / nblk;
    const int RW = (8 * MT + a.Ilx + a.Ily + 1) & ~1;
    const size_t sh = sizeof(double) * 2 * LS_KB * RW;
    if (cudaFuncSetAttribute(k_long_spread_mma<MT, NTW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) !=
        cudaSuccess)
        return 2;
    const int PCP = long_small_pcp(a.Pc);
    k_long_spread_mma<MT, NTW><<<nblk, std::max(nw * 32, 96), sh, st>>>(a, g0, gx, gy, per, PCP, part);
    k_long_sum<double><<<(G * a.Pc + 255) / 256, 256, 0, st>>>(part, grid, G, a.Pc, PCP, nblk);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int launch_long_spread_gemm(const LongArgs& a, const int4* g0, double gx, double gy, int nblk, void* part, void* grid,
                            bool f32, cudaStream_t st) {
    // fp64 opt-in (SOG_LONG_MMA=1): the DMMA product; measured slower than the register-tiled DFMA
    // kernel at c5 (6.3 vs 3.9 ms), so off by default
    static const bool mma = std::getenv("SOG_LONG_MMA") && std::atoi(std::getenv("SOG_LONG_MMA")) == 1;
    if (!f32 && mma) {
        int r = 1;
        switch ((a.Pc + 7) / 8) {
            case 1: r = spread_mma_go<1>(a, g0, gx, gy, nblk, (double*)part, (double*)grid, st); break;
            case 2: r = spread_mma_go<2>(a, g0, gx, gy, nblk, (double*)part, (double*)grid, st); break;
            case 3: r = spread_mma_go<3>(a, g0, gx, gy, nblk, (double*)part, (double*)grid, st); break;
            case 4: r = spread_mma_go<4>(a, g0, gx, gy, nblk, (double*)part, (double*)grid, st); break;
            default: break;
        }
        if (r != 1) return r;
    }
    return f32 ? spread_gemm_t(a, g0, gx, gy, nblk, (float*)part, (float*)grid, st)
               : spread_gemm_t(a, g0, gx, gy, nblk, (double*)part, (double*)grid, st);
}

template <int PCP, int NCY, typename T>
int gather_bc_go(const LongArgs& a, const int4* g0, const T* psi, d4* out, cudaStream_t st) {
    const size_t sh = sizeof(T) * ((size_t)a.Ilx * a.Ily * PCP + 2 * 128 * (size_t)a.Ilx + 2 * 128 * NCY);
    auto k = k_long_gather_bc<PCP, NCY, T>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) != cudaSuccess) return 2;
    k<<<(a.N + 127) / 128, 128, sh, st>>>(a, g0, psi, out);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

template <int NCY, typename T>
int gather_bc_p(const LongArgs& a, const int4* g0, const T* psi, d4* out, cudaStream_t st) {
    // even PCP for 2-wide loads: Pc rounded up to even
    switch ((a.Pc + 1) & ~1) {
#define C_(M_) case M_: return gather_bc_go<M_, NCY, T>(a, g0, psi, out, st);
        C_(2) C_(4) C_(6) C_(8) C_(10) C_(12) C_(14) C_(16) C_(18) C_(20) C_(22) C_(24) C_(26) C_(28) C_(30)
#undef C_
    }
    return 1;
}

template <typename T>
int gather_bc_t(const LongArgs& a, const int4* g0, const T* psi, d4* out, cudaStream_t st) {
    if (a.Ily <= 8) return gather_bc_p<8, T>(a, g0, psi, out, st);
    if (a.Ily <= 12) return gather_bc_p<12, T>(a, g0, psi, out, st);
    if (a.Ily <= 16) return gather_bc_p<16, T>(a, g0, psi, out, st);
    return 1;
}

int launch_long_gather_bc(const LongArgs& a, const int4* g0, const void* psi, d4* out, bool f32, cudaStream_t st) {
    return f32 ? gather_bc_t(a, g0, (const float*)psi, out, st) : gather_bc_t(a, g0, (const double*)psi, out, st);
}

int launch_long_scale(const void* in, void* out, const double* K, int nmode, int Pc, bool f32, cudaStream_t st) {
    const int nb = (nmode * Pc + 127) / 128;
    if (f32) k_long_scale<cuComplex><<<nb, 128, 0, st>>>((const cuComplex*)in, (cuComplex*)out, K, nmode, Pc);
    else k_long_scale<cuDoubleComplex><<<nb, 128, 0, st>>>((const cuDoubleComplex*)in, (cuDoubleComplex*)out, K, nmode, Pc);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int launch_long_to_nodes(const double* in, double* out, int G, int Pc, const double* M, cudaStream_t st) {
    k_long_to_nodes<<<(G * Pc + 255) / 256, 256, 0, st>>>(in, out, G, Pc, M);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace sog
