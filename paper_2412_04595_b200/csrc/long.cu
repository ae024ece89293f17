// Long-range stencil kernels (Algorithm 2, two-sided proxies) and their launchers.
#include "kernels_long.cuh"
#include "launch.h"

namespace sog {

#define SOG_ODD_P(M) M(5) M(7) M(9) M(11) M(13) M(15) M(17) M(19) M(21) M(23) M(25) M(27)

template <int PCMAX>
int long_dispatch(const LongArgs& a, int Pl, bool spread, double* grid, const double* psi, d4* out, cudaStream_t st) {
    int nb = (a.N + 127) / 128;
    switch (Pl) {
#define C_(P_)                                                                        \
    case P_:                                                                          \
        if (spread) k_long_spread_atomic<P_, PCMAX><<<nb, 128, 0, st>>>(a, grid);     \
        else k_long_gather<P_, PCMAX><<<nb, 128, 0, st>>>(a, psi, out);               \
        break;
        SOG_ODD_P(C_)
#undef C_
        default: return 1;
    }
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int launch_long_spread(const LongArgs& a, int Pl, double* grid, cudaStream_t st) {
    if (a.Pc <= 16) return long_dispatch<16>(a, Pl, true, grid, nullptr, nullptr, st);
    if (a.Pc <= 32) return long_dispatch<32>(a, Pl, true, grid, nullptr, nullptr, st);
    return 1;
}

int launch_long_gather(const LongArgs& a, int Pl, const double* psi, d4* out, cudaStream_t st) {
    if (a.Pc <= 16) return long_dispatch<16>(a, Pl, false, nullptr, psi, out, st);
    if (a.Pc <= 32) return long_dispatch<32>(a, Pl, false, nullptr, psi, out, st);
    return 1;
}

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
    int r = t.a.Pc <= 16 ? long_tile_dispatch<16>(t, Pl, st) : (t.a.Pc <= 32 ? long_tile_dispatch<32>(t, Pl, st) : 1);
    if (r) return r;
    int pcmax = t.a.Pc <= 16 ? 16 : 32;
    int n = t.a.Ilx * t.a.Ily * t.a.Pc;
    k_long_reduce<<<(n + 255) / 256, 256, 0, st>>>(t.part, grid, t.a.Ilx, t.a.Ily, t.a.Pc, pcmax, t.TX, t.TY, t.nty,
                                                   t.nchunk);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace sog
