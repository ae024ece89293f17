// Mid-range stencil kernels (Algorithm 1) and their launchers.
#include "kernels_mid.cuh"
#include "launch.h"

namespace sog {

#define SOG_ODD_P(M) M(5) M(7) M(9) M(11) M(13) M(15) M(17) M(19) M(21) M(23) M(25)

int launch_mid_gather(const MidArgs& a, int P, const double* psi, d4* out, double gx, double gy, double gz,
                      cudaStream_t st) {
    int nb = (a.N + 127) / 128;
    switch (P) {
#define C_(P_) case P_: k_mid_gather<P_><<<nb, 128, 0, st>>>(a, psi, out, gx, gy, gz); break;
        SOG_ODD_P(C_)
#undef C_
        default: return 1;
    }
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int launch_mid_spread_tile(const MidTileArgs& t, int P, const int4* g0, double* grid, cudaStream_t st) {
    const int nblk = t.ntx * t.nty * t.ntz;
    const size_t sh = sizeof(double) * MT_B * ((2 * P + 2 + MT_Z) & ~1);
    switch (P) {
#define C_(P_)                                                                                          \
    case P_:                                                                                            \
        if (cudaFuncSetAttribute(k_mid_spread_tile<P_>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                 (int)sh) != cudaSuccess) return 2;                                     \
        k_mid_spread_tile<P_><<<nblk, 256, sh, st>>>(t, g0, grid);                                      \
        break;
        SOG_ODD_P(C_)
#undef C_
        default: return 1;
    }
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int launch_stencil_origins(const d4* pos, int N, const MidArgs& a, int has_mid, double lhx, double lhy, double lhpx,
                           double lhpy, int4* g0, cudaStream_t st) {
    k_stencil_origins<<<(N + 255) / 256, 256, 0, st>>>(pos, N, a, has_mid, lhx, lhy, lhpx, lhpy, g0);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace sog
