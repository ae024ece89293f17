// Launchers of the near-field kernels with the single polynomial (R16-G): k_near3 (warp per target),
// k_near4 (target-stationary, opt-in) and k_near5 + k_near_fold (each pair once, opt-in).
#include <cstdlib>
#include "kernels_near4.cuh"
#include "kernels_near5.cuh"
#include "launch.h"
#include "sog_internal.h"

namespace sog {

template <int D>
int near4_go(const Near4Args& a, const NearPoly& p, int nw, dim3 grid, cudaStream_t st) {
    NearPolyArg<D> P;
    for (int n = 0; n <= D; ++n) P.c[n] = p.c[n];
    P.inv_h = p.inv_h;
    const size_t sh = near4_smem(a.cap, nw);
    if (cudaFuncSetAttribute(k_near4<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) != cudaSuccess) return 2;
    k_near4<D><<<grid, 32 * nw, sh, st>>>(a, P);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

size_t near4_smem(int cap, int nw) {
    return sizeof(unsigned short) * (size_t)nw * N4_Q * 32 + (2 * sizeof(double2) + 3 * sizeof(float)) * (size_t)cap;
}

// k_near3 with the single polynomial (R16-G) instead of the table
template <int PD>
int near3p_go(const Near3Args& a, const NearPoly& p, int ncell, cudaStream_t st) {
    NearPolyArg<PD> P;
    for (int n = 0; n <= PD; ++n) P.c[n] = p.c[n];
    P.inv_h = p.inv_h;
    const size_t sh = 10 * sizeof(double2) + NEAR3_WARPS * 160 * sizeof(int) + 16 * (size_t)a.cap;
    if (cudaFuncSetAttribute(k_near3<NEAR_D, PD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) != cudaSuccess)
        return 2;
    k_near3<NEAR_D, PD><<<ncell, 32 * NEAR3_WARPS, sh, st>>>(a, P);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int launch_near3p(const Near3Args& a, const NearPoly& p, int ncell, cudaStream_t st) {
    switch (p.D) {
        case 16: return near3p_go<16>(a, p, ncell, st);
        case 20: return near3p_go<20>(a, p, ncell, st);
        case 24: return near3p_go<24>(a, p, ncell, st);
        case 28: return near3p_go<28>(a, p, ncell, st);
        case 32: return near3p_go<32>(a, p, ncell, st);
        case 40: return near3p_go<40>(a, p, ncell, st);
        case 48: return near3p_go<48>(a, p, ncell, st);
        case 56: return near3p_go<56>(a, p, ncell, st);
        default: return 1;
    }
}

template <int PD>
int near5_go(const Near5Args& a, const NearPoly& p, int ncell, cudaStream_t st) {
    NearPolyArg<PD> P;
    for (int n = 0; n <= PD; ++n) P.c[n] = p.c[n];
    P.inv_h = p.inv_h;
    const size_t sh = near5_smem(a.cap);
    if (sh > 227 * 1024) return 1;
    if (cudaFuncSetAttribute(k_near5<PD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) != cudaSuccess) return 2;
    k_near5<PD><<<ncell, 32 * NEAR5_WARPS, sh, st>>>(a, P);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int launch_near5(const Near5Args& a, const NearPoly& p, int ncell, cudaStream_t st) {
    if (a.cap % 128) return 1;
    switch (p.D) {
        case 16: return near5_go<16>(a, p, ncell, st);
        case 20: return near5_go<20>(a, p, ncell, st);
        case 24: return near5_go<24>(a, p, ncell, st);
        case 28: return near5_go<28>(a, p, ncell, st);
        case 32: return near5_go<32>(a, p, ncell, st);
        case 40: return near5_go<40>(a, p, ncell, st);
        case 48: return near5_go<48>(a, p, ncell, st);
        case 56: return near5_go<56>(a, p, ncell, st);
        default: return 1;
    }
}

int launch_near_fold(d4* out, const d4* part, int N, cudaStream_t st) {
    if (N <= 0) return 0;
    const long long nt = 4LL * N;
    k_near_fold<><<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(out, part, N);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int launch_near4(const Near4Args& a, const NearPoly& p, int nw, cudaStream_t st) {
    if (nw < 1 || nw > N4_MAXW) return 1;
    const dim3 grid(a.g.ncx * a.g.ncy, (a.g.ncz + a.kc - 1) / a.kc);
    switch (p.D) {
        case 16: return near4_go<16>(a, p, nw, grid, st);
        case 20: return near4_go<20>(a, p, nw, grid, st);
        case 24: return near4_go<24>(a, p, nw, grid, st);
        case 28: return near4_go<28>(a, p, nw, grid, st);
        case 32: return near4_go<32>(a, p, nw, grid, st);
        case 40: return near4_go<40>(a, p, nw, grid, st);
        case 48: return near4_go<48>(a, p, nw, grid, st);
        case 56: return near4_go<56>(a, p, nw, grid, st);
        default: return 1;
    }
}

}  // namespace sog
