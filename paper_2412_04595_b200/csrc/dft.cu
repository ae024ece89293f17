// Long range without FFT (Algorithm 3, App. B): launchers of the direct-sum kernels (kernels_dft.cuh).
#include "kernels_dft.cuh"
#include "launch.h"

namespace sog {

template <int PCP, int NYT, typename T>
int dft_spread_nyt(const LongArgs& a, const DftArgs& d, int nblk, T* part, T* S, cudaStream_t st) {
    const int nky2 = (d.nky + NYT - 1) / NYT;
    int nthr = ((d.nkx * nky2 * (PCP / DFT_LT) + 31) / 32) * 32;
    if (nthr > 256) return 1;
    nthr = nthr < 2 * DFT_KB ? 2 * DFT_KB : nthr;
    const int RW = ((2 * d.nkx + 2 * NYT * nky2 + PCP) + 1) & ~1;
    const size_t sh = sizeof(T) * 2 * DFT_KB * RW;
    if (sh > 227 * 1024) return 1;
    if (cudaFuncSetAttribute(k_long_dft_spread<PCP, NYT, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) !=
        cudaSuccess)
        return 2;
    const int per = (a.N + nblk - 1) / nblk;
    k_long_dft_spread<PCP, NYT, T><<<nblk, nthr, sh, st>>>(a, d, per, part);
    const int G = 2 * d.nmode;
    k_long_sum<T><<<(G * a.Pc + 255) / 256, 256, 0, st>>>(part, S, G, a.Pc, PCP, nblk);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

// 2 ky modes per thread while the block fits 256 threads, else 4
template <int PCP, typename T>
int dft_spread_go(const LongArgs& a, const DftArgs& d, int nblk, T* part, T* S, cudaStream_t st) {
    if (d.nkx * ((d.nky + 1) / 2) * (PCP / DFT_LT) <= 256) return dft_spread_nyt<PCP, 2, T>(a, d, nblk, part, S, st);
    return dft_spread_nyt<PCP, 4, T>(a, d, nblk, part, S, st);
}

template <int PCP, typename T>
int dft_gather_go(const LongArgs& a, const DftArgs& d, const T* psi, d4* out, cudaStream_t st) {
    const size_t sh = sizeof(T) * 2 * (size_t)d.nmode * PCP;
    if (sh > 200 * 1024) return 1;
    if (cudaFuncSetAttribute(k_long_dft_gather<PCP, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) !=
        cudaSuccess)
        return 2;
    k_long_dft_gather<PCP, T><<<(a.N + 127) / 128, 128, sh, st>>>(a, d, psi, out);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

template <typename T>
int dft_spread_t(const LongArgs& a, const DftArgs& d, int nblk, T* part, T* S, cudaStream_t st) {
    switch (long_small_pcp(a.Pc)) {
        case 6: return dft_spread_go<6, T>(a, d, nblk, part, S, st);
        case 12: return dft_spread_go<12, T>(a, d, nblk, part, S, st);
        case 18: return dft_spread_go<18, T>(a, d, nblk, part, S, st);
        case 24: return dft_spread_go<24, T>(a, d, nblk, part, S, st);
        case 30: return dft_spread_go<30, T>(a, d, nblk, part, S, st);
    }
    return 1;
}

template <typename T>
int dft_gather_t(const LongArgs& a, const DftArgs& d, const T* psi, d4* out, cudaStream_t st) {
    switch (long_small_pcp(a.Pc)) {
        case 6: return dft_gather_go<6, T>(a, d, psi, out, st);
        case 12: return dft_gather_go<12, T>(a, d, psi, out, st);
        case 18: return dft_gather_go<18, T>(a, d, psi, out, st);
        case 24: return dft_gather_go<24, T>(a, d, psi, out, st);
        case 30: return dft_gather_go<30, T>(a, d, psi, out, st);
    }
    return 1;
}

int launch_long_dft_spread(const LongArgs& a, const DftArgs& d, int nblk, void* part, void* S, bool f32,
                           cudaStream_t st) {
    return f32 ? dft_spread_t(a, d, nblk, (float*)part, (float*)S, st)
               : dft_spread_t(a, d, nblk, (double*)part, (double*)S, st);
}

int launch_long_dft_gather(const LongArgs& a, const DftArgs& d, const void* psi, d4* out, bool f32, cudaStream_t st) {
    return f32 ? dft_gather_t(a, d, (const float*)psi, out, st) : dft_gather_t(a, d, (const double*)psi, out, st);
}

bool long_dft_ok(const DftArgs& d, int Pc) {
    const int pcp = long_small_pcp(Pc), nky4 = (d.nky + 3) / 4;
    return pcp > 0 && d.nkx * nky4 * (pcp / DFT_LT) <= 256 && 16 * (size_t)d.nmode * pcp <= 200 * 1024;
}

}  // namespace sog
