// Host planning and launchers of the shared-memory FFT kernels (kernels_fft.cuh).
#include <algorithm>
#include <cmath>
#include <vector>
#include "kernels_fft.cuh"
#include "launch.h"

namespace sog {

// radices (largest first): 8, 7, 5, 4, 3, 2; false when n is not 7-smooth or too long
bool fft_plan_stages(int n, FftStages& f, std::vector<double2>& tw, int E) {
    f = FftStages();
    f.n = n;
    if (n < 1 || n > FFT_MAXE) return false;
    std::vector<int> rs;
    int m = n;
    for (int r : {8, 7, 5, 4, 3, 2})
        while (m % r == 0 && (E == 0 || E % r == 0)) {
            rs.push_back(r);
            m /= r;
        }
    if (m != 1 || (int)rs.size() > FFT_MAXST) return false;
    tw.clear();
    int Ns = 1;
    for (size_t s = 0; s < rs.size(); ++s) {
        const int R = rs[s];
        f.R[s] = R;
        f.Ns[s] = Ns;
        f.mNs[s] = Ns > 1 ? (unsigned)((0x100000000ULL + Ns - 1) / Ns) : 0u;
        f.tw[s] = (int)tw.size();
        for (int k = 0; k < Ns; ++k)
            for (int r = 1; r < R; ++r) {
                // e^{-2 pi i k r / (Ns R)} in long double, rounded once
                const long double a = -2.0L * 3.14159265358979323846264338327950288L * (long double)(k * r) /
                                      (long double)(Ns * R);
                tw.push_back(make_double2((double)cosl(a), (double)sinl(a)));
            }
        Ns *= R;
    }
    f.nst = (int)rs.size();
    return true;
}

int fft_cols_per_cta(int n) {
    int B = 1;
    while (2 * B * n <= FFT_MAXE && B < 16) B *= 2;
    return B;
}

template <typename T, int LM, int B>
int zpass_go(void* X, long long M, int nyh, int zin0, int nin, int zout0, int nout, const FftStages& f, const void* tw,
             int L, const double* A, const double* Tx, int Ix, const double* Ty, const double* Tz, cudaStream_t st) {
    using C = typename Cplx<T>::C;
    int ntw = 0;
    for (int s = 0; s < f.nst; ++s) ntw = f.tw[s] + f.Ns[s] * (f.R[s] - 1);
    const size_t sh = sizeof(C) * ((size_t)f.n * B + ntw) + sizeof(T) * B * LM;
    if (sh > 227 * 1024) return 1;
    if (cudaFuncSetAttribute(k_zpass<T, LM, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) != cudaSuccess)
        return 2;
    const unsigned grid = (unsigned)((M + B - 1) / B);
    k_zpass<T, LM, B><<<grid, FFT_NTHR, sh, st>>>((C*)X, M, nyh, zin0, nin, zout0, nout, f, (const C*)tw, ntw, L, A,
                                                  Tx, Ix, Ty, Tz);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

template <typename T, int LM>
int zpass_b(void* X, long long M, int nyh, int zin0, int nin, int zout0, int nout, const FftStages& f, const void* tw,
            int L, const double* A, const double* Tx, int Ix, const double* Ty, const double* Tz, cudaStream_t st) {
    switch (fft_cols_per_cta(f.n)) {
        case 1: return zpass_go<T, LM, 1>(X, M, nyh, zin0, nin, zout0, nout, f, tw, L, A, Tx, Ix, Ty, Tz, st);
        case 2: return zpass_go<T, LM, 2>(X, M, nyh, zin0, nin, zout0, nout, f, tw, L, A, Tx, Ix, Ty, Tz, st);
        case 4: return zpass_go<T, LM, 4>(X, M, nyh, zin0, nin, zout0, nout, f, tw, L, A, Tx, Ix, Ty, Tz, st);
        case 8: return zpass_go<T, LM, 8>(X, M, nyh, zin0, nin, zout0, nout, f, tw, L, A, Tx, Ix, Ty, Tz, st);
        default: return zpass_go<T, LM, 16>(X, M, nyh, zin0, nin, zout0, nout, f, tw, L, A, Tx, Ix, Ty, Tz, st);
    }
}

template <typename T>
int zpass_l(void* X, long long M, int nyh, int zin0, int nin, int zout0, int nout, const FftStages& f,
            const void* tw, int L, const double* A, const double* Tx, int Ix, const double* Ty, const double* Tz,
            cudaStream_t st) {
    if (L <= 8) return zpass_b<T, 8>(X, M, nyh, zin0, nin, zout0, nout, f, tw, L, A, Tx, Ix, Ty, Tz, st);
    if (L <= 16) return zpass_b<T, 16>(X, M, nyh, zin0, nin, zout0, nout, f, tw, L, A, Tx, Ix, Ty, Tz, st);
    if (L <= 24) return zpass_b<T, 24>(X, M, nyh, zin0, nin, zout0, nout, f, tw, L, A, Tx, Ix, Ty, Tz, st);
    if (L <= 32) return zpass_b<T, 32>(X, M, nyh, zin0, nin, zout0, nout, f, tw, L, A, Tx, Ix, Ty, Tz, st);
    if (L <= 48) return zpass_b<T, 48>(X, M, nyh, zin0, nin, zout0, nout, f, tw, L, A, Tx, Ix, Ty, Tz, st);
    if (L <= 64) return zpass_b<T, 64>(X, M, nyh, zin0, nin, zout0, nout, f, tw, L, A, Tx, Ix, Ty, Tz, st);
    return 1;
}

// register-resident z pass: E elements per thread, every radix of the plan divides E
template <typename T, int E, int B>
int zpass_r_go(void* X, long long M, int zin0, int nin, int zout0, int nout, const FftStages& f, const void* tw,
               const void* mult, cudaStream_t st) {
    using C = typename Cplx<T>::C;
    const int Tc = f.n / E;
    if (f.n % E || B * Tc > 512) return 1;
    for (int s = 0; s < f.nst; ++s)
        if (E % f.R[s]) return 1;
    const size_t sh = sizeof(C) * (size_t)f.n * B;
    if (cudaFuncSetAttribute(k_zpass_r<T, E, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) != cudaSuccess)
        return 2;
    k_zpass_r<T, E, B><<<(unsigned)((M + B - 1) / B), B * Tc, sh, st>>>((C*)X, M, zin0, nin, zout0, nout, f,
                                                                     (const C*)tw, (const T*)mult);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int launch_zpass_r(void* X, long long M, int zin0, int nin, int zout0, int nout, const FftStages& f, const void* tw,
                   const void* mult, bool f32, int E, int B, cudaStream_t st) {
#define SOG_ZR(EE, BB)                                                                                          \
    if (E == EE && B == BB)                                                                                     \
        return f32 ? zpass_r_go<float, EE, BB>(X, M, zin0, nin, zout0, nout, f, tw, mult, st)                   \
                   : zpass_r_go<double, EE, BB>(X, M, zin0, nin, zout0, nout, f, tw, mult, st);
    SOG_ZR(10, 2) SOG_ZR(10, 4) SOG_ZR(8, 2) SOG_ZR(8, 4) SOG_ZR(12, 2) SOG_ZR(12, 4) SOG_ZR(16, 2) SOG_ZR(16, 4)
#undef SOG_ZR
    return 1;
}

int build_mult_table(void* out, long long M, int nyh, int Izs, int L, const double* A, const double* Tx, int Ix,
                     const double* Ty, const double* Tz, bool f32, void* tmp, cudaStream_t st) {
    const long long n = M * Izs;
    double* d = f32 ? (double*)tmp : (double*)out;
    k_mult_table<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d, M, nyh, Izs, L, A, Tx, Ix, Ty, Tz);
    if (f32) k_mult_table_f<<<(unsigned)((n + 255) / 256), 256, 0, st>>>((float*)out, d, n);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int launch_zpass(void* X, long long M, int nyh, int zin0, int nin, int zout0, int nout, const FftStages& f,
                 const void* tw, int L, const double* A, const double* Tx, int Ix, const double* Ty, const double* Tz,
                 bool f32, cudaStream_t st) {
    return f32 ? zpass_l<float>(X, M, nyh, zin0, nin, zout0, nout, f, tw, L, A, Tx, Ix, Ty, Tz, st)
               : zpass_l<double>(X, M, nyh, zin0, nin, zout0, nout, f, tw, L, A, Tx, Ix, Ty, Tz, st);
}

}  // namespace sog
