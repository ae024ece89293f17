// Host planning and launchers of the shared-memory FFT kernels (kernels_fft.cuh).
#include <algorithm>
#include <cmath>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
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

// ---- TMA z pass (fp64): tensor maps through the driver entry point (no libcuda link) ----
namespace {
PFN_cuTensorMapEncodeTiled_v12000 tmap_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}
}  // namespace

bool encode_tmap_f64(void* map128, const void* base, int rank, const unsigned long long* dims,
                     const unsigned long long* strides_bytes, const unsigned* box) {
    auto enc = tmap_encode();
    if (!enc || rank < 1 || rank > 5) return false;
    cuuint64_t d[5], st[4];
    cuuint32_t bx[5], es[5];
    for (int i = 0; i < rank; ++i) {
        if (dims[i] == 0) return false;
        d[i] = dims[i];
        bx[i] = box[i];
        es[i] = 1;
        if (i + 1 < rank) st[i] = strides_bytes[i];
    }
    static_assert(sizeof(CUtensorMap) == 128, "tensor map size");
    return enc(reinterpret_cast<CUtensorMap*>(map128), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)rank,
               const_cast<void*>(base), d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {
// 2D fp64 tensor [rows][cols] (row pitch cols doubles), box [box_rows][box_cols]
bool tmap_2d(ZrTmap& m, const void* base, long long cols, long long rows, int box_cols, int box_rows) {
    if (rows <= 0) return false;
    const unsigned long long dims[2] = {(unsigned long long)cols, (unsigned long long)rows};
    const unsigned long long strides[1] = {(unsigned long long)cols * sizeof(double)};
    const unsigned box[2] = {(unsigned)box_cols, (unsigned)box_rows};
    return encode_tmap_f64(&m, base, 2, dims, strides, box);
}
}  // namespace

template <int E, int B>
int zpass_t_go(void* X, long long M, int zin0, int nin, int zout0, int nout, const FftStages& f, const void* tw,
               const void* mult, cudaStream_t st) {
    const int Tc = f.n / E;
    if (f.n % E || B * Tc > 512) return 1;
    for (int s = 0; s < f.nst; ++s)
        if (E % f.R[s]) return 1;
    ZrTmap tin, tout, tmul;
    if (!tmap_2d(tin, X, 2 * M, nin, 2 * B, ZR_BOX) || !tmap_2d(tout, X, 2 * M, nout, 2 * B, ZR_BOX) ||
        !tmap_2d(tmul, mult, M, f.n, B, ZR_BOX))
        return 1;
    const size_t sh = zr_smem(f.n, B);
    if (sh > 227 * 1024) return 1;
    if (cudaFuncSetAttribute(k_zpass_t<E, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) != cudaSuccess)
        return 2;
    k_zpass_t<E, B><<<(unsigned)((M + B - 1) / B), B * Tc, sh, st>>>(tin, tout, tmul, M, zin0, nin, zout0, nout, f,
                                                                    (const double2*)tw);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

// 1 = not supported here (the caller keeps k_zpass_r): fp32, odd M, another (E, B)
int launch_zpass_t(void* X, long long M, int zin0, int nin, int zout0, int nout, const FftStages& f, const void* tw,
                   const void* mult, int E, int B, cudaStream_t st) {
    if (M % 2 || M * 2 > (1LL << 31)) return 1;
#define SOG_ZT(EE, BB) \
    if (E == EE && B == BB) return zpass_t_go<EE, BB>(X, M, zin0, nin, zout0, nout, f, tw, mult, st);
    SOG_ZT(10, 2) SOG_ZT(8, 2) SOG_ZT(12, 2) SOG_ZT(16, 2)
#undef SOG_ZT
    return 1;
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

// ---------------------------------------------------------------------------------------
// plane FFTs (rows r2c / c2r along y, complex along x): E elements per thread, BR rows or B columns
// per CTA; 1 = configuration not supported (the caller keeps the library transform)
template <typename T, int E, int BR>
int rows_go(bool inv, const void* in, void* out, long long nrows, int nyh, const FftStages& f, const void* tw,
            const void* wpost, cudaStream_t st) {
    using C = typename Cplx<T>::C;
    const int Tc = f.n / E;
    if (f.n % E || BR * Tc > (E >= 16 ? 256 : 512) || nyh != f.n + 1) return 1;
    for (int s = 0; s < f.nst; ++s)
        if (E % f.R[s]) return 1;
    const int ntw = f.tw[f.nst - 1] + f.Ns[f.nst - 1] * (f.R[f.nst - 1] - 1);
    const size_t sh = sizeof(C) * ((size_t)(f.n + 1) * BR + ntw);
    if (sh > 227 * 1024) return 1;
    const unsigned grid = (unsigned)((nrows + BR - 1) / BR);
    if (!inv) {
        if (cudaFuncSetAttribute(k_rows_r2c<T, E, BR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) != cudaSuccess)
            return 2;
        k_rows_r2c<T, E, BR><<<grid, BR * Tc, sh, st>>>((const T*)in, (C*)out, nrows, nyh, f, (const C*)tw,
                                                         (const C*)wpost);
    } else {
        if (cudaFuncSetAttribute(k_rows_c2r<T, E, BR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) != cudaSuccess)
            return 2;
        k_rows_c2r<T, E, BR><<<grid, BR * Tc, sh, st>>>((const C*)in, (T*)out, nrows, nyh, f, (const C*)tw,
                                                         (const C*)wpost);
    }
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

template <typename T, int E, int B>
int xfft_go(bool inv, void* X, long long planes, int Ix, int nyh, const FftStages& f, const void* tw, cudaStream_t st) {
    using C = typename Cplx<T>::C;
    const int Tc = Ix / E;
    if (f.n != Ix || Ix % E || B * Tc > (E >= 16 ? 256 : 512)) return 1;
    for (int s = 0; s < f.nst; ++s)
        if (E % f.R[s]) return 1;
    const int ntw = f.tw[f.nst - 1] + f.Ns[f.nst - 1] * (f.R[f.nst - 1] - 1);
    const size_t sh = sizeof(C) * ((size_t)Ix * B + ntw);
    if (sh > 227 * 1024) return 1;
    const int nbk = (nyh + B - 1) / B;
    const long long nblk = planes * nbk;
    if (nblk > 0x7fffffffLL) return 1;
    auto k = inv ? k_xfft<T, E, B, true> : k_xfft<T, E, B, false>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) != cudaSuccess) return 2;
    k<<<(unsigned)nblk, B * Tc, sh, st>>>((C*)X, Ix, nyh, nbk, f, (const C*)tw);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

#define SOG_PF_CASES(M_) M_(20, 2) M_(8, 4) M_(8, 8) M_(8, 16) M_(10, 4) M_(10, 8) M_(10, 16) M_(16, 4) M_(16, 8) M_(16, 16) \
    M_(20, 4) M_(20, 8) M_(20, 16) M_(12, 4) M_(12, 8) M_(12, 16)

int launch_rows_fft(bool inv, const void* in, void* out, long long nrows, int nyh, const FftStages& f, const void* tw,
                    const void* wpost, bool f32, int E, int BR, cudaStream_t st) {
#define C_(EE, BB)                                                                                  \
    if (E == EE && BR == BB)                                                                        \
        return f32 ? rows_go<float, EE, BB>(inv, in, out, nrows, nyh, f, tw, wpost, st)             \
                   : rows_go<double, EE, BB>(inv, in, out, nrows, nyh, f, tw, wpost, st);
    SOG_PF_CASES(C_)
#undef C_
    return 1;
}

int launch_xfft(bool inv, void* X, long long planes, int Ix, int nyh, const FftStages& f, const void* tw, bool f32,
                int E, int B, cudaStream_t st) {
#define C_(EE, BB)                                                                                  \
    if (E == EE && B == BB)                                                                         \
        return f32 ? xfft_go<float, EE, BB>(inv, X, planes, Ix, nyh, f, tw, st)                      \
                   : xfft_go<double, EE, BB>(inv, X, planes, Ix, nyh, f, tw, st);
    SOG_PF_CASES(C_)
#undef C_
    return 1;
}

bool plane_fft_supported(int n, int E, int B) {
    if (n % E || (n / E) * B > (E >= 16 ? 256 : 512) || sizeof(double2) * (size_t)(n + 1) * (B + 1) > 227 * 1024) return false;
    bool ok = false;
#define C_(EE, BB) ok = ok || (E == EE && B == BB);
    SOG_PF_CASES(C_)
#undef C_
    return ok;
}

}  // namespace sog
