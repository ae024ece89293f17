// Mid-range stencil kernels (Algorithm 1) and their launchers.
#include <cstdlib>
#include <cstring>
#include <vector>
#include "kernels_mid.cuh"
#include "launch.h"

namespace sog {

#define SOG_ODD_P(M) M(5) M(7) M(9) M(11) M(13) M(15) M(17) M(19) M(21) M(23) M(25)

int launch_stencil_origins(const d4* pos, int N, const MidArgs& a, int has_mid, double lhx, double lhy, double lhpx,
                           double lhpy, int4* g0, cudaStream_t st) {
    k_stencil_origins<<<(N + 255) / 256, 256, 0, st>>>(pos, N, a, has_mid, lhx, lhy, lhpx, lhpy, g0);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int launch_mid_sort_keys(const int4* g0, int N, const MidSortArgs& s, int* key, int* count, cudaStream_t st) {
    k_mid_key<<<(N + 255) / 256, 256, 0, st>>>(g0, N, s, key, count);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int launch_mid_sort_place(const int* key, int N, int* cursor, int* tmp, const int* mstart, int nkeys, const d4* pos_s,
                          const int4* g0, int p, d4* mpos, int4* minfo, cudaStream_t st) {
    k_mid_scatter<<<(N + 255) / 256, 256, 0, st>>>(key, N, cursor, tmp);
    k_mid_bucket<<<(int)(((long)nkeys * 32 + 255) / 256), 256, 0, st>>>(mstart, nkeys, tmp, pos_s, g0, p, mpos, minfo);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

// KB-window instantiations (R6-KB): supports up to 17 in fp64 (tol >= 2e-14 needs P <= 17),
// up to 11 in fp32 mode (tol >= 1e-5)
template <int P, typename T>
constexpr bool kb_compiled() { return sizeof(T) == 8 ? P <= 17 : P <= 11; }

template <int P, typename T, bool KB>
int spread_go_w(const MidZArgs& a, int nseg, T* grid, cudaStream_t st) {
    using R = SRec<P, T>;
    const size_t sh = R::BYTES;
    if (cudaFuncSetAttribute(k_mid_spread_z<P, T, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) !=
        cudaSuccess)
        return 2;
    k_mid_spread_z<P, T, KB><<<dim3(a.ntout * a.nty, nseg), R::NTHR, sh, st>>>(a, grid);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

template <int P, bool KB, int NP>
int spread_go_m(const MidZArgs& a, int nseg, double* grid, cudaStream_t st) {
    using R = SRec<P, double, NP>;
    const size_t sh = R::BYTES;
    auto k = k_mid_spread_zm<P, KB, NP>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) != cudaSuccess ||
        cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100) != cudaSuccess)
        return 2;
    k<<<dim3(a.ntout * a.nty, nseg), R::NTHR, sh, st>>>(a, grid);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

// fp64 accumulates on the FP64 tensor path (DMMA) with 4 producer warps unless SOG_SPREAD_MMA=0
// (the DFMA consumer); SOG_SPREAD_MMA = 2 or 3 selects 2 or 3 producer warps at P = 11 (GS window).
// c5: DFMA 7.87 ms, DMMA with 2 / 3 / 4 producer warps 5.56 / 5.45 / 5.13 ms.
static int spread_mma() {
    static const int v = std::getenv("SOG_SPREAD_MMA") ? std::atoi(std::getenv("SOG_SPREAD_MMA")) : 1;
    return v;
}

template <int P, typename T>
int spread_go(const MidZArgs& a, int nseg, T* grid, cudaStream_t st) {
    if constexpr (sizeof(T) == 8) {
        const int v = spread_mma();
        if constexpr (P == 11) {
            if (!a.kb && v == 2) return spread_go_m<P, false, 2>(a, nseg, grid, st);
            if (!a.kb && v == 3) return spread_go_m<P, false, 3>(a, nseg, grid, st);
        }
        if (v != 0) {
            if (!a.kb) return spread_go_m<P, false, 4>(a, nseg, grid, st);
            if constexpr (kb_compiled<P, T>()) return spread_go_m<P, true, 4>(a, nseg, grid, st);
            return 1;
        }
    }
    if (!a.kb) return spread_go_w<P, T, false>(a, nseg, grid, st);
    if constexpr (kb_compiled<P, T>()) return spread_go_w<P, T, true>(a, nseg, grid, st);
    return 1;
}

int launch_mid_spread_z(const MidZArgs& a, int P, int nseg, void* grid, bool f32, cudaStream_t st) {
    switch (P) {
#define C_(P_)                                                                                  \
    case P_:                                                                                    \
        return f32 ? spread_go<P_, float>(a, nseg, (float*)grid, st) : spread_go<P_, double>(a, nseg, (double*)grid, st);
        SOG_ODD_P(C_)
#undef C_
        default: return 1;
    }
}

// TMA boxes for the gather ring (fp64): the tensor map of Psi [Izs][Ixk][Iy] and the bank-grouped
// column assignment for the dense box pitch WY (kernels_mid.cuh, GatherTma).  SOG_GATHER_TMA=0: off.
template <int P, typename T, bool KB>
void gather_tma(const MidZArgs& a, const T* psi, GatherTma& tm) {
    using G = GRing<P, T, KB>;
    constexpr int NR = G::NR, WX = G::WX, WY = G::WY;
    std::memset(&tm, 0, sizeof tm);
    static const bool on = !(std::getenv("SOG_GATHER_TMA") && std::atoi(std::getenv("SOG_GATHER_TMA")) == 0);
    if (sizeof(T) != 8 || !on || 2 * NR > 8 || (WY * sizeof(T)) % 16 || ((size_t)a.Iy * sizeof(T)) % 16) return;
    const unsigned long long dims[3] = {(unsigned long long)a.Iy, (unsigned long long)a.Ixk, (unsigned long long)a.Izs};
    const unsigned long long strides[2] = {(unsigned long long)a.Iy * sizeof(T),
                                           (unsigned long long)a.Ixk * a.Iy * sizeof(T)};
    const unsigned box[3] = {(unsigned)WY, (unsigned)WX, 1u};
    if (!encode_tmap_f64(tm.map, psi, 3, dims, strides, box)) return;
    // member i of residue class r = (a WY + b) mod 16 -> half-warp group i, lane position r; the
    // members past the last group fill the free lanes (a 2-way conflict there)
    for (int i = 0; i < 128; ++i) tm.col[i] = -1;
    std::vector<int> cls[16], spill;
    for (int aa = 0; aa < P; ++aa)
        for (int bb = 0; bb < P; ++bb) cls[(aa * WY + bb) % 16].push_back(aa * P + bb);
    for (int r = 0; r < 16; ++r)
        for (size_t i = 0; i < cls[r].size(); ++i) {
            if ((int)i < 2 * NR) tm.col[(i / 2) * 32 + (i % 2) * 16 + r] = (short)cls[r][i];
            else spill.push_back(cls[r][i]);
        }
    for (int c : spill)
        for (int i = 128 - 1; i >= 0; --i)
            if (i < 32 * NR && tm.col[i] < 0) { tm.col[i] = (short)c; break; }
    tm.ok = 1;
}

template <int P, typename T, bool KB>
int gather_ring(const MidZArgs& a, int nseg, const T* psi, d4* out, cudaStream_t st) {
    const size_t sh = GRing<P, T, KB>::BYTES;
    if (cudaFuncSetAttribute(k_mid_gather_z<P, T, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh) !=
        cudaSuccess)
        return 2;
    GatherTma tm;
    gather_tma<P, T, KB>(a, psi, tm);
    k_mid_gather_z<P, T, KB><<<dim3(a.ntout * a.nty, nseg), 256, sh, st>>>(a, psi, out, tm);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

template <int P, typename T>
int gather_go(const MidZArgs& a, int nseg, int nmid, const T* psi, d4* out, cudaStream_t st) {
    if (!a.kb) {
        if constexpr (GRing<P, T, false>::FITS) return gather_ring<P, T, false>(a, nseg, psi, out, st);
    } else {
        if constexpr (kb_compiled<P, T>() && GRing<P, T, true>::FITS) return gather_ring<P, T, true>(a, nseg, psi, out, st);
    }
    if constexpr (sizeof(T) == 4) {
        return 1;   // fp32 mode: ring gather only
    } else {
        k_mid_gather_g<P><<<148 * 8, 256, 0, st>>>(a, psi, out, nmid);
        return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
    }
}

int launch_mid_gather_z(const MidZArgs& a, int P, int nseg, int nmid, const void* psi, d4* out, bool f32,
                        cudaStream_t st) {
    switch (P) {
#define C_(P_)                                                                                             \
    case P_:                                                                                               \
        return f32 ? gather_go<P_, float>(a, nseg, nmid, (const float*)psi, out, st)                      \
                   : gather_go<P_, double>(a, nseg, nmid, (const double*)psi, out, st);
        SOG_ODD_P(C_)
#undef C_
        default: return 1;
    }
}

int mid_spread_emax() { return SRec<11>::EMAX; }

size_t mid_gather_smem(int P) {
    switch (P) {
#define C_(P_) case P_: return GRing<P_>::FITS ? GRing<P_>::BYTES : 1;
        SOG_ODD_P(C_)
#undef C_
        default: return 0;
    }
}

template <typename C>
int mid_scale_go(C* spec, int Ix, int Izs, int nyh, int L, const double* A, const double* Tx, const double* Ty,
                 const double* Tz, cudaStream_t st) {
    dim3 g((nyh + 127) / 128, (Izs * Ix + MS_ROWS - 1) / MS_ROWS);
    if (L <= 8) k_mid_scale<8, C><<<g, 128, 0, st>>>(spec, Ix, Izs, nyh, L, A, Tx, Ty, Tz);
    else if (L <= 16) k_mid_scale<16, C><<<g, 128, 0, st>>>(spec, Ix, Izs, nyh, L, A, Tx, Ty, Tz);
    else if (L <= 24) k_mid_scale<24, C><<<g, 128, 0, st>>>(spec, Ix, Izs, nyh, L, A, Tx, Ty, Tz);
    else if (L <= 32) k_mid_scale<32, C><<<g, 128, 0, st>>>(spec, Ix, Izs, nyh, L, A, Tx, Ty, Tz);
    else if (L <= 48) k_mid_scale<48, C><<<g, 128, 0, st>>>(spec, Ix, Izs, nyh, L, A, Tx, Ty, Tz);
    else if (L <= 64) k_mid_scale<64, C><<<g, 128, 0, st>>>(spec, Ix, Izs, nyh, L, A, Tx, Ty, Tz);
    else return 1;
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int launch_mid_scale(void* spec, int Ix, int Izs, int nyh, int L, const double* A, const double* Tx, const double* Ty,
                     const double* Tz, bool f32, cudaStream_t st) {
    return f32 ? mid_scale_go((cuComplex*)spec, Ix, Izs, nyh, L, A, Tx, Ty, Tz, st)
               : mid_scale_go((cuDoubleComplex*)spec, Ix, Izs, nyh, L, A, Tx, Ty, Tz, st);
}

}  // namespace sog

namespace sog {

template <typename C>
int zfft_tr_go(const C* in, C* out, int nz, long long M, int Izs, int z0, bool fwd, cudaStream_t st) {
    dim3 g((unsigned)((M + TR_T - 1) / TR_T), (nz + TR_T - 1) / TR_T);
    if (fwd) k_tr_xz<C><<<g, TR_T * 8, 0, st>>>(in, out, nz, M, Izs, z0);
    else k_tr_zx<C><<<g, TR_T * 8, 0, st>>>(in, out, nz, M, Izs, z0);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int launch_zfft_transpose(const void* in, void* out, int nz, long long M, int Izs, int z0, bool fwd, bool f32,
                          cudaStream_t st) {
    return f32 ? zfft_tr_go((const cuComplex*)in, (cuComplex*)out, nz, M, Izs, z0, fwd, st)
               : zfft_tr_go((const cuDoubleComplex*)in, (cuDoubleComplex*)out, nz, M, Izs, z0, fwd, st);
}

template <typename C>
int scale_z_go(C* W, int Ix, int nyh, int Izs, int L, const double* A, const double* Tx, const double* Ty,
               const double* Tz, cudaStream_t st) {
    const long long M = (long long)Ix * nyh;
    dim3 g((Izs + 127) / 128, (unsigned)((M + MS_ROWS - 1) / MS_ROWS));
    if (L <= 8) k_scale_pencil_z<8, C><<<g, 128, 0, st>>>(W, Ix, nyh, Izs, L, A, Tx, Ty, Tz);
    else if (L <= 16) k_scale_pencil_z<16, C><<<g, 128, 0, st>>>(W, Ix, nyh, Izs, L, A, Tx, Ty, Tz);
    else if (L <= 24) k_scale_pencil_z<24, C><<<g, 128, 0, st>>>(W, Ix, nyh, Izs, L, A, Tx, Ty, Tz);
    else if (L <= 32) k_scale_pencil_z<32, C><<<g, 128, 0, st>>>(W, Ix, nyh, Izs, L, A, Tx, Ty, Tz);
    else if (L <= 48) k_scale_pencil_z<48, C><<<g, 128, 0, st>>>(W, Ix, nyh, Izs, L, A, Tx, Ty, Tz);
    else if (L <= 64) k_scale_pencil_z<64, C><<<g, 128, 0, st>>>(W, Ix, nyh, Izs, L, A, Tx, Ty, Tz);
    else return 1;
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int launch_scale_pencil_z(void* W, int Ix, int nyh, int Izs, int L, const double* A, const double* Tx,
                          const double* Ty, const double* Tz, bool f32, cudaStream_t st) {
    return f32 ? scale_z_go((cuComplex*)W, Ix, nyh, Izs, L, A, Tx, Ty, Tz, st)
               : scale_z_go((cuDoubleComplex*)W, Ix, nyh, Izs, L, A, Tx, Ty, Tz, st);
}

}  // namespace sog
