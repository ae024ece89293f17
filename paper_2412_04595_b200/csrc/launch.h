// Host launchers for the templated stencil kernels (one translation unit per family so the
// instantiations compile in parallel).  Return 0 on success, 1 for an unsupported template
// parameter, 2 for a CUDA launch error (query cudaGetLastError()).
#pragma once
#include <cuComplex.h>
#include <cuda_runtime.h>
#include <vector>
#include "kernels_common.cuh"

namespace sog {
struct MidArgs;
struct MidSortArgs;
struct MidZArgs;
struct LongArgs;
struct LongTileArgs;
struct DftArgs;
int launch_stencil_origins(const d4* pos, int N, const MidArgs& a, int has_mid, double lhx, double lhy, double lhpx,
                           double lhpy, int4* g0, cudaStream_t st);
int launch_mid_sort_keys(const int4* g0, int N, const MidSortArgs& s, int* key, int* count, cudaStream_t st);
int launch_mid_sort_place(const int* key, int N, int* cursor, int* tmp, const int* mstart, int nkeys, const d4* pos_s,
                          const int4* g0, int p, d4* mpos, int4* minfo, cudaStream_t st);
int launch_mid_spread_z(const MidZArgs& a, int P, int nseg, void* grid, bool f32, cudaStream_t st);
int launch_mid_gather_z(const MidZArgs& a, int P, int nseg, int nmid, const void* psi, d4* out, bool f32,
                        cudaStream_t st);
size_t mid_gather_smem(int P);
// fp64 tensor map (CUtensorMap, 128 bytes) through the driver entry point; dims / box innermost first,
// strides_bytes of dims 1..rank-1.  false: no driver entry point or an invalid shape
bool encode_tmap_f64(void* map128, const void* base, int rank, const unsigned long long* dims,
                     const unsigned long long* strides_bytes, const unsigned* box);
int launch_zfft_transpose(const void* in, void* out, int nz, long long M, int Izs, int z0, bool fwd, bool f32,
                          cudaStream_t st);
struct FftStages;
struct Near4Args;
struct Near3Args;
struct NearPoly;
int launch_near3p(const Near3Args& a, const NearPoly& p, int ncell, cudaStream_t st);
struct Near5Args;
// each pair once (kernels_near5.cuh), then out += the 13 forward-shell partials
int launch_near5(const Near5Args& a, const NearPoly& p, int ncell, cudaStream_t st);
int launch_near_fold(d4* out, const d4* part, int N, cudaStream_t st);
// target-stationary near field (kernels_near4.cuh): 1 = unsupported degree / warps
int launch_near4(const Near4Args& a, const NearPoly& p, int nw, cudaStream_t st);
size_t near4_smem(int cap, int nw);
// shared-memory FFT (kernels_fft.cuh): stage plan + twiddles (false: length not supported)
// E > 0: radices restricted to divisors of E (register-resident z pass)
bool fft_plan_stages(int n, FftStages& f, std::vector<double2>& tw, int E = 0);
// z pass of the mid solver: FFT along z, S5 scaling, inverse FFT, in place on the plane spectra
int launch_zpass(void* X, long long M, int nyh, int zin0, int nin, int zout0, int nout, const FftStages& f,
                 const void* tw, int L, const double* A, const double* Tx, int Ix, const double* Ty, const double* Tz,
                 bool f32, cudaStream_t st);
// the same with TMA row blocks (fp64, B = 2); 1 = not supported (use launch_zpass_r)
int launch_zpass_t(void* X, long long M, int zin0, int nin, int zout0, int nout, const FftStages& f, const void* tw,
                   const void* mult, int E, int B, cudaStream_t st);
int launch_zpass_r(void* X, long long M, int zin0, int nin, int zout0, int nout, const FftStages& f, const void* tw,
                   const void* mult, bool f32, int E, int B, cudaStream_t st);
// plane FFTs of S4 / S6 (kernels_fft.cuh): rows r2c (inv: c2r) of nrows real rows of 2 f.n samples <->
// nyh = f.n + 1 complex; x FFT of length Ix of every (plane, ky) column of X [planes][Ix][nyh], in
// place.  wpost = e^{-2 pi i k / (2 f.n)}, k <= f.n.  1 = (E, B) not compiled / too large.
int launch_rows_fft(bool inv, const void* in, void* out, long long nrows, int nyh, const FftStages& f, const void* tw,
                    const void* wpost, bool f32, int E, int BR, cudaStream_t st);
int launch_xfft(bool inv, void* X, long long planes, int Ix, int nyh, const FftStages& f, const void* tw, bool f32,
                int E, int B, cudaStream_t st);
bool plane_fft_supported(int n, int E, int B);
// S5 multiplier table [Izs][M] (fp64, or fp32 through the fp64 scratch tmp)
int build_mult_table(void* out, long long M, int nyh, int Izs, int L, const double* A, const double* Tx, int Ix,
                     const double* Ty, const double* Tz, bool f32, void* tmp, cudaStream_t st);
int launch_scale_pencil_z(void* W, int Ix, int nyh, int Izs, int L, const double* A, const double* Tx,
                          const double* Ty, const double* Tz, bool f32, cudaStream_t st);
int mid_spread_emax();
int launch_mid_scale(void* spec, int Ix, int Izs, int nyh, int L, const double* A, const double* Tx, const double* Ty,
                     const double* Tz, bool f32, cudaStream_t st);
int launch_long_gather2(const LongArgs& a, int Pl, const double* psi, double* psiT, d4* out, double gx, double gy,
                        cudaStream_t st);
int long_pcmax(int Pc);
int launch_long_spread_tile(const LongTileArgs& t, int Pl, double* grid, cudaStream_t st);
// register-tiled spread per column tile (k_long_spread_tgemm); 1 = unsupported shape (use the tile kernel)
int launch_long_spread_tgemm(const LongTileArgs& t, double* grid, cudaStream_t st);
bool long_small_ok(int Ilx, int Ily, int Pc);
int long_small_pcp(int Pc);
int launch_long_spread_gemm(const LongArgs& a, const int4* g0, double gx, double gy, int nblk, void* part, void* grid,
                            bool f32, cudaStream_t st);
int launch_long_gather_bc(const LongArgs& a, const int4* g0, const void* psi, d4* out, bool f32, cudaStream_t st);
int launch_long_scale(const void* in, void* out, const double* K, int nmode, int Pc, bool f32, cudaStream_t st);
int launch_long_to_nodes(const double* in, double* out, int G, int Pc, const double* M, cudaStream_t st);
// long range without FFT (Alg. 3): type-1 sums into S~[n][mode] complex, type-2 sums to the particles
int launch_long_dft_spread(const LongArgs& a, const DftArgs& d, int nblk, void* part, void* S, bool f32,
                           cudaStream_t st);
int launch_long_dft_gather(const LongArgs& a, const DftArgs& d, const void* psi, d4* out, bool f32, cudaStream_t st);
bool long_dft_ok(const DftArgs& d, int Pc);
// exclusive prefix sum of in[0..n) into out[0..n] (out[n] = total); temp from scan_temp_bytes
size_t scan_temp_bytes(int n);
int launch_exclusive_scan(const int* in, int* out, int n, void* temp, size_t temp_bytes, cudaStream_t st);
size_t select_temp_bytes(int n);
int launch_select_flagged(const d4* in, const int* flags, d4* out, int* nsel, int n, void* temp, size_t temp_bytes,
                          cudaStream_t st);
}  // namespace sog
