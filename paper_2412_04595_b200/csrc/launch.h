// Host launchers for the templated stencil kernels (one translation unit per family so the
// instantiations compile in parallel).  Return 0 on success, 1 for an unsupported template
// parameter, 2 for a CUDA launch error (query cudaGetLastError()).
#pragma once
#include <cuda_runtime.h>
#include "kernels_common.cuh"

namespace sog {
struct MidArgs;
struct LongArgs;
struct LongTileArgs;
struct MidTileArgs;
int launch_mid_spread_tile(const MidTileArgs& t, int P, const int4* g0, double* grid, cudaStream_t st);
int launch_stencil_origins(const d4* pos, int N, const MidArgs& a, int has_mid, double lhx, double lhy, double lhpx,
                           double lhpy, int4* g0, cudaStream_t st);
int launch_long_gather2(const LongArgs& a, int Pl, const double* psi, double* psiT, d4* out, double gx, double gy,
                        cudaStream_t st);
int long_pcmax(int Pc);
int launch_long_spread_tile(const LongTileArgs& t, int Pl, double* grid, cudaStream_t st);
int launch_mid_gather(const MidArgs& a, int P, const double* psi, d4* out, double gx, double gy, double gz,
                      cudaStream_t st);
}  // namespace sog
