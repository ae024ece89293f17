// x-slab decomposition: particle halos, the pencil transposes of the
// distributed mid-range FFT, Psi halo planes, long-range ownership masks.
//
// Rank r owns x in [X_r, X_{r+1}) and the mid-grid planes [I_r, I_r + Ixr), Ixr = Ix / R.  Its
// local particle set is [own | left halo | right halo]; halo particles are the neighbours'
// particles within H of the shared boundary, carried in the slab frame (x shifted by +-Lx
// across the periodic seam).  Local mid grids are [Izs][Ixk][Iy] with interior planes at
// local x in [XO, XO + Ixr); the FFT is 2D (z, y) per x plane, an all-to-all to ky chunks,
// 1D along x, and back.
#pragma once
#include <cuComplex.h>
#include "kernels_common.cuh"

namespace sog {

// own particles: d4 copy, halo flags (bit 0: within H of the left edge, bit 1: of the right
// edge) and the rank's input status, summed into st[] (block-reduced, then one atomic per block):
//   st[0] particles outside the rank's x slab (after the canonical wrap, R14)
//   st[1] non-finite position or charge, st[2] z outside [-Lz/2, Lz/2] (S1 rules)
//   st[4] sum q, st[5] sum |q| over the finite charges (neutrality)
// Particles that fail a check are parked at the slab centre with their (finite) charge so every
// later kernel stays in bounds; the evaluation is rejected on every rank after the agreement.
static __global__ void k_slab_flags(const double* __restrict__ xyz, const double* __restrict__ q, int n, double Lx,
                                    double Lz, double xlo, double xhi, double H, d4* __restrict__ own,
                                    int* __restrict__ fl, int* __restrict__ fr, double* __restrict__ st) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (i < n) {
        double x = xyz[3 * (size_t)i];
        const double y = xyz[3 * (size_t)i + 1], z = xyz[3 * (size_t)i + 2], qi = q[i];
        const bool fin = isfinite(x) && isfinite(y) && isfinite(z) && isfinite(qi);
        const double halfL = 0.5 * Lx;
        if (fin) {
            const double f = floor(__ddiv_rn(__dadd_rn(x, halfL), Lx));      // canonical wrap (R14)
            x = __dsub_rn(x, __dmul_rn(Lx, f));
            if (x >= halfL) x = __dsub_rn(x, Lx);
        }
        const bool inslab = fin && x >= xlo && x < xhi;
        const bool zok = fin && fabs(z) <= 0.5 * Lz;
        v[0] = fin && !inslab ? 1.0 : 0.0;
        v[1] = fin ? 0.0 : 1.0;
        v[2] = fin && !zok ? 1.0 : 0.0;
        v[3] = isfinite(qi) ? qi : 0.0;
        v[4] = isfinite(qi) ? fabs(qi) : 0.0;
        const bool ok = inslab && zok;
        const double xm = 0.5 * (xlo + xhi);
        own[i] = ok ? d4{x, y, z, qi} : d4{xm, 0.0, 0.0, v[3]};
        fl[i] = ok && x < xlo + H ? 1 : 0;
        fr[i] = ok && x >= xhi - H ? 1 : 0;
    }
#pragma unroll
    for (int k = 0; k < 5; ++k)
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    __shared__ double red[5][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0)
        for (int k = 0; k < 5; ++k) red[k][wid] = v[k];
    __syncthreads();
    if (threadIdx.x < 5) {
        double t = 0.0;
        for (int w = 0; w < nw; ++w) t += red[threadIdx.x][w];
        const int slot = threadIdx.x < 3 ? threadIdx.x : threadIdx.x + 1;
        if (t != 0.0) atomicAdd(&st[slot], t);
    }
}

// st[3] += halo sends over capacity (the select cannot overflow: its buffers hold every own
// particle) + a host-side capacity violation
static __global__ void k_halo_status(const int* __restrict__ nsel, int cap, int host_err, double* __restrict__ st) {
    st[3] += double((nsel[0] > cap) + (nsel[1] > cap) + host_err);
}

static __global__ void k_shift_x(d4* __restrict__ p, const int* __restrict__ n, double dx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < *n) p[i].x += dx;
}

// local input arrays (xyz N x 3, q) from [own | left halo | right halo]
static __global__ void k_slab_local(const d4* __restrict__ own, int nown, const d4* __restrict__ hl, int nl,
                                    const d4* __restrict__ hr, int nr, double* __restrict__ xyz, double* __restrict__ q) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nown + nl + nr) return;
    const d4 v = i < nown ? own[i] : (i < nown + nl ? hl[i - nown] : hr[i - nown - nl]);
    xyz[3 * (size_t)i] = v.x;
    xyz[3 * (size_t)i + 1] = v.y;
    xyz[3 * (size_t)i + 2] = v.z;
    q[i] = v.w;
}

// all-to-all packing of the 2D spectra spec2 [Izs][Ixr][nyh] <-> send/recv blocks
//   block for ky chunk s: [Izs][Ixr][kyc_s], kyc_s = min(kc, nyh - s kc), stored at s * blk
static __global__ void k_pack_fwd(const cuDoubleComplex* __restrict__ spec2, cuDoubleComplex* __restrict__ buf, int Izs,
                                  int Ixr, int nyh, int kc, int R, size_t blk) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t tot = (size_t)Izs * Ixr * nyh;
    if (idx >= tot) return;
    const int ky = int(idx % nyh);
    const size_t zx = idx / nyh;
    const int s = ky / kc, k = ky - s * kc, kyc = min(kc, nyh - s * kc);
    buf[s * blk + zx * kyc + k] = spec2[idx];
}

static __global__ void k_unpack_bwd(const cuDoubleComplex* __restrict__ buf, cuDoubleComplex* __restrict__ spec2,
                                    int Izs, int Ixr, int nyh, int kc, int R, size_t blk) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t tot = (size_t)Izs * Ixr * nyh;
    if (idx >= tot) return;
    const int ky = int(idx % nyh);
    const size_t zx = idx / nyh;
    const int s = ky / kc, k = ky - s * kc, kyc = min(kc, nyh - s * kc);
    spec2[idx] = buf[s * blk + zx * kyc + k];
}

// received blocks from rank s ([Izs][Ixr][kyc]) <-> x pencils specx [Izs][kyc][Ix]
static __global__ void k_unpack_fwd(const cuDoubleComplex* __restrict__ buf, cuDoubleComplex* __restrict__ specx,
                                    int Izs, int Ixr, int Ix, int kyc, size_t blk) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;   // over [Izs][kyc][Ix]
    const size_t tot = (size_t)Izs * kyc * Ix;
    if (idx >= tot) return;
    const int x = int(idx % Ix);
    const size_t zk = idx / Ix;
    const int k = int(zk % kyc), z = int(zk / kyc);
    const int s = x / Ixr, xl = x - s * Ixr;
    specx[idx] = buf[s * blk + ((size_t)z * Ixr + xl) * kyc + k];
}

static __global__ void k_pack_bwd(const cuDoubleComplex* __restrict__ specx, cuDoubleComplex* __restrict__ buf, int Izs,
                                  int Ixr, int Ix, int kyc, size_t blk) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t tot = (size_t)Izs * kyc * Ix;
    if (idx >= tot) return;
    const int x = int(idx % Ix);
    const size_t zk = idx / Ix;
    const int k = int(zk % kyc), z = int(zk / kyc);
    const int s = x / Ixr, xl = x - s * Ixr;
    buf[s * blk + ((size_t)z * Ixr + xl) * kyc + k] = specx[idx];
}

// S5 on x pencils: specx [Izs][kyc][Ix] *= mult(kz, kx, ky0 + k)  (same tables as k_mid_scale)
static __global__ void k_scale_pencil(cuDoubleComplex* __restrict__ specx, int Izs, int kyc, int Ix, int ky0, int nyh,
                                      int L, const double* __restrict__ A, const double* __restrict__ Tx,
                                      const double* __restrict__ Ty, const double* __restrict__ Tz) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t tot = (size_t)Izs * kyc * Ix;
    if (idx >= tot) return;
    const int x = int(idx % Ix);
    const size_t zk = idx / Ix;
    const int k = int(zk % kyc), z = int(zk / kyc);
    double m = 0.0;
    for (int l = 0; l < L; ++l)
        m = fma(A[l] * Tz[(size_t)l * Izs + z] * Tx[(size_t)l * Ix + x], Ty[(size_t)l * nyh + ky0 + k], m);
    const cuDoubleComplex v = specx[idx];
    specx[idx] = make_cuDoubleComplex(v.x * m, v.y * m);
}

// planes [x0, x0 + nx) of a [Izs][Ixk][Iy] grid <-> contiguous [Izs][nx][Iy]
static __global__ void k_planes_pack(const double* __restrict__ g, double* __restrict__ buf, int Izs, int Ixk, int Iy,
                                     int x0, int nx) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t tot = (size_t)Izs * nx * Iy;
    if (idx >= tot) return;
    const int y = int(idx % Iy);
    const size_t zx = idx / Iy;
    const int xl = int(zx % nx), z = int(zx / nx);
    buf[idx] = g[((size_t)z * Ixk + x0 + xl) * Iy + y];
}

static __global__ void k_planes_unpack(const double* __restrict__ buf, double* __restrict__ g, int Izs, int Ixk, int Iy,
                                       int x0, int nx) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t tot = (size_t)Izs * nx * Iy;
    if (idx >= tot) return;
    const int y = int(idx % Iy);
    const size_t zx = idx / Iy;
    const int xl = int(zx % nx), z = int(zx / nx);
    g[((size_t)z * Ixk + x0 + xl) * Iy + y] = buf[idx];
}

// long range: own particles only (halo particles are owned by the neighbours)
static __global__ void k_own_mask(const d4* __restrict__ pos_s, const int* __restrict__ perm, int n, int nown,
                                  d4* __restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    d4 v = pos_s[k];
    if (perm[k] >= nown) v.w = 0.0;
    out[k] = v;
}

}  // namespace sog
