// S1: validate + canonicalise + bin particles into near-field cells, deterministic
// counting sort (cell-major, original index order inside a cell), gather to sorted SoA.
#pragma once
#include "kernels_common.cuh"

namespace sog {

// R14 canonical wrap x - L floor((x + L/2)/L) in [-L/2, L/2), rounded step by step
// exactly like the oracle (no contraction).
__device__ __forceinline__ double canon(double x, double L) {
    double halfL = 0.5 * L;
    double f = floor(__ddiv_rn(__dadd_rn(x, halfL), L));
    double r = __dsub_rn(x, __dmul_rn(L, f));
    if (r >= halfL) r = __dsub_rn(r, L);
    return r;
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__global__ void k_prepare(const double* __restrict__ xyz, const double* __restrict__ q, int N, CellGeo g,
                          d4* __restrict__ pos, int* __restrict__ cell, int* __restrict__ count,
                          unsigned* __restrict__ flags, double* __restrict__ qsums) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    double qa = 0.0, qabs = 0.0;
    if (i < N) {
        double x = xyz[3 * (size_t)i], y = xyz[3 * (size_t)i + 1], z = xyz[3 * (size_t)i + 2];
        double qi = q[i];
        unsigned f = 0;
        if (!isfinite(x) || !isfinite(y) || !isfinite(z) || !isfinite(qi)) f |= FLAG_NONFINITE;
        if (g.px) x = canon(x, g.Lx);   // x-slab ranks receive own + halo particles in the slab frame
        y = canon(y, g.Ly);
        if (!(fabs(z) <= 0.5 * g.Lz)) f |= FLAG_ZRANGE;
        int cx = 0, cy = 0, cz = 0;
        if (!f) {
            cx = clampi((int)floor((x - g.x0) * g.sx), 0, g.ncx - 1);
            cy = clampi((int)floor((y + 0.5 * g.Ly) * g.sy), 0, g.ncy - 1);
            cz = clampi((int)floor((z + 0.5 * g.Lz) * g.sz), 0, g.ncz - 1);
        }
        if (f) { x = y = z = 0.0; qi = isfinite(qi) ? qi : 0.0; cx = cy = cz = 0; atomicOr(flags, f); }  // keep kernels in bounds
        int c = (cx * g.ncy + cy) * g.ncz + cz;
        pos[i] = d4{x, y, z, qi};
        cell[i] = c;
        atomicAdd(&count[c], 1);
        qa = qi;
        qabs = fabs(qi);
    }
    // block reduction of sum q and sum |q| (neutrality check)
    for (int o = 16; o > 0; o >>= 1) {
        qa += __shfl_xor_sync(0xffffffffu, qa, o);
        qabs += __shfl_xor_sync(0xffffffffu, qabs, o);
    }
    __shared__ double red[2][32];
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) { red[0][wid] = qa; red[1][wid] = qabs; }
    __syncthreads();
    if (wid == 0) {
        int nw = blockDim.x >> 5;
        qa = lane < nw ? red[0][lane] : 0.0;
        qabs = lane < nw ? red[1][lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) {
            qa += __shfl_xor_sync(0xffffffffu, qa, o);
            qabs += __shfl_xor_sync(0xffffffffu, qabs, o);
        }
        if (lane == 0) { atomicAdd(&qsums[0], qa); atomicAdd(&qsums[1], qabs); }
    }
}

// Exclusive scan of count[0..n) into start[0..n]; one block of 1024 threads.
__global__ void __launch_bounds__(1024) k_scan(const int* __restrict__ count, int n, int* __restrict__ start,
                                               int* __restrict__ cursor) {
    __shared__ int part[1024];
    int t = threadIdx.x;
    int chunk = (n + 1023) / 1024;
    int lo = min(n, t * chunk), hi = min(n, lo + chunk);
    int s = 0;
    for (int i = lo; i < hi; ++i) s += count[i];
    part[t] = s;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        int v = t >= o ? part[t - o] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    int run = part[t] - s;
    for (int i = lo; i < hi; ++i) {
        start[i] = run;
        cursor[i] = run;
        run += count[i];
    }
    if (t == 1023) start[n] = part[1023];
}

__global__ void k_scatter(const int* __restrict__ cell, int N, int* __restrict__ cursor, int* __restrict__ tmp) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N) tmp[atomicAdd(&cursor[cell[i]], 1)] = i;
}

// One warp per cell: order the cell's members by (z, original index) (rank counting), gather
// the sorted SoA and the permutation.  Cells are z-major inside an (x,y) column, so every
// column is z-sorted (the near-field z windows rely on it); the order is deterministic.
__global__ void k_cellsort(const int* __restrict__ start, int ncell, const int* __restrict__ tmp,
                           const d4* __restrict__ pos, d4* __restrict__ pos_s, int* __restrict__ perm,
                           int* __restrict__ iperm) {
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (warp >= ncell) return;
    int s = start[warp], n = start[warp + 1] - s;
    if (n <= 64) {
        // the cell's (z, index) pairs in registers (two per lane), ranks by broadcasting each pair:
        // the same order as the loop below without its dependent global loads per comparison
        const int e0 = lane, e1 = lane + 32;
        const int m0 = e0 < n ? tmp[s + e0] : 0, m1 = e1 < n ? tmp[s + e1] : 0;
        const double z0 = e0 < n ? pos[m0].z : 0.0, z1 = e1 < n ? pos[m1].z : 0.0;
        int r0 = 0, r1 = 0;
        for (int f = 0; f < n; ++f) {
            const int src = f & 31;
            const double zo = __shfl_sync(0xffffffffu, f < 32 ? z0 : z1, src);
            const int o = __shfl_sync(0xffffffffu, f < 32 ? m0 : m1, src);
            r0 += (zo < z0 || (zo == z0 && o < m0));
            r1 += (zo < z1 || (zo == z1 && o < m1));
        }
        if (e0 < n) {
            perm[s + r0] = m0;
            iperm[m0] = s + r0;
            st_d4(&pos_s[s + r0], ld_d4(&pos[m0]));
        }
        if (e1 < n) {
            perm[s + r1] = m1;
            iperm[m1] = s + r1;
            st_d4(&pos_s[s + r1], ld_d4(&pos[m1]));
        }
        return;
    }
    for (int e = lane; e < n; e += 32) {
        int my = tmp[s + e];
        const double zm = pos[my].z;
        int rank = 0;
        if (n <= 4096) {
            for (int f = 0; f < n; ++f) {
                const int o = tmp[s + f];
                const double zo = pos[o].z;
                rank += (zo < zm || (zo == zm && o < my));
            }
        } else {
            rank = e;   // pathological clustering: arrival order (z windows fall back to full columns)
        }
        perm[s + rank] = my;
        iperm[my] = s + rank;                  // inverse: caller / local index -> sorted index
        st_d4(&pos_s[s + rank], ld_d4(&pos[my]));
    }
}

}  // namespace sog
