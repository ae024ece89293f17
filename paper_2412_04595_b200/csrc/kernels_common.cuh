// Device-side helpers shared by the SOG kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#ifdef SOG_ASSERTS
#include <cassert>
#define SOG_ASSERT(c) assert(c)
#else
#define SOG_ASSERT(c) ((void)0)
#endif

namespace sog {

struct __align__(32) d4 {
    double x, y, z, w;
};

__device__ __forceinline__ d4 ld_d4(const d4* p) {
    const double2* q = reinterpret_cast<const double2*>(p);
    double2 a = __ldg(q), b = __ldg(q + 1);
    return d4{a.x, a.y, b.x, b.y};
}
__device__ __forceinline__ void st_d4(d4* p, d4 v) {
    double2* q = reinterpret_cast<double2*>(p);
    q[0] = make_double2(v.x, v.y);
    q[1] = make_double2(v.z, v.w);
}

// Validation flag bits written by k_prepare.
enum : unsigned { FLAG_NONFINITE = 1u, FLAG_ZRANGE = 2u };

// Geometry of the near-field cell grid (cells >= r_c; y periodic; z clamped; x periodic for a
// whole-box plan, or a non-periodic extended slab [x0, x0 + Lx) for an x-slab rank).
struct CellGeo {
    double Lx, Ly, Lz;
    double invLx, invLy;
    int ncx, ncy, ncz;
    double sx, sy, sz;      // cells per unit length (nc / L)
    double x0;              // x of the first cell edge (-Lx/2 for the whole box)
    int px;                 // 1: x periodic (whole box), 0: x-slab (no x images)
    int nzr;                // z neighbour reach in cells: cell height >= r_c / nzr (near field)
};

// One axis of a window stencil on a uniform grid x_g = (g - I/2) h (R6):
// nearest grid point g0 = floor(x/h + I/2 + 1/2) computed with explicitly rounded
// operations (no FMA contraction) so the integer decision matches the oracle bit for bit.
__device__ __forceinline__ int stencil_g0(double x, double h, double half_plus) {
    return (int)floor(__dadd_rn(__ddiv_rn(x, h), half_plus));
}

// Window weights W(x_g - x) = exp(-S ((x_g - x)/H)^2) at the P points g0-p..g0+p, and
// dW/dx_particle = 2 S (x_g - x)/H^2 W (R11).  invH2S = S / H^2.
template <int P, bool GRAD>
__device__ __forceinline__ void window_weights(double x, int g0, double h, double halfI,
                                               double invH2S, double* W, double* dW) {
    constexpr int p = (P - 1) / 2;
#pragma unroll
    for (int a = 0; a < P; ++a) {
        double d = ((double)(g0 - p + a) - halfI) * h - x;
        double e = exp(-invH2S * d * d);
        W[a] = e;
        if (GRAD) dW[a] = 2.0 * invH2S * d * e;
    }
}

// Same weights by the Gaussian recurrence (2 exps per axis instead of P):
//   d_k = d_0 + k h,  W_{k+1} = W_k R_k,  R_k = exp(-a h (2 d_0 + (2k+1) h)),  R_{k+1} = R_k gamma,
//   gamma = exp(-2 a h^2)   (a = S/H^2).  Relative deviation from direct exp ~ P ulps.
template <int P, bool GRAD>
__device__ __forceinline__ void window_weights_rec(double x, int g0, double h, double halfI, double invH2S,
                                                   double gamma, double* W, double* dW) {
    constexpr int p = (P - 1) / 2;
    const double d0 = ((double)(g0 - p) - halfI) * h - x;
    double w = exp(-invH2S * d0 * d0);
    double r = exp(-invH2S * h * (2.0 * d0 + h));
#pragma unroll
    for (int a = 0; a < P; ++a) {
        W[a] = w;
        if (GRAD) dW[a] = 2.0 * invH2S * (d0 + a * h) * w;
        w *= r;
        r *= gamma;
    }
}

// R6-KB (Kaiser-Bessel window as polynomials, Remark rmk::PWindow P:477-480): the particle's
// offset from its nearest grid point u = x/h + I/2 - g0 in [-1/2, 1/2], rounded as the oracle does
__device__ __forceinline__ double kb_offset(double x, double h, double halfI, int g0) {
    return __dsub_rn(__dadd_rn(__ddiv_rn(x, h), halfI), (double)g0);
}

// R6-KB monomial table, carried by value in the kernel arguments (constant bank): c[n P + j] is
// the u^n coefficient of stencil point j, n = 0..P+3 (degrees nu < P + 3 are zero-padded), so
// with P a compile-time constant every coefficient is an immediate constant-bank operand.
constexpr int KB_PMAX = 17;
constexpr int KB_TAB = KB_PMAX * (KB_PMAX + 4);
struct KBTab {
    double c[KB_TAB];
};

// W_j(u) = sum_n c[n P + j] u^n at the P stencil points (Horner, P independent chains) and dW_j/du
template <int P, bool GRAD>
__device__ __forceinline__ void kb_weights(double u, const KBTab& t, double* W, double* dW) {
    static_assert(P <= KB_PMAX, "KB window support above KB_PMAX");
    constexpr int NU = P + 3;
#pragma unroll
    for (int j = 0; j < P; ++j) {
        W[j] = t.c[NU * P + j];
        if (GRAD) dW[j] = 0.0;
    }
#pragma unroll
    for (int n = NU - 1; n >= 0; --n) {
#pragma unroll
        for (int j = 0; j < P; ++j) {
            if (GRAD) dW[j] = fma(dW[j], u, W[j]);
            W[j] = fma(W[j], u, t.c[n * P + j]);
        }
    }
}

// runtime-P front end: f(j, W_j, dW_j/du) for j < P (P odd in [5, KB_PMAX])
template <int P, bool GRAD, class F>
__device__ __forceinline__ void kb_emit(double u, const KBTab& t, F& f) {
    double W[P], dW[P];
    kb_weights<P, GRAD>(u, t, W, dW);
#pragma unroll
    for (int j = 0; j < P; ++j) f(j, W[j], GRAD ? dW[j] : 0.0);
}
template <bool GRAD, class F>
__device__ __forceinline__ void kb_emit_rt(int P, double u, const KBTab& t, F& f) {
    switch (P) {
        case 5: kb_emit<5, GRAD>(u, t, f); break;
        case 7: kb_emit<7, GRAD>(u, t, f); break;
        case 9: kb_emit<9, GRAD>(u, t, f); break;
        case 11: kb_emit<11, GRAD>(u, t, f); break;
        case 13: kb_emit<13, GRAD>(u, t, f); break;
        case 15: kb_emit<15, GRAD>(u, t, f); break;
        case 17: kb_emit<17, GRAD>(u, t, f); break;
        default: break;
    }
}

__device__ __forceinline__ int wrap(int g, int I) {
    g %= I;
    return g < 0 ? g + I : g;
}

// c += a b on the FP64 tensor path: mma.sync m8n8k4 f64 (DMMA).  Fragments (lane l, gid = l / 4,
// tig = l % 4): a = A[gid][tig] (8 x 4, row), b = B[tig][gid] (4 x 8, col), c = C[gid][2 tig + {0, 1}].
// 256 FMAs per warp instruction on the same FP64 pipe as DFMA (profiles/r02_fp64_peak.json), with
// two register operands per lane instead of one shared-memory operand per FMA.
__device__ __forceinline__ void dmma_884(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

}  // namespace sog
