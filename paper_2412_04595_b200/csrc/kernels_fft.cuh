// Shared-memory mixed-radix FFT for the mid-range solver (Algorithm 1 steps 2-4).
//
// cuFFT is no longer used for the mid grid: the z-pruned 3D FFT, the S5 scaling and the inverse
// are done by these kernels, each one pass over HBM:
//   k_fft_rows   y:  real rows of Iy -> nyh complex (forward) / back (inverse)       [z][x][.]
//   k_fft_cols   x:  complex columns of Ix at stride nyh, B adjacent ky per CTA       [z][.][ky]
//   k_zpass      z:  FFT along z of B adjacent (x, ky) columns, zero padding of the input
//                    rows implicit, S5 multiply by mult(k) (Eq. eq::widehat-tilde),
//                    inverse FFT, store of the rows the gather reads -- one kernel, in place.
// A CTA holds its B transforms in shared memory as [n][B] (row = one index of the transform, B
// adjacent columns, so global rows are contiguous B-element segments) and runs Stockham autosort
// stages of radix 2, 3, 4, 5, 7 or 8 (7-smooth lengths, rule R5/R7): per stage every thread loads
// its butterflies into registers, multiplies by the stage twiddles (host table, long double),
// applies the radix-R DFT, a barrier, stores them in natural order, a barrier.  Forward sign
// e^{-2 pi i / n}, unnormalised (the 1/(Ix Iy Izs) of the inverse is folded into the S5 table,
// R12).  The inverse uses conj(FFT(conj(x))).
#pragma once
#include <cuComplex.h>
#include <type_traits>
#include "kernels_common.cuh"

namespace sog {

constexpr int FFT_MAXST = 24;
constexpr int FFT_NTHR = 512;        // threads per CTA
constexpr int FFT_MAXE = 2560;       // complex elements per CTA (n x B): <= 5 per thread in registers

struct FftStages {
    int n = 0, nst = 0;
    int R[FFT_MAXST] = {};           // radix of stage s
    int Ns[FFT_MAXST] = {};          // product of the earlier radices
    unsigned mNs[FFT_MAXST] = {};    // ceil(2^32 / Ns): j / Ns = umulhi(j, mNs) for j < 2^18
    int tw[FFT_MAXST] = {};          // offset of stage s's twiddles: [Ns][R-1] complex
};

template <typename T>
struct Cplx;
template <>
struct Cplx<double> {
    using C = double2;
};
template <>
struct Cplx<float> {
    using C = float2;
};

template <typename C>
__device__ __forceinline__ C cmul(C a, C b) {
    C r;
    r.x = a.x * b.x - a.y * b.y;
    r.y = a.x * b.y + a.y * b.x;
    return r;
}
template <typename C>
__device__ __forceinline__ C cadd(C a, C b) {
    a.x += b.x;
    a.y += b.y;
    return a;
}
template <typename C>
__device__ __forceinline__ C csub(C a, C b) {
    a.x -= b.x;
    a.y -= b.y;
    return a;
}
template <typename C>
__device__ __forceinline__ C mul_mi(C a) {   // -i a
    C r;
    r.x = a.y;
    r.y = -a.x;
    return r;
}

// radix-R DFT in registers, forward sign: y_k = sum_j v_j e^{-2 pi i j k / R}
template <int R, typename C>
__device__ __forceinline__ void dft_small(C* v) {
    using T = decltype(v[0].x);
    if constexpr (R == 2) {
        const C a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    } else if constexpr (R == 4) {
        const C t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]), t2 = cadd(v[1], v[3]), t3 = mul_mi(csub(v[1], v[3]));
        v[0] = cadd(t0, t2);
        v[2] = csub(t0, t2);
        v[1] = cadd(t1, t3);
        v[3] = csub(t1, t3);
    } else if constexpr (R == 8) {
        // two radix-4 DFTs of the even / odd entries, twiddles W8^k, radix-2 across
        C e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
        dft_small<4>(e);
        dft_small<4>(o);
        const T h = T(0.70710678118654752440084436210485);
        // o1 *= W8 = (1 - i)/sqrt2, o2 *= -i, o3 *= W8^3 = (-1 - i)/sqrt2
        C w1, w3;
        w1.x = h * (o[1].x + o[1].y);
        w1.y = h * (o[1].y - o[1].x);
        w3.x = h * (o[3].y - o[3].x);
        w3.y = -h * (o[3].x + o[3].y);
        o[1] = w1;
        o[2] = mul_mi(o[2]);
        o[3] = w3;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[k] = cadd(e[k], o[k]);
            v[k + 4] = csub(e[k], o[k]);
        }
    } else {
        // odd R (3, 5, 7): pairs b_p = v_p + v_{R-p}, d_p = v_p - v_{R-p};
        // y_k = v_0 + sum_p cos(2 pi p k / R) b_p - i sum_p sin(2 pi p k / R) d_p, y_{R-k} with +i
        static_assert(R == 3 || R == 5 || R == 7, "radix");
        constexpr int H = (R - 1) / 2;
        // cos / sin (2 pi m / R), m = 1..H (compile-time after unrolling)
        auto cs = [](int m) -> T {
            if (R == 3) return T(-0.5);
            if (R == 5) return m == 1 ? T(0.30901699437494742410229341718282) : T(-0.80901699437494742410229341718282);
            return m == 1 ? T(0.62348980185873353052500488400424)
                          : (m == 2 ? T(-0.22252093395631440428890256449679) : T(-0.90096886790241912623610231950745));
        };
        auto sn = [](int m) -> T {
            if (R == 3) return T(0.86602540378443864676372317075294);
            if (R == 5) return m == 1 ? T(0.95105651629515357211643933337938) : T(0.58778525229247312916870595463907);
            return m == 1 ? T(0.78183148246802980870844452667406)
                          : (m == 2 ? T(0.97492791218182360701813168299393) : T(0.43388373911755812047576833284836));
        };
        C b[H], d[H];
#pragma unroll
        for (int p = 1; p <= H; ++p) {
            b[p - 1] = cadd(v[p], v[R - p]);
            d[p - 1] = csub(v[p], v[R - p]);
        }
        const C a0 = v[0];
        C y0 = a0;
#pragma unroll
        for (int p = 0; p < H; ++p) y0 = cadd(y0, b[p]);
#pragma unroll
        for (int k = 1; k <= H; ++k) {
            C re = a0, im;
            im.x = T(0);
            im.y = T(0);
#pragma unroll
            for (int p = 1; p <= H; ++p) {
                const int m = (p * k) % R;                    // cos(2 pi m/R), sin(2 pi m/R)
                const T c = m <= H ? cs(m) : cs(R - m);
                const T s = m <= H ? sn(m) : -sn(R - m);
                re.x = fma(c, b[p - 1].x, re.x);
                re.y = fma(c, b[p - 1].y, re.y);
                im.x = fma(s, d[p - 1].x, im.x);
                im.y = fma(s, d[p - 1].y, im.y);
            }
            // -i * im = (im.y, -im.x)
            v[k].x = re.x + im.y;
            v[k].y = re.y - im.x;
            v[R - k].x = re.x - im.y;
            v[R - k].y = re.y + im.x;
        }
        v[0] = y0;
    }
}

// one Stockham stage of radix R over the B columns of buf [n][B] (in place through registers)
template <int R, int B, typename C>
__device__ __forceinline__ void fft_stage(C* buf, int n, int Ns, unsigned mNs, const C* __restrict__ tw, int tid) {
    constexpr int K = (FFT_MAXE + R * FFT_NTHR - 1) / (R * FFT_NTHR);   // butterflies per thread
    const int nb = n / R, total = nb * B;
    C v[K][R];
    int dst[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int t = tid + k * FFT_NTHR;
        dst[k] = -1;
        if (t < total) {
            const int b = t & (B - 1), j = t / B;
            const int q = Ns > 1 ? (int)__umulhi((unsigned)j, mNs) : j;
            const int jk = j - q * Ns;
#pragma unroll
            for (int r = 0; r < R; ++r) v[k][r] = buf[(j + r * nb) * B + b];
            if (Ns > 1) {
                const C* w = tw + jk * (R - 1);
#pragma unroll
                for (int r = 1; r < R; ++r) v[k][r] = cmul(v[k][r], w[r - 1]);
            }
            dft_small<R>(v[k]);
            dst[k] = (q * R * Ns + jk) * B + b;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k)
        if (dst[k] >= 0) {
#pragma unroll
            for (int r = 0; r < R; ++r) buf[dst[k] + r * Ns * B] = v[k][r];
        }
    __syncthreads();
}

// the host orders the stages by radix 8, 7, 5, 4, 3, 2 (fft_plan_stages); one loop per radix keeps
// each radix's registers separate
template <int B, typename C>
__device__ __forceinline__ void fft_run(C* buf, const FftStages& f, const C* __restrict__ tw, int tid) {
    int s = 0;
#define SOG_FFT_RADIX_LOOP(RR) \
    for (; s < f.nst && f.R[s] == RR; ++s) fft_stage<RR, B>(buf, f.n, f.Ns[s], f.mNs[s], tw + f.tw[s], tid);
    SOG_FFT_RADIX_LOOP(8)
    SOG_FFT_RADIX_LOOP(7)
    SOG_FFT_RADIX_LOOP(5)
    SOG_FFT_RADIX_LOOP(4)
    SOG_FFT_RADIX_LOOP(3)
    SOG_FFT_RADIX_LOOP(2)
#undef SOG_FFT_RADIX_LOOP
}

// ---------------------------------------------------------------------------------------
// z pass: X [planes][M] complex (M = Ix * nyh columns m = x * nyh + ky).  Input rows z in
// [zin0, zin0 + nin) are read from planes z - zin0 (the others are the zero padding), output rows
// z in [zout0, zout0 + nout) are written to planes z - zout0 (in place: a CTA reads all rows of
// its columns before it writes any).  Between the forward and inverse transforms: multiply by
// mult(k) = sum_{l < L} A_l Tx_l(x) Ty_l(ky) Tz_l(kz) (R12; A holds the 1/(Ix Iy Izs) of the
// unnormalised inverse).  One CTA per batch of B columns; the stage twiddles are staged in shared
// memory.
__device__ __forceinline__ void cp_async_c(void* dst, const double2* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_c(void* dst, const float2* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <typename T, int LM, int B>
__global__ void __launch_bounds__(FFT_NTHR, 2) k_zpass(typename Cplx<T>::C* __restrict__ X, long long M, int nyh,
                                                     int zin0, int nin, int zout0, int nout, FftStages f,
                                                     const typename Cplx<T>::C* __restrict__ twg, int ntw, int L,
                                                     const double* __restrict__ A, const double* __restrict__ Tx,
                                                     int Ix, const double* __restrict__ Ty,
                                                     const double* __restrict__ Tz) {
    using C = typename Cplx<T>::C;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int tid = threadIdx.x, n = f.n;
    C* bufs = reinterpret_cast<C*>(smraw);                // [n][B]
    C* tw = bufs + n * B;                                 // [ntw] stage twiddles
    T* fac = reinterpret_cast<T*>(tw + ntw);              // [LM][B]: A_l Tx_l(x) Ty_l(ky) per column
    for (int e = tid; e < ntw; e += FFT_NTHR) tw[e] = twg[e];
    C zero;
    zero.x = T(0);
    zero.y = T(0);
    C* buf = bufs;
    const long long m0 = (long long)blockIdx.x * B;
    const int nbc = (int)min((long long)B, M - m0);
    {
        const C* src = X + m0;
        for (int e = tid; e < nin * B; e += FFT_NTHR) {
            const int zr = e / B, b = e & (B - 1);
            if (b < nbc) cp_async_c(&buf[zin0 * B + e], &src[(size_t)zr * M + b]);
            else buf[zin0 * B + e] = zero;
        }
        cp_async_commit();
    }
    // z padding rows
    for (int e = tid; e < zin0 * B; e += FFT_NTHR) buf[e] = zero;
    for (int e = (zin0 + nin) * B + tid; e < n * B; e += FFT_NTHR) buf[e] = zero;
    for (int e = tid; e < B * LM; e += FFT_NTHR) {
        const int l = e / B, b = e & (B - 1);
        T v = T(0);
        if (b < nbc && l < L) {
            const long long m = m0 + b;
            const int x = int(m / nyh), ky = int(m - (long long)x * nyh);
            v = T(A[l] * Tx[(size_t)l * Ix + x] * Ty[(size_t)l * nyh + ky]);
        }
        fac[e] = v;
    }
    cp_async_wait0();
    __syncthreads();
    fft_run<B>(buf, f, tw, tid);
    // S5 (thread per element; the LM factor loads are independent and issued together, the B
    // threads of one kz share each Tz_l(kz) load), then conj for the inverse
    for (int e = tid; e < n * B; e += FFT_NTHR) {
        const int kz = e / B, b = e & (B - 1);
        T m = T(0);
#pragma unroll
        for (int l = 0; l < LM; ++l) m = fma(fac[l * B + b], T(__ldg(&Tz[(size_t)min(l, L - 1) * n + kz])), m);
        C v = buf[e];
        v.x *= m;
        v.y *= -m;
        buf[e] = v;
    }
    __syncthreads();
    fft_run<B>(buf, f, tw, tid);
    C* dst = X + m0;
    for (int e = tid; e < nout * B; e += FFT_NTHR) {
        const int zr = e / B, b = e & (B - 1);
        if (b < nbc) {
            C v = buf[zout0 * B + e];
            v.y = -v.y;
            dst[(size_t)zr * M + b] = v;
        }
    }
}

}  // namespace sog

namespace sog {

// ---------------------------------------------------------------------------------------
// Register-resident z pass (k_zpass_r).  Thread (b, tau) of a CTA owns the E elements
// x[tau + Tc k], k < E (Tc = n / E) of column b for the whole transform.  A Stockham stage of radix
// R (R | E) is E / R butterflies on the thread's own registers (butterfly j = tau + Tc u reads
// x[j + r n/R] = register u + r E/R); its outputs go to shared memory in natural order and the next
// stage reads its E registers back (one exchange per stage, two barriers).  After the last
// forward stage the outputs a thread holds are again x[tau + Tc k] (Ns R = n), so the S5 multiply
// and the first inverse stage need no exchange, and the inverse's last stage stores its registers
// straight to the output rows.  The twiddles come from the host table through L1 (__ldg).
template <int R, int E, int B, typename C>
__device__ __forceinline__ void zr_stage(C (&x)[E], C* buf, int tau, int Tc, int b, int Ns, unsigned mNs,
                                         const C* __restrict__ tw, bool last) {
    constexpr int U = E / R;
    static_assert(E % R == 0, "radix must divide the elements per thread");
#pragma unroll
    for (int u = 0; u < U; ++u) {
        C v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = x[u + r * U];
        const int j = tau + Tc * u;
        const int q = Ns > 1 ? (int)__umulhi((unsigned)j, mNs) : j;
        const int jk = j - q * Ns;
        if (Ns > 1) {
            const C* w = tw + jk * (R - 1);
#pragma unroll
            for (int r = 1; r < R; ++r) v[r] = cmul(v[r], w[r - 1]);   // shared or global (L1) table
        }
        dft_small<R>(v);
#pragma unroll
        for (int r = 0; r < R; ++r) x[u + r * U] = v[r];
    }
    if (last) return;                       // outputs already at tau + Tc k (see above)
    __syncthreads();                        // the previous exchange's reads are done
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int j = tau + Tc * u;
        const int q = Ns > 1 ? (int)__umulhi((unsigned)j, mNs) : j;
        const int jk = j - q * Ns;
        const int dst = q * R * Ns + jk;
#pragma unroll
        for (int r = 0; r < R; ++r) buf[(dst + r * Ns) * B + b] = x[u + r * U];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < E; ++k) x[k] = buf[(tau + Tc * k) * B + b];
}

template <int E, int B, typename C>
__device__ __forceinline__ void zr_fft(C (&x)[E], C* buf, int tau, int Tc, int b, const FftStages& f,
                                       const C* __restrict__ tw) {
    int s = 0;
#define SOG_ZR_LOOP(RR)                                                                                         \
    if constexpr (E % RR == 0)                                                                                  \
        for (; s < f.nst && f.R[s] == RR; ++s)                                                                  \
            zr_stage<RR, E, B>(x, buf, tau, Tc, b, f.Ns[s], f.mNs[s], tw + f.tw[s], s == f.nst - 1);
    SOG_ZR_LOOP(8)
    SOG_ZR_LOOP(7)
    SOG_ZR_LOOP(5)
    SOG_ZR_LOOP(4)
    SOG_ZR_LOOP(3)
    SOG_ZR_LOOP(2)
#undef SOG_ZR_LOOP
}

// ---- TMA helpers (raw PTX; tensor maps encoded on the host per launch) ----
__device__ __forceinline__ unsigned zr_sa(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void zr_mbar_init(unsigned long long* b, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(zr_sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void zr_mbar_expect(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(zr_sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void zr_mbar_wait(unsigned long long* b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "ZW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra ZW_%=;\n}" ::"r"(zr_sa(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void zr_tma_load(void* dst, const void* tmap, int c0, int c1, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            zr_sa(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(zr_sa(bar))
        : "memory");
}
__device__ __forceinline__ void zr_tma_store(const void* tmap, int c0, int c1, const void* src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(tmap), "r"(c0),
                 "r"(c1), "r"(zr_sa(src))
                 : "memory");
}

// Opaque 128-byte tensor map (CUtensorMap), passed by value as a __grid_constant__ parameter
struct __align__(64) ZrTmap {
    unsigned long long w[16];
};
constexpr int ZR_BOX = 256;          // rows per TMA box
constexpr int ZR_PAD = ZR_BOX + 8;   // staging rows past n (the last box may run past the transform)
// byte offset of the S5 rows (128-byte aligned, as every TMA destination) and the total staging
__host__ __device__ constexpr size_t zr_mb_off(int n, int B) { return ((size_t)(n + ZR_PAD) * B * 16 + 127) & ~size_t(127); }
__host__ __device__ constexpr size_t zr_smem(int n, int B) { return zr_mb_off(n, B) + (size_t)(n + ZR_PAD) * B * 8; }

// k_zpass_r with the column block moved by TMA (fp64): the CTA's B adjacent (x, ky) columns of
// the written planes arrive in shared memory as boxes of ZR_BOX rows x B complex (one elected
// thread, mbarrier completion; rows outside the written planes are zero-filled by the tensor
// map's bounds), the S5 table rows of the same columns likewise, and the result rows leave by
// TMA stores clipped to the rows the gather reads.  No L1 traffic for the 32-byte row segments
// that made the thread-load version L1-bound.  Staging starts on a 128-byte aligned row.
template <int E, int B>
__global__ void __launch_bounds__(512) k_zpass_t(const __grid_constant__ ZrTmap tin, const __grid_constant__ ZrTmap tout,
                                                 const __grid_constant__ ZrTmap tmul, long long M, int zin0, int nin,
                                                 int zout0, int nout, FftStages f, const double2* __restrict__ tw) {
    static_assert(128 % (16 * B) == 0, "128-byte row groups");
    constexpr int RA = 128 / (16 * B);                    // rows per 128 bytes of staging
    extern __shared__ __align__(128) unsigned char smraw[];
    const int n = f.n, Tc = n / E;
    double2* buf = reinterpret_cast<double2*>(smraw);                       // [n + ZR_PAD][B]
    double* mb = reinterpret_cast<double*>(smraw + zr_mb_off(n, B));        // [n + ZR_PAD][B]
    __shared__ unsigned long long bar[2];
    const int t = threadIdx.x, b = t & (B - 1), tau = t / B;
    const int m0 = (int)((long long)blockIdx.x * B);
    const int zi = zin0 - zin0 % RA;
    if (t == 0) {
        zr_mbar_init(&bar[0], 1);
        zr_mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (t == 0) {
        const int nbx = (zin0 + nin - zi + ZR_BOX - 1) / ZR_BOX;
        zr_mbar_expect(&bar[0], (unsigned)(nbx * ZR_BOX * B * 16));
        for (int j = 0; j < nbx; ++j) zr_tma_load(buf + (size_t)(zi + ZR_BOX * j) * B, &tin, 2 * m0, zi - zin0 + ZR_BOX * j, &bar[0]);
        const int nbm = (n + ZR_BOX - 1) / ZR_BOX;
        zr_mbar_expect(&bar[1], (unsigned)(nbm * ZR_BOX * B * 8));
        for (int j = 0; j < nbm; ++j) zr_tma_load(mb + (size_t)ZR_BOX * j * B, &tmul, m0, ZR_BOX * j, &bar[1]);
    }
    zr_mbar_wait(&bar[0], 0);
    double2 x[E];
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const int z = tau + Tc * k;
        x[k] = (z >= zin0 && z < zin0 + nin) ? buf[(size_t)z * B + b] : make_double2(0.0, 0.0);
    }
    zr_fft<E, B>(x, buf, tau, Tc, b, f, tw);
    zr_mbar_wait(&bar[1], 0);
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const double m = mb[(size_t)(tau + Tc * k) * B + b];
        x[k].x *= m;
        x[k].y *= -m;
    }
    zr_fft<E, B>(x, buf, tau, Tc, b, f, tw);
    __syncthreads();                                      // the last exchange's reads are done
#pragma unroll
    for (int k = 0; k < E; ++k) {
        double2 v = x[k];
        v.y = -v.y;
        buf[(size_t)(tau + Tc * k) * B + b] = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (t == 0) {
        const int zo = zout0 - zout0 % RA;
        const int nbo = (zout0 + nout - zo + ZR_BOX - 1) / ZR_BOX;
        for (int j = 0; j < nbo; ++j) zr_tma_store(&tout, 2 * m0, zo - zout0 + ZR_BOX * j, buf + (size_t)(zo + ZR_BOX * j) * B);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
}

template <typename T, int E, int B>
__global__ void __launch_bounds__(512) k_zpass_r(typename Cplx<T>::C* __restrict__ X, long long M, int zin0, int nin,
                                                 int zout0, int nout, FftStages f,
                                                 const typename Cplx<T>::C* __restrict__ tw,
                                                 const T* __restrict__ mult) {
    using C = typename Cplx<T>::C;
    extern __shared__ __align__(16) unsigned char smraw[];
    C* buf = reinterpret_cast<C*>(smraw);                 // [n][B] exchange buffer
    const int n = f.n, Tc = n / E;
    const int t = threadIdx.x, b = t & (B - 1), tau = t / B;   // blockDim.x == B * Tc
    const long long m0 = (long long)blockIdx.x * B;
    const bool col = m0 + b < M;
    const size_t stride = (size_t)Tc * M;                 // rows tau + Tc k, k = 0, 1, ...
    C x[E];
    {
        const C* src = X + (size_t)tau * M + m0 + b - (size_t)zin0 * M;
#pragma unroll
        for (int k = 0; k < E; ++k) {
            const int z = tau + Tc * k;
            C v;
            v.x = T(0);
            v.y = T(0);
            if (col && z >= zin0 && z < zin0 + nin) v = src[k * stride];
            x[k] = v;
        }
    }
    zr_fft<E, B>(x, buf, tau, Tc, b, f, tw);
    // S5 on the registers: mult [kz][m] (plan-time table, R12), conj for the inverse transform
    {
        const T* mrow = mult + (size_t)tau * M + m0 + b;
#pragma unroll
        for (int k = 0; k < E; ++k) {
            const T m = col ? __ldg(&mrow[k * stride]) : T(0);
            x[k].x *= m;
            x[k].y *= -m;
        }
    }
    zr_fft<E, B>(x, buf, tau, Tc, b, f, tw);
    if (col) {
        C* dst = X + (size_t)tau * M + m0 + b - (size_t)zout0 * M;
#pragma unroll
        for (int k = 0; k < E; ++k) {
            const int z = tau + Tc * k;
            if (z >= zout0 && z < zout0 + nout) {
                C v = x[k];
                v.y = -v.y;
                dst[k * stride] = v;
            }
        }
    }
}

// S5 multiplier table mult[kz][m] = sum_{l < L} A_l Tx_l(x) Ty_l(ky) Tz_l(kz), m = x nyh + ky (R12),
// written once at plan time for the register-resident z pass
static __global__ void k_mult_table(double* __restrict__ out, long long M, int nyh, int Izs, int L, const double* __restrict__ A,
                             const double* __restrict__ Tx, int Ix, const double* __restrict__ Ty,
                             const double* __restrict__ Tz) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= M * Izs) return;
    const int kz = int(e / M);
    const long long m = e - (long long)kz * M;
    const int x = int(m / nyh), ky = int(m - (long long)x * nyh);
    double v = 0.0;
    for (int l = 0; l < L; ++l) v = fma(A[l] * Tx[(size_t)l * Ix + x], Ty[(size_t)l * nyh + ky] * Tz[(size_t)l * Izs + kz], v);
    out[e] = v;
}
static __global__ void k_mult_table_f(float* __restrict__ out, const double* __restrict__ in, long long n) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) out[e] = (float)in[e];
}

// ---------------------------------------------------------------------------------------
// Plane FFTs of S4 / S6 (x and y), in place of a 2D r2c / c2r library transform of the z-pruned
// planes; both are register-resident like k_zpass_r (zr_fft), one pass over HBM each.
//
// Rows (y): a real row of Iy = 2 n2 samples is the complex sequence z_n = x_2n + i x_2n+1 of length
// n2; with Z = FFT_n2(z) and W = e^{-2 pi i / Iy} the half spectrum is, for k = 0 .. n2,
//   X_k = (Z_k + conj Z_{n2-k}) / 2 - i W^k (Z_k - conj Z_{n2-k}) / 2          (Z_{n2} = Z_0)
// and the unnormalised inverse (x_m = sum_k X_k e^{+2 pi i k m / Iy} over the Hermitian extension)
// is z = IFFT_n2(Z'), Z'_k = (X_k + conj X_{n2-k}) + i W^{-k} (X_k - conj X_{n2-k}), x_2n = Re z_n,
// x_2n+1 = Im z_n.  A CTA transforms BR rows (row = (plane, x)); thread (b, tau), b = t mod BR.
// wpost[k] = W^k, k = 0 .. n2 (host table, long double).
// the stage twiddles of plan f (ntw = sum of Ns (R - 1)) copied into shared memory
template <typename C>
__device__ __forceinline__ const C* stage_twiddles(C* sm, const C* __restrict__ tw, const FftStages& f) {
    const int ntw = f.tw[f.nst - 1] + f.Ns[f.nst - 1] * (f.R[f.nst - 1] - 1);
    for (int i = threadIdx.x; i < ntw; i += blockDim.x) sm[i] = tw[i];
    return sm;
}

template <typename T, int E, int BR>
__global__ void __launch_bounds__(E >= 16 ? 256 : 512, E >= 16 ? 2 : 1) k_rows_r2c(const T* __restrict__ in, typename Cplx<T>::C* __restrict__ out,
                                                  long long nrows, int nyh, FftStages f,
                                                  const typename Cplx<T>::C* __restrict__ tw,
                                                  const typename Cplx<T>::C* __restrict__ wpost) {
    using C = typename Cplx<T>::C;
    extern __shared__ __align__(16) unsigned char smraw[];
    C* buf = reinterpret_cast<C*>(smraw);                 // [n2 + 1][BR], then the stage twiddles
    const int n2 = f.n, Tc = n2 / E;
    const int t = threadIdx.x, b = t & (BR - 1), tau = t / BR;
    const long long r0 = (long long)blockIdx.x * BR;
    const C* stw = stage_twiddles(buf + (n2 + 1) * BR, tw, f);
    const C* src = reinterpret_cast<const C*>(in);        // row r = complex [r n2, r n2 + n2)
    const int nt = blockDim.x;                            // BR Tc: BR n2 = nt E samples
    {
        C v[E];                                           // all loads in flight before the stores
#pragma unroll
        for (int k = 0; k < E; ++k) {
            const int idx = t + k * nt, bb = idx & (BR - 1), n = idx / BR;
            v[k].x = T(0);
            v[k].y = T(0);
            if (r0 + bb < nrows) v[k] = src[(size_t)(r0 + bb) * n2 + n];
        }
#pragma unroll
        for (int k = 0; k < E; ++k) {
            const int idx = t + k * nt;
            buf[(idx / BR) * BR + (idx & (BR - 1))] = v[k];
        }
    }
    __syncthreads();
    C x[E];
#pragma unroll
    for (int k = 0; k < E; ++k) x[k] = buf[(tau + Tc * k) * BR + b];
    zr_fft<E, BR>(x, buf, tau, Tc, b, f, stw);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < E; ++k) buf[(tau + Tc * k) * BR + b] = x[k];
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk <= E; ++kk) {                     // BR nyh = nt E + BR outputs
        const int idx = t + kk * nt, bb = idx & (BR - 1), k = idx / BR;
        if (idx >= BR * nyh || r0 + bb >= nrows) continue;
        const C zk = buf[(k == n2 ? 0 : k) * BR + bb];
        const C zc = buf[(k == 0 || k == n2 ? 0 : n2 - k) * BR + bb];
        C fe, d;
        fe.x = T(0.5) * (zk.x + zc.x);                    // (Z_k + conj Z_{n2-k}) / 2
        fe.y = T(0.5) * (zk.y - zc.y);
        d.x = T(0.5) * (zk.x - zc.x);                     // (Z_k - conj Z_{n2-k}) / 2
        d.y = T(0.5) * (zk.y + zc.y);
        const C w = wpost[k];
        const C wd = cmul(w, d);
        C X;
        X.x = fe.x + wd.y;                                // fe - i W^k d
        X.y = fe.y - wd.x;
        out[(size_t)(r0 + bb) * nyh + k] = X;
    }
}

template <typename T, int E, int BR>
__global__ void __launch_bounds__(E >= 16 ? 256 : 512) k_rows_c2r(const typename Cplx<T>::C* __restrict__ in, T* __restrict__ out,
                                                  long long nrows, int nyh, FftStages f,
                                                  const typename Cplx<T>::C* __restrict__ tw,
                                                  const typename Cplx<T>::C* __restrict__ wpost) {
    using C = typename Cplx<T>::C;
    extern __shared__ __align__(16) unsigned char smraw[];
    C* buf = reinterpret_cast<C*>(smraw);                 // [nyh][BR] (then the exchange buffer), twiddles
    const int n2 = f.n, Tc = n2 / E;
    const int t = threadIdx.x, b = t & (BR - 1), tau = t / BR;
    const long long r0 = (long long)blockIdx.x * BR;
    const C* stw = stage_twiddles(buf + (n2 + 1) * BR, tw, f);
    const int nt = blockDim.x;                            // BR nyh = nt E + BR inputs
    {
        C v[E + 1];                                       // all loads in flight before the stores
#pragma unroll
        for (int kk = 0; kk <= E; ++kk) {
            const int idx = t + kk * nt, bb = idx & (BR - 1), k = idx / BR;
            v[kk].x = T(0);
            v[kk].y = T(0);
            if (idx < BR * nyh && r0 + bb < nrows) v[kk] = in[(size_t)(r0 + bb) * nyh + k];
        }
#pragma unroll
        for (int kk = 0; kk <= E; ++kk) {
            const int idx = t + kk * nt;
            if (idx < BR * nyh) buf[idx] = v[kk];         // [k][BR]: idx = k BR + bb
        }
    }
    __syncthreads();
    C x[E];
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const int n = tau + Tc * k;
        const C a = buf[n * BR + b], c = buf[(n2 - n) * BR + b];
        C s, d;
        s.x = a.x + c.x;                                  // X_n + conj X_{n2-n}
        s.y = a.y - c.y;
        d.x = a.x - c.x;                                  // X_n - conj X_{n2-n}
        d.y = a.y + c.y;
        C w = wpost[n];
        w.y = -w.y;                                       // W^{-n}
        const C wd = cmul(w, d);
        // Z' = s + i W^{-n} d; the inverse is conj(FFT(conj Z'))
        x[k].x = s.x - wd.y;
        x[k].y = -(s.y + wd.x);
    }
    zr_fft<E, BR>(x, buf, tau, Tc, b, f, stw);
    if (r0 + b < nrows) {
        C* dst = reinterpret_cast<C*>(out) + (size_t)(r0 + b) * n2;
#pragma unroll
        for (int k = 0; k < E; ++k) {
            C v = x[k];
            v.y = -v.y;                                   // (x_2n, x_2n+1) = conj
            dst[tau + Tc * k] = v;
        }
    }
}

// x: FFT of length Ix along x of every (plane, ky) column of X [planes][Ix][nyh], in place; a CTA
// owns B adjacent ky of one plane.  INV: the unnormalised inverse, conj(FFT(conj)).
template <typename T, int E, int B, bool INV>
__global__ void __launch_bounds__(E >= 16 ? 256 : 512, E >= 16 ? 2 : 1) k_xfft(typename Cplx<T>::C* __restrict__ X, int Ix, int nyh, int nbk, FftStages f,
                                              const typename Cplx<T>::C* __restrict__ tw) {
    using C = typename Cplx<T>::C;
    extern __shared__ __align__(16) unsigned char smraw[];
    C* buf = reinterpret_cast<C*>(smraw);                 // [Ix][B], then the stage twiddles
    const C* stw = stage_twiddles(buf + Ix * B, tw, f);
    const int Tc = Ix / E;
    const int t = threadIdx.x, b = t & (B - 1), tau = t / B;
    const int pz = blockIdx.x / nbk, ky = (blockIdx.x - pz * nbk) * B + b;
    const bool col = ky < nyh;
    C* base = X + ((size_t)pz * Ix + tau) * nyh + ky;
    const size_t stride = (size_t)Tc * nyh;
    C x[E];
#pragma unroll
    for (int k = 0; k < E; ++k) {
        C v;
        v.x = T(0);
        v.y = T(0);
        if (col) v = base[k * stride];
        if (INV) v.y = -v.y;
        x[k] = v;
    }
    __syncthreads();                                      // twiddles staged
    zr_fft<E, B>(x, buf, tau, Tc, b, f, stw);
    if (col) {
#pragma unroll
        for (int k = 0; k < E; ++k) {
            C v = x[k];
            if (INV) v.y = -v.y;
            base[k * stride] = v;
        }
    }
}

}  // namespace sog
