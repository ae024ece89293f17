// C ABI (include/sog.h) and the per-evaluation orchestration of the SOG hot path on B200.
//
//   S1 k_prepare -> scan -> k_scatter -> k_cellsort             (validate, canonicalise, cell sort)
//      k_stencil_origins -> k_mid_key -> scan -> k_mid_scatter -> k_mid_bucket   (mid order)
//   S2 k_near3 (warp per target; k_near for tiny boxes)        (near field + nothing else)
//   S3-S7 k_mid_spread_z -> cuFFT D2Z -> k_mid_scale -> cuFFT Z2D -> k_mid_gather_z
//   S8-S12 k_long_spread -> cuFFT D2Z (batched 2D) -> k_long_scale -> Z2D -> k_long_gather
//   S13 k_combine                                               (self term, forces, unpermute, U)
// cuFFT supplies only the butterflies.  All other steps are the kernels in kernels_*.cuh.
#include <cuda_runtime.h>
#include <cufft.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sog.h"
#include "kernels_common.cuh"
#include "kernels_long.cuh"
#include "kernels_mid.cuh"
#include "launch.h"
#include "kernels_near.cuh"
#include "kernels_near3.cuh"
#include "kernels_sort.cuh"
#include "sog_internal.h"

namespace {
thread_local std::string g_err;
int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
}  // namespace

namespace sog {

__global__ void k_combine(const d4* __restrict__ nearo, const d4* __restrict__ mido, const d4* __restrict__ longo,
                          const d4* __restrict__ pos, const int* __restrict__ perm, int N, double selfc,
                          double* __restrict__ phi, double* __restrict__ force, double* __restrict__ energy) {
    // phi_i = Phi^N + Phi^mid + Phi^long - q_i sum_l w_l; F_i = -q_i grad phi
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    double e = 0.0;
    if (k < N) {
        d4 a = ld_d4(&nearo[k]), b = ld_d4(&mido[k]), c = ld_d4(&longo[k]);
        double q = ld_d4(&pos[k]).w;
        double ph = a.x + b.x + c.x - q * selfc;
        int i = perm[k];
        if (phi) phi[i] = ph;
        if (force) {
            force[3 * (size_t)i] = -q * (a.y + b.y + c.y);
            force[3 * (size_t)i + 1] = -q * (a.z + b.z + c.z);
            force[3 * (size_t)i + 2] = -q * (a.w + b.w + c.w);
        }
        e = 0.5 * q * ph;                                     // U = 1/2 sum q phi
    }
    for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(energy, e);
}

__global__ void k_components(const d4* __restrict__ nearo, const d4* __restrict__ mido, const d4* __restrict__ longo,
                             const int* __restrict__ perm, int N, double* __restrict__ out) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= N) return;
    int i = perm[k];
    const d4* src[3] = {nearo, mido, longo};
    for (int c = 0; c < 3; ++c) {
        d4 v = ld_d4(&src[c][k]);
        double* o = out + ((size_t)c * N + i) * 4;
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    }
}

}  // namespace sog

using namespace sog;

struct sog_plan {
    Params p;
    RuleKnobs knobs;
    CellGeo geo{};
    int ncell = 0;
    int offx[3] = {0, 0, 0}, noffx = 0, offy[3] = {0, 0, 0}, noffy = 0;
    NearTable near;
    double selfc = 0;
    cudaStream_t stream = nullptr;
    unsigned flags = 0;
    int device = 0;
    // workspace
    d4 *pos = nullptr, *pos_s = nullptr, *o_near = nullptr, *o_mid = nullptr, *o_long = nullptr;
    int *cell = nullptr, *tmp = nullptr, *perm = nullptr, *count = nullptr, *start = nullptr, *cursor = nullptr;
    int4* g0 = nullptr;             // stencil origins per sorted particle (mid x,y,z; long packed)
    unsigned* dflags = nullptr;
    double* qsums = nullptr;   // [0] sum q, [1] sum |q|, [2] energy
    double *d_cF = nullptr, *d_cdF = nullptr;
    // mid: S (spread output, its zero planes are never rewritten), Psi (inverse FFT output)
    double* mgrid = nullptr;
    double* mpsi = nullptr;
    cuDoubleComplex* mspec = nullptr;
    int *mkey = nullptr, *mcount = nullptr, *mstart = nullptr, *mcursor = nullptr, *mtmp = nullptr;
    d4* mpos = nullptr;
    int4* minfo = nullptr;
    int nkeys = 0, nseg_s = 1, nseg_g = 1, mz_cps_g = 1;
    MidZArgs mz{};
    void* scan_tmp = nullptr;
    size_t scan_bytes = 0;
    double *d_A = nullptr, *d_Tx = nullptr, *d_Ty = nullptr, *d_Tz = nullptr;
    cufftHandle mfwd = 0, minv = 0;
    bool has_mid = false;
    // long
    double* lgrid = nullptr;
    double* lpart = nullptr;        // long spread tile partials
    double* lpsiT = nullptr;        // long field, layer-fastest [Ilx][Ily][PCMAX]
    LongTileArgs lt{};
    cuDoubleComplex *lspec = nullptr, *lspec2 = nullptr;
    double *d_K = nullptr, *d_C = nullptr, *d_Tn = nullptr;
    bool long_small = false;        // small long grid: register-tiled spread + broadcast gather
    int lg_nblk = 0;
    double* lpart2 = nullptr;       // [lg_nblk][PCP][Ilx*Ily] spread partials
    double* ldbg = nullptr;         // debug: T basis -> proxy-node basis
    cufftHandle lfwd = 0, linv = 0;
    // host-buffer path
    double *h_xyz = nullptr, *h_q = nullptr, *h_phi = nullptr, *h_force = nullptr;
    // readback
    double* pinned = nullptr;   // [sum q, sum|q|, energy, flags]
    double last_energy = 0;
    cudaEvent_t ev[16] = {};
    double timings[11] = {};
    size_t bytes = 0;
};

namespace {

#define CK(x)                                                                                 \
    do {                                                                                      \
        cudaError_t e_ = (x);                                                                 \
        if (e_ != cudaSuccess) return fail(SOG_ECUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
    } while (0)
#define CKF(x)                                                                                \
    do {                                                                                      \
        cufftResult r_ = (x);                                                                 \
        if (r_ != CUFFT_SUCCESS) return fail(SOG_ECUDA, std::string(#x ": cufft error ") + std::to_string((int)r_)); \
    } while (0)

template <class T>
int dalloc(sog_plan* pl, T** ptr, size_t n) {
    if (n == 0) n = 1;
    cudaError_t e = cudaMalloc((void**)ptr, n * sizeof(T));
    if (e != cudaSuccess) return fail(SOG_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    pl->bytes += n * sizeof(T);
    return SOG_OK;
}

template <class T>
int upload(sog_plan* pl, T** ptr, const std::vector<T>& v) {
    int rc = dalloc(pl, ptr, v.size());
    if (rc) return rc;
    CK(cudaMemcpy(*ptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return SOG_OK;
}

void free_plan(sog_plan* pl) {
    if (!pl) return;
    void* ptrs[] = {pl->g0, pl->pos, pl->pos_s, pl->o_near, pl->o_mid, pl->o_long, pl->cell, pl->tmp, pl->perm,
                    pl->count, pl->start, pl->cursor, pl->dflags, pl->qsums, pl->d_cF, pl->d_cdF, pl->mgrid,
                    pl->mspec, pl->d_A, pl->d_Tx, pl->d_Ty, pl->d_Tz, pl->lgrid, pl->lspec, pl->lspec2,
                    pl->d_K, pl->d_C, pl->lpart, pl->lpsiT, pl->h_xyz, pl->h_q, pl->h_phi, pl->h_force,
                    pl->mpsi, pl->d_Tn, pl->lpart2, pl->ldbg, pl->mkey, pl->mcount, pl->mstart, pl->mcursor, pl->mtmp, pl->mpos, pl->minfo,
                    pl->scan_tmp};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (pl->pinned) cudaFreeHost(pl->pinned);
    for (cufftHandle h : {pl->mfwd, pl->minv, pl->lfwd, pl->linv})
        if (h) cufftDestroy(h);
    for (auto& e : pl->ev)
        if (e) cudaEventDestroy(e);
    delete pl;
}

int setup(sog_plan* pl) {
    Params& p = pl->p;
    CK(cudaGetDevice(&pl->device));
    const int N = int(p.N);
    std::vector<double> w, s;
    sog_weights(p, w, s);
    pl->selfc = 0;
    for (double v : w) pl->selfc += v;   // Phi^self / q = sum_l w_l
    // cell grid (cells >= r_c)
    CellGeo& g = pl->geo;
    g.Lx = p.Lx; g.Ly = p.Ly; g.Lz = p.Lz;
    g.invLx = 1.0 / p.Lx; g.invLy = 1.0 / p.Ly;
    g.ncx = std::max(1, int(std::floor(p.Lx / p.rc)));
    g.ncy = std::max(1, int(std::floor(p.Ly / p.rc)));
    g.ncz = std::max(1, int(std::floor(p.Lz / p.rc)));
    while ((long)g.ncx * g.ncy * g.ncz > 64L * 1024 * 1024) { g.ncx = std::max(1, g.ncx / 2); g.ncy = std::max(1, g.ncy / 2); }
    g.sx = g.ncx / p.Lx; g.sy = g.ncy / p.Ly; g.sz = g.ncz / p.Lz;
    pl->ncell = g.ncx * g.ncy * g.ncz;
    auto offs = [](int nc, int* o, int& n) {
        if (nc >= 3) { o[0] = -1; o[1] = 0; o[2] = 1; n = 3; }
        else if (nc == 2) { o[0] = 0; o[1] = 1; n = 2; }
        else { o[0] = 0; n = 1; }
    };
    offs(g.ncx, pl->offx, pl->noffx);
    offs(g.ncy, pl->offy, pl->noffy);
    std::string err;
    if (!build_near_table(p, pl->near, err)) return fail(SOG_EINVAL, err);
    int rc;
    if ((rc = dalloc(pl, &pl->pos, N)) || (rc = dalloc(pl, &pl->pos_s, N)) || (rc = dalloc(pl, &pl->o_near, N)) ||
        (rc = dalloc(pl, &pl->o_mid, N)) || (rc = dalloc(pl, &pl->o_long, N)) || (rc = dalloc(pl, &pl->cell, N)) ||
        (rc = dalloc(pl, &pl->tmp, N)) || (rc = dalloc(pl, &pl->perm, N)) || (rc = dalloc(pl, &pl->g0, N)) ||
        (rc = dalloc(pl, &pl->count, pl->ncell + 1)) || (rc = dalloc(pl, &pl->start, pl->ncell + 1)) ||
        (rc = dalloc(pl, &pl->cursor, pl->ncell + 1)) || (rc = dalloc(pl, &pl->dflags, 1)) ||
        (rc = dalloc(pl, &pl->qsums, 4)) || (rc = upload(pl, &pl->d_cF, pl->near.cF)) ||
        (rc = upload(pl, &pl->d_cdF, pl->near.cdF)))
        return rc;
    CK(cudaMallocHost((void**)&pl->pinned, 8 * sizeof(double)));
    // mid range
    pl->has_mid = p.m >= 0;
    if (pl->has_mid) {
        size_t G = (size_t)p.Ix * p.Iy * p.Izs, Gc = (size_t)p.Izs * p.Ix * (p.Iy / 2 + 1);
        if ((rc = dalloc(pl, &pl->mgrid, G)) || (rc = dalloc(pl, &pl->mpsi, G)) || (rc = dalloc(pl, &pl->mspec, Gc)))
            return rc;
        CK(cudaMemset(pl->mgrid, 0, G * sizeof(double)));
        // mid order (S1) and the z-sweep geometry of the spread / gather
        MidZArgs& z = pl->mz;
        const int pp = (p.P - 1) / 2;
        z.Ix = p.Ix; z.Iy = p.Iy; z.Izs = p.Izs;
        z.hx = p.hx(); z.hy = p.hy(); z.hz = p.hz();
        z.halfx = 0.5 * p.Ix; z.halfy = 0.5 * p.Iy; z.halfz = 0.5 * p.Izs;
        auto inv = [&](double h) { double H = (p.P - 1) * h / 2.0; return p.S / (H * H); };
        z.invH2Sx = inv(z.hx); z.invH2Sy = inv(z.hy); z.invH2Sz = inv(z.hz);
        z.Vh = z.hx * z.hy * z.hz;
        auto gam = [&](double h) { return std::exp(-2.0 * inv(h) * h * h); };
        z.gamma_x = gam(z.hx); z.gamma_y = gam(z.hy); z.gamma_z = gam(z.hz);
        z.ntx = (p.Ix + MZ_TX - 1) / MZ_TX; z.nty = (p.Iy + MZ_TY - 1) / MZ_TY; z.nzc = (p.Izs + MZ_ZC - 1) / MZ_ZC;
        // stencil starts of particles with |z| <= Lz/2 (one point of rounding margin each side)
        const int g_lo = std::max(pp, (int)std::floor(-0.5 * p.Lz / z.hz + 0.5 * p.Izs + 0.5) - 1);
        const int g_hi = std::min(p.Izs - 1 - pp, (int)std::floor(0.5 * p.Lz / z.hz + 0.5 * p.Izs + 0.5) + 1);
        z.c_lo = (g_lo - pp) / MZ_ZC;
        z.c_hi = (g_hi - pp) / MZ_ZC;
        z.c_hiw = std::min(z.nzc - 1, (g_hi - pp + p.P - 1) / MZ_ZC);
        const int ntile = z.ntx * z.nty;
        auto segs = [&](int nch, int& nseg, int cap) {
            nseg = std::max(1, std::min(nch, (4 * 148 + ntile - 1) / ntile));
            int cps = std::min(cap, (nch + nseg - 1) / nseg);
            nseg = (nch + cps - 1) / cps;
            return cps;
        };
        // spread: (chunks swept incl. warm-up) x (home tiles) must fit the CTA's range table
        auto nhome = [&](int T, int I, int nt) { return std::min(8, T + p.P - 1 >= I ? nt : (p.P - 1 + T - 1) / T + 2); };
        const int nh = nhome(MZ_TX, p.Ix, z.ntx) * nhome(MZ_TY, p.Iy, z.nty);
        const int cap_s = mid_spread_emax() / nh - (p.P - 2 + MZ_ZC) / MZ_ZC;
        if (cap_s < 1) return fail(SOG_EINVAL, "mid spread range table too small for this grid");
        const int cps_s = segs(z.c_hiw - z.c_lo + 1, pl->nseg_s, cap_s);
        const int cps_g = segs(z.c_hi - z.c_lo + 1, pl->nseg_g, 1 << 30);
        z.cps = cps_s;
        pl->mz_cps_g = cps_g;
        pl->nkeys = ntile * z.nzc;
        if ((rc = dalloc(pl, &pl->mkey, N)) || (rc = dalloc(pl, &pl->mtmp, N)) || (rc = dalloc(pl, &pl->mpos, N)) ||
            (rc = dalloc(pl, &pl->minfo, N)) || (rc = dalloc(pl, &pl->mcount, pl->nkeys + 1)) ||
            (rc = dalloc(pl, &pl->mstart, pl->nkeys + 1)) || (rc = dalloc(pl, &pl->mcursor, pl->nkeys + 1)))
            return rc;
        z.mpos = pl->mpos; z.minfo = pl->minfo; z.mstart = pl->mstart;
        if (!mid_gather_smem(p.P)) return fail(SOG_EINVAL, "mid window support outside the compiled range");
        std::vector<double> A, Tx, Ty, Tz;
        build_mid_tables(p, A, Tx, Ty, Tz);
        if ((rc = upload(pl, &pl->d_A, A)) || (rc = upload(pl, &pl->d_Tx, Tx)) || (rc = upload(pl, &pl->d_Ty, Ty)) ||
            (rc = upload(pl, &pl->d_Tz, Tz)))
            return rc;
        long long n[3] = {p.Izs, p.Ix, p.Iy};   // z slowest, y fastest (half axis)
        size_t ws = 0;
        CKF(cufftCreate(&pl->mfwd));
        CKF(cufftMakePlanMany64(pl->mfwd, 3, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_D2Z, 1, &ws));
        pl->bytes += ws;
        CKF(cufftCreate(&pl->minv));
        CKF(cufftMakePlanMany64(pl->minv, 3, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2D, 1, &ws));
        pl->bytes += ws;
    }
    // long range
    {
        size_t G = (size_t)p.Pc * p.Ilx * p.Ily, Gc = (size_t)p.Pc * p.Ilx * (p.Ily / 2 + 1);
        if ((rc = dalloc(pl, &pl->lgrid, G)) || (rc = dalloc(pl, &pl->lspec, Gc)) || (rc = dalloc(pl, &pl->lspec2, Gc)))
            return rc;
        std::vector<double> K, C;
        build_long_kernel(p, K);
        build_cheb_matrix(p.Pc, C);
        std::vector<double> Tn;
        build_cheb_nodes(p.Pc, Tn);
        if ((rc = upload(pl, &pl->d_K, K)) || (rc = upload(pl, &pl->d_C, C)) || (rc = upload(pl, &pl->d_Tn, Tn)) ||
            (rc = dalloc(pl, &pl->ldbg, G)))
            return rc;
        pl->long_small = long_small_ok(p.Ilx, p.Ily, p.Pc);
        if (pl->long_small) {
            pl->lg_nblk = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 4, (p.N + 255) / 256));
            if ((rc = dalloc(pl, &pl->lpart2, (size_t)pl->lg_nblk * long_small_pcp(p.Pc) * p.Ilx * p.Ily))) return rc;
        }
        // S8 tiling: one tile = whole grid when it fits one CTA, else 16x16 column tiles
        LongTileArgs& t = pl->lt;
        if (p.Ilx * p.Ily <= 256) { t.TX = p.Ilx; t.TY = p.Ily; }
        else { t.TX = std::min(16, p.Ilx); t.TY = std::min(16, p.Ily); }
        t.ntx = (p.Ilx + t.TX - 1) / t.TX;
        t.nty = (p.Ily + t.TY - 1) / t.TY;
        const int pl_half = (p.Pl - 1) / 2;
        t.full_range = (t.TX + 2 * pl_half + 2 >= p.Ilx) ? 1 : 0;
        int ntile = t.ntx * t.nty;
        t.nchunk = std::max(1, std::min(4 * 148 / ntile + 1, int((p.N + 255) / 256)));
        if (!t.full_range) t.nchunk = std::max(1, t.nchunk * 3);
        t.ncx = pl->geo.ncx;
        t.cells_per_x = pl->geo.ncy * pl->geo.ncz;
        t.cell_w = p.Lx / pl->geo.ncx;
        t.Lx = p.Lx;
        auto gam = [&](double h) { double H = (p.Pl - 1) * h / 2.0; return std::exp(-2.0 * p.Sl / (H * H) * h * h); };
        t.gamma_x = gam(p.hlx());
        t.gamma_y = gam(p.hly());
        int pcmax = p.Pc <= 16 ? 16 : 32;
        if ((rc = dalloc(pl, &pl->lpart, (size_t)ntile * t.nchunk * t.TX * t.TY * pcmax))) return rc;
        if ((rc = dalloc(pl, &pl->lpsiT, (size_t)p.Ilx * p.Ily * 32))) return rc;
        long long n[2] = {p.Ilx, p.Ily};
        size_t ws = 0;
        CKF(cufftCreate(&pl->lfwd));
        CKF(cufftMakePlanMany64(pl->lfwd, 2, n, nullptr, 1, (long long)p.Ilx * p.Ily, nullptr, 1,
                                (long long)p.Ilx * (p.Ily / 2 + 1), CUFFT_D2Z, p.Pc, &ws));
        pl->bytes += ws;
        CKF(cufftCreate(&pl->linv));
        CKF(cufftMakePlanMany64(pl->linv, 2, n, nullptr, 1, (long long)p.Ilx * (p.Ily / 2 + 1), nullptr, 1,
                                (long long)p.Ilx * p.Ily, CUFFT_Z2D, p.Pc, &ws));
        pl->bytes += ws;
    }
    pl->scan_bytes = std::max(scan_temp_bytes(pl->ncell), pl->nkeys ? scan_temp_bytes(pl->nkeys) : size_t(0));
    if ((rc = dalloc(pl, (char**)&pl->scan_tmp, pl->scan_bytes))) return rc;
    for (auto& e : pl->ev) CK(cudaEventCreate(&e));
    return SOG_OK;
}

int set_stream(sog_plan* pl, cudaStream_t s) {
    pl->stream = s;
    for (cufftHandle h : {pl->mfwd, pl->minv, pl->lfwd, pl->linv})
        if (h) CKF(cufftSetStream(h, s));
    return SOG_OK;
}

MidArgs mid_args(const sog_plan* pl) {
    const Params& p = pl->p;
    MidArgs a;
    a.pos = pl->pos_s;
    a.N = int(p.N);
    a.Ix = p.Ix; a.Iy = p.Iy; a.Izs = p.Izs;
    a.hx = p.hx(); a.hy = p.hy(); a.hz = p.hz();
    a.halfx = 0.5 * p.Ix; a.halfy = 0.5 * p.Iy; a.halfz = 0.5 * p.Izs;
    a.hpx = 0.5 * p.Ix + 0.5; a.hpy = 0.5 * p.Iy + 0.5; a.hpz = 0.5 * p.Izs + 0.5;
    auto inv = [&](double h) { double H = (p.P - 1) * h / 2.0; return p.S / (H * H); };
    a.invH2Sx = inv(a.hx); a.invH2Sy = inv(a.hy); a.invH2Sz = inv(a.hz);
    a.Vh = a.hx * a.hy * a.hz;
    return a;
}

LongArgs long_args(const sog_plan* pl) {
    const Params& p = pl->p;
    LongArgs a;
    a.pos = pl->pos_s;
    a.N = int(p.N);
    a.Ilx = p.Ilx; a.Ily = p.Ily; a.Pc = p.Pc; a.Pl = p.Pl;
    a.hx = p.hlx(); a.hy = p.hly();
    a.halfx = 0.5 * p.Ilx; a.halfy = 0.5 * p.Ily;
    a.hpx = 0.5 * p.Ilx + 0.5; a.hpy = 0.5 * p.Ily + 0.5;
    auto inv = [&](double h) { double H = (p.Pl - 1) * h / 2.0; return p.Sl / (H * H); };
    a.invH2Sx = inv(a.hx); a.invH2Sy = inv(a.hy);
    a.two_over_Lz = 2.0 / p.Lz;
    a.A = a.hx * a.hy;
    a.C = pl->d_C;
    return a;
}

int lchk(int r) {
    if (r == 1) return fail(SOG_EINVAL, "window support / proxy count outside the compiled range");
    if (r == 2) return fail(SOG_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(cudaGetLastError()));
    return SOG_OK;
}

void mark(sog_plan* pl, int k) {
    if (pl->flags & SOG_TIMING) cudaEventRecord(pl->ev[k], pl->stream);
}

// Sort + all three components into o_near / o_mid / o_long (sorted order).  stop_stage > 0
// returns early for sog_debug_stage.
int run_pipeline(sog_plan* pl, const double* xyz, const double* q, int stop_stage = 0) {
    const Params& p = pl->p;
    const int N = int(p.N);
    cudaStream_t st = pl->stream;
    mark(pl, 0);
    int rc;
    // S1
    CK(cudaMemsetAsync(pl->count, 0, sizeof(int) * (pl->ncell + 1), st));
    CK(cudaMemsetAsync(pl->dflags, 0, sizeof(unsigned), st));
    CK(cudaMemsetAsync(pl->qsums, 0, sizeof(double) * 4, st));
    int nb = (N + 255) / 256;
    k_prepare<<<nb, 256, 0, st>>>(xyz, q, N, pl->geo, pl->pos, pl->cell, pl->count, pl->dflags, pl->qsums);
    if ((rc = lchk(launch_exclusive_scan(pl->count, pl->start, pl->ncell, pl->scan_tmp, pl->scan_bytes, st)))) return rc;
    CK(cudaMemcpyAsync(pl->cursor, pl->start, sizeof(int) * pl->ncell, cudaMemcpyDeviceToDevice, st));
    k_scatter<<<nb, 256, 0, st>>>(pl->cell, N, pl->cursor, pl->tmp);
    k_cellsort<<<(pl->ncell * 32 + 255) / 256, 256, 0, st>>>(pl->start, pl->ncell, pl->tmp, pl->pos, pl->pos_s, pl->perm);
    {
        const Params& pp = pl->p;
        MidArgs ma{};
        if (pl->has_mid) ma = mid_args(pl);
        const double lhx = pp.hlx(), lhy = pp.hly();
        if ((rc = lchk(launch_stencil_origins(pl->pos_s, N, ma, pl->has_mid ? 1 : 0, lhx, lhy, 0.5 * pp.Ilx + 0.5,
                                              0.5 * pp.Ily + 0.5, pl->g0, st))))
            return rc;
    }
    if (pl->has_mid) {   // mid order: bucket by (stencil-start tile, z chunk)
        MidSortArgs ms{p.Ix, p.Iy, (p.P - 1) / 2, pl->mz.nty, pl->mz.nzc};
        CK(cudaMemsetAsync(pl->mcount, 0, sizeof(int) * (pl->nkeys + 1), st));
        if ((rc = lchk(launch_mid_sort_keys(pl->g0, N, ms, pl->mkey, pl->mcount, st)))) return rc;
        if ((rc = lchk(launch_exclusive_scan(pl->mcount, pl->mstart, pl->nkeys, pl->scan_tmp, pl->scan_bytes, st))))
            return rc;
        CK(cudaMemcpyAsync(pl->mcursor, pl->mstart, sizeof(int) * pl->nkeys, cudaMemcpyDeviceToDevice, st));
        if ((rc = lchk(launch_mid_sort_place(pl->mkey, N, pl->mcursor, pl->mtmp, pl->mstart, pl->nkeys, pl->pos_s,
                                             pl->g0, (p.P - 1) / 2, pl->mpos, pl->minfo, st))))
            return rc;
    }
    CK(cudaGetLastError());
    mark(pl, 1);
    // S2 near field
    if (!stop_stage) {
        const int D = pl->near.D;
        if (D != NEAR_D) return fail(SOG_EINVAL, "near table degree");
        if (pl->geo.ncx >= 3 && pl->geo.ncy >= 3 && p.N < (1 << 27)) {   // k_near3: warp per target
            Near3Args a;
            a.pos = pl->pos_s; a.start = pl->start; a.cF = pl->d_cF; a.out = pl->o_near;
            a.K = pl->near.K; a.du = pl->near.du; a.inv_du = pl->near.inv_du; a.rc2 = p.rc * p.rc;
            a.g = pl->geo;
            a.cap = 1536;
            a.rc2f = (float)(a.rc2 * (1.0 + 1e-5)) + 1e-5f;
            size_t sh = sizeof(double) * ((pl->near.K * (D + 1) + 1) & ~1) + 10 * sizeof(double2) +
                        NEAR3_WARPS * 160 * sizeof(int) + sizeof(float4) * a.cap;
            CK(cudaFuncSetAttribute(k_near3<NEAR_D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
            k_near3<NEAR_D><<<pl->ncell, 32 * NEAR3_WARPS, sh, st>>>(a);
        } else {
            NearArgs a;
            a.pos = pl->pos_s; a.start = pl->start; a.cF = pl->d_cF; a.cdF = pl->d_cdF; a.out = pl->o_near;
            a.N = N; a.K = pl->near.K; a.du = pl->near.du; a.inv_du = pl->near.inv_du; a.rc2 = p.rc * p.rc;
            a.g = pl->geo;
            for (int i = 0; i < 3; ++i) { a.ox[i] = pl->offx[i]; a.oy[i] = pl->offy[i]; }
            a.noffx = pl->noffx; a.noffy = pl->noffy;
            size_t sh = 2 * sizeof(double) * pl->near.K * (D + 1);
            CK(cudaFuncSetAttribute(k_near<NEAR_D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
            k_near<NEAR_D><<<(N + 255) / 256, 256, sh, st>>>(a);
        }
        CK(cudaGetLastError());
    }
    mark(pl, 2);
    // S3-S7 mid range
    if (pl->has_mid && (stop_stage == 0 || stop_stage == 1 || stop_stage == 2)) {
        if ((rc = lchk(launch_mid_spread_z(pl->mz, p.P, pl->nseg_s, pl->mgrid, st)))) return rc;
        mark(pl, 3);
        if (stop_stage == 1) return SOG_OK;
        CKF(cufftExecD2Z(pl->mfwd, pl->mgrid, pl->mspec));
        mark(pl, 4);
        if ((rc = lchk(launch_mid_scale(pl->mspec, p.Ix, p.Izs, p.Iy / 2 + 1, p.m + 1, pl->d_A, pl->d_Tx, pl->d_Ty,
                                        pl->d_Tz, st))))
            return rc;
        mark(pl, 5);
        CKF(cufftExecZ2D(pl->minv, pl->mspec, pl->mpsi));
        mark(pl, 6);
        if (stop_stage == 2) return SOG_OK;
        {
            MidZArgs g = pl->mz;
            g.cps = pl->mz_cps_g;
            if ((rc = lchk(launch_mid_gather_z(g, p.P, pl->nseg_g, N, pl->mpsi, pl->o_mid, st)))) return rc;
        }
    } else if (!pl->has_mid && !stop_stage) {
        CK(cudaMemsetAsync(pl->o_mid, 0, sizeof(d4) * N, st));
    }
    mark(pl, 7);
    // S8-S12 long range
    if (stop_stage == 0 || stop_stage == 3 || stop_stage == 4) {
        if (pl->long_small) {
            if ((rc = lchk(launch_long_spread_gemm(long_args(pl), pl->g0, pl->lt.gamma_x, pl->lt.gamma_y, pl->lg_nblk,
                                                   pl->lpart2, pl->lgrid, st))))
                return rc;
        } else {
            LongTileArgs t = pl->lt;
            t.a = long_args(pl);
            t.start = pl->start;
            t.part = pl->lpart;
            if ((rc = lchk(launch_long_spread_tile(t, p.Pl, pl->lgrid, st)))) return rc;
        }
        mark(pl, 8);
        if (stop_stage == 3) return SOG_OK;
        CKF(cufftExecD2Z(pl->lfwd, pl->lgrid, pl->lspec));
        int nmode = p.Ilx * (p.Ily / 2 + 1);
        k_long_scale<<<(nmode * p.Pc + 127) / 128, 128, 0, st>>>(pl->lspec, pl->lspec2, pl->d_K, nmode, p.Pc);
        CK(cudaGetLastError());
        CKF(cufftExecZ2D(pl->linv, pl->lspec2, pl->lgrid));
        mark(pl, 9);
        if (stop_stage == 4) return SOG_OK;
        if (pl->long_small) {
            if ((rc = lchk(launch_long_gather_bc(long_args(pl), pl->g0, pl->lgrid, pl->o_long, st)))) return rc;
        } else if ((rc = lchk(launch_long_gather2(long_args(pl), p.Pl, pl->lgrid, pl->lpsiT, pl->o_long,
                                                  pl->lt.gamma_x, pl->lt.gamma_y, st)))) {
            return rc;
        }
    }
    mark(pl, 10);
    return SOG_OK;
}

int check_flags(sog_plan* pl) {
    CK(cudaMemcpyAsync(pl->pinned, pl->qsums, 3 * sizeof(double), cudaMemcpyDeviceToHost, pl->stream));
    unsigned f = 0;
    CK(cudaMemcpyAsync(&pl->pinned[3], pl->dflags, sizeof(unsigned), cudaMemcpyDeviceToHost, pl->stream));
    CK(cudaStreamSynchronize(pl->stream));
    std::memcpy(&f, &pl->pinned[3], sizeof(unsigned));
    pl->last_energy = pl->pinned[2];
    if (f & FLAG_NONFINITE) return fail(SOG_ENONFINITE, "non-finite position or charge");
    if (f & FLAG_ZRANGE) return fail(SOG_EZRANGE, "z outside [-Lz/2, Lz/2]");
    if (std::fabs(pl->pinned[0]) > 1e-12 * pl->pinned[1]) return fail(SOG_ENONNEUTRAL, "system not charge neutral");
    return SOG_OK;
}

void collect_timings(sog_plan* pl) {
    if (!(pl->flags & SOG_TIMING)) return;
    cudaStreamSynchronize(pl->stream);
    // [0] sort, [1] near, [2] mid spread, [3] fwd, [4] scale, [5] inv, [6] gather,
    // [7] long spread, [8] long fft+scale+ifft, [9] long gather, [10] combine
    int pairs[11][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 4}, {4, 5}, {5, 6}, {6, 7}, {7, 8}, {8, 9}, {9, 10}, {10, 11}};
    for (int k = 0; k < 11; ++k) {
        float ms = 0;
        if (cudaEventElapsedTime(&ms, pl->ev[pairs[k][0]], pl->ev[pairs[k][1]]) != cudaSuccess) ms = 0;
        pl->timings[k] = ms;
    }
    cudaGetLastError();
}

}  // namespace

extern "C" {

const char* sog_last_error(void) { return g_err.c_str(); }

namespace {
// Fill p from the rules (or verbatim from explicit options) and validate.
int make_params(Params& p, RuleKnobs& knobs, int64_t N, double Lx, double Ly, double Lz, double tol,
                const sog_plan_opts* o) {
    g_err.clear();
    if (N < 1 || N > (int64_t(1) << 31) - 1) return fail(SOG_EINVAL, "N out of range");
    if (!(Lx > 0 && Ly > 0 && Lz > 0 && std::isfinite(Lx) && std::isfinite(Ly) && std::isfinite(Lz)))
        return fail(SOG_EINVAL, "box lengths must be positive and finite");
    if (!(tol >= 2e-14 && tol <= 1e-1)) return fail(SOG_EINFEASIBLE, "tol outside [2e-14, 1e-1]");
    p.N = N; p.Lx = Lx; p.Ly = Ly; p.Lz = Lz; p.tol = tol;
    std::string err;
    if (o && o->explicit_params) {
        static const double tb[6][3] = {{2.0, 1.9892536839080267, 0.9944464927622323},
                                        {1.62976708826776469, 2.7520026668023417, 1.0078069793438068},
                                        {1.48783512395703226, 3.7554672283554990, 0.9919117057598183},
                                        {1.32070036405934420, 4.3914554711638349, 1.0018891411481198},
                                        {1.21812525709410644, 5.6355288151271085, 1.0009014615603334},
                                        {1.14878150173321925, 7.2956245490719404, 1.0000368348358225}};
        if (o->row < 0 || o->row > 5) return fail(SOG_EINVAL, "row must be 0..5");
        p.row = o->row; p.b = tb[o->row][0]; p.r0 = tb[o->row][1]; p.omega = tb[o->row][2];
        p.rc = o->rc; p.sigma = p.rc / p.r0; p.M = o->M; p.m = o->m;
        p.Ix = o->Ix; p.Iy = o->Iy; p.Iz = o->Iz; p.Izs = o->Izs; p.P = o->P; p.S = o->S;
        p.Ilx = o->Ilx; p.Ily = o->Ily; p.Pl = o->Pl; p.Sl = o->Sl; p.Pc = o->Pc;
    } else {
        if (o && o->rc_factor > 0) knobs.rc_factor = o->rc_factor;
        if (o && o->eta > 0) knobs.eta = o->eta;
        if (!choose_params(p, knobs, err)) return fail(SOG_EINFEASIBLE, err);
    }
    if (!validate_params(p, err)) return fail(SOG_EINVAL, err);
    return SOG_OK;
}
}  // namespace

int sog_plan_choose(int64_t N, double Lx, double Ly, double Lz, double tol, const sog_plan_opts* o, char* buf,
                    size_t len) {
    Params p;
    RuleKnobs k;
    int rc = make_params(p, k, N, Lx, Ly, Lz, tol, o);
    if (rc) return rc;
    std::string s = describe(p);
    if (buf && len) {
        size_t n = std::min(len - 1, s.size());
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
    return int(s.size());
}

sog_plan* sog_plan_create_ex(int64_t N, double Lx, double Ly, double Lz, double tol, const sog_plan_opts* o) {
    sog_plan* pl = new sog_plan();
    if (make_params(pl->p, pl->knobs, N, Lx, Ly, Lz, tol, o) != SOG_OK) { delete pl; return nullptr; }
    if (o) pl->flags = o->flags;
    int rc = setup(pl);
    if (rc == SOG_OK) rc = set_stream(pl, o ? (cudaStream_t)o->cuda_stream : nullptr);
    if (rc != SOG_OK) { std::string keep = g_err; free_plan(pl); g_err = keep; return nullptr; }
    return pl;
}

sog_plan* sog_plan_create(int64_t N, double Lx, double Ly, double Lz, double tol) {
    return sog_plan_create_ex(N, Lx, Ly, Lz, tol, nullptr);
}

void sog_plan_destroy(sog_plan* p) { free_plan(p); }

int sog_eval(sog_plan* pl, const double* xyz, const double* q, double* phi, double* force) {
    if (!pl || !xyz || !q) return fail(SOG_EINVAL, "null argument");
    int rc = run_pipeline(pl, xyz, q);
    if (rc) return rc;
    const int N = int(pl->p.N);
    k_combine<<<(N + 255) / 256, 256, 0, pl->stream>>>(pl->o_near, pl->o_mid, pl->o_long, pl->pos_s, pl->perm, N,
                                                       pl->selfc, phi, force, pl->qsums + 2);
    CK(cudaGetLastError());
    mark(pl, 11);
    collect_timings(pl);
    if (!(pl->flags & SOG_NO_VALIDATE)) return check_flags(pl);
    return SOG_OK;
}

int sog_eval_host(sog_plan* pl, const double* xyz, const double* q, double* phi, double* force) {
    if (!pl || !xyz || !q) return fail(SOG_EINVAL, "null argument");
    const size_t N = pl->p.N;
    int rc;
    if (!pl->h_xyz) {
        if ((rc = dalloc(pl, &pl->h_xyz, 3 * N)) || (rc = dalloc(pl, &pl->h_q, N)) || (rc = dalloc(pl, &pl->h_phi, N)) ||
            (rc = dalloc(pl, &pl->h_force, 3 * N)))
            return rc;
    }
    CK(cudaMemcpyAsync(pl->h_xyz, xyz, 3 * N * sizeof(double), cudaMemcpyHostToDevice, pl->stream));
    CK(cudaMemcpyAsync(pl->h_q, q, N * sizeof(double), cudaMemcpyHostToDevice, pl->stream));
    rc = sog_eval(pl, pl->h_xyz, pl->h_q, phi ? pl->h_phi : nullptr, force ? pl->h_force : nullptr);
    if (rc) return rc;
    if (phi) CK(cudaMemcpyAsync(phi, pl->h_phi, N * sizeof(double), cudaMemcpyDeviceToHost, pl->stream));
    if (force) CK(cudaMemcpyAsync(force, pl->h_force, 3 * N * sizeof(double), cudaMemcpyDeviceToHost, pl->stream));
    CK(cudaStreamSynchronize(pl->stream));
    return SOG_OK;
}

int sog_eval_components(sog_plan* pl, const double* xyz, const double* q, double* out) {
    if (!pl || !xyz || !q || !out) return fail(SOG_EINVAL, "null argument");
    int rc = run_pipeline(pl, xyz, q);
    if (rc) return rc;
    const int N = int(pl->p.N);
    k_components<<<(N + 255) / 256, 256, 0, pl->stream>>>(pl->o_near, pl->o_mid, pl->o_long, pl->perm, N, out);
    CK(cudaGetLastError());
    return check_flags(pl);
}

int sog_debug_stage(sog_plan* pl, int stage, const double* xyz, const double* q, double* out, size_t len) {
    if (!pl || !xyz || !q || !out) return fail(SOG_EINVAL, "null argument");
    const Params& p = pl->p;
    size_t need;
    const double* src;
    if (stage == 1 || stage == 2) {
        if (!pl->has_mid) return fail(SOG_EINVAL, "plan has no mid-range part (m < 0)");
        need = (size_t)p.Ix * p.Iy * p.Izs;
        src = stage == 1 ? pl->mgrid : pl->mpsi;
    } else if (stage == 3 || stage == 4) {
        need = (size_t)p.Pc * p.Ilx * p.Ily;
        src = pl->ldbg;                 // converted from the T basis below
    } else {
        return fail(SOG_EINVAL, "stage must be 1..4");
    }
    if (len < need) return fail(SOG_EINVAL, "output buffer too small");
    int rc = run_pipeline(pl, xyz, q, stage);
    if (rc) return rc;
    if (stage >= 3) {   // T basis -> proxy nodes: S_b = sum_n C[b][n] S~_n, Psi_a = sum_m T_m(x_a) Psi~_m
        if ((rc = lchk(launch_long_to_nodes(pl->lgrid, pl->ldbg, p.Ilx * p.Ily, p.Pc, stage == 3 ? pl->d_C : pl->d_Tn,
                                            pl->stream))))
            return rc;
    }
    CK(cudaMemcpyAsync(out, src, need * sizeof(double), cudaMemcpyDeviceToDevice, pl->stream));
    return check_flags(pl);
}

int sog_last_energy(sog_plan* pl, double* U) {
    if (!pl || !U) return fail(SOG_EINVAL, "null argument");
    CK(cudaMemcpyAsync(pl->pinned + 2, pl->qsums + 2, sizeof(double), cudaMemcpyDeviceToHost, pl->stream));
    CK(cudaStreamSynchronize(pl->stream));
    *U = pl->pinned[2];
    return SOG_OK;
}

int sog_plan_describe(const sog_plan* pl, char* buf, size_t len) {
    if (!pl) return fail(SOG_EINVAL, "null plan");
    std::string s = describe(pl->p);
    char extra[512];
    std::snprintf(extra, sizeof extra,
                  "ncell=%d\nnear_table_pieces=%d\nnear_table_degree=%d\nnear_table_max_rel_err=%.3e\n"
                  "self_coefficient=%.17g\nworkspace_bytes=%zu\n",
                  pl->ncell, pl->near.K, pl->near.D, pl->near.max_rel_err, pl->selfc, pl->bytes);
    s += extra;
    if (buf && len) {
        size_t n = std::min(len - 1, s.size());
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
    return int(s.size());
}

int sog_get_timings(const sog_plan* pl, double* ms, int n) {
    if (!pl || !ms) return fail(SOG_EINVAL, "null argument");
    int k = std::min(n, 11);
    for (int i = 0; i < k; ++i) ms[i] = pl->timings[i];
    return k;
}

int sog_set_flags(sog_plan* pl, unsigned flags) {
    if (!pl) return fail(SOG_EINVAL, "null plan");
    pl->flags = flags;
    return SOG_OK;
}

int sog_set_stream(sog_plan* pl, void* s) {
    if (!pl) return fail(SOG_EINVAL, "null plan");
    return set_stream(pl, (cudaStream_t)s);
}

int sog_launches_per_eval(const sog_plan* pl) {
    if (!pl) return fail(SOG_EINVAL, "null plan");
    // prepare, scan (1 CUB kernel pair), scatter, cellsort, origins, near,
    // [mid: key, scan, scatter, bucket, spread, scale, gather], long: spread, reduce, scale,
    // [transpose,] gather, combine  (cuFFT launches are not counted)
    return 2 + 2 + 2 + 1 + (pl->has_mid ? 8 : 0) + (pl->long_small ? 4 : 5) + 1;
}

}  // extern "C"
