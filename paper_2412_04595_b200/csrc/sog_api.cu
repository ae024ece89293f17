// C ABI (include/sog.h) and the per-evaluation orchestration of the SOG hot path on B200.
//
//   S1 k_prepare -> scan -> k_scatter -> k_cellsort             (validate, canonicalise, cell sort)
//      k_stencil_origins -> k_mid_key -> scan -> k_mid_scatter -> k_mid_bucket   (mid order)
//   S2 k_near3 (warp per target; k_near for tiny boxes)        (near field + nothing else)
//   S3-S7 k_mid_spread_z -> cuFFT D2Z -> k_mid_scale -> cuFFT Z2D -> k_mid_gather_z
//   S8-S12 k_long_spread -> cuFFT D2Z (batched 2D) -> k_long_scale -> Z2D -> k_long_gather
//   S13 k_combine_g + k_sum_partials                            (self term, forces, unpermute, U)
// cuFFT supplies only the butterflies.  All other steps are the kernels in kernels_*.cuh.
#include <cuda_runtime.h>
#include <cufft.h>

#include <cmath>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sog.h"
#include "kernels_fft.cuh"
#include "kernels_common.cuh"
#include "kernels_dist.cuh"
#include "kernels_long.cuh"
#include "kernels_dft.cuh"
#include "kernels_mid.cuh"
#include "launch.h"
#include "kernels_near.cuh"
#include <nvtx3/nvToolsExt.h>
#include "kernels_near3.cuh"
#include "kernels_near5.cuh"
#include "kernels_near4.cuh"
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

// S13 in gather form: thread = caller (local) index i < nown, reading its sorted slot k = iperm[i]
// (full 32-byte sectors) and writing phi / force in caller order (coalesced stores)
__global__ void k_combine_g(const d4* __restrict__ nearo, const d4* __restrict__ mido, const d4* __restrict__ longo,
                            const d4* __restrict__ pos, const int* __restrict__ iperm, int nown, double selfc,
                            double* __restrict__ phi, double* __restrict__ force, double* __restrict__ epart) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double e = 0.0;
    if (i < nown) {
        const int k = iperm[i];
        const d4 a = ld_d4(&nearo[k]), b = ld_d4(&mido[k]), c = ld_d4(&longo[k]);
        const double q = ld_d4(&pos[k]).w;
        const double ph = a.x + b.x + c.x - q * selfc;
        if (phi) phi[i] = ph;
        if (force) {                                       // F = -q grad phi
            force[3 * (size_t)i] = -q * (a.y + b.y + c.y);
            force[3 * (size_t)i + 1] = -q * (a.z + b.z + c.z);
            force[3 * (size_t)i + 2] = -q * (a.w + b.w + c.w);
        }
        e = 0.5 * q * ph;                                  // U = 1/2 sum q phi
    }
    __shared__ double se[32];
    for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    if ((threadIdx.x & 31) == 0) se[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += se[w];
        epart[blockIdx.x] = t;
    }
}

// S13 in two passes (single GPU): sorted order with coalesced component reads -> tot[j] = (phi,
// F = -q grad phi) and the per-block energy partials, then caller order with one 32-byte random read
// per particle (the one-pass gather form reads four random 32-byte records per particle)
__global__ void k_combine_s(const d4* __restrict__ nearo, const d4* __restrict__ mido, const d4* __restrict__ longo,
                            const d4* __restrict__ pos, int n, double selfc, d4* __restrict__ tot,
                            double* __restrict__ epart) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    double e = 0.0;
    if (j < n) {
        const d4 a = ld_d4(&nearo[j]), b = ld_d4(&mido[j]), c = ld_d4(&longo[j]);
        const double q = ld_d4(&pos[j]).w;
        const double ph = a.x + b.x + c.x - q * selfc;
        st_d4(&tot[j], d4{ph, -q * (a.y + b.y + c.y), -q * (a.z + b.z + c.z), -q * (a.w + b.w + c.w)});
        e = 0.5 * q * ph;                                  // U = 1/2 sum q phi
    }
    __shared__ double se[32];
    for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    if ((threadIdx.x & 31) == 0) se[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += se[w];
        epart[blockIdx.x] = t;
    }
}
__global__ void k_combine_u(const d4* __restrict__ tot, const int* __restrict__ iperm, int n, double* __restrict__ phi,
                            double* __restrict__ force) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const d4 v = ld_d4(&tot[iperm[i]]);
    if (phi) phi[i] = v.x;
    if (force) {
        force[3 * (size_t)i] = v.y;
        force[3 * (size_t)i + 1] = v.z;
        force[3 * (size_t)i + 2] = v.w;
    }
}

// pipelined host path: fold one evaluation's input status into the accumulated status word
__global__ void k_status_accum(const unsigned* __restrict__ dflags, const double* __restrict__ qsums,
                               unsigned* __restrict__ acc) {
    unsigned f = *dflags;
    if (fabs(qsums[0]) > 1e-12 * qsums[1]) f |= 4u;      // not charge neutral (check_flags' rule)
    *acc |= f;
}

// out = sum of part[0..n) in a fixed order (one block)
__global__ void k_sum_partials(const double* __restrict__ part, int n, double* __restrict__ out) {
    __shared__ double s[1024];
    double t = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) t += part[i];
    s[threadIdx.x] = t;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = s[0];
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
    NearPoly npoly;                 // R16-G single polynomial (k_near4), when near4 is set
    bool near4 = false;
    int near_mode = 5;              // SOG_NEAR: 3 (table, k_near3), 4 (k_near4), 5 (k_near3 + polynomial: default),
                                    //   6 (k_near5: each pair once, + polynomial; one GPU, opt-in: slower)
    int n5_cap = 0;                 // k_near5 staged sources per piece
    bool nvtx_open = false;         // a stage NVTX range is open (mark())
    d4* npart = nullptr;            // k_near5 forward-shell partials [N][13]
    d4* o_tot = nullptr;            // two-pass combine (single GPU): (phi, F) in sorted order
    // pipelined host path (sog_eval_host_async): two device staging sets, copy-in / copy-out streams
    double *ax[2] = {}, *aq[2] = {}, *aphi[2] = {}, *aforce[2] = {};
    cudaStream_t cin = nullptr, cout = nullptr;
    cudaEvent_t ev_in[2] = {}, ev_comp[2] = {}, ev_out[2] = {};
    bool a_used[2] = {false, false};
    int aslot = 0;
    unsigned* astat = nullptr;      // input status accumulated over the calls since sog_host_wait
    int n4_kc = 1, n4_nw = 1, n4_cap = 0;
    double selfc = 0;
    cudaStream_t stream = nullptr;
    unsigned flags = 0;
    int device = 0;
    // workspace
    d4 *pos = nullptr, *pos_s = nullptr, *o_near = nullptr, *o_mid = nullptr, *o_long = nullptr;
    int *cell = nullptr, *tmp = nullptr, *perm = nullptr, *count = nullptr, *start = nullptr, *cursor = nullptr;
    int* iperm = nullptr;                   // inverse permutation (caller / local index -> sorted)
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
    cufftHandle mfwd = 0, minv = 0;     // z-pruned FFT: 2D over the written / read planes
    cufftHandle minv_full = 0, mzfft = 0;  // 2D inverse over all planes (debug stage 2); 1D along z
    cuDoubleComplex *mX = nullptr, *mY = nullptr;   // [planes][Ix*nyh] and zero-padded pencils [Ix*nyh][Izs]
    int zs0 = 0, nzf = 0, zg0 = 0, nzg = 0;         // spread-written planes, gather-read planes
    // fused z pass (kernels_fft.cuh): FFT along z + S5 + inverse in one kernel on the plane spectra
    bool zpass = false;
    int zr_E = 0, zr_B = 0;                         // register-resident variant (SOG_ZPASS=2)
    FftStages zst{};
    // plane FFTs (x, y) of S4 / S6 by k_rows_r2c / k_xfft / k_rows_c2r (SOG_PLANEFFT=0: cuFFT 2D)
    bool pfft = false;
    int pr_E = 0, pr_B = 0, px_E = 0, px_B = 0;
    FftStages prst{}, pxst{};
    void *d_prtw = nullptr, *d_pxtw = nullptr, *d_wpost = nullptr;
    void* d_ztw = nullptr;                          // twiddles (double2, or float2 in fp32 mode)
    void* d_mult = nullptr;                         // S5 table [Izs][Ix nyh] (register-resident z pass)
    bool has_mid = false;
    // long
    double* lgrid = nullptr;
    double* lpart = nullptr;        // long spread tile partials
    double* lpsiT = nullptr;        // long field, layer-fastest [Ilx][Ily][PCMAX]
    LongTileArgs lt{};
    cuDoubleComplex *lspec = nullptr, *lspec2 = nullptr;
    double *d_K = nullptr, *d_C = nullptr, *d_Tn = nullptr;
    KBTab kbl{};                                 // R6-KB long-window table (mid: in mz)
    bool long_small = false;        // small long grid: register-tiled spread + broadcast gather
    DftArgs dft{};                  // long_method = 1 (Alg. 3): mode set
    double *ldS = nullptr, *ldP = nullptr, *ldpart = nullptr, *d_Kd = nullptr;   // S~, Psi~ [Pc][mode] complex
    double* epart = nullptr;        // per-block partial energies of k_combine_g
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
    // SOG_GRAPH: the whole evaluation captured once per (xyz, q, phi, force) pointer tuple, replayed
    cudaGraphExec_t gexec = nullptr;
    const void* gkey[4] = {};
    cudaStream_t gstream = nullptr;         // private capture stream (the legacy stream cannot capture)
    // near field on a side stream, concurrent with the mid / long chain (ALU-bound pair kernel next
    // to the HBM-bound FFT steps); joined before the combine
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    double timings[11] = {};
    size_t bytes = 0;
    // ---- x-slab rank (R > 1); R == 1: the whole periodic box ----
    bool f32 = false;                      // fp32 mode (S2-S12 in fp32; grids hold floats)
    int R = 1, rank = 0;
    int Ncap = 0, Ncur = 0, Nown = 0;      // particle capacity / current local / own counts
    double xs0 = 0, xs1 = 0, Hh = 0;       // slab [xs0, xs1) and particle halo width
    int I0 = 0, Ixr = 0, XO = 0, Ixk = 0;  // interior planes [I0, I0+Ixr) at local x XO; local extent
    int kc = 0, HP = 0;                    // ky chunk per rank; Psi halo planes per side
    size_t blk = 0;                        // complex elements per all-to-all block
    cuDoubleComplex *spec2 = nullptr, *specx = nullptr, *sbuf = nullptr, *rbuf = nullptr;
    cufftHandle f2f = 0, f2i = 0, fxf = 0, fxi = 0;   // 2D (z,y) per x plane; 1D along x
    double *hsb = nullptr, *hrb = nullptr;             // Psi halo planes [2][Izs][HP][Iy]
    d4 *own = nullptr, *hsend = nullptr, *hrecv = nullptr, *pos_long = nullptr;
    int *fl = nullptr, *fr = nullptr, *nsel = nullptr;
    double* dstat = nullptr;                // [8] input status summed over ranks (k_slab_flags)
    double* pin_d = nullptr;                // pinned copy of dstat after the agreement
    int nown_cap = 0;                       // own-particle capacity
    double *lxyz = nullptr, *lq = nullptr;
    void* sel_tmp = nullptr;
    size_t sel_bytes = 0;
    int halo_cap = 0;
    int* pin_i = nullptr;                   // pinned [nl_send, nr_send, nl_recv, nr_recv, bad]
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
    void* ptrs[] = {pl->g0, pl->pos, pl->pos_s, pl->o_near, pl->o_mid, pl->o_long, pl->cell, pl->tmp, pl->perm, pl->iperm,
                    pl->count, pl->start, pl->cursor, pl->dflags, pl->qsums, pl->d_cF, pl->d_cdF, pl->mgrid,
                    pl->mspec, pl->d_A, pl->d_Tx, pl->d_Ty, pl->d_Tz, pl->lgrid, pl->lspec, pl->lspec2,
                    pl->d_K, pl->d_C, pl->lpart, pl->lpsiT, pl->h_xyz, pl->h_q, pl->h_phi, pl->h_force,
                    pl->mpsi, pl->d_Tn, pl->lpart2, pl->ldbg, pl->mkey, pl->mcount, pl->mstart, pl->mcursor, pl->mtmp, pl->mpos, pl->minfo,
                    pl->scan_tmp, pl->spec2, pl->specx, pl->sbuf, pl->rbuf, pl->hsb, pl->hrb, pl->own, pl->hsend,
                    pl->hrecv, pl->pos_long, pl->fl, pl->fr, pl->nsel, pl->dstat, pl->lxyz, pl->lq, pl->sel_tmp,
                    pl->ldS, pl->ldP, pl->ldpart, pl->d_Kd, pl->epart, pl->npart, pl->o_tot,
                    pl->ax[0], pl->ax[1], pl->aq[0], pl->aq[1], pl->aphi[0], pl->aphi[1], pl->aforce[0],
                    pl->aforce[1], pl->astat};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (int i = 0; i < 2; ++i)
        for (cudaEvent_t e : {pl->ev_in[i], pl->ev_comp[i], pl->ev_out[i]})
            if (e) cudaEventDestroy(e);
    if (pl->cin) cudaStreamDestroy(pl->cin);
    if (pl->cout) cudaStreamDestroy(pl->cout);
    if (pl->pinned) cudaFreeHost(pl->pinned);
    if (pl->pin_i) cudaFreeHost(pl->pin_i);
    if (pl->pin_d) cudaFreeHost(pl->pin_d);
    for (cufftHandle h : {pl->mfwd, pl->minv, pl->lfwd, pl->linv, pl->f2f, pl->f2i, pl->fxf, pl->fxi, pl->minv_full,
                          pl->mzfft})
        if (h) cufftDestroy(h);
    for (void* p : {(void*)pl->mX, (void*)pl->mY, pl->d_ztw, pl->d_mult, pl->d_prtw, pl->d_pxtw, pl->d_wpost})
        if (p) cudaFree(p);
    for (auto& e : pl->ev)
        if (e) cudaEventDestroy(e);
    if (pl->gexec) cudaGraphExecDestroy(pl->gexec);
    if (pl->gstream) cudaStreamDestroy(pl->gstream);
    if (pl->side) cudaStreamDestroy(pl->side);
    if (pl->ev_fork) cudaEventDestroy(pl->ev_fork);
    if (pl->ev_join) cudaEventDestroy(pl->ev_join);
    delete pl;
}

void kb_table(int P, double beta, int nu, int window, KBTab& t);

int setup(sog_plan* pl) {
    Params& p = pl->p;
    CK(cudaGetDevice(&pl->device));
    if (pl->Ncap <= 0) pl->Ncap = int(p.N);
    const int N = pl->Ncap;
    const bool slab = pl->R > 1;
    std::vector<double> w, s;
    sog_weights(p, w, s);
    pl->selfc = 0;
    for (double v : w) pl->selfc += v;   // Phi^self / q = sum_l w_l
    // cell grid (cells >= r_c)
    CellGeo& g = pl->geo;
    g.Lx = p.Lx; g.Ly = p.Ly; g.Lz = p.Lz;
    g.invLx = 1.0 / p.Lx; g.invLy = 1.0 / p.Ly;
    g.px = 1;
    g.x0 = -0.5 * p.Lx;
    if (slab) {   // non-periodic extended slab [xs0 - H, xs1 + H)
        g.Lx = (pl->xs1 - pl->xs0) + 2.0 * pl->Hh;
        g.invLx = 1.0 / g.Lx;
        g.x0 = pl->xs0 - pl->Hh;
        g.px = 0;
    }
    g.ncx = std::max(1, int(std::floor(g.Lx / p.rc)));
    g.ncy = std::max(1, int(std::floor(p.Ly / p.rc)));
    // cells of height >= r_c / nzr (SOG_NEAR_NZR, default 1; 2 and 3 measured slower at c2-c5): the z reach is +-nzr cells, so
    // the staged neighbourhood spans (2 nzr + 1) / nzr cell widths in z instead of 3
    {
        const char* env = std::getenv("SOG_NEAR_NZR");
        g.nzr = env ? std::max(1, std::min(4, std::atoi(env))) : 1;
    }
    g.ncz = std::max(1, int(std::floor(p.Lz * g.nzr / p.rc)));
    while ((long)g.ncx * g.ncy * g.ncz > 64L * 1024 * 1024) { g.ncx = std::max(1, g.ncx / 2); g.ncy = std::max(1, g.ncy / 2); }
    g.sx = g.ncx / g.Lx; g.sy = g.ncy / p.Ly; g.sz = g.ncz / p.Lz;
    if (slab && (g.ncx < 3 || g.ncy < 3)) return fail(SOG_EINVAL, "x-slab needs >= 3 near cells per axis");
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
    // target-stationary near field (k_near4) when the single polynomial validates and the cell grid
    // has >= 3 cells per periodic axis (SOG_NEAR=3: the warp-per-target k_near3 instead)
    {
        const char* env = std::getenv("SOG_NEAR");
        pl->near_mode = env ? std::atoi(env) : 5;
        if (slab && (pl->near_mode == 4 || pl->near_mode == 6)) pl->near_mode = 5;   // own-target filter: k_near3
        if (pl->near_mode == 6 && !(g.px && g.nzr == 1 && N < (1 << 27))) pl->near_mode = 5;
        if (pl->near_mode != 3 && !pl->f32 && g.ncx >= 3 && g.ncy >= 3 && build_near_poly(p, pl->npoly)) {
            const double m = std::max(1.0, double(pl->Ncap) / pl->ncell);       // mean particles per cell
            pl->n4_kc = std::max(1, std::min(g.ncz, int(140.0 / m)));
            pl->n4_nw = std::max(1, std::min(N4_MAXW, int(std::ceil(pl->n4_kc * m / 32.0))));
            const double expect = 3.0 * 3.0 * (pl->n4_kc + 2 * g.nzr) * m;       // staged records
            const int capmax = std::min(65535, int((227 * 1024 - sizeof(unsigned short) * (size_t)pl->n4_nw * N4_Q * 32) / 44));
            // expectation + 4 sigma (uniform input; rare overflows run in pieces)
            pl->n4_cap = std::max(256, std::min(capmax, int(expect + 4.0 * std::sqrt(expect) + 64)) & ~3);
            pl->near4 = true;
            if (pl->near_mode == 6) {   // k_near5: 14 staged cells, expectation + 4 sigma, 128-blocks
                const double e5 = 14.0 * m;
                pl->n5_cap = std::min(4096, (int(e5 + 4.0 * std::sqrt(e5) + 16) + 127) & ~127);
            }
        }
        if (!pl->near4 && pl->near_mode == 6) pl->near_mode = 5;
    }
    int rc;
    if ((rc = dalloc(pl, &pl->pos, N)) || (rc = dalloc(pl, &pl->pos_s, N)) || (rc = dalloc(pl, &pl->o_near, N)) ||
        (rc = dalloc(pl, &pl->o_mid, N)) || (rc = dalloc(pl, &pl->o_long, N)) || (rc = dalloc(pl, &pl->cell, N)) ||
        (rc = dalloc(pl, &pl->tmp, N)) || (rc = dalloc(pl, &pl->perm, N)) || (rc = dalloc(pl, &pl->iperm, N)) || (rc = dalloc(pl, &pl->g0, N)) ||
        (rc = dalloc(pl, &pl->count, pl->ncell + 1)) || (rc = dalloc(pl, &pl->start, pl->ncell + 1)) ||
        (rc = dalloc(pl, &pl->cursor, pl->ncell + 1)) || (rc = dalloc(pl, &pl->dflags, 1)) ||
        (rc = dalloc(pl, &pl->qsums, 4)) || (rc = dalloc(pl, &pl->epart, ((size_t)N + 255) / 256 + 1)) || (rc = upload(pl, &pl->d_cF, pl->near.cF)) ||
        (rc = upload(pl, &pl->d_cdF, pl->near.cdF)))
        return rc;
    if (pl->near4 && pl->near_mode == 6 && (rc = dalloc(pl, &pl->npart, (size_t)N * NEAR5_SLOTS))) return rc;
    if (!slab && !(std::getenv("SOG_COMBINE2") && std::atoi(std::getenv("SOG_COMBINE2")) == 0) &&
        (rc = dalloc(pl, &pl->o_tot, N)))
        return rc;
    CK(cudaMallocHost((void**)&pl->pinned, 8 * sizeof(double)));
    // mid range
    pl->has_mid = p.m >= 0;
    if (pl->has_mid) {
        const int nyh = p.Iy / 2 + 1;
        if (slab) {   // local extended planes: [XO halo | Ixr interior (tile-padded) | XO + 16 halo]
            pl->Ixr = p.Ix / pl->R;
            pl->I0 = pl->rank * pl->Ixr;
            // left/right local halo planes: every local particle (x within H of the slab) has its
            // stencil start s_x in [I0 - ceil(H/h) - 1 - p, ...): XO covers it, tile aligned
            const int hpl = int(std::ceil(pl->Hh / p.hx())) + 2 + p.P;
            pl->XO = MZ_TX * ((hpl + MZ_TX - 1) / MZ_TX);
            pl->Ixk = pl->XO + MZ_TX * ((pl->Ixr + MZ_TX - 1) / MZ_TX) + pl->XO + MZ_TX;
            pl->HP = (p.P - 1) / 2 + 1;
            pl->kc = (nyh + pl->R - 1) / pl->R;
            pl->blk = (size_t)p.Izs * pl->Ixr * pl->kc;
        } else {
            pl->Ixk = p.Ix;
        }
        size_t G = (size_t)pl->Ixk * p.Iy * p.Izs;
        if ((rc = dalloc(pl, &pl->mgrid, G)) || (rc = dalloc(pl, &pl->mpsi, G))) return rc;
        CK(cudaMemset(pl->mgrid, 0, G * sizeof(double)));
        CK(cudaMemset(pl->mpsi, 0, G * sizeof(double)));
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
        z.ntx = (pl->Ixk + MZ_TX - 1) / MZ_TX; z.nty = (p.Iy + MZ_TY - 1) / MZ_TY; z.nzc = (p.Izs + MZ_ZC - 1) / MZ_ZC;
        z.px = slab ? 0 : 1;
        z.xorig = slab ? pl->I0 - pl->XO : 0;
        z.Ixk = pl->Ixk;
        z.tlo = slab ? pl->XO / MZ_TX : 0;
        z.ntout = slab ? (pl->Ixr + MZ_TX - 1) / MZ_TX : z.ntx;
        // stencil starts of particles with |z| <= Lz/2 (one point of rounding margin each side)
        const int g_lo = std::max(pp, (int)std::floor(-0.5 * p.Lz / z.hz + 0.5 * p.Izs + 0.5) - 1);
        const int g_hi = std::min(p.Izs - 1 - pp, (int)std::floor(0.5 * p.Lz / z.hz + 0.5 * p.Izs + 0.5) + 1);
        z.c_lo = (g_lo - pp) / MZ_ZC;
        z.c_hi = (g_hi - pp) / MZ_ZC;
        z.c_hiw = std::min(z.nzc - 1, (g_hi - pp + p.P - 1) / MZ_ZC);
        const int ntile = z.ntout * z.nty;
        auto segs = [&](int nch, int& nseg, int cap) {
            nseg = std::max(1, std::min(nch, (4 * 148 + ntile - 1) / ntile));
            int cps = std::min(cap, (nch + nseg - 1) / nseg);
            nseg = (nch + cps - 1) / cps;
            return cps;
        };
        // spread: (chunks swept incl. warm-up) x (home tiles) must fit the CTA's range table
        auto nhome = [&](int T, int I, int nt) { return std::min(8, T + p.P - 1 >= I ? nt : (p.P - 1 + T - 1) / T + 2); };
        const int nh = (slab ? (p.P - 1 + MZ_TX - 1) / MZ_TX + 1 : nhome(MZ_TX, p.Ix, z.ntx)) * nhome(MZ_TY, p.Iy, z.nty);
        const int cap_s = mid_spread_emax() / nh - (p.P - 2 + MZ_ZC) / MZ_ZC;
        if (cap_s < 1) return fail(SOG_EINVAL, "mid spread range table too small for this grid");
        const int cps_s = segs(z.c_hiw - z.c_lo + 1, pl->nseg_s, cap_s);
        const int cps_g = segs(z.c_hi - z.c_lo + 1, pl->nseg_g, 1 << 30);
        z.cps = cps_s;
        pl->mz_cps_g = cps_g;
        pl->nkeys = z.ntx * z.nty * z.nzc;
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
        z.kb = p.window != 0 ? 1 : 0;                  // KB and ES: the polynomial-window kernels
        if (z.kb) kb_table(p.P, p.S, p.nu, p.window, z.kt);
        size_t ws = 0;
        if (!slab) {
            // z-pruned 3D FFT: 2D (x,y) over the planes the spread writes, 1D along z on zero-padded
            // z-contiguous pencils, 2D inverse over the planes the gather reads
            pl->zs0 = z.c_lo * MZ_ZC;
            pl->nzf = std::min(p.Izs, (z.c_hiw + 1) * MZ_ZC) - pl->zs0;
            pl->zg0 = z.c_lo * MZ_ZC;
            pl->nzg = std::min(p.Izs, (z.c_hi + 1) * MZ_ZC + p.P) - pl->zg0;
            const long long M = (long long)p.Ix * nyh;
            const size_t csz = pl->f32 ? sizeof(cuComplex) : sizeof(cuDoubleComplex);
            CK(cudaMalloc((void**)&pl->mX, csz * (size_t)M * p.Izs));
            pl->bytes += csz * (size_t)M * p.Izs;
            long long n2[2] = {p.Ix, p.Iy}, n1[1] = {p.Izs};
            const cufftType r2c = pl->f32 ? CUFFT_R2C : CUFFT_D2Z, c2r = pl->f32 ? CUFFT_C2R : CUFFT_Z2D;
            const cufftType c2c = pl->f32 ? CUFFT_C2C : CUFFT_Z2Z;
            CKF(cufftCreate(&pl->mfwd));
            CKF(cufftMakePlanMany64(pl->mfwd, 2, n2, nullptr, 1, (long long)p.Ix * p.Iy, nullptr, 1, M, r2c, pl->nzf, &ws));
            pl->bytes += ws;
            CKF(cufftCreate(&pl->minv));
            CKF(cufftMakePlanMany64(pl->minv, 2, n2, nullptr, 1, M, nullptr, 1, (long long)p.Ix * p.Iy, c2r, pl->nzg, &ws));
            pl->bytes += ws;
            CKF(cufftCreate(&pl->minv_full));
            CKF(cufftMakePlanMany64(pl->minv_full, 2, n2, nullptr, 1, M, nullptr, 1, (long long)p.Ix * p.Iy, c2r, p.Izs,
                                    &ws));
            pl->bytes += ws;
            CKF(cufftCreate(&pl->mzfft));
            CKF(cufftMakePlanMany64(pl->mzfft, 1, n1, nullptr, 1, p.Izs, nullptr, 1, p.Izs, c2c, M, &ws));
            pl->bytes += ws;
            // fused z pass (FFT along z + S5 + inverse FFT in one kernel, in place on the plane spectra):
            // SOG_ZPASS=2 (default) the register-resident kernel when a radix set dividing E = 8..16
            // covers Izs (c5: 5.35 ms vs 6.1 ms for the chain), 1 the shared-memory-stage kernel, 0 (or
            // an unsupported Izs) the transpose + cuFFT 1D + scale + cuFFT 1D + transpose chain
            {
                const char* env = std::getenv("SOG_ZPASS");
                const int mode = env ? std::atoi(env) : 2;
                std::vector<double2> tw;
                bool ok = false;
                if (mode == 2) {   // register-resident: E elements per thread, radices dividing E
                    for (int E : {10, 8, 12, 16}) {
                        if (p.Izs % E || p.Izs / E > 256) continue;
                        if (fft_plan_stages(p.Izs, pl->zst, tw, E)) {
                            pl->zr_E = E;
                            { const char* eb = std::getenv("SOG_ZPASS_B"); pl->zr_B = eb ? std::atoi(eb) : 2; }
                            ok = true;
                            break;
                        }
                    }
                } else if (mode == 1) {
                    ok = fft_plan_stages(p.Izs, pl->zst, tw);
                }
                if (ok) {
                    if (pl->f32) {
                        std::vector<float2> t2(tw.size());
                        for (size_t i = 0; i < tw.size(); ++i) t2[i] = make_float2((float)tw[i].x, (float)tw[i].y);
                        if ((rc = upload(pl, (float2**)&pl->d_ztw, t2))) return rc;
                    } else if ((rc = upload(pl, (double2**)&pl->d_ztw, tw))) {
                        return rc;
                    }
                    pl->zpass = true;
                }
            }
            // plane FFTs: rows of Iy = 2 n2 reals through a complex FFT of n2, x columns of Ix; E elements
            // per thread (radices dividing E), B rows / columns per CTA (SOG_PLANEFFT_B overrides both)
            if (p.Iy % 2 == 0 && !(std::getenv("SOG_PLANEFFT") && std::atoi(std::getenv("SOG_PLANEFFT")) == 0)) {
                // c5 (ncu, per launch): rows r2c / c2r 1.65 / 1.46 ms at 4 rows per CTA, x FFT 1.37 ms at
                // 8 columns, E = 20; cuFFT's 2D pair 3.56 / 3.61 ms
                const char* eb = std::getenv("SOG_PLANEFFT_B");
                const int Brow = eb ? std::atoi(eb) : 4, Bx = eb ? std::atoi(eb) : 8;
                std::vector<double2> twr, twx;
                const char* ee = std::getenv("SOG_PLANEFFT_E");
                const int Eonly = ee ? std::atoi(ee) : 0;
                auto pick = [&](int n, int B, FftStages& f, std::vector<double2>& tw, int& Esel) {
                    for (int E : {20, 16, 12, 10, 8})     // 12: lengths with radix 3 (576 = 2^6 3^2, 288, 96)
                        if (!Eonly || E == Eonly)
                            if (plane_fft_supported(n, E, B) && fft_plan_stages(n, f, tw, E)) {
                                Esel = E;
                                return true;
                            }
                    return false;
                };
                const int n2h = p.Iy / 2;
                if (pick(n2h, Brow, pl->prst, twr, pl->pr_E) && pick(p.Ix, Bx, pl->pxst, twx, pl->px_E)) {
                    pl->pr_B = Brow;
                    pl->px_B = Bx;
                    std::vector<double2> wp(n2h + 1);
                    for (int k = 0; k <= n2h; ++k) {
                        const long double a = -2.0L * 3.14159265358979323846264338327950288L * (long double)k /
                                              (long double)p.Iy;
                        wp[k] = make_double2((double)cosl(a), (double)sinl(a));
                    }
                    for (auto* pr : {&twr, &twx, &wp}) {
                        void** dst = pr == &twr ? &pl->d_prtw : pr == &twx ? &pl->d_pxtw : &pl->d_wpost;
                        if (pl->f32) {
                            std::vector<float2> t2(pr->size());
                            for (size_t i = 0; i < pr->size(); ++i)
                                t2[i] = make_float2((float)(*pr)[i].x, (float)(*pr)[i].y);
                            if ((rc = upload(pl, (float2**)dst, t2))) return rc;
                        } else if ((rc = upload(pl, (double2**)dst, *pr))) {
                            return rc;
                        }
                    }
                    pl->pfft = true;
                }
            }
            if (pl->zpass && pl->zr_E) {   // S5 table for the register-resident z pass
                const size_t n = (size_t)M * p.Izs;
                CK(cudaMalloc(&pl->d_mult, n * (pl->f32 ? sizeof(float) : sizeof(double))));
                pl->bytes += n * (pl->f32 ? sizeof(float) : sizeof(double));
                double* tmp = nullptr;
                if (pl->f32) CK(cudaMalloc((void**)&tmp, n * sizeof(double)));
                const int r = build_mult_table(pl->d_mult, M, nyh, p.Izs, p.m + 1, pl->d_A, pl->d_Tx, p.Ix, pl->d_Ty,
                                               pl->d_Tz, pl->f32, tmp, nullptr);
                CK(cudaDeviceSynchronize());
                if (tmp) cudaFree(tmp);
                if (r) return fail(SOG_ECUDA, "S5 multiplier table");
            }
            if (!pl->zpass) {   // zero-padded z pencils and their spectra for the cuFFT 1D chain
                CK(cudaMalloc((void**)&pl->mY, csz * (size_t)M * p.Izs));
                CK(cudaMemset(pl->mY, 0, csz * (size_t)M * p.Izs));   // z padding of the pencils stays zero
                pl->bytes += csz * (size_t)M * p.Izs;
                if ((rc = dalloc(pl, &pl->mspec, (size_t)p.Izs * p.Ix * nyh))) return rc;
            }
        } else {
            // distributed FFT: 2D (z, y) per interior x plane, all-to-all to ky chunks, 1D along x
            long long n2[2] = {p.Izs, p.Iy};
            long long ie[2] = {p.Izs, (long long)pl->Ixk * p.Iy}, oe[2] = {p.Izs, (long long)pl->Ixr * nyh};
            CKF(cufftCreate(&pl->f2f));
            CKF(cufftMakePlanMany64(pl->f2f, 2, n2, ie, 1, p.Iy, oe, 1, nyh, CUFFT_D2Z, pl->Ixr, &ws));
            pl->bytes += ws;
            CKF(cufftCreate(&pl->f2i));
            CKF(cufftMakePlanMany64(pl->f2i, 2, n2, oe, 1, nyh, ie, 1, p.Iy, CUFFT_Z2D, pl->Ixr, &ws));
            pl->bytes += ws;
            long long n1[1] = {p.Ix};
            CKF(cufftCreate(&pl->fxf));
            CKF(cufftMakePlanMany64(pl->fxf, 1, n1, nullptr, 1, p.Ix, nullptr, 1, p.Ix, CUFFT_Z2Z,
                                    (long long)p.Izs * pl->kc, &ws));
            pl->bytes += ws;
            const size_t nblk = pl->blk * pl->R;
            if ((rc = dalloc(pl, &pl->spec2, (size_t)p.Izs * pl->Ixr * nyh)) ||
                (rc = dalloc(pl, &pl->specx, (size_t)p.Izs * pl->kc * p.Ix)) || (rc = dalloc(pl, &pl->sbuf, nblk)) ||
                (rc = dalloc(pl, &pl->rbuf, nblk)) ||
                (rc = dalloc(pl, &pl->hsb, (size_t)2 * p.Izs * pl->HP * p.Iy)) ||
                (rc = dalloc(pl, &pl->hrb, (size_t)2 * p.Izs * pl->HP * p.Iy)))
                return rc;
        }
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
        else { t.TX = std::min(long_small_pcp(p.Pc) > 24 ? 8 : 16, p.Ilx); t.TY = std::min(16, p.Ily); }   // tgemm: <= 256 threads
        t.ntx = (p.Ilx + t.TX - 1) / t.TX;
        t.nty = (p.Ily + t.TY - 1) / t.TY;
        const int pl_half = (p.Pl - 1) / 2;
        t.full_range = (slab || t.TX + 2 * pl_half + 2 >= p.Ilx) ? 1 : 0;
        int ntile = t.ntx * t.nty;
        t.nchunk = std::max(1, std::min(4 * 148 / ntile + 1, int((p.N + 255) / 256)));
        if (!t.full_range && ntile < 4 * 148) t.nchunk = std::max(1, t.nchunk * 3);   // wide grids: tiles suffice
        t.ncx = pl->geo.ncx;
        t.cells_per_x = pl->geo.ncy * pl->geo.ncz;
        t.cell_w = p.Lx / pl->geo.ncx;
        t.Lx = p.Lx;
        t.ncy = pl->geo.ncy;
        t.ncz = pl->geo.ncz;
        t.cell_wy = p.Ly / pl->geo.ncy;
        t.Ly = p.Ly;
        auto gam = [&](double h) { double H = (p.Pl - 1) * h / 2.0; return std::exp(-2.0 * p.Sl / (H * H) * h * h); };
        t.gamma_x = gam(p.hlx());
        t.gamma_y = gam(p.hly());
        if (p.window != 0) kb_table(p.Pl, p.Sl, p.nul, p.window, pl->kbl);
        int pcmax = std::max(p.Pc <= 16 ? 16 : 32, long_small_pcp(p.Pc));   // tile kernel / tgemm partials
        if (t.nchunk > 1 && (rc = dalloc(pl, &pl->lpart, (size_t)ntile * t.nchunk * t.TX * t.TY * pcmax))) return rc;
        if ((rc = dalloc(pl, &pl->lpsiT, (size_t)p.Ilx * p.Ily * 32))) return rc;
        long long n[2] = {p.Ilx, p.Ily};
        size_t ws = 0;
        CKF(cufftCreate(&pl->lfwd));
        CKF(cufftMakePlanMany64(pl->lfwd, 2, n, nullptr, 1, (long long)p.Ilx * p.Ily, nullptr, 1,
                                (long long)p.Ilx * (p.Ily / 2 + 1), pl->f32 ? CUFFT_R2C : CUFFT_D2Z, p.Pc, &ws));
        pl->bytes += ws;
        CKF(cufftCreate(&pl->linv));
        CKF(cufftMakePlanMany64(pl->linv, 2, n, nullptr, 1, (long long)p.Ilx * (p.Ily / 2 + 1), nullptr, 1,
                                (long long)p.Ilx * p.Ily, pl->f32 ? CUFFT_C2R : CUFFT_Z2D, p.Pc, &ws));
        pl->bytes += ws;
        if (p.long_method == 1) {   // Alg. 3: direct sums over the R8-D modes
            if (slab) return fail(SOG_EINVAL, "the direct long range (long_method 1) is single-GPU only");
            DftArgs& d = pl->dft;
            d.Kx = p.Kx; d.Ky = p.Ky; d.nkx = 2 * p.Kx + 1; d.nky = p.Ky + 1; d.nmode = d.nkx * d.nky;
            const double twopi = 6.283185307179586476925286766559;
            d.kx1 = twopi / p.Lx; d.ky1 = twopi / p.Ly;
            if (!long_dft_ok(d, p.Pc)) return fail(SOG_EINVAL, "direct long range: too many modes (use long_method 0)");
            std::vector<double> Kd;
            build_long_kernel_direct(p, Kd);
            const size_t ns = 2 * (size_t)p.Pc * d.nmode;
            pl->lg_nblk = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 4, (p.N + 255) / 256));
            if ((rc = upload(pl, &pl->d_Kd, Kd)) || (rc = dalloc(pl, &pl->ldS, ns)) || (rc = dalloc(pl, &pl->ldP, ns)) ||
                (rc = dalloc(pl, &pl->ldpart, (size_t)pl->lg_nblk * long_small_pcp(p.Pc) * 2 * d.nmode)))
                return rc;
        }
    }
    pl->scan_bytes = std::max(scan_temp_bytes(pl->ncell), pl->nkeys ? scan_temp_bytes(pl->nkeys) : size_t(0));
    if ((rc = dalloc(pl, (char**)&pl->scan_tmp, pl->scan_bytes))) return rc;
    if (slab) {   // particle halos
        const int nown = pl->Ncap - 2 * pl->halo_cap;
        pl->nown_cap = nown;
        pl->sel_bytes = select_temp_bytes(nown);
        // the halo selects write into [left | right] halves of nown entries each, so clustered
        // input cannot overflow them; sends over halo_cap are rejected on every rank
        if ((rc = dalloc(pl, &pl->own, nown)) || (rc = dalloc(pl, &pl->hsend, 2 * (size_t)nown)) ||
            (rc = dalloc(pl, &pl->hrecv, 2 * pl->halo_cap)) || (rc = dalloc(pl, &pl->pos_long, N)) ||
            (rc = dalloc(pl, &pl->fl, nown)) || (rc = dalloc(pl, &pl->fr, nown)) || (rc = dalloc(pl, &pl->nsel, 4)) ||
            (rc = dalloc(pl, &pl->dstat, 8)) || (rc = dalloc(pl, &pl->lxyz, 3 * (size_t)N)) ||
            (rc = dalloc(pl, &pl->lq, N)) || (rc = dalloc(pl, (char**)&pl->sel_tmp, pl->sel_bytes)))
            return rc;
        CK(cudaMallocHost((void**)&pl->pin_i, 8 * sizeof(int)));
        CK(cudaMallocHost((void**)&pl->pin_d, 8 * sizeof(double)));
    }
    for (auto& e : pl->ev) CK(cudaEventCreate(&e));
    {   // SOG_NEAR_STREAM=off|low|high (default low): near-field side stream and its priority
        const char* env = std::getenv("SOG_NEAR_STREAM");
        const std::string mode = env ? env : "low";
        if (mode != "off") {
            int lo = 0, hi = 0;
            CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CK(cudaStreamCreateWithPriority(&pl->side, cudaStreamNonBlocking, mode == "high" ? hi : lo));
            CK(cudaEventCreateWithFlags(&pl->ev_fork, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&pl->ev_join, cudaEventDisableTiming));
        }
    }
    return SOG_OK;
}

int set_stream(sog_plan* pl, cudaStream_t s) {
    pl->stream = s;
    for (cufftHandle h : {pl->mfwd, pl->minv, pl->lfwd, pl->linv, pl->f2f, pl->f2i, pl->fxf, pl->fxi, pl->minv_full,
                          pl->mzfft})
        if (h) CKF(cufftSetStream(h, s));
    return SOG_OK;
}

MidArgs mid_args(const sog_plan* pl) {
    const Params& p = pl->p;
    MidArgs a;
    a.pos = pl->pos_s;
    a.N = pl->Ncur;
    a.Ix = p.Ix; a.Iy = p.Iy; a.Izs = p.Izs;
    a.hx = p.hx(); a.hy = p.hy(); a.hz = p.hz();
    a.halfx = 0.5 * p.Ix; a.halfy = 0.5 * p.Iy; a.halfz = 0.5 * p.Izs;
    a.hpx = 0.5 * p.Ix + 0.5; a.hpy = 0.5 * p.Iy + 0.5; a.hpz = 0.5 * p.Izs + 0.5;
    auto inv = [&](double h) { double H = (p.P - 1) * h / 2.0; return p.S / (H * H); };
    a.invH2Sx = inv(a.hx); a.invH2Sy = inv(a.hy); a.invH2Sz = inv(a.hz);
    a.Vh = a.hx * a.hy * a.hz;
    return a;
}

// R6-KB table: the degree-nu monomial coefficients, zero-padded to degree P + 3 (kernels_common.cuh)
void kb_table(int P, double beta, int nu, int window, KBTab& t) {
    std::vector<double> c;
    build_kb_poly(P, beta, nu, c, window);
    for (int i = 0; i < KB_TAB; ++i) t.c[i] = 0.0;
    for (int n = 0; n <= nu; ++n)
        for (int j = 0; j < P; ++j) t.c[n * P + j] = c[size_t(n) * P + j];
}

LongArgs long_args(const sog_plan* pl) {
    const Params& p = pl->p;
    LongArgs a;
    a.pos = pl->pos_s;
    a.N = pl->Ncur;
    a.Ilx = p.Ilx; a.Ily = p.Ily; a.Pc = p.Pc; a.Pl = p.Pl;
    a.hx = p.hlx(); a.hy = p.hly();
    a.halfx = 0.5 * p.Ilx; a.halfy = 0.5 * p.Ily;
    a.hpx = 0.5 * p.Ilx + 0.5; a.hpy = 0.5 * p.Ily + 0.5;
    auto inv = [&](double h) { double H = (p.Pl - 1) * h / 2.0; return p.Sl / (H * H); };
    a.invH2Sx = inv(a.hx); a.invH2Sy = inv(a.hy);
    a.two_over_Lz = 2.0 / p.Lz;
    a.A = a.hx * a.hy;
    a.C = pl->d_C;
    a.kb = p.window != 0 ? 1 : 0;
    a.kt = pl->kbl;
    return a;
}

int lchk(int r) {
    if (r == 1) return fail(SOG_EINVAL, "window support / proxy count outside the compiled range");
    if (r == 2) return fail(SOG_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(cudaGetLastError()));
    return SOG_OK;
}

// NVTX ranges (host-side, one per pipeline stage; a no-op unless a profiler injects NVTX): the
// range opened at mark k covers the launches of stage k
const char* const kStageName[] = {"sog S1 sort", "sog S2 near", "sog S3 mid spread", "sog S4 mid FFT",
                                  "sog S5 mid scale", "sog S6 mid IFFT", "sog S7 mid gather",
                                  "sog S8 long spread", "sog S9-S11 long FFT/scale/IFFT", "sog S12 long gather",
                                  "sog S13 combine"};
void mark(sog_plan* pl, int k) {
    if (pl->flags & SOG_TIMING) cudaEventRecord(pl->ev[k], pl->stream);
    if (pl->nvtx_open) nvtxRangePop();
    pl->nvtx_open = k < 11;
    if (pl->nvtx_open) nvtxRangePushA(kStageName[k]);
}

// ---- pipeline stages (sorted order outputs o_near / o_mid / o_long) --------------------------

// S1: validate, canonicalise, cell sort, stencil origins, mid order.  N = local particle count.
int st_sort(sog_plan* pl, const double* xyz, const double* q, int N) {
    const Params& p = pl->p;
    cudaStream_t st = pl->stream;
    int rc;
    pl->Ncur = N;
    CK(cudaMemsetAsync(pl->count, 0, sizeof(int) * (pl->ncell + 1), st));
    CK(cudaMemsetAsync(pl->dflags, 0, sizeof(unsigned), st));
    CK(cudaMemsetAsync(pl->qsums, 0, sizeof(double) * 4, st));
    if (N == 0) {   // an empty slab: empty buckets everywhere
        if (pl->has_mid) CK(cudaMemsetAsync(pl->mstart, 0, sizeof(int) * (pl->nkeys + 1), st));
        return SOG_OK;
    }
    const int nb = (N + 255) / 256;
    k_prepare<<<nb, 256, 0, st>>>(xyz, q, N, pl->geo, pl->pos, pl->cell, pl->count, pl->dflags, pl->qsums);
    if ((rc = lchk(launch_exclusive_scan(pl->count, pl->start, pl->ncell, pl->scan_tmp, pl->scan_bytes, st)))) return rc;
    CK(cudaMemcpyAsync(pl->cursor, pl->start, sizeof(int) * pl->ncell, cudaMemcpyDeviceToDevice, st));
    k_scatter<<<nb, 256, 0, st>>>(pl->cell, N, pl->cursor, pl->tmp);
    k_cellsort<<<(pl->ncell * 32 + 255) / 256, 256, 0, st>>>(pl->start, pl->ncell, pl->tmp, pl->pos, pl->pos_s, pl->perm,
                                                            pl->iperm);
    {
        MidArgs ma{};
        if (pl->has_mid) ma = mid_args(pl);
        if ((rc = lchk(launch_stencil_origins(pl->pos_s, N, ma, pl->has_mid ? 1 : 0, p.hlx(), p.hly(), 0.5 * p.Ilx + 0.5,
                                              0.5 * p.Ily + 0.5, pl->g0, st))))
            return rc;
    }
    if (pl->has_mid) {   // mid order: bucket by (stencil-start tile, z chunk)
        MidSortArgs ms{p.Ix, p.Iy, (p.P - 1) / 2, pl->mz.nty, pl->mz.nzc, pl->mz.px, pl->mz.xorig};
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
    return SOG_OK;
}

// S2 near field (+ nothing else; the self term is removed in the combine)
int st_near(sog_plan* pl) {
    const Params& p = pl->p;
    const int N = pl->Ncur;
    cudaStream_t st = pl->stream;
    int rc;
    if (N == 0) return SOG_OK;
    const int D = pl->near.D;
    if (D != NEAR_D) return fail(SOG_EINVAL, "near table degree");
    if (pl->f32 && pl->geo.ncx >= 3 && pl->geo.ncy >= 3) {   // fp32 mode: cell-relative fp32 (k_near3f)
        // (boxes with < 3 cells per periodic axis use the generic fp64 kernel below)
        Near3Args a;
        a.pos = pl->pos_s; a.start = pl->start; a.cF = pl->d_cF; a.out = pl->o_near;
        a.K = pl->near.K; a.du = pl->near.du; a.inv_du = pl->near.inv_du; a.rc2 = p.rc * p.rc;
        a.g = pl->geo;
        a.cap = 2048;
        size_t sh = sizeof(float) * ((pl->near.K * (D + 1) + 3) & ~3) + NEAR3_WARPS * 160 * sizeof(int) +
                    sizeof(float4) * a.cap;
        CK(cudaFuncSetAttribute(k_near3f<NEAR_D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
        k_near3f<NEAR_D><<<pl->ncell, 32 * NEAR3_WARPS, sh, st>>>(a);
    } else if (pl->near4 && pl->near_mode == 6) {   // k_near5: each pair once (+ fold of the partials)
        Near5Args a;
        a.pos = pl->pos_s; a.start = pl->start; a.out = pl->o_near; a.part = pl->npart;
        a.rc2 = p.rc * p.rc;
        a.rc2f = (float)(a.rc2 * (1.0 + 1e-5)) + 1e-5f;
        a.g = pl->geo;
        a.cap = pl->n5_cap;
        if ((rc = lchk(launch_near5(a, pl->npoly, pl->ncell, st)))) return rc;
        if ((rc = lchk(launch_near_fold(pl->o_near, pl->npart, N, st)))) return rc;
    } else if (pl->near4 && pl->near_mode == 5) {   // k_near3 with the single polynomial (R16-G)
        Near3Args a;
        a.pos = pl->pos_s; a.start = pl->start; a.cF = pl->d_cF; a.out = pl->o_near;
        a.K = pl->near.K; a.du = pl->near.du; a.inv_du = pl->near.inv_du; a.rc2 = p.rc * p.rc;
        a.g = pl->geo;
        a.cap = 1536;
        a.rc2f = (float)(a.rc2 * (1.0 + 1e-5)) + 1e-5f;
        if (pl->R > 1) { a.perm = pl->perm; a.nown = pl->Nown; }   // x-slab: own targets only
        if ((rc = lchk(launch_near3p(a, pl->npoly, pl->ncell, st)))) return rc;
    } else if (pl->near4) {   // k_near4: target-stationary, one polynomial (R16-G)
        Near4Args a;
        a.pos = pl->pos_s; a.start = pl->start; a.out = pl->o_near;
        a.g = pl->geo;
        a.rc2 = p.rc * p.rc;
        a.rc2f = (float)(a.rc2 * (1.0 + 1e-6)) + 1e-4f;
        a.rcz = (float)(p.rc * (1.0 + 1e-6)) + 1e-4f;
        a.kc = pl->n4_kc;
        a.cap = pl->n4_cap;
        if ((rc = lchk(launch_near4(a, pl->npoly, pl->n4_nw, st)))) return rc;
    } else if (pl->geo.ncx >= 3 && pl->geo.ncy >= 3 && N < (1 << 27)) {   // k_near3: warp per target
        Near3Args a;
        a.pos = pl->pos_s; a.start = pl->start; a.cF = pl->d_cF; a.out = pl->o_near;
        a.K = pl->near.K; a.du = pl->near.du; a.inv_du = pl->near.inv_du; a.rc2 = p.rc * p.rc;
        a.g = pl->geo;
        a.cap = 1536;                            // multiple of 128 (packed staging layout)
        a.rc2f = (float)(a.rc2 * (1.0 + 1e-5)) + 1e-5f;
        if (pl->R > 1) { a.perm = pl->perm; a.nown = pl->Nown; }   // x-slab: own targets only
        size_t sh = sizeof(double) * ((pl->near.K * (D + 1) + 1) & ~1) + 10 * sizeof(double2) +
                    NEAR3_WARPS * 160 * sizeof(int) + 16 * a.cap;
        CK(cudaFuncSetAttribute(k_near3<NEAR_D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
        k_near3<NEAR_D><<<pl->ncell, 32 * NEAR3_WARPS, sh, st>>>(a);
    } else {
        if (!pl->geo.px) return fail(SOG_EINVAL, "x-slab needs >= 3 near cells per axis");
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
    return SOG_OK;
}

int st_mid_spread(sog_plan* pl) {
    return lchk(launch_mid_spread_z(pl->mz, pl->p.P, pl->nseg_s, pl->mgrid, pl->f32, pl->stream));
}

int st_mid_gather(sog_plan* pl) {
    MidZArgs g = pl->mz;
    g.cps = pl->mz_cps_g;
    if (pl->R > 1) { g.tlo -= 1; g.ntout += 1; }   // own particles near the left edge start in the halo tile
    return lchk(launch_mid_gather_z(g, pl->p.P, pl->nseg_g, pl->Ncur, pl->mpsi, pl->o_mid, pl->f32, pl->stream));
}

// S8 (own particles only in an x-slab: the halo particles belong to the neighbours)
int st_long_spread(sog_plan* pl) {
    const Params& p = pl->p;
    cudaStream_t st = pl->stream;
    int rc;
    LongArgs la = long_args(pl);
    if (pl->R > 1) {
        k_own_mask<<<(pl->Ncur + 255) / 256, 256, 0, st>>>(pl->pos_s, pl->perm, pl->Ncur, pl->Nown, pl->pos_long);
        la.pos = pl->pos_long;
    }
    if (p.long_method == 1)
        return lchk(launch_long_dft_spread(la, pl->dft, pl->lg_nblk, pl->ldpart, pl->ldS, pl->f32, st));
    if (pl->long_small) {
        if ((rc = lchk(launch_long_spread_gemm(la, pl->g0, pl->lt.gamma_x, pl->lt.gamma_y, pl->lg_nblk, pl->lpart2,
                                               pl->lgrid, pl->f32, st))))
            return rc;
    } else {
        if (pl->f32) return fail(SOG_EINVAL, "fp32 mode needs a small long grid (register-tiled path)");
        LongTileArgs t = pl->lt;
        t.a = la;
        t.start = pl->start;
        t.part = pl->lpart;
        // wide grids: the register-tiled product per column tile; the per-column tile kernel when
        // the thread tile does not fit (Pc > 24)
        const int r = launch_long_spread_tgemm(t, pl->lgrid, st);
        if (r == 1) {
            if ((rc = lchk(launch_long_spread_tile(t, p.Pl, pl->lgrid, st)))) return rc;
        } else if ((rc = lchk(r))) {
            return rc;
        }
    }
    return SOG_OK;
}

// S9-S11
int st_long_solve(sog_plan* pl) {
    const Params& p = pl->p;
    cudaStream_t st = pl->stream;
    int rc;
    if (p.long_method == 1)
        return lchk(launch_long_scale(pl->ldS, pl->ldP, pl->d_Kd, pl->dft.nmode, p.Pc, pl->f32, st));
    const int nmode = p.Ilx * (p.Ily / 2 + 1);
    if (pl->f32) {
        CKF(cufftExecR2C(pl->lfwd, (float*)pl->lgrid, (cufftComplex*)pl->lspec));
        if ((rc = lchk(launch_long_scale(pl->lspec, pl->lspec2, pl->d_K, nmode, p.Pc, true, st)))) return rc;
        CKF(cufftExecC2R(pl->linv, (cufftComplex*)pl->lspec2, (float*)pl->lgrid));
    } else {
        CKF(cufftExecD2Z(pl->lfwd, pl->lgrid, pl->lspec));
        if ((rc = lchk(launch_long_scale(pl->lspec, pl->lspec2, pl->d_K, nmode, p.Pc, false, st)))) return rc;
        CKF(cufftExecZ2D(pl->linv, pl->lspec2, pl->lgrid));
    }
    return SOG_OK;
}

// S12
int st_long_gather(sog_plan* pl) {
    const Params& p = pl->p;
    if (p.long_method == 1)
        return lchk(launch_long_dft_gather(long_args(pl), pl->dft, pl->ldP, pl->o_long, pl->f32, pl->stream));
    if (pl->long_small)
        return lchk(launch_long_gather_bc(long_args(pl), pl->g0, pl->lgrid, pl->o_long, pl->f32, pl->stream));
    if (pl->f32) return fail(SOG_EINVAL, "fp32 mode needs a small long grid (register-tiled path)");
    return lchk(launch_long_gather2(long_args(pl), p.Pl, pl->lgrid, pl->lpsiT, pl->o_long, pl->lt.gamma_x,
                                    pl->lt.gamma_y, pl->stream));
}

// Whole-box pipeline: sort + all three components (sorted order).  stop_stage > 0 returns
// early for sog_debug_stage.
int run_pipeline(sog_plan* pl, const double* xyz, const double* q, int stop_stage = 0) {
    const Params& p = pl->p;
    cudaStream_t st = pl->stream;
    mark(pl, 0);
    int rc;
    if ((rc = st_sort(pl, xyz, q, int(p.N)))) return rc;
    mark(pl, 1);
    // near field: on the side stream, concurrent with the mid / long chain (not when per-stage
    // timings are collected: they need the stages in sequence)
    const bool overlap = !stop_stage && pl->side && !(pl->flags & SOG_TIMING);
    if (overlap) {
        CK(cudaEventRecord(pl->ev_fork, st));
        CK(cudaStreamWaitEvent(pl->side, pl->ev_fork, 0));
        pl->stream = pl->side;
        rc = st_near(pl);
        pl->stream = st;
        if (rc) return rc;
        CK(cudaEventRecord(pl->ev_join, pl->side));
    } else if (!stop_stage && (rc = st_near(pl))) {
        return rc;
    }
    mark(pl, 2);
    // S3-S7 mid range
    if (pl->has_mid && (stop_stage == 0 || stop_stage == 1 || stop_stage == 2)) {
        if ((rc = st_mid_spread(pl))) return rc;
        mark(pl, 3);
        if (stop_stage == 1) return SOG_OK;
        // S4: 2D FFTs of the written planes, transpose to zero-padded z pencils, FFT along z
        const int nyh = p.Iy / 2 + 1;
        const long long M = (long long)p.Ix * nyh;
        const size_t gp = (size_t)p.Ix * p.Iy;
        if (pl->pfft) {
            const size_t esz = pl->f32 ? sizeof(float) : sizeof(double);
            if ((rc = lchk(launch_rows_fft(false, (const char*)pl->mgrid + esz * gp * pl->zs0, pl->mX,
                                           (long long)pl->nzf * p.Ix, nyh, pl->prst, pl->d_prtw, pl->d_wpost, pl->f32,
                                           pl->pr_E, pl->pr_B, st))) ||
                (rc = lchk(launch_xfft(false, pl->mX, pl->nzf, p.Ix, nyh, pl->pxst, pl->d_pxtw, pl->f32, pl->px_E,
                                       pl->px_B, st))))
                return rc;
        } else if (pl->f32) {
            CKF(cufftExecR2C(pl->mfwd, (float*)pl->mgrid + gp * pl->zs0, (cufftComplex*)pl->mX));
        } else {
            CKF(cufftExecD2Z(pl->mfwd, pl->mgrid + gp * pl->zs0, pl->mX));
        }
        const bool full = stop_stage == 2;
        const int z0 = full ? 0 : pl->zg0, nz = full ? p.Izs : pl->nzg;
        if (pl->zpass) {
            // S4 (z), S5, S6 (z) in one kernel, in place on the plane spectra
            mark(pl, 4);
            if (pl->zr_E) {
                // TMA row blocks (fp64) unless SOG_ZPASS_TMA=0; 1 = not supported: thread loads
                static const bool tma = !(std::getenv("SOG_ZPASS_TMA") && std::atoi(std::getenv("SOG_ZPASS_TMA")) == 0);
                int zr = pl->f32 || !tma ? 1 : launch_zpass_t(pl->mX, M, pl->zs0, pl->nzf, z0, nz, pl->zst, pl->d_ztw,
                                                               pl->d_mult, pl->zr_E, pl->zr_B, st);
                if (zr == 1)
                    zr = launch_zpass_r(pl->mX, M, pl->zs0, pl->nzf, z0, nz, pl->zst, pl->d_ztw, pl->d_mult, pl->f32,
                                        pl->zr_E, pl->zr_B, st);
                if ((rc = lchk(zr))) return rc;
            } else if ((rc = lchk(launch_zpass(pl->mX, M, nyh, pl->zs0, pl->nzf, z0, nz, pl->zst, pl->d_ztw, p.m + 1,
                                               pl->d_A, pl->d_Tx, p.Ix, pl->d_Ty, pl->d_Tz, pl->f32, st)))) {
                return rc;
            }
            mark(pl, 5);
        } else {
        if ((rc = lchk(launch_zfft_transpose(pl->mX, pl->mY, pl->nzf, M, p.Izs, pl->zs0, true, pl->f32, st)))) return rc;
        if (pl->f32) CKF(cufftExecC2C(pl->mzfft, (cufftComplex*)pl->mY, (cufftComplex*)pl->mspec, CUFFT_FORWARD));
        else CKF(cufftExecZ2Z(pl->mzfft, pl->mY, pl->mspec, CUFFT_FORWARD));
        mark(pl, 4);
        // S5 on the z pencils
        if ((rc = lchk(launch_scale_pencil_z(pl->mspec, p.Ix, nyh, p.Izs, p.m + 1, pl->d_A, pl->d_Tx, pl->d_Ty, pl->d_Tz,
                                             pl->f32, st))))
            return rc;
        mark(pl, 5);
        // S6: inverse along z, back to planes (only those the gather reads; all for the debug stage)
        if (pl->f32) CKF(cufftExecC2C(pl->mzfft, (cufftComplex*)pl->mspec, (cufftComplex*)pl->mspec, CUFFT_INVERSE));
        else CKF(cufftExecZ2Z(pl->mzfft, pl->mspec, pl->mspec, CUFFT_INVERSE));
        if ((rc = lchk(launch_zfft_transpose(pl->mspec, pl->mX, nz, M, p.Izs, z0, false, pl->f32, st)))) return rc;
        }
        const cufftHandle inv = full ? pl->minv_full : pl->minv;
        if (pl->pfft) {
            const size_t esz = pl->f32 ? sizeof(float) : sizeof(double);
            if ((rc = lchk(launch_xfft(true, pl->mX, nz, p.Ix, nyh, pl->pxst, pl->d_pxtw, pl->f32, pl->px_E, pl->px_B,
                                       st))) ||
                (rc = lchk(launch_rows_fft(true, pl->mX, (char*)pl->mpsi + esz * gp * z0, (long long)nz * p.Ix, nyh,
                                           pl->prst, pl->d_prtw, pl->d_wpost, pl->f32, pl->pr_E, pl->pr_B, st))))
                return rc;
        } else if (pl->f32) {
            CKF(cufftExecC2R(inv, (cufftComplex*)pl->mX, (float*)pl->mpsi + gp * z0));
        } else {
            CKF(cufftExecZ2D(inv, pl->mX, pl->mpsi + gp * z0));
        }
        mark(pl, 6);
        if (stop_stage == 2) return SOG_OK;
        if ((rc = st_mid_gather(pl))) return rc;
    } else if (!pl->has_mid && !stop_stage) {
        CK(cudaMemsetAsync(pl->o_mid, 0, sizeof(d4) * pl->Ncur, st));
    }
    mark(pl, 7);
    // S8-S12 long range
    if (stop_stage == 0 || stop_stage == 3 || stop_stage == 4) {
        if ((rc = st_long_spread(pl))) return rc;
        mark(pl, 8);
        if (stop_stage == 3) return SOG_OK;
        if ((rc = st_long_solve(pl))) return rc;
        mark(pl, 9);
        if (stop_stage == 4) return SOG_OK;
        if ((rc = st_long_gather(pl))) return rc;
    }
    if (overlap) CK(cudaStreamWaitEvent(st, pl->ev_join, 0));
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
    if (o && o->precision != 0 && o->precision != 1) return fail(SOG_EINVAL, "precision must be 0 (fp64) or 1 (fp32)");
    if (o && o->precision == 1 && tol < 1e-5) return fail(SOG_EINFEASIBLE, "fp32 mode supports tol >= 1e-5");
    std::string err;
    if (o && o->explicit_params) {
        static const double tb[6][3] = {{2.0, 1.9892536839080267, 0.9944464927622323},
                                        {1.62976708826776469, 2.7520026668023417, 1.0078069793438068},
                                        {1.48783512395703226, 3.7554672283554990, 0.9919117057598183},
                                        {1.32070036405934420, 4.3914554711638349, 1.0018891411481198},
                                        {1.21812525709410644, 5.6355288151271085, 1.0009014615603334},
                                        {1.14878150173321925, 7.2956245490719404, 1.0000368348358225}};
        if (o->b > 1.0) {   // general b (NEXT #4): verbatim
            p.row = -1; p.b = o->b; p.r0 = o->r0; p.omega = o->omega;
        } else {
            if (o->row < 0 || o->row > 5) return fail(SOG_EINVAL, "row must be 0..5");
            p.row = o->row; p.b = tb[o->row][0]; p.r0 = tb[o->row][1]; p.omega = tb[o->row][2];
        }
        p.rc = o->rc; p.sigma = p.rc / p.r0; p.M = o->M; p.m = o->m;
        p.Ix = o->Ix; p.Iy = o->Iy; p.Iz = o->Iz; p.Izs = o->Izs; p.P = o->P; p.S = o->S;
        p.Ilx = o->Ilx; p.Ily = o->Ily; p.Pl = o->Pl; p.Sl = o->Sl; p.Pc = o->Pc;
        p.window = o->window;
        p.long_method = o->long_method;
        p.Kx = o->Kx;
        p.Ky = o->Ky;
        if (p.window != 0) {
            p.nu = p.m >= 0 ? (o->nu > 0 ? o->nu : p.P + knobs.kb_nu_extra) : 0;
            p.nul = o->nul > 0 ? o->nul : p.Pl + knobs.kb_nu_extra;
        }
    } else {
        if (o && (o->window < 0 || o->window > 2)) return fail(SOG_EINVAL, "window must be 0, 1 or 2");
        if (o && o->long_method != 0 && o->long_method != 1) return fail(SOG_EINVAL, "long_method must be 0 or 1");
        p.window = o ? o->window : 0;
        p.long_method = o ? o->long_method : 0;
        if (o && o->b != 0.0) {
            if (!(o->b > 1.0 && o->b <= 2.0)) return fail(SOG_EINVAL, "b must lie in (1, 2]");
            p.b = o->b;   // general b: choose_params runs the C^1 solve
        }
        if (o && o->rc_factor > 0) knobs.rc_factor = o->rc_factor;
        if (o && o->eta > 0) knobs.eta = o->eta;
        if (o && o->optimize) {
            if (!choose_params_opt(p, knobs, err)) return fail(SOG_EINFEASIBLE, err);
        } else if (!choose_params(p, knobs, err)) {
            return fail(SOG_EINFEASIBLE, err);
        }
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
    pl->f32 = o && o->precision == 1;
    int rc = setup(pl);
    if (rc == SOG_OK) rc = set_stream(pl, o ? (cudaStream_t)o->cuda_stream : nullptr);
    if (rc != SOG_OK) { std::string keep = g_err; free_plan(pl); g_err = keep; return nullptr; }
    return pl;
}

sog_plan* sog_plan_create(int64_t N, double Lx, double Ly, double Lz, double tol) {
    return sog_plan_create_ex(N, Lx, Ly, Lz, tol, nullptr);
}

void sog_plan_destroy(sog_plan* p) { free_plan(p); }

namespace {
int eval_body(sog_plan* pl, const double* xyz, const double* q, double* phi, double* force) {
    int rc = run_pipeline(pl, xyz, q);
    if (rc) return rc;
    const int N = int(pl->p.N);
    if (pl->o_tot) {
        k_combine_s<<<(N + 255) / 256, 256, 0, pl->stream>>>(pl->o_near, pl->o_mid, pl->o_long, pl->pos_s, N, pl->selfc,
                                                             pl->o_tot, pl->epart);
        k_combine_u<<<(N + 255) / 256, 256, 0, pl->stream>>>(pl->o_tot, pl->iperm, N, phi, force);
    } else {
        k_combine_g<<<(N + 255) / 256, 256, 0, pl->stream>>>(pl->o_near, pl->o_mid, pl->o_long, pl->pos_s, pl->iperm, N,
                                                             pl->selfc, phi, force, pl->epart);
    }
    k_sum_partials<<<1, 1024, 0, pl->stream>>>(pl->epart, (N + 255) / 256, pl->qsums + 2);
    CK(cudaGetLastError());
    mark(pl, 11);
    return SOG_OK;
}

// capture eval_body into a CUDA graph (the launch sequence has no host synchronisation), or
// reuse the instantiated one when the caller's buffers are the same as last time
int eval_graph(sog_plan* pl, const double* xyz, const double* q, double* phi, double* force) {
    const void* key[4] = {xyz, q, phi, force};
    if (!pl->gexec || std::memcmp(key, pl->gkey, sizeof key) != 0) {
        if (pl->gexec) { cudaGraphExecDestroy(pl->gexec); pl->gexec = nullptr; }
        const unsigned saved = pl->flags;
        pl->flags &= ~SOG_TIMING;                       // no event nodes in the graph
        // capture on a private stream (the plan's stream may be the legacy default stream); the
        // graph is launched on the plan's stream
        if (!pl->gstream) CK(cudaStreamCreateWithFlags(&pl->gstream, cudaStreamNonBlocking));
        const cudaStream_t user = pl->stream;
        CK(cudaStreamSynchronize(user));                // no pending plan work crosses into the capture
        int rc = set_stream(pl, pl->gstream);
        if (rc) return rc;
        CK(cudaStreamBeginCapture(pl->gstream, cudaStreamCaptureModeRelaxed));
        rc = eval_body(pl, xyz, q, phi, force);
        cudaGraph_t g = nullptr;
        const cudaError_t e = cudaStreamEndCapture(pl->gstream, &g);
        pl->flags = saved;
        const int rs = set_stream(pl, user);
        if (rs) { if (g) cudaGraphDestroy(g); return rs; }
        if (rc) { if (g) cudaGraphDestroy(g); return rc; }
        if (e != cudaSuccess) return fail(SOG_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
        const cudaError_t ei = cudaGraphInstantiate(&pl->gexec, g, 0);
        cudaGraphDestroy(g);
        if (ei != cudaSuccess) { pl->gexec = nullptr; return fail(SOG_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei)); }
        std::memcpy(pl->gkey, key, sizeof key);
    }
    nvtxRangePushA("sog_eval (CUDA graph replay)");
    const cudaError_t el = cudaGraphLaunch(pl->gexec, pl->stream);
    nvtxRangePop();
    CK(el);
    return SOG_OK;
}
}  // namespace

int sog_eval(sog_plan* pl, const double* xyz, const double* q, double* phi, double* force) {
    if (!pl || !xyz || !q) return fail(SOG_EINVAL, "null argument");
    const int rc = (pl->flags & SOG_GRAPH) && pl->R <= 1 ? eval_graph(pl, xyz, q, phi, force)
                                                         : eval_body(pl, xyz, q, phi, force);
    if (rc) return rc;
    if (!(pl->flags & SOG_GRAPH)) collect_timings(pl);
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

int sog_eval_host_async(sog_plan* pl, const double* xyz, const double* q, double* phi, double* force) {
    if (!pl || !xyz || !q) return fail(SOG_EINVAL, "null argument");
    if (pl->R > 1) return fail(SOG_EINVAL, "the pipelined host path is single-GPU (use sog_dist_eval)");
    const size_t N = pl->p.N;
    int rc;
    if (!pl->cin) {
        for (int i = 0; i < 2; ++i) {
            if ((rc = dalloc(pl, &pl->ax[i], 3 * N)) || (rc = dalloc(pl, &pl->aq[i], N)) ||
                (rc = dalloc(pl, &pl->aphi[i], N)) || (rc = dalloc(pl, &pl->aforce[i], 3 * N)))
                return rc;
            CK(cudaEventCreateWithFlags(&pl->ev_in[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&pl->ev_comp[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&pl->ev_out[i], cudaEventDisableTiming));
        }
        if ((rc = dalloc(pl, &pl->astat, 1))) return rc;
        CK(cudaMemset(pl->astat, 0, sizeof(unsigned)));
        CK(cudaStreamCreateWithFlags(&pl->cin, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&pl->cout, cudaStreamNonBlocking));
    }
    const int sl = pl->aslot;
    pl->aslot ^= 1;
    // inputs: staging set sl, once the evaluation two calls back has consumed it
    if (pl->a_used[sl]) CK(cudaStreamWaitEvent(pl->cin, pl->ev_comp[sl], 0));
    CK(cudaMemcpyAsync(pl->ax[sl], xyz, 3 * N * sizeof(double), cudaMemcpyHostToDevice, pl->cin));
    CK(cudaMemcpyAsync(pl->aq[sl], q, N * sizeof(double), cudaMemcpyHostToDevice, pl->cin));
    CK(cudaEventRecord(pl->ev_in[sl], pl->cin));
    // evaluation on the plan's stream once the inputs are in and set sl's previous outputs are out
    CK(cudaStreamWaitEvent(pl->stream, pl->ev_in[sl], 0));
    if (pl->a_used[sl]) CK(cudaStreamWaitEvent(pl->stream, pl->ev_out[sl], 0));
    const unsigned saved = pl->flags;
    pl->flags &= ~(unsigned)(SOG_GRAPH | SOG_TIMING);    // alternating pointers: no graph; no host syncs
    rc = eval_body(pl, pl->ax[sl], pl->aq[sl], phi ? pl->aphi[sl] : nullptr, force ? pl->aforce[sl] : nullptr);
    pl->flags = saved;
    if (rc) return rc;
    if (!(pl->flags & SOG_NO_VALIDATE)) k_status_accum<<<1, 1, 0, pl->stream>>>(pl->dflags, pl->qsums, pl->astat);
    CK(cudaEventRecord(pl->ev_comp[sl], pl->stream));
    // outputs back on the copy-out stream
    CK(cudaStreamWaitEvent(pl->cout, pl->ev_comp[sl], 0));
    if (phi) CK(cudaMemcpyAsync(phi, pl->aphi[sl], N * sizeof(double), cudaMemcpyDeviceToHost, pl->cout));
    if (force) CK(cudaMemcpyAsync(force, pl->aforce[sl], 3 * N * sizeof(double), cudaMemcpyDeviceToHost, pl->cout));
    CK(cudaEventRecord(pl->ev_out[sl], pl->cout));
    pl->a_used[sl] = true;
    return SOG_OK;
}

int sog_host_wait(sog_plan* pl) {
    if (!pl) return fail(SOG_EINVAL, "null plan");
    if (!pl->cin) return SOG_OK;
    CK(cudaStreamSynchronize(pl->cout));
    CK(cudaStreamSynchronize(pl->stream));
    unsigned f = 0;
    CK(cudaMemcpy(&f, pl->astat, sizeof(unsigned), cudaMemcpyDeviceToHost));
    CK(cudaMemset(pl->astat, 0, sizeof(unsigned)));
    double e = 0.0;
    CK(cudaMemcpy(&e, pl->qsums + 2, sizeof(double), cudaMemcpyDeviceToHost));
    pl->last_energy = e;
    if (f & FLAG_NONFINITE) return fail(SOG_ENONFINITE, "non-finite position or charge (pipelined call)");
    if (f & FLAG_ZRANGE) return fail(SOG_EZRANGE, "z outside [-Lz/2, Lz/2] (pipelined call)");
    if (f & 4u) return fail(SOG_ENONNEUTRAL, "system not charge neutral (pipelined call)");
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
    if (pl->f32) return fail(SOG_EINVAL, "debug stages are available in fp64 mode only");
    const Params& p = pl->p;
    size_t need;
    const double* src;
    if (stage == 1 || stage == 2) {
        if (!pl->has_mid) return fail(SOG_EINVAL, "plan has no mid-range part (m < 0)");
        need = (size_t)p.Ix * p.Iy * p.Izs;
        src = stage == 1 ? pl->mgrid : pl->mpsi;
    } else if (stage == 3 || stage == 4) {
        if (p.long_method == 1) return fail(SOG_EINVAL, "stages 3, 4 are the FFT long range's grids (long_method 0)");
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
    char extra[1024];
    std::snprintf(extra, sizeof extra,
                  "ncell=%d\nnear_table_pieces=%d\nnear_table_degree=%d\nnear_table_max_rel_err=%.3e\n"
                  "self_coefficient=%.17g\nworkspace_bytes=%zu\nzpass=%d\nnear_kernel=%d\nnear_poly_degree=%d\n"
                  "near_poly_err_F=%.3e\nnear_poly_err_dF=%.3e\n",
                  pl->ncell, pl->near.K, pl->near.D, pl->near.max_rel_err, pl->selfc, pl->bytes, pl->zpass ? 1 : 0,
                  pl->near4 ? pl->near_mode : 3, pl->npoly.D, pl->npoly.err_F, pl->npoly.err_dF);
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
    // launches of this library's own kernels per whole-box evaluation (CUB's scan kernels counted,
    // cuFFT's not): sort = prepare, scan (init + scan), scatter, cellsort, stencil origins; near
    // (+ fold for k_near5); mid = key, scan (2), place (scatter + bucket), spread, plane FFTs (rows +
    // x, forward and inverse: 4) or the cuFFT chain's transposes (2), z pass (1) or pencil scale (1),
    // gather; long = spread (+ sum), scale, [transpose,] gather; combine + energy sum
    int n = 1 + 2 + 1 + 1 + 1;
    n += 1 + (pl->near4 && pl->near_mode == 6 ? 1 : 0);
    if (pl->has_mid) n += 1 + 2 + 2 + 1 + (pl->pfft ? 4 : 0) + (pl->zpass ? 1 : 3) + 1;
    n += pl->p.long_method == 1 ? 4 : (pl->long_small ? 4 : 5);
    return n + (pl->o_tot ? 3 : 2);
}

}  // extern "C"

// =========================================================================================
// x-slab distributed evaluation.  One sog_plan per rank in slab mode; the
// exchange steps are expressed as per-rank send/receive lists and executed either by NCCL
// (one process per GPU) or by a loopback backend (R virtual ranks of one process on one
// device, device-to-device copies): the same decomposition runs in both.
// =========================================================================================
#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// NCCL is resolved at run time (the process's already-loaded libnccl.so.2, e.g. torch's),
// so libsog.so loads and runs single-GPU without it.
NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return api;
    auto sym = [&](auto& fp, const char* name) { fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name)); return fp != nullptr; };
    api.ok = sym(api.GetUniqueId, "ncclGetUniqueId") && sym(api.CommInitRank, "ncclCommInitRank") &&
             sym(api.CommDestroy, "ncclCommDestroy") && sym(api.GroupStart, "ncclGroupStart") &&
             sym(api.GroupEnd, "ncclGroupEnd") && sym(api.Send, "ncclSend") && sym(api.Recv, "ncclRecv") &&
             sym(api.AllReduce, "ncclAllReduce") && sym(api.GetErrorString, "ncclGetErrorString");
    return api;
}

struct Msg {
    int peer;
    void* ptr;
    size_t bytes;
};
struct Exch {
    std::vector<Msg> send, recv;
};

bool smooth7l(long n) {
    for (long f : {2L, 3L, 5L, 7L})
        while (n % f == 0) n /= f;
    return n == 1;
}

}  // namespace

struct sog_dist {
    int R = 1;
    bool loopback = false;
    std::vector<sog_plan*> pl;           // loopback: all R ranks; NCCL: this process's rank
    ncclComm_t comm = nullptr;
    cudaStream_t stream = nullptr;
    // SOG_TIMING: phase boundaries on the ranks' stream + the near field on plan 0's side stream
    bool timing = false;
    cudaEvent_t ev[12] = {}, nev[2] = {};
    double ms[12] = {};
};

namespace {

#define NCK(x)                                                                                     \
    do {                                                                                           \
        ncclResult_t r_ = (x);                                                                     \
        if (r_ != ncclSuccess) return fail(SOG_ENCCL, std::string(#x ": ") + nccl().GetErrorString(r_)); \
    } while (0)

// execute one exchange step: ex[i] belongs to local plan i
int run_exchange(sog_dist* d, std::vector<Exch>& ex) {
    if (d->loopback) {
        for (int r = 0; r < d->R; ++r) {
            std::vector<int> used(d->R, 0);
            for (const Msg& m : ex[r].send) {
                // the k-th message r -> m.peer matches the k-th receive posted at m.peer from r
                int k = used[m.peer]++, seen = 0;
                const Msg* dst = nullptr;
                for (const Msg& rv : ex[m.peer].recv)
                    if (rv.peer == r && seen++ == k) { dst = &rv; break; }
                if (!dst || dst->bytes < m.bytes) return fail(SOG_EINVAL, "loopback exchange: unmatched message");
                if (m.bytes) CK(cudaMemcpyAsync(dst->ptr, m.ptr, m.bytes, cudaMemcpyDeviceToDevice, d->stream));
            }
        }
        return SOG_OK;
    }
    NcclApi& api = nccl();
    NCK(api.GroupStart());
    for (const Msg& m : ex[0].send)
        if (m.bytes) NCK(api.Send(m.ptr, m.bytes, ncclUint8, m.peer, d->comm, d->stream));
    for (const Msg& m : ex[0].recv)
        if (m.bytes) NCK(api.Recv(m.ptr, m.bytes, ncclUint8, m.peer, d->comm, d->stream));
    NCK(api.GroupEnd());
    return SOG_OK;
}

__global__ void k_sum_into(double* __restrict__ a, const double* __restrict__ b, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] += b[i];
}

// sum of the long-range proxy grids over ranks (S8 is linear in the charges)
int run_allreduce(sog_dist* d, size_t n) {
    if (d->loopback) {
        double* a = d->pl[0]->lgrid;
        for (int r = 1; r < d->R; ++r)
            k_sum_into<<<(unsigned)((n + 255) / 256), 256, 0, d->stream>>>(a, d->pl[r]->lgrid, n);
        for (int r = 1; r < d->R; ++r)
            CK(cudaMemcpyAsync(d->pl[r]->lgrid, a, n * sizeof(double), cudaMemcpyDeviceToDevice, d->stream));
        CK(cudaGetLastError());
        return SOG_OK;
    }
    NCK(nccl().AllReduce(d->pl[0]->lgrid, d->pl[0]->lgrid, n, ncclFloat64, ncclSum, d->comm, d->stream));
    return SOG_OK;
}

// SOG_DEBUG_SYNC=1: synchronise after every x-slab step and report the first failing one
int dbg_sync(sog_dist* d, const char* what) {
    static const bool on = std::getenv("SOG_DEBUG_SYNC") != nullptr;
    if (!on) return SOG_OK;
    cudaError_t e = cudaStreamSynchronize(d->stream);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SOG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return SOG_OK;
}

void dmark(sog_dist* d, int k) {
    if (d->timing) cudaEventRecord(d->ev[k], d->stream);
}

int kyc_of(const sog_plan* pl, int s) {
    const int nyh = pl->p.Iy / 2 + 1;
    return std::max(0, std::min(pl->kc, nyh - s * pl->kc));
}

int dist_eval(sog_dist* d, const int64_t* nown, const double* const* xyz, const double* const* q, double* const* phi,
              double* const* force) {
    const int L = int(d->pl.size());
    const int R = d->R;
    std::vector<Exch> ex(L);
    int rc;
    auto left = [&](int r) { return (r + R - 1) % R; };
    auto right = [&](int r) { return (r + 1) % R; };
    dmark(d, 0);
    // ---- particle halos: select, agree on the input status, exchange counts, exchange particles ----
    // No rank returns before the agreement: a rank-local error (capacity, slab membership, invalid
    // input) is summed into every rank's status, so all ranks reject the evaluation together
    // instead of leaving the others blocked in a collective.
    for (int i = 0; i < L; ++i) {
        sog_plan* pl = d->pl[i];
        const Params& p = pl->p;
        const int64_t n64 = nown[i];
        const int host_err = (n64 < 0 || n64 > pl->nown_cap) ? 1 : 0;
        const int n = host_err ? 0 : int(n64);
        pl->Nown = n;
        cudaStream_t st = pl->stream;
        CK(cudaMemsetAsync(pl->dstat, 0, 8 * sizeof(double), st));
        CK(cudaMemsetAsync(pl->nsel, 0, 4 * sizeof(int), st));
        if (n > 0) {
            k_slab_flags<<<(n + 255) / 256, 256, 0, st>>>(xyz[i], q[i], n, p.Lx, p.Lz, pl->xs0, pl->xs1, pl->Hh, pl->own,
                                                         pl->fl, pl->fr, pl->dstat);
            if ((rc = lchk(launch_select_flagged(pl->own, pl->fl, pl->hsend, pl->nsel, n, pl->sel_tmp, pl->sel_bytes, st))) ||
                (rc = lchk(launch_select_flagged(pl->own, pl->fr, pl->hsend + pl->nown_cap, pl->nsel + 1, n, pl->sel_tmp,
                                                 pl->sel_bytes, st))))
                return rc;
            // across the periodic seam the halo copies carry the image shift of the receiver's frame
            if (pl->rank == 0)
                k_shift_x<<<(pl->halo_cap + 255) / 256, 256, 0, st>>>(pl->hsend, pl->nsel, p.Lx);
            if (pl->rank == R - 1)
                k_shift_x<<<(pl->halo_cap + 255) / 256, 256, 0, st>>>(pl->hsend + pl->nown_cap, pl->nsel + 1, -p.Lx);
        }
        k_halo_status<<<1, 1, 0, st>>>(pl->nsel, pl->halo_cap, host_err, pl->dstat);
        CK(cudaGetLastError());
        const int r = pl->rank;
        ex[i].send = {{left(r), pl->nsel, sizeof(int)}, {right(r), pl->nsel + 1, sizeof(int)}};
        ex[i].recv = {{right(r), pl->nsel + 2, sizeof(int)}, {left(r), pl->nsel + 3, sizeof(int)}};
    }
    if (d->loopback) {
        for (int i = 1; i < L; ++i)
            k_sum_into<<<1, 8, 0, d->stream>>>(d->pl[0]->dstat, d->pl[i]->dstat, 8);
        for (int i = 1; i < L; ++i)
            CK(cudaMemcpyAsync(d->pl[i]->dstat, d->pl[0]->dstat, 8 * sizeof(double), cudaMemcpyDeviceToDevice, d->stream));
    } else {
        NCK(nccl().AllReduce(d->pl[0]->dstat, d->pl[0]->dstat, 8, ncclFloat64, ncclSum, d->comm, d->stream));
    }
    if ((rc = run_exchange(d, ex))) return rc;
    for (int i = 0; i < L; ++i) {
        sog_plan* pl = d->pl[i];
        CK(cudaMemcpyAsync(pl->pin_i, pl->nsel, 4 * sizeof(int), cudaMemcpyDeviceToHost, pl->stream));
        CK(cudaMemcpyAsync(pl->pin_d, pl->dstat, 8 * sizeof(double), cudaMemcpyDeviceToHost, pl->stream));
    }
    CK(cudaStreamSynchronize(d->stream));
    {
        // identical on every rank (summed status)
        const double* sd = d->pl[0]->pin_d;
        if (sd[3] > 0) return fail(SOG_EINVAL, "x-slab capacity exceeded (own count or halo of clustered input) on some rank");
        if (sd[0] > 0) return fail(SOG_EINVAL, "own particle outside its rank's x slab");
        if (!(d->pl[0]->flags & SOG_NO_VALIDATE)) {
            if (sd[1] > 0) return fail(SOG_ENONFINITE, "non-finite position or charge");
            if (sd[2] > 0) return fail(SOG_EZRANGE, "z outside [-Lz/2, Lz/2]");
            if (std::fabs(sd[4]) > 1e-12 * sd[5]) return fail(SOG_ENONNEUTRAL, "system not charge neutral");
        } else if (sd[1] > 0 || sd[2] > 0) {
            return fail(SOG_EINVAL, "invalid particle (non-finite or z out of range)");
        }
    }
    for (int i = 0; i < L; ++i) {
        sog_plan* pl = d->pl[i];
        const int* c = pl->pin_i;
        const int r = pl->rank;
        ex[i].send = {{left(r), pl->hsend, sizeof(d4) * c[0]}, {right(r), pl->hsend + pl->nown_cap, sizeof(d4) * c[1]}};
        ex[i].recv = {{right(r), pl->hrecv + pl->halo_cap, sizeof(d4) * c[2]}, {left(r), pl->hrecv, sizeof(d4) * c[3]}};
    }
    if ((rc = run_exchange(d, ex))) return rc;
    dmark(d, 1);
    // ---- local particles: near field, mid spread, 2D FFTs, pack for the all-to-all ----
    for (int i = 0; i < L; ++i) {
        sog_plan* pl = d->pl[i];
        const Params& p = pl->p;
        cudaStream_t st = pl->stream;
        const int nl = pl->pin_i[3], nr = pl->pin_i[2], nloc = pl->Nown + nl + nr;
        if (nloc > 0)
            k_slab_local<<<(nloc + 255) / 256, 256, 0, st>>>(pl->own, pl->Nown, pl->hrecv, nl, pl->hrecv + pl->halo_cap, nr,
                                                            pl->lxyz, pl->lq);
        if ((rc = st_sort(pl, pl->lxyz, pl->lq, nloc)) || (rc = dbg_sync(d, "slab sort"))) return rc;
        // near field (own targets only) on the rank's side stream: it runs under the pencil
        // all-to-alls and the mid / long chain below; joined before the combine
        if (i == 0) dmark(d, 2);
        if (pl->side) {
            CK(cudaEventRecord(pl->ev_fork, st));
            CK(cudaStreamWaitEvent(pl->side, pl->ev_fork, 0));
            if (d->timing && i == 0) cudaEventRecord(d->nev[0], pl->side);
            pl->stream = pl->side;
            rc = st_near(pl);
            pl->stream = st;
            if (rc) return rc;
            if (d->timing && i == 0) cudaEventRecord(d->nev[1], pl->side);
            CK(cudaEventRecord(pl->ev_join, pl->side));
        } else if ((rc = st_near(pl))) {
            return rc;
        }
        if ((rc = dbg_sync(d, "slab near"))) return rc;
        if (!pl->has_mid) continue;
        if ((rc = st_mid_spread(pl)) || (rc = dbg_sync(d, "slab spread"))) return rc;
        CKF(cufftExecD2Z(pl->f2f, pl->mgrid + (size_t)pl->XO * p.Iy, pl->spec2));
        if ((rc = dbg_sync(d, "2D FFT"))) return rc;
        const size_t tot = (size_t)p.Izs * pl->Ixr * (p.Iy / 2 + 1);
        k_pack_fwd<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(pl->spec2, pl->sbuf, p.Izs, pl->Ixr, p.Iy / 2 + 1, pl->kc,
                                                                  R, pl->blk);
        CK(cudaGetLastError());
        ex[i].send.clear();
        ex[i].recv.clear();
        const int r = pl->rank;
        for (int s = 0; s < R; ++s) {
            ex[i].send.push_back({s, pl->sbuf + s * pl->blk, sizeof(cuDoubleComplex) * p.Izs * pl->Ixr * kyc_of(pl, s)});
            ex[i].recv.push_back({s, pl->rbuf + s * pl->blk, sizeof(cuDoubleComplex) * p.Izs * pl->Ixr * kyc_of(pl, r)});
        }
    }
    const bool has_mid = d->pl[0]->has_mid;
    dmark(d, 3);
    if (has_mid) {
        if ((rc = run_exchange(d, ex))) return rc;
        dmark(d, 4);
        // ---- x pencils: 1D FFT along x, S5 scaling, inverse, pack back ----
        for (int i = 0; i < L; ++i) {
            sog_plan* pl = d->pl[i];
            const Params& p = pl->p;
            cudaStream_t st = pl->stream;
            const int r = pl->rank, kyc = kyc_of(pl, r);
            const size_t tot = (size_t)p.Izs * kyc * p.Ix;
            if (tot) {
                k_unpack_fwd<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(pl->rbuf, pl->specx, p.Izs, pl->Ixr, p.Ix, kyc,
                                                                            pl->blk);
                if ((rc = dbg_sync(d, "unpack fwd"))) return rc;
                CKF(cufftExecZ2Z(pl->fxf, pl->specx, pl->specx, CUFFT_FORWARD));
                k_scale_pencil<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(pl->specx, p.Izs, kyc, p.Ix, r * pl->kc,
                                                                              p.Iy / 2 + 1, p.m + 1, pl->d_A, pl->d_Tx,
                                                                              pl->d_Ty, pl->d_Tz);
                CKF(cufftExecZ2Z(pl->fxf, pl->specx, pl->specx, CUFFT_INVERSE));
                k_pack_bwd<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(pl->specx, pl->sbuf, p.Izs, pl->Ixr, p.Ix, kyc,
                                                                          pl->blk);
                CK(cudaGetLastError());
            }
            ex[i].send.clear();
            ex[i].recv.clear();
            for (int s = 0; s < R; ++s) {
                ex[i].send.push_back({s, pl->sbuf + s * pl->blk, sizeof(cuDoubleComplex) * p.Izs * pl->Ixr * kyc});
                ex[i].recv.push_back({s, pl->rbuf + s * pl->blk, sizeof(cuDoubleComplex) * p.Izs * pl->Ixr * kyc_of(pl, s)});
            }
        }
        dmark(d, 5);
        if ((rc = run_exchange(d, ex))) return rc;
        dmark(d, 6);
        // ---- inverse 2D FFTs into the interior planes of Psi; edge planes for the neighbours ----
        for (int i = 0; i < L; ++i) {
            sog_plan* pl = d->pl[i];
            const Params& p = pl->p;
            cudaStream_t st = pl->stream;
            const size_t tot = (size_t)p.Izs * pl->Ixr * (p.Iy / 2 + 1);
            k_unpack_bwd<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(pl->rbuf, pl->spec2, p.Izs, pl->Ixr, p.Iy / 2 + 1,
                                                                        pl->kc, R, pl->blk);
            CKF(cufftExecZ2D(pl->f2i, pl->spec2, pl->mpsi + (size_t)pl->XO * p.Iy));
            if ((rc = dbg_sync(d, "inverse 2D FFT"))) return rc;
            const size_t hp = (size_t)p.Izs * pl->HP * p.Iy;
            k_planes_pack<<<(unsigned)((hp + 255) / 256), 256, 0, st>>>(pl->mpsi, pl->hsb, p.Izs, pl->Ixk, p.Iy, pl->XO,
                                                                        pl->HP);
            k_planes_pack<<<(unsigned)((hp + 255) / 256), 256, 0, st>>>(pl->mpsi, pl->hsb + hp, p.Izs, pl->Ixk, p.Iy,
                                                                        pl->XO + pl->Ixr - pl->HP, pl->HP);
            CK(cudaGetLastError());
            const int r = pl->rank;
            ex[i].send = {{left(r), pl->hsb, sizeof(double) * hp}, {right(r), pl->hsb + hp, sizeof(double) * hp}};
            ex[i].recv = {{right(r), pl->hrb + hp, sizeof(double) * hp}, {left(r), pl->hrb, sizeof(double) * hp}};
        }
        dmark(d, 7);
        if ((rc = run_exchange(d, ex))) return rc;
    }
    dmark(d, 8);
    // ---- halo planes in, mid gather, long spread of the own particles ----
    for (int i = 0; i < L; ++i) {
        sog_plan* pl = d->pl[i];
        const Params& p = pl->p;
        cudaStream_t st = pl->stream;
        if (pl->has_mid) {
            const size_t hp = (size_t)p.Izs * pl->HP * p.Iy;
            k_planes_unpack<<<(unsigned)((hp + 255) / 256), 256, 0, st>>>(pl->hrb, pl->mpsi, p.Izs, pl->Ixk, p.Iy,
                                                                          pl->XO - pl->HP, pl->HP);
            k_planes_unpack<<<(unsigned)((hp + 255) / 256), 256, 0, st>>>(pl->hrb + hp, pl->mpsi, p.Izs, pl->Ixk, p.Iy,
                                                                          pl->XO + pl->Ixr, pl->HP);
            CK(cudaGetLastError());
            if ((rc = dbg_sync(d, "psi halo"))) return rc;
            if (pl->Ncur && ((rc = st_mid_gather(pl)) || (rc = dbg_sync(d, "slab gather")))) return rc;
        } else if (pl->Ncur) {
            CK(cudaMemsetAsync(pl->o_mid, 0, sizeof(d4) * pl->Ncur, st));
        }
        if (pl->Ncur) {
            if ((rc = st_long_spread(pl))) return rc;
        } else {
            CK(cudaMemsetAsync(pl->lgrid, 0, sizeof(double) * p.Pc * p.Ilx * p.Ily, st));
        }
    }
    {
        const Params& p = d->pl[0]->p;
        dmark(d, 9);
        if ((rc = dbg_sync(d, "long spread")) || (rc = run_allreduce(d, (size_t)p.Pc * p.Ilx * p.Ily)) ||
            (rc = dbg_sync(d, "long allreduce")))
            return rc;
        dmark(d, 10);
    }
    // ---- long solve (redundant per rank: small grid), long gather, combine ----
    for (int i = 0; i < L; ++i) {
        sog_plan* pl = d->pl[i];
        if ((rc = st_long_solve(pl))) return rc;
        if (pl->side) CK(cudaStreamWaitEvent(pl->stream, pl->ev_join, 0));
        if (!pl->Ncur) continue;
        if ((rc = st_long_gather(pl))) return rc;
        k_combine_g<<<std::max(1, (pl->Nown + 255) / 256), 256, 0, pl->stream>>>(pl->o_near, pl->o_mid, pl->o_long, pl->pos_s,
                                                                    pl->iperm, pl->Nown, pl->selfc, phi[i], force[i],
                                                                    pl->epart);
        k_sum_partials<<<1, 1024, 0, pl->stream>>>(pl->epart, std::max(1, (pl->Nown + 255) / 256), pl->qsums + 2);
        CK(cudaGetLastError());
    }
    if (d->timing) {
        dmark(d, 11);
        CK(cudaStreamSynchronize(d->stream));
        // [0] halos, [1] sort, [2] spread + 2D FFT + pack, [3] all-to-all fwd, [4] x FFT + S5 + pack,
        // [5] all-to-all bwd, [6] inverse 2D FFT + plane pack, [7] Psi halo planes, [8] gather + long
        // spread, [9] long all-reduce, [10] long solve + gather + combine, [11] near field (side stream)
        const int pr[11][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 4}, {4, 5}, {5, 6}, {6, 7}, {7, 8}, {8, 9}, {9, 10}, {10, 11}};
        for (int k = 0; k < 11; ++k) {
            float ms = 0;
            if (!has_mid && k >= 3 && k <= 7) { d->ms[k] = 0; continue; }
            if (cudaEventElapsedTime(&ms, d->ev[pr[k][0]], d->ev[pr[k][1]]) != cudaSuccess) ms = 0;
            d->ms[k] = ms;
        }
        float ms = 0;
        if (cudaEventElapsedTime(&ms, d->nev[0], d->nev[1]) != cudaSuccess) ms = 0;
        d->ms[11] = ms;
        cudaGetLastError();
    }
    return SOG_OK;
}

// plan of one x-slab rank (slab geometry, capacities); p holds the global parameters
int dist_plan_setup(sog_plan* pl, int rank, int R, int64_t nown_max) {
    const Params& p = pl->p;
    pl->R = R;
    pl->rank = rank;
    pl->xs0 = -0.5 * p.Lx + p.Lx * rank / R;
    pl->xs1 = (rank == R - 1) ? 0.5 * p.Lx : -0.5 * p.Lx + p.Lx * (rank + 1) / R;
    const double hx = p.Lx / p.Ix;
    pl->Hh = std::max(p.rc, ((p.P - 1) / 2 + 1.5) * hx) * (1.0 + 1e-9);
    if (p.Lx / R < pl->Hh) return fail(SOG_EINVAL, "x slab narrower than the halo (r_c / window): use fewer ranks");
    if (p.Ix % R) return fail(SOG_EINVAL, "mid grid Ix must be a multiple of the rank count");
    if (p.Iy / 2 + 1 < R) return fail(SOG_EINVAL, "mid grid too small for the pencil transpose");
    const double frac = pl->Hh / (p.Lx / R);
    pl->halo_cap = int(std::min<double>(double(nown_max), std::ceil(double(nown_max) * frac * 1.5 + 1024.0)));
    pl->Ncap = int(nown_max + 2 * int64_t(pl->halo_cap));
    return setup(pl);
}

}  // namespace

extern "C" {

// One-process check of the NCCL plumbing (run-time symbol binding and call conventions) on the
// current device: a 1-rank communicator, grouped send/recv to itself and an all-reduce.
int sog_nccl_selftest(void) {
    if (!nccl().ok) return fail(SOG_ENCCL, "libnccl.so.2 not available");
    const NcclApi& api = nccl();
    ncclUniqueId id;
    NCK(api.GetUniqueId(&id));
    ncclComm_t comm;
    NCK(api.CommInitRank(&comm, 1, id, 0));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    const size_t n = 1 << 16;
    double *a = nullptr, *b = nullptr;
    CK(cudaMalloc(&a, n * sizeof(double)));
    CK(cudaMalloc(&b, n * sizeof(double)));
    std::vector<double> h(n), g(n);
    for (size_t i = 0; i < n; ++i) h[i] = 0.5 * double(i) - 7.0;
    CK(cudaMemcpy(a, h.data(), n * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemset(b, 0, n * sizeof(double)));
    NCK(api.GroupStart());
    NCK(api.Send(a, n * sizeof(double), ncclUint8, 0, comm, st));
    NCK(api.Recv(b, n * sizeof(double), ncclUint8, 0, comm, st));
    NCK(api.GroupEnd());
    NCK(api.AllReduce(b, b, n, ncclFloat64, ncclSum, comm, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(g.data(), b, n * sizeof(double), cudaMemcpyDeviceToHost));
    cudaFree(a);
    cudaFree(b);
    cudaStreamDestroy(st);
    api.CommDestroy(comm);
    for (size_t i = 0; i < n; ++i)
        if (g[i] != h[i]) return fail(SOG_ENCCL, "NCCL self-test: wrong data");
    return SOG_OK;
}

int sog_nccl_unique_id(void* id128) {
    if (!id128) return fail(SOG_EINVAL, "null argument");
    if (!nccl().ok) return fail(SOG_ENCCL, "libnccl.so.2 not available");
    ncclUniqueId id;
    NCK(nccl().GetUniqueId(&id));
    std::memcpy(id128, &id, sizeof(id) < 128 ? sizeof(id) : 128);
    return SOG_OK;
}

static sog_dist* dist_create(int64_t N_total, int64_t nown_max, double Lx, double Ly, double Lz, double tol,
                             const sog_plan_opts* o, int R, int first, int count, bool loopback, const void* id128) {
    if (R < 2 || nown_max < 1) { fail(SOG_EINVAL, "x-slab needs >= 2 ranks and a positive capacity"); return nullptr; }
    if (o && o->precision == 1) { fail(SOG_EINVAL, "x-slab ranks run in fp64"); return nullptr; }
    sog_dist* d = new sog_dist();
    d->R = R;
    d->loopback = loopback;
    d->stream = o ? (cudaStream_t)o->cuda_stream : nullptr;
    Params p;
    RuleKnobs k;
    if (make_params(p, k, N_total, Lx, Ly, Lz, tol, o) != SOG_OK) { delete d; return nullptr; }
    if (!(o && o->explicit_params) && p.m >= 0) {   // Ix a multiple of R (even, FFT friendly)
        long n = p.Ix;
        while (n % R || (n & 1) || !smooth7l(n)) ++n;
        p.Ix = int(n);
    }
    for (int r = first; r < first + count; ++r) {
        sog_plan* pl = new sog_plan();
        pl->p = p;
        pl->knobs = k;
        if (o) pl->flags = o->flags;
        d->pl.push_back(pl);
        int rc = dist_plan_setup(pl, r, R, nown_max);
        if (rc == SOG_OK) rc = set_stream(pl, d->stream);
        if (rc != SOG_OK) { std::string keep = g_err; sog_dist_destroy(d); g_err = keep; return nullptr; }
    }
    if (!loopback) {
        if (!nccl().ok) { fail(SOG_ENCCL, "libnccl.so.2 not available"); sog_dist_destroy(d); return nullptr; }
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof(id));
        ncclResult_t r = nccl().CommInitRank(&d->comm, R, id, first);
        if (r != ncclSuccess) {
            fail(SOG_ENCCL, std::string("ncclCommInitRank: ") + nccl().GetErrorString(r));
            sog_dist_destroy(d);
            return nullptr;
        }
    }
    return d;
}

sog_dist* sog_dist_create(int64_t N_total, int64_t nown_max, double Lx, double Ly, double Lz, double tol,
                          const sog_plan_opts* opts, int rank, int nranks, const void* nccl_id) {
    if (!nccl_id || rank < 0 || rank >= nranks) { fail(SOG_EINVAL, "bad rank / NCCL id"); return nullptr; }
    return dist_create(N_total, nown_max, Lx, Ly, Lz, tol, opts, nranks, rank, 1, false, nccl_id);
}

sog_dist* sog_dist_create_loopback(int64_t N_total, int64_t nown_max, double Lx, double Ly, double Lz, double tol,
                                   const sog_plan_opts* opts, int nranks) {
    return dist_create(N_total, nown_max, Lx, Ly, Lz, tol, opts, nranks, 0, nranks, true, nullptr);
}

int sog_dist_eval(sog_dist* d, const int64_t* n_own, const double* const* xyz, const double* const* q,
                  double* const* phi, double* const* force) {
    if (!d || !n_own || !xyz || !q || !phi || !force) return fail(SOG_EINVAL, "null argument");
    return dist_eval(d, n_own, xyz, q, phi, force);
}

int sog_dist_local_ranks(const sog_dist* d) { return d ? int(d->pl.size()) : fail(SOG_EINVAL, "null"); }

int sog_dist_set_flags(sog_dist* d, unsigned flags) {
    if (!d) return fail(SOG_EINVAL, "null");
    for (sog_plan* pl : d->pl) pl->flags = flags & ~SOG_TIMING;   // the plans' own stage events stay off
    const bool t = (flags & SOG_TIMING) != 0;
    if (t && !d->ev[0]) {
        for (auto& e : d->ev) CK(cudaEventCreate(&e));
        for (auto& e : d->nev) CK(cudaEventCreate(&e));
    }
    d->timing = t;
    return SOG_OK;
}

int sog_dist_get_timings(const sog_dist* d, double* ms, int n) {
    if (!d || !ms) return fail(SOG_EINVAL, "null argument");
    const int k = std::min(n, 12);
    for (int i = 0; i < k; ++i) ms[i] = d->ms[i];
    return k;
}

int sog_dist_describe(const sog_dist* d, char* buf, size_t len) {
    if (!d || d->pl.empty()) return fail(SOG_EINVAL, "null");
    const sog_plan* pl = d->pl[0];
    std::string s = describe(pl->p);
    char extra[512];
    std::snprintf(extra, sizeof extra, "ranks=%d\nslab_planes=%d\nhalo=%.17g\nhalo_capacity=%d\nlocal_capacity=%d\n",
                  d->R, pl->Ixr, pl->Hh, pl->halo_cap, pl->Ncap);
    s += extra;
    if (buf && len) {
        size_t n = std::min(len - 1, s.size());
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
    return int(s.size());
}

void sog_dist_destroy(sog_dist* d) {
    if (!d) return;
    for (auto& e : d->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : d->nev)
        if (e) cudaEventDestroy(e);
    if (d->comm && nccl().ok) nccl().CommDestroy(d->comm);
    for (sog_plan* pl : d->pl) free_plan(pl);
    delete d;
}

}  // extern "C"
