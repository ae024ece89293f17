/*
 * sog.h -- C ABI of the B200-native spectral sum-of-Gaussians (SOG) solver for
 * quasi-2D electrostatics (periodic in x,y, free in z), arXiv 2412.04595.
 *
 * Operation (section 2.1, Eq. eq::Phi): for N point charges q_i at
 * r_i in the box [-Lx/2,Lx/2) x [-Ly/2,Ly/2) x [-Lz/2,Lz/2], periodic in x,y,
 * charge neutral (sum q = 0), compute
 *     phi_i = sum_j sum'_{n in Z^2 x {0}} q_j / |r_ij + n o L|          (self excluded)
 *     F_i   = -q_i grad phi(r_i)
 * by the spectral SOG split (Eq. eq::SOGdecomp; Eq. eq::splitting):
 *     phi = Phi^N (near, cell list) + Phi^mid (Algorithm 1)
 *         + Phi^long (Algorithm 2 with two-sided Chebyshev proxies) - q_i sum_l w_l
 * to the requested tolerance `tol` (relative L-inf potential error).
 *
 * Conventions (all entry points):
 *   - Every function is thread-compatible, not thread-safe: one plan per host thread.
 *   - A plan is not reentrant; sog_eval calls on one plan are serialised on its stream.
 *   - Errors: functions return a negative sog_status (or NULL) and never throw; the
 *     message is available from sog_last_error() (thread-local, valid until the next
 *     call on that thread).  Outputs are unspecified after an error.
 *   - Device pointers are CUDA device pointers on the plan's device; host pointers are
 *     ordinary (pageable or pinned) host memory.  The caller owns every buffer it
 *     passes; the plan owns all of its workspace.
 *   - Layouts: xyz is N x 3 row-major (x0,y0,z0,x1,...) fp64; q, phi are N fp64;
 *     force is N x 3 row-major fp64; all in the caller's particle order.
 */
#ifndef SOG_H
#define SOG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sog_plan sog_plan; /* opaque; owns all device workspace and cuFFT plans */

typedef enum {
    SOG_OK = 0,
    SOG_EINVAL = -1,        /* bad argument (N, box, tol, pointer, option)                 */
    SOG_ENONNEUTRAL = -2,   /* |sum q| > 1e-12 sum|q|                           */
    SOG_EZRANGE = -3,       /* some z outside the closed interval [-Lz/2, Lz/2] */
    SOG_ENONFINITE = -4,    /* non-finite position or charge                                */
    SOG_EINFEASIBLE = -5,   /* tol outside [2e-14, 1e-1] (Table 1 force floor)       */
    SOG_ECUDA = -6,         /* CUDA runtime or cuFFT failure                                 */
    SOG_ENCCL = -7,         /* NCCL unavailable or an NCCL call failed (x-slab ranks)        */
    SOG_ENOMEM = -8         /* device allocation failed                                      */
} sog_status;

/* flags for sog_plan_opts.flags / sog_set_flags */
#define SOG_NO_VALIDATE 1u  /* skip the validation readback (the only host sync in sog_eval) */

/*
 * Optional plan overrides.  Zero-initialise and set what you need.
 *   explicit_params = 0: parameters come from the plan rules R1-R9, with
 *                        rc_factor / eta overriding R2 / R4 when > 0.
 *   explicit_params = 1: every parameter below is used verbatim (e.g. a plan chosen by
 *                        the CPU oracle); the library only validates them.
 * Field meanings follow PAPER.md: row = Table 1 row 0..5 (b, r0, omega);
 * rc = cutoff r_c (sigma = rc/r0); M, m = last Gaussian and last mid-range
 * Gaussian; Ix,Iy = mid grid in x,y; Iz = interior z count (h_z = Lz/Iz);
 * Izs = extended z grid I_z^* (P:580); P, S = window support (odd) and shape;
 * Ilx, Ily = long grid; Pl, Sl = long window; Pc = Chebyshev proxy layers.
 */
typedef struct {
    double rc_factor;
    double eta;
    int explicit_params;
    int row;
    double rc;
    int M, m;
    int Ix, Iy, Iz, Izs, P;
    double S;
    int Ilx, Ily, Pl;
    double Sl;
    int Pc;
    void* cuda_stream;      /* cudaStream_t to enqueue on; NULL = the legacy default stream */
    unsigned flags;         /* SOG_NO_VALIDATE ... */
    int precision;          /* 0: fp64 (default); 1: fp32 mode (S2-S12 in fp32 storage and
                               arithmetic, positions/outputs fp64 at the boundary; tol >= 1e-5,
                               whole-box plans with small long grids; parity bar 1e-5) */
    int window;             /* 0: Gaussian window (Eq. eq::GS; default); 1: Kaiser-Bessel window,
                               2: "exponential of semicircle" (ES) window (R6-ES; transform by
                               quadrature) (Remark rmk::PWindow) evaluated as per-stencil-point polynomials
                               of degree nu (mid) / nul (long) from Chebyshev interpolation; with
                               window = 1, S and Sl are the KB shapes beta and the support half-width is
                               P h / 2 (R6-KB) */
    int nu, nul;            /* KB polynomial degrees for explicit_params (0: P + 3 / Pl + 3); <= P + 3 */
    int long_method;        /* 0: Alg. 2, window + 2D FFT per proxy layer (default); 1: Alg. 3 without
                               FFT (App. B): direct type-1/type-2 Fourier sums over
                               kx = 2 pi n / Lx, |n| <= Kx, ky = 2 pi n / Ly, 0 <= n <= Ky (DESIGN.md
                               R8-D), for boxes with few modes (cubic / tall: c2, c4, c5); single-GPU */
    int Kx, Ky;             /* direct long range mode bounds for explicit_params */
    int optimize;           /* 1: R20, eq::optimiz with B200-calibrated costs: the
                               plan of least predicted time over r_c factors {2.75 .. 3.75} x eta
                               {0.2 .. 0.5} (rc_factor / eta ignored) */
    double b;               /* > 1: a general SOG base b in (1, 2] instead of the Table-1 row (NEXT #4):
                               (r0, omega) from the C^1 continuity solve (Eq. eq::2.35z;
                               DESIGN.md R22), e.g. Table 4's b = 1.17.  With explicit_params,
                               b > 1 takes (b, r0, omega) verbatim from the three fields and row is ignored */
    double r0, omega;
} sog_plan_opts;

/* Build a plan for N particles in the box (Lx,Ly,Lz) at tolerance tol on the current
 * CUDA device.  Chooses parameters (R1-R9), precomputes tables (SOG weights, near-kernel
 * polynomial table, window/deconvolution tables, long-range kernel matrices K_ab),
 * allocates workspace and cuFFT plans.  Returns NULL on error (see sog_last_error). */
sog_plan* sog_plan_create(int64_t N, double Lx, double Ly, double Lz, double tol);
sog_plan* sog_plan_create_ex(int64_t N, double Lx, double Ly, double Lz, double tol,
                             const sog_plan_opts* opts);

/* Run only the parameter rules R1-R9 (no device work, no GPU needed) and write the
 * key=value description of the plan sog_plan_create_ex would build into buf (same format
 * as sog_plan_describe).  Returns the number of bytes needed, or a negative sog_status. */
int sog_plan_choose(int64_t N, double Lx, double Ly, double Lz, double tol, const sog_plan_opts* opts,
                    char* buf, size_t len);

/* Evaluate potentials and forces.  xyz, q: device inputs (caller order, see layouts);
 * phi, force: device outputs (either may be NULL to skip).  Enqueued on the plan's stream;
 * unless SOG_NO_VALIDATE is set, synchronises once to read the validation flags and
 * returns SOG_EZRANGE / SOG_ENONFINITE / SOG_ENONNEUTRAL on invalid input. */
int sog_eval(sog_plan* p, const double* xyz, const double* q, double* phi, double* force);

/* Same as sog_eval with HOST buffers: copies inputs host->device, evaluates, copies
 * results back, and returns after the results are in host memory. */
int sog_eval_host(sog_plan* p, const double* xyz, const double* q, double* phi, double* force);

/* Pipelined host-buffer evaluation of independent systems back to back (same plan, same N): the
 * copy of the inputs is enqueued on a copy-in stream, the evaluation on the plan's stream once they
 * have arrived, and the copy of phi / force (either may be NULL) on a copy-out stream once it has
 * finished; the call returns without waiting.  Two device staging sets alternate, so the copies of
 * one call overlap the evaluation of the previous one (PCIe copies under the compute).  Host
 * buffers must stay valid, and inputs unmodified, until sog_host_wait(); pinned host memory makes
 * the copies asynchronous.  No CUDA graph (the staging pointers alternate) and no per-call host
 * synchronisation: input validation (unless SOG_NO_VALIDATE) is accumulated on the device and
 * reported by sog_host_wait.  Single-GPU plans only (SOG_EINVAL for an x-slab rank's plan). */
int sog_eval_host_async(sog_plan* p, const double* xyz, const double* q, double* phi, double* force);
/* Wait for every pending sog_eval_host_async call (results in host memory); returns
 * SOG_ENONFINITE / SOG_EZRANGE / SOG_ENONNEUTRAL if any of them had invalid input. */
int sog_host_wait(sog_plan* p);

/* Per-component outputs for parity testing: out is a DEVICE buffer of 3*N*4 doubles laid
 * out [component][i][4] with component 0 = near (Phi^N, grad Phi^N), 1 = mid, 2 = long,
 * and the 4 values (phi, dphi/dx, dphi/dy, dphi/dz), caller order, self term NOT removed. */
int sog_eval_components(sog_plan* p, const double* xyz, const double* q, double* out);

/* Intermediate grids for stage parity (device buffer `out` of `len` doubles):
 *   stage 1: mid spread grid S        [Izs][Ix][Iy]  (z slowest)  (Alg. 1 step 1)
 *   stage 2: mid scaled field Psi     [Izs][Ix][Iy]               (Alg. 1 step 4)
 *   stage 3: long proxy grids S_b     [Pc][Ilx][Ily]           (Alg. 2 step 1)
 *   stage 4: long scaled fields Psi_a [Pc][Ilx][Ily]           (Alg. 2 step 4) */
int sog_debug_stage(sog_plan* p, int stage, const double* xyz, const double* q, double* out, size_t len);

/* Potential energy U = 1/2 sum q_i phi_i of the last sog_eval; host scalar. */
int sog_last_energy(sog_plan* p, double* U);

void sog_plan_destroy(sog_plan* p); /* NULL-safe */

/* Thread-local message for the last failing call on this thread ("" if none). */
const char* sog_last_error(void);

/* key=value lines describing the chosen plan (parameters, grid sizes, memory).
 * Returns the number of bytes needed (excluding NUL); writes at most len bytes. */
int sog_plan_describe(const sog_plan* p, char* buf, size_t len);

/* Per-stage device times (ms) of the last sog_eval with SOG_TIMING set via sog_set_flags:
 * [0] sort, [1] near, [2] mid spread, [3] mid FFT fwd, [4] mid scale, [5] mid FFT inv,
 * [6] mid gather, [7] long spread, [8] long FFT+scale+IFFT, [9] long gather, [10] combine.
 * Returns the number of entries written (<= n). */
#define SOG_TIMING 2u
/* Replay the evaluation as one CUDA graph: captured at the first sog_eval and re-captured when the
 * (xyz, q, phi, force) pointers change; stage timings are not collected in this mode. */
#define SOG_GRAPH 4u
int sog_get_timings(const sog_plan* p, double* ms, int n);

int sog_set_flags(sog_plan* p, unsigned flags);
int sog_set_stream(sog_plan* p, void* cuda_stream);

/* Number of kernel launches sog_eval enqueues (for the bench's gpu_launches). */
int sog_launches_per_eval(const sog_plan* p);

/* ---------------------------------------------------------------------------------------
 * x-slab decomposition over R ranks (north_star "partitioned across the 8
 * GPUs of one box by x-slabs").  Rank r owns the particles with canonical x in
 *   [-Lx/2 + r Lx/R, -Lx/2 + (r+1) Lx/R)     (the last slab is closed at +Lx/2 by the wrap)
 * and the mid-grid planes [r Ix/R, (r+1) Ix/R).  One evaluation exchanges: particle halos
 * (particles within H = max(r_c, (p + 1.5) h_x) of a slab edge) with the two neighbours; the
 * pencil all-to-all of the distributed 3D FFT (2D (z,y) FFTs per x plane, ky chunks, 1D FFT
 * along x, and back); the Psi edge planes needed by the gather; and a sum of the long-range
 * proxy grids (all-reduce).  The result equals the single-GPU evaluation up to rounding.
 * The plan parameters are those of the global system of N_total particles (Ix rounded up to
 * a multiple of R when the rules choose it); n_own_max bounds every rank's own count.
 * --------------------------------------------------------------------------------------- */
typedef struct sog_dist sog_dist;

/* One-process check of the library's NCCL plumbing (libnccl.so.2 resolved at run time): a 1-rank
 * communicator on the current device, grouped send/recv to itself and an all-reduce; SOG_OK or
 * SOG_ENCCL with the reason in sog_last_error(). */
int sog_nccl_selftest(void);

/* 128 bytes of ncclUniqueId for sog_dist_create (call on one rank, broadcast to the others,
 * e.g. with torch.distributed).  SOG_ENCCL if libnccl.so.2 cannot be loaded. */
int sog_nccl_unique_id(void* id128);

/* One process per GPU (NCCL over NVLink): this process is `rank` of `nranks`.  Every rank
 * calls it collectively with the same N_total, n_own_max, box, tol, opts and id. */
sog_dist* sog_dist_create(int64_t N_total, int64_t n_own_max, double Lx, double Ly, double Lz, double tol,
                          const sog_plan_opts* opts, int rank, int nranks, const void* nccl_id);

/* All nranks ranks as virtual ranks of this process on the current device (exchanges are
 * device-to-device copies): the same decomposition, for testing on one GPU. */
sog_dist* sog_dist_create_loopback(int64_t N_total, int64_t n_own_max, double Lx, double Ly, double Lz, double tol,
                                   const sog_plan_opts* opts, int nranks);

/* Evaluate.  Arrays of length sog_dist_local_ranks(d) (1 for NCCL ranks, nranks for loopback);
 * entry i: n_own[i] particles of local rank i, device arrays xyz (n x 3), q (n), outputs phi
 * (n), force (n x 3) in that rank's own particle order.  Collective: every rank calls it.
 * SOG_EINVAL if a particle is outside its rank's slab or a halo exceeds its capacity. */
int sog_dist_eval(sog_dist* d, const int64_t* n_own, const double* const* xyz, const double* const* q,
                  double* const* phi, double* const* force);

int sog_dist_local_ranks(const sog_dist* d);
/* SOG_NO_VALIDATE / SOG_TIMING for every local rank.  With SOG_TIMING each evaluation synchronises at
 * its end and records per-phase device times of local rank 0 (CUDA events on the ranks' stream; the
 * collective phases include waiting for the slowest peer):
 *   [0] particle halos (select, status agreement, exchanges), [1] sort, [2] mid spread + 2D FFTs + pack,
 *   [3] all-to-all forward, [4] x FFT + S5 + pack, [5] all-to-all back, [6] inverse 2D FFTs + plane
 *   pack, [7] Psi halo planes, [8] mid gather + long spread, [9] long-grid all-reduce,
 *   [10] long solve + gather + combine, [11] near field (own targets, on the side stream). */
int sog_dist_set_flags(sog_dist* d, unsigned flags);
int sog_dist_get_timings(const sog_dist* d, double* ms, int n);   /* writes min(n, 12) values, returns it */
int sog_dist_describe(const sog_dist* d, char* buf, size_t len);   /* plan + slab key=value lines */
void sog_dist_destroy(sog_dist* d);                                 /* NULL-safe */

#ifdef __cplusplus
}
#endif
#endif /* SOG_H */
