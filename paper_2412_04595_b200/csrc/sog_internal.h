// Internal definitions shared by the host runtime (plan.cpp, sog_api.cu) and kernels.
// Nothing here is visible through the C ABI (include/sog.h).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace sog {

// Plan parameters (rules R1-R9).  Names follow PAPER.md notation.
struct Params {
    int64_t N = 0;
    double Lx = 0, Ly = 0, Lz = 0, tol = 0;
    int row = -1;                  // Table 1 row
    double b = 0, r0 = 0, omega = 0;
    double rc = 0, sigma = 0;      // r_c, sigma = r_c / r0
    int M = 0, m = -1;             // last Gaussian, last mid-range Gaussian
    // mid-range grid / window
    int Ix = 0, Iy = 0, Iz = 0, Izs = 0, P = 0;
    double S = 0;
    // long-range grid / window / proxies
    int Ilx = 0, Ily = 0, Pl = 0;
    double Sl = 0;
    int Pc = 0;
    // window (R6 / R6-KB / R6-ES): 0 = Gaussian (Eq. eq::GS), 1 = Kaiser-Bessel, 2 = exponential of
    // semicircle, the last two as per-stencil-point polynomials of degree nu (mid) / nul (long); S, Sl
    // hold beta for KB / ES
    int window = 0, nu = 0, nul = 0;
    // long range: 0 = Alg. 2 (window + 2D FFT), 1 = Alg. 3 without FFT (App. B): direct Fourier
    // sums over kx = 2 pi n / Lx, |n| <= Kx, ky = 2 pi n / Ly, 0 <= n <= Ky (R8-D)
    int long_method = 0, Kx = 0, Ky = 0;
    // derived
    double hx() const { return Lx / Ix; }
    double hy() const { return Ly / Iy; }
    double hz() const { return Lz / Iz; }
    double Lzs() const { return hz() * Izs; }
    double hlx() const { return Lx / Ilx; }
    double hly() const { return Ly / Ily; }
};

struct RuleKnobs {
    double rc_factor = 3.25;  // R2 (GPU-tuned: bench sweep)
    double eta = 0.3;         // R4
    double kappa = 1.15;      // R5/R8
    double win_c = 0.3;       // R6
    double pad_c = 10.0;      // R7
    double cheb_c = 0.1;      // R9
    double fft_cost = 30.0;   // R6 cost model (grid point vs stencil point, B200-measured)
    double long_fft_cost = 30.0;
    double kb_beta = 2.2;     // R6-KB: beta = kb_beta * P
    double es_beta = 2.3;     // R6-ES: beta = es_beta * P
    int kb_nu_extra = 3;      // R6-KB: nu = P + kb_nu_extra
    double kb_rate_a = 0.4, kb_rate_b = 0.92;   // R6-KB: window error ~ 10^(a - b P)
};

// plan.cpp
bool choose_params(Params& p, const RuleKnobs& k, std::string& err);   // rules R1-R9 (p.b > 1, p.row < 0: general b)
// NEXT #4: C^1 solve for a general b (binary128): the smallest root r0 whose error terms are <= tol
bool c1_solve(double b, double tol, double& r0, double& omega);
// R20: eq::optimiz with B200-calibrated costs: the least predicted time over r_c factor x eta grids
bool choose_params_opt(Params& p, const RuleKnobs& k, std::string& err);
double plan_cost(const Params& p);
bool validate_params(const Params& p, std::string& err);
void sog_weights(const Params& p, std::vector<double>& w, std::vector<double>& s);
double erfcinv_host(double y);

// Near-field kernel table: F(u) and dF/du, u = r^2, piecewise Taylor polynomials (R16),
// NEAR_D = polynomial degree (the kernels are instantiated for it).
constexpr int NEAR_D = 10;
struct NearTable {
    int K = 0, D = 0;          // pieces, degree
    double du = 0, inv_du = 0; // piece width in u
    std::vector<double> cF;    // K x (D+1)   F coefficients (Horner, highest last)
    std::vector<double> cdF;   // K x (D+1)   dF/du coefficients (degree D-1, last = 0)
    double max_rel_err = 0;    // validated at plan time against the direct sum
};
bool build_near_table(const Params& p, NearTable& t, std::string& err);
// R16-G: one polynomial of degree D <= NEAR_POLY_DMAX in t = 2u/r_c^2 - 1 for F(u) on [0, r_c^2]
// (monomial coefficients c[0..D]); false when no supported degree meets the 1e-15 validation
constexpr int NEAR_POLY_DMAX = 56;
struct NearPoly {
    int D = 0;
    double inv_h = 0;            // dt/du
    double c[NEAR_POLY_DMAX + 1] = {};
    double err_F = 0, err_dF = 0;
};
bool build_near_poly(const Params& p, NearPoly& t);

// Mid-range scaling tables: mult(k) = sum_{l<=m} A_l Tx[l][ix] Ty[l][iy] Tz[l][iz] (R12);
// Ty covers the half axis iy < Iy/2+1, Tx and Tz the full axes (fftfreq order).
void build_mid_tables(const Params& p, std::vector<double>& A, std::vector<double>& Tx,
                      std::vector<double>& Ty, std::vector<double>& Tz);
// Long-range kernel matrices per half mode (mode = ix*(Ily/2+1)+iy), in the Chebyshev T
// basis: K~[mode][m][n] = sum_ab C[a][m] K_ab C[b][n], K_ab from R9/R10.
void build_long_kernel(const Params& p, std::vector<double>& K);
// R8-D direct long range: K~ = C^T K C per mode, modes ordered (ix = 0..2Kx, iy = 0..Ky), K with
// pi / (Lx Ly) and no window (App. B, Eq. eq::gridnonfft P:1243)
void build_long_kernel_direct(const Params& p, std::vector<double>& K);
// R6-KB: monomial coefficients c[n * P + j] (n = 0..nu) in u = x/h + I/2 - g0 of the degree-nu
// Chebyshev interpolant of W_KB((j - p - u) h), H = P h / 2 (Remark rmk::PWindow)
void build_kb_poly(int P, double beta, int nu, std::vector<double>& c, int window = 1);   // 1 KB, 2 ES
// Fourier transform of the KB window of half-width H (sinh / sin branches)
double kb_hat(double k, double H, double beta);
double poly_window_hat(int window, double k, double H, double beta);   // KB (1) closed form, ES (2) quadrature
// Chebyshev -> Lagrange coefficient matrix C[b][n]: L_b(x) = sum_n C[b][n] T_n(x).
void build_cheb_matrix(int Pc, std::vector<double>& C);
// Tn[a][m] = T_m(x_a) at the first-kind nodes x_a = cos((a+1/2) pi / Pc).
void build_cheb_nodes(int Pc, std::vector<double>& Tn);

std::string describe(const Params& p);

}  // namespace sog
