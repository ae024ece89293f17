// Host-side plan construction: parameter rules R1-R9 and precomputed tables.
// Independent of the CPU oracle (oracle/plan.py); tests/test_plan_parity.py compares them.
#include <algorithm>
#include <quadmath.h>
#include <cmath>
#include <cstdio>
#include <map>
#include <sstream>
#include <thread>

#include "sog_internal.h"

namespace sog {

namespace {

// Table 1: b, r0, omega, force error.
struct Row { double b, r0, omega, ferr; };
const Row kTable1[6] = {
    {2.0, 1.9892536839080267, 0.9944464927622323, 9.93e-3},
    {1.62976708826776469, 2.7520026668023417, 1.0078069793438068, 6.21e-4},
    {1.48783512395703226, 3.7554672283554990, 0.9919117057598183, 7.98e-5},
    {1.32070036405934420, 4.3914554711638349, 1.0018891411481198, 5.76e-7},
    {1.21812525709410644, 5.6355288151271085, 1.0009014615603334, 5.14e-10},
    {1.14878150173321925, 7.2956245490719404, 1.0000368348358225, 1.98e-14},
};
constexpr double kTolMin = 2e-14, kTolMax = 1e-1;
constexpr double kPi = 3.14159265358979323846;

bool smooth7(long n) {
    for (long f : {2L, 3L, 5L, 7L})
        while (n % f == 0) n /= f;
    return n == 1;
}
// smallest even n' >= n with prime factors in {2,3,5,7} (cuFFT-friendly sizes)
long friendly_even(long n) {
    if (n < 2) n = 2;
    if (n & 1) ++n;
    while (!smooth7(n)) n += 2;
    return n;
}

// R7-Z: padded z size, the smallest even 2^a 3^b or 2^a 5^b >= n (a radix set of the fused z pass)
// unless that exceeds 4096, else friendly_even (oracle/plan.py z_friendly_even)
long z_friendly_even(long n) {
    const long base = friendly_even(n);
    if (base > 4096) return base;
    for (long m = base;; m += 2) {
        long r = m;
        while (r % 2 == 0) r /= 2;
        long r3 = r, r5 = r;
        while (r3 % 3 == 0) r3 /= 3;
        while (r5 % 5 == 0) r5 /= 5;
        if (r3 == 1 || r5 == 1) return m;
    }
}

// Largest h keeping the Thm 4.2 aliasing term exp(-pi^2 mu (P-1)^2/(4 s^2 S)) <= eps,
// mu = s^2 - H^2/S, H = (P-1) h / 2.  0 if infeasible.
double h_alias(int P, double S, double eps, double s) {
    double a = P - 1.0;
    double rhs = 1.0 - 4.0 * S * std::log(1.0 / eps) / (kPi * kPi * a * a);
    if (rhs <= 0.0) return 0.0;
    return 2.0 * s * std::sqrt(S) / a * std::sqrt(rhs);
}

template <class Cost>
bool choose_window(double s, double eps_w, double tol, double kappa, Cost cost, int& Pout,
                   double& Sout, double& hout) {
    double S = erfcinv_host(eps_w);
    S = S * S;
    double h_nyq = kPi * s / (2.0 * kappa * std::sqrt(std::log(1.0 / tol)));
    bool found = false;
    double best = 0;
    for (int P = 3; P < 61; P += 2) {
        double ha = h_alias(P, S, eps_w, s);
        if (ha <= 0.0) continue;
        double h = std::min(h_nyq, ha);
        double c = cost(P, h);
        if (!found || c < best) { best = c; Pout = P; hout = h; found = true; }
    }
    Sout = S;
    return found;
}

// R6-KB: support P = smallest odd >= 5 with 10^(a - b P) <= eps_w, beta = kb_beta P, the mesh at
// the Nyquist bound (the window does not constrain h), nu = P + kb_nu_extra
void choose_window_kb(double s, double eps_w, double tol, const RuleKnobs& k, int window, int& Pout, double& beta,
                      double& h, int& nu) {
    int P = 5;
    while (std::pow(10.0, k.kb_rate_a - k.kb_rate_b * P) > eps_w) P += 2;
    Pout = P;
    beta = (window == 2 ? k.es_beta : k.kb_beta) * P;   // R6-ES / R6-KB
    h = kPi * s / (2.0 * k.kappa * std::sqrt(std::log(1.0 / tol)));
    nu = P + k.kb_nu_extra;
}

// Chebyshev T_n(x), n < P
void cheb_T(double x, int P, double* T) {
    T[0] = 1.0;
    if (P > 1) T[1] = x;
    for (int n = 1; n + 1 < P; ++n) T[n + 1] = 2.0 * x * T[n] - T[n - 1];
}

// Lagrange basis at first-kind Chebyshev nodes via discrete orthogonality:
// L_a(x) = (1/P) [1 + 2 sum_{n>=1} T_n(x_a) T_n(x)]   (App. A.2)
void lagrange(double x, int P, const std::vector<double>& Tnodes, double* L) {
    std::vector<double> T(P);
    cheb_T(x, P, T.data());
    for (int a = 0; a < P; ++a) {
        double acc = 0.0;
        for (int n = 1; n < P; ++n) acc += Tnodes[a * P + n] * T[n];
        L[a] = (1.0 + 2.0 * acc) / P;
    }
}

std::vector<double> node_T(int P) {
    std::vector<double> Tn(P * P);
    for (int a = 0; a < P; ++a) {
        double xa = std::cos((a + 0.5) * kPi / P);
        cheb_T(xa, P, &Tn[a * P]);
    }
    return Tn;
}

// R9: max error of sum_ab L_a(z) g(z_a - z_b) L_b(z'), g(d) = exp(-d^2/s^2), 65x65 test grid
double cheb_two_sided_error(int P, double Lz, double s) {
    const int nt = 65;
    std::vector<double> Tn = node_T(P), za(P), G(P * P), Lt(nt * P);
    for (int a = 0; a < P; ++a) za[a] = 0.5 * Lz * std::cos((a + 0.5) * kPi / P);
    for (int a = 0; a < P; ++a)
        for (int b = 0; b < P; ++b) {
            double d = (za[a] - za[b]) / s;
            G[a * P + b] = std::exp(-d * d);
        }
    for (int i = 0; i < nt; ++i) lagrange(-1.0 + 2.0 * i / (nt - 1), P, Tn, &Lt[i * P]);
    std::vector<double> LG(nt * P, 0.0);
    for (int i = 0; i < nt; ++i)
        for (int b = 0; b < P; ++b) {
            double acc = 0;
            for (int a = 0; a < P; ++a) acc += Lt[i * P + a] * G[a * P + b];
            LG[i * P + b] = acc;
        }
    double err = 0;
    for (int i = 0; i < nt; ++i)
        for (int j = 0; j < nt; ++j) {
            double acc = 0;
            for (int b = 0; b < P; ++b) acc += LG[i * P + b] * Lt[j * P + b];
            double zi = 0.5 * Lz * (-1.0 + 2.0 * i / (nt - 1));
            double zj = 0.5 * Lz * (-1.0 + 2.0 * j / (nt - 1));
            double d = (zi - zj) / s;
            err = std::max(err, std::fabs(acc - std::exp(-d * d)));
        }
    return err;
}

}  // namespace

// erfc^{-1}(y) for y in (0, 1]: Newton on erfc from an asymptotic start.
double erfcinv_host(double y) {
    if (y >= 1.0) return 0.0;
    double t = std::sqrt(-std::log(y));
    double x = t - (std::log(t) + 0.5 * std::log(kPi)) / (2.0 * t);   // asymptotic start
    if (!(x > 0)) x = 0.5;
    for (int it = 0; it < 100; ++it) {
        double f = std::erfc(x) - y;
        double df = -2.0 / std::sqrt(kPi) * std::exp(-x * x);
        double dx = f / df;
        x -= dx;
        if (std::fabs(dx) < 1e-17 * std::fabs(x)) break;
    }
    return x;
}

void sog_weights(const Params& p, std::vector<double>& w, std::vector<double>& s) {
    // w_l = (pi/2)^{-1/2} b^{-l} sigma^{-1} log b, s_l = sqrt(2) b^l sigma; omega on w_0
    w.resize(p.M + 1);
    s.resize(p.M + 1);
    const double c = std::pow(kPi / 2.0, -0.5) * std::log(p.b) / p.sigma;
    for (int l = 0; l <= p.M; ++l) {
        w[l] = c * std::pow(p.b, -double(l));
        s[l] = std::sqrt(2.0) * std::pow(p.b, double(l)) * p.sigma;
    }
    w[0] *= p.omega;
}

// NEXT #4: the C^1 continuity solve for a general b (Eq. eq::2.35z), sigma = 1:
//   r0 F(r0) = 1 and r0^2 F'(r0) = -1, F(r) = omega w_0 e^{-r^2/2} + G(r), G = sum_{l>=1} w_l e^{-r^2/s_l^2}.
// Eliminating omega: h(r) = 1 - r^2 + r^3 G(r) + r^2 G'(r) = 0, omega = (1/r - G(r)) e^{r^2/2} / w_0.
// The smallest root whose eq::convrate near-field / omega terms are below tol (reading R22).
// Sign changes of h on a 0.02 grid in r in [1, 20] (double), each bracket refined by bisection in
// binary128 (libquadmath): for b -> 1 |h| between roots is ~1e-13, so double cannot locate r0 and
// omega's e^{r^2/2} amplifies rounding.
static void c1_G(__float128 r, __float128 b, __float128 c, __float128& g, __float128& dg) {
    g = 0; dg = 0;
    for (int l = 1;; ++l) {
        const __float128 s2 = 2 * powq(b, 2 * l), w = c * powq(b, -l);
        const __float128 e = w * expq(-r * r / s2);
        g += e;
        dg += e * (-2 * r / s2);
        if (w < (__float128)1e-40) break;
    }
}
static __float128 c1_h(__float128 r, __float128 b, __float128 c) {
    __float128 g, dg;
    c1_G(r, b, c, g, dg);
    return 1 - r * r + r * r * r * g + r * r * dg;
}
bool c1_solve(double bd, double tol, double& r0, double& omega) {
    if (!(bd > 1.0 && bd <= 2.0)) return false;
    const __float128 pi = 4 * atanq((__float128)1), b = bd, c = sqrtq(2 / pi) * logq(b);
    // grid scan in double
    const double cd = std::sqrt(2.0 / kPi) * std::log(bd);
    const int nl = int(130.0 / std::log(bd)) + 2;
    auto hd = [&](double r) {
        double g = 0, dg = 0;
        for (int l = 1; l <= nl; ++l) {
            const double s2 = 2.0 * std::pow(bd, 2.0 * l), e = cd * std::pow(bd, -double(l)) * std::exp(-r * r / s2);
            g += e;
            dg += e * (-2.0 * r / s2);
        }
        return 1 - r * r + r * r * r * g + r * r * dg;
    };
    double rp = 1.0, hp = hd(rp);
    for (int i = 1; i <= 950; ++i) {
        const double rn = 1.0 + 0.02 * i, hn = hd(rn);
        if (hp * hn < 0) {
            __float128 lo = rp, hi = rn, hlo = c1_h(lo, b, c);
            if (hlo * c1_h(hi, b, c) <= 0) {
                for (int it = 0; it < 64; ++it) {
                    const __float128 mid = (lo + hi) / 2, hm = c1_h(mid, b, c);
                    if (hlo * hm <= 0) hi = mid;
                    else { lo = mid; hlo = hm; }
                }
                const __float128 r = (lo + hi) / 2;
                __float128 g, dg;
                c1_G(r, b, c, g, dg);
                const __float128 om = (1 / r - g) * expq(r * r / 2) / c;
                const __float128 s0 = sqrtq((__float128)2), sm1 = s0 / b, wm1 = c * b;
                const __float128 e1 = expq(-r * r / (sm1 * sm1)), e0 = expq(-r * r / (s0 * s0));
                const __float128 te = fabsq(wm1 * e1) + fabsq((om - 1) * c * e0);
                const __float128 tf = fabsq(wm1 / (sm1 * sm1) * e1) + fabsq((om - 1) * c / (s0 * s0) * e0);
                if ((te > tf ? te : tf) <= (__float128)tol) {
                    r0 = double(r);
                    omega = double(om);
                    return true;
                }
            }
        }
        rp = rn;
        hp = hn;
    }
    return false;
}

bool choose_params(Params& p, const RuleKnobs& k, std::string& err) {
    if (!(p.tol >= kTolMin && p.tol <= kTolMax)) { err = "tol outside [2e-14, 1e-1]"; return false; }
    if (p.b > 1.0 && p.row < 0) {
        // NEXT #4: a caller-chosen b, (r0, omega) from the C^1 solve
        if (!c1_solve(p.b, p.tol, p.r0, p.omega)) { err = "no C^1 root for this b below tol"; return false; }
    } else {
        // R1: coarsest Table-1 row whose force error <= tol
        int row = -1;
        for (int r = 0; r < 6; ++r) if (kTable1[r].ferr <= p.tol) { row = r; break; }
        if (row < 0) { err = "infeasible tolerance"; return false; }
        p.row = row;
        p.b = kTable1[row].b; p.r0 = kTable1[row].r0; p.omega = kTable1[row].omega;
    }
    // R2
    const double rho = double(p.N) / (p.Lx * p.Ly * p.Lz);
    p.rc = std::min(k.rc_factor * std::pow(rho, -1.0 / 3.0), 0.5 * std::min(p.Lx, p.Ly));
    p.sigma = p.rc / p.r0;
    const double s0 = std::sqrt(2.0) * p.sigma;
    const double Lmax = std::max(p.Lx, std::max(p.Ly, p.Lz));
    // R3: smallest M with s_M >= Lmax / tol
    const double target = Lmax / p.tol;
    int M = std::max(0, int(std::ceil(std::log(target / s0) / std::log(p.b))));
    while (s0 * std::pow(p.b, M) < target) ++M;
    while (M > 0 && s0 * std::pow(p.b, M - 1) >= target) --M;
    p.M = M;
    // R4: m = max{l : s_l <= eta Lz}
    int m = -1;
    for (int l = 0; l <= M; ++l) if (s0 * std::pow(p.b, l) <= k.eta * p.Lz) m = l;
    p.m = std::min(m, M - 1);
    const double eps_w = k.win_c * p.tol;
    const double N = double(p.N);
    if (p.m >= 0) {
        const double sm = s0 * std::pow(p.b, p.m);
        const double padimg = sm * std::sqrt(std::log(k.pad_c / p.tol));
        auto cost_mid = [&](int P, double h) {
            double pad = std::max(2.0 * ((P - 1) * h / 2.0 + h), padimg);
            return double(P) * P * P + k.fft_cost * (p.Lx * p.Ly * (p.Lz + pad)) / (N * h * h * h);
        };
        double h;
        if (p.window == 1 || p.window == 2)
            choose_window_kb(s0, eps_w, p.tol, k, p.window, p.P, p.S, h, p.nu);
        else if (!choose_window(s0, eps_w, p.tol, k.kappa, cost_mid, p.P, p.S, h)) { err = "no mid window"; return false; }
        p.Ix = friendly_even(long(std::ceil(p.Lx / h)));
        p.Iy = friendly_even(long(std::ceil(p.Ly / h)));
        p.Iz = std::max(1L, long(std::ceil(p.Lz / h)));
        const double hz = p.hz();
        const double Hz = (p.P - 1) * hz / 2.0;
        const double pad = std::max(2.0 * (Hz + hz), padimg);          // R7
        p.Izs = z_friendly_even(long(std::ceil((p.Lz + pad) / hz)));   // R7, R7-Z
    }
    const double sl = s0 * std::pow(p.b, p.m + 1);
    auto cost_long = [&](int P, double h) {
        return double(P) * P + k.long_fft_cost * (p.Lx * p.Ly) / (N * h * h);
    };
    double hl;
    if (p.window == 1 || p.window == 2)
        choose_window_kb(sl, eps_w, p.tol, k, p.window, p.Pl, p.Sl, hl, p.nul);
    else if (!choose_window(sl, eps_w, p.tol, k.kappa, cost_long, p.Pl, p.Sl, hl)) { err = "no long window"; return false; }
    p.Ilx = std::max(friendly_even(long(std::ceil(p.Lx / hl))), friendly_even(p.Pl));
    p.Ily = std::max(friendly_even(long(std::ceil(p.Ly / hl))), friendly_even(p.Pl));
    // R9
    p.Pc = 0;
    for (int P = 2; P < 65; ++P)
        if (cheb_two_sided_error(P, p.Lz, sl) <= std::max(k.cheb_c * p.tol, 5e-14)) { p.Pc = P; break; }
    if (!p.Pc) { err = "Chebyshev order > 64 needed"; return false; }
    if (p.long_method == 1) {   // R8-D: the narrowest long-range Gaussian's spectrum below tol^(kappa^2)
        const double kcut = 2.0 * k.kappa * std::sqrt(std::log(1.0 / p.tol)) / sl;
        p.Kx = int(std::ceil(kcut * p.Lx / (2.0 * kPi)));
        p.Ky = int(std::ceil(kcut * p.Ly / (2.0 * kPi)));
    }
    return true;
}

double plan_cost(const Params& p) {
    // seconds: near per pair, mid stencil point, mid grid point, long particle x Pl^2 x Pc, long grid point x layer
    const double c_pair = 1.35e-11, c_st = 1.39e-12, c_grid = 2.6e-11, c_long = 4.33e-13, c_lgrid = 3.6e-11;
    const double N = double(p.N), rho = N / (p.Lx * p.Ly * p.Lz);
    const double vol = std::min(4.0 / 3.0 * kPi * p.rc * p.rc * p.rc, kPi * p.rc * p.rc * p.Lz);
    double t = c_pair * N * rho * vol;
    if (p.m >= 0) t += c_st * N * double(p.P) * p.P * p.P + c_grid * double(p.Ix) * p.Iy * p.Izs;
    t += c_long * N * double(p.Pl) * p.Pl * p.Pc + c_lgrid * double(p.Ilx) * p.Ily * p.Pc;
    return t;
}

bool choose_params_opt(Params& p, const RuleKnobs& k, std::string& err) {
    static const double rcs[] = {2.75, 3.0, 3.25, 3.5, 3.75};
    static const double etas[] = {0.2, 0.25, 0.3, 0.35, 0.4, 0.5};
    Params best;
    double bc = -1.0;
    for (double f : rcs)
        for (double e : etas) {
            Params q = p;
            RuleKnobs kk = k;
            kk.rc_factor = f;
            kk.eta = e;
            std::string er;
            if (!choose_params(q, kk, er)) { err = er; continue; }
            if (q.Pc > 32 || q.Pl > 25 || (q.m >= 0 && q.P > 25)) continue;   // GPU compiled range
            const double c = plan_cost(q);
            if (bc < 0.0 || c < bc) { best = q; bc = c; }
        }
    if (bc < 0.0) return false;
    p = best;
    return true;
}

bool validate_params(const Params& p, std::string& err) {
    auto bad = [&](const char* m) { err = m; return false; };
    if (p.N < 1 || p.N > (int64_t(1) << 31) - 1) return bad("N out of range [1, 2^31)");
    if (!(p.Lx > 0 && p.Ly > 0 && p.Lz > 0) || !std::isfinite(p.Lx + p.Ly + p.Lz)) return bad("invalid box");
    if (p.row > 5 || (p.row < 0 && !(p.b > 1.0 && p.b <= 2.0 && p.r0 > 0))) return bad("row must be 0..5 (or a general b)");
    if (!(p.rc > 0) || p.rc > 0.5 * std::min(p.Lx, p.Ly) * (1 + 1e-15)) return bad("r_c must be in (0, min(Lx,Ly)/2]");
    if (p.M < 1 || p.M > 4000) return bad("M out of range");
    if (p.m < -1 || p.m >= p.M) return bad("m must be in [-1, M-1]");
    if (p.m >= 0) {
        if (p.Ix < 2 || p.Iy < 2 || p.Iz < 1 || p.Izs < 2 || (p.Izs & 1)) return bad("bad mid grid");
        if (p.P < 5 || p.P > 25 || !(p.P & 1)) return bad("mid window support must be odd in [5,25]");
        if (!(p.S > 0)) return bad("bad mid window shape");
        if (p.Ix < p.P || p.Iy < p.P) return bad("mid grid smaller than the window support");
        // R7: the z stencil must not leave the extended grid
        double hz = p.hz();
        if (p.Izs * hz < p.Lz + (p.P - 1) * hz + 2.0 * hz * (1 - 1e-12)) return bad("Izs too small for the z stencil (R7)");
    }
    if (p.Ilx < 2 || p.Ily < 2 || (p.Ily & 1)) return bad("bad long grid (Ily must be even)");
    if (p.Pl < 5 || p.Pl > 25 || !(p.Pl & 1)) return bad("long window support must be odd in [5,25]");
    if (!(p.Sl > 0)) return bad("bad long window shape");
    if (p.Ilx < p.Pl || p.Ily < p.Pl) return bad("long grid smaller than the window support");
    if (p.Pc < 2 || p.Pc > 32) return bad("Pc must be in [2,32]");
    if (p.window < 0 || p.window > 2) return bad("window must be 0 (Gaussian), 1 (Kaiser-Bessel) or 2 (ES)");
    if (p.long_method != 0 && p.long_method != 1) return bad("long_method must be 0 (FFT) or 1 (direct)");
    if (p.long_method == 1 && (p.Kx < 0 || p.Ky < 0 || p.Kx > 63 || p.Ky > 63))
        return bad("direct long range: mode bounds Kx, Ky must be in [0, 63]");
    if (p.window == 1 || p.window == 2) {
        if ((p.m >= 0 && p.P > 17) || p.Pl > 17) return bad("KB window support must be <= 17");
        if (p.m >= 0 && (p.nu < 2 || p.nu > p.P + 3)) return bad("KB mid polynomial degree nu must be in [2, P+3]");
        if (p.nul < 2 || p.nul > p.Pl + 3) return bad("KB long polynomial degree nul must be in [2, Pl+3]");
        // deconvolution divides by the window transform: keep every grid mode inside its
        // positive (sinh) branch, k_max H = pi P / 2 < beta
        if (p.m >= 0 && !(p.S > 0.5 * kPi * p.P)) return bad("KB mid shape beta must exceed pi P / 2");
        if (!(p.Sl > 0.5 * kPi * p.Pl)) return bad("KB long shape beta must exceed pi Pl / 2");
    }
    return true;
}

// R16-G (k_near4): ONE polynomial for F(u) on [0, r_c^2], so every lane evaluates the same
// coefficients (kernel-parameter / constant-bank operands, no table lookups).  The degree-D
// Chebyshev interpolant of F in t = 2u/r_c^2 - 1 (long double, D + 1 first-kind nodes) is
// re-expanded in powers of t (long double) and rounded once; F and dF/dt come from one joint
// Horner.  The monomial form keeps sum |c_n| = F(0) (an alternating series for a sum of decaying
// exponentials), so Horner loses nothing.  D = the smallest supported degree whose F and F'
// errors on a dense sample are <= 1e-15 of F(0) and of max |F'| (validated, long double).
bool build_near_poly(const Params& p, NearPoly& t) {
    std::vector<double> w, s;
    sog_weights(p, w, s);
    const long double umax = (long double)p.rc * p.rc, h = umax / 2;
    auto Fl = [&](long double u, long double* dF) {
        long double F = 0, d = 0;
        for (int l = 0; l <= p.M; ++l) {
            const long double a = 1.0L / ((long double)s[l] * s[l]);
            const long double e = (long double)w[l] * expl(-u * a);
            F += e;
            d -= e * a;
        }
        if (dF) *dF = d;
        return F;
    };
    long double dF0 = 0;
    const long double F0 = Fl(0, &dF0);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int D : {16, 20, 24, 28, 32, 40, 48, 56}) {
        if (D > NEAR_POLY_DMAX) break;
        const int n1 = D + 1;
        std::vector<long double> f(n1), a(n1), mono(n1 + 1, 0.0L), Tm(n1 + 1), Tc(n1 + 1), Tn(n1 + 1);
        for (int i = 0; i < n1; ++i) f[i] = Fl(h * (1.0L + cosl((i + 0.5L) * pi / n1)), nullptr);
        for (int n = 0; n < n1; ++n) {
            long double acc = 0;
            for (int i = 0; i < n1; ++i) acc += f[i] * cosl(n * (i + 0.5L) * pi / n1);
            a[n] = acc * (n == 0 ? 1.0L : 2.0L) / n1;
        }
        std::fill(Tm.begin(), Tm.end(), 0.0L);
        std::fill(Tc.begin(), Tc.end(), 0.0L);
        Tm[0] = 1.0L;
        Tc[1] = 1.0L;
        mono[0] += a[0];
        mono[1] += a[1];
        for (int n = 2; n < n1; ++n) {
            for (int e = 0; e <= n1; ++e) Tn[e] = (e > 0 ? 2.0L * Tc[e - 1] : 0.0L) - Tm[e];
            for (int e = 0; e <= n1; ++e) mono[e] += a[n] * Tn[e];
            Tm.swap(Tc);
            Tc.swap(Tn);
        }
        NearPoly q;
        q.D = D;
        q.inv_h = double(1.0L / h);
        long double cond = 0;
        for (int n = 0; n <= D; ++n) {
            q.c[n] = double(mono[n]);
            cond += fabsl(mono[n]);
        }
        // validation in the arithmetic the kernel uses (double Horner) against the long-double sum
        double eF = 0, edF = 0, mdF = 0;
        for (int i = 0; i <= 4000; ++i) {
            const double u = double(umax) * i / 4000.0;
            const double tt = u * q.inv_h - 1.0;
            double F = q.c[D], dF = 0;
            for (int n = D - 1; n >= 0; --n) {
                dF = dF * tt + F;
                F = F * tt + q.c[n];
            }
            long double dFe = 0;
            const long double Fe = Fl(u, &dFe);
            eF = std::max(eF, double(fabsl((long double)F - Fe)));
            edF = std::max(edF, double(fabsl((long double)(dF * q.inv_h) - dFe)));
            mdF = std::max(mdF, double(fabsl(dFe)));
        }
        q.err_F = eF / double(F0);
        q.err_dF = edF / mdF;
        if (q.err_F <= 1e-15 && q.err_dF <= 1e-15 && cond <= 2.0L * F0) {
            t = q;
            return true;
        }
    }
    return false;
}

bool build_near_table(const Params& p, NearTable& t, std::string& err) {
    // F(u) = sum_l w_l exp(-u/s_l^2) (Eq. eq::SOGField) as piecewise Taylor polynomials
    // in u = r^2 on [0, r_c^2]; pieces narrow enough that du/(2 s_0^2) <= 1/4 (R16).
    std::vector<double> w, s;
    sog_weights(p, w, s);
    const double s0sq = s[0] * s[0];
    const double umax = p.rc * p.rc;
    // pieces with du / (2 s_0^2) <= 1/8 and degree NEAR_D = 10: Taylor remainders at |d| <= du/2
    // of the narrowest Gaussian ~1e-17 (F), ~3e-16 (F'); the table stays small (shared memory)
    t.K = std::max(1, int(std::ceil(4.0 * umax / s0sq)));
    t.D = NEAR_D;
    t.du = umax / t.K;
    t.inv_du = t.K / umax;
    const int D = t.D;
    t.cF.assign(size_t(t.K) * (D + 1), 0.0);
    t.cdF.assign(size_t(t.K) * (D + 1), 0.0);
    std::vector<long double> c(D + 2);
    for (int k = 0; k < t.K; ++k) {
        long double uk = (k + 0.5L) * (long double)t.du;
        for (int n = 0; n <= D + 1; ++n) c[n] = 0.0L;
        for (int l = 0; l <= p.M; ++l) {
            long double a = -1.0L / ((long double)s[l] * s[l]);
            long double term = (long double)w[l] * expl(a * uk);
            for (int n = 0; n <= D + 1; ++n) {
                c[n] += term;
                term *= a / (n + 1);
            }
        }
        for (int n = 0; n <= D; ++n) t.cF[size_t(k) * (D + 1) + n] = double(c[n]);
        for (int n = 0; n < D; ++n) t.cdF[size_t(k) * (D + 1) + n] = double((n + 1) * c[n + 1]);
    }
    // validate against the direct sum on a dense sample
    double maxrel = 0;
    for (int i = 0; i <= 4000; ++i) {
        double u = umax * i / 4000.0;
        int k = std::min(t.K - 1, int(u * t.inv_du));
        double d = u - (k + 0.5) * t.du;
        double F = t.cF[size_t(k) * (D + 1) + D], dF = 0;
        for (int n = D - 1; n >= 0; --n) {
            dF = dF * d + F;
            F = F * d + t.cF[size_t(k) * (D + 1) + n];
        }
        long double Fe = 0, dFe = 0;
        for (int l = 0; l <= p.M; ++l) {
            long double e = (long double)w[l] * expl(-(long double)u / ((long double)s[l] * s[l]));
            Fe += e;
            dFe += -e / ((long double)s[l] * s[l]);
        }
        maxrel = std::max(maxrel, double(std::fabs((long double)F - Fe) / Fe));
        maxrel = std::max(maxrel, double(std::fabs((long double)dF - dFe) / std::fabs(dFe)));
    }
    t.max_rel_err = maxrel;
    if (maxrel > 1e-14) {
        char buf[128];
        std::snprintf(buf, sizeof buf, "near table validation failed: rel err %.3e", maxrel);
        err = buf;
        return false;
    }
    return true;
}

void build_mid_tables(const Params& p, std::vector<double>& A, std::vector<double>& Tx,
                      std::vector<double>& Ty, std::vector<double>& Tz) {
    // mult(k) = pi^{3/2} sum_{l<=m} w_l s_l^3 exp(-s_l^2 |k|^2/4) / (W_x W_y W_z)^2 with
    // W_hat(k) = sqrt(pi/S) H exp(-k^2 H^2/(4S)), k_d = 2 pi n / L_d (L_z -> L_z^*).
    // Per axis and per l:  T[l][i] = (S / (pi H^2)) exp(-k^2 (s_l^2/4 - H^2/(2S)))  (one exp:
    // no overflow of the separate Gaussian / deconvolution factors).
    std::vector<double> w, s;
    sog_weights(p, w, s);
    const int L = p.m + 1;
    A.resize(L);
    // cuFFT's inverse is unnormalised: the 1/(Ix Iy Izs) of ifftn is folded into A_l (R12).
    const double inv_n = 1.0 / (double(p.Ix) * p.Iy * p.Izs);
    for (int l = 0; l < L; ++l) A[l] = std::pow(kPi, 1.5) * w[l] * s[l] * s[l] * s[l] * inv_n;
    auto axis = [&](int I, double Lper, double h, bool half, std::vector<double>& T) {
        int n = half ? I / 2 + 1 : I;
        T.resize(size_t(L) * n);
        double H = (p.window != 0 ? p.P : p.P - 1) * h / 2.0;
        for (int l = 0; l < L; ++l)
            for (int i = 0; i < n; ++i) {
                int f = (half || i < (I + 1) / 2) ? i : i - I;   // numpy fftfreq ordering
                double kk = 2.0 * kPi * f / Lper;
                if (p.window != 0) {   // R6-KB / R6-ES: exp(-k^2 s_l^2/4) / W(k)^2
                    const double wh = poly_window_hat(p.window, kk, H, p.S);
                    T[size_t(l) * n + i] = std::exp(-kk * kk * s[l] * s[l] / 4.0) / (wh * wh);
                    continue;
                }
                double e = kk * kk * (s[l] * s[l] / 4.0 - H * H / (2.0 * p.S));
                T[size_t(l) * n + i] = p.S / (kPi * H * H) * std::exp(-e);
            }
    };
    // spectrum layout [Izs][Ix][Iy/2+1]: y is the half (real-to-complex) axis
    axis(p.Ix, p.Lx, p.hx(), false, Tx);
    axis(p.Iy, p.Ly, p.hy(), true, Ty);
    axis(p.Izs, p.Lzs(), p.hz(), false, Tz);
}

// K_ab(kdot) accumulated in long double: pi sum_{l>m} w_l s_l^2 exp(-s_l^2 k^2/4) E_l(z_a - z_b) without the
// window / normalisation factors (R9, R10).  The T-basis transform K~ = C^T K C below concentrates the
// smooth K into low orders; double rounding of K_ab would leave ~1e-15 absolute noise in every K~
// entry, which the gather's T'_n (~n^2) amplifies in the forces, so the whole chain is long double
// and K~ is rounded once.
static const long double kPiL = 3.141592653589793238462643383279502884L;
static void cheb_matrix_l(int P, std::vector<long double>& C) {   // L_b(x) = sum_n C[b][n] T_n(x)
    C.resize(size_t(P) * P);
    for (int b = 0; b < P; ++b)
        for (int n = 0; n < P; ++n)
            C[size_t(b) * P + n] = (n == 0 ? 1.0L : 2.0L * cosl(n * (b + 0.5L) * kPiL / P)) / P;
}
static void cheb_transform(int P, const std::vector<long double>& Kl, const std::vector<long double>& C, double* out) {
    std::vector<long double> KC(size_t(P) * P, 0.0L);
    for (int a = 0; a < P; ++a)
        for (int n = 0; n < P; ++n) {
            long double t = 0.0L;
            for (int b = 0; b < P; ++b) t += Kl[size_t(a) * P + b] * C[size_t(b) * P + n];
            KC[size_t(a) * P + n] = t;
        }
    for (int m = 0; m < P; ++m)
        for (int n = 0; n < P; ++n) {
            long double t = 0.0L;
            for (int a = 0; a < P; ++a) t += C[size_t(a) * P + m] * KC[size_t(a) * P + n];
            out[size_t(m) * P + n] = double(t);
        }
}

// Gaussian part of K~ (T basis, no window / normalisation factor) for every distinct |kdot|^2 of the
// mode set: K depends on kdot only through |kdot|^2 (E_l(d) is k-independent), so wide grids (the
// confined s1: 3840 x 1921 modes, ~1.4e6 distinct |k|^2) are built once per value, on all host threads.
static void long_kernel_unique(const Params& p, const std::vector<long double>& k2u, std::vector<double>& Ku) {
    std::vector<double> w, s;
    sog_weights(p, w, s);
    const int P = p.Pc, L = p.M - p.m;
    std::vector<long double> Cl, zal(P), E(size_t(L) * P * P), E0(size_t(L) * P * P);
    cheb_matrix_l(P, Cl);
    for (int a = 0; a < P; ++a) zal[a] = 0.5L * p.Lz * cosl((a + 0.5L) * kPiL / P);
    for (int l = 0; l < L; ++l) {
        const long double ss = (long double)s[p.m + 1 + l] * s[p.m + 1 + l];
        for (int a = 0; a < P; ++a)
            for (int b = 0; b < P; ++b) {
                const long double d2 = (zal[a] - zal[b]) * (zal[a] - zal[b]);
                E[(size_t(l) * P + a) * P + b] = expl(-d2 / ss);
                E0[(size_t(l) * P + a) * P + b] = expm1l(-d2 / ss);            // R10 at kdot = 0
            }
    }
    Ku.assign(k2u.size() * P * P, 0.0);
    const size_t nu = k2u.size();
    unsigned nth = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    if (nu < 64) nth = 1;
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nth; ++t)
        th.emplace_back([&, t]() {
            std::vector<long double> Kl(size_t(P) * P);
            for (size_t u = t; u < nu; u += nth) {
                const long double k2 = k2u[u];
                std::fill(Kl.begin(), Kl.end(), 0.0L);
                for (int l = 0; l < L; ++l) {
                    const long double ss = (long double)s[p.m + 1 + l] * s[p.m + 1 + l];
                    const long double g = ss * k2 / 4.0L;
                    // s_l grows with l: once exp(-g) < 1e-323 every later term rounds to 0 in the double K~
                    if (k2 != 0.0L && g > 745.0L) break;
                    const long double f = (long double)w[p.m + 1 + l] * ss * (k2 == 0.0L ? 1.0L : expl(-g));
                    const long double* El = (k2 == 0.0L ? E0.data() : E.data()) + size_t(l) * P * P;
                    for (int ab = 0; ab < P * P; ++ab) Kl[ab] += f * El[ab];
                }
                cheb_transform(P, Kl, Cl, &Ku[u * P * P]);
            }
        });
    for (auto& x : th) x.join();
}

void build_long_kernel(const Params& p, std::vector<double>& K) {
    // K_ab(kdot) = pi sum_{l=m+1}^{M} w_l s_l^2 exp(-s_l^2 |kdot|^2/4) E_l(z_a - z_b) / (W_x W_y)^2,
    // E_l(d) = exp(-d^2/s_l^2) for kdot != 0 and expm1(-d^2/s_l^2) at kdot = 0 (R10).
    const int P = p.Pc, nx = p.Ilx, ny = p.Ily / 2 + 1;
    const int Pw = p.window != 0 ? p.Pl : p.Pl - 1;   // support width in mesh steps (R6 / R6-KB)
    const double Hx = Pw * p.hlx() / 2.0, Hy = Pw * p.hly() / 2.0;
    // distinct |kdot|^2 (integer key (fx^2, fy^2) scaled by the box; one key per value when Lx == Ly)
    const bool sq = p.Lx == p.Ly;
    std::map<std::pair<long long, long long>, size_t> key;
    std::vector<long double> k2u;
    std::vector<size_t> mode_u(size_t(nx) * ny);
    for (int ix = 0; ix < nx; ++ix) {
        const long long fx = ix < (nx + 1) / 2 ? ix : ix - nx;
        for (int iy = 0; iy < ny; ++iy) {
            const long long a2 = fx * fx, b2 = (long long)iy * iy;
            const std::pair<long long, long long> kk = sq ? std::make_pair(a2 + b2, 0LL) : std::make_pair(a2, b2);
            auto it = key.find(kk);
            if (it == key.end()) {
                it = key.emplace(kk, k2u.size()).first;
                const long double kx = 2.0L * kPiL * fx / p.Lx, ky = 2.0L * kPiL * iy / p.Ly;
                k2u.push_back(kx * kx + ky * ky);
            }
            mode_u[size_t(ix) * ny + iy] = it->second;
        }
    }
    std::vector<double> Ku;
    long_kernel_unique(p, k2u, Ku);
    K.assign(size_t(nx) * ny * P * P, 0.0);
    for (int ix = 0; ix < nx; ++ix) {
        const int fx = ix < (nx + 1) / 2 ? ix : ix - nx;
        const double kx = 2.0 * kPi * fx / p.Lx;
        for (int iy = 0; iy < ny; ++iy) {
            const double ky = 2.0 * kPi * iy / p.Ly;
            // 1 / (W_x W_y)^2
            double Wx = p.window != 0 ? poly_window_hat(p.window, kx, Hx, p.Sl)
                                      : std::sqrt(kPi / p.Sl) * Hx * std::exp(-kx * kx * Hx * Hx / (4.0 * p.Sl));
            double Wy = p.window != 0 ? poly_window_hat(p.window, ky, Hy, p.Sl)
                                      : std::sqrt(kPi / p.Sl) * Hy * std::exp(-ky * ky * Hy * Hy / (4.0 * p.Sl));
            // pi and the 1/(Ilx Ily) of the (unnormalised) cuFFT inverse are folded in here (R12)
            const double dec = kPi / (Wx * Wx * Wy * Wy) / (double(p.Ilx) * p.Ily);
            const double* src = &Ku[mode_u[size_t(ix) * ny + iy] * P * P];
            double* dst = &K[(size_t(ix) * ny + iy) * P * P];
            for (int e = 0; e < P * P; ++e) dst[e] = src[e] * dec;
        }
    }
}

void build_cheb_nodes(int Pc, std::vector<double>& Tn) { Tn = node_T(Pc); }

void build_long_kernel_direct(const Params& p, std::vector<double>& K) {
    // K_ab(kdot) = pi/(Lx Ly) sum_{l>m} w_l s_l^2 exp(-s_l^2 |kdot|^2/4) E_l(z_a - z_b), E_l =
    // exp(-d^2/s_l^2) (expm1 at kdot = 0, R10), then K~ = C^T K C (T basis, as build_long_kernel)
    const int P = p.Pc, nx = 2 * p.Kx + 1, ny = p.Ky + 1;
    std::vector<long double> k2u;
    for (int ix = 0; ix < nx; ++ix)
        for (int iy = 0; iy < ny; ++iy) {
            const long double kx = 2.0L * kPiL * (ix - p.Kx) / p.Lx, ky = 2.0L * kPiL * iy / p.Ly;
            k2u.push_back(kx * kx + ky * ky);
        }
    std::vector<double> Ku;
    long_kernel_unique(p, k2u, Ku);
    K.assign(Ku.size(), 0.0);
    const double f = kPi / (p.Lx * p.Ly);
    for (size_t e = 0; e < Ku.size(); ++e) K[e] = Ku[e] * f;
}


double kb_hat(double k, double H, double beta) {
    // int_{-H}^{H} I0(beta sqrt(1 - (x/H)^2)) / I0(beta) e^{-ikx} dx
    //   = 2H sinh(sqrt(beta^2 - (kH)^2)) / (I0(beta) sqrt(beta^2 - (kH)^2))   (sin form past kH = beta)
    const double a = beta * beta - (k * H) * (k * H);
    const double r = std::sqrt(std::fabs(a));
    const double f = r == 0.0 ? 1.0 : (a > 0.0 ? std::sinh(r) / r : std::sin(r) / r);
    return 2.0 * H * f / std::cyl_bessel_i(0.0, beta);
}

// ES transform H int_{-pi/2}^{pi/2} exp(beta (cos t - 1)) cos(k H sin t) cos t dt (x = H sin t; the
// integrand is entire in t): 192-point Gauss-Legendre, nodes by Newton on P_n in long double
double es_hat(double k, double H, double beta) {
    static std::vector<long double> xs, ws;
    if (xs.empty()) {
        const int n = 192;
        const long double pi = 3.141592653589793238462643383279502884L;
        xs.resize(n);
        ws.resize(n);
        for (int i = 0; i < n; ++i) {
            long double x = std::cos(pi * (i + 0.75L) / (n + 0.5L)), dp = 0;
            for (int it = 0; it < 100; ++it) {
                long double p0 = 1, p1 = x;
                for (int m = 2; m <= n; ++m) {
                    const long double p2 = ((2 * m - 1) * x * p1 - (m - 1) * p0) / m;
                    p0 = p1;
                    p1 = p2;
                }
                dp = n * (x * p1 - p0) / (x * x - 1);
                const long double dx = p1 / dp;
                x -= dx;
                if (std::fabs(dx) < 1e-19L) break;
            }
            xs[i] = x;
            ws[i] = 2.0L / ((1 - x * x) * dp * dp);
        }
    }
    const long double half = 1.5707963267948966192313216916397514L;
    long double acc = 0;
    for (size_t i = 0; i < xs.size(); ++i) {
        const long double t = half * xs[i];
        acc += ws[i] * std::exp((long double)beta * (std::cos(t) - 1)) * std::cos((long double)k * H * std::sin(t)) * std::cos(t);
    }
    return double((long double)H * half * acc);
}

double poly_window_hat(int window, double k, double H, double beta) {
    return window == 2 ? es_hat(k, H, beta) : kb_hat(k, H, beta);
}

void build_kb_poly(int P, double beta, int nu, std::vector<double>& c, int window) {
    // Chebyshev interpolation in t = 2u at the nu+1 first-kind points (discrete orthogonality),
    // then the series sum_n a_n T_n(2u) re-expanded in powers of u, all in long double.
    const int p = (P - 1) / 2, n1 = nu + 1;
    const long double half_w = 0.5L * P, pi = 3.141592653589793238462643383279502884L;
    const long double i0b = std::cyl_bessel_il(0.0L, (long double)beta);
    c.assign(size_t(n1) * P, 0.0);
    std::vector<long double> f(n1), a(n1), Tm(n1), Tc(n1), Tn(n1), mono(n1);
    for (int j = 0; j < P; ++j) {
        for (int i = 0; i < n1; ++i) {
            const long double t = std::cos((i + 0.5L) * pi / n1);
            const long double x = (long double)(j - p) - 0.5L * t;      // (x_g - x) / h
            const long double r = 1.0L - (x / half_w) * (x / half_w);
            f[i] = r < 0 ? 0.0L
                         : (window == 2 ? std::exp((long double)beta * (std::sqrt(r) - 1.0L))    // ES
                                        : std::cyl_bessel_il(0.0L, (long double)beta * std::sqrt(r)) / i0b);
        }
        for (int n = 0; n < n1; ++n) {
            long double acc = 0;
            for (int i = 0; i < n1; ++i) acc += f[i] * std::cos(n * (i + 0.5L) * pi / n1);
            a[n] = acc * (n == 0 ? 1.0L : 2.0L) / n1;
        }
        // T_n(2u) as monomials in u: T_0 = 1, T_1 = 2u, T_{n+1} = 4u T_n - T_{n-1}
        std::fill(mono.begin(), mono.end(), 0.0L);
        std::fill(Tm.begin(), Tm.end(), 0.0L);
        std::fill(Tc.begin(), Tc.end(), 0.0L);
        Tm[0] = 1.0L;
        mono[0] += a[0];
        if (n1 > 1) { Tc[1] = 2.0L; mono[1] += 2.0L * a[1]; }
        for (int n = 2; n < n1; ++n) {
            for (int e = 0; e < n1; ++e) Tn[e] = (e > 0 ? 4.0L * Tc[e - 1] : 0.0L) - Tm[e];
            for (int e = 0; e < n1; ++e) mono[e] += a[n] * Tn[e];
            Tm.swap(Tc);
            Tc.swap(Tn);
        }
        for (int e = 0; e < n1; ++e) c[size_t(e) * P + j] = double(mono[e]);
    }
}

void build_cheb_matrix(int Pc, std::vector<double>& C) {
    std::vector<double> Tn = node_T(Pc);
    C.resize(size_t(Pc) * Pc);
    for (int b = 0; b < Pc; ++b)
        for (int n = 0; n < Pc; ++n) C[b * Pc + n] = (n == 0 ? 1.0 : 2.0 * Tn[b * Pc + n]) / Pc;
}

std::string describe(const Params& p) {
    std::ostringstream o;
    o.precision(17);
    o << "N=" << p.N << "\nLx=" << p.Lx << "\nLy=" << p.Ly << "\nLz=" << p.Lz << "\ntol=" << p.tol
      << "\nrow=" << p.row << "\nb=" << p.b << "\nr0=" << p.r0 << "\nomega=" << p.omega
      << "\nrc=" << p.rc << "\nsigma=" << p.sigma << "\nM=" << p.M << "\nm=" << p.m
      << "\nIx=" << p.Ix << "\nIy=" << p.Iy << "\nIz=" << p.Iz << "\nIzs=" << p.Izs
      << "\nP=" << p.P << "\nS=" << p.S << "\nIlx=" << p.Ilx << "\nIly=" << p.Ily
      << "\nPl=" << p.Pl << "\nSl=" << p.Sl << "\nPc=" << p.Pc << "\nwindow=" << p.window
      << "\nnu=" << p.nu << "\nnul=" << p.nul << "\nlong_method=" << p.long_method << "\nKx=" << p.Kx
      << "\nKy=" << p.Ky << "\n";
    return o.str();
}

}  // namespace sog
