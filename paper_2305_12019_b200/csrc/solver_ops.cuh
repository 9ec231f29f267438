// Fused per-iteration operators of the inexact sGS-ADMM loop
// (reference pkg/src/gdwd/solver.py:493-555 and subsolvers.py).  Each Op
// plugs into zmv / ztmv / vmap (zops.cuh).  Expression order follows the
// reference's numpy expressions so elementwise results round identically
// (the library is compiled with -fmad=false; numpy never contracts).
#pragma once
#include "common.cuh"
#include "zops.cuh"

namespace gdwd {

constexpr double TINY = 1e-300;  // psqmr.py:14
constexpr int HIST_W = 16;       // history row: 11 KKT fields + sigma beta reused psqmr eps
enum HistCol { H_GAP = 8, H_OBJP = 9, H_OBJD = 10, H_SIGMA = 11, H_BETA = 12, H_REUSE = 13, H_PSQMR = 14, H_EPS = 15 };

// Device-resident scalars of one solve.
struct Scal {
  int k;          // index of the iteration (body) being executed
  int stopped;    // 1 => all later kernels of the solve are no-ops
  int iters_done; // completed iterations
  int converged;
  int reuse;      // Step-1c reuse decision of the current iteration
  int double_count;
  int error;      // 6: r <= 0 (AssertionError), 7: psqmr needs proximal switch
  int ps_iters, ps_active, ps_conv, ps_brk, ps_total, need_prox, pad0;
  double sigma, sigma_next;
  double sdual;       // sum w^(1/(q+1)) a+^(q/(q+1)) of the last KKT pass
  double eta[11];     // last KKT residuals (KKT_FIELDS order)
  double gnorm, wu2, w2;
  double smw_coef, smw_s2;
  double ps_tau, ps_rho, ps_theta, ps_alpha, ps_thnew, ps_cA, ps_cB, ps_rhonew, ps_resn;
  double ys;          // SMW: 1 + ybar^T J^{-1} ybar - 1
  double yjy;         // SMW: ybar^T G^{-1} ybar (the sum inside ys)
  double ytzw;        // Gram space: y . ztw_bar (= zy . w_bar)
  double pv[16];      // proximal: V^T v of the last projection
  double px_beta;     // proximal: beta of the current solve
  double ft_ys, ft_ya, ft_zal2;  // fused tail: y.(xi - r), y.alpha, ||Z~ alpha||^2 after Step 3
  unsigned pk_bar, pk_pad;       // persistent kernel: grid-barrier counter value at the end of the last launch
};

constexpr int PX_MAXL = 16;  // ell - 1 <= 16 eigenvectors in the proximal operator

struct Dev {
  int64_t n, d, m;  // m = d + 1
  int64_t bot;      // index of the scalar slot (beta, h_bot) in x/h vectors: d, or n in Gram space
  double C, q, mu, mu2, zscale, tau, yty, ynorm, kappa, e1, e2, qp1, one_c;
  double tol_feas, tol_cgap, tol_cap;
  int max_iter, sched_len;
  const double *y, *e, *wl, *zy, *jac, *jy;
  const double *kap, *gam;  // Gram-space SMW2: K jy, GK (y/|y|)
  double *r, *xi, *al, *ztw, *rnew, *dr, *ztwb, *s1, *g, *tq;
  double *u, *rho, *h, *h2, *xb, *x;
  double *pr, *pres, *pq, *pu, *pd, *pAd, *pAq;
  // Gram-space SMW2: n-coefficient temporaries and the d-space outputs
  double *cres, *cdiff;
  // fused tail (zft.cuh): Z~ (xi - r) and Z~ alpha after Step 3
  double *zp0, *zp1;
  double* aln;  // alpha after the fused tail's Step 3 (alpha itself is still being read)
  double *wd, *ud, *rhod;
  // proximal backend (subsolvers.py:159-256): V = top-(ell-1) eigenvectors of
  // Z~ Z~^T, eigenvector-major [L][d]; coefficient vectors for inv / fwd
  const double* pxV;
  const double *px_cinv, *px_cfwd;  // 1/(mu^2+lam_i) - base, lam_i - lam_ell
  double px_base, px_fwd0, px_schur;  // 1/(mu^2+lam_ell), mu^2+lam_ell, Schur scalar
  int px_L;
  double *px_sa, *px_hp, *px_tmp, *px_zaz;  // d-vectors
  const double *eps_tab, *tol_tab, *sched;
  double* hist;
  Scal* S;
};

// ---------------------------------------------------------------------------
// scalar rules
// ---------------------------------------------------------------------------
GDWD_DEV double sigma_rule(double sigma, double ep, double ed) {  // solver.py:343-362
  if (ep == 0.0 && ed == 0.0) return sigma;
  const double chi = (ed == 0.0) ? INFINITY : ep / ed;
  const double ichi = (ep == 0.0) ? INFINITY : ed / ep;
  const double worst = chi > ichi ? chi : ichi;
  const double zeta = worst > 500.0 ? 2.2 : (worst > 50.0 ? 1.65 : 1.1);
  if (chi > 5.0) return sigma * zeta;
  if (ichi > 5.0) return sigma / zeta;
  return sigma;
}

GDWD_DEV double bisect_margin(double a, double sigma, double q, double wt, double tol) {  // subsolvers.py:264-280
  double lo = 1e-12;
  double hi = (a > 0.0 ? a : 0.0) + pow((q * wt) / sigma, 1.0 / (q + 2.0)) + 1.0;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    const double gg = sigma * (mid - a) - (q * wt) / np_pow(mid, q + 1.0);
    if (fabs(gg) <= tol) return mid;
    // Once lo and hi are adjacent doubles, mid rounds onto one of them and
    // the bracket can stop changing; from then on every remaining step
    // repeats the same mid, residual and branch (the 1e-17 width test never
    // fires below one ulp), so leaving now returns the same 0.5*(lo+hi) the
    // reference reaches after all 200 steps.
    if (gg < 0.0) {
      if (mid == lo) break;
      lo = mid;
    } else {
      if (mid == hi) break;
      hi = mid;
    }
    if (hi - lo <= 1e-17 * (1.0 > hi ? 1.0 : hi)) break;
  }
  return 0.5 * (lo + hi);
}

// bisect_margin run by a whole warp (all 32 lanes call it with the same
// arguments and get the same root).  Each round, lane m evaluates the
// residual at node m of the next five levels of the bisection tree (31
// nodes, breadth-first; a node's bracket is rebuilt from its path with the
// same mid = 0.5*(lo+hi) roundings) together with the per-node outcomes of
// the sequential step -- exit (|g| <= tol), stuck bracket, the child bracket
// and its width test.  Ballots of those flags let every lane walk the five
// levels with integer operations; the value returned (or the bracket carried
// into the next round) is then shuffled from the lane of the node where the
// walk stopped.  Brackets, mids and exits are the sequential routine's, one
// residual evaluation per five steps.
GDWD_DEV double bisect_margin_warp(double a, double sigma, double q, double wt, double tol) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  double lo = 1e-12;
  double hi = (a > 0.0 ? a : 0.0) + pow((q * wt) / sigma, 1.0 / (q + 2.0)) + 1.0;
  const int m1 = lane + 1;  // 1-based heap index of this lane's node (lane 31: unused)
  const int depth = 31 - __clz(m1);
  int it = 0;
  for (;;) {
    double nlo = lo, nhi = hi;
    for (int l = depth - 1; l >= 0; --l) {  // path bit 1: residual < 0, lo = mid
      const double mid = 0.5 * (nlo + nhi);
      if ((m1 >> l) & 1) nlo = mid;
      else nhi = mid;
    }
    const double mid = 0.5 * (nlo + nhi);
    const double gg = sigma * (mid - a) - (q * wt) / np_pow(mid, q + 1.0);
    const bool neg = gg < 0.0;
    const double clo = neg ? mid : nlo, chi = neg ? nhi : mid;  // the bracket after this step
    const unsigned bneg = __ballot_sync(FULL, neg);
    const unsigned bret = __ballot_sync(FULL, fabs(gg) <= tol || (neg ? mid == nlo : mid == nhi));
    const unsigned bwid = __ballot_sync(FULL, chi - clo <= 1e-17 * (1.0 > chi ? 1.0 : chi));
    int node = 0, par = 0, src = -1;
    bool child = false;
#pragma unroll
    for (int lev = 0; lev < 5; ++lev) {
      const unsigned b = 1u << node;
      if (bret & b) {  // |g| <= tol returns mid; a stuck bracket returns 0.5*(lo+hi) = the same mid
        src = node;
        break;
      }
      if (++it >= 200 || (bwid & b)) {  // loop end / width break: 0.5*(lo+hi) of the new bracket
        src = node;
        child = true;
        break;
      }
      par = node;
      node = 2 * node + ((bneg & b) ? 2 : 1);
    }
    if (src >= 0) return __shfl_sync(FULL, child ? 0.5 * (clo + chi) : mid, src);
    lo = __shfl_sync(FULL, clo, par);
    hi = __shfl_sync(FULL, chi, par);
  }
}

// One coordinate of newton_r_sweep (subsolvers.py:321-364): same update and
// the sweep's two activity-test forms (``/ s**(q+1)`` first, then
// ``* s**(-(q+1))``).  scalar_form=1 reproduces the scalar newton_r
// (subsolvers.py:283-318), which uses the first form throughout; *iters
// receives its iteration count.
template <bool WARP>
GDWD_DEV double newton_margin_t(double a, double sigma, double q, double wt, double r0, double tol,
                                int max_newton, int scalar_form, int* iters) {
  const double mq = -q, qp1 = q + 1.0;
  const double c = (q * wt) / sigma;
  double s = r0;
  double foc = (mq * wt) / np_pow(s, qp1) + sigma * (s - a);
  int it = 0;
  if (!(fabs(foc) > tol)) {
    if (iters) *iters = 0;
    return s;
  }
  // iterates whose residual was tested in the form later iterates use (the
  // sweep tests r0 with the other form, so it is not recorded there)
  double seen[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) seen[j] = NAN;
  if (scalar_form) seen[0] = s;
  for (it = 0; it < max_newton; ++it) {
    const double sp = np_pow(s, qp1);
    const double nxt = (s * ((q + 2.0) * c + a * sp)) / ((q + 1.0) * c + sp * s);
    if (!isfinite(nxt) || nxt <= 0.0) {
      if (iters) *iters = it;
      if constexpr (WARP) return bisect_margin_warp(a, sigma, q, wt, tol);
      else return bisect_margin(a, sigma, q, wt, tol);
    }
    s = nxt;
    foc = scalar_form ? (mq * wt) / np_pow(s, qp1) + sigma * (s - a)
                      : (mq * wt) * np_pow(s, -qp1) + sigma * (s - a);
    if (!(fabs(foc) > tol)) {
      if (iters) *iters = it + 1;
      return s;
    }
    // The update is a fixed map of s: once it returns to an iterate already
    // tested (a fixed point or a cycle of length <= 8) every later iterate
    // and residual repeats, |foc| <= tol can no longer happen, and the
    // reference ends in the same bisection after max_newton updates.
    bool cyc = false;
#pragma unroll
    for (int j = 0; j < 8; ++j) cyc |= s == seen[j];
    if (cyc) break;
#pragma unroll
    for (int j = 7; j > 0; --j) seen[j] = seen[j - 1];
    seen[0] = s;
  }
  if (iters) *iters = max_newton;
  if constexpr (WARP) return bisect_margin_warp(a, sigma, q, wt, tol);
  else return bisect_margin(a, sigma, q, wt, tol);
}
GDWD_DEV double newton_margin(double a, double sigma, double q, double wt, double r0, double tol,
                              int max_newton = 50, int scalar_form = 0, int* iters = nullptr) {
  return newton_margin_t<false>(a, sigma, q, wt, r0, tol, max_newton, scalar_form, iters);
}
// the same root computed by a whole warp (uniform arguments in all lanes)
GDWD_DEV double newton_margin_warp(double a, double sigma, double q, double wt, double r0, double tol,
                                   int max_newton = 50, int scalar_form = 0, int* iters = nullptr) {
  return newton_margin_t<true>(a, sigma, q, wt, r0, tol, max_newton, scalar_form, iters);
}

GDWD_DEV double np_max0(double x) { return isnan(x) ? x : (x > 0.0 ? x : 0.0); }   // np.maximum(x, 0)
GDWD_DEV double np_min0(double x) { return isnan(x) ? x : (x < 0.0 ? x : 0.0); }   // np.minimum(x, 0)

// Completes iteration k-1 once ||Z alpha||^2 (`zal2`) is known: dual
// objective, gap, the stopping test (solver.py:293-304,334,548-554); then
// commits sigma and opens the history row of iteration k.
GDWD_DEV void finish_previous(const Dev& D, double zal2) {
  Scal* S = D.S;
  const int k = S->k;
  if (k > 0) {
    const double od = D.kappa * S->sdual - D.zscale * sqrt(zal2);
    const double op = S->eta[9];
    const double gap = fabs(op - od) / (1.0 + fabs(op) + fabs(od));
    S->eta[10] = od;
    S->eta[8] = gap;
    double* hr = D.hist + (int64_t)(k - 1) * HIST_W;
    hr[H_OBJD] = od;
    hr[H_GAP] = gap;
    const double* e = S->eta;
    const double ep = fmax(fmax(e[3], e[4]), e[5]);
    const double ed = fmax(e[6], e[7]);
    const double ec = fmax(fmax(e[0], e[1]), e[2]);
    if (fmax(ep, ed) < D.tol_feas && fmin(ec, gap) < D.tol_cgap && fmax(ec, gap) < D.tol_cap) {
      S->stopped = 1;
      S->converged = 1;
      return;
    }
  }
  if (k >= D.max_iter) {
    S->stopped = 1;
    return;
  }
  S->sigma = S->sigma_next;
  double* hr = D.hist + (int64_t)k * HIST_W;
  hr[H_SIGMA] = S->sigma;
  hr[H_EPS] = D.eps_tab[k];
  hr[H_REUSE] = 1.0;
  hr[H_PSQMR] = 0.0;
}

// ---------------------------------------------------------------------------
// KA: h = [-Z(xi - r - a/sigma) + mu^2 u + (mu/sigma) rho ; -y.rhs], fused
// with Z alpha of the previous iteration (its dual objective, gap and the
// stopping test, solver.py:293-304,334,548-554) -- one X pass, 2 RHS.
// ---------------------------------------------------------------------------
struct OpRhsAlpha {
  static constexpr int R = 2, NN = 1, ND = 1;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV void input(int64_t i, double (&t)[R], double (&na)[NN]) const {
    const double sig = D.S->sigma_next;
    t[0] = (D.xi[i] - D.r[i]) - D.al[i] / sig;
    t[1] = D.al[i];
    na[0] += D.y[i] * t[0];
  }
  GDWD_DEV void epi(int64_t j, const double (&v)[R], double (&da)[ND]) const {
    const double sig = D.S->sigma_next;
    D.h[j] = (-v[0] + D.mu2 * D.u[j]) + (D.mu / sig) * D.rho[j];
    da[0] += v[1] * v[1];
  }
  GDWD_DEV void fin(const double (&ns)[NN], const double (&ds)[ND]) const {
    D.h[D.bot] = -ns[0];
    finish_previous(D, ds[0]);
  }
};

// Dense GEMV with the explicit inverse (DIRECT: A^{-1}; replaces the two
// triangular solves of cholesky.py:60-61).  out = M hv.
struct OpGemvSolve {
  static constexpr int NN = 1;
  static constexpr bool HAS_FIN = false;
  Dev D;
  const double* hv;
  double* out;
  int pred;  // 1: run only when the Step-1c reuse test failed
  GDWD_DEV bool skip() const { return D.S->stopped || (pred && D.S->reuse); }
  GDWD_DEV double wval(int64_t j) const { return hv[j]; }
  GDWD_DEV void row(int64_t i, double dot, double (&)[NN]) const { out[i] = dot; }
  GDWD_DEV void fin(const double (&)[NN]) const {}
};

// copy src -> dst when the reuse test passed (solver.py:521-522)
struct OpCopyIfReuse {
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = false;
  Dev D;
  const double* src;
  double* dst;
  GDWD_DEV bool skip() const { return D.S->stopped || !D.S->reuse; }
  GDWD_DEV void elem(int64_t i, double (&)[NR]) const { dst[i] = src[i]; }
  GDWD_DEV void fin(const double (&)[NR]) const {}
};

struct OpCopy {  // dst = src
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = false;
  Dev D;
  const double* src;
  double* dst;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV void elem(int64_t i, double (&)[NR]) const { dst[i] = src[i]; }
  GDWD_DEV void fin(const double (&)[NR]) const {}
};

// KT: ztw_bar = Z^T w_bar, then c = ztw_bar + y beta_bar + xi - alpha/sigma,
// r+ = Newton (solver.py:501-504), dr = r+ - r, y.dr (solver.py:507-509).
struct OpZtNewton {
  static constexpr int NN = 1;
  static constexpr bool HAS_FIN = true;
  // <= 85 registers (3 CTAs per SM instead of 2 at the 100 the Newton epilogue
  // asks for): c3's pass 328 -> 268 us (6.0 TB/s); 4 CTAs (64 registers) the same
  static constexpr int ZT_MINB = 3;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV double wval(int64_t j) const { return D.xb[j]; }
  GDWD_DEV void row(int64_t i, double dot, double (&na)[NN]) const {
    const Scal* S = D.S;
    const double sig = S->sigma, bb = D.xb[D.bot];
    D.ztwb[i] = dot;
    const double a = ((dot + D.y[i] * bb) + D.xi[i]) - D.al[i] / sig;
    const double rn = newton_margin(a, sig, D.q, D.wl[i], D.r[i], D.tol_tab[S->k]);
    D.rnew[i] = rn;
    const double dri = rn - D.r[i];
    D.dr[i] = dri;
    na[0] += D.y[i] * dri;
  }
  GDWD_DEV void fin(const double (&ns)[NN]) const { D.h2[D.bot] = D.h[D.bot] + ns[0]; }
};

// KC: h2 = h + [Z dr; y.dr], reuse residual ||h2 - A [w_bar; beta_bar]||
// with A x via Z ztw_bar (solver.py:506-524); one X pass, 2 RHS.
struct OpDrZtwb {
  static constexpr int R = 2, NN = 1, ND = 2;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV void input(int64_t i, double (&t)[R], double (&)[NN]) const {
    t[0] = D.dr[i];
    t[1] = D.ztwb[i];
  }
  GDWD_DEV void epi(int64_t j, const double (&v)[R], double (&da)[ND]) const {
    const double bb = D.xb[D.bot];
    const double h2j = D.h[j] + v[0];
    D.h2[j] = h2j;
    const double ax = (v[1] + D.mu2 * D.xb[j]) + D.zy[j] * bb;
    const double rj = h2j - ax;
    da[0] += rj * rj;
    da[1] += D.zy[j] * D.xb[j];
  }
  GDWD_DEV void fin(const double (&)[NN], const double (&ds)[ND]) const {
    Scal* S = D.S;
    const double bb = D.xb[D.bot];
    const double rb = D.h2[D.bot] - (ds[1] + D.yty * bb);
    const double rr = hypot(sqrt(ds[0]), rb);
    const int reuse = rr <= 5.0 * D.eps_tab[S->k];
    S->reuse = reuse;
    if (!reuse) S->double_count += 1;
    D.hist[(int64_t)S->k * HIST_W + H_REUSE] = reuse ? 1.0 : 0.0;
  }
};

struct OpSetReuse {  // use_sgs = False
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV void elem(int64_t, double (&)[NR]) const {}
  GDWD_DEV void fin(const double (&)[NR]) const { D.S->reuse = 1; }
};

// ztw = Z^T w after a re-solve (solver.py:530)
struct OpZtStore {
  static constexpr int NN = 1;
  static constexpr bool HAS_FIN = false;
  Dev D;
  const double* wv;
  double* out;
  int pred;
  GDWD_DEV bool skip() const { return D.S->stopped || (pred && D.S->reuse); }
  GDWD_DEV double wval(int64_t j) const { return wv[j]; }
  GDWD_DEV void row(int64_t i, double dot, double (&)[NN]) const { out[i] = dot; }
  GDWD_DEV void fin(const double (&)[NN]) const {}
};

// Step 2a: g = w - rho/(sigma mu), ||g|| (solver.py:535-536)
struct OpStep2a {
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV void elem(int64_t j, double (&a)[NR]) const {
    const double gj = D.x[j] - D.rho[j] / (D.S->sigma * D.mu);
    a[0] += gj * gj;
  }
  GDWD_DEV void fin(const double (&s)[NR]) const { D.S->gnorm = sqrt(s[0]); }
};

// Step 2b: ball projection u, rho update (solver.py:537,542), ||w-u||, ||w||
struct OpStep2b {
  static constexpr int NR = 2;
  static constexpr bool HAS_FIN = true;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV void elem(int64_t j, double (&a)[NR]) const {
    const double sig = D.S->sigma, gn = D.S->gnorm;
    const double wj = D.x[j];
    const double gj = wj - D.rho[j] / (sig * D.mu);
    const double uj = (gn <= D.zscale) ? gj : (D.zscale / gn) * gj;
    D.u[j] = uj;
    D.rho[j] = D.rho[j] - ((D.tau * sig) * D.mu) * (wj - uj);
    const double dw = wj - uj;
    a[0] += dw * dw;
    a[1] += wj * wj;
  }
  GDWD_DEV void fin(const double (&s)[NR]) const {
    D.S->wu2 = s[0];
    D.S->w2 = s[1];
  }
};

// Step 3 + KKT sample terms (solver.py:533,538-541,311-333) and the
// per-iteration scalar logic: residuals, sigma update (or replay).
struct OpStep3 {
  static constexpr int NR = 10;
  static constexpr bool HAS_FIN = true;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV void elem(int64_t i, double (&a)[NR]) const {
    const double sig = D.S->sigma, bet = D.x[D.bot];
    const double C = D.C;
    const double rr = D.rnew[i];
    D.r[i] = rr;
    const double yi = D.y[i], ei = D.e[i], zt = D.ztw[i], ali = D.al[i];
    const double xv = np_max0((((rr - zt) - yi * bet) + ali / sig) - (C / sig) * ei);
    D.xi[i] = xv;
    const double pg = ((zt + yi * bet) + xv) - rr;
    const double an = ali - (D.tau * sig) * pg;
    D.al[i] = an;
    const double wl = D.wl[i];
    const double s = (D.q * wl) / np_pow(rr, D.qp1);
    const double d2 = an - s;
    const double mn = np_min0(an);
    const double mx = np_max0(an - C * ei);
    a[0] += yi * an;
    a[1] += xv * (C * ei - an);
    a[2] += d2 * d2;
    a[3] += pg * pg;
    a[4] += mn * mn;
    a[5] += mx * mx;
    a[6] += wl / np_pow(rr, D.q);
    a[7] += ei * xv;
    a[8] += np_pow(wl, D.e1) * np_pow(np_max0(an), D.e2);
    a[9] += (rr <= 0.0) ? 1.0 : 0.0;
  }
  GDWD_DEV void fin(const double (&s)[NR]) const {
    Scal* S = D.S;
    const int k = S->k;
    const double oc = D.one_c;
    if (s[9] > 0.0) {
      S->error = 6;
      S->stopped = 1;
      return;
    }
    double* e = S->eta;
    e[0] = fabs(s[0]) / oc;
    e[1] = fabs(s[1]) / oc;
    e[2] = s[2] / oc;
    e[3] = sqrt(s[3]) / oc;
    e[4] = (D.mu * sqrt(S->wu2)) / oc;
    e[5] = fmax(sqrt(S->w2) - D.zscale, 0.0) / oc;
    e[6] = sqrt(s[4]) / oc;
    e[7] = sqrt(s[5]) / oc;
    e[9] = s[6] + D.C * s[7];
    S->sdual = s[8];
    double* hr = D.hist + (int64_t)k * HIST_W;
    for (int f = 0; f < 8; ++f) hr[f] = e[f];
    hr[H_OBJP] = e[9];
    hr[H_BETA] = D.x[D.bot];
    const double ep = fmax(fmax(e[3], e[4]), e[5]);
    const double ed = fmax(e[6], e[7]);
    if (D.sched && k + 1 < D.sched_len) S->sigma_next = D.sched[k + 1];
    else S->sigma_next = sigma_rule(S->sigma, ep, ed);
    S->iters_done = k + 1;
    S->k = k + 1;
  }
};

// ---------------------------------------------------------------------------
// Fused tail of an X-space iteration (zft.cuh, SURVEY App. C fusion P2): one
// pass over X computes ztw = Z~^T w after a re-solve (solver.py:530; the
// reused ztw_bar otherwise, :521-522), Step 3 with the KKT sample sums
// (solver.py:538-541, 311-333) exactly as OpStep3, and the next iteration's
// products Z~ (xi - r) and Z~ alpha.  The next right-hand side
// Z~ (xi - r - alpha/sigma) is then Z~ (xi - r) - (Z~ alpha)/sigma_next
// (OpRhsParts, no pass over X): the same vector up to rounding.
// ---------------------------------------------------------------------------
struct OpTail {
  static constexpr int R = 2, NN = 2, ND = 1;
  struct Pf {
    double rn, y, e, al, zb;  // prefetched per-sample inputs
  };
  struct U {
    double sig, bet, tsig, csig;  // sigma, beta, tau*sigma, C/sigma
    int reuse;
  };
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV bool need_dot() const { return !D.S->reuse; }
  GDWD_DEV double wval(int64_t j) const { return D.x[j]; }
  GDWD_DEV U uniform() const {
    const Scal* S = D.S;
    U u;
    u.sig = S->sigma;
    u.bet = D.x[D.bot];
    u.tsig = D.tau * u.sig;
    u.csig = D.C / u.sig;
    u.reuse = S->reuse;
    return u;
  }
  static constexpr int NPF = 5;  // per-sample inputs, staged by cp.async (zft.cuh)
  GDWD_DEV const double* pf_src(int f, int64_t i) const {
    return (f == 0 ? D.rnew : f == 1 ? D.y : f == 2 ? D.e : f == 3 ? D.al : D.ztwb) + i;
  }
  GDWD_DEV void load_pf(const double* slot, Pf& p) const {
    p.rn = slot[0];
    p.y = slot[1];
    p.e = slot[2];
    p.al = slot[3];
    p.zb = slot[4];
  }
  // the OpStep3 elementwise update (same expressions); sums y.(xi - r), y.alpha
  GDWD_DEV void input(int64_t i, double dot, const Pf& p, const U& u, double (&t)[R], bool write,
                      double (&na)[NN]) const {
    const double rr = p.rn;
    const double yi = p.y, ei = p.e, zt = u.reuse ? p.zb : dot, ali = p.al;
    const double xv = np_max0((((rr - zt) - yi * u.bet) + ali / u.sig) - u.csig * ei);
    const double pg = ((zt + yi * u.bet) + xv) - rr;
    const double an = ali - u.tsig * pg;
    if (write) {
      D.ztw[i] = zt;
      D.r[i] = rr;
      D.xi[i] = xv;
      D.aln[i] = an;  // into alpha by OpKktTail: other ranks of the cluster may still read alpha
      na[0] += yi * (xv - rr);
      na[1] += yi * an;
    }
    t[0] = xv - rr;
    t[1] = an;
  }
  GDWD_DEV void epi(int64_t j, const double (&v)[R], double (&da)[ND]) const {
    D.zp0[j] = v[0];
    D.zp1[j] = v[1];
    da[0] += v[1] * v[1];
  }
  GDWD_DEV void fin(const double (&s)[NN], const double (&ds)[ND]) const {
    Scal* S = D.S;
    S->ft_ys = s[0];
    S->ft_ya = s[1];
    S->ft_zal2 = ds[0];
  }
};

// KKT sample sums of Step 3 after the fused tail (OpStep3's sums and fin,
// from the stored r, xi, alpha, ztw; pg recomputed with the same expression)
struct OpKktTail {
  static constexpr int NR = 10;
  static constexpr bool HAS_FIN = true;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV void elem(int64_t i, double (&a)[NR]) const {
    const double bet = D.x[D.bot], C = D.C;
    const double rr = D.r[i], yi = D.y[i], ei = D.e[i], zt = D.ztw[i], xv = D.xi[i], an = D.aln[i];
    D.al[i] = an;
    const double pg = ((zt + yi * bet) + xv) - rr;
    const double wl = D.wl[i];
    const double s = (D.q * wl) / np_pow(rr, D.qp1);
    const double d2 = an - s;
    const double mn = np_min0(an);
    const double mx = np_max0(an - C * ei);
    a[0] += yi * an;
    a[1] += xv * (C * ei - an);
    a[2] += d2 * d2;
    a[3] += pg * pg;
    a[4] += mn * mn;
    a[5] += mx * mx;
    a[6] += wl / np_pow(rr, D.q);
    a[7] += ei * xv;
    a[8] += np_pow(wl, D.e1) * np_pow(np_max0(an), D.e2);
    a[9] += (rr <= 0.0) ? 1.0 : 0.0;
  }
  GDWD_DEV void fin(const double (&s)[NR]) const { OpStep3{D}.fin(s); }
};

// h = [-(Z~(xi - r) - Z~ alpha / sigma) + mu^2 u + (mu/sigma) rho ;
//      -(y.(xi - r) - y.alpha / sigma)] from the fused tail's products, and
// the previous iteration's dual objective, gap and stopping test (the
// OpRhsAlpha fin) -- a d-space map, no pass over X.
struct OpRhsParts {
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV void elem(int64_t j, double (&)[NR]) const {
    const double sig = D.S->sigma_next;
    D.h[j] = (-(D.zp0[j] - D.zp1[j] / sig) + D.mu2 * D.u[j]) + (D.mu / sig) * D.rho[j];
  }
  GDWD_DEV void fin(const double (&)[NR]) const {
    Scal* S = D.S;
    D.h[D.bot] = -(S->ft_ys - S->ft_ya / S->sigma_next);
    finish_previous(D, S->ft_zal2);
  }
};

// ---------------------------------------------------------------------------
// SMW solve (subsolvers.py:127-151) with the explicit G^{-1}
// ---------------------------------------------------------------------------
struct OpSmwS1 {  // s1 = Z^T (h/mu^2) + y t2
  static constexpr int NN = 1;
  static constexpr bool HAS_FIN = false;
  Dev D;
  const double* hv;
  int pred;
  GDWD_DEV bool skip() const { return D.S->stopped || (pred && D.S->reuse); }
  GDWD_DEV double wval(int64_t j) const { return hv[j] / D.mu2; }
  GDWD_DEV void row(int64_t i, double dot, double (&)[NN]) const {
    const double t2 = hv[D.bot] / D.yty;
    D.s1[i] = dot + D.y[i] * t2;
  }
  GDWD_DEV void fin(const double (&)[NN]) const {}
};

struct OpSmwG {  // g = G^{-1} s1 ; ybar.J^{-1}s
  static constexpr int NN = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  const double* hv;
  int pred;
  GDWD_DEV bool skip() const { return D.S->stopped || (pred && D.S->reuse); }
  GDWD_DEV double wval(int64_t j) const { return D.s1[j]; }
  GDWD_DEV void row(int64_t i, double dot, double (&na)[NN]) const {
    D.g[i] = dot;
    na[0] += (D.y[i] / D.ynorm) * dot;
  }
  GDWD_DEV void fin(const double (&ns)[NN]) const {
    const double t2 = hv[D.bot] / D.yty;
    const double s2 = D.ynorm * t2;
    const double bd = ns[0] + (-s2);
    D.S->smw_coef = bd / D.S->ys;
    D.S->smw_s2 = s2;
  }
};

struct OpSmwP {  // p1 = Z v[:n]; x = [t1 - p1/mu^2 ; t2 - p2/|y|^2]
  static constexpr int R = 1, NN = 1, ND = 1;
  Dev D;
  const double* hv;
  double* out;
  int pred;
  GDWD_DEV bool skip() const { return D.S->stopped || (pred && D.S->reuse); }
  GDWD_DEV void input(int64_t i, double (&t)[R], double (&na)[NN]) const {
    const double v = D.g[i] - D.S->smw_coef * D.jy[i];
    t[0] = v;
    na[0] += D.y[i] * v;
  }
  GDWD_DEV void epi(int64_t j, const double (&v)[R], double (&)[ND]) const {
    out[j] = hv[j] / D.mu2 - v[0] / D.mu2;
  }
  GDWD_DEV void fin(const double (&ns)[NN], const double (&)[ND]) const {
    const double vn = (-D.S->smw_s2) - D.S->smw_coef * (-1.0);
    const double p2 = ns[0] + D.ynorm * vn;
    out[D.bot] = hv[D.bot] / D.yty - p2 / D.yty;
  }
};


// ---------------------------------------------------------------------------
// Gram-space SMW2.  Every d-vector of the SMW2 iteration stays in span(Z~)
// (u = rho = w = 0 initially; h, w_bar, w, g, u, rho are linear combinations
// of Z~ columns), so each is carried as n coefficients c with v = Z~ c and
// every Z~ / Z~^T product becomes a GEMV with the n x n Gram K = Z~^T Z~
// (L2-resident) instead of a pass over X.  D.h/h2/xb/x hold coefficients
// (+ the scalar slot at D.bot = n); D.u / D.rho hold the coefficients of u
// and rho.  Norms are quadratic forms c^T K c of difference vectors formed
// first (no cancellation at large sigma).
// ---------------------------------------------------------------------------
struct GsKAlpha {  // ||Z alpha||^2 = alpha^T K alpha, then finish iteration k-1
  static constexpr int NN = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV double wval(int64_t j) const { return D.al[j]; }
  GDWD_DEV void row(int64_t i, double dot, double (&na)[NN]) const { na[0] += D.al[i] * dot; }
  GDWD_DEV void fin(const double (&ns)[NN]) const { finish_previous(D, ns[0]); }
};

struct GsRhs {  // c_h = -rhs + mu^2 c_u + (mu/sigma) c_rho ; h_bot = -y.rhs
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV void elem(int64_t i, double (&a)[NR]) const {
    const double sig = D.S->sigma;
    const double rhs = (D.xi[i] - D.r[i]) - D.al[i] / sig;
    D.h[i] = (-rhs + D.mu2 * D.u[i]) + (D.mu / sig) * D.rho[i];
    a[0] += D.y[i] * rhs;
  }
  GDWD_DEV void fin(const double (&s)[NR]) const { D.h[D.bot] = -s[0]; }
};

struct GsX {  // x = [t1 - v/mu^2 ; t2 - p2/|y|^2] in coefficients (subsolvers.py:145-151)
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  const double* hv;
  double* out;
  int pred;
  GDWD_DEV bool skip() const { return D.S->stopped || (pred && D.S->reuse); }
  GDWD_DEV void elem(int64_t i, double (&a)[NR]) const {
    const double v = D.g[i] - D.S->smw_coef * D.jy[i];
    out[i] = hv[i] / D.mu2 - v / D.mu2;
    a[0] += D.y[i] * v;
  }
  GDWD_DEV void fin(const double (&s)[NR]) const {
    const double vn = (-D.S->smw_s2) - D.S->smw_coef * (-1.0);
    const double p2 = s[0] + D.ynorm * vn;
    out[D.bot] = hv[D.bot] / D.yty - p2 / D.yty;
  }
};

struct GsResid1 {  // h2 = h + [dr; y.dr]; c_res = c_h2 - (ztw_bar + mu^2 c_xb + y beta_bar)
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV void elem(int64_t i, double (&a)[NR]) const {
    const double bb = D.xb[D.bot];
    const double h2 = D.h[i] + D.dr[i];
    D.h2[i] = h2;
    const double ax = (D.ztwb[i] + D.mu2 * D.xb[i]) + D.y[i] * bb;
    D.cres[i] = h2 - ax;
    a[0] += D.y[i] * D.ztwb[i];
  }
  GDWD_DEV void fin(const double (&s)[NR]) const { D.S->ytzw = s[0]; }
};

struct GsResid2 {  // ||res_top||^2 = c_res^T K c_res ; reuse test (solver.py:516-524)
  static constexpr int NN = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV double wval(int64_t j) const { return D.cres[j]; }
  GDWD_DEV void row(int64_t i, double dot, double (&na)[NN]) const { na[0] += D.cres[i] * dot; }
  GDWD_DEV void fin(const double (&ns)[NN]) const {
    Scal* S = D.S;
    const double bb = D.xb[D.bot];
    const double rb = D.h2[D.bot] - (S->ytzw + D.yty * bb);
    const double rr = hypot(sqrt(ns[0] > 0.0 ? ns[0] : 0.0), rb);
    const int reuse = rr <= 5.0 * D.eps_tab[S->k];
    S->reuse = reuse;
    if (!reuse) S->double_count += 1;
    D.hist[(int64_t)S->k * HIST_W + H_REUSE] = reuse ? 1.0 : 0.0;
  }
};

struct GsStep2a {  // g = w - rho/(sigma mu) ; ||g||^2 = c_g^T K c_g
  static constexpr int NN = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV double cg(int64_t j) const { return D.x[j] - D.rho[j] / (D.S->sigma * D.mu); }
  GDWD_DEV double wval(int64_t j) const { return cg(j); }
  GDWD_DEV void row(int64_t i, double dot, double (&na)[NN]) const { na[0] += cg(i) * dot; }
  GDWD_DEV void fin(const double (&ns)[NN]) const { D.S->gnorm = sqrt(ns[0] > 0.0 ? ns[0] : 0.0); }
};

struct GsStep2b {  // u, rho updates in coefficients; c_w - c_u ; ||w||^2 = c_w . ztw
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV void elem(int64_t i, double (&a)[NR]) const {
    const double sig = D.S->sigma, gn = D.S->gnorm;
    const double wi = D.x[i];
    const double gi = wi - D.rho[i] / (sig * D.mu);
    const double ui = (gn <= D.zscale) ? gi : (D.zscale / gn) * gi;
    D.u[i] = ui;
    D.rho[i] = D.rho[i] - ((D.tau * sig) * D.mu) * (wi - ui);
    D.cdiff[i] = wi - ui;
    a[0] += wi * D.ztw[i];
  }
  GDWD_DEV void fin(const double (&s)[NR]) const { D.S->w2 = s[0]; }
};

struct GsStep2c {  // ||w - u||^2 = (c_w - c_u)^T K (c_w - c_u)
  static constexpr int NN = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV double wval(int64_t j) const { return D.cdiff[j]; }
  GDWD_DEV void row(int64_t i, double dot, double (&na)[NN]) const { na[0] += D.cdiff[i] * dot; }
  GDWD_DEV void fin(const double (&ns)[NN]) const { D.S->wu2 = ns[0] > 0.0 ? ns[0] : 0.0; }
};

// d-space iterates from coefficients (end of solve / callback): w, u (+beta)
struct GsMaterialize2 {
  static constexpr int R = 2, NN = 1, ND = 1;
  Dev D;
  GDWD_DEV bool skip() const { return false; }
  GDWD_DEV void input(int64_t i, double (&t)[R], double (&)[NN]) const {
    t[0] = D.x[i];
    t[1] = D.u[i];
  }
  GDWD_DEV void epi(int64_t j, const double (&v)[R], double (&)[ND]) const {
    D.wd[j] = v[0];
    D.ud[j] = v[1];
  }
  GDWD_DEV void fin(const double (&)[NN], const double (&)[ND]) const { D.wd[D.d] = D.x[D.bot]; }
};

struct GsMaterialize1 {  // rho
  static constexpr int R = 1, NN = 1, ND = 1;
  Dev D;
  GDWD_DEV bool skip() const { return false; }
  GDWD_DEV void input(int64_t i, double (&t)[R], double (&)[NN]) const { t[0] = D.rho[i]; }
  GDWD_DEV void epi(int64_t j, const double (&v)[R], double (&)[ND]) const { D.rhod[j] = v[0]; }
  GDWD_DEV void fin(const double (&)[NN], const double (&)[ND]) const {}
};

// ---------------------------------------------------------------------------
// PSQMR (linalg/psqmr.py:27-95) on A = [Z Z^T + mu^2 I, zy; zy^T, y^Ty]
// with the Jacobi preconditioner (solver.py:428-438).
// ---------------------------------------------------------------------------
struct OpApplyZt {  // tq = Z^T v_top
  static constexpr int NN = 1;
  static constexpr bool HAS_FIN = false;
  Dev D;
  const double* v;
  int pred;
  int mode;  // 0: initial residual (predicated on reuse), 1: PSQMR step (needs ps_active)
  GDWD_DEV bool skip() const {
    if (D.S->stopped) return true;
    return mode == 0 ? (pred && D.S->reuse) : !D.S->ps_active;
  }
  GDWD_DEV double wval(int64_t j) const { return v[j]; }
  GDWD_DEV void row(int64_t i, double dot, double (&)[NN]) const { D.tq[i] = dot; }
  GDWD_DEV void fin(const double (&)[NN]) const {}
};

// r = b - A x0 (init, psqmr.py:49) -- pred >= 0 flags; active test skipped
struct OpInitResidual {
  static constexpr int R = 1, NN = 1, ND = 1;
  Dev D;
  const double* x0;
  const double* b;
  int pred;
  GDWD_DEV bool skip() const { return D.S->stopped || (pred && D.S->reuse); }
  GDWD_DEV void input(int64_t i, double (&t)[R], double (&)[NN]) const { t[0] = D.tq[i]; }
  GDWD_DEV void epi(int64_t j, const double (&v)[R], double (&da)[ND]) const {
    const double ax = (v[0] + D.mu2 * x0[j]) + D.zy[j] * x0[D.bot];
    D.pr[j] = b[j] - ax;
    da[0] += D.zy[j] * x0[j];
  }
  GDWD_DEV void fin(const double (&)[NN], const double (&ds)[ND]) const {
    const double ax = ds[0] + D.yty * x0[D.bot];
    D.pr[D.bot] = b[D.bot] - ax;
  }
};

struct OpPsInit {
  static constexpr int NR = 3;
  static constexpr bool HAS_FIN = true;
  Dev D;
  const double* x0;
  double* xo;
  int pred;
  double tolmul;
  GDWD_DEV bool skip() const { return D.S->stopped || (pred && D.S->reuse); }
  GDWD_DEV void elem(int64_t j, double (&a)[NR]) const {
    xo[j] = x0[j];
    const double rj = D.pr[j];
    D.pres[j] = rj;
    const double qj = rj / D.jac[j];
    D.pq[j] = qj;
    D.pd[j] = 0.0;
    D.pAd[j] = 0.0;
    a[0] += rj * rj;
    a[1] += qj * qj;
    a[2] += rj * qj;
  }
  GDWD_DEV void fin(const double (&s)[NR]) const {
    Scal* S = D.S;
    const double tol = tolmul * D.eps_tab[S->k];
    S->ps_resn = sqrt(s[0]);
    S->ps_iters = 0;
    S->ps_conv = 0;
    S->ps_brk = 0;
    if (S->ps_resn <= tol) {
      S->ps_conv = 1;
      S->ps_active = 0;
      return;
    }
    S->ps_tau = sqrt(s[1]);
    S->ps_rho = s[2];
    S->ps_theta = 0.0;
    S->ps_active = 1;
  }
};

// Aq = A q  (second half of the operator) fused with sigma = q.Aq, alpha
struct OpPsApply {
  static constexpr int R = 1, NN = 1, ND = 2;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped || !D.S->ps_active; }
  GDWD_DEV void input(int64_t i, double (&t)[R], double (&)[NN]) const { t[0] = D.tq[i]; }
  GDWD_DEV void epi(int64_t j, const double (&v)[R], double (&da)[ND]) const {
    const double qj = D.pq[j];
    const double aq = (v[0] + D.mu2 * qj) + D.zy[j] * D.pq[D.bot];
    D.pAq[j] = aq;
    da[0] += D.zy[j] * qj;
    da[1] += qj * aq;
  }
  GDWD_DEV void fin(const double (&)[NN], const double (&ds)[ND]) const {
    Scal* S = D.S;
    const double qd = D.pq[D.bot];
    const double aqd = ds[0] + D.yty * qd;
    D.pAq[D.bot] = aqd;
    const double sg = ds[1] + qd * aqd;
    if (fabs(sg) < TINY) {
      S->ps_brk = 1;
      S->ps_active = 0;
      return;
    }
    S->ps_alpha = S->ps_rho / sg;
  }
};

// The same two PSQMR operator applications with A's block Z~ Z~^T taken
// from the explicit d x d Gram Gd (symmetric: row j of Gd dotted with the
// top of the vector is (Z~ Z~^T v)_j): one GEMV over Gd instead of a Z~^T
// pass and a Z~ pass.  Rows are features; the "sample sums" of the row
// kernel are the feature sums of OpPsApply / OpInitResidual.
struct OpPsApplyGram {
  static constexpr int NN = 2;
  static constexpr bool HAS_FIN = true;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped || !D.S->ps_active; }
  GDWD_DEV double wval(int64_t j) const { return D.pq[j]; }
  GDWD_DEV void row(int64_t j, double dot, double (&da)[NN]) const {
    const double qj = D.pq[j];
    const double aq = (dot + D.mu2 * qj) + D.zy[j] * D.pq[D.bot];
    D.pAq[j] = aq;
    da[0] += D.zy[j] * qj;
    da[1] += qj * aq;
  }
  GDWD_DEV void fin(const double (&ds)[NN]) const {
    Scal* S = D.S;
    const double qd = D.pq[D.bot];
    const double aqd = ds[0] + D.yty * qd;
    D.pAq[D.bot] = aqd;
    const double sg = ds[1] + qd * aqd;
    if (fabs(sg) < TINY) {
      S->ps_brk = 1;
      S->ps_active = 0;
      return;
    }
    S->ps_alpha = S->ps_rho / sg;
  }
};
struct OpInitResidualGram {
  static constexpr int NN = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  const double* x0;
  const double* b;
  int pred;
  GDWD_DEV bool skip() const { return D.S->stopped || (pred && D.S->reuse); }
  GDWD_DEV double wval(int64_t j) const { return x0[j]; }
  GDWD_DEV void row(int64_t j, double dot, double (&da)[NN]) const {
    const double ax = (dot + D.mu2 * x0[j]) + D.zy[j] * x0[D.bot];
    D.pr[j] = b[j] - ax;
    da[0] += D.zy[j] * x0[j];
  }
  GDWD_DEV void fin(const double (&ds)[NN]) const {
    const double ax = ds[0] + D.yty * x0[D.bot];
    D.pr[D.bot] = b[D.bot] - ax;
  }
};

struct OpPsV1 {  // r -= alpha Aq ; u = M^{-1} r ; ||u||, r.u
  static constexpr int NR = 2;
  static constexpr bool HAS_FIN = true;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped || !D.S->ps_active; }
  GDWD_DEV void elem(int64_t j, double (&a)[NR]) const {
    const double rj = D.pr[j] - D.S->ps_alpha * D.pAq[j];
    D.pr[j] = rj;
    const double uj = rj / D.jac[j];
    D.pu[j] = uj;
    a[0] += uj * uj;
    a[1] += rj * uj;
  }
  GDWD_DEV void fin(const double (&s)[NR]) const {
    Scal* S = D.S;
    const double th = (S->ps_tau > TINY) ? sqrt(s[0]) / S->ps_tau : 0.0;
    const double c2 = 1.0 / (1.0 + th * th);
    S->ps_tau = (S->ps_tau * th) * sqrt(c2);
    S->ps_cA = (c2 * S->ps_theta) * S->ps_theta;
    S->ps_cB = c2 * S->ps_alpha;
    S->ps_thnew = th;
    S->ps_rhonew = s[1];
  }
};

struct OpPsV2 {  // d, x, Ad, res updates; ||res||; q = u + beta q
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  double* xo;
  double tolmul;
  int max_steps;
  GDWD_DEV bool skip() const { return D.S->stopped || !D.S->ps_active; }
  GDWD_DEV void elem(int64_t j, double (&a)[NR]) const {
    const Scal* S = D.S;
    const double cA = S->ps_cA, cB = S->ps_cB;
    const double qj = D.pq[j];
    const double dj = cA * D.pd[j] + cB * qj;
    D.pd[j] = dj;
    xo[j] = xo[j] + dj;
    const double adj = cA * D.pAd[j] + cB * D.pAq[j];
    D.pAd[j] = adj;
    const double rs = D.pres[j] - adj;
    D.pres[j] = rs;
    a[0] += rs * rs;
    D.pq[j] = D.pu[j] + (S->ps_rhonew / S->ps_rho) * qj;
  }
  GDWD_DEV void fin(const double (&s)[NR]) const {
    Scal* S = D.S;
    S->ps_iters += 1;
    S->ps_resn = sqrt(s[0]);
    if (S->ps_resn <= tolmul * D.eps_tab[S->k]) {
      S->ps_conv = 1;
      S->ps_active = 0;
      return;
    }
    if (fabs(S->ps_rho) < TINY) {
      S->ps_brk = 1;
      S->ps_active = 0;
      return;
    }
    S->ps_rho = S->ps_rhonew;
    S->ps_theta = S->ps_thnew;
    if (S->ps_iters >= max_steps) S->ps_active = 0;
  }
};


// End of a device-resident PSQMR call (psqmr.py:65-93 as captured in a CUDA
// graph WHILE node): the step count joins the totals and the history; a run
// that did not converge (step cap or breakdown) is the permanent switch to
// the proximal backend (solver.py:479-483), which the host builds -- the
// solve stops here (every later kernel is a no-op) with error 7 and the
// number of the failed solve, and the host resumes the iteration.
struct OpPsEnd {
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  int pred;   // 1: the Step-1c re-solve (skipped when the reuse test passed)
  int which;  // 1: first solve of the iteration, 2: the re-solve
  GDWD_DEV bool skip() const { return D.S->stopped || (pred && D.S->reuse); }
  GDWD_DEV void elem(int64_t, double (&)[NR]) const {}
  GDWD_DEV void fin(const double (&)[NR]) const {
    Scal* S = D.S;
    S->ps_total += S->ps_iters;
    D.hist[(int64_t)S->k * HIST_W + H_PSQMR] += (double)S->ps_iters;
    if (!S->ps_conv) {
      S->error = 7;
      S->need_prox = which;
      S->stopped = 1;
    }
  }
};

// ---------------------------------------------------------------------------
// Proximal backend (subsolvers.py:169-256).  inv(v) = base v + V (c_inv .* V^T v)
// and fwd(v) = (mu^2 + lam_ell) v + V (c_fwd .* V^T v) over the top-(ell-1)
// eigenvectors; d-space, replicated across shards.
// ---------------------------------------------------------------------------
struct OpPxDot {  // pv = V^T src
  static constexpr int NR = PX_MAXL;
  static constexpr bool HAS_FIN = true;
  Dev D;
  const double* src;
  int pred;
  GDWD_DEV bool skip() const { return D.S->stopped || (pred && D.S->reuse); }
  GDWD_DEV void elem(int64_t j, double (&a)[NR]) const {
    const double v = src[j];
#pragma unroll
    for (int i = 0; i < NR; ++i)
      if (i < D.px_L) a[i] += D.pxV[(int64_t)i * D.d + j] * v;
  }
  GDWD_DEV void fin(const double (&s)[NR]) const {
#pragma unroll
    for (int i = 0; i < NR; ++i) D.S->pv[i] = s[i];
  }
};

GDWD_DEV double px_lowrank(const Dev& D, int64_t j, const double* coef) {
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < PX_MAXL; ++i)
    if (i < D.px_L) acc += D.pxV[(int64_t)i * D.d + j] * (coef[i] * D.S->pv[i]);
  return acc;
}

// sa = fwd(w) - mu^2 w - Z ztw (solver.py:484-488); hp = h_top + sa
struct OpPxShift {
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = false;
  Dev D;
  const double* aw;
  const double* hv;
  int pred;
  GDWD_DEV bool skip() const { return D.S->stopped || (pred && D.S->reuse); }
  GDWD_DEV void elem(int64_t j, double (&)[NR]) const {
    const double fw = D.px_fwd0 * aw[j] + px_lowrank(D, j, D.px_cfwd);
    const double sa = (fw - D.mu2 * aw[j]) - D.px_zaz[j];
    D.px_sa[j] = sa;
    D.px_hp[j] = hv[j] + sa;
  }
  GDWD_DEV void fin(const double (&)[NR]) const {}
};

// hp = h_top + sa with a stored sa (second solve of an iteration)
struct OpPxShifted {
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = false;
  Dev D;
  const double* hv;
  int pred;
  GDWD_DEV bool skip() const { return D.S->stopped || (pred && D.S->reuse); }
  GDWD_DEV void elem(int64_t j, double (&)[NR]) const { D.px_hp[j] = hv[j] + D.px_sa[j]; }
  GDWD_DEV void fin(const double (&)[NR]) const {}
};

// beta = (h_bot - zy . inv(hp)) / schur  (solver_proximal first half)
struct OpPxBeta {
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  const double* hv;
  int pred;
  GDWD_DEV bool skip() const { return D.S->stopped || (pred && D.S->reuse); }
  GDWD_DEV void elem(int64_t j, double (&a)[NR]) const {
    const double iv = D.px_base * D.px_hp[j] + px_lowrank(D, j, D.px_cinv);
    a[0] += D.zy[j] * iv;
  }
  GDWD_DEV void fin(const double (&s)[NR]) const {
    double beta = (hv[D.bot] - s[0]);
    beta /= D.px_schur;
    D.S->px_beta = beta;
  }
};

// tmp = hp - zy beta
struct OpPxRhs2 {
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = false;
  Dev D;
  int pred;
  GDWD_DEV bool skip() const { return D.S->stopped || (pred && D.S->reuse); }
  GDWD_DEV void elem(int64_t j, double (&)[NR]) const { D.px_tmp[j] = D.px_hp[j] - D.zy[j] * D.S->px_beta; }
  GDWD_DEV void fin(const double (&)[NR]) const {}
};

// out = [inv(tmp) ; beta]
struct OpPxW {
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = true;
  Dev D;
  double* out;
  int pred;
  GDWD_DEV bool skip() const { return D.S->stopped || (pred && D.S->reuse); }
  GDWD_DEV void elem(int64_t j, double (&)[NR]) const {
    out[j] = D.px_base * D.px_tmp[j] + px_lowrank(D, j, D.px_cinv);
  }
  GDWD_DEV void fin(const double (&)[NR]) const { out[D.bot] = D.S->px_beta; }
};

// sGS residual in proximal mode (solver.py:510-520): h2 = h + Z dr (epilogue
// of a Z dr pass), ax = fwd(w_bar) + zy beta_bar, res = h2 + sa - ax
struct OpPxH2 {
  static constexpr int R = 1, NN = 1, ND = 1;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV void input(int64_t i, double (&t)[R], double (&na)[NN]) const {
    t[0] = D.dr[i];
    na[0] += D.y[i] * D.dr[i];
  }
  GDWD_DEV void epi(int64_t j, const double (&v)[R], double (&)[ND]) const { D.h2[j] = D.h[j] + v[0]; }
  GDWD_DEV void fin(const double (&ns)[NN], const double (&)[ND]) const { D.h2[D.bot] = D.h[D.bot] + ns[0]; }
};

struct OpPxResid {
  static constexpr int NR = 2;
  static constexpr bool HAS_FIN = true;
  Dev D;
  GDWD_DEV bool skip() const { return D.S->stopped; }
  GDWD_DEV void elem(int64_t j, double (&a)[NR]) const {
    const double bb = D.xb[D.bot];
    const double fw = D.px_fwd0 * D.xb[j] + px_lowrank(D, j, D.px_cfwd);
    const double ax = fw + D.zy[j] * bb;
    const double rj = (D.h2[j] + D.px_sa[j]) - ax;
    a[0] += rj * rj;
    a[1] += D.zy[j] * D.xb[j];
  }
  GDWD_DEV void fin(const double (&s)[NR]) const {
    Scal* S = D.S;
    const double bb = D.xb[D.bot];
    const double rb = D.h2[D.bot] - (s[1] + D.yty * bb);
    const double rr = hypot(sqrt(s[0]), rb);
    const int reuse = rr <= 5.0 * D.eps_tab[S->k];
    S->reuse = reuse;
    if (!reuse) S->double_count += 1;
    D.hist[(int64_t)S->k * HIST_W + H_REUSE] = reuse ? 1.0 : 0.0;
  }
};

struct OpZtwStore {  // zaz = Z ztw (the anchor's Z Z^T w term)
  static constexpr int R = 1, NN = 1, ND = 1;
  Dev D;
  const double* src;
  int pred;
  GDWD_DEV bool skip() const { return D.S->stopped || (pred && D.S->reuse); }
  GDWD_DEV void input(int64_t i, double (&t)[R], double (&)[NN]) const { t[0] = src[i]; }
  GDWD_DEV void epi(int64_t j, const double (&v)[R], double (&)[ND]) const { D.px_zaz[j] = v[0]; }
  GDWD_DEV void fin(const double (&)[NN], const double (&)[ND]) const {}
};

// ---------------------------------------------------------------------------
// setup / seam ops
// ---------------------------------------------------------------------------
struct OpPlainZ {  // out = Z t (+ n-dot y.t into *dot)
  static constexpr int R = 1, NN = 1, ND = 1;
  const double* t;
  const double* y;
  double* out;
  double* dot;
  GDWD_DEV bool skip() const { return false; }
  GDWD_DEV void input(int64_t i, double (&tv)[R], double (&na)[NN]) const {
    tv[0] = t[i];
    if (y) na[0] += y[i] * t[i];
  }
  GDWD_DEV void epi(int64_t j, const double (&v)[R], double (&)[ND]) const { out[j] = v[0]; }
  GDWD_DEV void fin(const double (&ns)[NN], const double (&)[ND]) const {
    if (dot) *dot = ns[0];
  }
};

struct OpPlainZt {  // out = Z^T w
  static constexpr int NN = 1;
  static constexpr bool HAS_FIN = false;
  const double* w;
  double* out;
  GDWD_DEV bool skip() const { return false; }
  GDWD_DEV double wval(int64_t j) const { return w[j]; }
  GDWD_DEV void row(int64_t i, double dot, double (&)[NN]) const { out[i] = dot; }
  GDWD_DEV void fin(const double (&)[NN]) const {}
};

// kkt_residuals (solver.py:311-340) of a caller-supplied iterate, without
// touching solver state.  Sample sums in the Z~^T w pass, ||Z~ alpha||^2 in
// the Z~ alpha pass, the d-space norms in a map; out[0..13) receives
// [y.a, xi.(Ce - a), |a - s|^2, |p|^2, |min(a,0)|^2, |max(a - Ce,0)|^2,
//  sum wl / r^q, e.xi, sum wl^(1/(q+1)) max(a,0)^(q/(q+1)), #(r <= 0),
//  ||Z~ a||^2, ||w - u||^2, ||w||^2].
struct KktArgs {
  const double *r, *xi, *al, *w, *u, *y, *e, *wl;
  double beta, C, q, qp1, e1, e2;
  double* out;
};
struct OpKktZt {
  static constexpr int NN = 10;
  static constexpr bool HAS_FIN = true;
  KktArgs K;
  GDWD_DEV bool skip() const { return false; }
  GDWD_DEV double wval(int64_t j) const { return K.w[j]; }
  GDWD_DEV void row(int64_t i, double dot, double (&a)[NN]) const {
    const double rr = K.r[i], xv = K.xi[i], an = K.al[i], yi = K.y[i], ei = K.e[i], wl = K.wl[i], C = K.C;
    const double s = (K.q * wl) / np_pow(rr, K.qp1);
    const double d2 = an - s;
    const double pg = ((dot + K.beta * yi) + xv) - rr;
    const double mn = np_min0(an), mx = np_max0(an - C * ei);
    a[0] += yi * an;
    a[1] += xv * (C * ei - an);
    a[2] += d2 * d2;
    a[3] += pg * pg;
    a[4] += mn * mn;
    a[5] += mx * mx;
    a[6] += wl / np_pow(rr, K.q);
    a[7] += ei * xv;
    a[8] += np_pow(wl, K.e1) * np_pow(np_max0(an), K.e2);
    a[9] += (rr <= 0.0) ? 1.0 : 0.0;
  }
  GDWD_DEV void fin(const double (&a)[NN]) const {
#pragma unroll
    for (int f = 0; f < NN; ++f) K.out[f] = a[f];
  }
};
struct OpKktZa {  // ||Z~ alpha||^2
  static constexpr int R = 1, NN = 1, ND = 1;
  KktArgs K;
  GDWD_DEV bool skip() const { return false; }
  GDWD_DEV void input(int64_t i, double (&t)[R], double (&)[NN]) const { t[0] = K.al[i]; }
  GDWD_DEV void epi(int64_t, const double (&v)[R], double (&da)[ND]) const { da[0] += v[0] * v[0]; }
  GDWD_DEV void fin(const double (&)[NN], const double (&ds)[ND]) const { K.out[10] = ds[0]; }
};
struct OpKktD {  // ||w - u||^2, ||w||^2
  static constexpr int NR = 2;
  static constexpr bool HAS_FIN = true;
  KktArgs K;
  GDWD_DEV bool skip() const { return false; }
  GDWD_DEV void elem(int64_t j, double (&a)[NR]) const {
    const double wj = K.w[j], dj = wj - K.u[j];
    a[0] += dj * dj;
    a[1] += wj * wj;
  }
  GDWD_DEV void fin(const double (&a)[NR]) const {
    K.out[11] = a[0];
    K.out[12] = a[1];
  }
};

// scores = beta + X^T w and the train-error count y sgn(score) <= 0
// (solver.py:610-642; np.sign(0) = 0 counts as wrong, NaN never does)
struct OpScore {
  static constexpr int NN = 1;
  static constexpr bool HAS_FIN = true;
  const double* w;
  double beta;
  const double* y;  // nullable
  double* out;      // nullable
  double* wrong;    // device scalar (count as a double: exact below 2^53)
  GDWD_DEV bool skip() const { return false; }
  GDWD_DEV double wval(int64_t j) const { return w[j]; }
  GDWD_DEV void row(int64_t i, double dot, double (&na)[NN]) const {
    const double s = beta + dot;
    if (out) out[i] = s;
    if (y) {
      const double sg = s > 0.0 ? 1.0 : (s < 0.0 ? -1.0 : s);  // np.sign (0 and NaN pass through)
      na[0] += (y[i] * sg <= 0.0) ? 1.0 : 0.0;
    }
  }
  GDWD_DEV void fin(const double (&ns)[NN]) const { *wrong = ns[0]; }
};

struct OpJyG {  // jy = G^{-1} (y/|y|) ; ys = 1 + (y/|y|).jy - 1  (subsolvers.py:114-117)
  static constexpr int NN = 1;
  static constexpr bool HAS_FIN = true;
  const double* y;
  double ynorm;
  double* jy;
  Scal* S;
  GDWD_DEV bool skip() const { return false; }
  GDWD_DEV double wval(int64_t j) const { return y[j] / ynorm; }
  GDWD_DEV void row(int64_t i, double dot, double (&na)[NN]) const {
    jy[i] = dot;
    na[0] += (y[i] / ynorm) * dot;
  }
  GDWD_DEV void fin(const double (&ns)[NN]) const {
    S->ys = 1.0 + ns[0] - 1.0;
    S->yjy = ns[0];
  }
};

// out = M v (rows of an n x n Gram-space matrix), v[j] / vscale
struct OpGemvStore {
  static constexpr int NN = 1;
  static constexpr bool HAS_FIN = false;
  const double* v;
  double vscale;
  double* out;
  GDWD_DEV bool skip() const { return false; }
  GDWD_DEV double wval(int64_t j) const { return v[j] / vscale; }
  GDWD_DEV void row(int64_t i, double dot, double (&)[NN]) const { out[i] = dot; }
  GDWD_DEV void fin(const double (&)[NN]) const {}
};

struct OpNewtonSweep {  // standalone newton_r_sweep / newton_r (subsolvers.py:283-364)
  static constexpr int NR = 1;
  static constexpr bool HAS_FIN = false;
  const double *a, *w, *r0;
  double* out;
  int* iters;
  double sigma, q, tol;
  int max_newton, scalar_form;
  GDWD_DEV bool skip() const { return false; }
  GDWD_DEV void elem(int64_t i, double (&)[NR]) const {
    int it = 0;
    out[i] = newton_margin(a[i], sigma, q, w[i], r0[i], tol, max_newton, scalar_form & 1, &it);
    if (iters) iters[i] = it;
  }
  GDWD_DEV void fin(const double (&)[NR]) const {}
};

// the same sweep with one warp per coordinate (newton_margin_warp, the form
// the persistent Gram-space kernel uses)
__global__ void newton_warp_kernel(OpNewtonSweep op, int64_t n) {
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    int it = 0;
    const double r = newton_margin_warp(op.a[i], op.sigma, op.q, op.w[i], op.r0[i], op.tol, op.max_newton,
                                        op.scalar_form & 1, &it);
    if ((threadIdx.x & 31) == 0) {
      op.out[i] = r;
      if (op.iters) op.iters[i] = it;
    }
  }
}

}  // namespace gdwd
