// Persistent cooperative kernel for the Gram-space SMW2 iteration, three
// grid barriers per iteration (two with use_sgs = False).
//
// Same iteration as persist.cuh (reference solver.py:493-555 with the SMW
// solve of subsolvers.py:127-151, every d-vector carried as n coefficients
// over the Gram K = Z~^T Z~), re-associated so that only two row sweeps
// remain.  With G = I + K/mu^2, GK = G^{-1} K = mu^2 (I - G^{-1}) and
// K GK = mu^2 (K - GK), the products the 4-barrier kernel sweeps for follow
// from those it already has:
//   * x_bar = t1 - v/mu^2 with v = GK t1 + c' jy  (t1 = c_h/mu^2,
//     c' = t2 |y| - coef, jy = G^{-1} y/|y|), so
//       ztw_bar = K x_bar = GK t1 - c' kap/mu^2,       kap = K jy   (fixed);
//   * coef needs ybar^T g = gam^T t1 + t2 |y| ybar^T jy, gam = GK ybar
//     (fixed, GK symmetric): a local dot over the staged t1, so the Newton
//     prox (Step 1b) runs in the same phase as the first sweep;
//   * the re-solved w = (h + dr)/mu^2 - v'/mu^2 has
//       K w = GK t1 + GK dr/mu^2 - c'' kap/mu^2         (c'' = t2' |y| - coef');
//   * K g = K w - K rho/(sigma mu), K (w - g) = K rho/(sigma mu); K rho of
//     the own rows is swept once per launch and then follows rho's update
//     by linearity (K rho -= tau sigma mu (K w - K u), K u = s K g).
// Phases of iteration k:
//   A  stage u, rho (k-1 commit), c_h, t1; local sums -> coef, beta_bar;
//      rows: [K alpha ; GK t1] -> ztw_bar, x_bar, Newton r+, dr
//   -- barrier 1: alpha^T K alpha (finish k-1: dual objective, stop test), y.dr
//   D  stage c_res = h2 - A x_bar, dr/mu^2;  rows: [K c_res ; GK dr/mu^2]
//   -- barrier 2: c_res^T K c_res (reuse test), ybar.g', y.g'
//   H  (no sweep) w, ztw = K w, g, norms' row terms, Step 3, KKT sample terms
//   -- barrier 3: 14 sums -> ||g||, ||w - u||, ||w||, eta, sigma rule
// Rounding differs from the 4-barrier association (not bitwise equal to it);
// parity is to the reference's trajectories at the same tolerances.
#pragma once
#include "persist.cuh"

namespace gdwd {

constexpr int PK3_MAXR = PK_MAX_OWN;  // owned rows per CTA (host: n <= PK_MAX_OWN * grid)

// One warp: row a (length n) against NA staged vectors and row b against NB,
// both rows streamed together (8 double2 loads of each in flight per lane,
// predicated at the ragged end; pad columns are zero), two FMA chains per
// right-hand side, butterfly sums (every lane ends with the same values).
template <int NA, int NB>
GDWD_DEV void pk_row_dot_ab(const double* ra, const double* const (&xa)[NA], const double* rb,
                            const double* const (&xb)[NB], int64_t n, double (&oa)[NA], double (&ob)[NB]) {
  const int lane = threadIdx.x & 31;
  double a0[NA + NB], a1[NA + NB];
#pragma unroll
  for (int v = 0; v < NA + NB; ++v) a0[v] = a1[v] = 0.0;
  constexpr int U = 8;
  for (int64_t j0 = 2 * lane; j0 < n + 2 * lane; j0 += U * 64) {
    double2 za[U], zb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * 64;
      za[u] = j < n ? __ldg(reinterpret_cast<const double2*>(ra + j)) : make_double2(0.0, 0.0);
      zb[u] = j < n ? __ldg(reinterpret_cast<const double2*>(rb + j)) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * 64;
      const bool ok = j < n;
#pragma unroll
      for (int v = 0; v < NA; ++v) {
        const double2 x = ok ? *reinterpret_cast<const double2*>(xa[v] + j) : make_double2(0.0, 0.0);
        a0[v] = __fma_rn(za[u].x, x.x, a0[v]);
        a1[v] = __fma_rn(za[u].y, x.y, a1[v]);
      }
#pragma unroll
      for (int v = 0; v < NB; ++v) {
        const double2 x = ok ? *reinterpret_cast<const double2*>(xb[v] + j) : make_double2(0.0, 0.0);
        a0[NA + v] = __fma_rn(zb[u].x, x.x, a0[NA + v]);
        a1[NA + v] = __fma_rn(zb[u].y, x.y, a1[NA + v]);
      }
    }
  }
#pragma unroll
  for (int v = 0; v < NA + NB; ++v) a0[v] += a1[v];
  warp_sum<NA + NB>(a0);
#pragma unroll
  for (int v = 0; v < NA; ++v) oa[v] = a0[v];
#pragma unroll
  for (int v = 0; v < NB; ++v) ob[v] = a0[NA + v];
}


// ---------------------------------------------------------------------------
// Tensor memory as a resident store for the CTA's own Gram rows.  TMEM is 128
// lanes x 512 columns x 32 bit per SM and a warp reaches only its lane
// quarter (warp % 4), so warp w keeps its row (r = w, at most 16 rows per CTA)
// in quarter w % 4, row block w / 4.  Lane l holds the row's columns
// 2l + 64u, 2l + 64u + 1 (u < U = ceil(n/64)) as 4 words per chunk u -- the
// same distribution the L2 row dot uses, so a 32x32b load of 32 words hands
// each lane 8 chunks.  Reads run at ~400 B/cycle/SM (profiles/probes/
// tmem_probe.cu) against ~110 B/cycle/SM from L2.
// ---------------------------------------------------------------------------
GDWD_DEV void tm_ld32(uint32_t addr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
}
GDWD_DEV void tm_ld16(uint32_t addr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(addr));
}
GDWD_DEV void tm_st4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
GDWD_DEV void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
GDWD_DEV void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// copy row `row` (length n, zero beyond n) into this warp's TMEM block at `addr`
// Row into TMEM, 16 chunks' loads in flight per batch (one L2 round trip per
// batch, not per chunk).  With x != nullptr it also returns row . x in
// pk_row_dot<1>'s order (the same chunks, FMA chains and butterfly), so the
// launch's K rho needs no second pass over the row.
GDWD_DEV double tm_put_row(uint32_t addr, const double* row, int64_t n, const double* x = nullptr) {
  const int lane = threadIdx.x & 31;
  const int U = (int)((n + 63) / 64);
  constexpr int B = 16;
  double a0 = 0.0, a1 = 0.0;
  for (int u0 = 0; u0 < U; u0 += B) {
    double2 z[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int64_t j = 2 * lane + 64 * (int64_t)(u0 + u);
      z[u] = j < n ? __ldg(reinterpret_cast<const double2*>(row + j)) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      if (u0 + u < U)
        tm_st4(addr + 4 * (u0 + u), __double2loint(z[u].x), __double2hiint(z[u].x), __double2loint(z[u].y),
               __double2hiint(z[u].y));
      if (x) {
        const int64_t j = 2 * lane + 64 * (int64_t)(u0 + u);
        const double2 xv = j < n ? *reinterpret_cast<const double2*>(x + j) : make_double2(0.0, 0.0);
        a0 = __fma_rn(z[u].x, xv.x, a0);
        a1 = __fma_rn(z[u].y, xv.y, a1);
      }
    }
  }
  tm_wait_st();
  double v[1] = {a0 + a1};
  if (x) warp_sum<1>(v);
  return v[0];
}

// Row a from TMEM against NA staged vectors, row b against NB staged vectors
// with b from TMEM (B_TM) or streamed from L2; same chunk order, FMA chains
// and butterfly as pk_row_dot_ab.
template <int NA, int NB, bool B_TM>
GDWD_DEV void pk_row_dot_tm(uint32_t ta, const double* const (&xa)[NA], uint32_t tb, const double* rb,
                            const double* const (&xb)[NB], int64_t n, double (&oa)[NA], double (&ob)[NB]) {
  const int lane = threadIdx.x & 31;
  double a0[NA + NB], a1[NA + NB];
#pragma unroll
  for (int v = 0; v < NA + NB; ++v) a0[v] = a1[v] = 0.0;
  const int U = (int)((n + 63) / 64);
  // B from L2: 16 chunks (16 double2 loads per lane) in flight per batch --
  // the row's latency is its number of L2 round trips; A (and B_TM) from
  // TMEM in 8-chunk loads inside the batch
  constexpr int UB = B_TM ? 8 : 16;
  for (int u0 = 0; u0 < U; u0 += UB) {
    double2 zb[B_TM ? 1 : UB];
    if constexpr (!B_TM) {
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int64_t j = 2 * lane + 64 * (int64_t)(u0 + u);
        zb[u] = j < n ? __ldg(reinterpret_cast<const double2*>(rb + j)) : make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int h = 0; h < UB / 4; ++h) {  // TMEM words of 4 chunks at a time (register budget)
      if (u0 + 4 * h >= U) break;        // warp-uniform: never address past the row block
      uint32_t wa[16], wb[B_TM ? 16 : 1];
      tm_ld16(ta + 4 * (u0 + 4 * h), wa);
      if constexpr (B_TM) tm_ld16(tb + 4 * (u0 + 4 * h), wb);
      tm_wait_ld();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j = 2 * lane + 64 * (int64_t)(u0 + 4 * h + u);
        const bool ok = j < n;
        // chunks past the row (>= U) read a neighbouring block: zero them
        const double kx = ok ? __hiloint2double(wa[4 * u + 1], wa[4 * u]) : 0.0;
        const double ky = ok ? __hiloint2double(wa[4 * u + 3], wa[4 * u + 2]) : 0.0;
#pragma unroll
        for (int v = 0; v < NA; ++v) {
          const double2 x = ok ? *reinterpret_cast<const double2*>(xa[v] + j) : make_double2(0.0, 0.0);
          a0[v] = __fma_rn(kx, x.x, a0[v]);
          a1[v] = __fma_rn(ky, x.y, a1[v]);
        }
        double gx, gy;
        if constexpr (B_TM) {
          gx = ok ? __hiloint2double(wb[4 * u + 1], wb[4 * u]) : 0.0;
          gy = ok ? __hiloint2double(wb[4 * u + 3], wb[4 * u + 2]) : 0.0;
        } else {
          gx = zb[4 * h + u].x;
          gy = zb[4 * h + u].y;
        }
#pragma unroll
        for (int v = 0; v < NB; ++v) {
          const double2 x = ok ? *reinterpret_cast<const double2*>(xb[v] + j) : make_double2(0.0, 0.0);
          a0[NA + v] = __fma_rn(gx, x.x, a0[NA + v]);
          a1[NA + v] = __fma_rn(gy, x.y, a1[NA + v]);
        }
      }
    }
  }
#pragma unroll
  for (int v = 0; v < NA + NB; ++v) a0[v] += a1[v];
  warp_sum<NA + NB>(a0);
#pragma unroll
  for (int v = 0; v < NA; ++v) oa[v] = a0[v];
#pragma unroll
  for (int v = 0; v < NB; ++v) ob[v] = a0[NA + v];
}

GDWD_DEV void tm_ld8(uint32_t addr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(addr));
}

// Row a from TMEM, row b streamed from L2 (K resident, GK not: n <= 2048).
// Per 8-chunk group: the group's 8 L2 loads of b are issued first, the TMEM
// words of a (one 32x32b.x32 load) and their FMAs run while they are in
// flight, then b is consumed (64 live registers, no spills).  Per-chain chunk
// order, FMA chains and butterfly are those of pk_row_dot_ab (bitwise the
// same sums).
template <int NA, int NB>
GDWD_DEV void pk_row_dot_tm1(uint32_t ta, const double* const (&xa)[NA], const double* rb,
                             const double* const (&xb)[NB], int64_t n, double (&oa)[NA], double (&ob)[NB]) {
  const int lane = threadIdx.x & 31;
  double a0[NA + NB], a1[NA + NB];
#pragma unroll
  for (int v = 0; v < NA + NB; ++v) a0[v] = a1[v] = 0.0;
  const int U = (int)((n + 63) / 64);
#pragma unroll 1
  for (int u0 = 0; u0 < U; u0 += 8) {
    double2 zb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t j = 2 * lane + 64 * (int64_t)(u0 + u);
      zb[u] = j < n ? __ldg(reinterpret_cast<const double2*>(rb + j)) : make_double2(0.0, 0.0);
    }
    uint32_t wa[32];
    tm_ld32(ta + 4 * u0, wa);  // past U: a neighbouring block (inside the allocation), zeroed below
    tm_wait_ld();
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t j = 2 * lane + 64 * (int64_t)(u0 + u);
      const bool ok = j < n;
      const double kx = ok ? __hiloint2double(wa[4 * u + 1], wa[4 * u]) : 0.0;
      const double ky = ok ? __hiloint2double(wa[4 * u + 3], wa[4 * u + 2]) : 0.0;
#pragma unroll
      for (int v = 0; v < NA; ++v) {
        const double2 x = ok ? *reinterpret_cast<const double2*>(xa[v] + j) : make_double2(0.0, 0.0);
        a0[v] = __fma_rn(kx, x.x, a0[v]);
        a1[v] = __fma_rn(ky, x.y, a1[v]);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t j = 2 * lane + 64 * (int64_t)(u0 + u);
      const bool ok = j < n;
#pragma unroll
      for (int v = 0; v < NB; ++v) {
        const double2 x = ok ? *reinterpret_cast<const double2*>(xb[v] + j) : make_double2(0.0, 0.0);
        a0[NA + v] = __fma_rn(zb[u].x, x.x, a0[NA + v]);
        a1[NA + v] = __fma_rn(zb[u].y, x.y, a1[NA + v]);
      }
    }
  }
#pragma unroll
  for (int v = 0; v < NA + NB; ++v) a0[v] += a1[v];
  warp_sum<NA + NB>(a0);
#pragma unroll
  for (int v = 0; v < NA; ++v) oa[v] = a0[v];
#pragma unroll
  for (int v = 0; v < NB; ++v) ob[v] = a0[NA + v];
}

struct PK3Args {
  Dev D;
  const double* K;    // n x ld
  const double* GK;   // G^{-1} K = mu^2 (I - G^{-1}), n x ld
  const double* kap;  // K jy
  const double* gam;  // GK (y/|y|)
  int64_t ld;
  double* part;  // [2][PK_NPART][gridDim]
  int count;
  int diag;  // 1 = skip the row sweeps (barrier / staging floor)
  unsigned long long* tstamp;
  int use_sgs;
  unsigned* ctr;  // grid barrier counter, zero at launch (null: cooperative-groups grid.sync)
};

template <int TM>  // own rows in TMEM: 0 none, 1 K, 2 K and GK (host picks by n)
__global__ void __launch_bounds__(PK_THREADS, 1) gram_smw_persistent3(PK3Args A) {
  const unsigned long long pk_entry = pk_now();
  cg::grid_group grid = cg::this_grid();
  const Dev& D = A.D;
  const int64_t n = D.n;
  extern __shared__ double pksm[];
  const int64_t ns = (n + 3) / 2 * 2;  // slot stride: > n, even (16-byte aligned double2 reads)
  // exchange slots (bulk-copied): A: xi r alpha x ; D: dr x_bar ztw_bar, c_res (staged)
  double* const s0 = pksm;
  double* const s1 = pksm + ns;
  double* const s2 = pksm + 2 * ns;
  double* const s3 = pksm + 3 * ns;
  double* const st1 = pksm + 4 * ns;  // A: t1 ; D: dr/mu^2
  // resident for the launch: y, jy, gam, u, rho, c_h
  double* const sy = pksm + 5 * ns;
  double* const sjy = pksm + 6 * ns;
  double* const sgam = pksm + 7 * ns;
  double* const su = pksm + 8 * ns;
  double* const srho = pksm + 9 * ns;
  double* const sh = pksm + 10 * ns;
  __shared__ unsigned long long bar;
  __shared__ double red[PK_WARPS * PK_NPART];
  __shared__ PKS S;
  // owned rows (r = i - i0): values carried between the phases of an iteration
  __shared__ double o_al[PK3_MAXR], o_s1[PK3_MAXR], o_ztwb[PK3_MAXR], o_xb[PK3_MAXR], o_rn[PK3_MAXR],
      o_dr[PK3_MAXR], o_krho[PK3_MAXR], o_gdr[PK3_MAXR], o_gp[PK3_MAXR], o_kw[PK3_MAXR], o_kg[PK3_MAXR];
  __shared__ double ot_e[PK3_MAXR], ot_wl[PK3_MAXR], ot_pw[PK3_MAXR];  // Step 3 operands, w^(1/(q+1))
  __shared__ double sc_scal[8];  // scalar results of side-by-side chains
  unsigned parity = 0;
  const unsigned vbytes = (unsigned)(((n + 1) / 2 * 2) * sizeof(double));
  auto issue = [&](int cnt, const double* const* src, double* const* dst) {
    if (threadIdx.x == PK_THREADS - 32) {
      asm volatile("fence.proxy.async;" ::: "memory");  // generic writes (global sources, reused slots)
      mbar_arrive_expect_tx(&bar, cnt * vbytes);
      for (int v = 0; v < cnt; ++v) bulk_g2s(dst[v], src[v], vbytes, &bar);
    }
  };
  auto wait_in = [&]() {
    mbar_wait(&bar, parity);
    parity ^= 1;
  };
  auto issue_a = [&]() {
    const double* src[4] = {D.xi, D.r, D.al, D.x};
    double* dst[4] = {s0, s1, s2, s3};
    issue(4, src, dst);
  };
  // Grid barrier: one release-add per CTA on a counter that only grows, then
  // an acquire poll for this barrier's target (bar.sync before and after
  // carries the ordering to and from the CTA's other threads); no fence.sc.
  // the counter only grows: this launch starts where the previous one of the
  // solve left it (no reset between launches)
  unsigned bar_target = A.ctr ? D.S->pk_bar : 0u;
  auto pk_bar = [&]() {
    if (!A.ctr) {
      grid.sync();
      return;
    }
    __syncthreads();
    bar_target += gridDim.x;
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(A.ctr) : "memory");
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(A.ctr) : "memory");
      } while ((int)(v - bar_target) < 0);
    }
    __syncthreads();
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i0 = n * blockIdx.x / gridDim.x, i1 = n * (blockIdx.x + 1) / gridDim.x;
  const int nrows = (int)(i1 - i0);
  const int nsweep = A.diag == 1 ? 0 : nrows;
  const double mu = D.mu, mu2 = D.mu2, yty = D.yty, ynorm = D.ynorm;
  const bool mu2_one = mu2 == 1.0;  // x / 1.0 == x exactly: skip the division
  const double ys = D.S->ys, yjy = D.S->yjy;  // yjy: (y/|y|)^T jy
  int slot = 0;

  if (threadIdx.x == 0) {
    const Scal* G = D.S;
    S.k = G->k; S.stopped = G->stopped; S.converged = G->converged; S.reuse = G->reuse; S.pending = 0;
    S.gnorm = G->gnorm;
    S.double_count = G->double_count; S.iters_done = G->iters_done; S.error = G->error;
    S.sigma = G->sigma; S.sigma_next = G->sigma_next; S.sdual = G->sdual;
    for (int f = 0; f < 11; ++f) S.eta[f] = G->eta[f];
    for (int v = 0; v < 11; ++v) pksm[v * ns + n] = 0.0;  // odd-tail pads read as zeros
    mbar_init(&bar, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  {
    const double* src[5] = {D.y, D.jy, A.gam, D.u, D.rho};
    double* dst[5] = {sy, sjy, sgam, su, srho};
    issue(5, src, dst);
    wait_in();
    if (threadIdx.x == 0) srho[n] = 0.0;  // bulk copies of odd n bring the pad slot along
  }
  // own Gram rows into tensor memory (once per launch)
  __shared__ uint32_t tm_base;
  uint32_t tmK = 0, tmG = 0;
  if (TM) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tm_base)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t blk = 4u * (uint32_t)((n + 63) / 64) * (uint32_t)TM;  // columns per row block
    tmK = tm_base + ((uint32_t)(32 * (warp & 3)) << 16) + blk * (uint32_t)(warp >> 2);
    tmG = tmK + blk / 2;
    if (warp < nsweep) {
      // K rho of the own rows with the TMEM load (see below)
      const double kr = tm_put_row(tmK, A.K + (i0 + warp) * A.ld, n, srho);
      if (lane == 0) o_krho[warp] = kr;
      if (TM == 2) tm_put_row(tmG, A.GK + (i0 + warp) * A.ld, n);
    }
  }
  // K rho of the own rows, swept once per launch (u, rho may have been
  // advanced outside this kernel); within the launch it follows rho's update
  // by linearity: K rho -= tau sigma mu (K w - K u), K u = s K g
  for (int r = TM ? nsweep : warp; r < nsweep; r += PK_WARPS) {
    const double* rows[1] = {A.K + (i0 + r) * A.ld};
    const double* xs[1] = {srho};
    double o[1];
    pk_row_dot<1>(rows, n, xs, o);
    if (lane == 0) o_krho[r] = o[0];
  }
  // Step 3 operands that do not change during the solve
  if (warp == 0 && lane < nrows) {
    ot_e[lane] = D.e[i0 + lane];
    ot_wl[lane] = D.wl[i0 + lane];
    ot_pw[lane] = np_pow(D.wl[i0 + lane], D.e1);
  }
  const int k_end = S.k + A.count;
  const int k_begin = S.k;
  if (A.tstamp && threadIdx.x == 0) {
    A.tstamp[(size_t)blockIdx.x * 32 + 27] = pk_entry;
    A.tstamp[(size_t)blockIdx.x * 32 + 28] = pk_now();
  }
#define PK3_TS(pt)                                                                         \
  do {                                                                                     \
    if (A.tstamp && threadIdx.x == 0 && S.k - k_begin < PK_TS_ITERS)                       \
      A.tstamp[((size_t)(S.k - k_begin) * gridDim.x + blockIdx.x) * 32 + (pt)] = pk_now(); \
  } while (0)
  issue_a();
  for (;;) {
    if (S.stopped || S.k >= k_end) {
      wait_in();
      break;
    }
    const int k = S.k;
    const double eps = D.eps_tab[k], tol = D.tol_tab[k];
    PK3_TS(0);
    const bool pending = S.pending != 0;
    const double sig = S.sigma_next;  // sigma of iteration k (committed after barrier 1)
    double h2bot_l = 0.0;             // h2's scalar slot (every thread, after barrier 1)
    // ------------- phase A: u, rho (k-1); c_h, t1; sweep [K alpha, K rho ; GK t1]; Newton ----
    {
      const double sp = S.sigma_pend, gn = S.gnorm;
      double yr = 0.0, gt = 0.0;
      wait_in();  // xi r alpha x
      if (threadIdx.x == 0) s2[n] = 0.0;  // alpha is swept: zero pad (synced by block_sum)
      PK3_TS(1);
      // 4 independent elements per thread, predicated (no early exit), so
      // their division chains overlap; uniform factors computed once
      // rho / (sigma mu) on coefficients (not an elementwise quantity of the
      // reference, whose rho is a d-vector): one reciprocal, a multiply each
      const double spmu = sp * mu, ispmu = 1.0 / spmu, tsm = (D.tau * sp) * mu, mus = mu / sig;
      const bool proj = !(gn <= D.zscale);
      const double zsg = proj ? D.zscale / gn : 1.0;
#pragma unroll 1
      for (int64_t j0 = threadIdx.x; j0 < n; j0 += 4 * PK_THREADS) {
        double rhs[4], t1[4], ch[4], uu[4], rr[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t j = j0 + u * PK_THREADS < n ? j0 + u * PK_THREADS : j0;
          double uj = su[j], rj = srho[j];
          if (pending) {  // Step 2 of iteration k-1 (solver.py:535-542)
            const double wj = s3[j];
            const double gj = wj - rj * ispmu;
            uj = proj ? zsg * gj : gj;
            rj = rj - tsm * (wj - uj);
          }
          rhs[u] = (s0[j] - s1[j]) - s2[j] / sig;
          ch[u] = (-rhs[u] + mu2 * uj) + mus * rj;
          t1[u] = mu2_one ? ch[u] : ch[u] / mu2;
          uu[u] = uj;
          rr[u] = rj;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t j = j0 + u * PK_THREADS;
          if (j < n) {
            if (pending) {
              su[j] = uu[u];
              srho[j] = rr[u];
            }
            sh[j] = ch[u];
            st1[j] = t1[u];
            yr += sy[j] * rhs[u];
            gt += sgam[j] * t1[u];
          }
        }
      }
      if (pending && warp == 0 && lane < nsweep) {  // K rho of the own rows, same update
        const double kgr = o_kg[lane];
        const double kur = proj ? zsg * kgr : kgr;
        o_krho[lane] = o_krho[lane] - tsm * (o_kw[lane] - kur);
      }
      PK3_TS(2);
      double v2[2] = {yr, gt};
      block_sum<2>(v2, red);
      if (threadIdx.x == 0) {
        // SMW solve scalars (subsolvers.py:138-151) from the local sums
        const double hbot = -v2[0];
        const double t2 = hbot / yty;
        const double s2 = ynorm * t2;
        const double ybg = v2[1] + t2 * (ynorm * yjy);  // ybar^T g
        const double coef = (ybg + (-s2)) / ys;
        const double yv = ynorm * (ybg - coef * yjy);   // y^T v
        const double vn = (-s2) - coef * (-1.0);
        const double p2 = yv + ynorm * vn;
        S.hbot = hbot;
        S.s2 = s2;
        S.coef = coef;
        S.beta_b = hbot / yty - p2 / yty;
        S.cp = t2 * ynorm - coef;  // c'
        S.pending = 0;
      }
      __syncthreads();
      PK3_TS(3);
      const double t2 = S.hbot / yty, coef = S.coef, cp = S.cp, bb = S.beta_b;
      double qa = 0.0, ydr = 0.0;
      for (int r = warp; r < nsweep; r += PK_WARPS) {
        const int64_t i = i0 + r;
        const double* Ki = A.K + i * A.ld;
        const double* GKi = A.GK + i * A.ld;
        const double xii = s0[i], ri = s1[i], ali = s2[i], wli = D.wl[i], kapi = A.kap[i];
        const double yi = sy[i], jyi = sjy[i], hi = sh[i];
        double oK[1], oG[1];
        {
          const double* xa[1] = {s2};
          const double* xg[1] = {st1};
          if (TM == 2) pk_row_dot_tm<1, 1, true>(tmK, xa, tmG, GKi, xg, n, oK, oG);
          else if (TM) pk_row_dot_tm1<1, 1>(tmK, xa, GKi, xg, n, oK, oG);
          else pk_row_dot_ab<1, 1>(Ki, xa, GKi, xg, n, oK, oG);  // K alpha, GK t1
        }
        // every lane holds the same sums (butterfly), so all lanes run Newton
        const double s1i = oG[0];
        const double gi = s1i + t2 * (ynorm * jyi);
        const double vi = gi - coef * jyi;
        const double xbi = mu2_one ? hi - vi : hi / mu2 - vi / mu2;
        const double ztwbi = mu2_one ? s1i - cp * kapi : s1i - (cp * kapi) / mu2;
        const double a = ((ztwbi + yi * bb) + xii) - ali / sig;
        double rn;
        if (A.diag == 2) rn = ri + 1e-3 * a;  // diagnostics: no Newton solve
        else if (A.diag == 3) rn = __shfl_sync(0xffffffffu, lane == 0 ? newton_margin(a, sig, D.q, wli, ri, tol) : 0.0, 0);
        else rn = newton_margin_warp(a, sig, D.q, wli, ri, tol);
        const double dri = rn - ri;
        if (lane == 0) {
          qa += ali * oK[0];
          ydr += yi * dri;
          D.dr[i] = dri;
          D.xb[i] = xbi;
          D.ztwb[i] = ztwbi;
          o_al[r] = ali;
          o_s1[r] = s1i;
          o_ztwb[r] = ztwbi;
          o_xb[r] = xbi;
          o_rn[r] = rn;
          o_dr[r] = dri;
        }
      }
      PK3_TS(4);
      double pv[2] = {qa, ydr};
      pk_write_lane0<2>(A.part, slot, pv, red);
      PK3_TS(5);
      pk_bar();
      if (A.use_sgs) {  // phase D inputs
        const double* src[3] = {D.dr, D.xb, D.ztwb};
        double* dst[3] = {s0, s1, s2};
        issue(3, src, dst);
      }
      double tot[2];
      pk_cross_sum<2>(A.part, slot, tot, red);
      slot ^= 1;
      PK3_TS(6);
      h2bot_l = S.hbot + tot[1];
      // thread 0 finishes iteration k-1 while the other warps start phase D;
      // the stop decision is read after D's first block barrier (phase D
      // writes only per-iteration scratch before then)
      if (threadIdx.x == 0) {
        S.h2bot = h2bot_l;
        if (blockIdx.x == 0) {
          D.h[D.bot] = S.hbot;
          D.xb[D.bot] = S.beta_b;
        }
        // finish iteration k-1 (solver.py:293-304,334,548-555)
        if (k > 0) {
          const double od = D.kappa * S.sdual - D.zscale * sqrt(tot[0]);
          const double op = S.eta[9];
          const double gap = fabs(op - od) / (1.0 + fabs(op) + fabs(od));
          S.eta[10] = od;
          S.eta[8] = gap;
          if (blockIdx.x == 0) {
            double* hr = D.hist + (int64_t)(k - 1) * HIST_W;
            hr[H_OBJD] = od;
            hr[H_GAP] = gap;
          }
          const double ep = fmax(fmax(S.eta[3], S.eta[4]), S.eta[5]);
          const double ed = fmax(S.eta[6], S.eta[7]);
          const double ec = fmax(fmax(S.eta[0], S.eta[1]), S.eta[2]);
          if (fmax(ep, ed) < D.tol_feas && fmin(ec, gap) < D.tol_cgap && fmax(ec, gap) < D.tol_cap) {
            S.stopped = 1;
            S.converged = 1;
          }
        }
        if (!S.stopped && k >= D.max_iter) S.stopped = 1;
        if (!S.stopped) {
          S.sigma = S.sigma_next;
          if (blockIdx.x == 0) {
            double* hr = D.hist + (int64_t)k * HIST_W;
            hr[H_SIGMA] = S.sigma;
            hr[H_EPS] = D.eps_tab[k];
            hr[H_REUSE] = 1.0;
            hr[H_PSQMR] = 0.0;
          }
        }
      }
    }
    // ---------------- phase D: Step 1c residual, speculative re-solve -------------
    if (A.use_sgs) {
      const double bb = S.beta_b;
      const double t2 = h2bot_l / yty;
      double ytz = 0.0;
      wait_in();  // dr x_bar ztw_bar
      if (threadIdx.x == 0) s0[n] = s3[n] = 0.0;  // swept vectors: zero pads (synced by block_sum)
      PK3_TS(7);
#pragma unroll 1
      for (int64_t j0 = threadIdx.x; j0 < n; j0 += 4 * PK_THREADS) {
        double cr[4], dm[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t j = j0 + u * PK_THREADS < n ? j0 + u * PK_THREADS : j0;
          const double drj = s0[j];
          const double h2 = sh[j] + drj;
          const double ax = (s2[j] + mu2 * s1[j]) + sy[j] * bb;
          cr[u] = h2 - ax;  // c_res
          dm[u] = mu2_one ? drj : drj / mu2;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t j = j0 + u * PK_THREADS;
          if (j < n) {
            s3[j] = cr[u];
            if (!mu2_one) st1[j] = dm[u];
            ytz += sy[j] * s2[j];
          }
        }
      }
      double v1[1] = {ytz};
      block_sum<1>(v1, red);
      if (threadIdx.x == 0) S.ytzw = v1[0];
      __syncthreads();
      if (S.stopped) break;  // iteration k-1 was the last (decided after barrier 1)
      PK3_TS(8);
      const double* sdr = mu2_one ? s0 : st1;
      double q = 0.0, syg = 0.0, yg = 0.0;
      for (int r = warp; r < nsweep; r += PK_WARPS) {
        const int64_t i = i0 + r;
        const double* rows[2] = {A.K + i * A.ld, A.GK + i * A.ld};
        const double* xs[2] = {s3, sdr};
        const double s1i = o_s1[r], jyi = sjy[i], yi = sy[i];
        double o[2];
        if (TM) {
          const double* xa1[1] = {s3};
          const double* xb1[1] = {sdr};
          double oa[1], ob[1];
          if (TM == 2) pk_row_dot_tm<1, 1, true>(tmK, xa1, tmG, rows[1], xb1, n, oa, ob);
          else pk_row_dot_tm1<1, 1>(tmK, xa1, rows[1], xb1, n, oa, ob);
          o[0] = oa[0];
          o[1] = ob[0];
        } else {
          pk_row_dot<2>(rows, n, xs, o);
        }
        if (lane == 0) {
          q += s3[i] * o[0];
          const double gpi = (s1i + o[1]) + t2 * (ynorm * jyi);
          o_gdr[r] = o[1];
          o_gp[r] = gpi;
          syg += (yi / ynorm) * gpi;
          yg += yi * gpi;
        }
      }
      PK3_TS(9);
      double pv[3] = {q, syg, yg};
      pk_write_lane0<3>(A.part, slot, pv, red);
      PK3_TS(10);
      pk_bar();
      double t[3];
      pk_cross_sum<3>(A.part, slot, t, red);
      slot ^= 1;
      PK3_TS(11);
      // the reuse test (warp 0) and the re-solve's scalars (warp 1,
      // speculatively) are independent chains: run them side by side
      if (threadIdx.x == 0) {
        const double rb = S.h2bot - (S.ytzw + yty * bb);
        const double rr = hypot(sqrt(t[0] > 0.0 ? t[0] : 0.0), rb);
        S.reuse = rr <= 5.0 * eps;
      } else if (threadIdx.x == 32) {
        const double s2 = ynorm * t2;
        const double coef = (t[1] + (-s2)) / ys;
        const double yv = t[2] - coef * (ynorm * yjy);
        const double vn = (-s2) - coef * (-1.0);
        const double p2 = yv + ynorm * vn;
        sc_scal[0] = coef;
        sc_scal[1] = t2 * ynorm - coef;  // c''
        sc_scal[2] = S.h2bot / yty - p2 / yty;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        if (S.reuse) {
          S.beta = bb;
        } else {
          S.double_count += 1;
          S.coef = sc_scal[0];
          S.cp = sc_scal[1];
          S.beta = sc_scal[2];
        }
        if (blockIdx.x == 0) {
          D.hist[(int64_t)k * HIST_W + H_REUSE] = S.reuse ? 1.0 : 0.0;
          D.x[D.bot] = S.beta;
        }
      }
      __syncthreads();
    } else {
      __syncthreads();
      if (S.stopped) break;
      if (threadIdx.x == 0) {
        S.reuse = 1;
        S.beta = S.beta_b;
        if (blockIdx.x == 0) D.x[D.bot] = S.beta;
      }
      __syncthreads();
    }
    // ------------- phase H: w, ztw = K w, g; Step 3 and the KKT sample terms -------------
    {
      const bool reuse = S.reuse != 0;
      const double bet = S.beta, C = D.C, coef = S.coef, cpp = S.cp;
      double acc[PK_NPART];
#pragma unroll
      for (int f = 0; f < PK_NPART; ++f) acc[f] = 0.0;
      if (warp == 0 && lane < nrows) {  // one owned sample per lane
        const int r = lane;
        const int64_t i = i0 + r;
        double wi, kwi;
        if (reuse) {
          wi = o_xb[r];
          kwi = o_ztwb[r];
        } else {  // x = (h + dr)/mu^2 - v'/mu^2 (subsolvers.py:145-151)
          const double vi = o_gp[r] - coef * sjy[i];
          const double hd = sh[i] + o_dr[r];
          wi = mu2_one ? hd - vi : hd / mu2 - vi / mu2;
          const double kap = A.kap[i];
          kwi = (o_s1[r] + o_gdr[r]) - (mu2_one ? cpp * kap : (cpp * kap) / mu2);
        }
        const double isgmu = 1.0 / (sig * mu);
        const double gi = wi - srho[i] * isgmu;
        const double di = wi - gi;                     // w - u when u = g (no projection)
        const double kdi = o_krho[r] * isgmu;          // K (w - g)
        const double kgi = kwi - kdi;                  // K g
        o_kw[r] = kwi;
        o_kg[r] = kgi;
        acc[10] = gi * kgi;
        acc[11] = di * kdi;
        acc[12] = di * kgi;
        acc[13] = wi * kwi;
        D.x[i] = wi;
        D.ztw[i] = kwi;
        // Step 3 + KKT sample terms (solver.py:533,538-541,311-333; OpStep3)
        const double rr = o_rn[r];
        D.r[i] = rr;
        const double yi = sy[i], ei = ot_e[r], zt = kwi, ali = o_al[r];
        const double xv = np_max0((((rr - zt) - yi * bet) + ali / sig) - (C / sig) * ei);
        D.xi[i] = xv;
        const double pg = ((zt + yi * bet) + xv) - rr;
        const double an = ali - (D.tau * sig) * pg;
        D.al[i] = an;
        const double wl = ot_wl[r];
        const double s = (D.q * wl) / np_pow(rr, D.qp1);
        const double d2 = an - s;
        const double mn = np_min0(an);
        const double mx = np_max0(an - C * ei);
        acc[0] = yi * an;
        acc[1] = xv * (C * ei - an);
        acc[2] = d2 * d2;
        acc[3] = pg * pg;
        acc[4] = mn * mn;
        acc[5] = mx * mx;
        acc[6] = wl / np_pow(rr, D.q);
        acc[7] = ei * xv;
        acc[8] = ot_pw[r] * np_pow(np_max0(an), D.e2);
        acc[9] = (rr <= 0.0) ? 1.0 : 0.0;
      }
      PK3_TS(12);
      if (warp == 0) {
        warp_sum<PK_NPART>(acc);
        if (lane == 0) {
          double* p = A.part + (size_t)slot * gridDim.x * PK_NPART + blockIdx.x;
#pragma unroll
          for (int f = 0; f < PK_NPART; ++f) p[(size_t)f * gridDim.x] = acc[f];
        }
      }
      PK3_TS(13);
      pk_bar();
      issue_a();  // next iteration's phase A inputs
      double t[PK_NPART];
      pk_cross_sum<PK_NPART>(A.part, slot, t, red);
      slot ^= 1;
      PK3_TS(14);
      // the eight normalised residuals by lane 0 of warps 0-7 side by side
      // (one sqrt and one division each; warp 4 also forms ||g|| and ||w-u||)
      if (lane == 0 && warp < 8) {
        const double oc = D.one_c;
        double ev;
        switch (warp) {
          case 0: ev = fabs(t[0]) / oc; break;
          case 1: ev = fabs(t[1]) / oc; break;
          case 2: ev = t[2] / oc; break;
          case 3: ev = sqrt(t[3]) / oc; break;
          case 4: {
            const double gg = t[10] > 0.0 ? t[10] : 0.0;
            const double gn = sqrt(gg);
            double wu2;
            if (gn <= D.zscale) {
              wu2 = t[11] > 0.0 ? t[11] : 0.0;
            } else {  // w - u = d + (1 - s) g with s = z_scale / ||g||
              const double om = 1.0 - D.zscale / gn;
              const double v = t[11] + 2.0 * om * t[12] + om * om * gg;
              wu2 = v > 0.0 ? v : 0.0;
            }
            S.gnorm = gn;
            S.wu2 = wu2;
            ev = (D.mu * sqrt(wu2)) / oc;
            break;
          }
          case 5: ev = fmax(sqrt(t[13]) - D.zscale, 0.0) / oc; break;
          case 6: ev = sqrt(t[4]) / oc; break;
          default: ev = sqrt(t[5]) / oc; break;
        }
        sc_scal[warp] = ev;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        S.w2 = t[13];
        S.pending = 1;
        S.sigma_pend = S.sigma;
        if (t[9] > 0.0 && A.diag == 0) {
          S.error = 6;
          S.stopped = 1;
        } else {
          double* e = S.eta;
#pragma unroll
          for (int f = 0; f < 8; ++f) e[f] = sc_scal[f];
          e[9] = t[6] + D.C * t[7];
          S.sdual = t[8];
          if (blockIdx.x == 0) {
            double* hr = D.hist + (int64_t)k * HIST_W;
            for (int f = 0; f < 8; ++f) hr[f] = e[f];
            hr[H_OBJP] = e[9];
            hr[H_BETA] = S.beta;
          }
          const double ep = fmax(fmax(e[3], e[4]), e[5]);
          const double ed = fmax(e[6], e[7]);
          if (D.sched && k + 1 < D.sched_len) S.sigma_next = D.sched[k + 1];
          else S.sigma_next = sigma_rule(S.sigma, ep, ed);
          S.iters_done = k + 1;
          S.k = k + 1;
        }
      }
      __syncthreads();
    }
  }
  // the k-1 Step 2 update still pending at the end is applied to the owned
  // rows; owners write u, rho (resident here for the whole launch) back
  if (S.pending) {
    const double sp = S.sigma_pend, gn = S.gnorm;
    for (int64_t j = i0 + threadIdx.x; j < i1; j += PK_THREADS) {
      const double wj = D.x[j];
      const double gj = wj - srho[j] * (1.0 / (sp * mu));  // as in the staging loop
      const double uj = (gn <= D.zscale) ? gj : (D.zscale / gn) * gj;
      srho[j] = srho[j] - ((D.tau * sp) * mu) * (wj - uj);
      su[j] = uj;
    }
  }
  for (int64_t j = i0 + threadIdx.x; j < i1; j += PK_THREADS) {
    D.u[j] = su[j];
    D.rho[j] = srho[j];
  }
  __syncthreads();
  if (TM && warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm_base));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    Scal* G = D.S;
    G->k = S.k; G->stopped = S.stopped; G->converged = S.converged; G->reuse = S.reuse;
    G->double_count = S.double_count; G->iters_done = S.iters_done; G->error = S.error;
    G->sigma = S.sigma; G->sigma_next = S.sigma_next; G->sdual = S.sdual; G->gnorm = S.gnorm;
    G->wu2 = S.wu2; G->w2 = S.w2;
    for (int f = 0; f < 11; ++f) G->eta[f] = S.eta[f];
    G->pk_bar = bar_target;
  }
}
#undef PK3_TS

}  // namespace gdwd
