// Persistent cooperative Dormand-Prince 5(4) solver for ONE large system (mesolve / sesolve).
//
// One launch integrates the whole tlist: every CTA of a cooperative grid owns a contiguous
// slab of 32-row blocks; the six RHS evaluations of an attempt (integrator.hpp:91-102) are
// fused CSR SpMV passes whose epilogue forms the next stage input, the stage-7 pass also
// produces the embedded-error partials (integrator.hpp:105-116), and the accept/reject PI
// controller (integrator.hpp:119-145) runs redundantly — and identically — in every CTA after
// a deterministic grid reduction. Observations (evolve.cpp:160-165, 284-297) evaluate the
// Hairer dense output (integrator.hpp:127-131,150-154) lazily, only at the indices the e_ops
// touch, fused into the next attempt's first pass. No host round trip per step.
//
// Passes per attempt: 6 (stage 2 gathers y + h*a21*k1 on the fly), each followed by one grid
// barrier. See DESIGN.md §4 for the byte model.
#include <cstdio>

#include "engine.cuh"
#include "grid_engine.h"

namespace qsg {

namespace {

constexpr int kThreads = 512;

struct Pending {
  double theta;  // NaN: observe buffer Y directly
  int grid_idx;  // -1: save-only
  int save_idx;  // -1: no state save
};

struct Bufs {
  double2* b[11];
};

// logical buffer ids
enum { Y = 0, YO = 1, K1 = 2, K2 = 3, K3 = 4, K4 = 5, K5 = 6, K6 = 7, K7 = 8, SA = 9, SB = 10 };

__device__ __forceinline__ double2 dense_at(double2* const* B, const int* bi, int c, double theta,
                                            double h) {
  // integrator.hpp:127-131 (rc1..rc5) and :150-154 (evaluation), per element.
  // After an accepted step the FSAL swap (:138) put the step's k1 under the K7 label and its
  // k7 under the K1 label.
  const double2 yo = B[bi[YO]][c];
  if (isnan(theta)) return B[bi[Y]][c];
  const double2 y1 = B[bi[Y]][c];
  const double2 k1 = B[bi[K7]][c];
  const double2 k7 = B[bi[K1]][c];
  const double2 k3 = B[bi[K3]][c], k4 = B[bi[K4]][c], k5 = B[bi[K5]][c], k6 = B[bi[K6]][c];
  using namespace dp;
  const double th1 = 1.0 - theta;
  double2 rc2 = csub(y1, yo);
  double2 rc3 = csub(cscale(h, k1), rc2);
  double2 rc4 = csub(csub(rc2, cscale(h, k7)), rc3);
  double2 rc5;
  rc5.x = h * (d1 * k1.x + d3 * k3.x + d4 * k4.x + d5 * k5.x + d6 * k6.x + d7 * k7.x);
  rc5.y = h * (d1 * k1.y + d3 * k3.y + d4 * k4.y + d5 * k5.y + d6 * k6.y + d7 * k7.y);
  double2 o;
  o.x = yo.x + theta * (rc2.x + th1 * (rc3.x + theta * (rc4.x + th1 * rc5.x)));
  o.y = yo.y + theta * (rc2.y + th1 * (rc3.y + theta * (rc4.y + th1 * rc5.y)));
  return o;
}

// Observation pass for up to `np` pending events: expectation partials into reduction slots
// and state saves. ME: expect_e = sum_{(i,j) in A_e} A(i,j) * rho_h(j,i) with
// rho_h = (rho + rho^dag)/2 (evolve.cpp:286-295); SE: <psi|E psi> (evolve.cpp:341-345).
template <int MODE>
__device__ void observe_pass(const GridProblem& P, double2* const* B, const int* bi,
                             const Pending* pend, int np, double h_last, double* slots,
                             double* smem, int rank, int G) {
  const int gtid = rank * blockDim.x + threadIdx.x;
  const int gstride = G * blockDim.x;
  for (int e = 0; e < P.n_e; ++e) {
    for (int q = 0; q < np; ++q) {
      double2 acc = make_double2(0.0, 0.0);
      if (pend[q].grid_idx >= 0) {
        if (MODE == 0) {
          const int beg = P.eo_off[e], end = P.eo_off[e + 1];
          for (int p = beg + gtid; p < end; p += gstride) {
            const int i = P.eo_i[p], j = P.eo_j[p];
            // rho(j,i) = y[i*d + j], rho(i,j) = y[j*d + i]
            const double2 rji = dense_at(B, bi, i * P.d + j, pend[q].theta, h_last);
            const double2 rij = dense_at(B, bi, j * P.d + i, pend[q].theta, h_last);
            const double2 rh = cscale(0.5, cadd(rji, cconj(rij)));
            acc = cadd(acc, cmul(P.eo_v[p], rh));
          }
        } else {
          const int* rp = P.se_rowptr + static_cast<long long>(e) * (P.n + 1);
          const long long off = P.se_off[e];
          for (int r = gtid; r < P.n; r += gstride) {
            double2 ev = make_double2(0.0, 0.0);
            for (int p = rp[r]; p < rp[r + 1]; ++p)
              ev = cadd(ev, cmul(P.se_val[off + p], dense_at(B, bi, P.se_col[off + p], pend[q].theta, h_last)));
            const double2 g = dense_at(B, bi, r, pend[q].theta, h_last);
            acc = cadd(acc, cmul(cconj(g), ev));
          }
        }
      }
      const double sx = block_sum(acc.x, smem);
      const double sy = block_sum(acc.y, smem);
      if (threadIdx.x == 0) {
        const int s = 2 * (q * P.n_e + e);
        slots[static_cast<long long>(s) * G + rank] = sx;
        slots[static_cast<long long>(s + 1) * G + rank] = sy;
      }
    }
  }
  // state saves: every CTA writes its own rows
  for (int q = 0; q < np; ++q) {
    if (pend[q].save_idx < 0) continue;
    double2* out = P.states + static_cast<long long>(pend[q].save_idx) * P.n;
    for (int r = gtid; r < P.n; r += gstride) {
      if (MODE == 0) {
        const int i = r % P.d, j = r / P.d;
        const double2 a = dense_at(B, bi, r, pend[q].theta, h_last);          // rho(i,j)
        const double2 b = dense_at(B, bi, i * P.d + j, pend[q].theta, h_last);  // rho(j,i)
        out[r] = cscale(0.5, cadd(a, cconj(b)));
      } else {
        out[r] = dense_at(B, bi, r, pend[q].theta, h_last);
      }
    }
  }
}

// CTA 0 folds the observation slots (written before the last barrier) into expect[].
__device__ void observe_commit(const GridProblem& P, const Pending* pend, int np,
                               const double* slots, int G) {
  if (blockIdx.x != 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int nv = 2 * np * P.n_e;
  for (int s = warp; s < nv; s += nw) {
    double v = 0.0;
    for (int g = lane; g < G; g += 32) v += slots[static_cast<long long>(s) * G + g];
    v = warp_sum(v);
    if (lane == 0) {
      const int q = (s / 2) / P.n_e, e = (s / 2) % P.n_e;
      if (pend[q].grid_idx >= 0) {
        double* dst = reinterpret_cast<double*>(P.expect + static_cast<long long>(pend[q].grid_idx) * P.n_e + e);
        dst[s & 1] = v;
      }
    }
  }
  __syncthreads();  // s_pend is rewritten right after
}

// every CTA reads slot s (partials of all G CTAs) in the same order -> identical value
__device__ __forceinline__ double grid_value(const double* red, int s, int G, double* smem) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (warp == 0) {
    double v = 0.0;
    for (int g = lane; g < G; g += 32) v += red[static_cast<long long>(s) * G + g];
    v = warp_sum(v);
    if (lane == 0) smem[0] = v;
  }
  __syncthreads();
  return smem[0];
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) dp5_grid_kernel(const __grid_constant__ GridProblem P) {
  __shared__ double s_red[kThreads / 32];
  __shared__ double s_val;
  __shared__ Pending s_pend[kMaxPending];

  const int G = gridDim.x, rank = blockIdx.x;
  const int W = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = P.n;
  const int nblk = (n + 31) >> 5;
  const int bpc = (nblk + G - 1) / G;
  const int b0 = rank * bpc, b1 = min(nblk, b0 + bpc);
  double2* const* B = P.buf;
  int bi[11];
#pragma unroll
  for (int i = 0; i < 11; ++i) bi[i] = i;

  const double atol = P.atol, rtol = P.rtol;
  const double t0 = P.t0, tf = P.tf, eps_t = P.eps_t;
  double* red = P.red;
  double* obs_slots[2] = {red + static_cast<long long>(kSlotObs0) * G,
                          red + static_cast<long long>(kSlotObs0 + kObsSlots) * G};
  int obs_par = 0;

  double t = t0, t_old = t0, h = 0.0, h_last = 0.0, facold = 1e-4;
  long long steps = 0, rejected = 0, rhs_evals = 0, attempts_total = 0;
  int status = kRunning;
  double fail_t = 0.0;
  int next = 0, np = 0;
  const int kcap = max(1, min(kMaxPending, kObsSlots / (2 * max(1, P.n_e))));

  auto push_pending = [&](double theta) {
    // all threads run this identically; thread 0 also records it in shared memory
    const int gi = P.ev_grid[next], si = P.ev_save[next];
    if (threadIdx.x == 0) s_pend[np] = Pending{theta, gi, si};
    ++np;
    ++next;
  };

  // ---------------- start (integrator.hpp:61-69) + initial_step (:157-187) ----------------
  // events at t0 observe y0 directly (evolve.cpp:134-137)
  while (next < P.n_ev && P.ev_t[next] <= t0 + eps_t && np < kcap) push_pending(__longlong_as_double(0x7ff8000000000000ll));
  __syncthreads();
  {
    // pass S1: k1 = G(t0) y ; d0, d1 partials
    double d0 = 0.0, d1 = 0.0;
    for (int b = b0 + warp; b < b1; b += W) {
      const int rb = b << 5, row = rb + lane;
      const double2* y = B[bi[Y]];
      double2 k = gen_row(P.gen, P.params, b, t, [&](int c) { return y[c]; });
      if (row < n) {
        B[bi[K1]][row] = k;
        const double2 yy = y[row];
        const double sc = atol + rtol * cabs_(yy);
        d0 += cnorm(make_double2(yy.x / sc, yy.y / sc));
        d1 += cnorm(make_double2(k.x / sc, k.y / sc));
      }
    }
    if (np) observe_pass<MODE>(P, B, bi, s_pend, np, h_last, obs_slots[obs_par], s_red, rank, G);
    d0 = block_sum(d0, s_red);
    d1 = block_sum(d1, s_red);
    if (threadIdx.x == 0) {
      red[static_cast<long long>(kSlotD0) * G + rank] = d0;
      red[static_cast<long long>(kSlotD1) * G + rank] = d1;
    }
    grid_barrier(P.bar, G);
    rhs_evals += 1;
    if (np) {
      observe_commit(P, s_pend, np, obs_slots[obs_par], G);
      obs_par ^= 1;
      np = 0;
    }
    d0 = sqrt(grid_value(red, kSlotD0, G, &s_val) / static_cast<double>(n));
    d1 = sqrt(grid_value(red, kSlotD1, G, &s_val) / static_cast<double>(n));
    double h0 = (d0 < 1e-5 || d1 < 1e-5) ? 1e-6 : 0.01 * d0 / d1;
    h0 = fmin(h0, tf - t);
    if (!(h0 > 0)) h0 = 1e-6;
    // pass S2: k2 = G(t0+h0)(y + h0 k1) ; d2 partial
    double d2 = 0.0;
    for (int b = b0 + warp; b < b1; b += W) {
      const int rb = b << 5, row = rb + lane;
      const double2* y = B[bi[Y]];
      const double2* k1 = B[bi[K1]];
      double2 k = gen_row(P.gen, P.params, b, t + h0, [&](int c) {
        const double2 a = y[c], b2 = k1[c];
        return make_double2(a.x + h0 * b2.x, a.y + h0 * b2.y);
      });
      if (row < n) {
        const double2 yy = y[row], kk1 = k1[row];
        const double sc = atol + rtol * cabs_(yy);
        const double2 df = csub(k, kk1);
        d2 += cnorm(make_double2(df.x / sc, df.y / sc));
      }
    }
    d2 = block_sum(d2, s_red);
    if (threadIdx.x == 0) red[static_cast<long long>(kSlotD2) * G + rank] = d2;
    grid_barrier(P.bar, G);
    rhs_evals += 1;
    d2 = sqrt(grid_value(red, kSlotD2, G, &s_val) / static_cast<double>(n)) / h0;
    double h1;
    if (fmax(d1, d2) <= 1e-15) h1 = fmax(1e-6, h0 * 1e-3);
    else h1 = pow(0.01 / fmax(d1, d2), 0.2);
    h = fmin(fmin(100.0 * h0, h1), tf - t);
  }

  // ---------------- main loop (evolve.cpp:156-167) ----------------
  while (next < P.n_ev && status == kRunning) {
    if (steps >= P.max_steps) {
      status = kFailMaxSteps;
      fail_t = t;
      break;
    }
    int attempts = 0;
    for (;;) {  // Dopri5::step (integrator.hpp:78-147)
      const double hh = fmin(h, tf - t);
      const bool clamped = hh < h;
      if (!(hh > 0.0)) { status = kFailPastEnd; fail_t = t; break; }
      if (hh <= fabs(t) * 1e-15 + 1e-300) { status = kFailUnderflow; fail_t = t; break; }
      if (++attempts > 1000) { status = kFailRejected; fail_t = t; break; }
      ++attempts_total;
      using namespace dp;
      // ---- stage 2: k2 = G(t + c2 h)(y + h a21 k1); ysti3 -> SA
      {
        const double2* y = B[bi[Y]];
        const double2* k1 = B[bi[K1]];
        double2* k2o = B[bi[K2]];
        double2* so = B[bi[SA]];
        for (int b = b0 + warp; b < b1; b += W) {
          const int rb = b << 5, row = rb + lane;
          double2 k = gen_row(P.gen, P.params, b, t + c2 * hh, [&](int c) {
            const double2 a = y[c], q = k1[c];
            return make_double2(a.x + hh * (a21 * q.x), a.y + hh * (a21 * q.y));
          });
          if (row < n) {
            const double2 yy = y[row], q1 = k1[row];
            k2o[row] = k;
            so[row] = make_double2(yy.x + hh * (a31 * q1.x + a32 * k.x), yy.y + hh * (a31 * q1.y + a32 * k.y));
          }
        }
        if (np) observe_pass<MODE>(P, B, bi, s_pend, np, h_last, obs_slots[obs_par], s_red, rank, G);
        grid_barrier(P.bar, G);
        if (np) {
          observe_commit(P, s_pend, np, obs_slots[obs_par], G);
          obs_par ^= 1;
          np = 0;
        }
      }
      // ---- stage 3: k3 = G(t + c3 h) SA; ysti4 -> SB
      {
        const double2* y = B[bi[Y]];
        const double2* x = B[bi[SA]];
        const double2 *k1 = B[bi[K1]], *k2 = B[bi[K2]];
        double2* ko = B[bi[K3]];
        double2* so = B[bi[SB]];
        for (int b = b0 + warp; b < b1; b += W) {
          const int rb = b << 5, row = rb + lane;
          double2 k = gen_row(P.gen, P.params, b, t + c3 * hh, [&](int c) { return x[c]; });
          if (row < n) {
            const double2 yy = y[row], q1 = k1[row], q2 = k2[row];
            ko[row] = k;
            so[row] = make_double2(yy.x + hh * (a41 * q1.x + a42 * q2.x + a43 * k.x),
                                   yy.y + hh * (a41 * q1.y + a42 * q2.y + a43 * k.y));
          }
        }
        grid_barrier(P.bar, G);
      }
      // ---- stage 4: k4 = G(t + c4 h) SB; ysti5 -> SA
      {
        const double2* y = B[bi[Y]];
        const double2* x = B[bi[SB]];
        const double2 *k1 = B[bi[K1]], *k2 = B[bi[K2]], *k3 = B[bi[K3]];
        double2* ko = B[bi[K4]];
        double2* so = B[bi[SA]];
        for (int b = b0 + warp; b < b1; b += W) {
          const int rb = b << 5, row = rb + lane;
          double2 k = gen_row(P.gen, P.params, b, t + c4 * hh, [&](int c) { return x[c]; });
          if (row < n) {
            const double2 yy = y[row], q1 = k1[row], q2 = k2[row], q3 = k3[row];
            ko[row] = k;
            so[row] = make_double2(yy.x + hh * (a51 * q1.x + a52 * q2.x + a53 * q3.x + a54 * k.x),
                                   yy.y + hh * (a51 * q1.y + a52 * q2.y + a53 * q3.y + a54 * k.y));
          }
        }
        grid_barrier(P.bar, G);
      }
      // ---- stage 5: k5 = G(t + c5 h) SA; ysti6 -> SB
      {
        const double2* y = B[bi[Y]];
        const double2* x = B[bi[SA]];
        const double2 *k1 = B[bi[K1]], *k2 = B[bi[K2]], *k3 = B[bi[K3]], *k4 = B[bi[K4]];
        double2* ko = B[bi[K5]];
        double2* so = B[bi[SB]];
        for (int b = b0 + warp; b < b1; b += W) {
          const int rb = b << 5, row = rb + lane;
          double2 k = gen_row(P.gen, P.params, b, t + c5 * hh, [&](int c) { return x[c]; });
          if (row < n) {
            const double2 yy = y[row], q1 = k1[row], q2 = k2[row], q3 = k3[row], q4 = k4[row];
            ko[row] = k;
            so[row] = make_double2(
                yy.x + hh * (a61 * q1.x + a62 * q2.x + a63 * q3.x + a64 * q4.x + a65 * k.x),
                yy.y + hh * (a61 * q1.y + a62 * q2.y + a63 * q3.y + a64 * q4.y + a65 * k.y));
          }
        }
        grid_barrier(P.bar, G);
      }
      // ---- stage 6: k6 = G(t + h) SB; ysti7 (= y1 candidate) -> SA
      {
        const double2* y = B[bi[Y]];
        const double2* x = B[bi[SB]];
        const double2 *k1 = B[bi[K1]], *k3 = B[bi[K3]], *k4 = B[bi[K4]], *k5 = B[bi[K5]];
        double2* ko = B[bi[K6]];
        double2* so = B[bi[SA]];
        for (int b = b0 + warp; b < b1; b += W) {
          const int rb = b << 5, row = rb + lane;
          double2 k = gen_row(P.gen, P.params, b, t + hh, [&](int c) { return x[c]; });
          if (row < n) {
            const double2 yy = y[row], q1 = k1[row], q3 = k3[row], q4 = k4[row], q5 = k5[row];
            ko[row] = k;
            so[row] = make_double2(
                yy.x + hh * (a71 * q1.x + a73 * q3.x + a74 * q4.x + a75 * q5.x + a76 * k.x),
                yy.y + hh * (a71 * q1.y + a73 * q3.y + a74 * q4.y + a75 * q5.y + a76 * k.y));
          }
        }
        grid_barrier(P.bar, G);
      }
      // ---- stage 7 (FSAL): k7 = G(t + h) SA; embedded error partial
      double err;
      {
        const double2* y = B[bi[Y]];
        const double2* x = B[bi[SA]];
        const double2 *k1 = B[bi[K1]], *k3 = B[bi[K3]], *k4 = B[bi[K4]], *k5 = B[bi[K5]], *k6 = B[bi[K6]];
        double2* ko = B[bi[K7]];
        double esq = 0.0;
        for (int b = b0 + warp; b < b1; b += W) {
          const int rb = b << 5, row = rb + lane;
          double2 k = gen_row(P.gen, P.params, b, t + hh, [&](int c) { return x[c]; });
          if (row < n) {
            const double2 yy = y[row], y1 = x[row], q1 = k1[row], q3 = k3[row], q4 = k4[row],
                          q5 = k5[row], q6 = k6[row];
            ko[row] = k;
            double2 e;
            e.x = hh * (e1 * q1.x + e3 * q3.x + e4 * q4.x + e5 * q5.x + e6 * q6.x + e7 * k.x);
            e.y = hh * (e1 * q1.y + e3 * q3.y + e4 * q4.y + e5 * q5.y + e6 * q6.y + e7 * k.y);
            const double sc = atol + rtol * fmax(cabs_(yy), cabs_(y1));
            const double qq = cabs_(e) / sc;
            esq += qq * qq;
          }
        }
        esq = block_sum(esq, s_red);
        if (threadIdx.x == 0) red[static_cast<long long>(kSlotErr) * G + rank] = esq;
        grid_barrier(P.bar, G);
        err = sqrt(grid_value(red, kSlotErr, G, &s_val) / static_cast<double>(n));
        if (!isfinite(err)) err = 10.0;
      }
      rhs_evals += 6;
      if (err <= 1.0) {  // accept (integrator.hpp:119-142)
        const double fac11 = pow(err, expo1);
        double fac = fac11 / pow(facold, beta);
        fac = fmax(facc2, fmin(facc1, fac / safe));
        const double h_new = hh / fac;
        facold = fmax(err, 1e-4);
        t_old = t;
        t += hh;
        h_last = hh;
        {  // y_old <- y, y <- ysti7, FSAL k1 <-> k7
          const int oy = bi[Y], oyo = bi[YO];
          bi[YO] = oy;
          bi[Y] = bi[SA];
          bi[SA] = oyo;
          const int k1p = bi[K1];
          bi[K1] = bi[K7];
          bi[K7] = k1p;
        }
        ++steps;
        if (!clamped) h = h_new;
        else h = fmax(h, h_new);
        break;
      }
      ++rejected;
      h = hh / fmin(facc1, pow(err, expo1) / safe);
    }
    if (status != kRunning) break;
    // observation events reached by this step (evolve.cpp:160-165)
    for (;;) {
      while (next < P.n_ev && P.ev_t[next] <= t + eps_t && np < kcap)
        push_pending((fmin(P.ev_t[next], t) - t_old) / h_last);
      const bool more = next < P.n_ev && P.ev_t[next] <= t + eps_t;
      const bool last = t >= tf - eps_t;
      if (!(more || (last && np))) break;
      // flush now: either the pending list is full or the solve is ending
      __syncthreads();
      observe_pass<MODE>(P, B, bi, s_pend, np, h_last, obs_slots[obs_par], s_red, rank, G);
      grid_barrier(P.bar, G);
      observe_commit(P, s_pend, np, obs_slots[obs_par], G);
      obs_par ^= 1;
      np = 0;
    }
    __syncthreads();
    if (t >= tf - eps_t) break;
  }

  // trailing events observe the final state (evolve.cpp:169)
  if (status == kRunning) {
    if (np) {
      __syncthreads();
      observe_pass<MODE>(P, B, bi, s_pend, np, h_last, obs_slots[obs_par], s_red, rank, G);
      grid_barrier(P.bar, G);
      observe_commit(P, s_pend, np, obs_slots[obs_par], G);
      obs_par ^= 1;
      np = 0;
    }
    while (next < P.n_ev) {
      while (next < P.n_ev && np < kcap) push_pending(__longlong_as_double(0x7ff8000000000000ll));
      __syncthreads();
      observe_pass<MODE>(P, B, bi, s_pend, np, h_last, obs_slots[obs_par], s_red, rank, G);
      grid_barrier(P.bar, G);
      observe_commit(P, s_pend, np, obs_slots[obs_par], G);
      obs_par ^= 1;
      np = 0;
    }
    status = kDone;
  }
  if (rank == 0 && threadIdx.x == 0) {
    GridCtl* c = P.ctl;
    c->t = t;
    c->h = h;
    c->status = status;
    c->fail_t = fail_t;
    c->steps = steps;
    c->rejected = rejected;
    c->rhs_evals = rhs_evals;
    c->attempts = attempts_total;
    c->final_buf = bi[Y];
  }
}

template <int MODE>
cudaError_t launch_one(const GridProblem& P, int grid, cudaStream_t s) {
  void* args[] = {const_cast<GridProblem*>(&P)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(dp5_grid_kernel<MODE>), dim3(grid),
                                     dim3(kThreads), args, 0, s);
}

template <int MODE>
int occupancy_one() {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dp5_grid_kernel<MODE>, kThreads, 0);
  return nb;
}

}  // namespace

int grid_threads() { return kThreads; }

int grid_max_blocks_per_sm(int mode) { return mode == 0 ? occupancy_one<0>() : occupancy_one<1>(); }

cudaError_t launch_grid_dp5(const GridProblem& P, int mode, int grid, cudaStream_t s) {
  return mode == 0 ? launch_one<0>(P, grid, s) : launch_one<1>(P, grid, s);
}

}  // namespace qsg
