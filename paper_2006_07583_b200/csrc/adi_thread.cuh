// adi_thread.cuh — thread-per-line kernels for SHORT grid lines (the paper's own grids,
// configs 1-2: 41..~160 nodes per line).
//
// On lines this short a warp-per-line tile (adi_line.cuh) leaves most lanes idle and the
// CTA count is a few per sweep.  Here ONE THREAD runs one grid line through the whole
// half-step, sequentially, as the paper's CPU code does per line ("no data
// dependency among the N linear systems"): K fixed-point sweeps of eq. 8 / eq. 9
//     u <- S - alpha D̄(x),   x <- X - beta D([gL, u, gR])
// with every CFD derivative a stencil of App. A followed by the Thomas solve with the
// no-pivot LU of P̄ / P (the per-position tables l, 1/d, c of
// setup_axis), every MFD derivative the D4 / G4 rows of App. B; then the fused epilogue
// (the next explicit half, S' = u - alpha D̄(x) + dt/2 F, X' = 2x - X), or the FINAL /
// PROLOGUE variants, with the same arrays, layouts and KParams as the line kernels.
//
// The line's working arrays (u, x and a temporary) live in shared memory as
// [array][position][thread] (consecutive threads, consecutive banks); the bases S, X are
// read from global memory (L1-resident at these sizes).  A line's half-step is one long
// dependent chain, so the kernel is built for latency: the LU tables are staged in shared
// memory once per CTA (l, 1/d and c/d per position: the backward step is then ONE
// dependent FMA, z = r/d - (c/d) z, with r/d off the chain), every array is addressed
// through __restrict__ shared pointers, and the loops are unrolled so the loads of later
// positions are issued ahead of the recurrence.
#pragma once
#include "adi_line.cuh"

namespace adi {

// doubles of the staged CFD LU tables ([2 systems][3][n + 1], rounded to 2 for alignment)
__host__ __device__ inline int thread_tab_doubles(int n) { return (6 * (n + 1) + 1) & ~1; }

template <int METHOD, int MODE>
__global__ void __launch_bounds__(128) adi_thread_kernel(const __grid_constant__ KParams P) {
  extern __shared__ __align__(16) double tsm[];
  const int T = blockDim.x, t = threadIdx.x;
  const int n = P.n;
  const int np = n + 2;   // stored positions 0..n+1 (the MFD ū_{n+1} slot)
  const int line = P.line0 + blockIdx.x * T + t;
  const int b = blockIdx.z;
  // CFD: the LU tables of both systems, [u-op, x-op][l, 1/d, c/d][n + 1]
  double* __restrict__ tab = tsm;
  if (METHOD == M_CFD) {
    const int n1 = n + 1;
    for (int i = t; i < n1; i += T) {
      const double ul = P.tabU[i], ui = P.tabU[n1 + i], uc = P.tabU[2 * n1 + i];
      const double xl = P.tabX[i], xi = P.tabX[n1 + i], xc = P.tabX[2 * n1 + i];
      tab[i] = ul; tab[n1 + i] = ui; tab[2 * n1 + i] = uc * ui;
      tab[3 * n1 + i] = xl; tab[4 * n1 + i] = xi; tab[5 * n1 + i] = xc * xi;
    }
    __syncthreads();
  }
  if (line < P.line_lo || line >= P.nlines) return;
  double* const arr = tsm + (METHOD == M_CFD ? thread_tab_doubles(n) : 0);
  double* __restrict__ U = arr + t;                          // u (pressure of this direction), slots 0 and n (CFD) / n+1 (MFD)
  double* __restrict__ X = arr + (size_t)np * T + t;         // x (velocity of this direction)
  double* __restrict__ R = arr + (size_t)2 * np * T + t;     // temporary (stencil, Thomas)
  auto u = [&](int p) -> double& { return U[(size_t)p * T]; };
  auto x = [&](int p) -> double& { return X[(size_t)p * T]; };
  auto r = [&](int p) -> double& { return R[(size_t)p * T]; };
  const int uhi = (METHOD == M_CFD) ? n - 1 : n;   // u active on [1, uhi]
  const int pR = (METHOD == M_CFD) ? n : n + 1;    // position of ū's right Dirichlet value
  const double* Sb = P.S_in ? P.S_in + (long long)b * P.s_batch + (long long)line * P.s_line : nullptr;
  const double* Xb = P.X_in + (long long)b * P.x_batch + (long long)line * P.x_line;
  const double* Ub = P.U_in ? P.U_in + (long long)b * P.u_batch + (long long)line * P.u_line : nullptr;

  // Dirichlet values of this line for this half-step
  double gL = 0.0, gR = 0.0;
  if (MODE == KM_PROLOGUE) {
    gL = Ub[0];
    gR = Ub[(long long)pR * P.u_pt];
  } else {
    if (P.edgeL) gL = P.edgeL[line] * P.gb;
    if (P.edgeR) gR = P.edgeR[line] * P.gb;
  }
  // the source at position p (F = phi gf + the point source g/h^2), times dt/2
  const int ipt = (P.pt_line && line == P.pt_line[b]) ? P.pt_pos[b] : -1;
  const double* ph = P.phi_src ? P.phi_src + (long long)line * P.s_line : nullptr;
  auto src = [&](int p) -> double {
    double f = ph ? ph[p] * P.gf : 0.0;
    if (p == ipt) f += P.pt_amp * P.gf;
    return P.half_dt * f;
  };

  // ---- the two derivative operators on this line (App. A / App. B)
  // u-op: out_p = B_p - alpha D̄(x)_p on the u positions [1, uhi]; out may alias B
  auto uop = [&](auto&& B, auto&& out) {
    if (METHOD == M_CFD) {
      const double* __restrict__ tl = tab;
      const double* __restrict__ ti = tab + (n + 1);
      const double* __restrict__ tc = tab + 2 * (n + 1);   // c/d
      r(1) = (-x(0) - 9.0 * x(1) + 9.0 * x(2) + x(3)) * (1.0 / 3.0);
#pragma unroll 4
      for (int p = 2; p <= n - 2; ++p) r(p) = x(p + 1) - x(p - 1);
      r(n - 1) = (-x(n - 3) - 9.0 * x(n - 2) + 9.0 * x(n - 1) + x(n)) * (1.0 / 3.0);
      double y = r(1);
#pragma unroll 8
      for (int p = 2; p <= n - 1; ++p) { y = fma(-tl[p], y, r(p)); r(p) = y; }
      double z = y * ti[n - 1];
      r(n - 1) = z;
#pragma unroll 8
      for (int p = n - 2; p >= 1; --p) { z = fma(-tc[p], z, r(p) * ti[p]); r(p) = z; }
#pragma unroll 4
      for (int p = 1; p <= n - 1; ++p) out(p) = fma(-P.cu, r(p), B(p));
    } else {
      const double a = P.cu, cA = P.mA, cB = P.mB;
      double s = 0.0;
      for (int k = 0; k < 6; ++k) s = fma(c_d4r0[k], x(k), s);
      r(1) = fma(-a, s, B(1));
#pragma unroll 4
      for (int p = 2; p <= n - 1; ++p) r(p) = fma(cA, x(p + 1) - x(p - 2), fma(cB, x(p - 1) - x(p), B(p)));
      s = 0.0;
      for (int k = 0; k < 6; ++k) s = fma(-c_d4r0[5 - k], x(n - 5 + k), s);
      r(n) = fma(-a, s, B(n));
#pragma unroll 4
      for (int p = 1; p <= n; ++p) out(p) = r(p);
    }
  };
  // x-op: out_p = B_p - beta D([gL, u, gR])_p on the nodes [0, n]; out may alias B
  auto xop = [&](auto&& B, auto&& out) {
    if (METHOD == M_CFD) {
      const double* __restrict__ tl = tab + 3 * (n + 1);
      const double* __restrict__ ti = tab + 4 * (n + 1);
      const double* __restrict__ tc = tab + 5 * (n + 1);   // c/d
      r(0) = (-17.0 * u(0) + 9.0 * u(1) + 9.0 * u(2) - u(3)) * (1.0 / 3.0);
#pragma unroll 4
      for (int p = 1; p <= n - 1; ++p) r(p) = u(p + 1) - u(p - 1);
      r(n) = (u(n - 3) - 9.0 * u(n - 2) - 9.0 * u(n - 1) + 17.0 * u(n)) * (1.0 / 3.0);
      double y = r(0);
#pragma unroll 8
      for (int p = 1; p <= n; ++p) { y = fma(-tl[p], y, r(p)); r(p) = y; }
      double z = y * ti[n];
      r(n) = z;
#pragma unroll 8
      for (int p = n - 1; p >= 0; --p) { z = fma(-tc[p], z, r(p) * ti[p]); r(p) = z; }
#pragma unroll 4
      for (int p = 0; p <= n; ++p) out(p) = fma(-P.cx, r(p), B(p));
    } else {
      const double bb = P.cx, cC = P.mC, cD = P.mD;
      double s = 0.0;
      for (int k = 0; k < 6; ++k) s = fma(c_g4r0[k], u(k), s);
      r(0) = fma(-bb, s, B(0));
      s = 0.0;
      for (int k = 0; k < 5; ++k) s = fma(c_g4r1[k], u(k), s);
      r(1) = fma(-bb, s, B(1));
#pragma unroll 4
      for (int p = 2; p <= n - 2; ++p) r(p) = fma(cC, u(p + 2) - u(p - 1), fma(cD, u(p) - u(p + 1), B(p)));
      s = 0.0;
      for (int k = 0; k < 4; ++k) s = fma(-c_g4r1[4 - k], u(n - 3 + k), s);
      s = fma(-c_g4r1[0], gR, s);
      r(n - 1) = fma(-bb, s, B(n - 1));
      s = 0.0;
      for (int k = 0; k < 5; ++k) s = fma(-c_g4r0[5 - k], u(n - 4 + k), s);
      s = fma(-c_g4r0[0], gR, s);
      r(n) = fma(-bb, s, B(n));
#pragma unroll 4
      for (int p = 0; p <= n; ++p) out(p) = r(p);
    }
  };
  auto gS = [&](int p) -> double { return Sb[p]; };
  auto gX = [&](int p) -> double { return Xb[p]; };
  double acc = 0.0;   // finiteness check (ADI_CHECK_FINITE)

  if (MODE == KM_PROLOGUE) {
    // U (the column through the Dirichlet rows) and W̄ of this line
    for (int p = 0; p <= pR; ++p) u(p) = Ub[(long long)p * P.u_pt];
    for (int p = 0; p <= n; ++p) x(p) = Xb[p];
    // W* = W - beta D(U) -> X_out (through R, then into the output)
    double* Xo = P.X_out + (long long)b * P.x_batch + (long long)line * P.x_line;
    xop(gX, [&](int p) -> double& { return r(p); });
    for (int p = 0; p <= n; ++p) { Xo[p] = r(p); acc += r(p); }
    // S1 = U + dt/2 F - alpha D̄(W) -> S_out (transposed)
    for (int p = 1; p <= uhi; ++p) u(p) = u(p) + src(p);
    uop(u, u);
  } else {
    for (int p = 0; p <= n; ++p) x(p) = Xb[p];
    u(0) = gL;
    u(pR) = gR;
    const int KK = P.Kdev ? *P.Kdev : P.K;
    for (int k = 0; k < KK; ++k) {
      uop(gS, u);
      xop(gX, x);
    }
    if (MODE == KM_SWEEP) {
      // the next explicit half (fused): S' = (u_K + dt/2 F) - alpha D̄(x_K), X' = 2 x_K - X
      for (int p = 1; p <= uhi; ++p) u(p) = u(p) + src(p);
      uop(u, u);
      for (int p = 0; p <= n; ++p) x(p) = fma(2.0, x(p), -Xb[p]);
    }
  }
  // ---- stores: S' (or U) transposed, X' along the line
  if (MODE == KM_FINAL) {
    double* Ut = P.U_out + (long long)b * P.u_batch + (long long)line * P.u_line;
    for (int p = 0; p <= n; ++p) { Ut[(long long)p * P.u_pt] = u(p); acc += u(p); }
    if (METHOD == M_MFD) Ut[(long long)(n + 1) * P.u_pt] = gR;   // ū_{n+1} at this time
  } else {
    double* So = P.S_out + (long long)b * P.s_batch + (long long)line * P.so_line;
    for (int p = 1; p <= uhi; ++p) { So[(long long)p * P.so_pt] = u(p); acc += u(p); }
  }
  if (MODE != KM_PROLOGUE) {
    double* Xo = P.X_out + (long long)b * P.x_batch + (long long)line * P.x_line;
    for (int p = 0; p <= n; ++p) { Xo[p] = x(p); acc += x(p); }
  }
  if (P.flag && !isfinite(acc)) atomicOr(P.flag, 1);
}

// threads per CTA of the thread kernels for lines of n cells: three [n+2][T] arrays of
// doubles and the CFD LU tables within 200 KB of shared memory
inline int thread_tpb(int n) {
  int T = 128;
  while (T > 32 && ((size_t)3 * (n + 2) * T + thread_tab_doubles(n)) * 8 > 200 * 1024) T /= 2;
  return T;
}
inline size_t thread_smem(int n, int T) { return ((size_t)3 * (n + 2) * T + thread_tab_doubles(n)) * sizeof(double); }

}  // namespace adi
