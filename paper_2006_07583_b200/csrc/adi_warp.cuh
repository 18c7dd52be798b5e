// adi_warp.cuh — warp-per-line kernels for SHORT grid lines (at most 64 stored positions:
// the paper's 41-node grids of configs 1-2).
//
// A half-step on such a line is 17 operator applications in a row (K fixed-point sweeps
// of eq. 8 / eq. 9 and the fused epilogue), each a short stencil and, for CFD, a
// tridiagonal solve: one long dependent chain per line.  The thread-per-line kernels
// (adi_thread.cuh) run it sequentially in one thread, ~25k dependent instructions; here
// the 32 lanes of a warp share the line, two positions per lane:
//   * stencils (App. A / App. B): the operand goes through a 64-double shared buffer, each
//     lane reads the neighbours it needs, the line-end closure rows are computed by the
//     lanes owning those positions with the same formulas as the thread kernels;
//   * the CFD solve keeps the paper's no-pivot LU of P̄ / P (the tables
//     l, 1/d, c of setup_axis): the forward recurrence y_p = r_p - l_p y_(p-1) and the
//     backward recurrence z_p = y_p/d_p - (c_p/d_p) z_(p+1) are first-order linear
//     recurrences, evaluated as warp scans of affine maps (Kogge-Stone, 5 shuffle steps).
//     A lane first folds its two positions into one map; the maps' multipliers depend only
//     on the tables, so their scan prefixes are computed once per kernel and each solve
//     scans only the offsets.  Same recurrences as the thread kernels, reassociated.
// Same arrays, layouts, modes (SWEEP, FINAL, PROLOGUE) and KParams as the other kernels.
#pragma once
#include "adi_line.cuh"

namespace adi {

constexpr int WK_LANES = 32, WK_POS = 2 * WK_LANES;   // positions per line held by a warp
constexpr int WK_WARPS = 4;                          // lines (warps) per CTA

// the scan multipliers of one recurrence system (u-op or x-op), per lane
struct WkSys {
  double l[2], iv[2], m[2];   // l_q, 1/d_q, c_q/d_q at this lane's positions (0 outside the system)
  double fk[5], bk[5];        // multipliers of the forward / backward scan steps
};

// the system's tables at positions q0, q1 in [lo, hi] and the scan prefixes of the maps
__device__ __forceinline__ void wk_setup(WkSys& S, const double* tab, int n, int lo, int hi, int lane) {
  const int n1 = n + 1;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int q = 2 * lane + j;
    const bool in = q >= lo && q <= hi;
    S.l[j] = (in && q > lo) ? tab[q] : 0.0;
    S.iv[j] = in ? tab[n1 + q] : 0.0;
    S.m[j] = (in && q < hi) ? tab[2 * n1 + q] * tab[n1 + q] : 0.0;
  }
  // forward: y(q1) = B + A y(q0 - 1), A = l(q1) l(q0); backward: z(q0) = B + A z(q1 + 1), A = m(q0) m(q1)
  double fa = S.l[1] * S.l[0], ba = S.m[0] * S.m[1];
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int d = 1 << s;
    S.fk[s] = fa;
    S.bk[s] = ba;
    const double fp = __shfl_up_sync(0xffffffffu, fa, d);
    const double bn = __shfl_down_sync(0xffffffffu, ba, d);
    if (lane >= d) fa *= fp;
    if (lane + d < WK_LANES) ba *= bn;
  }
}

// z = T^{-1} r on the system (r, z: this lane's two positions; 0 outside the system)
__device__ __forceinline__ void wk_solve(const WkSys& S, const double (&r)[2], double (&z)[2], int lane) {
  // forward: lane map y(q1) = (r1 - l1 r0) + l1 l0 y_in, inclusive scan, then y_in from lane - 1
  double B = fma(-S.l[1], r[0], r[1]);
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int d = 1 << s;
    const double Bp = __shfl_up_sync(0xffffffffu, B, d);
    if (lane >= d) B = fma(S.fk[s], Bp, B);
  }
  double yin = __shfl_up_sync(0xffffffffu, B, 1);
  if (lane == 0) yin = 0.0;
  double y[2];
  y[0] = fma(-S.l[0], yin, r[0]);
  y[1] = fma(-S.l[1], y[0], r[1]);
  // backward: g = y/d, lane map z(q0) = (g0 - m0 g1) + m0 m1 z_in, suffix scan, z_in from lane + 1
  const double g0 = y[0] * S.iv[0], g1 = y[1] * S.iv[1];
  double C = fma(-S.m[0], g1, g0);
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int d = 1 << s;
    const double Cn = __shfl_down_sync(0xffffffffu, C, d);
    if (lane + d < WK_LANES) C = fma(S.bk[s], Cn, C);
  }
  double zin = __shfl_down_sync(0xffffffffu, C, 1);
  if (lane == WK_LANES - 1) zin = 0.0;
  z[1] = fma(-S.m[1], zin, g1);
  z[0] = fma(-S.m[0], z[1], g0);
}

template <int METHOD, int MODE>
__global__ void __launch_bounds__(32 * WK_WARPS) adi_warp_kernel(const __grid_constant__ KParams P) {
  __shared__ double wbuf[WK_WARPS][WK_POS];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int line = P.line0 + blockIdx.x * WK_WARPS + w;
  const int b = blockIdx.z;
  if (line < P.line_lo || line >= P.nlines) return;   // whole warps: no CTA barrier below
  double* const buf = wbuf[w];
  const int n = P.n;
  const int q0 = 2 * lane;
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

  // CFD: the two recurrence systems (u-op: P̄ on [1, n-1]; x-op: P on [0, n])
  WkSys SU, SX;
  if (METHOD == M_CFD) {
    wk_setup(SU, P.tabU, n, 1, n - 1, lane);
    wk_setup(SX, P.tabX, n, 0, n, lane);
  }

  // the operand of an operator into the warp's buffer (positions 2 lane, 2 lane + 1)
  auto publish = [&](const double (&a)[2]) {
    __syncwarp();   // the previous operator's reads are done
    buf[q0] = a[0];
    buf[q0 + 1] = a[1];
    __syncwarp();
  };
  auto at = [&](int p) -> double { return buf[p < 0 ? 0 : (p >= WK_POS ? WK_POS - 1 : p)]; };

  // u-op: out_p = B_p - alpha D̄(x)_p on [1, uhi]; the other positions keep out's value
  auto uop = [&](const double (&xo)[2], const double (&B)[2], double (&out)[2]) {
    publish(xo);
    double r[2];
    if (METHOD == M_CFD) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int p = q0 + j;
        double v = 0.0;
        if (p == 1) v = (-at(0) - 9.0 * at(1) + 9.0 * at(2) + at(3)) * (1.0 / 3.0);
        else if (p == n - 1) v = (-at(n - 3) - 9.0 * at(n - 2) + 9.0 * at(n - 1) + at(n)) * (1.0 / 3.0);
        else if (p >= 2 && p <= n - 2) v = at(p + 1) - at(p - 1);
        r[j] = v;
      }
      double z[2];
      wk_solve(SU, r, z, lane);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int p = q0 + j;
        if (p >= 1 && p <= n - 1) out[j] = fma(-P.cu, z[j], B[j]);
      }
    } else {
      const double a = P.cu, cA = P.mA, cB = P.mB;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int p = q0 + j;
        if (p == 1) {
          double s = 0.0;
          for (int k = 0; k < 6; ++k) s = fma(c_d4r0[k], at(k), s);
          r[j] = fma(-a, s, B[j]);
        } else if (p == n) {
          double s = 0.0;
          for (int k = 0; k < 6; ++k) s = fma(-c_d4r0[5 - k], at(n - 5 + k), s);
          r[j] = fma(-a, s, B[j]);
        } else {
          r[j] = fma(cA, at(p + 1) - at(p - 2), fma(cB, at(p - 1) - at(p), B[j]));
        }
        if (p >= 1 && p <= n) out[j] = r[j];
      }
    }
  };
  // x-op: out_p = B_p - beta D([gL, u, gR])_p on [0, n]
  auto xop = [&](const double (&uo)[2], const double (&B)[2], double (&out)[2]) {
    publish(uo);
    double r[2];
    if (METHOD == M_CFD) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int p = q0 + j;
        double v = 0.0;
        if (p == 0) v = (-17.0 * at(0) + 9.0 * at(1) + 9.0 * at(2) - at(3)) * (1.0 / 3.0);
        else if (p == n) v = (at(n - 3) - 9.0 * at(n - 2) - 9.0 * at(n - 1) + 17.0 * at(n)) * (1.0 / 3.0);
        else if (p >= 1 && p <= n - 1) v = at(p + 1) - at(p - 1);
        r[j] = v;
      }
      double z[2];
      wk_solve(SX, r, z, lane);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int p = q0 + j;
        if (p <= n) out[j] = fma(-P.cx, z[j], B[j]);
      }
    } else {
      const double bb = P.cx, cC = P.mC, cD = P.mD;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int p = q0 + j;
        double s = 0.0;
        if (p == 0) {
          for (int k = 0; k < 6; ++k) s = fma(c_g4r0[k], at(k), s);
          r[j] = fma(-bb, s, B[j]);
        } else if (p == 1) {
          for (int k = 0; k < 5; ++k) s = fma(c_g4r1[k], at(k), s);
          r[j] = fma(-bb, s, B[j]);
        } else if (p == n - 1) {
          for (int k = 0; k < 4; ++k) s = fma(-c_g4r1[4 - k], at(n - 3 + k), s);
          s = fma(-c_g4r1[0], gR, s);
          r[j] = fma(-bb, s, B[j]);
        } else if (p == n) {
          for (int k = 0; k < 5; ++k) s = fma(-c_g4r0[5 - k], at(n - 4 + k), s);
          s = fma(-c_g4r0[0], gR, s);
          r[j] = fma(-bb, s, B[j]);
        } else {
          r[j] = fma(cC, at(p + 2) - at(p - 1), fma(cD, at(p) - at(p + 1), B[j]));
        }
        if (p <= n) out[j] = r[j];
      }
    }
  };

  // this lane's bases and state (positions q0, q0 + 1; 0 outside the line)
  double u[2] = {0.0, 0.0}, x[2] = {0.0, 0.0}, S[2] = {0.0, 0.0}, X[2] = {0.0, 0.0};
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int p = q0 + j;
    if (p <= n) X[j] = Xb[p];
    if (MODE != KM_PROLOGUE && Sb && p >= 1 && p <= uhi) S[j] = Sb[p];
    if (MODE == KM_PROLOGUE && p <= pR) u[j] = Ub[(long long)p * P.u_pt];
    x[j] = X[j];
  }
  double acc = 0.0;   // finiteness check (ADI_CHECK_FINITE)
  if (MODE == KM_PROLOGUE) {
    // W* = W - beta D(U) -> X_out; S1 = U + dt/2 F - alpha D̄(W) -> S_out (transposed)
    double ws[2] = {X[0], X[1]};
    xop(u, X, ws);
    double* Xo = P.X_out + (long long)b * P.x_batch + (long long)line * P.x_line;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int p = q0 + j;
      if (p <= n) { Xo[p] = ws[j]; acc += ws[j]; }
      if (p >= 1 && p <= uhi) u[j] = u[j] + src(p);
    }
    double o[2] = {u[0], u[1]};
    uop(x, u, o);
    u[0] = o[0]; u[1] = o[1];
  } else {
    // Dirichlet slots of ū
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int p = q0 + j;
      if (p == 0) u[j] = gL;
      if (p == pR) u[j] = gR;
    }
    const int KK = P.Kdev ? *P.Kdev : P.K;
    for (int k = 0; k < KK; ++k) {
      uop(x, S, u);
      xop(u, X, x);
    }
    if (MODE == KM_SWEEP) {
      // the next explicit half (fused): S' = (u_K + dt/2 F) - alpha D̄(x_K), X' = 2 x_K - X
      double base[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int p = q0 + j;
        base[j] = (p >= 1 && p <= uhi) ? u[j] + src(p) : u[j];
      }
      double o[2] = {base[0], base[1]};
      uop(x, base, o);
      u[0] = o[0]; u[1] = o[1];
#pragma unroll
      for (int j = 0; j < 2; ++j) x[j] = fma(2.0, x[j], -X[j]);
    }
  }
  // stores: S' (or U) transposed, X' along the line
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int p = q0 + j;
    if (MODE == KM_FINAL) {
      double* Ut = P.U_out + (long long)b * P.u_batch + (long long)line * P.u_line;
      if (p <= n) { Ut[(long long)p * P.u_pt] = u[j]; acc += u[j]; }
      if (METHOD == M_MFD && p == n + 1) Ut[(long long)p * P.u_pt] = gR;   // ū_{n+1} at this time
    } else if (p >= 1 && p <= uhi) {
      double* So = P.S_out + (long long)b * P.s_batch + (long long)line * P.so_line;
      So[(long long)p * P.so_pt] = u[j];
      acc += u[j];
    }
    if (MODE != KM_PROLOGUE && p <= n) {
      double* Xo = P.X_out + (long long)b * P.x_batch + (long long)line * P.x_line;
      Xo[p] = x[j];
      acc += x[j];
    }
  }
  if (P.flag && !isfinite(acc)) atomicOr(P.flag, 1);
}

}  // namespace adi
