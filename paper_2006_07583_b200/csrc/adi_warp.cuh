// adi_warp.cuh — warp-per-line kernels for SHORT grid lines (at most 32 NPL stored
// positions, NPL <= 12: the paper's grids of configs 1-2, 41..321 nodes).
//
// A half-step on such a line is 17 operator applications in a row (K fixed-point sweeps
// of eq. 8 / eq. 9 and the fused epilogue), each a short stencil and, for CFD, a
// tridiagonal solve: one long dependent chain per line.  The thread-per-line kernels
// (adi_thread.cuh) run it sequentially in one thread; here the 32 lanes of a warp share
// the line, NPL consecutive positions per lane:
//   * stencils (App. A / App. B): the operand goes through a shared buffer of the line,
//     each lane reads the neighbours it needs, and the line-end closure rows are computed
//     by the lanes owning those positions with the same formulas as the thread kernels;
//   * the CFD solve keeps the paper's no-pivot LU of P̄ / P (the tables
//     l, 1/d, c of setup_axis): the forward recurrence y_p = r_p - l_p y_(p-1) and the
//     backward recurrence z_p = y_p/d_p - (c_p/d_p) z_(p+1) are first-order linear
//     recurrences.  Each lane folds its NPL positions into one affine map (a sequential
//     pass), the warp scans the maps (Kogge-Stone, 5 shuffle steps), and each lane re-runs
//     its positions from the scanned carry.  The maps' multipliers depend only on the
//     tables, so their scan prefixes are computed once per kernel; each solve scans only
//     the offsets.  Same recurrences as the thread kernels, reassociated.
// Same arrays, layouts, modes (SWEEP, FINAL, PROLOGUE) and KParams as the other kernels.
#pragma once
#include "adi_line.cuh"

namespace adi {

constexpr int WK_LANES = 32;
constexpr int WK_WARPS = 4;     // lines (warps) per CTA
constexpr int WK_NPL_MAX = 12;  // positions per lane of the largest instantiation (384 per line)

// the LU tables of one system (u-op or x-op) staged per CTA: [l, 1/d, c/d][WK_LANES NPL],
// each entry 0 outside the system [lo, hi] (l also 0 at lo, c/d also 0 at hi)
__device__ __forceinline__ void wk_stage(double* t, int P, const double* tab, int n, int lo, int hi, int tid,
                                         int nthr) {
  const int n1 = n + 1;
  for (int q = tid; q < P; q += nthr) {
    const bool in = q >= lo && q <= hi;
    t[q] = (in && q > lo) ? tab[q] : 0.0;
    t[P + q] = in ? tab[n1 + q] : 0.0;
    t[2 * P + q] = (in && q < hi) ? tab[2 * n1 + q] * tab[n1 + q] : 0.0;
  }
}

// scan multipliers of the lane maps: forward y(last) = B + A y(first - 1), A = prod(-l);
// backward z(first) = C + A z(last + 1), A = prod(-m)
template <int NPL>
__device__ __forceinline__ void wk_prefix(const double* t, int lane, double (&fk)[5], double (&bk)[5]) {
  constexpr int P = WK_LANES * NPL;
  double fa = 1.0, ba = 1.0;
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    fa *= -t[NPL * lane + j];
    ba *= -t[2 * P + NPL * lane + j];
  }
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int d = 1 << s;
    fk[s] = fa;
    bk[s] = ba;
    const double fp = __shfl_up_sync(0xffffffffu, fa, d);
    const double bn = __shfl_down_sync(0xffffffffu, ba, d);
    if (lane >= d) fa *= fp;
    if (lane + d < WK_LANES) ba *= bn;
  }
}

// z = T^{-1} r on a staged system (r, z: this lane's NPL positions; 0 outside the system)
template <int NPL>
__device__ __forceinline__ void wk_solve(const double* t, const double (&fk)[5], const double (&bk)[5],
                                         const double (&r)[NPL], double (&z)[NPL], int lane) {
  constexpr int P = WK_LANES * NPL;
  const double* tl = t + NPL * lane;
  const double* ti = t + P + NPL * lane;
  const double* tm = t + 2 * P + NPL * lane;
  // forward: the lane's map from y_in = 0, inclusive scan, then y_in from lane - 1
  double B = 0.0;
#pragma unroll
  for (int j = 0; j < NPL; ++j) B = fma(-tl[j], B, r[j]);
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int d = 1 << s;
    const double Bp = __shfl_up_sync(0xffffffffu, B, d);
    if (lane >= d) B = fma(fk[s], Bp, B);
  }
  double y = __shfl_up_sync(0xffffffffu, B, 1);
  if (lane == 0) y = 0.0;
  double g[NPL];
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    y = fma(-tl[j], y, r[j]);
    g[j] = y * ti[j];
  }
  // backward: z_q = g_q - m_q z_(q+1); the lane's map from z_in = 0, suffix scan
  double C = 0.0;
#pragma unroll
  for (int j = NPL - 1; j >= 0; --j) C = fma(-tm[j], C, g[j]);
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int d = 1 << s;
    const double Cn = __shfl_down_sync(0xffffffffu, C, d);
    if (lane + d < WK_LANES) C = fma(bk[s], Cn, C);
  }
  double zz = __shfl_down_sync(0xffffffffu, C, 1);
  if (lane == WK_LANES - 1) zz = 0.0;
#pragma unroll
  for (int j = NPL - 1; j >= 0; --j) {
    zz = fma(-tm[j], zz, g[j]);
    z[j] = zz;
  }
}

// shared memory of a CTA: the CFD tables (2 systems x 3 x 32 NPL) and the operand
// buffers (WK_WARPS x 32 NPL) -- 13.8 KB at NPL = 12
template <int NPL>
constexpr size_t warp_smem_bytes() {
  return sizeof(double) * (size_t)(6 + WK_WARPS) * WK_LANES * NPL;
}

template <int METHOD, int MODE, int NPL>
__global__ void __launch_bounds__(32 * WK_WARPS) adi_warp_kernel(const __grid_constant__ KParams P) {
  constexpr int NP = WK_LANES * NPL;   // positions a warp holds
  extern __shared__ __align__(16) double wsm[];
  double* const tabU = wsm;               // CFD: [l, 1/d, c/d][NP] of the u-op system
  double* const tabX = wsm + 3 * NP;      // ... of the x-op system
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = P.n;
  if (METHOD == M_CFD) {
    wk_stage(tabU, NP, P.tabU, n, 1, n - 1, threadIdx.x, blockDim.x);
    wk_stage(tabX, NP, P.tabX, n, 0, n, threadIdx.x, blockDim.x);
    __syncthreads();
  }
  const int line = P.line0 + blockIdx.x * WK_WARPS + w;
  const int b = blockIdx.z;
  if (line < P.line_lo || line >= P.nlines) return;   // whole warps: no CTA barrier below
  double* const buf = wsm + 6 * NP + w * NP;
  const int q0 = NPL * lane;
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

  double fkU[5], bkU[5], fkX[5], bkX[5];
  if (METHOD == M_CFD) {
    wk_prefix<NPL>(tabU, lane, fkU, bkU);
    wk_prefix<NPL>(tabX, lane, fkX, bkX);
  }

  // the operand of an operator into the warp's buffer
  auto publish = [&](const double (&a)[NPL]) {
    __syncwarp();   // the previous operator's reads are done
#pragma unroll
    for (int j = 0; j < NPL; ++j) buf[q0 + j] = a[j];
    __syncwarp();
  };
  auto at = [&](int p) -> double { return buf[p < 0 ? 0 : (p >= NP ? NP - 1 : p)]; };

  // u-op: out_p = B_p - alpha D̄(x)_p on [1, uhi]; the other positions keep out's value
  auto uop = [&](const double (&xo)[NPL], const double (&B)[NPL], double (&out)[NPL]) {
    publish(xo);
    double r[NPL];
    if (METHOD == M_CFD) {
#pragma unroll
      for (int j = 0; j < NPL; ++j) {
        const int p = q0 + j;
        double v = 0.0;
        if (p == 1) v = (-at(0) - 9.0 * at(1) + 9.0 * at(2) + at(3)) * (1.0 / 3.0);
        else if (p == n - 1) v = (-at(n - 3) - 9.0 * at(n - 2) + 9.0 * at(n - 1) + at(n)) * (1.0 / 3.0);
        else if (p >= 2 && p <= n - 2) v = at(p + 1) - at(p - 1);
        r[j] = v;
      }
      double z[NPL];
      wk_solve<NPL>(tabU, fkU, bkU, r, z, lane);
#pragma unroll
      for (int j = 0; j < NPL; ++j) {
        const int p = q0 + j;
        if (p >= 1 && p <= n - 1) out[j] = fma(-P.cu, z[j], B[j]);
      }
    } else {
      const double a = P.cu, cA = P.mA, cB = P.mB;
#pragma unroll
      for (int j = 0; j < NPL; ++j) {
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
  auto xop = [&](const double (&uo)[NPL], const double (&B)[NPL], double (&out)[NPL]) {
    publish(uo);
    double r[NPL];
    if (METHOD == M_CFD) {
#pragma unroll
      for (int j = 0; j < NPL; ++j) {
        const int p = q0 + j;
        double v = 0.0;
        if (p == 0) v = (-17.0 * at(0) + 9.0 * at(1) + 9.0 * at(2) - at(3)) * (1.0 / 3.0);
        else if (p == n) v = (at(n - 3) - 9.0 * at(n - 2) - 9.0 * at(n - 1) + 17.0 * at(n)) * (1.0 / 3.0);
        else if (p >= 1 && p <= n - 1) v = at(p + 1) - at(p - 1);
        r[j] = v;
      }
      double z[NPL];
      wk_solve<NPL>(tabX, fkX, bkX, r, z, lane);
#pragma unroll
      for (int j = 0; j < NPL; ++j) {
        const int p = q0 + j;
        if (p <= n) out[j] = fma(-P.cx, z[j], B[j]);
      }
    } else {
      const double bb = P.cx, cC = P.mC, cD = P.mD;
#pragma unroll
      for (int j = 0; j < NPL; ++j) {
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

  // this lane's bases and state (positions q0 .. q0 + NPL - 1; 0 outside the line)
  double u[NPL], x[NPL], S[NPL], X[NPL];
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    const int p = q0 + j;
    X[j] = (p <= n) ? Xb[p] : 0.0;
    S[j] = (MODE != KM_PROLOGUE && Sb && p >= 1 && p <= uhi) ? Sb[p] : 0.0;
    u[j] = (MODE == KM_PROLOGUE && p <= pR) ? Ub[(long long)p * P.u_pt] : 0.0;
    x[j] = X[j];
  }
  double acc = 0.0;   // finiteness check (ADI_CHECK_FINITE)
  if (MODE == KM_PROLOGUE) {
    // W* = W - beta D(U) -> X_out; S1 = U + dt/2 F - alpha D̄(W) -> S_out (transposed)
    double ws[NPL];
#pragma unroll
    for (int j = 0; j < NPL; ++j) ws[j] = X[j];
    xop(u, X, ws);
    double* Xo = P.X_out + (long long)b * P.x_batch + (long long)line * P.x_line;
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      const int p = q0 + j;
      if (p <= n) { Xo[p] = ws[j]; acc += ws[j]; }
      if (p >= 1 && p <= uhi) u[j] = u[j] + src(p);
    }
    double o[NPL];
#pragma unroll
    for (int j = 0; j < NPL; ++j) o[j] = u[j];
    uop(x, u, o);
#pragma unroll
    for (int j = 0; j < NPL; ++j) u[j] = o[j];
  } else {
    // Dirichlet slots of ū
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
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
      double base[NPL], o[NPL];
#pragma unroll
      for (int j = 0; j < NPL; ++j) {
        const int p = q0 + j;
        base[j] = (p >= 1 && p <= uhi) ? u[j] + src(p) : u[j];
        o[j] = base[j];
      }
      uop(x, base, o);
#pragma unroll
      for (int j = 0; j < NPL; ++j) {
        u[j] = o[j];
        x[j] = fma(2.0, x[j], -X[j]);
      }
    }
  }
  // stores: S' (or U) transposed, X' along the line
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
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

// positions per lane for lines of n cells (n + 2 stored positions), 0 if too long
inline int warp_npl(int n) {
  for (int npl : {2, 4, 6, 8, 10, 12})
    if (n + 2 <= WK_LANES * npl) return npl;
  return 0;
}

}  // namespace adi
