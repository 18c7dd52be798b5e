// adi_kernels.cuh — sm_100a line-sweep kernels for the Peaceman–Rachford ADI
// step of arXiv:2006.07583 (CFD: App. A; MFD: PAPER.md:255-344,
// App. B; ADI iterations: App. C).
//
// ONE kernel template does a whole ADI half-step for a tile of grid lines:
//   load S (pressure-like carried field) and X (the velocity of this direction)
//   -> K fixed-point sweeps entirely on chip (eq. 8 / eq. 9):
//        u <- S - alpha D̄(x)          (u-op)
//        x <- X - beta  D([gL,u,gR])   (x-op)
//   -> epilogue (fused next explicit half): S' = u - alpha D̄(x) + dt/2 F(t1),
//      X' = x - beta D([gL,u,gR]) = 2x - X
//   -> store S', X'.
// The row sweep (lines = rows, x contiguous) and the column sweep (lines =
// columns) are the same code with different strides, so no transpose is ever
// materialised.  HBM traffic is 32 B per point per half-step (+8 B for a dense
// source) — DESIGN.md §5.
//
// Work decomposition: a CTA owns NL lines x (NT/NL) chunks of
// M consecutive points; each thread owns one chunk IN REGISTERS.  Long lines
// are cut into segments with a halo (MFD: exact, finite stencil support;
// CFD: the P^{-1} influence decays like (2-sqrt 3)^d).
// Chunks exchange edge values through shared memory once per operator
// application (one __syncthreads per op).
//
// CFD tridiagonal solves (P, P̄ with the global no-pivot LU)
// are split across chunks by a truncated SPIKE scheme: each chunk solves
// locally with zero carries, publishes (y_last, z_first, z_last), and adds the
// carry responses K_i*ycarry + J_i*zcarry; carries from >= 2 chunks away are
// below 1e-18 relative for M = 16 and are dropped.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace adi {

enum { M_CFD = 0, M_MFD = 1 };
enum { KM_SWEEP = 0, KM_FINAL = 1, KM_PROLOGUE = 2 };

struct Seg {
  int start;    // line position of the first point of chunk 0 (may be < 0)
  int nchunks;  // active chunks per line in this tile
  int out_lo;   // positions [out_lo, out_hi) are written by this tile
  int out_hi;
};

struct KParams {
  int n;        // cells along the line; positions 0..n
  int nlines;   // interior pressure lines
  int NL;       // lines per tile (power of two, divides NT)
  int plo, phi; // chunks entirely inside [plo, phi] use the interior fast path
  const Seg* segs;
  // fields: element of (batch b, line l, position p)
  const double* S_in;  double* S_out;  // S layout: b*s_batch + l*s_line + (p-1)*s_pt
  const double* X_in;  double* X_out;  // X layout: b*x_batch + l*x_line + p*x_pt
  const double* U_in;  double* U_out;  // U layout: b*u_batch + (l+1)*u_line + p*u_pt
  long long s_line, s_pt, s_batch;
  long long x_line, x_pt, x_batch;
  long long u_line, u_pt, u_batch;
  // Dirichlet data of this line's two ends: edgeL[l+1]*gb, edgeR[l+1]*gb
  const double* edgeL; const double* edgeR;
  double gb;
  // source F = phi*gf (+ point source pt_amp at (pt_line[b], pt_pos[b]))
  const double* phi_src; double gf;
  const int* pt_line; const int* pt_pos; double pt_amp;
  // operator scales
  double cu;        // u-op: alpha/h (MFD) or 3 alpha/h (CFD)
  double cx;        // x-op: beta/h  (MFD) or 3 beta/h  (CFD)
  double half_dt;
  int K;
  // CFD per-position LU tables, 3 x (n+1): l, 1/d, c   (u-op: P̄, x-op: P)
  const double* tabU; const double* tabX;
  int* flag;        // set to 1 if a non-finite value is stored
};

// ---------------------------------------------------------------------------
// constants (host fills them once; see adi_runtime.cu)
// ---------------------------------------------------------------------------
constexpr int MMAX = 32;
// MFD closures (App. B), interior (1/24, -9/8, 9/8, -1/24)
__constant__ double c_d4r0[6];   // D4 row 0
__constant__ double c_g4r0[6];   // G4 row 0
__constant__ double c_g4r1[5];   // G4 row 1
// CFD interior chunk (converged LU of tridiag(1,4,1)): multiplier l*, 1/d*,
// fix-up responses K_i (to ycarry) and J_i (to zcarry) for a chunk of M points
__constant__ double c_cl, c_cinvd;
__constant__ double c_cK[MMAX], c_cJ[MMAX];
__constant__ double c_cF, c_cKs, c_cKe, c_cJs, c_cJe;

// ---------------------------------------------------------------------------
// shared-memory exchange area
// ---------------------------------------------------------------------------
// dynamic slots: 2 buffers x 4 values;  static slots (CFD): 2 systems x 5 + 4
constexpr int DYN = 4;
constexpr int NSTAT = 14;
enum { ST_F = 0, ST_KS = 1, ST_KE = 2, ST_JS = 3, ST_JE = 4 };  // + 5*sys
enum { ST_SF = 10, ST_SL = 11, ST_VF = 12, ST_VL = 13 };        // base first/last

struct Xch {
  double* a;     // base of the exchange area
  int stride;    // entries per slot = NT + 4*NL
  int pad;       // 2*NL
  __device__ double* dyn(int buf, int k) const { return a + (buf * DYN + k) * stride + pad; }
  __device__ double* st(int k) const { return a + (2 * DYN + k) * stride + pad; }
};

__device__ __forceinline__ bool finite_(double v) { return isfinite(v); }

// ---------------------------------------------------------------------------
// Thread context
// ---------------------------------------------------------------------------
template <int M>
struct Ctx {
  int t, NL, line, chunk, s, n;  // s = line position of chunk element 0
  bool live;      // thread owns an existing chunk of an existing line
  bool interior;  // fast path allowed
  double gL, gR;  // Dirichlet values of this line for this half-step
};

// ===========================================================================
// MFD operators (App. B).  u at cb positions 1..n (cell centres), x at nodes
// 0..n; ū_0 = gL (slot u[pos 0]), ū_{n+1} = gR (scalar).
// ===========================================================================
template <int M>
struct Mfd {
  // u-op: out = B - a * D4 x  (a = alpha/h); neighbours xm2,xm1 (prev chunk), xp1
  template <bool INTERIOR>
  static __device__ __forceinline__ void uop(const Ctx<M>& c, const double (&x)[M],
                                             const double (&B)[M], double (&out)[M], double a,
                                             double xm2, double xm1, double xp1) {
    const double cA = a * (1.0 / 24.0), cB = a * (9.0 / 8.0);
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const double xl2 = (i >= 2) ? x[i - 2] : (i == 1 ? xm1 : xm2);
      const double xl1 = (i >= 1) ? x[i - 1] : xm1;
      const double xr1 = (i + 1 < M) ? x[i + 1] : xp1;
      if (INTERIOR) {
        out[i] = fma(cA, xr1 - xl2, fma(cB, xl1 - x[i], B[i]));
      } else {
        const int p = c.s + i;
        if (p >= 2 && p <= c.n - 1) {
          out[i] = fma(cA, xr1 - xl2, fma(cB, xl1 - x[i], B[i]));
        } else if (p == 1) {
          if (i >= 1 && i + 4 < M) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 6; ++k) s = fma(c_d4r0[k], x[i - 1 + k], s);
            out[i] = fma(-a, s, B[i]);
          }
        } else if (p == c.n) {
          if (i >= 5) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 6; ++k) s = fma(-c_d4r0[5 - k], x[i - 5 + k], s);
            out[i] = fma(-a, s, B[i]);
          }
        }
      }
    }
  }
  // x-op: out = B - b * G4 ū ; neighbours um1 (prev chunk), up1, up2 (next chunk)
  template <bool INTERIOR>
  static __device__ __forceinline__ void xop(const Ctx<M>& c, const double (&u)[M],
                                             const double (&B)[M], double (&out)[M], double b,
                                             double um1, double up1, double up2) {
    const double cC = b * (1.0 / 24.0), cD = b * (9.0 / 8.0);
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const double ul1 = (i >= 1) ? u[i - 1] : um1;
      const double ur1 = (i + 1 < M) ? u[i + 1] : up1;
      const double ur2 = (i + 2 < M) ? u[i + 2] : (i + 1 == M ? up2 : up1);
      if (INTERIOR) {
        out[i] = fma(cC, ur2 - ul1, fma(cD, u[i] - ur1, B[i]));
      } else {
        const int p = c.s + i;
        const int n = c.n;
        if (p >= 2 && p <= n - 2) {
          out[i] = fma(cC, ur2 - ul1, fma(cD, u[i] - ur1, B[i]));
        } else if (p == 0) {
          if (i + 5 < M) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 6; ++k) s = fma(c_g4r0[k], u[i + k], s);
            out[i] = fma(-b, s, B[i]);
          }
        } else if (p == 1) {
          if (i >= 1 && i + 3 < M) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 5; ++k) s = fma(c_g4r1[k], u[i - 1 + k], s);
            out[i] = fma(-b, s, B[i]);
          }
        } else if (p == n - 1) {
          if (i >= 2 && i + 1 < M) {
            // -reverse(g1) on ū_{n-3..n+1}; ū_{n+1} = gR
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) s = fma(-c_g4r1[4 - k], u[i - 2 + k], s);
            s = fma(-c_g4r1[0], c.gR, s);
            out[i] = fma(-b, s, B[i]);
          }
        } else if (p == n) {
          if (i >= 4) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 5; ++k) s = fma(-c_g4r0[5 - k], u[i - 4 + k], s);
            s = fma(-c_g4r0[0], c.gR, s);
            out[i] = fma(-b, s, B[i]);
          }
        }
      }
    }
  }
};

// ===========================================================================
// CFD operators (App. A).  x at nodes 0..n; u at nodes 1..n-1 with slots
// u[pos 0] = gL, u[pos n] = gR.  D̄ = P̄^{-1}Q̄ (u-op), D = P^{-1}Q (x-op).
// Stencil values are computed in units of (3/h)^{-1}: interior rows are
// f_{p+1} - f_{p-1}; the closure rows are divided by 3.
// ===========================================================================
template <int M>
struct Cfd {
  // raw stencil r of the u-op (Q̄ x) into r[]; needs x_{s-1}, x_{s+M}
  template <bool INTERIOR>
  static __device__ __forceinline__ void rhs_u(const Ctx<M>& c, const double (&x)[M],
                                               double (&r)[M], double xm1, double xp1) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const double xl = (i >= 1) ? x[i - 1] : xm1;
      const double xr = (i + 1 < M) ? x[i + 1] : xp1;
      if (INTERIOR) {
        r[i] = xr - xl;
      } else {
        const int p = c.s + i, n = c.n;
        double v = 0.0;
        if (p >= 2 && p <= n - 2) v = xr - xl;
        else if (p == 1) { if (i >= 1 && i + 2 < M) v = (-x[i - 1] - 9.0 * x[i] + 9.0 * x[i + 1] + x[i + 2]) * (1.0 / 3.0); }
        else if (p == n - 1) { if (i >= 2 && i + 1 < M) v = (-x[i - 2] - 9.0 * x[i - 1] + 9.0 * x[i] + x[i + 1]) * (1.0 / 3.0); }
        r[i] = v;
      }
    }
  }
  // raw stencil of the x-op (Q ū); needs ū_{s-1}, ū_{s+M}
  template <bool INTERIOR>
  static __device__ __forceinline__ void rhs_x(const Ctx<M>& c, const double (&u)[M],
                                               double (&r)[M], double um1, double up1) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const double ul = (i >= 1) ? u[i - 1] : um1;
      const double ur = (i + 1 < M) ? u[i + 1] : up1;
      if (INTERIOR) {
        r[i] = ur - ul;
      } else {
        const int p = c.s + i, n = c.n;
        double v = 0.0;
        if (p >= 1 && p <= n - 1) v = ur - ul;
        else if (p == 0) { if (i + 3 < M) v = (-17.0 * u[i] + 9.0 * u[i + 1] + 9.0 * u[i + 2] - u[i + 3]) * (1.0 / 3.0); }
        else if (p == n) { if (i >= 3) v = (u[i - 3] - 9.0 * u[i - 2] - 9.0 * u[i - 1] + 17.0 * u[i]) * (1.0 / 3.0); }
        r[i] = v;
      }
    }
  }
};

}  // namespace adi

namespace adi {

// ===========================================================================
// CFD: one operator application out = B - coef * T^{-1} r(o) on the tile
// (T = P̄ for the u-op, P for the x-op), truncated-SPIKE across chunks.
// Phase 1 (local solve, publish), __syncthreads, phase 2 (carries, fix-up).
// Also returns the operand neighbour values of the NEXT op (this op's output
// at the previous chunk's last and the next chunk's first position) without a
// second barrier.
// ===========================================================================
template <int M, bool UOP>
__device__ __forceinline__ void cfd_apply(const Ctx<M>& c, const KParams& P, const Xch& X,
                                          int buf, const double (&o)[M], const double (&B)[M],
                                          double (&out)[M], double coef, double om1, double op1,
                                          double& nom1, double& nop1) {
  const int t = c.t, NL = c.NL;
  const int sys = UOP ? 0 : 1;
  const double* tab = UOP ? P.tabU : P.tabX;
  const int np1 = c.n + 1;
  double yl_e, ws, we;
  // ---------------- phase 1: local solve with zero carries ----------------
  if (c.interior) {
    if (UOP) Cfd<M>::template rhs_u<true>(c, o, out, om1, op1);
    else Cfd<M>::template rhs_x<true>(c, o, out, om1, op1);
    const double l = c_cl, iv = c_cinvd;
    out[0] = out[0];
#pragma unroll
    for (int i = 1; i < M; ++i) out[i] = fma(-l, out[i - 1], out[i]);
    yl_e = out[M - 1];
#pragma unroll
    for (int i = M - 2; i >= 0; --i) out[i] = fma(-iv, out[i + 1], out[i]);
    ws = iv * out[0];
    we = iv * out[M - 1];
  } else {
    if (UOP) Cfd<M>::template rhs_u<false>(c, o, out, om1, op1);
    else Cfd<M>::template rhs_x<false>(c, o, out, om1, op1);
    double yp = 0.0;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const int p = c.s + i;
      const double l = (p >= 0 && p < np1) ? __ldg(tab + p) : 0.0;
      out[i] = fma(-l, yp, out[i]);
      yp = out[i];
    }
    yl_e = out[M - 1];
    double z = 0.0;
    we = 0.0;
#pragma unroll
    for (int i = M - 1; i >= 0; --i) {
      const int p = c.s + i;
      const bool in = (p >= 0 && p < np1);
      const double iv = in ? __ldg(tab + np1 + p) : 0.0;
      const double cc = in ? __ldg(tab + 2 * np1 + p) : 0.0;
      z = (out[i] - cc * z) * iv;
      if (i == M - 1) we = z;
    }
    ws = z;
  }
  if (!c.live) { yl_e = 0.0; ws = 0.0; we = 0.0; }
  X.dyn(buf, 0)[t] = yl_e;
  X.dyn(buf, 1)[t] = ws;
  X.dyn(buf, 2)[t] = we;
  __syncthreads();
  // ---------------- phase 2: carries and fix-up ----------------
  const double ylm1 = X.dyn(buf, 0)[t - NL], ylm2 = X.dyn(buf, 0)[t - 2 * NL];
  const double ylp1 = X.dyn(buf, 0)[t + NL];
  const double wsp1 = X.dyn(buf, 1)[t + NL], wsp2 = X.dyn(buf, 1)[t + 2 * NL];
  const double wem1 = X.dyn(buf, 2)[t - NL];
  const int so = 5 * sys;
  const double Fm1 = X.st(so + ST_F)[t - NL], Fme = X.st(so + ST_F)[t];
  const double Ksp1 = X.st(so + ST_KS)[t + NL], Jsp1 = X.st(so + ST_JS)[t + NL];
  const double Ksp2 = X.st(so + ST_KS)[t + 2 * NL];
  const double Kem1 = X.st(so + ST_KE)[t - NL], Jem1 = X.st(so + ST_JE)[t - NL];
  const double ycarry = fma(Fm1, ylm2, ylm1);            // true y at s-1
  const double ycn = fma(Fme, ycarry, yl_e);             // true y at s+M-1
  const double zcarry = fma(Jsp1, fma(Ksp2, ylp1, wsp2), fma(Ksp1, ycn, wsp1));  // true z at s+M
  double z0;
  if (c.interior) {
    const double iv = c_cinvd;
    z0 = fma(c_cJ[0], zcarry, fma(c_cK[0], ycarry, iv * out[0]));
    const double cy = coef * ycarry, cz = coef * zcarry, ci = coef * iv;
#pragma unroll
    for (int i = 0; i < M; ++i) out[i] = fma(-c_cJ[i], cz, fma(-c_cK[i], cy, fma(-ci, out[i], B[i])));
  } else {
    double g = 1.0;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const int p = c.s + i;
      const double l = (p >= 0 && p < np1) ? __ldg(tab + p) : 0.0;
      g *= -l;
      out[i] = fma(g, ycarry, out[i]);
    }
    double z = zcarry;
#pragma unroll
    for (int i = M - 1; i >= 0; --i) {
      const int p = c.s + i;
      const bool in = (p >= 0 && p < np1);
      const double iv = in ? __ldg(tab + np1 + p) : 0.0;
      const double cc = in ? __ldg(tab + 2 * np1 + p) : 0.0;
      z = (out[i] - cc * z) * iv;
      out[i] = z;
    }
    z0 = out[0];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const int p = c.s + i;
      const bool act = UOP ? (p >= 1 && p <= c.n - 1) : (p >= 0 && p <= c.n);
      double slot = 0.0;
      if (UOP) slot = (p == 0) ? c.gL : ((p == c.n) ? c.gR : 0.0);
      out[i] = act ? fma(-coef, out[i], B[i]) : slot;
    }
  }
  // operand neighbours of the next op
  nop1 = fma(-coef, zcarry, X.st(UOP ? ST_SF : ST_VF)[t + NL]);
  nom1 = fma(-coef, fma(Jem1, z0, fma(Kem1, ylm2, wem1)), X.st(UOP ? ST_SL : ST_VL)[t - NL]);
}

// CFD statics of a chunk for one system: F, K_s, K_e, J_s, J_e
template <int M>
__device__ __forceinline__ void cfd_statics(const Ctx<M>& c, const double* tab, int np1,
                                            double& F, double& Ks, double& Ke, double& Js,
                                            double& Je) {
  if (c.interior) {
    F = c_cF; Ks = c_cKs; Ke = c_cKe; Js = c_cJs; Je = c_cJe;
    return;
  }
  double G[M];
  double g = 1.0;
#pragma unroll
  for (int i = 0; i < M; ++i) {
    const int p = c.s + i;
    const double l = (p >= 0 && p < np1) ? __ldg(tab + p) : 0.0;
    g *= -l;
    G[i] = g;
  }
  F = G[M - 1];
  double k = 0.0, j = 1.0;
#pragma unroll
  for (int i = M - 1; i >= 0; --i) {
    const int p = c.s + i;
    const bool in = (p >= 0 && p < np1);
    const double iv = in ? __ldg(tab + np1 + p) : 0.0;
    const double cc = in ? __ldg(tab + 2 * np1 + p) : 0.0;
    k = (G[i] - cc * k) * iv;
    j *= -cc * iv;
    if (i == M - 1) { Ke = k; Je = j; }
  }
  Ks = k;
  Js = j;
}

// ===========================================================================
// MFD: publish the first two / last two values of a chunk array and read the
// neighbours' (one __syncthreads).
// ===========================================================================
template <int M>
__device__ __forceinline__ void mfd_exchange(const Ctx<M>& c, const Xch& X, int buf,
                                             const double (&a)[M], double& m2, double& m1,
                                             double& p1, double& p2) {
  const int t = c.t, NL = c.NL;
  X.dyn(buf, 0)[t] = c.live ? a[0] : 0.0;
  X.dyn(buf, 1)[t] = c.live ? a[1] : 0.0;
  X.dyn(buf, 2)[t] = c.live ? a[M - 2] : 0.0;
  X.dyn(buf, 3)[t] = c.live ? a[M - 1] : 0.0;
  __syncthreads();
  m2 = X.dyn(buf, 2)[t - NL];
  m1 = X.dyn(buf, 3)[t - NL];
  p1 = X.dyn(buf, 0)[t + NL];
  p2 = X.dyn(buf, 1)[t + NL];
}

// ===========================================================================
// The tile kernel.
// ===========================================================================
template <int METHOD, int M, int NT, int MODE>
__global__ void __launch_bounds__(NT, 1) adi_tile_kernel(const KParams P) {
  extern __shared__ double smem[];
  const int t = threadIdx.x;
  const int NL = P.NL;
  const Seg sg = P.segs[blockIdx.y];
  const int l = t & (NL - 1);
  const int ch = t / NL;
  const int line = blockIdx.x * NL + l;
  const long long b = blockIdx.z;
  const int n = P.n;

  Ctx<M> c;
  c.t = t; c.NL = NL; c.line = line; c.chunk = ch; c.n = n;
  c.s = sg.start + ch * M;
  c.live = (line < P.nlines) && (ch < sg.nchunks);
  c.interior = c.live && c.s >= P.plo && c.s + M - 1 <= P.phi;

  Xch X;
  X.stride = NT + 4 * NL;
  X.pad = 2 * NL;
  X.a = smem;
  for (int k = t; k < (2 * DYN + NSTAT) * X.stride; k += NT) smem[k] = 0.0;

  // ---- Dirichlet values of this line (ū at position 0 and at n (CFD) / n+1 (MFD))
  const int pR = (METHOD == M_CFD) ? n : n + 1;
  const double* Ub = P.U_in + b * P.u_batch + (long long)(line + 1) * P.u_line;
  c.gL = 0.0; c.gR = 0.0;
  if (c.live) {
    if (MODE == KM_PROLOGUE) {
      c.gL = Ub[0];
      c.gR = Ub[(long long)pR * P.u_pt];
    } else {
      if (P.edgeL) c.gL = P.edgeL[line + 1] * P.gb;
      if (P.edgeR) c.gR = P.edgeR[line + 1] * P.gb;
    }
  }
  const int uhi = (METHOD == M_CFD) ? n - 1 : n;  // u active on [1, uhi]

  // ---- load the chunk
  double u[M], x[M], S[M], V[M];
  const double* Sb = P.S_in + b * P.s_batch + (long long)line * P.s_line;
  const double* Xb = P.X_in + b * P.x_batch + (long long)line * P.x_line;
#pragma unroll
  for (int i = 0; i < M; ++i) {
    const int p = c.s + i;
    const bool xin = c.live && p >= 0 && p <= n;
    const bool uin = c.live && p >= 1 && p <= uhi;
    x[i] = xin ? Xb[(long long)p * P.x_pt] : 0.0;
    V[i] = x[i];
    if (MODE == KM_PROLOGUE) {
      u[i] = (c.live && p >= 0 && p <= n) ? Ub[(long long)p * P.u_pt] : 0.0;
      S[i] = 0.0;
    } else {
      S[i] = uin ? Sb[(long long)(p - 1) * P.s_pt] : 0.0;
      u[i] = (p == 0) ? c.gL : ((METHOD == M_CFD && p == n) ? c.gR : 0.0);
      if (!c.live) u[i] = 0.0;
    }
  }
  __syncthreads();  // exchange area zeroed

  // source factor at this chunk's points, dt/2 F(t)
  auto add_source = [&](double (&dst)[M], const double (&src)[M]) {
    const double* ph = P.phi_src ? P.phi_src + (long long)line * P.s_line : nullptr;
    const int ptl = P.pt_line ? P.pt_line[b] : -1;
    const int ptp = P.pt_pos ? P.pt_pos[b] : -1;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const int p = c.s + i;
      const bool uin = c.live && p >= 1 && p <= uhi;
      double f = 0.0;
      if (uin && ph) f = ph[(long long)(p - 1) * P.s_pt] * P.gf;
      if (uin && line == ptl && p == ptp) f += P.pt_amp * P.gf;
      dst[i] = fma(P.half_dt, f, src[i]);
    }
  };

  if (METHOD == M_CFD) {
    // ---------------- CFD ----------------
    const int np1 = n + 1;
    if (c.live) {
      double F, Ks, Ke, Js, Je;
      cfd_statics<M>(c, P.tabU, np1, F, Ks, Ke, Js, Je);
      X.st(ST_F)[t] = F; X.st(ST_KS)[t] = Ks; X.st(ST_KE)[t] = Ke; X.st(ST_JS)[t] = Js; X.st(ST_JE)[t] = Je;
      cfd_statics<M>(c, P.tabX, np1, F, Ks, Ke, Js, Je);
      X.st(5 + ST_F)[t] = F; X.st(5 + ST_KS)[t] = Ks; X.st(5 + ST_KE)[t] = Ke; X.st(5 + ST_JS)[t] = Js; X.st(5 + ST_JE)[t] = Je;
      X.st(ST_SF)[t] = S[0]; X.st(ST_SL)[t] = S[M - 1];
      X.st(ST_VF)[t] = V[0]; X.st(ST_VL)[t] = V[M - 1];
      // initial operand exchange: x (and u in the prologue)
      X.dyn(1, 0)[t] = x[0]; X.dyn(1, 1)[t] = x[M - 1];
      X.dyn(1, 2)[t] = u[0]; X.dyn(1, 3)[t] = u[M - 1];
    }
    __syncthreads();
    double xm1 = X.dyn(1, 1)[t - NL], xp1 = X.dyn(1, 0)[t + NL];
    double um1 = X.dyn(1, 3)[t - NL], up1 = X.dyn(1, 2)[t + NL];
    __syncthreads();  // buffer 1 is reused by the second op
    if (MODE == KM_PROLOGUE) {
      double d1, d2;
      cfd_apply<M, false>(c, P, X, 0, u, V, x, P.cx, um1, up1, d1, d2);  // W* = W - beta D(U)
      add_source(S, u);                                                    // S = U + dt/2 F
      cfd_apply<M, true>(c, P, X, 1, V, S, u, P.cu, xm1, xp1, d1, d2);     // S1 = S - alpha D̄(W)
    } else {
      int buf = 0;
      for (int k = 0; k < P.K; ++k) {
        cfd_apply<M, true>(c, P, X, buf, x, S, u, P.cu, xm1, xp1, um1, up1);
        buf ^= 1;
        cfd_apply<M, false>(c, P, X, buf, u, V, x, P.cx, um1, up1, xm1, xp1);
        buf ^= 1;
      }
      if (MODE == KM_SWEEP) {
        double d1, d2;
        add_source(S, u);
        cfd_apply<M, true>(c, P, X, buf, x, S, u, P.cu, xm1, xp1, d1, d2);
#pragma unroll
        for (int i = 0; i < M; ++i) x[i] = fma(2.0, x[i], -V[i]);
      }
    }
  } else {
    // ---------------- MFD ----------------
    double xm2, xm1, xp1, xp2, um2, um1, up1, up2;
    mfd_exchange<M>(c, X, 0, x, xm2, xm1, xp1, xp2);
    const double au = P.cu, bx = P.cx;
    if (MODE == KM_PROLOGUE) {
      mfd_exchange<M>(c, X, 1, u, um2, um1, up1, up2);
      if (c.interior) Mfd<M>::template xop<true>(c, u, V, x, bx, um1, up1, up2);
      else Mfd<M>::template xop<false>(c, u, V, x, bx, um1, up1, up2);
      add_source(S, u);
      if (c.interior) Mfd<M>::template uop<true>(c, V, S, u, au, xm2, xm1, xp1);
      else Mfd<M>::template uop<false>(c, V, S, u, au, xm2, xm1, xp1);
    } else {
      int buf = 1;
      for (int k = 0; k < P.K; ++k) {
        if (c.interior) Mfd<M>::template uop<true>(c, x, S, u, au, xm2, xm1, xp1);
        else Mfd<M>::template uop<false>(c, x, S, u, au, xm2, xm1, xp1);
        mfd_exchange<M>(c, X, buf, u, um2, um1, up1, up2);
        buf ^= 1;
        if (c.interior) Mfd<M>::template xop<true>(c, u, V, x, bx, um1, up1, up2);
        else Mfd<M>::template xop<false>(c, u, V, x, bx, um1, up1, up2);
        if (k + 1 < P.K || MODE == KM_SWEEP) {
          mfd_exchange<M>(c, X, buf, x, xm2, xm1, xp1, xp2);
          buf ^= 1;
        }
      }
      if (MODE == KM_SWEEP) {
        add_source(S, u);
        if (c.interior) Mfd<M>::template uop<true>(c, x, S, u, au, xm2, xm1, xp1);
        else Mfd<M>::template uop<false>(c, x, S, u, au, xm2, xm1, xp1);
#pragma unroll
        for (int i = 0; i < M; ++i) x[i] = fma(2.0, x[i], -V[i]);
      }
    }
  }

  // ---- store the owned output range
  if (!c.live) return;
  double acc = 0.0;
  double* So = P.S_out + b * P.s_batch + (long long)line * P.s_line;
  double* Xo = P.X_out + b * P.x_batch + (long long)line * P.x_line;
  double* Uo = P.U_out ? P.U_out + b * P.u_batch + (long long)(line + 1) * P.u_line : nullptr;
#pragma unroll
  for (int i = 0; i < M; ++i) {
    const int p = c.s + i;
    if (p < sg.out_lo || p >= sg.out_hi || p < 0 || p > n) continue;
    Xo[(long long)p * P.x_pt] = x[i];
    acc += x[i];
    if (MODE == KM_FINAL) {
      Uo[(long long)p * P.u_pt] = u[i];  // interior values and the Dirichlet slots
      acc += u[i];
      if (METHOD == M_MFD && p == n) Uo[(long long)(n + 1) * P.u_pt] = c.gR;
      if (METHOD == M_MFD && p == 0) Uo[0] = c.gL;
    } else if (p >= 1 && p <= uhi) {
      So[(long long)(p - 1) * P.s_pt] = u[i];
      acc += u[i];
    }
  }
  if (P.flag && !finite_(acc)) atomicOr(P.flag, 1);
}

}  // namespace adi
