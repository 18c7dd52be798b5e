// adi_line.cuh — sm_100a line-sweep kernels for the Peaceman–Rachford ADI step
// of arXiv:2006.07583 (CFD: App. A; MFD: PAPER.md:255-344,
// App. B; ADI iterations: App. C).
//
// ONE kernel template performs a whole ADI half-step for NW grid lines:
//   load S (pressure-like carried field) and X (the velocity of this direction)
//   -> K fixed-point sweeps entirely on chip (eq. 8 / eq. 9):
//        u <- S - alpha D̄(x)          (u-op)
//        x <- X - beta  D([gL,u,gR])   (x-op)
//   -> epilogue (the next explicit half, fused): S' = u - alpha D̄(x) + dt/2 F,
//      X' = x - beta D([gL,u,gR]) = 2x - X
//   -> store S' and X'.
//
// Layout.  Every kernel reads its lines CONTIGUOUSLY: the row
// sweep reads S and V̄ row-major, the column sweep reads S^T and W̄^T.  The
// carried field S changes layout every half-step: each kernel writes S'
// transposed (NW consecutive lines give NW*8-byte runs), so the next sweep
// again reads contiguous lines.  No explicit transpose kernel runs in a step.
//
// Decomposition.  One WARP owns one segment of one line:
// lane l owns chunk l of M consecutive points, the iterated u and x in
// registers, the read-only bases S and X in a padded shared-memory tile.
// Neighbouring chunks exchange edge values by warp shuffles only — no shared
// mailbox, no barrier inside the sweeps.  Long lines are cut into 32*M-point
// segments with a halo (MFD: exact, finite stencil support; CFD: the P^{-1}
// influence decays like (2-sqrt 3)^d).
//
// CFD tridiagonal solves (P, P̄, global no-pivot LU) are
// split across chunks by a truncated SPIKE scheme (local solve, exchange of
// (y_last, z_first, z_last), carry fix-up) and, inside a
// chunk, across NSUB interleaved sub-chunks for instruction-level parallelism.
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

// Lines and positions are grid POSITIONS (the line index is the position in the
// cross direction; interior lines are 1..).  Element (batch b, line L, position p):
//   S_in : b*s_batch + L*s_line  + p          (lines contiguous)
//   X_in : b*x_batch + L*x_line  + p
//   S_out: b*s_batch + L*so_line + p*so_pt    (written transposed)
//   X_out: b*x_batch + L*x_line  + p
//   U_in / U_out: b*u_batch + L*u_line + p*u_pt  (prologue / final)
struct KParams {
  int n;        // cells along the line; positions 0..n
  int line0;    // line of (blockIdx.x = 0, warp 0); 4-aligned
  int line_lo;  // lines [line_lo, nlines) are processed
  int nlines;
  int plo, phi; // chunks entirely inside [plo, phi] use the interior fast path
  const Seg* segs;
  const double* S_in;  double* S_out;
  const double* X_in;  double* X_out;
  const double* U_in;  double* U_out;
  long long s_line, so_line, so_pt, s_batch;
  long long x_line, x_batch;
  long long u_line, u_pt, u_batch;
  // Dirichlet data of this line's two ends: edgeL[l+1]*gb, edgeR[l+1]*gb
  const double* edgeL; const double* edgeR;
  double gb;
  // source F = phi*gf (+ point source pt_amp at (pt_line[b], pt_pos[b])); phi in S_in layout
  const double* phi_src; double gf;
  const int* pt_line; const int* pt_pos; double pt_amp;
  double cu;        // u-op scale: alpha/h (MFD) or 3 alpha/h (CFD)
  double cx;        // x-op scale: beta/h  (MFD) or 3 beta/h  (CFD)
  double half_dt;
  int K;
  // CFD per-position LU tables, 3 x (n+1): l, 1/d, c   (u-op: P̄, x-op: P)
  const double* tabU; const double* tabX;
  int* flag;        // set to 1 if a non-finite value is stored
};

constexpr int MMAX = 64;
// MFD closures (App. B), interior (1/24, -9/8, 9/8, -1/24)
__constant__ double c_d4r0[6];   // D4 row 0
__constant__ double c_g4r0[6];   // G4 row 0
__constant__ double c_g4r1[5];   // G4 row 1
// CFD interior chunk (converged LU of tridiag(1,4,1)): multiplier l*, 1/d*,
// chunk-level responses (for the neighbours' carries) and sub-chunk responses
__constant__ double c_cl, c_cinvd;
__constant__ double c_cF, c_cKs, c_cKe, c_cJs, c_cJe;
__constant__ double c_sK[MMAX], c_sJ[MMAX];
__constant__ double c_sF;
enum { ST_F = 0, ST_KS = 1, ST_KE = 2, ST_JS = 3, ST_JE = 4 };  // CFD chunk statics

template <int M>
struct Ctx {
  int t, line, chunk, s, n;  // s = line position of chunk element 0
  bool live;      // thread owns an existing chunk of an existing line
  bool interior;  // fast path allowed
  bool nbint;     // chunks c-2 .. c+2 all exist and are interior (CFD constant statics)
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
                                             const double* __restrict__ B, double (&out)[M], double a,
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
                                             const double* __restrict__ B, double (&out)[M], double b,
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


template <int M>
struct MfdSplit {
  // load the op's bases into the (dead) output registers: one burst of 128-bit
  // shared loads, issued before any arithmetic so their latency overlaps
  static __device__ __forceinline__ void bases(const double* __restrict__ B, double (&out)[M]) {
    const double2* B2 = reinterpret_cast<const double2*>(B);
#pragma unroll
    for (int i = 0; i < M / 2; ++i) {
      const double2 v = B2[i];
      out[2 * i] = v.x;
      out[2 * i + 1] = v.y;
    }
  }
  // u-op: out_i = B_i + cA (x_{i+1} - x_{i-2}) + cB (x_{i-1} - x_i), out preloaded with B
  static __device__ __forceinline__ void u_inner(const double (&x)[M], double (&out)[M], double cA,
                                                 double cB) {
#pragma unroll
    for (int i = 2; i <= M - 2; ++i) out[i] = fma(cA, x[i + 1] - x[i - 2], fma(cB, x[i - 1] - x[i], out[i]));
  }
  static __device__ __forceinline__ void u_edges(const double (&x)[M], double (&out)[M], double cA,
                                                 double cB, double xm2, double xm1, double xp1) {
    out[0] = fma(cA, x[1] - xm2, fma(cB, xm1 - x[0], out[0]));
    out[1] = fma(cA, x[2] - xm1, fma(cB, x[0] - x[1], out[1]));
    out[M - 1] = fma(cA, xp1 - x[M - 3], fma(cB, x[M - 2] - x[M - 1], out[M - 1]));
  }
  // x-op: out_i = B_i + cC (u_{i+2} - u_{i-1}) + cD (u_i - u_{i+1}), out preloaded with B
  static __device__ __forceinline__ void x_inner(const double (&u)[M], double (&out)[M], double cC,
                                                 double cD) {
#pragma unroll
    for (int i = 1; i <= M - 3; ++i) out[i] = fma(cC, u[i + 2] - u[i - 1], fma(cD, u[i] - u[i + 1], out[i]));
  }
  static __device__ __forceinline__ void x_edges(const double (&u)[M], double (&out)[M], double cC,
                                                 double cD, double um1, double up1, double up2) {
    out[0] = fma(cC, u[2] - um1, fma(cD, u[0] - u[1], out[0]));
    out[M - 2] = fma(cC, up1 - u[M - 3], fma(cD, u[M - 2] - u[M - 1], out[M - 2]));
    out[M - 1] = fma(cC, up2 - u[M - 2], fma(cD, u[M - 1] - up1, out[M - 1]));
  }
};

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
// TMA bulk copies (cp.async.bulk) with per-warp mbarrier completion
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!ok);
}
// global -> shared, `bytes` (multiple of 16, 16-byte aligned ends), completes on mbarrier
__device__ __forceinline__ void bulk_g2s(double* dst, const double* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// shared -> global (bulk group)
__device__ __forceinline__ void bulk_s2g(double* dst, const double* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void fence_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ double shup(double v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }
__device__ __forceinline__ double shdn(double v, int d) { return __shfl_down_sync(0xffffffffu, v, d); }

// prev chunk's a[M-2], a[M-1]; next chunk's a[0], a[1] (0 outside the warp's segment)
template <int M>
__device__ __forceinline__ void warp_edges(int lane, const double (&a)[M], double& pm2, double& pm1,
                                           double& np1, double& np2) {
  pm2 = shup(a[M - 2], 1);
  pm1 = shup(a[M - 1], 1);
  np1 = shdn(a[0], 1);
  np2 = shdn(a[1], 1);
  pm2 = lane == 0 ? 0.0 : pm2;
  pm1 = lane == 0 ? 0.0 : pm1;
  np1 = lane == 31 ? 0.0 : np1;
  np2 = lane == 31 ? 0.0 : np2;
}

template <int M>
__device__ __forceinline__ void cfd_statics(const Ctx<M>& c, const double* tab, int np1,
                                            double* st /* 5 */) {
  if (c.interior) {
    st[0] = c_cF; st[1] = c_cKs; st[2] = c_cKe; st[3] = c_cJs; st[4] = c_cJe;
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
  st[0] = G[M - 1];
  double k = 0.0, j = 1.0;
#pragma unroll
  for (int i = M - 1; i >= 0; --i) {
    const int p = c.s + i;
    const bool in = (p >= 0 && p < np1);
    const double iv = in ? __ldg(tab + np1 + p) : 0.0;
    const double cc = in ? __ldg(tab + 2 * np1 + p) : 0.0;
    k = (G[i] - cc * k) * iv;
    j *= -cc * iv;
    if (i == M - 1) { st[2] = k; st[4] = j; }
  }
  st[1] = k;
  st[3] = j;
}


constexpr int NSUB = 4;

// ===========================================================================
// CFD: one operator application out = B - coef * T^{-1} r(o) on the warp's
// segment (T = P̄ for the u-op, P for the x-op).  Phase 1: local solve with
// zero carries (NSUB interleaved sub-chunks); exchange (y_e, z_s, z_e) by
// shuffles; phase 2: carries + fix-up.  Also returns this op's output at the
// previous chunk's last and the next chunk's first position (the operand
// neighbours of the next op).  st: statics of this warp's chunks [5][32].
// ===========================================================================
template <int M, bool UOP>
__device__ __forceinline__ void cfd_apply(const Ctx<M>& c, const KParams& P, int lane,
                                          const double* st, const double (&o)[M],
                                          const double* __restrict__ B, double (&out)[M],
                                          double coef, double om1, double op1, double Bn_first,
                                          double Bp_last, double& nom1, double& nop1) {
  constexpr int L = M / NSUB;
  const double* tab = UOP ? P.tabU : P.tabX;
  const int np1 = c.n + 1;
  double yl_e, ws, we;
  double ysub[NSUB];
  // ---------------- phase 1: local solve with zero carries ----------------
  if (c.interior) {
    if (UOP) Cfd<M>::template rhs_u<true>(c, o, out, om1, op1);
    else Cfd<M>::template rhs_x<true>(c, o, out, om1, op1);
    const double l = c_cl, iv = c_cinvd, FL = c_sF;
#pragma unroll
    for (int i = 1; i < L; ++i)
#pragma unroll
      for (int j = 0; j < NSUB; ++j) out[j * L + i] = fma(-l, out[j * L + i - 1], out[j * L + i]);
#pragma unroll
    for (int j = 0; j < NSUB; ++j) ysub[j] = out[j * L + L - 1];
#pragma unroll
    for (int i = L - 2; i >= 0; --i)
#pragma unroll
      for (int j = 0; j < NSUB; ++j) out[j * L + i] = fma(-iv, out[j * L + i + 1], out[j * L + i]);
    double Y[NSUB];
    Y[0] = ysub[0];
#pragma unroll
    for (int j = 1; j < NSUB; ++j) Y[j] = fma(FL, Y[j - 1], ysub[j]);
    yl_e = Y[NSUB - 1];
    double zc = 0.0;
#pragma unroll
    for (int j = NSUB - 2; j >= 0; --j) zc = fma(c_sJ[0], zc, fma(c_sK[0], Y[j], iv * out[(j + 1) * L]));
    ws = fma(c_sJ[0], zc, iv * out[0]);
    we = fma(c_sK[L - 1], Y[NSUB - 2], iv * out[M - 1]);
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
  // ---------------- exchange (shuffles) ----------------
  double ylm1 = shup(yl_e, 1), ylm2 = shup(yl_e, 2), ylp1 = shdn(yl_e, 1);
  double wsp1 = shdn(ws, 1), wsp2 = shdn(ws, 2), wem1 = shup(we, 1);
  ylm1 = lane == 0 ? 0.0 : ylm1;
  ylm2 = lane <= 1 ? 0.0 : ylm2;
  wem1 = lane == 0 ? 0.0 : wem1;
  ylp1 = lane == 31 ? 0.0 : ylp1;
  wsp1 = lane == 31 ? 0.0 : wsp1;
  wsp2 = lane >= 30 ? 0.0 : wsp2;
  double Fm1, Fme, Ksp1, Jsp1, Ksp2, Kem1, Jem1;
  if (c.nbint) {
    Fm1 = Fme = c_cF; Ksp1 = Ksp2 = c_cKs; Jsp1 = c_cJs; Kem1 = c_cKe; Jem1 = c_cJe;
  } else {
    auto at = [&](int k, int cc) { return (cc >= 0 && cc < 32) ? st[k * 32 + cc] : 0.0; };
    Fm1 = at(ST_F, lane - 1); Fme = at(ST_F, lane);
    Ksp1 = at(ST_KS, lane + 1); Jsp1 = at(ST_JS, lane + 1); Ksp2 = at(ST_KS, lane + 2);
    Kem1 = at(ST_KE, lane - 1); Jem1 = at(ST_JE, lane - 1);
  }
  // ---------------- phase 2: carries and fix-up ----------------
  const double ycarry = fma(Fm1, ylm2, ylm1);   // true y at s-1
  const double ycn = fma(Fme, ycarry, yl_e);    // true y at s+M-1
  const double zcarry = fma(Jsp1, fma(Ksp2, ylp1, wsp2), fma(Ksp1, ycn, wsp1));  // true z at s+M
  double z0;
  if (c.interior) {
    const double iv = c_cinvd, FL = c_sF;
    double ycT[NSUB], zcT[NSUB];
    ycT[0] = ycarry;
#pragma unroll
    for (int j = 1; j < NSUB; ++j) ycT[j] = fma(FL, ycT[j - 1], ysub[j - 1]);
    zcT[NSUB - 1] = zcarry;
#pragma unroll
    for (int j = NSUB - 2; j >= 0; --j)
      zcT[j] = fma(c_sJ[0], zcT[j + 1], fma(c_sK[0], ycT[j + 1], iv * out[(j + 1) * L]));
    z0 = fma(c_sJ[0], zcT[0], fma(c_sK[0], ycT[0], iv * out[0]));
    const double ci = coef * iv;
#pragma unroll
    for (int j = 0; j < NSUB; ++j) {
      const double cy = coef * ycT[j], cz = coef * zcT[j];
#pragma unroll
      for (int i = 0; i < L; ++i)
        out[j * L + i] = fma(-c_sJ[i], cz, fma(-c_sK[i], cy, fma(-ci, out[j * L + i], B[j * L + i])));
    }
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
  nop1 = fma(-coef, zcarry, Bn_first);
  nom1 = fma(-coef, fma(Jem1, z0, fma(Kem1, ylm2, wem1)), Bp_last);
}

// Occupancy targets (resident CTAs per SM) for the NW-warp CTAs.
template <int METHOD>
struct Occ {
  static constexpr int value = (METHOD == M_MFD) ? 3 : 2;
};

// shared memory of one CTA: padded staging of S and X for NW lines (+ CFD statics)
template <int METHOD, int M, int NW>
constexpr size_t line_smem_bytes() {
  return sizeof(double) * (size_t)(2 * NW * (32 * (M + 2) + 4) + (METHOD == M_CFD ? NW * 10 * 32 : 0) + NW);
}

// ===========================================================================
// The line kernel.  CTA = NW warps = NW consecutive lines x one segment of
// 32*M positions.
// ===========================================================================
template <int METHOD, int M, int NW, int MODE>
__global__ void __launch_bounds__(32 * NW, (Occ<METHOD>::value)) adi_line_kernel(const KParams P) {
  constexpr int NT = 32 * NW;
  constexpr int NPOS = 32 * M;   // positions per segment
  constexpr int PADM = M + 2;    // padded chunk stride: 16-byte rows, conflict-free 128-bit loads
  constexpr int LSTR = 32 * PADM + 4;  // line stride of the staging tile
  extern __shared__ double smem[];
  double* stS = smem;             // [NW][32][PADM]: S (or U in the prologue)
  double* stX = stS + NW * LSTR;  // [NW][32][PADM]: X
  double* stc = stX + NW * LSTR;  // CFD statics [NW][2 sys][5][32]
  unsigned long long* wbars =
      (unsigned long long*)(stc + (METHOD == M_CFD ? NW * 10 * 32 : 0));  // [NW] per-warp mbarriers

  const int t = threadIdx.x;
  const int w = t >> 5, lane = t & 31;
  const Seg sg = P.segs[blockIdx.y];
  const int line = P.line0 + blockIdx.x * NW + w;   // cross position of this line
  const long long b = blockIdx.z;
  const int n = P.n;
  const int uhi = (METHOD == M_CFD) ? n - 1 : n;  // u active on [1, uhi]
  const int pR = (METHOD == M_CFD) ? n : n + 1;   // position of ū's right Dirichlet value
  const int nact = sg.nchunks * M;
  const bool lineok = line >= P.line_lo && line < P.nlines;

  Ctx<M> c;
  c.t = t; c.line = line; c.chunk = lane; c.n = n;
  c.s = sg.start + lane * M;
  c.live = lineok && (lane < sg.nchunks);
  // dead chunks also run the branch-free interior path: their values only reach
  // the tile halo, which absorbs any bounded garbage
  const bool inner = c.s >= P.plo && c.s + M - 1 <= P.phi;
  c.interior = !c.live || inner;
  c.nbint = c.live && inner && lane >= 2 && lane + 2 < sg.nchunks && c.s - 2 * M >= P.plo &&
            c.s + 3 * M - 1 <= P.phi;

  // ---- load this warp's line segment into the staging tile.  A chunk that starts
  // at a position >= 0 arrives by one TMA bulk copy per lane and array (256 B,
  // rows are padded so it never crosses a row end), completed on the warp's
  // mbarrier; a chunk starting before position 0 (dead positions of a single-tile
  // line) and the strided prologue read of U use 8-byte cp.async with zero fill.
  double* lS = stS + w * LSTR;
  double* lX = stX + w * LSTR;
  unsigned long long* wbar = wbars + w;
  unsigned wpar = 0;  // parity of the warp mbarrier's next phase
  const bool live_chunk = lineok && lane < sg.nchunks;
  const bool bulk = live_chunk && c.s >= 0;
  {
    const double* Sl = P.S_in ? P.S_in + b * P.s_batch + (long long)line * P.s_line : nullptr;
    const double* Xl = P.X_in + b * P.x_batch + (long long)line * P.x_line;
    const double* Ul = P.U_in ? P.U_in + b * P.u_batch + (long long)line * P.u_line : nullptr;
    const unsigned nb = __popc(__ballot_sync(0xffffffffu, bulk));
    if (lane == 0) {
      mbar_init(wbar, 1);
      mbar_expect_tx(wbar, nb * M * 8 * (MODE == KM_PROLOGUE ? 1 : 2));
    }
    __syncwarp();
    if (bulk) {
      bulk_g2s(lX + lane * PADM, Xl + c.s, M * 8, wbar);
      if (MODE != KM_PROLOGUE) bulk_g2s(lS + lane * PADM, Sl + c.s, M * 8, wbar);
    }
    if (!live_chunk) {
      // dead chunk: zero its slots (neighbours read their edges; stale shared
      // memory could hold NaN, which no halo absorbs)
      double2* zs = reinterpret_cast<double2*>(lS + lane * PADM);
      double2* zx = reinterpret_cast<double2*>(lX + lane * PADM);
#pragma unroll
      for (int i = 0; i < PADM / 2; ++i) {
        zs[i] = make_double2(0.0, 0.0);
        zx[i] = make_double2(0.0, 0.0);
      }
    }
    if (live_chunk && (!bulk || MODE == KM_PROLOGUE)) {
#pragma unroll 4
      for (int i = 0; i < M; ++i) {
        const int p = c.s + i;
        const bool xin = p >= 0 && p <= n;
        const bool uin = p >= 1 && p <= uhi;
        if (!bulk) {
          cp_async8(lX + lane * PADM + i, xin ? Xl + p : P.X_in, xin);
          if (MODE != KM_PROLOGUE) cp_async8(lS + lane * PADM + i, uin ? Sl + p : P.X_in, uin);
        }
        if (MODE == KM_PROLOGUE) cp_async8(lS + lane * PADM + i, xin ? Ul + (long long)p * P.u_pt : P.X_in, xin);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  // Dirichlet values of this line
  c.gL = 0.0; c.gR = 0.0;
  if (lineok) {
    if (MODE == KM_PROLOGUE) {
      const double* Ub = P.U_in + b * P.u_batch + (long long)line * P.u_line;
      c.gL = Ub[0];
      c.gR = Ub[(long long)pR * P.u_pt];
    } else {
      if (P.edgeL) c.gL = P.edgeL[line] * P.gb;
      if (P.edgeR) c.gR = P.edgeR[line] * P.gb;
    }
  }
  // source pattern of this segment (shared by the batch): prefetched into L2
  // now, staged into the S tile before the epilogue
  const bool want_phi = (MODE != KM_FINAL) && P.phi_src;
  const double* phl = want_phi ? P.phi_src + (long long)line * P.s_line : nullptr;
  if (want_phi && c.live) {
    const double* a0 = phl + max(c.s, 1);
    asm volatile("prefetch.global.L2 [%0];" ::"l"(a0));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(a0 + 16));
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  mbar_wait(wbar, wpar);
  wpar ^= 1u;
  __syncwarp();

  double* Sm = lS + lane * PADM;  // this chunk's bases in shared memory
  double* Vm = lX + lane * PADM;
  double u[M], x[M];
#pragma unroll
  for (int i = 0; i < M; ++i) {
    const int p = c.s + i;
    x[i] = c.live ? Vm[i] : 0.0;
    if (MODE == KM_PROLOGUE) {
      u[i] = c.live ? Sm[i] : 0.0;
    } else {
      u[i] = (p == 0) ? c.gL : ((METHOD == M_CFD && p == n) ? c.gR : 0.0);
      if (!c.live) u[i] = 0.0;
    }
  }

  // Stage this segment's source pattern into the S tile (coalesced, async).
  // Only legal once S is dead (after the last u-op that uses it as a base).
  auto stage_phi = [&]() {
    if (!want_phi) return;
    __syncwarp();
    fence_async_shared();   // generic-proxy reads of the S tile before the TMA overwrite
    const unsigned nb = __popc(__ballot_sync(0xffffffffu, bulk));
    if (lane == 0) mbar_expect_tx(wbar, nb * M * 8);
    __syncwarp();
    if (bulk) bulk_g2s(lS + lane * PADM, phl + c.s, M * 8, wbar);
    if (live_chunk && !bulk) {
#pragma unroll 4
      for (int i = 0; i < M; ++i) {
        const int p = c.s + i;
        const bool uin = p >= 1 && p <= uhi;
        cp_async8(lS + lane * PADM + i, uin ? phl + p : P.X_in, uin);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  // dst = src + dt/2 F at this chunk's points (F = phi*gf + point source); with
  // a dense source, dst must be the S tile holding the staged phi
  auto add_source = [&](double* dst, const double (&src)[M]) {
    const int ptl = P.pt_line ? P.pt_line[b] : -1;
    const int ptp = P.pt_pos ? P.pt_pos[b] : -1;
    if (want_phi) {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      mbar_wait(wbar, wpar);
      wpar ^= 1u;
      __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const int p = c.s + i;
      double f = want_phi ? dst[i] * P.gf : 0.0;
      if (c.live && line == ptl && p == ptp) f += P.pt_amp * P.gf;
      dst[i] = fma(P.half_dt, f, src[i]);
    }
  };

  if (METHOD == M_CFD) {
    // ---------------- CFD ----------------
    const int np1 = n + 1;
    double* stU = stc + (w * 2 + 0) * 5 * 32;
    double* stXs = stc + (w * 2 + 1) * 5 * 32;
    {
      double q[5];
      cfd_statics<M>(c, P.tabU, np1, q);
#pragma unroll
      for (int k = 0; k < 5; ++k) stU[k * 32 + lane] = c.live ? q[k] : 0.0;
      cfd_statics<M>(c, P.tabX, np1, q);
#pragma unroll
      for (int k = 0; k < 5; ++k) stXs[k * 32 + lane] = c.live ? q[k] : 0.0;
    }
    double d0, d1, xm1, xp1, um1, up1;
    const double SLp = lane > 0 ? lS[(lane - 1) * PADM + M - 1] : 0.0;
    const double SFn = lane < 31 ? lS[(lane + 1) * PADM] : 0.0;
    const double VLp = lane > 0 ? lX[(lane - 1) * PADM + M - 1] : 0.0;
    const double VFn = lane < 31 ? lX[(lane + 1) * PADM] : 0.0;
    __syncwarp();
    warp_edges<M>(lane, x, d0, xm1, xp1, d1);
    warp_edges<M>(lane, u, d0, um1, up1, d1);
    if (MODE == KM_PROLOGUE) {
      double e1, e2;
      double wv[M];
#pragma unroll
      for (int i = 0; i < M; ++i) wv[i] = x[i];
      stage_phi();
      cfd_apply<M, false>(c, P, lane, stXs, u, Vm, x, P.cx, um1, up1, 0.0, 0.0, e1, e2);
      add_source(Sm, u);
      cfd_apply<M, true>(c, P, lane, stU, wv, Sm, u, P.cu, xm1, xp1, 0.0, 0.0, e1, e2);
    } else {
      for (int k = 0; k < P.K; ++k) {
        cfd_apply<M, true>(c, P, lane, stU, x, Sm, u, P.cu, xm1, xp1, SFn, SLp, um1, up1);
        if (MODE == KM_SWEEP && k + 1 == P.K) stage_phi();
        cfd_apply<M, false>(c, P, lane, stXs, u, Vm, x, P.cx, um1, up1, VFn, VLp, xm1, xp1);
      }
      if (MODE == KM_SWEEP) {
        double e1, e2;
        add_source(Sm, u);
        cfd_apply<M, true>(c, P, lane, stU, x, Sm, u, P.cu, xm1, xp1, 0.0, 0.0, e1, e2);
#pragma unroll
        for (int i = 0; i < M; ++i) x[i] = fma(2.0, x[i], -Vm[i]);
      }
    }
  } else {
    // ---------------- MFD ----------------
    const double au = P.cu, bx = P.cx;
    const double cA = au * (1.0 / 24.0), cB = au * (9.0 / 8.0);
    const double cC = bx * (1.0 / 24.0), cD = bx * (9.0 / 8.0);
    double xm2, xm1, xp1, xp2, um2, um1, up1, up2;
    auto u_op = [&](const double (&opd)[M], const double* __restrict__ B) {
      if (c.interior) { MfdSplit<M>::bases(B, u); MfdSplit<M>::u_inner(opd, u, cA, cB); }
      warp_edges<M>(lane, opd, xm2, xm1, xp1, xp2);
      if (c.interior) MfdSplit<M>::u_edges(opd, u, cA, cB, xm2, xm1, xp1);
      else Mfd<M>::template uop<false>(c, opd, B, u, au, xm2, xm1, xp1);
    };
    auto x_op = [&](const double* __restrict__ B) {
      if (c.interior) { MfdSplit<M>::bases(B, x); MfdSplit<M>::x_inner(u, x, cC, cD); }
      warp_edges<M>(lane, u, um2, um1, up1, up2);
      if (c.interior) MfdSplit<M>::x_edges(u, x, cC, cD, um1, up1, up2);
      else Mfd<M>::template xop<false>(c, u, B, x, bx, um1, up1, up2);
    };
    if (MODE == KM_PROLOGUE) {
      double wv[M];
#pragma unroll
      for (int i = 0; i < M; ++i) wv[i] = x[i];
      stage_phi();
      x_op(Vm);            // W* = W - beta D(U)
      add_source(Sm, u);   // S = U + dt/2 F
      u_op(wv, Sm);        // S1 = S - alpha D̄(W)
    } else {
      for (int k = 0; k < P.K; ++k) {
        u_op(x, Sm);
        if (MODE == KM_SWEEP && k + 1 == P.K) stage_phi();
        x_op(Vm);
      }
      if (MODE == KM_SWEEP) {
        add_source(Sm, u);
        u_op(x, Sm);
#pragma unroll
        for (int i = 0; i < M; ++i) x[i] = fma(2.0, x[i], -Vm[i]);
      }
    }
  }

  // ---- stage the outputs in the tile (own chunk), then store the owned range.
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < M; ++i) {
    Sm[i] = u[i];
    Vm[i] = x[i];
    if (c.live) acc += u[i] + x[i];
  }
  // X: this warp's own line, contiguous.  Chunks entirely inside the owned range
  // leave by one TMA bulk store each; partial chunks element by element.
  const bool xown_all = live_chunk && c.s >= sg.out_lo && c.s + M <= sg.out_hi && c.s >= 0 &&
                        c.s + M - 1 <= n;
  double* Xo = P.X_out + b * P.x_batch + (long long)line * P.x_line;
  fence_async_shared();
  __syncwarp();
  if (xown_all) bulk_s2g(Xo + c.s, Vm, M * 8);
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  if (live_chunk && !xown_all) {
#pragma unroll 4
    for (int i = 0; i < M; ++i) {
      const int p = c.s + i;
      if (p >= sg.out_lo && p < sg.out_hi && p >= 0 && p <= n) Xo[p] = Vm[i];
    }
  }
  __syncthreads();
  // S (or U): transposed — a thread stores one position of a pair of lines (16 B)
#pragma unroll 4
  for (int k = 0; k < (NW / 2) * M; ++k) {
    const int e = t + NT * k;
    const int pr = e % (NW / 2), pos = e / (NW / 2);
    const int l0 = 2 * pr;
    const int ln = P.line0 + blockIdx.x * NW + l0;
    const int p = sg.start + pos;
    if (pos >= nact || p < sg.out_lo || p >= sg.out_hi || p < 0 || p > n) continue;
    const bool ok0 = ln >= P.line_lo && ln < P.nlines;
    const bool ok1 = ln + 1 >= P.line_lo && ln + 1 < P.nlines;
    const int si = (pos / M) * PADM + pos % M;
    const double v0 = stS[l0 * LSTR + si], v1 = stS[(l0 + 1) * LSTR + si];
    if (MODE == KM_FINAL) {
      double* Ub = P.U_out + b * P.u_batch + (long long)p * P.u_pt + (long long)ln * P.u_line;
      if (ok0 && ok1) *reinterpret_cast<double2*>(Ub) = make_double2(v0, v1);
      else { if (ok0) Ub[0] = v0; if (ok1) Ub[P.u_line] = v1; }
      if (METHOD == M_MFD && p == n) {
        double* Ut = P.U_out + b * P.u_batch + (long long)(n + 1) * P.u_pt + (long long)ln * P.u_line;
        if (ok0) Ut[0] = P.edgeR ? P.edgeR[ln] * P.gb : 0.0;
        if (ok1) Ut[P.u_line] = P.edgeR ? P.edgeR[ln + 1] * P.gb : 0.0;
      }
    } else if (p >= 1 && p <= uhi) {
      double* So = P.S_out + b * P.s_batch + (long long)p * P.so_pt + (long long)ln * P.so_line;
      if (ok0 && ok1) *reinterpret_cast<double2*>(So) = make_double2(v0, v1);
      else { if (ok0) So[0] = v0; if (ok1) So[P.so_line] = v1; }
    }
  }
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  if (P.flag && !isfinite(acc)) atomicOr(P.flag, 1);
}

}  // namespace adi
