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
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace adi {

enum { M_CFD = 0, M_MFD = 1 };
enum { KM_SWEEP = 0, KM_FINAL = 1, KM_PROLOGUE = 2,
       // stopping-rule attempts: SWEEP / FINAL that also accumulate the last sweep's
       // squared changes (Alg. 3/4 test) and exit at once when the stage is decided
       KM_SWEEP_T = 4, KM_FINAL_T = 5 };

struct Seg {
  int start;    // line position of the first point of chunk 0 (may be < 0)
  int nchunks;  // active chunks per line in this tile
  int out_lo;   // positions [out_lo, out_hi) are written by this tile
  int out_hi;
  int edge;     // 1: generic tile (short lines): per-chunk closures and LU tables
  int end;      // lean tiles: 0 interior, 1 line start (start = 0), 2 line end at
                // chunk 31 element 31 (position n), 3 line end at element 30 (n+1 dead)
};

// Staging tiles arrive by TMA tensor copies of an OVERLAPPING-ROW view of a
// pitched line array: d0 = 34 doubles, d1 = pair offset
// (16 B), d2 = 32-position chunk (256 B), d3 = line, d4 = batch.  One box
// {34, 1, 32, 1, 1} is a line segment in the padded [chunk][34] layout the
// lanes read conflict-free.  Coordinates are taken relative to position
// -TMA_P0 so that segment starts before position 0 stay non-negative.
constexpr int TMA_P0 = 32;
constexpr int BUF_GUARD_FRONT = 64;   // doubles before / after every staged array
constexpr int BUF_GUARD_TAIL = 192;

// Lines and positions are grid POSITIONS (the line index is the position in the
// cross direction; interior lines are 1..).  Element (batch b, line L, position p):
//   S_in : b*s_batch + L*s_line  + p          (lines contiguous)
//   X_in : b*x_batch + L*x_line  + p
//   S_out: b*s_batch + L*so_line + p*so_pt    (written transposed)
//   X_out: b*x_batch + L*x_line  + p
//   U_in / U_out: b*u_batch + L*u_line + p*u_pt  (prologue / final)
constexpr int MAX_TRANKS = 8;   // ranks of a fused transpose (KParams peer table)
struct KParams {
  CUtensorMap tmS;   // S_in (or nothing in the prologue)
  CUtensorMap tmX;   // X_in
  CUtensorMap tmF;   // phi_src (batch extent 1)
  CUtensorMap tmC;   // heterogeneous media (HET kernels): (kappa, rho^-1) fp32 pairs, batch extent 1
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
  double mA, mB, mC, mD;  // MFD interior stencil: cu/24, 9cu/8, cx/24, 9cx/8
  double half_dt;
  int K;
  // NEXT row f4 (FULL kernels): Cerjan taper G(k) = taper[d], d = min(k, n - k) < nb;
  // damp = 1: V' *= G(line) G(p) (row sweep); 2: u, w *= G before the fused a2, W*
  // recomputed (column sweep / final); 0: none
  const double* taper;
  int nb;
  int damp;
  // inner stopping rule (Alg. 3/4): an attempt (KM_*_T) runs K sweeps, adds the
  // owned squared changes of u and x in its last sweep to norms[0], norms[1], and
  // does nothing when *gate is set (the stage is already decided)
  const int* Kdev;   // if set: the sweep count (else K)
  double* norms;
  const int* gate;
  // CFD per-position LU tables, 3 x (n+1): l, 1/d, c   (u-op: P̄, x-op: P)
  const double* tabU; const double* tabX;
  int* flag;        // if set: becomes 1 when a non-finite value is stored
  // profiling aid (adi_set_trace): per tile, warp 0 records
  // {tile, smid, t_start, t_loaded, t_ops_done, t_end, t_after_barrier} (%globaltimer ns)
  unsigned long long* trace;
  long long trace_cap;
  int seg0, nseg_all;   // this launch's first segment, all segments of the axis (trace index)
  // ADI_PREFETCH: the tile this many CTAs later in launch order (about one resident wave
  // per unit) has its staging tiles prefetched into L2 at this tile's start; 0 = off
  int pf_ahead;
  // carry mode (KM_SWEEP, last step of a call): before the fused a2 the
  // kernel also writes this step's final state, U^{m+1} = u_K to U_out (transposed) and
  // W̄^{m+1} = x_K to X_out2, so the next call needs no prologue; 0 = off
  int carry;
  double* X_out2;
  // origin of the TMA-staged arrays (band-local arrays): TMA line
  // coordinate = line - tline0, position coordinate = position - tpos0 (even)
  int tline0, tpos0;
  // positions of U present in a band-local array (column sweep): [pos_lo, pos_hi)
  int pos_lo, pos_hi;
  // asynchronous output (ADI_ASYNC_STORE): S'^T leaves by TMA tensor
  // stores of boxes {4 lines, 4 positions} through tmSo (line coordinate = line -
  // so_line0, position coordinate = p - so_pos0), X' by bulk copies; tma_so = 0: off
  CUtensorMap tmSo;
  int so_line0, so_pos0, tma_so;
  // fused transpose (ADI_DIST_TRANSPOSE with ADI_DIST_FUSED): the transposed
  // S' store of position p goes straight into the array of the rank q that owns p
  // (tcut[q] <= p < tcut[q + 1]), at tso[q] + b tsb[q] + p tpt[q] + line -- peer memory
  // over NVLink (P2P), or another rank's array of a local group.  tnp = 0: own S_out
  int tnp;
  int tcut[MAX_TRANKS + 1];
  double* tso[MAX_TRANKS];
  long long tpt[MAX_TRANKS], tsb[MAX_TRANKS];
};

// per-tile %globaltimer stamps for adi_set_trace (tools/tile_trace.py, trace_sync.py): only in
// libraries built with -DADI_TILE_TRACE=1 (tools/build_variant.sh), out of production kernels
#ifndef ADI_TILE_TRACE
#define ADI_TILE_TRACE 0
#endif
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

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
// Line ends of lean CFD tiles: the lean solve applies T* = L*U*
// (constant pivots); the true operator with the end rows (and identity rows at
// positions outside the system) is A = T* + U V^T of rank <= 3, so
// A^{-1} r = z - M (V^T z), z = T*^{-1} r, M = T*^{-1} U (I + V^T T*^{-1} U)^{-1}.
// Case = system (0: u-op P̄, 1: x-op P) * 3 + end (0 start, 1 end at n, 2 end at
// n+1); V acts on 4 chunk elements (0..3 at the start, 28..31 at the end), M on the
// 32 elements of the end chunk (T*^{-1} U decays like (2-sqrt 3)^d).
// M is applied as its exact entries on the 4 elements next to the end rows (c_wbN)
// and, further in, as a geometric tail: M[i][j] = c_wbF[j] * rho^d, d = distance
// from the line end, rho = -l* (c_rho[d] = rho^d; checked on the host to ~1e-18).
__constant__ double c_wbV[6][3][4];
__constant__ double c_wbN[6][4][3];
__constant__ double c_wbF[6][3];
__constant__ double c_rho[32];

// V^T z of the end correction (zz: z on the 4 elements next to the end rows)
template <int CS>
__device__ __forceinline__ void wb_g(const double (&zz)[4], double& g0, double& g1, double& g2) {
  g0 = 0.0; g1 = 0.0; g2 = 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    g0 = fma(c_wbV[CS][0][q], zz[q], g0);
    g1 = fma(c_wbV[CS][1][q], zz[q], g1);
    g2 = fma(c_wbV[CS][2][q], zz[q], g2);
  }
}
// out += coef * M g on the end chunk (out = B - coef z, z <- z - M g)
template <int CS, bool START, int M>
__device__ __forceinline__ void wb_apply(double (&out)[M], double coef, double g0, double g1, double g2) {
  const double ck = coef * fma(c_wbF[CS][2], g2, fma(c_wbF[CS][1], g1, c_wbF[CS][0] * g0));
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = START ? q : M - 4 + q;
    out[i] = fma(coef, fma(c_wbN[CS][q][2], g2, fma(c_wbN[CS][q][1], g1, c_wbN[CS][q][0] * g0)), out[i]);
  }
#pragma unroll
  for (int q = 4; q < M; ++q) {
    const int i = START ? q : M - 1 - q;
    out[i] = fma(ck, c_rho[q], out[i]);
  }
}
enum { ST_F = 0, ST_KS = 1, ST_KE = 2, ST_JS = 3, ST_JE = 4 };  // CFD chunk statics

template <int M>
struct Ctx {
  int t, line, chunk, s, n;  // s = line position of chunk element 0
  bool live;      // thread owns an existing chunk of an existing line
  bool interior;  // fast path allowed
  bool nbint;     // chunks c-2 .. c+2 all exist and are interior (CFD constant statics)
  double gL, gR;  // Dirichlet values of this line for this half-step
  int endc;       // lean tiles: -1 interior, 0 line start, 1 end at n, 2 end at n+1
  bool me;        // this lane owns the chunk with the line end (lane 0 / lane 31)
};

// ===========================================================================
// MFD operators (App. B).  u at cb positions 1..n (cell centres), x at nodes
// 0..n; ū_0 = gL (slot u[pos 0]), ū_{n+1} = gR (scalar).
// ===========================================================================
template <int M>
struct Mfd {
  // u-op: out = B - a * D4 x  (a = alpha/h); neighbours xm2,xm1 (prev chunk), xp1
  // (NOB: B = 0, the HET kernels' first pass)
  template <bool INTERIOR, bool NOB = false>
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
        out[i] = fma(cA, xr1 - xl2, fma(cB, xl1 - x[i], (NOB ? 0.0 : B[i])));
      } else {
        const int p = c.s + i;
        if (p >= 2 && p <= c.n - 1) {
          out[i] = fma(cA, xr1 - xl2, fma(cB, xl1 - x[i], (NOB ? 0.0 : B[i])));
        } else if (p == 1) {
          if (i >= 1 && i + 4 < M) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 6; ++k) s = fma(c_d4r0[k], x[i - 1 + k], s);
            out[i] = fma(-a, s, (NOB ? 0.0 : B[i]));
          }
        } else if (p == c.n) {
          if (i >= 5) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 6; ++k) s = fma(-c_d4r0[5 - k], x[i - 5 + k], s);
            out[i] = fma(-a, s, (NOB ? 0.0 : B[i]));
          }
        }
      }
    }
  }
  // x-op: out = B - b * G4 ū ; neighbours um1 (prev chunk), up1, up2 (next chunk)
  template <bool INTERIOR, bool NOB = false>
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
        out[i] = fma(cC, ur2 - ul1, fma(cD, u[i] - ur1, (NOB ? 0.0 : B[i])));
      } else {
        const int p = c.s + i;
        const int n = c.n;
        if (p >= 2 && p <= n - 2) {
          out[i] = fma(cC, ur2 - ul1, fma(cD, u[i] - ur1, (NOB ? 0.0 : B[i])));
        } else if (p == 0) {
          if (i + 5 < M) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 6; ++k) s = fma(c_g4r0[k], u[i + k], s);
            out[i] = fma(-b, s, (NOB ? 0.0 : B[i]));
          }
        } else if (p == 1) {
          if (i >= 1 && i + 3 < M) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 5; ++k) s = fma(c_g4r1[k], u[i - 1 + k], s);
            out[i] = fma(-b, s, (NOB ? 0.0 : B[i]));
          }
        } else if (p == n - 1) {
          if (i >= 2 && i + 1 < M) {
            // -reverse(g1) on ū_{n-3..n+1}; ū_{n+1} = gR
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) s = fma(-c_g4r1[4 - k], u[i - 2 + k], s);
            s = fma(-c_g4r1[0], c.gR, s);
            out[i] = fma(-b, s, (NOB ? 0.0 : B[i]));
          }
        } else if (p == n) {
          if (i >= 4) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 5; ++k) s = fma(-c_g4r0[5 - k], u[i - 4 + k], s);
            s = fma(-c_g4r0[0], c.gR, s);
            out[i] = fma(-b, s, (NOB ? 0.0 : B[i]));
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

// MFD closure rows at the line end of a lean tile (same arithmetic as Mfd<M>::uop/xop)
template <int M, bool NOB = false>
__device__ __forceinline__ void mfd_end_u(const Ctx<M>& c, const double (&x)[M], const double* __restrict__ B,
                                          double (&out)[M], double a) {
  static_assert(M == 32, "end fix-ups assume 32-point chunks");
  if (c.endc == 0) {
    out[0] = c.gL;  // ū_0
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) s = fma(c_d4r0[k], x[k], s);
    out[1] = fma(-a, s, (NOB ? 0.0 : B[1]));
  } else {
    const int i = (c.endc == 1) ? 31 : 30;  // position n
    double s = 0.0;
    if (c.endc == 1) {
#pragma unroll
      for (int k = 0; k < 6; ++k) s = fma(-c_d4r0[5 - k], x[26 + k], s);
      out[31] = fma(-a, s, (NOB ? 0.0 : B[31]));
    } else {
#pragma unroll
      for (int k = 0; k < 6; ++k) s = fma(-c_d4r0[5 - k], x[25 + k], s);
      out[30] = fma(-a, s, (NOB ? 0.0 : B[30]));
      out[31] = 0.0;
    }
    (void)i;
  }
}
template <int M, bool NOB = false>
__device__ __forceinline__ void mfd_end_x(const Ctx<M>& c, const double (&u)[M], const double* __restrict__ B,
                                          double (&out)[M], double b) {
  if (c.endc == 0) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) s = fma(c_g4r0[k], u[k], s);
    out[0] = fma(-b, s, (NOB ? 0.0 : B[0]));
    s = 0.0;
#pragma unroll
    for (int k = 0; k < 5; ++k) s = fma(c_g4r1[k], u[k], s);
    out[1] = fma(-b, s, (NOB ? 0.0 : B[1]));
  } else if (c.endc == 1) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) s = fma(-c_g4r1[4 - k], u[28 + k], s);
    s = fma(-c_g4r1[0], c.gR, s);
    out[30] = fma(-b, s, (NOB ? 0.0 : B[30]));
    s = 0.0;
#pragma unroll
    for (int k = 0; k < 5; ++k) s = fma(-c_g4r0[5 - k], u[27 + k], s);
    s = fma(-c_g4r0[0], c.gR, s);
    out[31] = fma(-b, s, (NOB ? 0.0 : B[31]));
  } else {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) s = fma(-c_g4r1[4 - k], u[27 + k], s);
    s = fma(-c_g4r1[0], c.gR, s);
    out[29] = fma(-b, s, (NOB ? 0.0 : B[29]));
    s = 0.0;
#pragma unroll
    for (int k = 0; k < 5; ++k) s = fma(-c_g4r0[5 - k], u[26 + k], s);
    s = fma(-c_g4r0[0], c.gR, s);
    out[30] = fma(-b, s, (NOB ? 0.0 : B[30]));
    out[31] = 0.0;
  }
}

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
__device__ __forceinline__ void fence_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// bulk (non-tensor) copy shared -> global of `bytes` (16-byte aligned, a multiple of 16)
__device__ __forceinline__ void bulk_store(double* g, const double* sm, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(smem_u32(sm)),
               "r"(bytes)
               : "memory");
}
// TMA tensor store of one box of a 3-d map (coordinates d0, d1, d2) from shared memory
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tm, const double* sm, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   (unsigned long long)tm),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(sm))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

__device__ __forceinline__ double shup(double v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }
__device__ __forceinline__ double shdn(double v, int d) { return __shfl_down_sync(0xffffffffu, v, d); }

// prev chunk's a[M-2], a[M-1]; next chunk's a[0], a[1] (0 outside the warp's segment)
// ZEND = false (interior-only tiles): the values beyond the segment ends stay whatever the
// shuffle returns; like zeros they are truncation the halo absorbs (bounded)
template <int M, bool ZEND = true>
__device__ __forceinline__ void warp_edges(int lane, const double (&a)[M], double& pm2, double& pm1,
                                           double& np1, double& np2) {
  pm2 = shup(a[M - 2], 1);
  pm1 = shup(a[M - 1], 1);
  np1 = shdn(a[0], 1);
  np2 = shdn(a[1], 1);
  if (ZEND) {
    pm2 = lane == 0 ? 0.0 : pm2;
    pm1 = lane == 0 ? 0.0 : pm1;
    np1 = lane == 31 ? 0.0 : np1;
    np2 = lane == 31 ? 0.0 : np2;
  }
}

// Heterogeneous media (NEXT row f3; Alg. 3/4 "K.*( )", "R.*( )"):
// the second pass of a HET operator.  The first pass ran the homogeneous code with
// kappa = rho = 1 and no base (out = -ch T^{-1} r, or the stencil times ch); here
// out_i = B_i + m_i out_i with m_i = kappa_i (u-op) or rho^-1_i (x-op) from the staged
// fp32 pairs, at the positions the operator defines ([lo, hi]); the other positions
// keep their Dirichlet slots (lean tiles: restored after an unpredicated pass).
//
// fp32 -> fp64 of a positive normal float (adi_set_media admits only those): exact,
// two integer operations instead of a conversion-unit F2F
__device__ __forceinline__ double f32pos_to_f64(float f) {
  const unsigned b = __float_as_uint(f);
  return __hiloint2double((int)((b >> 3) + 0x38000000u), (int)(b << 29));
}
// 128-bit shared load of 4 floats (two (kappa, rho^-1) pairs); kept whole so the lanes'
// 272-byte-strided rows stay bank-conflict free
__device__ __forceinline__ float4 lds_f4(const void* p) {
  float4 v;
  asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}
template <int M, int METHOD, bool UOP, bool EDGE>
__device__ __forceinline__ void het_apply(const Ctx<M>& c, const double* Crow, const double* __restrict__ B,
                                          double (&out)[M], int lo, int hi) {
  const double2* B2 = reinterpret_cast<const double2*>(B);
#pragma unroll
  for (int i = 0; i < M / 2; ++i) {
    const float4 q = lds_f4(Crow + 2 * i);
    const double2 b = B2[i];
    const double m0 = f32pos_to_f64(UOP ? q.x : q.y), m1 = f32pos_to_f64(UOP ? q.z : q.w);
    if (!EDGE) {
      out[2 * i] = fma(m0, out[2 * i], b.x);
      out[2 * i + 1] = fma(m1, out[2 * i + 1], b.y);
    } else {
      const int p = c.s + 2 * i;
      if (p >= lo && p <= hi && c.live) out[2 * i] = fma(m0, out[2 * i], b.x);
      if (p + 1 >= lo && p + 1 <= hi && c.live) out[2 * i + 1] = fma(m1, out[2 * i + 1], b.y);
    }
  }
  if (!EDGE && c.me) {
    // the slots of the line-end chunk (as the homogeneous end fix-ups leave them)
    static_assert(M == 32, "end fix-ups assume 32-point chunks");
    if (UOP) {
      if (c.endc == 0) out[0] = c.gL;
      else if (c.endc == 1) { if (METHOD == M_CFD) out[31] = c.gR; }
      else { if (METHOD == M_CFD) out[30] = c.gR; out[31] = 0.0; }
    } else if (c.endc == 2) {
      out[31] = 0.0;
    }
  }
}

// CFD LU tables of the line ends staged in shared memory by edge tiles:
// [system 2][l, 1/d, c][ETAB], entries 0..63 = positions 0..63, entries 64..127 =
// positions n-63..n.  Non-interior chunks only touch positions within 64 of an
// end (plo <= 32, checked by the runtime), so the staged entries cover them.
constexpr int ETAB = 128;
struct EdgeTab {
  const double* t;  // [3][ETAB] of one system
  int n;
  __device__ __forceinline__ double get(int arr, int p) const {
    const int i = p < 64 ? p : 64 + p - (n - 63);
    return t[arr * ETAB + i];
  }
};

template <int M>
__device__ __forceinline__ void cfd_statics(const Ctx<M>& c, const EdgeTab& T, int np1,
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
    const double l = (p >= 0 && p < np1) ? T.get(0, p) : 0.0;
    g *= -l;
    G[i] = g;
  }
  st[0] = G[M - 1];
  double k = 0.0, j = 1.0;
#pragma unroll
  for (int i = M - 1; i >= 0; --i) {
    const int p = c.s + i;
    const bool in = (p >= 0 && p < np1);
    const double iv = in ? T.get(1, p) : 0.0;
    const double cc = in ? T.get(2, p) : 0.0;
    k = (G[i] - cc * k) * iv;
    j *= -cc * iv;
    if (i == M - 1) { st[2] = k; st[4] = j; }
  }
  st[1] = k;
  st[3] = j;
}


#ifndef ADI_NSUB
#define ADI_NSUB 4
#endif
constexpr int NSUB = ADI_NSUB;
// CFD fix-up truncation: with 32-point sub-chunks the carry responses
// K_i (i >= 27) and J_i (i <= 3) are below 3e-17 and are not applied
#ifndef ADI_TRIM
#define ADI_TRIM 1
#endif
constexpr bool TRIM = ADI_TRIM && (32 / NSUB == 32);
// CFD interior solve: fold the base into the backward sweep (see cfd_apply)
#ifndef ADI_EARLY_BASE
#define ADI_EARLY_BASE 1
#endif
constexpr bool EARLY_BASE = ADI_EARLY_BASE;
// MFD SWEEP tiles: peel the last of the K sweeps (see line_tile)
#ifndef ADI_MFD_PEEL
#define ADI_MFD_PEEL 1
#endif
constexpr int TRIM_K = 27, TRIM_J = 4;

// ===========================================================================
// CFD: one operator application out = B - coef * T^{-1} r(o) on the warp's
// segment (T = P̄ for the u-op, P for the x-op).  Phase 1: local solve with
// zero carries (NSUB interleaved sub-chunks); exchange (y_e, z_s, z_e) by
// shuffles; phase 2: carries + fix-up.  Also returns this op's output at the
// previous chunk's last and the next chunk's first position (the operand
// neighbours of the next op).  st: statics of this warp's chunks [5][32].
// ===========================================================================
template <int M, bool UOP, bool EDGE, bool NOB = false, bool ZEND = true>
__device__ __forceinline__ void cfd_apply(const Ctx<M>& c, const KParams& P, int lane,
                                          const double* st, const double* etab, const double (&o)[M],
                                          const double* __restrict__ B, double (&out)[M],
                                          double coef, double om1, double op1, double Bn_first,
                                          double Bp_last, double& nom1, double& nop1) {
  constexpr int L = M / NSUB;
  const EdgeTab T{etab + (UOP ? 0 : 3 * ETAB), c.n};
  const int np1 = c.n + 1;
  double yl_e, ws, we;
  double ysub[NSUB];
  // raw backward values the carries need (interior path): sub-chunk starts, the last
  // element, the 4 elements at the chunk start / end (line-end Woodbury window)
  double wsub[NSUB], wlast = 0.0, wzs[4] = {0.0, 0.0, 0.0, 0.0}, wze[4] = {0.0, 0.0, 0.0, 0.0};
  // ---------------- phase 1: local solve with zero carries ----------------
  if (c.interior) {
    if (UOP) Cfd<M>::template rhs_u<true>(c, o, out, om1, op1);
    else Cfd<M>::template rhs_x<true>(c, o, out, om1, op1);
    if (!EDGE && c.me) {
      // closure rows of Q̄ / Q at the line end; zero rows outside the system
      static_assert(M == 32, "end fix-ups assume 32-point chunks");
      if (UOP) {
        if (c.endc == 0) { out[0] = 0.0; out[1] = (-o[0] - 9.0 * o[1] + 9.0 * o[2] + o[3]) * (1.0 / 3.0); }
        else if (c.endc == 1) { out[31] = 0.0; out[30] = (-o[28] - 9.0 * o[29] + 9.0 * o[30] + o[31]) * (1.0 / 3.0); }
        else { out[31] = 0.0; out[30] = 0.0; out[29] = (-o[27] - 9.0 * o[28] + 9.0 * o[29] + o[30]) * (1.0 / 3.0); }
      } else {
        if (c.endc == 0) out[0] = (-17.0 * o[0] + 9.0 * o[1] + 9.0 * o[2] - o[3]) * (1.0 / 3.0);
        else if (c.endc == 1) out[31] = (o[28] - 9.0 * o[29] - 9.0 * o[30] + 17.0 * o[31]) * (1.0 / 3.0);
        else { out[31] = 0.0; out[30] = (o[27] - 9.0 * o[28] - 9.0 * o[29] + 17.0 * o[30]) * (1.0 / 3.0); }
      }
    }
    const double l = c_cl, iv = c_cinvd, FL = c_sF;
#pragma unroll
    for (int i = 1; i < L; ++i)
#pragma unroll
      for (int j = 0; j < NSUB; ++j) out[j * L + i] = fma(-l, out[j * L + i - 1], out[j * L + i]);
#pragma unroll
    for (int j = 0; j < NSUB; ++j) ysub[j] = out[j * L + L - 1];
    if constexpr (EARLY_BASE) {
      // backward sweep with the base folded in as soon as each w_i is final: out_i
      // becomes t_i = B_i - coef iv w_i (the first term of the fix-up, same rounding
      // order), so the base loads and these FMAs fill the latency-bound recurrence
      // instead of stalling the fix-up after the exchange.  The raw w the carries need
      // (sub-chunk starts, the last element, the line-end window) are kept aside.
      const double ci = -coef * iv;
      double wn[NSUB];
#pragma unroll
      for (int j = 0; j < NSUB; ++j) wn[j] = out[j * L + L - 1];
      wlast = wn[NSUB - 1];
      wze[3] = wlast;
#pragma unroll
      for (int i = L - 2; i >= 0; --i)
#pragma unroll
        for (int j = 0; j < NSUB; ++j) {
          const double w = fma(-iv, wn[j], out[j * L + i]);
          out[j * L + i + 1] = NOB ? ci * wn[j] : fma(ci, wn[j], B[j * L + i + 1]);
          wn[j] = w;
          const int e = j * L + i;
          if (e < 4) wzs[e] = w;
          else if (e >= M - 4) wze[e - (M - 4)] = w;
        }
#pragma unroll
      for (int j = 0; j < NSUB; ++j) {
        wsub[j] = wn[j];
        out[j * L] = NOB ? ci * wn[j] : fma(ci, wn[j], B[j * L]);
      }
    } else {
#pragma unroll
      for (int i = L - 2; i >= 0; --i)
#pragma unroll
        for (int j = 0; j < NSUB; ++j) out[j * L + i] = fma(-iv, out[j * L + i + 1], out[j * L + i]);
#pragma unroll
      for (int j = 0; j < NSUB; ++j) wsub[j] = out[j * L];
      wlast = out[M - 1];
#pragma unroll
      for (int q = 0; q < 4; ++q) { wzs[q] = out[q]; wze[q] = out[M - 4 + q]; }
    }
    double Y[NSUB];
    Y[0] = ysub[0];
#pragma unroll
    for (int j = 1; j < NSUB; ++j) Y[j] = fma(FL, Y[j - 1], ysub[j]);
    yl_e = Y[NSUB - 1];
    double zc = 0.0;
#pragma unroll
    for (int j = NSUB - 2; j >= 0; --j) zc = fma(c_sJ[0], zc, fma(c_sK[0], Y[j], iv * wsub[j + 1]));
    ws = fma(c_sJ[0], zc, iv * wsub[0]);
    if constexpr (NSUB > 1) we = fma(c_sK[L - 1], Y[NSUB - 2 < 0 ? 0 : NSUB - 2], iv * wlast);
    else we = iv * wlast;
  } else {
    if (UOP) Cfd<M>::template rhs_u<false>(c, o, out, om1, op1);
    else Cfd<M>::template rhs_x<false>(c, o, out, om1, op1);
    double yp = 0.0;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const int p = c.s + i;
      const double l = (p >= 0 && p < np1) ? T.get(0, p) : 0.0;
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
      const double iv = in ? T.get(1, p) : 0.0;
      const double cc = in ? T.get(2, p) : 0.0;
      z = (out[i] - cc * z) * iv;
      if (i == M - 1) we = z;
    }
    ws = z;
  }
  if (!c.live) { yl_e = 0.0; ws = 0.0; we = 0.0; }
  // ---------------- exchange (shuffles) ----------------
  double ylm1 = shup(yl_e, 1), ylm2 = shup(yl_e, 2), ylp1 = shdn(yl_e, 1);
  double wsp1 = shdn(ws, 1), wsp2 = shdn(ws, 2), wem1 = shup(we, 1);
  if (ZEND) {
    ylm1 = lane == 0 ? 0.0 : ylm1;
    ylm2 = lane <= 1 ? 0.0 : ylm2;
    wem1 = lane == 0 ? 0.0 : wem1;
    ylp1 = lane == 31 ? 0.0 : ylp1;
    wsp1 = lane == 31 ? 0.0 : wsp1;
    wsp2 = lane >= 30 ? 0.0 : wsp2;
  }
  double Fm1, Fme, Ksp1, Jsp1, Ksp2, Kem1, Jem1;
  if (!EDGE && !ZEND) {
    // interior-only tile: constant statics everywhere (the segment ends are halo)
    Fm1 = Fme = c_cF; Ksp1 = Ksp2 = c_cKs; Jsp1 = c_cJs; Kem1 = c_cKe; Jem1 = c_cJe;
  } else if (!EDGE) {
    // interior tile: every chunk of the segment has the interior statics; the
    // segment ends carry nothing (truncated SPIKE)
    Fm1 = lane >= 1 ? c_cF : 0.0; Fme = c_cF;
    Ksp1 = lane <= 30 ? c_cKs : 0.0; Jsp1 = lane <= 30 ? c_cJs : 0.0; Ksp2 = lane <= 29 ? c_cKs : 0.0;
    Kem1 = lane >= 1 ? c_cKe : 0.0; Jem1 = lane >= 1 ? c_cJe : 0.0;
  } else if (c.nbint) {
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
      zcT[j] = fma(c_sJ[0], zcT[j + 1], fma(c_sK[0], ycT[j + 1], iv * wsub[j + 1]));
    z0 = fma(c_sJ[0], zcT[0], fma(c_sK[0], ycT[0], iv * wsub[0]));
    double g0 = 0.0, g1 = 0.0, g2 = 0.0;  // V^T z of the line-end correction
    constexpr int C0 = UOP ? 0 : 3;
    if (!EDGE && c.me) {
      double zz[4];
      if (c.endc == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) zz[q] = fma(c_sJ[q], zcT[0], fma(c_sK[q], ycT[0], iv * wzs[q]));
        wb_g<C0>(zz, g0, g1, g2);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          zz[q] = fma(c_sJ[L - 4 + q], zcT[NSUB - 1], fma(c_sK[L - 4 + q], ycT[NSUB - 1],
                                                           iv * wze[q]));
        if (c.endc == 1) wb_g<C0 + 1>(zz, g0, g1, g2);
        else wb_g<C0 + 2>(zz, g0, g1, g2);
      }
    }
    // the signs ride on the per-chunk scalars (exact), so each constant is a plain
    // constant-bank operand of its DFMA instead of a register loaded by LDC
    const double ci = -coef * iv;
#pragma unroll
    for (int j = 0; j < NSUB; ++j) {
      const double cy = -coef * ycT[j], cz = -coef * zcT[j];
#pragma unroll
      for (int i = 0; i < L; ++i) {
        // truncated responses (TRIM, 32-point sub-chunks): |K_i| < 3e-17 for i >= 27 and
        // |J_i| < 3e-17 for i <= 3 (relative to the carries) -- below round-off, dropped
        double acc = EARLY_BASE ? out[j * L + i] : fma(ci, out[j * L + i], NOB ? 0.0 : B[j * L + i]);
        if (!(TRIM && i >= TRIM_K)) acc = fma(c_sK[i], cy, acc);
        if (!(TRIM && i < TRIM_J)) acc = fma(c_sJ[i], cz, acc);
        out[j * L + i] = acc;
      }
    }
    if (!EDGE && c.me) {
      if (c.endc == 0) wb_apply<C0, true, M>(out, coef, g0, g1, g2);
      else if (c.endc == 1) wb_apply<C0 + 1, false, M>(out, coef, g0, g1, g2);
      else wb_apply<C0 + 2, false, M>(out, coef, g0, g1, g2);
      // positions outside the system hold the Dirichlet slots (u-op) or nothing
      if (UOP) {
        if (c.endc == 0) out[0] = c.gL;
        else if (c.endc == 1) out[31] = c.gR;
        else { out[30] = c.gR; out[31] = 0.0; }
      } else if (c.endc == 2) {
        out[31] = 0.0;
      }
    }
  } else {
    double g = 1.0;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const int p = c.s + i;
      const double l = (p >= 0 && p < np1) ? T.get(0, p) : 0.0;
      g *= -l;
      out[i] = fma(g, ycarry, out[i]);
    }
    double z = zcarry;
#pragma unroll
    for (int i = M - 1; i >= 0; --i) {
      const int p = c.s + i;
      const bool in = (p >= 0 && p < np1);
      const double iv = in ? T.get(1, p) : 0.0;
      const double cc = in ? T.get(2, p) : 0.0;
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
      out[i] = act ? fma(-coef, out[i], NOB ? 0.0 : B[i]) : slot;
    }
  }
  nop1 = fma(-coef, zcarry, Bn_first);
  nom1 = fma(-coef, fma(Jem1, z0, fma(Kem1, ylm2, wem1)), Bp_last);
}

// Occupancy targets (resident CTAs per SM) for the NW-warp CTAs.
template <int METHOD, bool EDGE, int MODE, bool HET = false, bool FULL = false>
struct Occ {
#ifndef ADI_CFD_OCC
#define ADI_CFD_OCC 3
#endif
  // 168 registers: MFD, and the lean CFD kernel (u_K parked in shared memory);
  // the generic CFD kernel keeps 255 registers
  // (the norm pass of the stopping rule keeps the previous iterates: 255 registers)
  // HET (three staging tiles per line): 2, the CFD edge kernel 1 (shared memory)
  // FULL (the f4 variant): 3 lean (168 registers; a same-box A/B 9.88 vs 9.98 ms/step at 2), 2 edge
#ifndef ADI_FULL_OCC
#define ADI_FULL_OCC 3
#endif
  static constexpr int value = FULL ? (EDGE ? 2 : ADI_FULL_OCC)
                               : HET ? ((METHOD == M_CFD && EDGE) ? 1 : 2)
                               : (MODE == KM_SWEEP_T || MODE == KM_FINAL_T) ? 2
                               : (METHOD == M_MFD) ? 3 : (EDGE ? 2 : ADI_CFD_OCC);
};

__host__ __device__ constexpr int PADM_OF(int M) { return M + 2; }
// line stride of the staging tile: 32 padded chunks, rounded to 128 B (TMA destination)
__host__ __device__ constexpr int LSTR_OF(int M) { return (32 * (M + 2) + 15) / 16 * 16; }

// shared memory of one CTA: padded staging of S and X (HET: and the media pairs) for
// NW lines (+ CFD statics; the CFD chunk statics are only needed by edge tiles)
template <int METHOD, int M, int NW, bool EDGE, bool HET = false>
constexpr size_t line_smem_bytes() {
#ifndef ADI_SMEM_PAD
#define ADI_SMEM_PAD 0   // (experiments only: extra bytes per CTA to lower the resident CTAs)
#endif
  return sizeof(double) * (size_t)((HET ? 3 : 2) * NW * LSTR_OF(M) +
                                   (METHOD == M_CFD && EDGE ? NW * 10 * 32 + 6 * ETAB : 0) + NW) +
         128 + ADI_SMEM_PAD;
}

// TMA tensor copy of one line segment (box {34,1,32,1,1}) into the staging tile
__device__ __forceinline__ void tma_load_seg(double* dst, const CUtensorMap* tm, int c1, int c2, int line,
                                             int b, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"((unsigned long long)tm), "r"(0), "r"(c1), "r"(c2), "r"(line), "r"(b), "r"(smem_u32(bar))
      : "memory");
}

// 256-bit global stores (STG.E.256, sm_100): the transposed S' of a CTA's 4 lines is one
// 32-byte sector per position, written by one thread (MFD rows -6%)
#ifndef ADI_S256
#define ADI_S256 1
#endif
// one 32-byte global store (STG.E.256, sm_100); dst 32-byte aligned
__device__ __forceinline__ void st256(double* dst, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

// L2 prefetch of the same box (no shared-memory destination, no completion)
__device__ __forceinline__ void tma_prefetch_seg(const CUtensorMap* tm, int c1, int c2, int line, int b) {
  asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(
                   (unsigned long long)tm),
               "r"(0), "r"(c1), "r"(c2), "r"(line), "r"(b)
               : "memory");
}

// unroll factor of the output store loops (several shared loads in flight per lane)
#ifndef ADI_STORE_UNROLL
#define ADI_STORE_UNROLL 4
#endif
constexpr int STORE_UNROLL = ADI_STORE_UNROLL;
// MFD interior tiles: the epilogue operator accumulates onto u_K in registers (1) or
// reads a staged base u_K + dt/2 F (0)
#ifndef ADI_CARRY_TILE
#define ADI_CARRY_TILE 1
#endif
// carry mode: W̄^{m+1} = x_K leaves through the warp's X tile with the
// coalesced pair store of the epilogue (1) instead of per-lane 16-byte stores from
// registers, 256 B apart across lanes (0)
constexpr bool CARRY_TILE = ADI_CARRY_TILE;
#ifndef ADI_MFD_EPI_REG
#define ADI_MFD_EPI_REG 1
#endif
constexpr bool MFD_EPI_REG = ADI_MFD_EPI_REG;
// the SWEEP tiles' outputs leave asynchronously (bulk copies of X', TMA tensor stores of
// S'^T from a [position][4 lines] re-staging): the tile's slot frees as soon as the copy
// engine has read shared memory instead of after every store instruction has issued
#ifndef ADI_ASYNC_STORE_CODE
#define ADI_ASYNC_STORE_CODE 1
#endif

// ===========================================================================
// One tile = NW lines x one segment.  EDGE = false: all 32 chunks of every line
// are interior and live (the lean path, no generic closures, no per-chunk
// predicates); EDGE = true: line ends, dead chunks, short lines.
// ===========================================================================
// PACK (fragment tiles): a warp carries the FC-chunk middle fragments of
// 32 / FC lines -- lanes [g FC, (g+1) FC) hold line g's chunks; the CTA's 4 warps hold
// 16 consecutive lines.  MFD SWEEP interior segments only; the shuffles at the fragment
// seams read the next fragment's values, which the 28-point halos absorb
constexpr int FRAG_CH = 8;
template <int METHOD, int M, int NW, int MODE_, bool EDGE, bool HET = false, bool FULL = false,
          bool NOEND = false, bool PACK = false>
__device__ __forceinline__ void line_tile(const KParams& P, const Seg& sg, double* smem) {
  // FULL (NEXT row f4, CFD only, readings F1-F2): every position 0..n is
  // unknown and both operators are the full D = P^{-1} Q (the x-op's operator)
  static_assert(!FULL || METHOD == M_CFD, "the full-matrix variant is CFD");
  constexpr bool UOPK = !FULL;   // cfd_apply flavour of the pressure operator
  // stopping-rule attempts are SWEEP / FINAL tiles with the last-sweep test
  constexpr bool TEST = (MODE_ == KM_SWEEP_T || MODE_ == KM_FINAL_T);
  constexpr int MODE = (MODE_ == KM_SWEEP_T) ? KM_SWEEP : (MODE_ == KM_FINAL_T) ? KM_FINAL : MODE_;
  constexpr int NT = 32 * NW;
  constexpr int PADM = PADM_OF(M);
  constexpr int LSTR = LSTR_OF(M);
  constexpr unsigned BOX_BYTES = 32u * PADM * 8u;
  static_assert(M == 32, "the TMA box assumes 32-point chunks");
  static_assert(NW == 4, "the transposed store pairs the 4 lines of a CTA by half-warps");
  double* stS = smem;             // [NW][LSTR]: S (or U in the prologue), later phi, then S'
  double* stX = stS + NW * LSTR;  // [NW][LSTR]: X, then X'
  double* stC = stX + NW * LSTR;  // HET: [NW][LSTR] (kappa, rho^-1) fp32 pairs
  double* stc = stC + (HET ? NW * LSTR : 0);  // CFD statics [NW][2 sys][5][32] (edge tiles)
  double* etab = stc + NW * 10 * 32;  // CFD line-end LU tables [2][3][ETAB] (edge tiles)
  unsigned long long* wbars =
      (unsigned long long*)(stc + (METHOD == M_CFD && EDGE ? NW * 10 * 32 + 6 * ETAB : 0));  // [NW] mbarriers

  const int t = threadIdx.x;
  const int w = t >> 5, lane = t & 31;
  static_assert(!PACK || (METHOD == M_MFD && MODE_ == KM_SWEEP && !EDGE && !HET && !FULL && NOEND),
                "fragment tiles: MFD interior SWEEP");
  constexpr int LPW = PACK ? 32 / FRAG_CH : 1;   // lines per warp
  const int grp = PACK ? lane / FRAG_CH : 0;      // this lane's line within the warp
  const int cl = PACK ? lane % FRAG_CH : lane;    // this lane's chunk within its line
  const int line = PACK ? P.line0 + (blockIdx.x * NW + w) * LPW + grp
                        : P.line0 + blockIdx.x * NW + w;   // cross position of this line
  const int b = blockIdx.z;
  const int n = P.n;
  const int ulo = FULL ? 0 : 1;
  const int uhi = (METHOD == M_CFD && !FULL) ? n - 1 : n;  // u active on [ulo, uhi]
  const int pR = (METHOD == M_CFD) ? n : n + 1;   // position of ū's right Dirichlet value
  const bool lineok = line >= P.line_lo && line < P.nlines;
  const bool tr = ADI_TILE_TRACE && P.trace && t == 0;   // (compiled out of production builds)
  // trace index unique across the launches of one kernel kind (segment offset seg0 of nseg_all)
  const long long tile =
      (long long)blockIdx.x + (long long)gridDim.x * (P.seg0 + blockIdx.y + (long long)P.nseg_all * b);
  unsigned long long tr0 = tr ? gtimer() : 0ull, tr1 = 0ull, tr2 = 0ull;

  Ctx<M> c;
  c.t = t; c.line = line; c.chunk = cl; c.n = n;
  c.s = sg.start + cl * M;
  if (EDGE) {
    c.live = lineok && (lane < sg.nchunks);
    // dead chunks also run the branch-free interior path: their values only reach
    // the tile halo, which absorbs any bounded garbage
    const bool inner = c.s >= P.plo && c.s + M - 1 <= P.phi;
    c.interior = !c.live || inner;
    c.nbint = c.live && inner && lane >= 2 && lane + 2 < sg.nchunks && c.s - 2 * M >= P.plo &&
              c.s + 3 * M - 1 <= P.phi;
  } else {
    c.live = true;      // lines beyond the range compute on finite data; nothing is stored
    c.interior = true;
    c.nbint = true;
  }
  c.endc = EDGE ? -1 : sg.end - 1;
  // NOEND: a launch of interior segments only, the line-end fix-ups compile away
  c.me = !EDGE && !NOEND && ((sg.end == 1 && lane == 0) || (sg.end >= 2 && lane == 31));

  // ---- load: one TMA tensor copy per array and warp (zero fill outside the array)
  double* lS = stS + w * LSTR;
  double* lX = stX + w * LSTR;
  double* lC = stC + w * LSTR;
  unsigned long long* wbar = wbars + w;
  unsigned wpar = 0;  // parity of the warp mbarrier's next phase
  // TMA coordinates are relative to the staged arrays' own origin: a band-local array
  // starts at line tline0 (row sweep) or position tpos0 (column sweep)
  const int sh = sg.start + TMA_P0 - P.tpos0;
  const int tl = line - P.tline0;
  const int c1 = (sh & 31) >> 1, c2 = sh >> 5;
  // PACK: the 4 fragment lines' leader lanes each copy FRAG_CH chunks (8-chunk boxes) into
  // the line's quarter of the tile, on the warp's one barrier (same byte count in total)
  const int go = PACK ? grp * FRAG_CH * PADM : 0;
  if (lane == 0) {
    mbar_init(wbar, 1);
    mbar_expect_tx(wbar, BOX_BYTES * ((MODE == KM_PROLOGUE ? 1u : 2u) + (HET ? 1u : 0u)));
  }
  if (PACK) __syncwarp();   // the barrier exists before the other leaders' copies
  if (PACK ? cl == 0 : lane == 0) {
    tma_load_seg(lX + go, &P.tmX, c1, c2, tl, b, wbar);
    if (HET) tma_load_seg(lC, &P.tmC, c1, c2, tl, 0, wbar);   // one medium for the batch
    if (MODE != KM_PROLOGUE) tma_load_seg(lS + go, &P.tmS, c1, c2, tl, b, wbar);
  }
  if (!EDGE && !PACK && P.pf_ahead > 0 && lane == 0) {
    // L2 prefetch of the staging tiles of the tile pf_ahead CTAs later in launch order:
    // CTAs are dispatched in linear block order, so that tile starts about one resident
    // wave later and its TMA loads then hit L2 -- the HBM reads of the next wave overlap
    // this wave's sweeps (same tensor maps and coordinates as the loads above)
    const long long gx = gridDim.x, gy = gridDim.y;
    const long long lin = blockIdx.x + gx * (blockIdx.y + gy * (long long)blockIdx.z) + P.pf_ahead;
    if (lin < gx * gy * (long long)gridDim.z) {
      const int tx = (int)(lin % gx);
      const long long r = lin / gx;
      const int ty = (int)(r % gy), tz = (int)(r / gy);
      const int tline = P.line0 + tx * NW + w;
      if (tline >= P.line_lo && tline < P.nlines) {
        const int tsh = P.segs[ty].start + TMA_P0 - P.tpos0;
        const int tc1 = (tsh & 31) >> 1, tc2 = tsh >> 5;
        tma_prefetch_seg(&P.tmX, tc1, tc2, tline - P.tline0, tz);
        if (HET) tma_prefetch_seg(&P.tmC, tc1, tc2, tline - P.tline0, 0);
        if (MODE != KM_PROLOGUE) tma_prefetch_seg(&P.tmS, tc1, tc2, tline - P.tline0, tz);
      }
    }
  }
  __syncwarp();  // the barrier is initialised before any lane waits on it
  if (MODE == KM_PROLOGUE) {
    // U is read across its rows (stride u_pt), cooperatively by the CTA: thread e
    // takes line e&3 at segment position e>>2, so one warp instruction reads 8 rows
    // x 4 consecutive lines = 8 full 32-byte sectors (8-byte cp.async, zero fill)
    const double* Ub = P.U_in + (long long)b * P.u_batch;
    const int lg0 = P.line0 + blockIdx.x * NW;
#pragma unroll 4
    for (int k = 0; k < 32 * M * NW / NT; ++k) {
      const int e = t + NT * k;
      const int wl = e % NW, pos = e / NW;
      const int ln = lg0 + wl;
      const int p = sg.start + pos;
      const bool in = ln >= P.line_lo && ln < P.nlines && (!EDGE || pos < sg.nchunks * M) && p >= 0 && p <= n &&
                      p >= P.pos_lo && p < P.pos_hi;
      cp_async8(stS + wl * LSTR + (pos / M) * PADM + pos % M,
                in ? Ub + (long long)p * P.u_pt + (long long)ln * P.u_line : P.X_in, in);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  if (METHOD == M_CFD && EDGE) {
    // stage the line-end LU tables (same for all lines of the tile)
    const int np1 = n + 1;
    for (int k = t; k < 6 * ETAB; k += NT) {
      const int sys = k / (3 * ETAB), arr = (k / ETAB) % 3, i = k % ETAB;
      const int p = i < 64 ? i : n - 63 + (i - 64);
      const double* tab = sys ? P.tabX : P.tabU;
      etab[k] = (p >= 0 && p <= n) ? tab[arr * np1 + p] : 0.0;
    }
    __syncthreads();
  }
  // Dirichlet values of this line (edge tiles only use them)
  c.gL = 0.0; c.gR = 0.0;
  if ((EDGE || sg.end) && lineok) {
    if (MODE == KM_PROLOGUE) {
      const double* Ub = P.U_in + (long long)b * P.u_batch + (long long)line * P.u_line;
      c.gL = (P.pos_lo <= 0) ? Ub[0] : 0.0;                               // (a band without the
      c.gR = (pR < P.pos_hi) ? Ub[(long long)pR * P.u_pt] : 0.0;          //  line end: not used)
    } else {
      if (P.edgeL) c.gL = P.edgeL[line] * P.gb;
      if (P.edgeR) c.gR = P.edgeR[line] * P.gb;
    }
  }
  const bool want_phi = (MODE != KM_FINAL) && P.phi_src;
  const int KK = P.Kdev ? *P.Kdev : P.K;   // sweeps (the stopping rule's choice, if any)
  if (want_phi && (PACK ? cl == 0 : lane == 0)) {
    // the source pattern is staged late (after the last u-op): warm L2 now
    asm volatile(
        "cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(
            (unsigned long long)&P.tmF),
        "r"(0), "r"(c1), "r"(c2), "r"(tl), "r"(0)
        : "memory");
  }
  if (MODE == KM_PROLOGUE) {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();  // the U gather filled every warp's tile
  }
  mbar_wait(wbar, wpar);
  wpar ^= 1u;
  __syncwarp();
  if (tr) tr1 = gtimer();

  double* Sm = lS + lane * PADM;  // this chunk's bases in shared memory
  double* Vm = lX + lane * PADM;
  const double* Cm = lC + lane * PADM;  // HET: this chunk's (kappa, rho^-1) pairs
  double u[M], x[M];
  {
    const double2* V2 = reinterpret_cast<const double2*>(Vm);
    const double2* S2 = reinterpret_cast<const double2*>(Sm);
#pragma unroll
    for (int i = 0; i < M / 2; ++i) {
      const double2 v = V2[i];
      x[2 * i] = v.x;
      x[2 * i + 1] = v.y;
      if (MODE == KM_PROLOGUE) {
        const double2 q = S2[i];
        u[2 * i] = q.x;
        u[2 * i + 1] = q.y;
      }
    }
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const int p = c.s + i;
      if (EDGE && !c.live) { x[i] = 0.0; u[i] = 0.0; continue; }
      if (MODE != KM_PROLOGUE) u[i] = (EDGE && p == 0) ? c.gL : ((EDGE && METHOD == M_CFD && p == n) ? c.gR : 0.0);
    }
  }

  // Stage this segment's source pattern into the S tile (TMA).  Only legal once
  // S is dead (after the last u-op that uses it as a base).
  auto stage_phi = [&]() {
    if (!want_phi) return;
    fence_async_shared();   // generic-proxy reads of the S tile before the async overwrite
    __syncwarp();
    if (lane == 0) mbar_expect_tx(wbar, BOX_BYTES);
    if (PACK) __syncwarp();
    if (PACK ? cl == 0 : lane == 0) tma_load_seg(lS + go, &P.tmF, c1, c2, tl, 0, wbar);
  };
  // dst = src + dt/2 F at this chunk's points (F = phi*gf + point source); with
  // a dense source, dst is the S tile holding the staged phi
  auto add_source = [&](double* dst, const double (&src)[M]) {
    int ipt = -1;
    if (P.pt_line && line == P.pt_line[b] && (!EDGE || c.live)) ipt = P.pt_pos[b] - c.s;
    const double ptf = P.pt_amp * P.gf;
    if (want_phi) {
      mbar_wait(wbar, wpar);
      wpar ^= 1u;
      __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < M; ++i) {
      double f = want_phi ? dst[i] * P.gf : 0.0;
      if (i == ipt) f += ptf;
      dst[i] = fma(P.half_dt, f, src[i]);
    }
  };

  // u = u + dt/2 F in registers, the source pattern staged in `ph` (the S tile)
  auto add_source_reg = [&](const double* ph, double (&uu)[M]) {
    int ipt = -1;
    if (P.pt_line && line == P.pt_line[b]) ipt = P.pt_pos[b] - c.s;
    const double ptf = P.pt_amp * P.gf;
    if (want_phi) {
      mbar_wait(wbar, wpar);
      wpar ^= 1u;
      __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < M; ++i) {
      double f = want_phi ? ph[i] * P.gf : 0.0;
      if (i == ipt) f += ptf;
      uu[i] = fma(P.half_dt, f, uu[i]);
    }
  };

  // dst = dst + dt/2 F in place (dst: S tile holding u_K or U); phi read from global,
  // warmed in L2 at tile start (CFD: keeps one 32-point array live)
  auto add_source_global = [&](double* dst) {
    int ipt = -1;
    if (P.pt_line && line == P.pt_line[b] && (!EDGE || c.live)) ipt = P.pt_pos[b] - c.s;
    const double ptf = P.pt_amp * P.gf;
    const double2* ph = reinterpret_cast<const double2*>(P.phi_src + (long long)line * P.s_line + c.s);
#pragma unroll
    for (int i = 0; i < M / 2; ++i) {
      // (lines past the last row of a CTA group compute but store nothing: no read)
      const double2 f2 = (want_phi && lineok) ? __ldg(ph + i) : make_double2(0.0, 0.0);
      double f0 = f2.x * P.gf, f1 = f2.y * P.gf;
      if (2 * i == ipt) f0 += ptf;
      if (2 * i + 1 == ipt) f1 += ptf;
      dst[2 * i] = fma(P.half_dt, f0, dst[2 * i]);
      dst[2 * i + 1] = fma(P.half_dt, f1, dst[2 * i + 1]);
    }
  };

  // u = u + dt/2 F in registers, phi read from global (warmed in L2 at tile start)
  auto add_source_global_reg = [&](double (&uu)[M]) {
    int ipt = -1;
    if (P.pt_line && line == P.pt_line[b] && (!EDGE || c.live)) ipt = P.pt_pos[b] - c.s;
    const double ptf = P.pt_amp * P.gf;
    const double2* ph = reinterpret_cast<const double2*>(P.phi_src + (long long)line * P.s_line + c.s);
#pragma unroll
    for (int i = 0; i < M / 2; ++i) {
      const double2 f2 = (want_phi && lineok) ? __ldg(ph + i) : make_double2(0.0, 0.0);
      double f0 = f2.x * P.gf, f1 = f2.y * P.gf;
      if (2 * i == ipt) f0 += ptf;
      if (2 * i + 1 == ipt) f1 += ptf;
      uu[2 * i] = fma(P.half_dt, f0, uu[2 * i]);
      uu[2 * i + 1] = fma(P.half_dt, f1, uu[2 * i + 1]);
    }
  };

  // carry mode: this step's final state before the fused a2 -- W̄^{m+1} = x_K from
  // registers (own line, owned positions), U^{m+1} = u_K from the S tiles, transposed,
  // with the FINAL kernel's position range and the MFD right Dirichlet row n+1
  auto carry_store = [&](const double (&xk)[M]) {
    if (!CARRY_TILE && lineok && (!EDGE || c.live)) {
      const int xlo = max(sg.out_lo, 0), xhi = min(sg.out_hi, n + 1);
      double* Xo = P.X_out2 + (long long)b * P.x_batch + (long long)line * P.x_line;
      // 16-byte pairs (segment starts and line pitches are even)
#pragma unroll
      for (int i = 0; i < M; i += 2) {
        const int p = c.s + i;
        if (p >= xlo && p + 1 < xhi) *reinterpret_cast<double2*>(Xo + p) = make_double2(xk[i], xk[i + 1]);
        else {
          if (p >= xlo && p < xhi) Xo[p] = xk[i];
          if (p + 1 >= xlo && p + 1 < xhi) Xo[p + 1] = xk[i + 1];
        }
      }
    }
    __syncthreads();   // every warp's u_K is in its S tile
    const int pr = lane >> 4;
    const int ln = P.line0 + blockIdx.x * NW + 2 * pr;
    const bool ok0 = ln >= P.line_lo && ln < P.nlines;
    const bool ok1 = ln + 1 >= P.line_lo && ln + 1 < P.nlines;
    const int plo_ = max(sg.out_lo, 0), phi_ = min(sg.out_hi, n + 1);
    const double* r0 = stS + (2 * pr) * LSTR;
    const double* r1 = r0 + LSTR;
    const int lg0 = P.line0 + blockIdx.x * NW;
    if (ADI_S256 && P.u_line == 1 && lg0 >= P.line_lo && lg0 + NW <= P.nlines) {
      // the CTA's 4 lines of a position as one 32-byte store (as the S' store)
      for (int pos = t; pos < 32 * M; pos += NT) {
        const int p = sg.start + pos;
        if (p < plo_ || p >= phi_) continue;
        const int si = (pos >> 5) * PADM + (pos & 31);
        st256(P.U_out + (long long)b * P.u_batch + (long long)p * P.u_pt + lg0, stS[si], stS[LSTR + si],
              stS[2 * LSTR + si], stS[3 * LSTR + si]);
        if (METHOD == M_MFD && p == n) {
          double e[4];
          for (int l = 0; l < 4; ++l) e[l] = P.edgeR ? P.edgeR[lg0 + l] * P.gb : 0.0;
          st256(P.U_out + (long long)b * P.u_batch + (long long)(n + 1) * P.u_pt + lg0, e[0], e[1], e[2], e[3]);
        }
      }
      __syncthreads();   // the S tiles are read before the epilogue reuses them
      return;
    }
    for (int pos = 16 * w + (lane & 15); pos < 32 * M; pos += 16 * NW) {
      const int p = sg.start + pos;
      if (p < plo_ || p >= phi_) continue;
      const int si = (pos >> 5) * PADM + (pos & 31);
      const double v0 = r0[si], v1 = r1[si];
      double* Ub = P.U_out + (long long)b * P.u_batch + (long long)p * P.u_pt + (long long)ln * P.u_line;
      if (ok0 && ok1) *reinterpret_cast<double2*>(Ub) = make_double2(v0, v1);
      else { if (ok0) Ub[0] = v0; if (ok1) Ub[P.u_line] = v1; }
      if (METHOD == M_MFD && p == n) {
        double* Ut = P.U_out + (long long)b * P.u_batch + (long long)(n + 1) * P.u_pt + (long long)ln * P.u_line;
        if (ok0) Ut[0] = P.edgeR ? P.edgeR[ln] * P.gb : 0.0;
        if (ok1) Ut[P.u_line] = P.edgeR ? P.edgeR[ln + 1] * P.gb : 0.0;
      }
    }
    __syncthreads();   // the S tiles are read before the epilogue reuses them
  };

  // carry mode with CARRY_TILE, after the epilogue operator (x = x_K no longer an
  // operand): x_K replaces V^m in the X tile as x becomes 2 x_K - V^m, then the warp
  // stores W̄^{m+1} from the tile in coalesced pairs (the X-store pattern below)
  auto carry_x_tile = [&]() {
#pragma unroll
    for (int i = 0; i < M; ++i) { const double t = Vm[i]; Vm[i] = x[i]; x[i] = fma(2.0, x[i], -t); }
    __syncwarp();
    if (lineok) {
      const int xlo = max(sg.out_lo, 0), xhi = min(sg.out_hi, n + 1);
      double* Xo = P.X_out2 + (long long)b * P.x_batch + (long long)line * P.x_line;
#pragma unroll STORE_UNROLL
      for (int p = (xlo & ~1) + 2 * lane; p < xhi; p += 64) {
        const int q = p - sg.start;
        const double2 v = *reinterpret_cast<const double2*>(lX + (q >> 5) * PADM + (q & 31));
        if (p >= xlo && p + 1 < xhi) *reinterpret_cast<double2*>(Xo + p) = v;
        else {
          if (p >= xlo) Xo[p] = v.x;
          if (p + 1 >= xlo && p + 1 < xhi) Xo[p + 1] = v.y;
        }
      }
    }
    __syncwarp();   // the tile is read before the epilogue stages X' over it
  };

  // stopping rule (Alg. 3/4): this warp's share of
  // ||u_s - u_{s-1}||^2 and ||x_s - x_{s-1}||^2 over its owned positions
  auto norm_add = [&](const double (&un)[M], const double (&uo)[M], const double (&xn)[M],
                      const double (&xo)[M]) {
    double su = 0.0, sx = 0.0;
    if (lineok && (!EDGE || c.live)) {
      const int ua = max(sg.out_lo, 1), ub = min(sg.out_hi, uhi + 1);
      const int xa = max(sg.out_lo, 0), xb = min(sg.out_hi, n + 1);
#pragma unroll
      for (int i = 0; i < M; ++i) {
        const int p = c.s + i;
        const double du = (p >= ua && p < ub) ? un[i] - uo[i] : 0.0;
        const double dx = (p >= xa && p < xb) ? xn[i] - xo[i] : 0.0;
        su = fma(du, du, su);
        sx = fma(dx, dx, sx);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      su += __shfl_xor_sync(0xffffffffu, su, o);
      sx += __shfl_xor_sync(0xffffffffu, sx, o);
    }
    if (lane == 0) {
      atomicAdd(P.norms, su);
      atomicAdd(P.norms + 1, sx);
    }
  };

  if (METHOD == M_CFD) {
    // ---------------- CFD ----------------
    const int np1 = n + 1;
    double* stU = stc + (w * 2 + 0) * 5 * 32;
    double* stXs = stc + (w * 2 + 1) * 5 * 32;
    if (EDGE) {
      double q[5];
      cfd_statics<M>(c, EdgeTab{etab, n}, np1, q);
#pragma unroll
      for (int k = 0; k < 5; ++k) stU[k * 32 + lane] = c.live ? q[k] : 0.0;
      cfd_statics<M>(c, EdgeTab{etab + 3 * ETAB, n}, np1, q);
#pragma unroll
      for (int k = 0; k < 5; ++k) stXs[k * 32 + lane] = c.live ? q[k] : 0.0;
    }
    double d0, d1, xm1, xp1, um1, up1;
    // HET: coefficients at the previous chunk's last / the next chunk's first position
    // (the neighbour outputs of each operator)
    double kP = 0.0, kN = 0.0, rP = 0.0, rN = 0.0;
    if constexpr (HET) {
      const float* Cf = reinterpret_cast<const float*>(lC);
      if (lane > 0) { kP = (double)Cf[2 * ((lane - 1) * PADM + M - 1)]; rP = (double)Cf[2 * ((lane - 1) * PADM + M - 1) + 1]; }
      if (lane < 31) { kN = (double)Cf[2 * ((lane + 1) * PADM)]; rN = (double)Cf[2 * ((lane + 1) * PADM) + 1]; }
    }
    const double SLp = lane > 0 ? lS[(lane - 1) * PADM + M - 1] : 0.0;
    const double SFn = lane < 31 ? lS[(lane + 1) * PADM] : 0.0;
    const double VLp = lane > 0 ? lX[(lane - 1) * PADM + M - 1] : 0.0;
    const double VFn = lane < 31 ? lX[(lane + 1) * PADM] : 0.0;
    __syncwarp();
    warp_edges<M, !NOEND>(lane, x, d0, xm1, xp1, d1);
    warp_edges<M, !NOEND>(lane, u, d0, um1, up1, d1);
    if (MODE == KM_PROLOGUE) {
      // at most two 32-point arrays live: U stays in the S tile, W is re-read from
      // the X tile, W* is staged for output before the u-op
      double e1, e2;
      cfd_apply<M, false, EDGE, HET, !NOEND>(c, P, lane, stXs, etab, u, Vm, x, P.cx, um1, up1, 0.0, 0.0, e1, e2);
      if constexpr (HET) het_apply<M, METHOD, false, EDGE>(c, Cm, Vm, x, 0, n);
      add_source_global(Sm);   // S = U + dt/2 F
      double wv[M];
      {
        double2* V2 = reinterpret_cast<double2*>(Vm);
#pragma unroll
        for (int i = 0; i < M / 2; ++i) {
          const double2 v = V2[i];
          wv[2 * i] = v.x;
          wv[2 * i + 1] = v.y;
          V2[i] = make_double2(x[2 * i], x[2 * i + 1]);
        }
      }
      cfd_apply<M, UOPK, EDGE, HET, !NOEND>(c, P, lane, FULL ? stXs : stU, etab, wv, Sm, u, P.cu, xm1, xp1, 0.0, 0.0, e1, e2);
      if constexpr (HET) het_apply<M, METHOD, true, EDGE>(c, Cm, Sm, u, 1, uhi);
    } else {
      double uo[TEST ? M : 1], xo[TEST ? M : 1];
      for (int k = 0; k < KK; ++k) {
        if constexpr (TEST) {
          if (k + 1 == KK) {
#pragma unroll
            for (int i = 0; i < M; ++i) { uo[i] = u[i]; xo[i] = x[i]; }
          }
        }
        if constexpr (HET) {
          cfd_apply<M, true, EDGE, true, !NOEND>(c, P, lane, stU, etab, x, Sm, u, P.cu, xm1, xp1, 0.0, 0.0, um1, up1);
          het_apply<M, METHOD, true, EDGE>(c, Cm, Sm, u, 1, uhi);
          um1 = fma(kP, um1, SLp);
          up1 = fma(kN, up1, SFn);
        } else {
          cfd_apply<M, UOPK, EDGE, false, !NOEND>(c, P, lane, FULL ? stXs : stU, etab, x, Sm, u, P.cu, xm1, xp1, SFn, SLp, um1, up1);
        }
        if (k + 1 == KK) {
          // park u_K in the (now dead) S tile: u is then dead across every x-op,
          // which keeps one 32-point array live instead of two (no spills at 3 CTAs/SM)
          double2* S2 = reinterpret_cast<double2*>(Sm);
#pragma unroll
          for (int i = 0; i < M / 2; ++i) S2[i] = make_double2(u[2 * i], u[2 * i + 1]);
        }
        if constexpr (HET) {
          cfd_apply<M, false, EDGE, true, !NOEND>(c, P, lane, stXs, etab, u, Vm, x, P.cx, um1, up1, 0.0, 0.0, xm1, xp1);
          het_apply<M, METHOD, false, EDGE>(c, Cm, Vm, x, 0, n);
          xm1 = fma(rP, xm1, VLp);
          xp1 = fma(rN, xp1, VFn);
        } else {
          cfd_apply<M, false, EDGE, false, !NOEND>(c, P, lane, stXs, etab, u, Vm, x, P.cx, um1, up1, VFn, VLp, xm1, xp1);
        }
        if constexpr (TEST) {
          if (k + 1 == KK) norm_add(u, uo, x, xo);
        }
      }
      // f4: the Cerjan taper at this chunk's points, G(line) G(p) (F2)
      auto taper_at = [&](int k, int nn) -> double {
        const int d = min(k, nn - k);
        return (d >= 0 && d < P.nb) ? P.taper[d] : 1.0;
      };
      if (FULL && P.damp == 2) {
        // column sweep of the full variant: U^{m+1} = G u_K, W^{m+1} = G w_K (parked u_K in
        // the S tile); FINAL stores them, SWEEP continues with the fused a2 of step m+1:
        // W* = Gw - beta D(Gu) (explicitly: the 2w - W* identity does not survive the taper)
        // and S1 = Gu + dt/2 F - alpha D(Gw)
        const double gl = taper_at(line, P.nlines - 1);
#pragma unroll
        for (int i = 0; i < M; ++i) {
          const double g = gl * taper_at(c.s + i, n);
          x[i] *= g;
          Sm[i] *= g;
        }
        if (MODE == KM_SWEEP) {
          double e1, e2, d0, d1;
#pragma unroll
          for (int i = 0; i < M; ++i) { u[i] = Sm[i]; Vm[i] = x[i]; }   // operand Gu, base Gw
          __syncwarp();
          warp_edges<M, !NOEND>(lane, u, d0, um1, up1, d1);
          cfd_apply<M, false, EDGE, false, !NOEND>(c, P, lane, stXs, etab, u, Vm, x, P.cx, um1, up1, 0.0, 0.0, e1, e2);
#pragma unroll
          for (int i = 0; i < M; ++i) { u[i] = Vm[i]; Vm[i] = x[i]; }   // operand Gw; Vm = W*
          __syncwarp();
          warp_edges<M, !NOEND>(lane, u, d0, xm1, xp1, d1);
          add_source_global(Sm);   // S = Gu + dt/2 F
          cfd_apply<M, false, EDGE, false, !NOEND>(c, P, lane, stXs, etab, u, Sm, x, P.cu, xm1, xp1, 0.0, 0.0, e1, e2);
#pragma unroll
          for (int i = 0; i < M; ++i) { u[i] = x[i]; x[i] = Vm[i]; }    // u = S1, x = W*
        }
      } else if (MODE == KM_SWEEP) {
        double e1, e2;
        bool carried = false;
        if constexpr (!HET && !FULL) {
          if (P.carry) { carry_store(x); carried = true; }   // U^{m+1} (u_K parked in the S tile), W̄^{m+1}
        }
        add_source_global(Sm);   // S = u_K + dt/2 F
        cfd_apply<M, UOPK, EDGE, HET, !NOEND>(c, P, lane, FULL ? stXs : stU, etab, x, Sm, u, P.cu, xm1, xp1, 0.0, 0.0, e1, e2);
        if constexpr (HET) het_apply<M, METHOD, true, EDGE>(c, Cm, Sm, u, 1, uhi);
        if (CARRY_TILE && carried) carry_x_tile();
        else {
#pragma unroll
          for (int i = 0; i < M; ++i) x[i] = fma(2.0, x[i], -Vm[i]);
        }
        if (FULL && P.damp == 1) {   // row sweep of the full variant: V^{m+1} = G (2x - X)
          const double gl = taper_at(line, P.nlines - 1);
#pragma unroll
          for (int i = 0; i < M; ++i) x[i] *= gl * taper_at(c.s + i, n);
        }
      }
    }
  } else {
    // ---------------- MFD ----------------
    const double au = P.cu, bx = P.cx;
    const double cA = P.mA, cB = P.mB, cC = P.mC, cD = P.mD;
    double xm2, xm1, xp1, xp2, um2, um1, up1, up2;
    auto u_op = [&](const double (&opd)[M], const double* __restrict__ B) {
      if constexpr (HET) {
        // unit coefficient, no base; then out = B + ch kappa_i out (het_apply)
        if (c.interior) {
#pragma unroll
          for (int i = 0; i < M; ++i) u[i] = 0.0;
          MfdSplit<M>::u_inner(opd, u, cA, cB);
        }
        warp_edges<M, !NOEND>(lane, opd, xm2, xm1, xp1, xp2);
        if (c.interior) MfdSplit<M>::u_edges(opd, u, cA, cB, xm2, xm1, xp1);
        else Mfd<M>::template uop<false, true>(c, opd, B, u, au, xm2, xm1, xp1);
        if (!EDGE && c.me) mfd_end_u<M, true>(c, opd, B, u, au);
        het_apply<M, METHOD, true, EDGE>(c, Cm, B, u, 1, uhi);
      } else {
        if (c.interior) { MfdSplit<M>::bases(B, u); MfdSplit<M>::u_inner(opd, u, cA, cB); }
        warp_edges<M, !NOEND>(lane, opd, xm2, xm1, xp1, xp2);
        if (c.interior) MfdSplit<M>::u_edges(opd, u, cA, cB, xm2, xm1, xp1);
        else Mfd<M>::template uop<false>(c, opd, B, u, au, xm2, xm1, xp1);
        if (!EDGE && c.me) mfd_end_u<M>(c, opd, B, u, au);
      }
    };
    auto x_op = [&](const double* __restrict__ B) {
      if constexpr (HET) {
        if (c.interior) {
#pragma unroll
          for (int i = 0; i < M; ++i) x[i] = 0.0;
          MfdSplit<M>::x_inner(u, x, cC, cD);
        }
        warp_edges<M, !NOEND>(lane, u, um2, um1, up1, up2);
        if (c.interior) MfdSplit<M>::x_edges(u, x, cC, cD, um1, up1, up2);
        else Mfd<M>::template xop<false, true>(c, u, B, x, bx, um1, up1, up2);
        if (!EDGE && c.me) mfd_end_x<M, true>(c, u, B, x, bx);
        het_apply<M, METHOD, false, EDGE>(c, Cm, B, x, 0, n);
      } else {
        if (c.interior) { MfdSplit<M>::bases(B, x); MfdSplit<M>::x_inner(u, x, cC, cD); }
        warp_edges<M, !NOEND>(lane, u, um2, um1, up1, up2);
        if (c.interior) MfdSplit<M>::x_edges(u, x, cC, cD, um1, up1, up2);
        else Mfd<M>::template xop<false>(c, u, B, x, bx, um1, up1, up2);
        if (!EDGE && c.me) mfd_end_x<M>(c, u, B, x, bx);
      }
    };
    if (MODE == KM_PROLOGUE) {
      // at most two 32-point arrays live (as for CFD): U stays in the S tile, W is
      // re-read from the X tile, W* is staged for output before the u-op
      x_op(Vm);                 // W* = W - beta D(U)
      add_source_global(Sm);    // S = U + dt/2 F
      double wv[M];
      {
        double2* V2 = reinterpret_cast<double2*>(Vm);
#pragma unroll
        for (int i = 0; i < M / 2; ++i) {
          const double2 v = V2[i];
          wv[2 * i] = v.x;
          wv[2 * i + 1] = v.y;
          V2[i] = make_double2(x[2 * i], x[2 * i + 1]);
        }
      }
      u_op(wv, Sm);             // S1 = S - alpha D̄(W)
    } else {
      double uo[TEST ? M : 1], xo[TEST ? M : 1];
      if constexpr (TEST || MODE != KM_SWEEP || !ADI_MFD_PEEL) {
        for (int k = 0; k < KK; ++k) {
          if constexpr (TEST) {
            if (k + 1 == KK) {
#pragma unroll
              for (int i = 0; i < M; ++i) { uo[i] = u[i]; xo[i] = x[i]; }
            }
          }
          u_op(x, Sm);
          if (MODE == KM_SWEEP && k + 1 == KK && !(!HET && P.carry)) stage_phi();
          x_op(Vm);
          if constexpr (TEST) {
            if (k + 1 == KK) norm_add(u, uo, x, xo);
          }
        }
      } else {
        // the last sweep peeled: the source staging between its two operators is then
        // straight-line code, and the loop carries u and x in fixed registers (with the
        // conditional TMA inside the loop, ptxas re-homed u around it: 64 moves a sweep)
        for (int k = 0; k + 1 < KK; ++k) {
          u_op(x, Sm);
          x_op(Vm);
        }
        if (KK > 0) {
          u_op(x, Sm);
          if (!(!HET && P.carry)) stage_phi();
          x_op(Vm);
        }
      }
      if (MODE == KM_SWEEP) {
        bool carried = false;
        if constexpr (!HET) {
          if (P.carry) {
            // carry mode: u_K to the S tile (no source pattern staged there), the final
            // state out, then S' = (u_K - alpha D̄(x_K)) + dt/2 F with the source from global
            double2* S2 = reinterpret_cast<double2*>(Sm);
#pragma unroll
            for (int i = 0; i < M / 2; ++i) S2[i] = make_double2(u[2 * i], u[2 * i + 1]);
            carry_store(x);
            u_op(x, Sm);
            add_source_global_reg(u);
            if (CARRY_TILE) carry_x_tile();
            carried = true;
          }
        }
        if (carried) {
        } else if constexpr (NOEND && !HET && MFD_EPI_REG) {
          // interior tiles: the epilogue operator accumulates onto u_K in registers and
          // the source comes last (S' = u_K - alpha D̄(x_K) + dt/2 F), so the TMA of the
          // source pattern, issued after the last u-op, has two operators of slack
          MfdSplit<M>::u_inner(x, u, cA, cB);
          warp_edges<M, false>(lane, x, xm2, xm1, xp1, xp2);
          MfdSplit<M>::u_edges(x, u, cA, cB, xm2, xm1, xp1);
          add_source_reg(Sm, u);
        } else {
          add_source(Sm, u);
          u_op(x, Sm);
        }
        if (!(CARRY_TILE && carried)) {
#pragma unroll
          for (int i = 0; i < M; ++i) x[i] = fma(2.0, x[i], -Vm[i]);
        }
      }
    }
  }
  if (tr) tr2 = gtimer();

  // ---- stage the outputs in the tile (own chunk); the CFD FINAL u_K is already parked
  double acc = 0.0;
  {
    double2* S2 = reinterpret_cast<double2*>(Sm);
    double2* V2 = reinterpret_cast<double2*>(Vm);
#pragma unroll
    for (int i = 0; i < M / 2; ++i) {
      if (!(METHOD == M_CFD && MODE == KM_FINAL)) S2[i] = make_double2(u[2 * i], u[2 * i + 1]);
      if (MODE != KM_PROLOGUE) V2[i] = make_double2(x[2 * i], x[2 * i + 1]);
    }
    if (P.flag && lineok && (!EDGE || c.live)) {
#pragma unroll
      for (int i = 0; i < M; ++i) acc += Sm[i] + Vm[i];
    }
  }
  __syncthreads();
  const unsigned long long tr3 = tr ? gtimer() : 0ull;   // (trace: after the CTA barrier)

  // (X' along the line stays in 16-byte pairs: 32-byte runs per lane measured slower)
  // asynchronous outputs (ADI_ASYNC_STORE): lean SWEEP tiles whose 4 lines are all processed
  constexpr bool ASYNC_ST = ADI_ASYNC_STORE_CODE && MODE == KM_SWEEP && !EDGE && !HET && !FULL && !TEST && !PACK;
  bool async_s = false;
  if constexpr (ASYNC_ST) {
    const int lg0 = P.line0 + blockIdx.x * NW;
    async_s = P.tma_so && !P.carry && lg0 >= P.line_lo && lg0 + NW <= P.nlines;
  }
  if constexpr (PACK) {
    // fragment tiles.  X': the 8 lanes of a line store its owned positions in pairs
    {
      const int xlo = max(sg.out_lo, 0), xhi = min(sg.out_hi, n + 1);
      const double* tX = lX + grp * FRAG_CH * PADM;   // this line's chunks
      double* Xo = P.X_out + (long long)b * P.x_batch + (long long)line * P.x_line;
      if (lineok) {
        for (int p = (xlo & ~1) + 2 * cl; p < xhi; p += 2 * FRAG_CH) {
          const int q = p - sg.start;
          const double2 v = *reinterpret_cast<const double2*>(tX + (q >> 5) * PADM + (q & 31));
          if (p >= xlo && p + 1 < xhi) *reinterpret_cast<double2*>(Xo + p) = v;
          else {
            if (p >= xlo) Xo[p] = v.x;
            if (p + 1 >= xlo && p + 1 < xhi) Xo[p + 1] = v.y;
          }
        }
      }
    }
    // S'^T: the CTA's 16 consecutive lines make 128 contiguous bytes per position; thread
    // t stores lines 4 (t & 3) .. +3 -- one fragment slot of each warp row, i.e. warp
    // (t & 3)'s 4 fragments -- of position plo_ + (t >> 2) + 32 k, as one 32-byte store
    {
      const int plo_ = max(sg.out_lo, ulo), phi_ = min(sg.out_hi, uhi + 1);
      const int wq = t & 3;                                   // the warp whose 4 fragment lines
      const double* r0 = stS + wq * LSTR;                     // line 4 wq + g: fragment g of warp wq
      const int ln = P.line0 + blockIdx.x * NW * LPW + 4 * wq;
      bool ok[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) ok[g] = ln + g >= P.line_lo && ln + g < P.nlines;
      const bool all = ok[0] && ok[1] && ok[2] && ok[3];
      int own = 0;   // fused transpose: the owner of position p (positions grow along the loop)
      for (int p = plo_ + (t >> 2); p < phi_; p += NT / 4) {
        const int q = p - sg.start;
        const int si = (q >> 5) * PADM + (q & 31);
        double v[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) v[g] = r0[g * FRAG_CH * PADM + si];
        double* So;
        long long sl = P.so_line;
        if (P.tnp > 0) {
          while (own + 1 < P.tnp && p >= P.tcut[own + 1]) ++own;
          So = P.tso[own] + (long long)b * P.tsb[own] + (long long)p * P.tpt[own] + (long long)ln;
          sl = 1;
        } else {
          So = P.S_out + (long long)b * P.s_batch + (long long)p * P.so_pt + (long long)ln * P.so_line;
        }
        if (all && sl == 1) {
          asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(So), "d"(v[0]), "d"(v[1]), "d"(v[2]),
                       "d"(v[3])
                       : "memory");
        } else {
#pragma unroll
          for (int g = 0; g < 4; ++g)
            if (ok[g]) So[g * sl] = v[g];
        }
      }
      if (P.tnp > 0) __threadfence_system();   // (peer stores, as in the tiles' fused store)
    }
  } else if (ASYNC_ST && P.tma_so && !P.carry && lineok) {
    // X': this lane's chunk ∩ the owned range as one bulk copy (16-byte aligned body;
    // an odd first / last position by a plain store)
    const int xlo = max(sg.out_lo, 0), xhi = min(sg.out_hi, n + 1);
    double* Xo = P.X_out + (long long)b * P.x_batch + (long long)line * P.x_line;
    int a = max(xlo, c.s), e = min(xhi, c.s + M);
    if (a < e) {
      if (a & 1) { Xo[a] = Vm[a - c.s]; ++a; }
      if ((e & 1) && e > a) { Xo[e - 1] = Vm[e - 1 - c.s]; --e; }
      if (e > a) {
        fence_async_shared();
        bulk_store(Xo + a, Vm + (a - c.s), (unsigned)(e - a) * 8u);
      }
    }
    bulk_commit();
  } else if (lineok) {
    const int xlo = max(sg.out_lo, 0), xhi = min(sg.out_hi, n + 1);
    double* Xo = P.X_out + (long long)b * P.x_batch + (long long)line * P.x_line;
#pragma unroll STORE_UNROLL
    for (int p = (xlo & ~1) + 2 * lane; p < xhi; p += 64) {
      const int q = p - sg.start;
      const double2 v = *reinterpret_cast<const double2*>(lX + (q >> 5) * PADM + (q & 31));
      if (p >= xlo && p + 1 < xhi) *reinterpret_cast<double2*>(Xo + p) = v;
      else {
        if (p >= xlo) Xo[p] = v.x;
        if (p + 1 >= xlo && p + 1 < xhi) Xo[p + 1] = v.y;
      }
    }
  }
  if (ASYNC_ST && async_s) {
    // S'^T: re-stage the 4 lines as [position][4] in the X tiles (once the bulk copies of X'
    // have read them), then TMA tensor stores of {4 lines, 4 positions} boxes over the
    // owned range; its ragged ends (< 4 positions) by plain stores
    bulk_wait_read();
    __syncthreads();
    double* stg = stX;   // [1024][4] doubles (the 4 X tiles hold 4 * LSTR >= 4096)
    for (int q = t; q < 32 * M; q += NT) {
      const int si = (q >> 5) * PADM + (q & 31);
      double2* d = reinterpret_cast<double2*>(stg + 4 * q);
      d[0] = make_double2(stS[si], stS[LSTR + si]);
      d[1] = make_double2(stS[2 * LSTR + si], stS[3 * LSTR + si]);
    }
    fence_async_shared();
    __syncthreads();
    const int lg0 = P.line0 + blockIdx.x * NW;
    const int plo_ = max(sg.out_lo, ulo), phi_ = min(sg.out_hi, uhi + 1);
    const int q0 = (plo_ - sg.start + 3) & ~3, q1 = (phi_ - sg.start) & ~3;
    for (int k = q0 + 4 * t; k < q1; k += 4 * NT)
      tma_store_3d(&P.tmSo, stg + 4 * k, lg0 - P.so_line0, sg.start + k - P.so_pos0, b);
    bulk_commit();
    // ragged ends: positions [plo_, start + q0) and [start + max(q0, q1), phi_)
    {
      const int nh = max(min(sg.start + q0, phi_) - plo_, 0);
      const int tail0 = max(sg.start + max(q0, q1), plo_);
      const int nt = max(phi_ - tail0, 0);
      if (t < 4 * (nh + nt)) {
        const int k = t >> 2, l = t & 3;
        const int p = (k < nh) ? plo_ + k : tail0 + (k - nh);
        double* So = P.S_out + (long long)b * P.s_batch + (long long)p * P.so_pt + (long long)(lg0 + l) * P.so_line;
        *So = stg[4 * (p - sg.start) + l];
      }
    }
    bulk_wait_read();
  } else if (!PACK)
  // S (or U): transposed.  Half-warp h of warp w stores line pair h at positions
  // 16 w + (lane & 15) + 64 k: the two half-warps fill one 32-byte sector each
  {
    const int pr = lane >> 4;
    const int ln = P.line0 + blockIdx.x * NW + 2 * pr;
    const bool ok0 = ln >= P.line_lo && ln < P.nlines;
    const bool ok1 = ln + 1 >= P.line_lo && ln + 1 < P.nlines;
    int plo_, phi_;   // output positions of this tile for S / U
    if (MODE == KM_FINAL) { plo_ = max(sg.out_lo, 0); phi_ = min(sg.out_hi, n + 1); }
    else { plo_ = max(sg.out_lo, ulo); phi_ = min(sg.out_hi, uhi + 1); }
    const double* r0 = stS + (2 * pr) * LSTR;
    const double* r1 = r0 + LSTR;
    const bool all4 = P.line0 + (int)blockIdx.x * NW >= P.line_lo && P.line0 + (int)blockIdx.x * NW + NW <= P.nlines;
    if (ADI_S256 && MODE != KM_FINAL && P.tnp > 0 && all4) {
      // fused transpose, one 32-byte sector (the CTA's 4 lines) per thread and position
      const long long lg0 = P.line0 + (long long)blockIdx.x * NW;
      int q = 0;
#pragma unroll STORE_UNROLL
      for (int pos = t; pos < 32 * M; pos += NT) {
        const int p = sg.start + pos;
        if (p < plo_ || p >= phi_) continue;
        while (q + 1 < P.tnp && p >= P.tcut[q + 1]) ++q;
        const int si = (pos >> 5) * PADM + (pos & 31);
        double* So = P.tso[q] + (long long)b * P.tsb[q] + (long long)p * P.tpt[q] + lg0;
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(So), "d"(stS[si]), "d"(stS[LSTR + si]),
                     "d"(stS[2 * LSTR + si]), "d"(stS[3 * LSTR + si])
                     : "memory");
      }
      __threadfence_system();
    } else if (MODE != KM_FINAL && P.tnp > 0) {
      // fused transpose: position p lands in the array of its owner q
      // (the cuts are few and sorted; positions grow along a lane's loop), as P2P stores
      int q = 0;
#pragma unroll STORE_UNROLL
      for (int pos = 16 * w + (lane & 15); pos < 32 * M; pos += 16 * NW) {
        const int p = sg.start + pos;
        if (p < plo_ || p >= phi_) continue;
        while (q + 1 < P.tnp && p >= P.tcut[q + 1]) ++q;
        const int si = (pos >> 5) * PADM + (pos & 31);
        double* So = P.tso[q] + (long long)b * P.tsb[q] + (long long)p * P.tpt[q] + (long long)ln;
        if (ok0 && ok1) *reinterpret_cast<double2*>(So) = make_double2(r0[si], r1[si]);
        else { if (ok0) So[0] = r0[si]; if (ok1) So[1] = r1[si]; }
      }
      // this thread's peer stores are performed at system scope before the kernel can
      // complete (and the barrier after it release them to the owners)
      __threadfence_system();
    } else if (ADI_S256 && MODE == KM_FINAL && all4 && P.u_line == 1) {
      // U (FINAL): the CTA's 4 lines of a position as one 32-byte store; MFD row n+1 = gR
      const long long lg0 = P.line0 + (long long)blockIdx.x * NW;
#pragma unroll STORE_UNROLL
      for (int pos = t; pos < 32 * M; pos += NT) {
        const int p = sg.start + pos;
        if (p < plo_ || p >= phi_) continue;
        const int si = (pos >> 5) * PADM + (pos & 31);
        st256(P.U_out + (long long)b * P.u_batch + (long long)p * P.u_pt + lg0, stS[si], stS[LSTR + si],
              stS[2 * LSTR + si], stS[3 * LSTR + si]);
        if (METHOD == M_MFD && p == n) {
          double e[4];
          for (int l = 0; l < 4; ++l) e[l] = P.edgeR ? P.edgeR[lg0 + l] * P.gb : 0.0;
          st256(P.U_out + (long long)b * P.u_batch + (long long)(n + 1) * P.u_pt + lg0, e[0], e[1], e[2], e[3]);
        }
      }
    } else if (ADI_S256 && MODE != KM_FINAL && all4) {
      // a whole 32-byte sector per thread: the CTA's 4 lines at one position
      const long long lg0 = P.line0 + (long long)blockIdx.x * NW;
#pragma unroll STORE_UNROLL
      for (int pos = t; pos < 32 * M; pos += NT) {
        const int p = sg.start + pos;
        if (p < plo_ || p >= phi_) continue;
        const int si = (pos >> 5) * PADM + (pos & 31);
        double* So = P.S_out + (long long)b * P.s_batch + (long long)p * P.so_pt + lg0;
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(So), "d"(stS[si]), "d"(stS[LSTR + si]),
                     "d"(stS[2 * LSTR + si]), "d"(stS[3 * LSTR + si])
                     : "memory");
      }
    } else {
#pragma unroll STORE_UNROLL
      for (int pos = 16 * w + (lane & 15); pos < 32 * M; pos += 16 * NW) {
        const int p = sg.start + pos;
        if (p < plo_ || p >= phi_) continue;
        const int si = (pos >> 5) * PADM + (pos & 31);
        const double v0 = r0[si], v1 = r1[si];
        if (MODE == KM_FINAL) {
          double* Ub = P.U_out + (long long)b * P.u_batch + (long long)p * P.u_pt + (long long)ln * P.u_line;
          if (ok0 && ok1) *reinterpret_cast<double2*>(Ub) = make_double2(v0, v1);
          else { if (ok0) Ub[0] = v0; if (ok1) Ub[P.u_line] = v1; }
          if (METHOD == M_MFD && p == n) {
            double* Ut = P.U_out + (long long)b * P.u_batch + (long long)(n + 1) * P.u_pt + (long long)ln * P.u_line;
            if (ok0) Ut[0] = P.edgeR ? P.edgeR[ln] * P.gb : 0.0;
            if (ok1) Ut[P.u_line] = P.edgeR ? P.edgeR[ln + 1] * P.gb : 0.0;
          }
        } else {
          double* So = P.S_out + (long long)b * P.s_batch + (long long)p * P.so_pt + (long long)ln * P.so_line;
          if (ok0 && ok1) *reinterpret_cast<double2*>(So) = make_double2(v0, v1);
          else { if (ok0) So[0] = v0; if (ok1) So[P.so_line] = v1; }
        }
      }
    }
  }
  if (ASYNC_ST && P.tma_so && !P.carry && !async_s) bulk_wait_read();   // the X' copies read the tile
  if (P.flag && !isfinite(acc)) atomicOr(P.flag, 1);
  if (tr && tile < P.trace_cap) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    unsigned long long* r = P.trace + tile * 8;
    r[0] = tile; r[1] = smid; r[2] = tr0; r[3] = tr1; r[4] = tr2; r[5] = gtimer(); r[6] = tr3;
  }
}

// ===========================================================================
// The line kernel: grid (line groups, segments, batch), NW warps per CTA.  The
// interior segments (EDGE = false) and the segments holding line ends (EDGE =
// true) are separate launches, so the main kernel carries only the lean path.
//   MODE = KM_SWEEP   : S_in, X_in -> K sweeps -> S'^T (S_out), X' (X_out)
//   MODE = KM_FINAL   : as SWEEP without the fused explicit half; writes U_out
//   MODE = KM_PROLOGUE: U_in, X_in -> a2 (explicit half only)
// ===========================================================================
template <int METHOD, int M, int NW, int MODE, bool EDGE, bool HET = false, bool FULL = false,
          bool NOEND = false, bool PACK = false>
__global__ void __launch_bounds__(32 * NW, (Occ<METHOD, EDGE, MODE, HET, FULL>::value))
    adi_line_kernel(const __grid_constant__ KParams P) {
  extern __shared__ __align__(128) double smem_raw[];
  // TMA destinations need 128-byte alignment
  // (pointer arithmetic on the shared array keeps the shared address space visible)
  double* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u) / 8u;
  if (P.gate && *P.gate) return;   // stopping rule: the stage was decided by an earlier attempt
  const Seg sg = P.segs[blockIdx.y];
  line_tile<METHOD, M, NW, MODE, EDGE, HET, FULL, NOEND, PACK>(P, sg, smem);
}

// The stopping rule after the attempt with k sweeps (Alg. 3/4 "until test <= eps or
// k >= k_max"): test = ||u_k - u_{k-1}||_F + ||x_k - x_{k-1}||_F from the attempt's
// sums; a passing test (or k = kmax) closes the gate and records k.  One thread.
__global__ void decide_sweeps_kernel(const double* norms, double eps, int k, int kmax, int* gate, int* kout) {
  if (*gate) return;
  if (sqrt(norms[0]) + sqrt(norms[1]) <= eps || k >= kmax) {
    *gate = 1;
    *kout = k;
  }
}

}  // namespace adi
