/*
 * adi.h — C-ABI of the B200-native Peaceman–Rachford ADI library
 * (arXiv:2006.07583, Otero, Rojas, Moya & Castillo).  Library: libadi.so.
 *
 * The library advances the 2-D velocity–pressure acoustic system (eq. 1,
 * PAPER.md:57-63) with the Peaceman–Rachford splitting of Crank–Nicolson
 * (eqs. 4-6).  Each ADI stage resolves its implicit
 * pressure/velocity coupling with K fixed-point sweeps along grid lines
 * (eqs. 8-9; Alg. 3/4), K fixed
 * (default K = k_max = 8).  Two spatial
 * variants:
 *   ADI_CFD — nodal compact FD: every derivative is a stencil Q, Q̄ plus a
 *             tridiagonal solve with P, P̄ (Appendix A).
 *   ADI_MFD — staggered mimetic FD: D4 / G4 stencils with wide boundary
 *             closures (Appendix B).
 * Everything is IEEE fp64.  All compute runs in the library's sm_100a CUDA
 * kernels; there is no CPU fallback — without a usable CUDA device every
 * call returns ADI_ECUDA.
 *
 * ---------------------------------------------------------------------------
 * Grid and state layout (row index = y, column index = x; row-major, C order).
 * nx, ny are node counts per direction (N = n-1 cells, spacing h).
 *
 *   CFD (nodal):
 *     U  : ny x nx            pressure incl. the Dirichlet boundary
 *     V  : (ny-2) x nx        V̄ = rows 1..ny-2 of the horizontal velocity
 *     W  : ny x (nx-2)        W̄ = columns 1..nx-2 of the vertical velocity
 *   MFD (staggered):
 *     U  : (ny+1) x (nx+1)    pressure on X_cb x Y_cb incl. the boundary
 *     V  : (ny-1) x nx        V̄: x nodes x y cell centres
 *     W  : ny x (nx-1)        W̄: y nodes x x cell centres
 *   CFD_FULL (f4, see ADI_CFD_FULL): U, V, W all ny x nx (every node).
 * The velocity lines on the boundary that the paper never updates are not
 * part of the state.  The pressure-interior block ("I") is
 * (ny-2) x (nx-2) for CFD and (ny-1) x (nx-1) for MFD.
 *
 * Time: step m advances t^m = t0 + m*dt to t^{m+1}.  Source and boundary
 * time functions are given as tables sampled at HALF steps,
 * g[j] = g(t0 + j*dt/2), because the method needs t^m, t^m + dt/2 and
 * t^{m+1}.  A table must cover every step run:
 * adi_step returns ADI_EINVAL if 2*(m_end) >= ng.  A NULL table means the
 * constant 1.
 *
 * Ownership: the library owns all device memory (cudaMalloc).  Host pointers
 * are read or written only during the call; tables and patterns are copied.
 * Device pointers passed to *_device calls must stay valid for the call and
 * are accessed on the handle's stream.
 *
 * Errors: every call returns a status (ADI_OK = 0, negative = error,
 * positive = warning, state still usable); adi_last_error() gives the
 * message.  Arguments are validated before any allocation.
 * Threading: one host thread per handle at a time.
 * ---------------------------------------------------------------------------
 */
#ifndef ADI_H_
#define ADI_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct adi_ctx* adi_handle;

/* ADI_CFD_FULL: the full-matrix CFD variant.
 * "By simply replacing reduced operators P̄ and Q̄, and reduced matrices Ū, V̄, W̄,
 * by their full matrix versions [...] the boundary wave fields can be also
 * obtained.  These values can be further damped by the absorbing technique [of
 * Cerjan et al.]."  Every node is unknown: U, V, W and a dense source pattern are
 * all ny x nx; every derivative is D = P^{-1} Q (full, n+1 rows); there is no
 * Dirichlet data (adi_set_boundary with edges returns ADI_EINVAL).  After each
 * step U, V, W are multiplied by the Cerjan taper G(x) G(y) set by
 * ADI_ABSORB_WIDTH / ADI_ABSORB_RATE (readings F1-F2).  The literal
 * CFD closure's growth remains: the layer delays it.  No band
 * decomposition, stopping rule or media for this variant (ADI_EINVAL). */
enum adi_method { ADI_CFD = 0, ADI_MFD = 1, ADI_CFD_FULL = 2 };

enum adi_status {
  ADI_OK = 0,
  ADI_EINVAL = -1,      /* bad argument / shape / too small grid (N < 8) / short table */
  ADI_ENOMEM = -2,      /* device or host allocation failed */
  ADI_ECUDA = -3,       /* CUDA runtime error (incl. no device) */
  ADI_EZEROPIVOT = -4,  /* zero pivot in the LU of P or P̄ */
  ADI_ENONFINITE = -5,  /* a field became NaN/Inf (checked when ADI_CHECK_FINITE=1) */
  ADI_ESTATE = -6,      /* call out of order (e.g. step before set_fields) */
  ADI_ENCCL = -7,       /* NCCL unavailable or failed (adi_create_dist, adi_nccl_unique_id) */
  ADI_WUNSTABLE = 1     /* warning: c*dt/h above the inner-iteration limit
                           (2/sqrt(6) ~ 0.8165 MFD, 2/sqrt(3) ~ 1.155 CFD; SURVEY SA-3) */
};

enum adi_param {
  ADI_K_SWEEPS = 0,     /* fixed-point sweeps per stage, integer >= 1; default 8 */
  ADI_RHO = 1,          /* density rho > 0 (kappa = rho c^2); default 1 */
  ADI_CHECK_FINITE = 2, /* 1: adi_step synchronizes and checks for NaN/Inf; default 0 */
  ADI_TILE_CHUNKS = 3,  /* cap on chunks (32 points each) per line in one tile; 0 = auto.
                           Testing aid: forces the segmented (halo) tiling on small grids. */
  ADI_TIMING = 4,       /* 1: bracket every kernel launch with CUDA events on the handle's
                           stream (read with adi_get_kernel_times); default 0 */
  ADI_EPS = 5,          /* inner stopping rule of Alg. 3/4: 0 (default)
                           = fixed ADI_K_SWEEPS sweeps [G10]; eps > 0 = each stage stops at the
                           first sweep k in [ADI_K_MIN, ADI_K_SWEEPS] with
                           ||U_k - U_{k-1}||_F + ||V_k - V_{k-1}||_F <= eps (Frobenius norms over
                           the stage's whole interior pressure / velocity matrices), else at
                           ADI_K_SWEEPS.  Costs one extra pass of the stage's sweeps; decided on
                           the device (no host round trip).  Whole grid only (no band). */
  ADI_K_MIN = 6,        /* first sweep tested by the stopping rule; integer >= 2, default 6 */
  ADI_ABSORB_WIDTH = 7, /* ADI_CFD_FULL only: Cerjan layer width nb in points, integer in
                           [0, min(nx, ny)/2]; default 0 (no layer).  After each step the fields
                           are multiplied by G(x)G(y), G = exp(-(a (nb - d))^2) at distance d < nb
                           (points) from the nearest edge, else 1 */
  ADI_ABSORB_RATE = 8,  /* ADI_CFD_FULL only: the rate a > 0 of the taper; default 0.015 */
  ADI_PREFETCH = 9,     /* performance knob, no effect on results: each line tile of the lean
                           kernels prefetches into L2 (TMA prefetch) the staging tiles of the tile
                           v resident-CTA waves ahead in the same launch, so that the HBM reads of
                           the next wave overlap this wave's sweeps; integer in [0, 8], 0 = off;
                           default 0 (measured slower: DESIGN.md §5.6) */
  ADI_CARRY = 10,       /* 1 (default): the last column kernel of a call also computes the next
                           step's explicit half (a2), so that the next adi_step skips its
                           prologue kernel, unless a set_* call came in between.  Same results
                           up to rounding order (the one-call computation).  Used for plain
                           handles only (no band / dist, no ADI_EPS, no media, not
                           ADI_CFD_FULL); 0 = always run the prologue */
  ADI_GRAPH = 11,       /* 1: adi_step(n) captures its kernels (prologue, n x {rows, columns},
                           Dirichlet columns) into one CUDA graph and launches it: one host
                           launch per call instead of 2n+2 (short lines are launch-bound, the
                           paper's own observation).  Same kernels, same
                           results bit for bit.  Plain and banded handles without ADI_EPS;
                           ignored for adi_create_dist ranks.  Default 0 */
  ADI_THREAD_LINES = 12, /* the short-line kernels (one warp -- ADI_WARP_LINES --
                           or one thread per grid line through a half-step, with the no-pivot
                           LU of App. A) instead of the 1024-position line tiles: -1 (default)
                           for lines of at most 382 cells (warp kernels; 64 with
                           ADI_WARP_LINES = 0), 1 wherever they fit (warp: <= 382 cells, thread:
                           <= ~260), 0 never.  Plain handles of ADI_CFD / ADI_MFD with fixed K
                           (no band, media, stopping rule, ADI_CFD_FULL, ADI_TILE_CHUNKS);
                           results agree with the tile kernels to rounding (parity-tested
                           against the oracle) */
  ADI_ASYNC_STORE = 13, /* 1: the lean ADI-rows / ADI-columns tiles store their outputs
                           asynchronously -- X' by bulk copies, S'^T by TMA tensor stores of
                           {4 lines, 4 positions} boxes from a re-staged tile;
                           0 (default): thread stores.  Bitwise the same results; measured no
                           faster (the store phase is bound by the memory system) */
  ADI_DIST_FUSED = 14,  /* transpose-mode handles (ADI_DIST_TRANSPOSE, <= 8 ranks): 1 (default
                           where available) fuses the all-to-all of S into the kernels -- the
                           row and column kernels store their transposed S' straight into the
                           owning rank's array (peer memory over NVLink through CUDA IPC
                           mappings, or the other ranks' arrays of an adi_create_dist_local
                           group), and the exchange becomes a barrier (a one-element NCCL
                           all-reduce, or stream waits in a local group); 0: the NCCL / loopback
                           all-to-all.  Collective: set it to the same value on every rank,
                           between calls.  EINVAL where no peer mapping exists (halo mode, more
                           than 8 ranks, IPC unavailable: adi_create_dist_ex then leaves the
                           handle unfused on every rank).  Results are bitwise the same;
                           DESIGN.md §7.2 */
  ADI_WARP_LINES = 15,  /* 1 (default): where ADI_THREAD_LINES selects the short-line kernels and
                           every line has at most 384 stored positions (382 cells), one WARP runs
                           a line (2..12 positions per lane; the CFD solves as warp scans of the
                           paper's LU recurrences); 0: one thread per line.
                           Results agree to rounding */
  ADI_STEP_INDEX = 16,  /* the handle's time level m (steps taken; t = m dt): the index into the
                           source and boundary time tables of the next step.  Integer >= 0,
                           between calls; drops the carried explicit half (ADI_CARRY).  With
                           adi_set_fields, restarts a run from an initial state */
  ADI_FRAG_TILES = 17,  /* performance knob: 1 (default) runs the MFD sweeps of whole lines whose
                           1024-position tiles leave a short middle gap (4096 positions: 4 tiles
                           and a 168-position gap instead of 5 tiles) as the lean tiles plus one
                           8-chunk fragment per line, 4 lines' fragments per warp (DESIGN.md
                           §5.12); 0: the standard tile plan.  Results agree to rounding */
};

/* Kernel kinds launched by adi_step (index of adi_get_kernel_times arrays). */
enum adi_kernel_kind {
  ADI_KK_PROLOGUE = 0,  /* explicit y-half of the first step of a call (a2) */
  ADI_KK_ROW = 1,       /* ADI-rows: K sweeps along x + fused C / V^{m+1} (a3, a4) */
  ADI_KK_COL = 2,       /* ADI-columns: K sweeps along y + fused a2 of the next step (a6) */
  ADI_KK_FINAL = 3,     /* ADI-columns of the last step of a call, writes U, W̄ (a6) */
  ADI_KK_EDGE = 4,      /* Dirichlet columns of U */
  ADI_NKINDS = 5
};

typedef struct adi_stats {
  long long steps;      /* steps taken since creation */
  double t;             /* t0 + steps*dt */
  int nonfinite;        /* 1 if a non-finite value was produced (needs ADI_CHECK_FINITE) */
  int k_sweeps;
  long long kernel_launches; /* kernels launched by adi_step since creation */
  /* the last-sweep residuals (ADI_EPS > 0): for the last row [0] and column [1] stage,
   * the Alg. 3/4 test ||U_k - U_{k-1}||_F + ||V_k - V_{k-1}||_F at the chosen sweep
   * last_k; -1 and K when the rule is off (reading them
   * synchronizes the handle's stream) */
  double last_test[2];
  int last_k[2];
  /* device memory the handle allocated (field arrays with their guards, tables excluded,
   * halo buffers included): a band of adi_create_dist holds its band + halo rows only */
  long long device_bytes;
  /* host-side launches (kernel launches, or one per graph launch with ADI_GRAPH = 1) */
  long long host_launches;
} adi_stats;

/* Create a solver for one grid (batch = 1).  nx, ny >= 9 nodes (N >= 8);
 * h > 0 grid spacing, dt > 0, c > 0 wave speed; method ADI_CFD or ADI_MFD.
 * Returns ADI_WUNSTABLE (handle valid) when c*dt/h exceeds the K-sweep
 * iteration limit.  Fields start at zero, t0 = 0.  The handle lives on the calling
 * thread's current CUDA device; every later call on it runs on that device and
 * restores the caller's current device (handles on several devices may coexist in
 * one process; one host thread per handle at a time). */
int adi_create(int nx, int ny, double h, double dt, double c, int method, adi_handle* out);

/* As adi_create with `batch` independent grids ("shots") of the same shape
 * advanced together by every adi_step (config 5).  Field arrays of the
 * *_fields calls then hold `batch` consecutive grids. */
int adi_create_batch(int nx, int ny, double h, double dt, double c, int method, int batch,
                     adi_handle* out);

int adi_set_param(adi_handle h, int key, double value);

/* Stream on which all work of this handle is enqueued (cudaStream_t as void*;
 * NULL = the legacy default stream). */
int adi_set_stream(adi_handle h, void* cuda_stream);

/* Set the state at the current time from HOST arrays (shapes above, times batch).
 * With a band set (adi_set_band) only the rows the band uses are read: y positions
 * [y0 - halo, y1 + halo) of U and W̄ and the V̄ rows of those positions; the other
 * rows of the arrays are not accessed.  ESTATE while a call is in progress. */
int adi_set_fields(adi_handle h, const double* U, const double* V, const double* W);
/* Same from DEVICE arrays (contiguous, same shapes). */
int adi_set_fields_device(adi_handle h, const double* dU, const double* dV, const double* dW);

/* Source term F(x,y,t) of eq. 1 on the pressure-interior points, entering
 * eqs. 5-6 as dt/2 (F^m + F^{m+1}):
 *   F = phi(x,y) * g(t)                      if phi != NULL (phi: I-block, host), plus
 *   F = g(t) / h^2 at U-array point (ix, iy) if ix >= 1 (point source; batch 1;
 *   ADI_CFD_FULL: any node, ix >= 0).
 * g: table at half steps, ng entries (NULL: g = 1). */
int adi_set_source(adi_handle h, const double* phi, int ix, int iy, const double* g, int ng);

/* Point sources for a batch: shot b has F = g(t)/h^2 at U-array point (ix[b], iy[b]). */
int adi_set_point_sources(adi_handle h, const int* ix, const int* iy, const double* g, int ng);

/* Dirichlet data u0 = b(x,y) g(t) on the pressure boundary.
 * edges: host array of the four U edges concatenated: row 0 (y = 0, length
 * ncolsU), last row (y = 1, ncolsU), column 0 (x = 0, nrowsU), last column
 * (x = 1, nrowsU); NULL = homogeneous.  g: table at half steps (NULL: 1). */
int adi_set_boundary(adi_handle h, const double* edges, const double* g, int ng);

/* Heterogeneous media: the material matrices K = kappa(x,y)
 * and R = rho^-1(x,y) of Alg. 1-4 ("K.*( )", "R.*( )" after the
 * derivative).  Host arrays, fp32, C order, one
 * medium for every grid of a batch:
 *   kappa  : the U layout (nrowsU x ncolsU); interior points used
 *   rinv_v : rho^-1 on the V̄ layout (V's shape above)
 *   rinv_w : rho^-1 on the W̄ layout (W's shape above)
 * (CFD is nodal: rinv_v = R[1:-1, :], rinv_w = R[:, 1:-1] of one nodal field.)
 * The step then uses alpha_i = dt/2 kappa_i and beta_j = dt/2 rho^-1_j per point
 * in place of the scalars c, ADI_RHO; all arithmetic stays fp64 (the fp32 inputs
 * are promoted exactly).  Copied synchronously; all three NULL returns to the
 * scalar medium.  Errors: ADI_EINVAL if only some are NULL or a used value is not
 * finite, normal and > 0; ADI_ESTATE during a call; ADI_WUNSTABLE (fields set) if
 * sqrt(max kappa * max rho^-1) dt/h exceeds the inner-iteration limit.  Not
 * combinable with ADI_EPS > 0 (adi_step returns ADI_EINVAL). */
int adi_set_media(adi_handle h, const float* kappa, const float* rinv_v, const float* rinv_w);

/* Enqueue n >= 0 time steps on the handle's stream (asynchronous unless
 * ADI_CHECK_FINITE is set). */
int adi_step(adi_handle h, int n);

/* The phases of adi_step(n), for drivers that must act between the half-steps
 * (the multi-GPU band decomposition exchanges halos after the row sweep):
 *   adi_step_begin(h, n)            explicit y-half of the first step (a2)
 *   n x { adi_step_rows(h);         ADI-rows of the step (a3, a4)
 *         adi_step_cols(h); }       ADI-columns (a6; + a2 of the next step, or the
 *                                   final U, W̄ of the call)
 *   adi_step_end(h)                 Dirichlet columns of U; non-finite check
 * adi_step(h, n) is exactly this sequence.  All are asynchronous on the stream. */
int adi_step_begin(adi_handle h, int n);
int adi_step_rows(adi_handle h);
int adi_step_cols(adi_handle h);
int adi_step_end(adi_handle h);

/* Band decomposition of one grid over several handles / GPUs.
 * adi_set_band restricts this handle to the y positions [y0, y1) of the pressure
 * grid (0 <= y0 < y1 <= number of y positions): its row sweep processes the
 * interior rows inside the band, its column sweep outputs only positions in
 * the band.  The handle's arrays are re-laid out to hold the band plus `halo`
 * positions on each side only (device memory ~ 1/P of the grid): the state rows inside
 * both the old and the new extent are kept, rows new to the extent are zero (call
 * adi_set_fields after widening a band).  adi_set/get_fields move only those rows.
 * The column sweep plans its tiles over the band's own positions.  Between adi_step_rows and adi_step_cols the halo of
 * `halo` positions on each side must be refreshed from the neighbour bands
 * (kind 0: S2 and W*), and before adi_step_begin of every call but the first
 * after adi_set_fields (kind 1: U and W̄).  side 0 = low-y neighbour, 1 = high.
 * adi_halo_pack writes this band's edge positions that the neighbour on `side`
 * needs into a contiguous device buffer of adi_halo_bytes bytes;
 * adi_halo_unpack stores the neighbour's message into this band's halo.
 * EINVAL: a band thinner than the halo, or the handle of an adi_create_dist (fixed band);
 * a refused band leaves the handle unchanged. */
int adi_set_band(adi_handle h, int y0, int y1);
int adi_band_info(adi_handle h, int* y0, int* y1, int* halo, int* npos);

/* One rank of a grid line-sharded over `nranks` processes, one GPU each (
 * DESIGN.md §7), with the exchange INSIDE the library: the handle owns the band
 * adi_dist_bands gives `rank` (adi_set_band), and adi_step performs the halo exchanges
 * itself, as NCCL grouped ncclSend/ncclRecv on the handle's stream: U and W̄ before
 * a call's prologue (skipped right after adi_set_fields), S and W* after every row
 * sweep.  The handle lives on the calling thread's current CUDA device.
 * nccl_unique_id: the 128 bytes of adi_nccl_unique_id from one rank, given to all;
 * every rank must call adi_step with the same n (collective).  adi_set_fields /
 * adi_get_fields move the band's rows (see adi_set_band).  nranks = 1: a plain handle.
 * libnccl.so.2 is loaded at run time; ADI_ENCCL if it is missing or fails.  Not for
 * ADI_CFD_FULL with nranks > 1 (ADI_EINVAL).  The step phases (adi_step_begin ..)
 * do not exchange: drivers that call them exchange through adi_halo_pack/unpack. */
int adi_create_dist(int nx, int ny, double h, double dt, double c, int method, int batch,
                    const void* nccl_unique_id, int rank, int nranks, adi_handle* out);
/* The decomposition of adi_create_dist_ex / adi_create_dist_local_ex:
 *   ADI_DIST_HALO (the default of adi_create_dist): bands of y positions; each rank keeps
 *     its band plus a halo and exchanges the halo rows with its two neighbours (§7.1-7.2);
 *   ADI_DIST_TRANSPOSE (the north_star's plan): rank r owns the rows Y_r for the
 *     row sweep and the columns X_r for the column sweep (the cuts of adi_dist_bands over the
 *     y and the x positions); S moves to its next owner by an all-to-all (NCCL grouped
 *     send/recv, or loopback copies) after the prologue, every row sweep and every column
 *     sweep but the last (§7.3).  adi_set/get_fields: U and W̄ on the columns, V̄ on the
 *     rows (a get returns the owned ones: adi_dist_info).  No media, no halo calls. */
enum { ADI_DIST_HALO = 0, ADI_DIST_TRANSPOSE = 1 };
int adi_create_dist_ex(int nx, int ny, double h, double dt, double c, int method, int batch,
                       const void* nccl_unique_id, int rank, int nranks, int mode, adi_handle* out);
/* This rank's decomposition: mode, the owned rows [rows0, rows1) (y positions: V̄ and, in
 * halo mode, U and W̄) and columns [cols0, cols1) (x positions: U and W̄ in transpose
 * mode; all columns in halo mode).  A plain handle: mode halo, everything owned. */
int adi_dist_info(adi_handle h, int* mode, int* rows0, int* rows1, int* cols0, int* cols1);
int adi_nccl_unique_id(void* out128);
/* All `nranks` ranks of the same decomposition in ONE process on the current device
 * (out[0..nranks-1]), exchanging through loopback device copies instead of NCCL: the
 * code path of adi_create_dist (band-local arrays, pack -> transfer -> unpack, the
 * column sweep's halo-free segments overlapping the transfer) with only the transport
 * replaced.  For verification on one GPU: the ranks are stepped together by
 * adi_step_dist_local (adi_step on one of them returns ADI_ESTATE), which runs every
 * rank's phase before any rank's next one, so no rank's kernel waits on another's.
 * adi_set/get_fields, adi_get_stats and adi_destroy work per rank as for
 * adi_create_dist.  Destroy all handles. */
int adi_create_dist_local(int nx, int ny, double h, double dt, double c, int method, int batch, int nranks,
                          adi_handle* out);
int adi_create_dist_local_ex(int nx, int ny, double h, double dt, double c, int method, int batch, int nranks,
                             int mode, adi_handle* out);
int adi_step_dist_local(adi_handle* handles, int nranks, int n);
/* The band cuts of y positions [0, npos) over nranks: cuts[0..nranks] (host logic only). */
int adi_dist_bands(int npos, int nranks, int* cuts);
/* The halo (positions on each side of a band) that the band decomposition of `method`
 * (ADI_CFD / ADI_MFD) exchanges: the bound of a half-step's domain of influence
 * (DESIGN.md §5.3).  Host logic only; the value adi_band_info reports for a handle.
 * EINVAL for another method. */
int adi_plan_halo(int method, int* halo);
int adi_halo_bytes(adi_handle h, int kind, int side, size_t* bytes);
int adi_halo_pack(adi_handle h, int kind, int side, void* dev_buf);
int adi_halo_unpack(adi_handle h, int kind, int side, const void* dev_buf);

/* Asynchronous forms of adi_set_fields / adi_get_fields: the copies (and the
 * W̄ transposes) are only ENQUEUED on the handle's stream, in order with the
 * handle's steps.  The host arrays should be page-locked (cudaHostAlloc /
 * cudaHostRegister) for the copies to overlap other work; they must stay valid
 * and, for the set, unmodified until the stream has been synchronized.  Same
 * shapes, band rule and errors as the synchronous calls. */
int adi_set_fields_async(adi_handle h, const double* U, const double* V, const double* W);
int adi_get_fields_async(adi_handle h, double* U, double* V, double* W);

/* Copy the state to HOST arrays (synchronizes the stream).  With a band set only
 * the band's rows [y0, y1) are written (the top band also writes the U rows above
 * its last position); the other rows of the arrays are left untouched. */
int adi_get_fields(adi_handle h, double* U, double* V, double* W);
/* Copy the state to DEVICE arrays, enqueued on the handle's stream. */
int adi_get_fields_device(adi_handle h, double* dU, double* dV, double* dW);

int adi_get_stats(adi_handle h, adi_stats* s);

/* Testing aid (compute-sanitizer is not available on every host): with ADI_GUARD_CHECK=1
 * in the environment when the handle's arrays are allocated, the guard regions around
 * every field array hold a canary pattern instead of zeros; this call (synchronizes the
 * stream) counts the 8-byte guard words that no longer hold it, i.e. out-of-bounds writes
 * by a kernel or a copy.  Without the variable the guards are zeros and *bad counts them
 * all. */
int adi_check_guards(adi_handle h, long long* bad);

/* With ADI_TIMING = 1: synchronize the stream, then for each kernel kind k < nkinds
 * return the summed device time ms[k] (CUDA events around each launch) and the
 * launch count since the previous call; the accumulators are reset.  Either array
 * may be NULL. */
int adi_get_kernel_times(adi_handle h, double* ms, long long* launches, int nkinds);

/* Profiling aid.  While dev_buf != NULL, every launch of the line kernel of the given
 * kind (ADI_KK_*) records, for each tile id < cap, 8 unsigned 64-bit words at
 * dev_buf[8 * tile]: {tile, SM id, t_start, t_loaded, t_ops_done, t_end, 0, 0}, times
 * from the %globaltimer register (ns).  A later launch of that kind overwrites the
 * records.  dev_buf is device memory owned by the caller and must hold 64 * cap bytes;
 * NULL turns tracing off.  EINVAL for cap < 0 or an unknown kind, and in a library built
 * without -DADI_TILE_TRACE=1 (the production build: the timer reads are compiled out). */
int adi_set_trace(adi_handle h, void* dev_buf, long long cap, int kind);

/* Sweeps used by the last step's ADI-rows / ADI-columns stages (ADI_K_SWEEPS when
 * ADI_EPS = 0).  Synchronizes the stream. */
int adi_get_last_sweeps(adi_handle h, int* k_rows, int* k_cols);

/* Message for the last error on this handle ("" if none); valid until the next call. */
const char* adi_last_error(adi_handle h);

void adi_destroy(adi_handle h);

/* Library version string and the compiled device architecture ("sm_100a"). */
const char* adi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ADI_H_ */
