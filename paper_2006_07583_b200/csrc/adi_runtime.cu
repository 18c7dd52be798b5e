// adi_runtime.cu — host runtime and C-ABI (include/adi.h) of the B200 ADI
// library.  Builds the operators of App. A/B once per handle, plans the line
// tiles, owns the device buffers and enqueues the per-step kernels:
//
//   adi_step(n):  PROLOGUE (y)  : U, W̄        -> S1, W*          (a2, Alg.1/2 l.8,10)
//                 n x { ROW (x) : S1, V̄       -> S2, V̄^{m+1}     (a3+a4, l.11-14)
//                       COL (y) : S2, W*      -> S1', W*'        (a6 + a2 of m+1, l.15)
//                 }   the last COL is FINAL   -> U^{m+n}, W̄^{m+n}
//                 EDGE          : Dirichlet columns of U at t^{m+n}
//
// Every arithmetic step runs in the kernels of adi_line.cuh.  The host only
// computes the operator coefficient tables (exact rationals of the paper, LU
// without pivoting — PAPER.md:113,192) and scalar time factors.
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>   // types only: libnccl is loaded at run time (adi_create_dist)

#include "adi.h"
#include "adi_line.cuh"
#include "adi_thread.cuh"
#include "adi_warp.cuh"

namespace adi {

constexpr int TM = 32;     // points per thread chunk
constexpr int NW = 4;      // lines (warps) per CTA: S' is written in 32-byte runs
constexpr int TCH = 32;    // chunks per line segment (one per lane)

// segment halo of the line tiles and of the band decomposition
#ifndef ADI_HALO_CFD
#define ADI_HALO_CFD 56
#endif
#ifndef ADI_HALO_MFD
#define ADI_HALO_MFD 28
#endif
inline int plan_halo(int method) { return method == ADI_CFD ? ADI_HALO_CFD : ADI_HALO_MFD; }

struct Axis {
  int n = 0;            // cells along the sweep direction
  int nlines = 0;       // interior pressure lines of the grid
  int l0 = 0, l1 = 0;   // lines processed by this handle (band decomposition)
  int o0 = 0, o1 = 1 << 30;  // output positions of this handle (band decomposition)
  int halo = 0;
  int NL = 1;
  int plo = 0, phi = -1;
  std::vector<Seg> segs;   // interior segments (edge == 0) first
  int nint = 0;            // number of lean segments (edge == 0)
  int nmid = 0;            // of which without a line end (the first nmid)
  int nfree = 0;           // of which reading no halo position of a band (the first nfree): a
                           // band's column sweep launches them before its halo exchange lands
  Seg* d_segs = nullptr;
  // the fragment plan of the MFD SWEEP launches: fsegs = lean tiles
  // (interior first, fnmid of them, then the two line-end tiles), ffrag = the middle
  // fragment of FRAG_CH chunks that the PACK kernel runs for 4 lines per warp
  bool fplan = false;
  std::vector<Seg> fsegs;
  int fnmid = 0;
  Seg* d_fsegs = nullptr;    // fsegs then ffrag
  double* d_tabU = nullptr;  // CFD only
  double* d_tabX = nullptr;
  int* d_ptl = nullptr;      // per batch: point source line / position for this direction
  int* d_ptp = nullptr;
};

}  // namespace adi

struct adi_ctx {
  int dev = 0;          // the CUDA device the handle was created on (DevGuard)
  int method, nx, ny, batch;
  double h, dt, c, rho;
  int K = 8;
  int check_finite = 0;
  int tile_chunks = 0;  // 0 = auto
  int prefetch = 0;     // ADI_PREFETCH: L2 prefetch distance in resident waves (0 = off)
  int timing = 0;
  double eps = 0.0;      // ADI_EPS: inner stopping rule off (fixed K sweeps) when 0
  int kmin = 6;          // ADI_K_MIN
  double* d_norms = nullptr;  // [2 stages][K+1][2] per-sweep squared changes (rows, columns)
  int d_norms_cap = 0;
  int* d_k = nullptr;         // [4]: chosen sweeps (rows, columns) of the last step, gates
  unsigned long long* trace = nullptr;  // adi_set_trace
  long long trace_cap = 0;
  int trace_kind = -1;
  struct Rec { int kind; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  cudaStream_t stream = nullptr;
  // shapes
  int nxu, nyu, nxi, nyi, nxv, nyv;
  size_t nU, nV, nW, nS;  // per grid, dense (user layout)
  // internal layouts are POSITION-INDEXED full grids: the entry of
  // (y position, x position) sits at row y, index x (or row x, index y for the
  // transposed arrays), whatever the field; rows are pitched to multiples of 4
  // doubles and padded by >= 32 so a 32-point chunk never crosses a row end.
  //   U  [y][x] pu     Sa [y][x] pa (S)     Sb [x][y] pb (S^T)
  //   V  [y][x] pv (V̄, rows 1..nyi)        W  [x][y] pw (W̄^T, rows 1..nxi)
  //   phi [y][x] pa,  phiT [x][y] pb
  int pu, pa, pb, pv, pw;
  size_t aU, aS, aV, aW;  // allocation per grid (batch strides)
  // band-local storage: the arrays hold the y positions [ya, yb) only
  // (a whole grid: [0, nyu)).  Row-indexed arrays ([y][x]: U, Sa, V, V2, phi, Ca) and
  // column-indexed arrays ([x][y]: Sb, W, W2, W3, phiT, Cb) keep ABSOLUTE position
  // indexing through an offset base pointer (rows_in / cols_in); the allocation itself
  // is rows_raw / cols_raw.  ya is even (16-byte TMA alignment of the staged rows).
  int ya = 0, yb = 0;
  long long dev_bytes = 0;   // device memory this handle allocated (adi_get_stats)
  std::vector<std::pair<double*, size_t>> allocs;   // the guarded field arrays (adi_check_guards)
  double* Ubase = nullptr;
  // device buffers
  double *U = nullptr, *V = nullptr, *W = nullptr;
  double *V2 = nullptr, *W2 = nullptr, *Sa = nullptr, *Sb = nullptr;
  // carry mode: W3 receives the next step's W* from the last column
  // kernel of a call, Sa its S1; carry_valid: the next call may skip its prologue
  double* W3 = nullptr;
  bool carry_valid = false;
  bool call_carry = false;   // this call ends with the carry kernel (decided by adi_step_begin)
  int cols_phase = 0;        // column launches: 0 all segments, 1 halo-free ones, 2 the rest
  cudaEvent_t split_wait = nullptr;   // set by an in-flight halo exchange (dist handles)
  int call_K = 8;            // K of the call in progress (the stopping rule's buffer size)
  int carry_on = 1;     // ADI_CARRY
  double* phi = nullptr;    // source pattern, S layout (row-major)
  double* phiT = nullptr;   // its transpose (column sweep)
  double* edges = nullptr;  // y0 | y1 | x0 | x1
  // heterogeneous media (adi_set_media, NEXT row f3): (kappa, rho^-1) fp32 pairs per
  // position, Ca [y][x] pa (row sweep: rho^-1 at V̄ points), Cb [x][y] pb (column
  // sweep: rho^-1 at W̄ points); one medium for the whole batch
  double* Ca = nullptr;
  double* Cb = nullptr;
  bool het = false;
  // NEXT row f4 (ADI_CFD_FULL): the full-matrix CFD variant; every node is unknown, the
  // interior index i is position i (off = 0; the reduced variants: off = 1)
  bool full = false;
  int off = 1;
  int absorb_nb = 0;          // ADI_ABSORB_WIDTH (Cerjan layer, points)
  double absorb_a = 0.015;    // ADI_ABSORB_RATE
  double* d_taper = nullptr;  // taper[d], d < absorb_nb
  // adi_create_dist: this rank's band of a line-sharded grid; NCCL halo exchange inside
  // adi_step (the protocol of dist.step_distributed)
  bool dist = false;
  int rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  bool fresh = true;             // every rank holds its band + halo rows (after set_fields)
  double* hbuf[2][2][2] = {};    // [kind][side][send, recv]
  size_t hcount[2][2][2] = {};   // elements
  // transport of the halo messages: NCCL (comm) or, for the ranks of one process on one
  // device (adi_create_dist_local), loopback copies from the neighbours' send buffers
  bool loop = false;
  adi_ctx* peer[2] = {nullptr, nullptr};   // loopback: the low / high neighbour handle
  // ADI_DIST_TRANSPOSE (the north_star's decomposition): rank r
  // owns the rows Y_r = [ty0, ty1) for the row sweep and the columns X_r = [tx0, tx1) for the
  // column sweep; S changes owner between the half-steps by an all-to-all.  Row-side
  // arrays (Sa, V, V2, phi) hold rows [ya, yb) ⊇ Y_r; the row sweep writes S2^T into Sb
  // ([x][y in [ya, yb)]).  Column-side arrays Sc (S2^T input), W, W2, phiT hold the rows
  // x in [xa, xb) ⊇ X_r with all y (pitch pc); the column sweep writes S1'^T into Sd and U
  // ([y][x in [xa, xb)], pitch pd = pu).
  bool tmode = false;
  int ty0 = 0, ty1 = 0, tx0 = 0, tx1 = 0, xa = 0, xb = 0, pc = 0, pd = 0;
  size_t aC = 0;                      // per-grid size of Sc, Sd (common batch stride)
  double *Sc = nullptr, *Sd = nullptr;
  std::vector<int> cut_y, cut_x;      // the ranks' Y_q, X_q
  adi_ctx** group = nullptr;          // loopback: all ranks (adi_create_dist_local)
  std::vector<double*> tsend, trecv;  // NCCL staging per peer (transpose mode)
  // fused transpose (ADI_DIST_FUSED): the S' stores of the row / column
  // kernels write straight into the owning rank's Sc / Sa; the all-to-all becomes a barrier.
  // tpeer[q]: rank q's arrays as addressed from this process (the group's own pointers, or
  // CUDA IPC mappings of the peers' allocations); ipc_open: the mappings to close
  struct TPeer { double* Sc; double* Sa; long long pc, pa, aC, aS; };
  std::vector<TPeer> tpeer;
  bool tfused = false;
  std::vector<void*> ipc_open;
  double* dbar = nullptr;             // the barrier's one-element all-reduce buffer
  std::vector<size_t> tcount;
  cudaStream_t cs = nullptr;               // exchange stream (overlaps the column sweep)
  cudaEvent_t ev_pack = nullptr, ev_recv = nullptr;
  // internal layouts: Sa, V, V2 row-major; Sb = S^T; W, W2 = W̄^T (columns contiguous)
  int* flag = nullptr;
  adi::Axis ax, ay;
  // time tables (host)
  std::vector<double> gf, gb;
  bool has_pt = false;
  long long m = 0;  // steps taken
  long long launches = 0;
  long long host_launches = 0;   // launch API calls (a graph launch counts once)
  // ADI_GRAPH: each adi_step(n) is captured into a CUDA graph and launched at once; the
  // executable graph is kept and updated in place while the captured topology repeats
  int graph_on = 0;
  int small = -1;   // ADI_THREAD_LINES: -1 auto (short lines), 0 off, 1 on where possible
  int warp_lines = 1;   // ADI_WARP_LINES: short lines (<= 64 positions) on the warp-per-line kernels
  int frag_on = 1;      // ADI_FRAG_TILES: the MFD fragment plan where it applies
  int async_store = 0;   // ADI_ASYNC_STORE: the SWEEP tiles' outputs by TMA / bulk copies (measured:
                         // no gain, the store phase is bound by the memory system)
  bool capturing = false;
  cudaStream_t gstream = nullptr;   // capture stream when the handle's stream is the legacy one
  cudaGraphExec_t gexec = nullptr;
  bool fields_set = false;
  int nonfinite = 0;
  std::string err;
  // band decomposition (multi-GPU): this handle owns y positions [band_y0, band_y1)
  int band_y0 = 0, band_y1 = 1 << 30;
  // state of a call in progress (adi_step_begin .. adi_step_end)
  bool in_call = false;
  long long call_m1 = 0;
  double *Vcur = nullptr, *Valt = nullptr, *Wcur = nullptr, *Walt = nullptr;
  // TMA tensor maps of the staged arrays (keyed by base pointer)
  struct TMap { const double* ptr; CUtensorMap map; int box = 32; };   // box: chunks per copy
  std::vector<TMap> tmaps;
  struct SMap { const double* ptr; CUtensorMap map; int l0, p0; };
  std::vector<SMap> smaps;   // TMA store maps of the S' outputs (ADI_ASYNC_STORE)
};

namespace {

const char* kVersion = "adi-b200 0.1 (sm_100a)";
// __constant__ memory and function attributes are per device: the tables are uploaded
// once per device a handle is created on (one handle per device and host thread, but
// handles on several devices in one process are allowed)
constexpr int kMaxDev = 64;
std::mutex g_const_mu;
bool g_const_ready[kMaxDev] = {};

// Every call on a handle runs on the handle's device and restores the caller's
// current device afterwards.
struct DevGuard {
  int prev = -1;
  explicit DevGuard(const adi_ctx* h) {
    int cur = 0;
    if (h && cudaGetDevice(&cur) == cudaSuccess && cur != h->dev && cudaSetDevice(h->dev) == cudaSuccess)
      prev = cur;
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int fail(adi_ctx* h, int code, const std::string& msg) {
  if (h) h->err = msg;
  return code;
}

#define CUDA_TRY(h, call)                                                                  \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail((h), ADI_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)

// ---- NCCL, loaded at run time (adi_create_dist) ---------------------------------
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) =
      nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;
bool nccl_load() {
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
  // the process may already hold a libnccl (e.g. torch's); the soname resolves to it
  void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) return false;
  auto sym = [&](const char* n) { return dlsym(lib, n); };
  g_nccl.getUniqueId = (decltype(g_nccl.getUniqueId))sym("ncclGetUniqueId");
  g_nccl.commInitRank = (decltype(g_nccl.commInitRank))sym("ncclCommInitRank");
  g_nccl.commDestroy = (decltype(g_nccl.commDestroy))sym("ncclCommDestroy");
  g_nccl.send = (decltype(g_nccl.send))sym("ncclSend");
  g_nccl.recv = (decltype(g_nccl.recv))sym("ncclRecv");
  g_nccl.groupStart = (decltype(g_nccl.groupStart))sym("ncclGroupStart");
  g_nccl.allReduce = (decltype(g_nccl.allReduce))sym("ncclAllReduce");   // (optional: fused transpose)
  g_nccl.groupEnd = (decltype(g_nccl.groupEnd))sym("ncclGroupEnd");
  g_nccl.errorString = (decltype(g_nccl.errorString))sym("ncclGetErrorString");
  g_nccl.ok = g_nccl.getUniqueId && g_nccl.commInitRank && g_nccl.commDestroy && g_nccl.send && g_nccl.recv &&
              g_nccl.groupStart && g_nccl.groupEnd && g_nccl.errorString;
  return g_nccl.ok;
}
#define NCCL_TRY(h, call)                                                                          \
  do {                                                                                             \
    ncclResult_t r_ = (call);                                                                      \
    if (r_ != ncclSuccess) return fail((h), ADI_ENCCL, std::string(#call) + ": " + g_nccl.errorString(r_)); \
  } while (0)

// Host -> device copies of set-up data.  They go on the handle's stream and are
// waited for: a plain cudaMemcpy from pageable memory may return before the DMA
// lands, and a non-blocking user stream would not wait for the legacy stream.
#define H2D_SYNC(h, dst, src, bytes)                                                             \
  do {                                                                                           \
    CUDA_TRY((h), cudaMemcpyAsync((dst), (src), (bytes), cudaMemcpyHostToDevice, (h)->stream)); \
    CUDA_TRY((h), cudaStreamSynchronize((h)->stream));                                           \
  } while (0)

// ---- device arrays read by the line kernels' TMA copies carry guard regions
// (adi_line.cuh: a staged row may start TMA_P0 positions before a line and end
// past the last line); allocations are zeroed.
// ADI_GUARD_CHECK=1 in the environment (a testing aid in place of compute-sanitizer, which
// this pool does not offer): the guards are filled with a canary byte pattern instead of
// zeros, and adi_check_guards reports guard words that a kernel or copy overwrote
constexpr unsigned char kCanary = 0xA5;
static bool guard_canary() {
  const char* e = std::getenv("ADI_GUARD_CHECK");
  return e && e[0] == '1';
}
double* dalloc(size_t n) {
  void* raw = nullptr;
  const size_t tot = (n + adi::BUF_GUARD_FRONT + adi::BUF_GUARD_TAIL) * sizeof(double);
  if (cudaMalloc(&raw, tot) != cudaSuccess) { cudaGetLastError(); return nullptr; }
  // zeroed synchronously: later work may run on a non-blocking stream
  if (cudaMemset(raw, 0, tot) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    cudaGetLastError(); cudaFree(raw); return nullptr;
  }
  if (guard_canary()) {
    char* c = static_cast<char*>(raw);
    if (cudaMemset(c, kCanary, adi::BUF_GUARD_FRONT * sizeof(double)) != cudaSuccess ||
        cudaMemset(c + tot - adi::BUF_GUARD_TAIL * sizeof(double), kCanary, adi::BUF_GUARD_TAIL * sizeof(double)) !=
            cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
      cudaGetLastError(); cudaFree(raw); return nullptr;
    }
  }
  return static_cast<double*>(raw) + adi::BUF_GUARD_FRONT;
}
void dfree(double* p) {
  if (p) cudaFree(p - adi::BUF_GUARD_FRONT);
}
double* halloc(adi_ctx* h, size_t n) {
  double* p = dalloc(n);
  if (p) {
    h->dev_bytes += (long long)((n + adi::BUF_GUARD_FRONT + adi::BUF_GUARD_TAIL) * sizeof(double));
    h->allocs.push_back({p, n});
  }
  return p;
}
void hfree(adi_ctx* h, double* raw, size_t n) {
  if (!raw) return;
  for (size_t k = 0; k < h->allocs.size(); ++k)
    if (h->allocs[k].first == raw) { h->allocs.erase(h->allocs.begin() + k); break; }
  dfree(raw);
  h->dev_bytes -= (long long)((n + adi::BUF_GUARD_FRONT + adi::BUF_GUARD_TAIL) * sizeof(double));
}
// absolute-position views of band-local arrays (adi_ctx::ya)
double* rows_in(const adi_ctx* h, double* raw, int pitch) { return raw ? raw - (ptrdiff_t)h->ya * pitch : nullptr; }
double* cols_in(const adi_ctx* h, double* raw) { return raw ? raw - h->ya : nullptr; }
double* rows_raw(const adi_ctx* h, double* p, int pitch) { return p ? p + (ptrdiff_t)h->ya * pitch : nullptr; }
double* cols_raw(const adi_ctx* h, double* p) { return p ? p + h->ya : nullptr; }
int padp(int npos) { return (npos + 34 + 3) / 4 * 4; }
constexpr size_t kSrcSlack = 1152;   // doubles behind the source pattern arrays (see adi_set_source)
// pitches and per-grid sizes of the y extent [ya, yb)
void set_extent(adi_ctx* h, int ya, int yb) {
  h->ya = ya;
  h->yb = yb;
  const int ny = yb - ya;
  h->pb = padp(ny);
  h->pw = padp(ny);
  h->aU = (size_t)ny * h->pu;
  h->aS = std::max((size_t)ny * h->pa, (size_t)h->nxu * h->pb);
  h->aV = (size_t)ny * h->pv;
  h->aW = std::max((size_t)h->nxu * h->pw, (size_t)ny * h->nxi);  // W2 also serves as a dense scratch
}

// ---- TMA tensor maps (driver entry point fetched through the runtime)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;

// the overlapping-row view of a pitched line array (adi_line.cuh, TMA_P0)
int encode_lines(adi_ctx* h, const double* base, int pitch, int rows, size_t bstride, int batch,
                 CUtensorMap* out, int boxch = 32) {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
      cudaGetLastError();
      return fail(h, ADI_ECUDA, "cuTensorMapEncodeTiled unavailable");
    }
    g_encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  const cuuint64_t dims[5] = {34, 16, (cuuint64_t)((pitch + adi::TMA_P0 + 31) / 32 + 1), (cuuint64_t)rows,
                              (cuuint64_t)batch};
  const cuuint64_t strides[4] = {16, 256, (cuuint64_t)pitch * 8, (cuuint64_t)bstride * 8};
  const cuuint32_t box[5] = {34, 1, (cuuint32_t)boxch, 1, 1};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  const CUresult r = g_encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)(base - adi::TMA_P0), dims, strides,
                              box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
#ifndef ADI_L2PROMO
#define ADI_L2PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
                              ADI_L2PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(h, ADI_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return ADI_OK;
}

// the TMA STORE map of a transposed S' output array (ADI_ASYNC_STORE): dims {lines
// (contiguous), positions, batch}, box {4 lines, 4 positions, 1}; line / position origins
int tmap_store_for(adi_ctx* h, const double* ptr, CUtensorMap* out, int* line0, int* pos0) {
  for (auto& e : h->smaps)
    if (e.ptr == ptr) { *out = e.map; *line0 = e.l0; *pos0 = e.p0; return ADI_OK; }
  adi_ctx::SMap e{};
  e.ptr = ptr;
  const double* raw;
  cuuint64_t d0, d1;
  size_t pitch, bs = h->aS;
  if (ptr == h->Sb) {          // row sweep output [x][y]: lines y (origin ya), positions x
    raw = cols_raw(h, const_cast<double*>(ptr)); d0 = h->yb - h->ya; d1 = h->nxu; pitch = h->pb;
    e.l0 = h->ya; e.p0 = 0;
  } else if (ptr == h->Sa) {   // column sweep output [y][x]: lines x, positions y (origin ya)
    raw = rows_raw(h, const_cast<double*>(ptr), h->pa); d0 = h->nxu; d1 = h->yb - h->ya; pitch = h->pa;
    e.l0 = 0; e.p0 = h->ya;
  } else if (h->tmode && ptr == h->Sd) {   // transpose mode: [y][x in [xa, xb)]
    raw = ptr + h->xa; d0 = h->xb - h->xa; d1 = h->nyu; pitch = h->pd; bs = h->aC;
    e.l0 = h->xa; e.p0 = 0;
  } else {
    return fail(h, ADI_EINVAL, "internal: no store map for this array");
  }
  if (!g_encode) {
    CUtensorMap tmp;
    int rc = encode_lines(h, h->Sa, h->pa, 1, h->aS, 1, &tmp);   // (fetches the entry point)
    if (rc) return rc;
  }
  const cuuint64_t dims[3] = {d0, d1, (cuuint64_t)h->batch};
  const cuuint64_t strides[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)bs * 8};
  const cuuint32_t box[3] = {4, 4, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = g_encode(&e.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)raw, dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(h, ADI_ECUDA, "cuTensorMapEncodeTiled (store) failed: " + std::to_string((int)r));
  h->smaps.push_back(e);
  *out = e.map;
  *line0 = e.l0;
  *pos0 = e.p0;
  return ADI_OK;
}

// tensor map of one of the handle's staged arrays
int tmap_for(adi_ctx* h, const double* ptr, CUtensorMap* out, int boxch = 32) {
  for (auto& e : h->tmaps)
    if (e.ptr == ptr && e.box == boxch) { *out = e.map; return ADI_OK; }
  int pitch, rows, batch = h->batch;
  size_t bs;
  const int nyb = h->yb - h->ya;   // rows of the band-local row-indexed arrays
  const double* raw = nullptr;     // the allocation (TMA coordinates: tline0 / tpos0)
  if (h->tmode && (ptr == h->Sc || ptr == h->W || ptr == h->W2 || ptr == h->phiT)) {
    adi_ctx::TMap e;
    e.ptr = ptr;
    const size_t bs = (ptr == h->W || ptr == h->W2) ? h->aW : h->aC;
    e.box = boxch;
    int rc = encode_lines(h, ptr + (ptrdiff_t)h->xa * h->pc, h->pc, h->xb - h->xa, bs,
                          ptr == h->phiT ? 1 : h->batch, &e.map, boxch);
    if (rc) return rc;
    h->tmaps.push_back(e);
    *out = e.map;
    return ADI_OK;
  }
  auto rr = [&](int pt) { return rows_raw(h, const_cast<double*>(ptr), pt); };
  auto rc_ = [&]() { return cols_raw(h, const_cast<double*>(ptr)); };
  if (ptr == h->Sa) { pitch = h->pa; rows = nyb; bs = h->aS; raw = rr(pitch); }
  else if (ptr == h->Sb) { pitch = h->pb; rows = h->nxu; bs = h->aS; raw = rc_(); }
  else if (ptr == h->V || ptr == h->V2) { pitch = h->pv; rows = nyb; bs = h->aV; raw = rr(pitch); }
  else if (ptr == h->W || ptr == h->W2 || ptr == h->W3) { pitch = h->pw; rows = h->nxu; bs = h->aW; raw = rc_(); }
  else if (ptr == h->phi) { pitch = h->pa; rows = nyb; bs = h->aS; batch = 1; raw = rr(pitch); }
  else if (ptr == h->phiT) { pitch = h->pb; rows = h->nxu; bs = h->aS; batch = 1; raw = rc_(); }
  else if (ptr == h->Ca) { pitch = h->pa; rows = nyb; bs = h->aS; batch = 1; raw = rr(pitch); }
  else if (ptr == h->Cb) { pitch = h->pb; rows = h->nxu; bs = h->aS; batch = 1; raw = rc_(); }
  else return fail(h, ADI_EINVAL, "internal: no tensor map for this array");
  adi_ctx::TMap e;
  e.ptr = ptr;
  e.box = boxch;
  int rc = encode_lines(h, raw, pitch, rows, bs, batch, &e.map, boxch);
  if (rc) return rc;
  h->tmaps.push_back(e);
  *out = e.map;
  return ADI_OK;
}

// ---- Woodbury data of the lean CFD end tiles.  The lean solve
// applies T* = L*U* on the segment (forward y_p = r_p - l y_{p-1}, backward
// z_p = iv (y_p - z_{p+1}); first pivot 1/iv).  The operator with the line-end rows
// of P̄ (u-op) or P (x-op), and identity rows at positions outside the system, is
// A = T* + U V^T with U = [e_rows].  Work on a 64-position window at the end:
// start: window = segment positions 0..63, end chunk = window 0..31; end: window =
// positions e-63..e (e = segment end), end chunk = window 32..63.
void wb_setup(double l, double iv, double V[6][3][4], double Mx[6][32][3]) {
  typedef long double R;
  const R dd = 1.0L / (R)iv;             // pivot of U*
  const R a = (R)l * dd, b = (R)l + dd;  // T* sub-diagonal and diagonal (after the first row)
  struct Ent { int row, col; R v; };
  for (int cs = 0; cs < 6; ++cs) {
    const int sys = cs / 3, e = cs % 3;  // sys 0: u-op (P̄), 1: x-op (P)
    Ent E[8];
    int ne = 0;
    auto put = [&](int r, int c, R v) { E[ne++] = Ent{r, c, v}; };
    if (e == 0) {
      if (sys == 0) { put(0, 0, 1 - dd); put(0, 1, -1); put(1, 0, -a); put(1, 1, 6 - b); put(1, 2, 5); }
      else { put(0, 0, 6 - dd); put(0, 1, 17); }
    } else if (e == 1) {  // position n = window 63
      if (sys == 0) { put(62, 61, 6 - a); put(62, 62, 6 - b); put(62, 63, -1); put(63, 62, -a); put(63, 63, 1 - b); }
      else { put(63, 62, 18 - a); put(63, 63, 6 - b); }
    } else {              // position n+1 = window 63 (dead)
      if (sys == 0) {
        put(61, 60, 6 - a); put(61, 61, 6 - b); put(61, 62, -1); put(62, 61, -a); put(62, 62, 1 - b);
        put(62, 63, -1); put(63, 62, -a); put(63, 63, 1 - b);
      } else {
        put(62, 61, 18 - a); put(62, 62, 6 - b); put(62, 63, -1); put(63, 62, -a); put(63, 63, 1 - b);
      }
    }
    std::vector<int> rows;
    for (int q = 0; q < ne; ++q)
      if (std::find(rows.begin(), rows.end(), E[q].row) == rows.end()) rows.push_back(E[q].row);
    const int k = (int)rows.size();
    // W_j = T*^{-1} e_{rows[j]} on the window
    R W[3][64] = {};
    for (int j = 0; j < k; ++j) {
      R y[64], z[64];
      R prev = 0;
      for (int q = 0; q < 64; ++q) { y[q] = (q == rows[j] ? 1 : 0) - (R)l * prev; prev = y[q]; }
      R nxt = 0;
      for (int q = 63; q >= 0; --q) { z[q] = (R)iv * (y[q] - nxt); nxt = z[q]; }
      for (int q = 0; q < 64; ++q) W[j][q] = z[q];
    }
    // C = I + V^T W, its inverse (k <= 3, Gauss-Jordan)
    R C[3][3] = {}, Ci[3][3] = {};
    for (int j = 0; j < 3; ++j) { C[j][j] = 1; Ci[j][j] = 1; }
    for (int t = 0; t < ne; ++t) {
      const Ent& x = E[t];
      const int j = (int)(std::find(rows.begin(), rows.end(), x.row) - rows.begin());
      for (int q = 0; q < k; ++q) C[j][q] += x.v * W[q][x.col];
    }
    for (int c = 0; c < k; ++c) {
      int pv = c;
      for (int r = c + 1; r < k; ++r)
        if (std::fabs((double)C[r][c]) > std::fabs((double)C[pv][c])) pv = r;
      for (int q = 0; q < 3; ++q) { std::swap(C[c][q], C[pv][q]); std::swap(Ci[c][q], Ci[pv][q]); }
      const R inv = 1 / C[c][c];
      for (int q = 0; q < 3; ++q) { C[c][q] *= inv; Ci[c][q] *= inv; }
      for (int r = 0; r < k; ++r)
        if (r != c) {
          const R f = C[r][c];
          for (int q = 0; q < 3; ++q) { C[r][q] -= f * C[c][q]; Ci[r][q] -= f * Ci[c][q]; }
        }
    }
    // V over 4 chunk elements (0..3 at the start = window 0..3; 28..31 at the end = window 60..63)
    const int w0 = (e == 0) ? 0 : 60;
    for (int j = 0; j < 3; ++j)
      for (int q = 0; q < 4; ++q) V[cs][j][q] = 0.0;
    for (int t = 0; t < ne; ++t) {
      const Ent& x = E[t];
      const int j = (int)(std::find(rows.begin(), rows.end(), x.row) - rows.begin());
      V[cs][j][x.col - w0] += (double)x.v;
    }
    // M = W C^{-1} on the end chunk
    const int c0 = (e == 0) ? 0 : 32;
    for (int i = 0; i < 32; ++i)
      for (int j = 0; j < 3; ++j) {
        R acc = 0;
        for (int q = 0; q < k; ++q) acc += W[q][c0 + i] * Ci[q][j];
        Mx[cs][i][j] = (j < k) ? (double)acc : 0.0;
      }
  }
}

// ---- constants: MFD closures as the printed rationals (App. B), CFD interior LU
int init_constants(adi_ctx* h) {
  if (h->dev < 0 || h->dev >= kMaxDev) return fail(h, ADI_ECUDA, "device ordinal out of range");
  std::lock_guard<std::mutex> lock(g_const_mu);
  if (g_const_ready[h->dev]) return ADI_OK;
  const double d4r0[6] = {-4751.0 / 5192.0, 909.0 / 1298.0, 6091.0 / 15576.0,
                          -1165.0 / 5192.0, 129.0 / 2596.0, -25.0 / 15576.0};
  const double g4r0[6] = {-47888.0 / 14245.0, 1790.0 / 407.0, -14545.0 / 9768.0,
                          8997.0 / 16280.0, -2335.0 / 22792.0, 25.0 / 9768.0};
  const double g4r1[5] = {16.0 / 105.0, -31.0 / 24.0, 29.0 / 24.0, -3.0 / 40.0, 1.0 / 168.0};
  CUDA_TRY(h, cudaMemcpyToSymbol(adi::c_d4r0, d4r0, sizeof d4r0));
  CUDA_TRY(h, cudaMemcpyToSymbol(adi::c_g4r0, g4r0, sizeof g4r0));
  CUDA_TRY(h, cudaMemcpyToSymbol(adi::c_g4r1, g4r1, sizeof g4r1));
  // interior rows (1, 4, 1): the no-pivot LU recursion d <- 4 - 1/d converges to 2+sqrt(3)
  double d = 4.0;
  for (int i = 0; i < 200; ++i) d = 4.0 - 1.0 / d;
  const double l = 1.0 / d, invd = 1.0 / d;
  const int M = adi::TM;
  double G[adi::MMAX], Kc[adi::MMAX], Jc[adi::MMAX];
  double g = 1.0;
  for (int i = 0; i < M; ++i) { g *= -l; G[i] = g; }
  double k = 0.0, j = 1.0;
  for (int i = M - 1; i >= 0; --i) {
    k = (G[i] - k) * invd;  // c = 1
    j *= -invd;
    Kc[i] = k;
    Jc[i] = j;
  }
  for (int i = M; i < adi::MMAX; ++i) Kc[i] = Jc[i] = 0.0;
  const double F = G[M - 1], Ks = Kc[0], Ke = Kc[M - 1], Js = Jc[0], Je = Jc[M - 1];
  CUDA_TRY(h, cudaMemcpyToSymbol(adi::c_cl, &l, sizeof l));
  CUDA_TRY(h, cudaMemcpyToSymbol(adi::c_cinvd, &invd, sizeof invd));
  CUDA_TRY(h, cudaMemcpyToSymbol(adi::c_cF, &F, sizeof F));
  CUDA_TRY(h, cudaMemcpyToSymbol(adi::c_cKs, &Ks, sizeof Ks));
  CUDA_TRY(h, cudaMemcpyToSymbol(adi::c_cKe, &Ke, sizeof Ke));
  CUDA_TRY(h, cudaMemcpyToSymbol(adi::c_cJs, &Js, sizeof Js));
  CUDA_TRY(h, cudaMemcpyToSymbol(adi::c_cJe, &Je, sizeof Je));
  // responses of an interior sub-chunk of L = M / NSUB points (same formulas)
  {
    const int L = M / adi::NSUB;
    double Gs[adi::MMAX], sK[adi::MMAX], sJ[adi::MMAX];
    double gg = 1.0;
    for (int i = 0; i < L; ++i) { gg *= -l; Gs[i] = gg; }
    double kk = 0.0, jj = 1.0;
    for (int i = L - 1; i >= 0; --i) {
      kk = (Gs[i] - kk) * invd;
      jj *= -invd;
      sK[i] = kk;
      sJ[i] = jj;
    }
    for (int i = L; i < adi::MMAX; ++i) sK[i] = sJ[i] = 0.0;
    const double sF = Gs[L - 1];
    CUDA_TRY(h, cudaMemcpyToSymbol(adi::c_sK, sK, sizeof sK));
    CUDA_TRY(h, cudaMemcpyToSymbol(adi::c_sJ, sJ, sizeof sJ));
    CUDA_TRY(h, cudaMemcpyToSymbol(adi::c_sF, &sF, sizeof sF));
  }
  // line-end corrections of the lean CFD tiles (adi_line.cuh, c_wbV / c_wbM)
  {
    double V[6][3][4], Mx[6][32][3], N[6][4][3], F[6][3], rho[32];
    wb_setup(l, invd, V, Mx);
    // near entries exact; the rest as the geometric tail F_j rho^d (d = distance
    // from the line end) -- T*^{-1} e_r is geometric away from the rows
    rho[0] = 1.0;
    for (int q = 1; q < 32; ++q) rho[q] = rho[q - 1] * (-l);
    for (int cs = 0; cs < 6; ++cs) {
      const bool start = (cs % 3) == 0;
      for (int q = 0; q < 4; ++q)
        for (int j = 0; j < 3; ++j) N[cs][q][j] = Mx[cs][start ? q : 28 + q][j];
      for (int j = 0; j < 3; ++j) {
        F[cs][j] = Mx[cs][start ? 4 : 27][j] / rho[4];
        double mx = 0.0, err = 0.0;
        for (int i = 0; i < 32; ++i) mx = std::max(mx, std::fabs(Mx[cs][i][j]));
        for (int q = 4; q < 32; ++q)
          err = std::max(err, std::fabs(F[cs][j] * rho[q] - Mx[cs][start ? q : 31 - q][j]));
        if (mx > 0 && err > 1e-15 * mx)
          return fail(h, ADI_ECUDA, "internal: line-end correction is not geometric");
      }
    }
    CUDA_TRY(h, cudaMemcpyToSymbol(adi::c_wbV, V, sizeof V));
    CUDA_TRY(h, cudaMemcpyToSymbol(adi::c_wbN, N, sizeof N));
    CUDA_TRY(h, cudaMemcpyToSymbol(adi::c_wbF, F, sizeof F));
    CUDA_TRY(h, cudaMemcpyToSymbol(adi::c_rho, rho, sizeof rho));
  }
  g_const_ready[h->dev] = true;
  return ADI_OK;
}

// ---- CFD LU tables (position-indexed, 3 x (n+1)): l, 1/d, c.  P̄ (u-op) lives on
// positions 1..n-1 (eq. 14), P (x-op) on 0..n (eq. 12); LU without pivoting.
bool cfd_table(int n, bool bar, std::vector<double>& tab, double& maxdev_lo, int& plo) {
  const int np1 = n + 1;
  tab.assign(3 * np1, 0.0);
  const int p0 = bar ? 1 : 0, p1 = bar ? n - 1 : n;
  std::vector<double> a(np1, 1.0), bb(np1, 4.0), cc(np1, 1.0);
  if (bar) { bb[1] = 6; cc[1] = 6; a[n - 1] = 6; bb[n - 1] = 6; cc[n - 1] = 0; }
  else { bb[0] = 6; cc[0] = 18; a[n] = 18; bb[n] = 6; cc[n] = 0; }
  double dprev = 0.0;
  for (int p = p0; p <= p1; ++p) {
    double l = (p == p0) ? 0.0 : a[p] / dprev;
    double d = bb[p] - l * ((p == p0) ? 0.0 : cc[p - 1]);
    if (d == 0.0) return false;
    tab[p] = l;
    tab[np1 + p] = 1.0 / d;
    tab[2 * np1 + p] = (p == p1) ? 0.0 : cc[p];
    dprev = d;
  }
  // first position from which (l, 1/d) equal the interior constants to 2 ulp
  double dstar = 4.0;
  for (int i = 0; i < 200; ++i) dstar = 4.0 - 1.0 / dstar;
  plo = p1;
  for (int p = p0 + 1; p < p1; ++p) {
    bool ok = true;
    for (int q = p; q < std::min(p1, p + 8); ++q)
      ok = ok && std::fabs(tab[np1 + q] * dstar - 1.0) < 5e-16 && std::fabs(tab[q] * dstar - 1.0) < 5e-16;
    if (ok) { plo = p; break; }
  }
  maxdev_lo = 0.0;
  return true;
}

// ---- tile planning along one axis.  The owned positions
// [lo_all, hi_all) (the whole line, or a band of the decomposition, §7) are split
// evenly into S segments; a segment's tile covers its part plus `halo` on each
// side, except at a line end, where the tile contains the end itself (exact).
bool plan_axis(adi::Axis& A, int method, int cap, int lo_all, int hi_all) {
  const int M = adi::TM;
  const int chmax = cap > 0 ? std::min(cap, adi::TCH) : adi::TCH;
  const int P = A.n + 1;                       // positions 0..n
  const int halo = adi::plan_halo(method);
  A.halo = halo;
  A.segs.clear();
  lo_all = std::max(lo_all, 0);
  hi_all = std::min(hi_all, P);
  // Chunk starts are kept even (16-byte aligned rows for the TMA copies).
  const int D = (M - P % M) % M;
  const int nch1 = (P + D) / M;
  // the whole line in one tile -- unless only a band of it is owned (a band-local handle
  // holds the band and its halo rows only)
  if (nch1 <= chmax && lo_all <= 0 && hi_all >= P) {
    const int ds = (D / 2) & ~1;   // dead positions before 0 (even); the rest after n
    A.segs.push_back({-ds, nch1, lo_all, hi_all, 1});
    return true;
  }
  const int CH = chmax;
  const int R = hi_all - lo_all;
  if (R <= 0) return true;
  for (int S = 1; S <= R / 2 + 1; ++S) {
    std::vector<adi::Seg> segs;
    bool fits = true;
    for (int s = 0; s < S && fits; ++s) {
      const int lo = lo_all + (int)((long long)s * R / S), hi = lo_all + (int)((long long)(s + 1) * R / S);
      const int a = lo - halo, e = hi + halo;   // positions the tile must hold
      adi::Seg g{};
      g.out_lo = lo;
      g.out_hi = hi;
      if (a <= 0 && e >= P) { fits = false; break; }      // would need the whole line
      if (a <= 0) {                                       // holds the line start
        g.start = 0;
        g.nchunks = (e + M - 1) / M;
      } else if (e >= P) {                                // holds the line end
        // end the last chunk at n (or n+1, one dead position, to keep the start even);
        // with the full chunk count the line end sits in chunk 31 (lean end tile)
        // (a short line -- a band of it -- takes a generic tile of the chunks it needs)
        // (a band-local array starts at (lo_all - halo) & ~1: the lean end tile must not start below)
        const int ext_lo = lo_all > 0 ? ((lo_all - halo) & ~1) : 2;
        g.nchunks = (CH == adi::TCH && P - CH * M >= std::max(2, ext_lo)) ? CH : (P - a + M - 1) / M;
        g.start = P - g.nchunks * M;
        if (g.start & 1) g.start += 1;
        if (g.start > a) { g.nchunks += 1; g.start -= M; }
        if (g.start < 1) { fits = false; break; }
      } else {
        g.start = a & ~1;
        g.nchunks = (e - g.start + M - 1) / M;
      }
      if (g.nchunks > CH) fits = false;
      segs.push_back(g);
    }
    if (fits) { A.segs = segs; return true; }
  }
  return false;
}

int setup_axis(adi_ctx* h, adi::Axis& A, int n, int nlines, int nlmin) {
  A.n = n;
  A.nlines = nlines;
  // lines are positions off..nlines-1+off (the full variant: every line)
  if (A.l1 == 0 && A.l0 == 0) { A.l0 = h->off; A.l1 = nlines + h->off; }
  (void)nlmin;
  // the owned positions: the whole line, or this handle's band (adi_set_band)
  if (!plan_axis(A, h->method, h->tile_chunks, A.o0, A.o1))
    return fail(h, ADI_EINVAL, "tile planning failed (grid too small for the tile cap)");
  {
    std::vector<adi::Seg> keep;
    for (adi::Seg g : A.segs)
      if (g.out_lo < g.out_hi) keep.push_back(g);
    A.segs = keep;
    if (A.segs.empty()) A.segs.push_back({0, 0, 0, 0, 1});  // nothing to output: an idle tile
  }
  if (A.d_segs) { cudaFree(A.d_segs); A.d_segs = nullptr; }
  if (A.d_fsegs) { cudaFree(A.d_fsegs); A.d_fsegs = nullptr; }
  A.fplan = false;
  A.fsegs.clear();
  if (A.d_tabU) { cudaFree(A.d_tabU); A.d_tabU = nullptr; }
  if (A.d_tabX) { cudaFree(A.d_tabX); A.d_tabX = nullptr; }
  if (h->method == ADI_CFD) {
    std::vector<double> tu, tx;
    double dev;
    int plo_u, plo_x;
    if (!cfd_table(n, true, tu, dev, plo_u) || !cfd_table(n, false, tx, dev, plo_x))
      return fail(h, ADI_EZEROPIVOT, "zero pivot in the LU of P or P-bar");
    A.plo = std::max(std::max(plo_u, plo_x), 2);
    // edge tiles stage the LU tables of positions within 64 of a line end (adi_line.cuh)
    if (n >= 64 && A.plo > 32)
      return fail(h, ADI_EINVAL, "CFD LU pivots do not converge near the line ends");
    A.phi = n - 2;
    CUDA_TRY(h, cudaMalloc(&A.d_tabU, tu.size() * sizeof(double)));
    CUDA_TRY(h, cudaMalloc(&A.d_tabX, tx.size() * sizeof(double)));
    H2D_SYNC(h, A.d_tabU, tu.data(), tu.size() * sizeof(double));
    H2D_SYNC(h, A.d_tabX, tx.data(), tx.size() * sizeof(double));
  } else {
    A.plo = 2;
    A.phi = n - 2;
  }
  for (adi::Seg& g : A.segs) {
    // Lean tiles: the active chunks avoid the end rows (positions
    // 0, 1 and n-1, n), or the segment starts at the line start, or the line end
    // sits in chunk 31.  The lean kernel also runs the chunks beyond nchunks on the
    // (finite) data past the segment; they only move the truncation boundary further
    // from the owned range.  Everything else (short lines) takes the generic kernel.
    const int last = g.start + g.nchunks * adi::TM - 1;
    const int full = g.start + adi::TCH * adi::TM - 1;
    g.edge = 0;
    g.end = 0;
    if (g.nchunks <= 0) g.edge = 1;
    else if (g.start >= 2 && last <= n - 2) g.end = 0;
    else if (g.start == 0 && last <= n - 2) g.end = 1;
    else if (g.nchunks == adi::TCH && g.start >= 2 && full == n) g.end = 2;
    else if (g.nchunks == adi::TCH && g.start >= 2 && full == n + 1) g.end = 3;
    else g.edge = 1;
  }
  // launch order: lean interior segments (no line end), lean line-end segments, generic
  std::stable_partition(A.segs.begin(), A.segs.end(), [](const adi::Seg& g) { return g.edge == 0; });
  std::stable_partition(A.segs.begin(), A.segs.end(), [](const adi::Seg& g) { return g.edge == 0 && g.end == 0; });
  A.nint = 0;
  A.nmid = 0;
  for (const adi::Seg& g : A.segs) { A.nint += (g.edge == 0); A.nmid += (g.edge == 0 && g.end == 0); }
  {
    // band decomposition: the interior segments whose staged positions stay inside the
    // owned range [o0, o1) need no halo; they go first (overlap)
    const int npos = A.n + 1;
    auto free_of_halo = [&](const adi::Seg& g) {
      return !((A.o0 > 0 && g.start < A.o0) || (A.o1 < npos && g.start + adi::TCH * adi::TM + 2 > A.o1));
    };
    std::stable_partition(A.segs.begin(), A.segs.begin() + A.nmid, free_of_halo);
    A.nfree = 0;
    for (int k = 0; k < A.nmid; ++k) A.nfree += free_of_halo(A.segs[k]);
  }
  CUDA_TRY(h, cudaMalloc(&A.d_segs, A.segs.size() * sizeof(adi::Seg)));
  H2D_SYNC(h, A.d_segs, A.segs.data(), A.segs.size() * sizeof(adi::Seg));
  // the fragment plan (MFD, whole lines, lean tiles only): the two line-end tiles own
  // 1024 - halo positions, k interior tiles 1024 - 2 halo each, and the gap between them
  // goes to one FRAG_CH-chunk fragment -- used when that is fewer tile-times than the
  // standard plan (4.25 instead of 5 at 4096 positions)
  {
    const int P = A.n + 1, H = A.halo, L = adi::TCH * adi::TM, FL = adi::FRAG_CH * adi::TM;
    const bool whole = A.o0 <= 0 && A.o1 >= P && h->tile_chunks == 0;
    const bool lean = A.nint == (int)A.segs.size() && A.nint - A.nmid == 2;
    const int span = P - 2 * (L - H);
    if (h->method == ADI_MFD && whole && lean && span > 0) {
      const int k = span / (L - 2 * H), gap = span - k * (L - 2 * H);
      if (gap > 0 && gap <= FL - 2 * H && 2 + k + 0.25 < (double)A.segs.size() - 0.5) {
        std::vector<adi::Seg> mid, ends;
        for (const adi::Seg& g : A.segs)
          if (g.end != 0) ends.push_back(g);   // (the standard plan's line-start / line-end tiles)
        adi::Seg s0 = ends[0].end == 1 ? ends[0] : ends[1], s1 = ends[0].end == 1 ? ends[1] : ends[0];
        s0.out_lo = 0; s0.out_hi = L - H;               // line start: positions [0, L - H)
        s1.out_lo = s1.start + H; s1.out_hi = P;        // line end
        const int k1 = (k + 1) / 2, k2 = k - k1;
        int lo = L - H;
        for (int i = 0; i < k1; ++i, lo += L - 2 * H)
          mid.push_back({lo - H, adi::TCH, lo, lo + L - 2 * H, 0, 0});
        const int glo = lo;
        int hi = s1.out_lo;
        for (int i = 0; i < k2; ++i, hi -= L - 2 * H)
          mid.push_back({hi - (L - 2 * H) - H, adi::TCH, hi - (L - 2 * H), hi, 0, 0});
        const int ghi = hi;
        adi::Seg fr{(glo - H) & ~1, adi::FRAG_CH, glo, ghi, 0, 0};
        // (the line-end tile's start is even, so the gap may differ from span's remainder)
        bool ok = ghi > glo && ghi - glo <= FL - 2 * H && fr.start >= 2 && fr.start + FL >= ghi + H &&
                  fr.start + FL - 1 <= A.n - 2;
        for (const adi::Seg& g : mid) ok = ok && (g.start & 1) == 0 && g.start >= 2 && g.start + L - 1 <= A.n - 2;
        if (ok) {
          A.fsegs = mid;
          A.fnmid = (int)mid.size();
          A.fsegs.push_back(s0);
          A.fsegs.push_back(s1);
          A.fsegs.push_back(fr);
          CUDA_TRY(h, cudaMalloc(&A.d_fsegs, A.fsegs.size() * sizeof(adi::Seg)));
          H2D_SYNC(h, A.d_fsegs, A.fsegs.data(), A.fsegs.size() * sizeof(adi::Seg));
          A.fplan = true;
        }
      }
    }
  }
  return ADI_OK;
}

cudaEvent_t take_event(adi_ctx* h) {
  if (!h->pool.empty()) {
    cudaEvent_t e = h->pool.back();
    h->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
// bracket a launch with events when timing is on
struct TimeScope {
  adi_ctx* h;
  int kind;
  cudaEvent_t a = nullptr;
  // (inside an ADI_GRAPH capture the records become external event nodes of the graph,
  // recorded when the graph runs)
  static void rec(adi_ctx* h, cudaEvent_t e) {
    if (h->capturing) cudaEventRecordWithFlags(e, h->stream, cudaEventRecordExternal);
    else cudaEventRecord(e, h->stream);
  }
  TimeScope(adi_ctx* hh, int k) : h(hh), kind(k) {
    if (h->timing) { a = take_event(h); rec(h, a); }
  }
  ~TimeScope() {
    if (h->timing) {
      cudaEvent_t b = take_event(h);
      rec(h, b);
      h->recs.push_back({kind, a, b});
    }
  }
};

template <int METHOD, int MODE, bool EDGE, bool HET, bool FULL = false, bool NOEND = false>
int launch_e(adi_ctx* h, const adi::Axis& A, adi::KParams p, int seg0, int nseg) {
  auto kern = adi::adi_line_kernel<METHOD, adi::TM, adi::NW, MODE, EDGE, HET, FULL, NOEND>;
  const size_t smem = adi::line_smem_bytes<METHOD, adi::TM, adi::NW, EDGE, HET>();
  // per device: the shared-memory attribute, and the resident CTAs of this
  // instantiation (a race between threads only repeats idempotent calls)
  static int wave[kMaxDev] = {};
  const int dev = h->dev;
  if (wave[dev] == 0) {
    CUDA_TRY(h, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int nsm = 0, occ = 0;
    CUDA_TRY(h, cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CUDA_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * adi::NW, smem));
    wave[dev] = std::max(nsm * occ, 1);
  }
  if (nseg <= 0) return ADI_OK;
  p.pf_ahead = EDGE ? 0 : h->prefetch * wave[dev];
  const int nl = std::max(A.l1 - (A.l0 & ~3), 0);
  p.segs = A.d_segs + seg0;
  p.seg0 = seg0;
  p.nseg_all = (int)A.segs.size();
  dim3 grid((nl + adi::NW - 1) / adi::NW, (unsigned)nseg, h->batch);
  kern<<<grid, 32 * adi::NW, smem, h->stream>>>(p);
  CUDA_TRY(h, cudaGetLastError());
  h->launches++;
  if (!h->capturing) h->host_launches++;
  return ADI_OK;
}

// the fragment tiles of the fragment plan: 4 lines per warp, 16 per CTA (one segment)
int launch_frag(adi_ctx* h, const adi::Axis& A, adi::KParams p) {
  auto kern = adi::adi_line_kernel<adi::M_MFD, adi::TM, adi::NW, adi::KM_SWEEP, false, false, false, true, true>;
  const size_t smem = adi::line_smem_bytes<adi::M_MFD, adi::TM, adi::NW, false, false>();
  static bool set_[kMaxDev] = {};
  if (!set_[h->dev]) {
    CUDA_TRY(h, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    set_[h->dev] = true;
  }
  // TMA copies of FRAG_CH chunks (each fragment line's leader lane loads its line)
  int rc;
  if ((rc = tmap_for(h, p.S_in, &p.tmS, adi::FRAG_CH))) return rc;
  if ((rc = tmap_for(h, p.X_in, &p.tmX, adi::FRAG_CH))) return rc;
  if (p.phi_src && (rc = tmap_for(h, p.phi_src, &p.tmF, adi::FRAG_CH))) return rc;
  const int nl = std::max(A.l1 - (A.l0 & ~3), 0);
  const int lpc = adi::NW * (32 / adi::FRAG_CH);   // lines per CTA
  p.segs = A.d_fsegs + (A.fsegs.size() - 1);
  p.seg0 = 0;
  p.nseg_all = 1;
  p.pf_ahead = 0;
  dim3 grid((nl + lpc - 1) / lpc, 1, h->batch);
  kern<<<grid, 32 * adi::NW, smem, h->stream>>>(p);
  CUDA_TRY(h, cudaGetLastError());
  h->launches++;
  if (!h->capturing) h->host_launches++;
  return ADI_OK;
}

// interior segments first (lean kernel), then the segments with line ends
#ifndef ADI_SPLIT_END
#define ADI_SPLIT_END 1
#endif
// phase 0: every segment; phase 1: the first nfree (no halo read); phase 2: the others
template <int METHOD, int MODE, bool HET = false, bool FULL = false>
int launch_t(adi_ctx* h, const adi::Axis& A, const adi::KParams& p) {
  if (A.l1 <= A.l0) return ADI_OK;
  const int phase = (&A == &h->ay) ? h->cols_phase : 0;   // adi_step_cols of a band (overlap)
  const int nseg = (int)A.segs.size();
  int rc;
  if (METHOD == adi::M_MFD && MODE == adi::KM_SWEEP && !HET && !FULL && A.fplan && h->frag_on && phase == 0 &&
      !p.carry && !p.trace) {   // (ADI_ASYNC_STORE: the tiles' stores; PACK stores by threads)
    // the fragment plan: interior tiles, the two line-end tiles, then
    // the middle fragments packed 4 lines per warp
    adi::Axis F;
    F.l0 = A.l0; F.l1 = A.l1;
    F.segs = std::vector<adi::Seg>(A.fsegs.begin(), A.fsegs.end() - 1);
    F.d_segs = A.d_fsegs;
    rc = launch_e<METHOD, MODE, false, HET, FULL, true>(h, F, p, 0, A.fnmid);
    if (!rc) rc = launch_e<METHOD, MODE, false, HET, FULL, false>(h, F, p, A.fnmid, 2);
    if (!rc) rc = launch_frag(h, A, p);
    return rc;
  }
  if (phase == 1) return launch_e<METHOD, MODE, false, HET, FULL, true>(h, A, p, 0, A.nfree);
  const int s0 = (phase == 2) ? A.nfree : 0;
  if (ADI_SPLIT_END) {
    // interior segments without the line-end code, then the lean line-end segments
    rc = launch_e<METHOD, MODE, false, HET, FULL, true>(h, A, p, s0, A.nmid - s0);
    if (!rc) rc = launch_e<METHOD, MODE, false, HET, FULL, false>(h, A, p, A.nmid, A.nint - A.nmid);
  } else {
    rc = (phase == 2) ? launch_e<METHOD, MODE, false, HET, FULL, true>(h, A, p, s0, A.nmid - s0) : ADI_OK;
    if (!rc) rc = launch_e<METHOD, MODE, false, HET, FULL, false>(h, A, p, phase == 2 ? A.nmid : 0,
                                                               A.nint - (phase == 2 ? A.nmid : 0));
  }
  if (rc) return rc;
  return launch_e<METHOD, MODE, true, HET, FULL, false>(h, A, p, A.nint, nseg - A.nint);
}

// the full-matrix CFD variant (NEXT row f4)
template <int MODE>
int launch_full(adi_ctx* h, const adi::Axis& A, const adi::KParams& p) {
  return launch_t<adi::M_CFD, MODE, false, true>(h, A, p);
}

// heterogeneous-media kernels (fixed K sweeps: the stopping rule is not combined with media)
template <int METHOD>
int launch_het(adi_ctx* h, int mode, const adi::Axis& A, const adi::KParams& p) {
  if (mode == adi::KM_SWEEP) return launch_t<METHOD, adi::KM_SWEEP, true>(h, A, p);
  if (mode == adi::KM_FINAL) return launch_t<METHOD, adi::KM_FINAL, true>(h, A, p);
  if (mode == adi::KM_PROLOGUE) return launch_t<METHOD, adi::KM_PROLOGUE, true>(h, A, p);
  return fail(h, ADI_EINVAL, "internal: no media kernel for this mode");
}

// ---- thread-per-line kernels for short lines (adi_thread.cuh) ----------
#ifndef ADI_THREAD_AUTO_MAX
#define ADI_THREAD_AUTO_MAX 64    // cells per line up to which the auto mode uses them (measured: faster at 40, slower at 80)
#endif
#ifndef ADI_WARP_AUTO_MAX
#define ADI_WARP_AUTO_MAX 382     // cells per line up to which the auto mode uses the warp kernels (§5.9)
#endif
// warp-per-line kernels (adi_warp.cuh): lines of at most 384 stored positions
bool warp_fits(const adi_ctx* h) {
  return h->warp_lines && adi::warp_npl(std::max(h->ax.n, h->ay.n)) > 0;
}
// the short-line kernels (warp- or thread-per-line) run this handle's sweeps
bool thread_mode(const adi_ctx* h) {
  if (h->small == 0 || h->het || h->full || h->eps > 0.0 || h->tile_chunks > 0) return false;
  if (h->band_y0 > 0 || h->band_y1 < h->ay.n + 1 || (h->dist && h->nranks > 1)) return false;
  const int nmax = std::max(h->ax.n, h->ay.n);
  if (h->small < 0) return warp_fits(h) ? nmax <= ADI_WARP_AUTO_MAX : nmax <= ADI_THREAD_AUTO_MAX;
  return warp_fits(h) || adi::thread_smem(nmax, 32) <= 200 * 1024;
}

template <int METHOD, int MODE>
int launch_thread(adi_ctx* h, const adi::Axis& A, const adi::KParams& p) {
  auto kern = adi::adi_thread_kernel<METHOD, MODE>;
  const int T = adi::thread_tpb(A.n);
  const size_t smem = adi::thread_smem(A.n, T);
  static size_t set_for[kMaxDev] = {};
  if (set_for[h->dev] < smem) {
    CUDA_TRY(h, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    set_for[h->dev] = 200 * 1024;
  }
  const int nl = std::max(A.l1 - p.line0, 0);
  if (nl <= 0) return ADI_OK;
  dim3 grid((nl + T - 1) / T, 1, h->batch);
  kern<<<grid, T, smem, h->stream>>>(p);
  CUDA_TRY(h, cudaGetLastError());
  h->launches++;
  if (!h->capturing) h->host_launches++;
  return ADI_OK;
}

template <int METHOD, int MODE, int NPL>
int launch_warp_n(adi_ctx* h, const adi::Axis& A, const adi::KParams& p) {
  auto kern = adi::adi_warp_kernel<METHOD, MODE, NPL>;
  const int nl = std::max(A.l1 - p.line0, 0);
  if (nl <= 0) return ADI_OK;
  dim3 grid((nl + adi::WK_WARPS - 1) / adi::WK_WARPS, 1, h->batch);
  kern<<<grid, 32 * adi::WK_WARPS, adi::warp_smem_bytes<NPL>(), h->stream>>>(p);
  CUDA_TRY(h, cudaGetLastError());
  h->launches++;
  if (!h->capturing) h->host_launches++;
  return ADI_OK;
}
// positions per lane from the handle's longer line (both sweeps use one instantiation)
template <int METHOD, int MODE>
int launch_warp(adi_ctx* h, const adi::Axis& A, const adi::KParams& p) {
  switch (adi::warp_npl(std::max(h->ax.n, h->ay.n))) {
    case 2: return launch_warp_n<METHOD, MODE, 2>(h, A, p);
    case 4: return launch_warp_n<METHOD, MODE, 4>(h, A, p);
    case 6: return launch_warp_n<METHOD, MODE, 6>(h, A, p);
    case 8: return launch_warp_n<METHOD, MODE, 8>(h, A, p);
    case 10: return launch_warp_n<METHOD, MODE, 10>(h, A, p);
    case 12: return launch_warp_n<METHOD, MODE, 12>(h, A, p);
    default: return fail(h, ADI_EINVAL, "internal: line too long for the warp kernels");
  }
}

// the fused transpose is in use for this call's kernels (the stopping rule's attempts keep
// the all-to-all: their stores are provisional)
bool tm_fused_now(const adi_ctx* h) { return h->tmode && h->tfused && h->eps <= 0.0; }

int launch(adi_ctx* h, int mode, const adi::Axis& A, const adi::KParams& p0, int kind) {
  TimeScope ts(h, kind);
  if (thread_mode(h) && (mode == adi::KM_SWEEP || mode == adi::KM_FINAL || mode == adi::KM_PROLOGUE) &&
      !p0.carry) {
    adi::KParams p = p0;
    const bool cfd = h->method == ADI_CFD;
    if (warp_fits(h)) {
      if (mode == adi::KM_SWEEP) return cfd ? launch_warp<adi::M_CFD, adi::KM_SWEEP>(h, A, p)
                                            : launch_warp<adi::M_MFD, adi::KM_SWEEP>(h, A, p);
      if (mode == adi::KM_FINAL) return cfd ? launch_warp<adi::M_CFD, adi::KM_FINAL>(h, A, p)
                                            : launch_warp<adi::M_MFD, adi::KM_FINAL>(h, A, p);
      return cfd ? launch_warp<adi::M_CFD, adi::KM_PROLOGUE>(h, A, p)
                 : launch_warp<adi::M_MFD, adi::KM_PROLOGUE>(h, A, p);
    }
    if (mode == adi::KM_SWEEP) return cfd ? launch_thread<adi::M_CFD, adi::KM_SWEEP>(h, A, p)
                                          : launch_thread<adi::M_MFD, adi::KM_SWEEP>(h, A, p);
    if (mode == adi::KM_FINAL) return cfd ? launch_thread<adi::M_CFD, adi::KM_FINAL>(h, A, p)
                                          : launch_thread<adi::M_MFD, adi::KM_FINAL>(h, A, p);
    return cfd ? launch_thread<adi::M_CFD, adi::KM_PROLOGUE>(h, A, p)
               : launch_thread<adi::M_MFD, adi::KM_PROLOGUE>(h, A, p);
  }
  adi::KParams p = p0;
  p.trace = (kind == h->trace_kind) ? h->trace : nullptr;
  p.trace_cap = h->trace_cap;
  int rc;
  if (p.S_in && (rc = tmap_for(h, p.S_in, &p.tmS))) return rc;
  if ((rc = tmap_for(h, p.X_in, &p.tmX))) return rc;
  if (tm_fused_now(h) && (mode == adi::KM_SWEEP || mode == adi::KM_PROLOGUE) && (p.S_out == h->Sb || p.S_out == h->Sd)) {
    // fused transpose: the row kernel's S2^T (positions x) lands in the owners' Sc, the
    // column / prologue kernel's S1'^T (positions y) in the owners' Sa
    const bool rows = (p.S_out == h->Sb);
    const std::vector<int>& cut = rows ? h->cut_x : h->cut_y;
    p.tnp = h->nranks;
    for (int q = 0; q < h->nranks; ++q) {
      const adi_ctx::TPeer& t = h->tpeer[q];
      p.tcut[q] = cut[q];
      p.tso[q] = rows ? t.Sc : t.Sa;
      p.tpt[q] = rows ? t.pc : t.pa;
      p.tsb[q] = rows ? t.aC : t.aS;
    }
    p.tcut[h->nranks] = 1 << 30;
  } else if (mode == adi::KM_SWEEP && p.S_out && !h->het && !h->full && !p.carry && h->async_store) {
    if ((rc = tmap_store_for(h, p.S_out, &p.tmSo, &p.so_line0, &p.so_pos0))) return rc;
    p.tma_so = 1;
  }
  if (p.phi_src && (rc = tmap_for(h, p.phi_src, &p.tmF))) return rc;
  if (h->het) {
    if ((rc = tmap_for(h, (&A == &h->ay) ? h->Cb : h->Ca, &p.tmC))) return rc;
    return h->method == ADI_CFD ? launch_het<adi::M_CFD>(h, mode, A, p) : launch_het<adi::M_MFD>(h, mode, A, p);
  }
  if (h->full) {
    if (mode == adi::KM_SWEEP) return launch_full<adi::KM_SWEEP>(h, A, p);
    if (mode == adi::KM_FINAL) return launch_full<adi::KM_FINAL>(h, A, p);
    if (mode == adi::KM_PROLOGUE) return launch_full<adi::KM_PROLOGUE>(h, A, p);
    return fail(h, ADI_EINVAL, "internal: no full-variant kernel for this mode");
  }
  if (h->method == ADI_CFD) {
    if (mode == adi::KM_SWEEP) return launch_t<adi::M_CFD, adi::KM_SWEEP>(h, A, p);
    if (mode == adi::KM_FINAL) return launch_t<adi::M_CFD, adi::KM_FINAL>(h, A, p);
    if (mode == adi::KM_SWEEP_T) return launch_t<adi::M_CFD, adi::KM_SWEEP_T>(h, A, p);
    if (mode == adi::KM_FINAL_T) return launch_t<adi::M_CFD, adi::KM_FINAL_T>(h, A, p);
    return launch_t<adi::M_CFD, adi::KM_PROLOGUE>(h, A, p);
  }
  if (mode == adi::KM_SWEEP) return launch_t<adi::M_MFD, adi::KM_SWEEP>(h, A, p);
  if (mode == adi::KM_FINAL) return launch_t<adi::M_MFD, adi::KM_FINAL>(h, A, p);
  if (mode == adi::KM_SWEEP_T) return launch_t<adi::M_MFD, adi::KM_SWEEP_T>(h, A, p);
  if (mode == adi::KM_FINAL_T) return launch_t<adi::M_MFD, adi::KM_FINAL_T>(h, A, p);
  return launch_t<adi::M_MFD, adi::KM_PROLOGUE>(h, A, p);
}

// batched out[c][r] = in[r][c] for an R x C matrix (row pitches ip, op; 32x32 shared tiles)
__global__ void transpose_kernel(const double* __restrict__ in, double* __restrict__ out, int R, int C,
                                 long long ip, long long op, long long ibs, long long obs) {
  __shared__ double tile[32][33];
  const double* ib = in + blockIdx.z * ibs;
  double* ob = out + blockIdx.z * obs;
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int r = r0 + k, cc = c0 + threadIdx.x;
    if (r < R && cc < C) tile[k][threadIdx.x] = ib[(long long)r * ip + cc];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int cc = c0 + k, r = r0 + threadIdx.x;
    if (r < R && cc < C) ob[(long long)cc * op + r] = tile[threadIdx.x][k];
  }
}

int transpose(adi_ctx* h, const double* in, double* out, int R, int C, long long ip, long long op,
              int batch, long long ibs, long long obs) {
  dim3 grid((C + 31) / 32, (R + 31) / 32, batch);
  transpose_kernel<<<grid, dim3(32, 8), 0, h->stream>>>(in, out, R, C, ip, op, ibs, obs);
  CUDA_TRY(h, cudaGetLastError());
  return ADI_OK;
}

// Dirichlet columns (x = 0, x = 1) of U at time factor gb, all rows (corners included)
__global__ void edge_cols_kernel(double* U, int r0, int r1, int nxu, int pu, long long ubatch,
                                 const double* ex0, const double* ex1, double gb, int lo, int hi) {
  const int r = r0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= r1) return;
  double* Ub = U + blockIdx.y * ubatch + (long long)r * pu;
  if (lo) Ub[0] = ex0 ? ex0[r] * gb : 0.0;
  if (hi) Ub[nxu - 1] = ex1 ? ex1[r] * gb : 0.0;
}
double tabv(const std::vector<double>& g, long long j) { return g.empty() ? 1.0 : g[(size_t)j]; }

adi::KParams base_params(adi_ctx* h, const adi::Axis& A, bool ydir) {
  adi::KParams p;
  std::memset(&p, 0, sizeof p);
  p.n = A.n;
  p.line0 = A.l0 & ~3;     // CTA line groups are 4-aligned (32-byte transposed writes)
  p.line_lo = A.l0;
  p.nlines = A.l1;
  p.plo = A.plo;
  p.phi = A.phi;
  p.segs = A.d_segs;
  if (!ydir) {  // lines = interior rows y; S_in = Sa, S_out = Sb (= S^T)
    p.s_line = h->pa; p.so_line = 1; p.so_pt = h->pb;
    p.x_line = h->pv;
    p.u_line = h->pu; p.u_pt = 1;
    p.edgeL = h->edges ? h->edges + 2 * h->nxu : nullptr;
    p.edgeR = h->edges ? h->edges + 2 * h->nxu + h->nyu : nullptr;
    p.phi_src = h->phi;
  } else {      // lines = interior columns x; S_in = Sb, S_out = Sa; X = W̄^T
    p.s_line = h->pb; p.so_line = 1; p.so_pt = h->pa;
    p.x_line = h->pw;
    p.u_line = 1; p.u_pt = h->pu;
    p.edgeL = h->edges ? h->edges : nullptr;
    p.edgeR = h->edges ? h->edges + h->nxu : nullptr;
    p.phi_src = h->phiT;
  }
  p.s_batch = (long long)h->aS;
  p.x_batch = (long long)(ydir ? h->aW : h->aV);
  p.u_batch = (long long)h->aU;
  if (h->tmode && ydir) {   // column side of the transpose decomposition (adi_ctx::tmode)
    p.s_line = h->pc; p.so_pt = h->pd;
    p.x_line = h->pc;
    p.u_line = 1; p.u_pt = h->pd;
    p.s_batch = (long long)h->aC;
  }
  p.pt_line = h->has_pt ? A.d_ptl : nullptr;
  p.pt_pos = h->has_pt ? A.d_ptp : nullptr;
  p.pt_amp = 1.0 / (h->h * h->h);
  // with media the kernels' scalars are those of a unit medium (kappa = rho = 1); the
  // per-point kappa_i, rho^-1_i multiply them in the HET second pass
  const double kappa = h->het ? 1.0 : h->rho * h->c * h->c;
  const double rho = h->het ? 1.0 : h->rho;
  const double alpha = kappa * h->dt / 2.0, beta = h->dt / (2.0 * rho);
  const double f = (h->method == ADI_CFD) ? 3.0 : 1.0;
  p.cu = f * alpha / h->h;
  p.cx = f * beta / h->h;
  p.mA = p.cu * (1.0 / 24.0);
  p.mB = p.cu * (9.0 / 8.0);
  p.mC = p.cx * (1.0 / 24.0);
  p.mD = p.cx * (9.0 / 8.0);
  p.half_dt = h->dt / 2.0;
  p.taper = h->d_taper;
  p.nb = h->full ? h->absorb_nb : 0;
  p.damp = (h->full && h->absorb_nb > 0) ? (ydir ? 2 : 1) : 0;
  p.K = h->K;
  p.tabU = A.d_tabU;
  p.tabX = A.d_tabX;
  p.flag = h->check_finite ? h->flag : nullptr;
  // band-local arrays: the row sweep's lines and the column sweep's positions start at ya
  p.tline0 = ydir ? 0 : h->ya;
  p.tpos0 = ydir ? h->ya : 0;
  p.pos_lo = ydir ? h->ya : -(1 << 30);
  p.pos_hi = ydir ? h->yb : (1 << 30);
  if (h->tmode && ydir) {   // column-side arrays: the lines (rows) x start at xa, all y
    p.tline0 = h->xa;
    p.tpos0 = 0;
    p.pos_lo = 0;
    p.pos_hi = h->nyu;
  }
  return p;
}

// Inner stopping rule for one stage (Alg. 3/4), decided on the device:
// attempts with k = kmin..K sweeps are enqueued; each is the stage's own kernel
// (outputs stored) that also sums its last sweep's squared changes, followed by a
// one-thread decision.  Once a test passes the gate closes and the later attempts
// exit at once, so the outputs are those of the chosen k (the stage's inputs are
// never overwritten).
int stage_with_rule(adi_ctx* h, int mode_t, const adi::Axis& A, adi::KParams p, int kind, int which) {
  const int K = h->call_K;   // d_norms was sized by adi_step_begin for this K
  double* norms = h->d_norms + (size_t)which * 2 * (K + 1);
  CUDA_TRY(h, cudaMemsetAsync(norms, 0, sizeof(double) * 2 * (K + 1), h->stream));
  CUDA_TRY(h, cudaMemsetAsync(h->d_k + 2 + which, 0, sizeof(int), h->stream));
  p.Kdev = nullptr;
  p.gate = h->d_k + 2 + which;
  for (int k = h->kmin; k <= K; ++k) {
    adi::KParams q = p;
    q.K = k;
    q.norms = norms + 2 * k;
    int rc = launch(h, mode_t, A, q, kind);
    if (rc) return rc;
    adi::decide_sweeps_kernel<<<1, 1, 0, h->stream>>>(norms + 2 * k, h->eps, k, K,
                                                        h->d_k + 2 + which, h->d_k + which);
    CUDA_TRY(h, cudaGetLastError());
    h->launches++;
    h->host_launches++;
  }
  return ADI_OK;
}

void free_ctx(adi_ctx* h) {
  for (auto& k : h->hbuf)
    for (auto& sd : k)
      for (double*& b : sd)
        if (b) { cudaFree(b); b = nullptr; }
  if (h->comm && g_nccl.ok) g_nccl.commDestroy(h->comm);
  h->comm = nullptr;
  if (h->group) delete[] h->group;
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->gstream) cudaStreamDestroy(h->gstream);
  if (h->ev_pack) cudaEventDestroy(h->ev_pack);
  if (h->ev_recv) cudaEventDestroy(h->ev_recv);
  if (h->cs) cudaStreamDestroy(h->cs);
  for (adi_ctx* q : h->peer)
    if (q)
      for (adi_ctx*& back : q->peer)
        if (back == h) back = nullptr;
  for (auto& r : h->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : h->pool) cudaEventDestroy(e);
  if (h->tmode) {
    auto cr = [&](double* q) { return q ? q + (ptrdiff_t)h->xa * h->pc : nullptr; };
    for (double* q : {h->Ubase ? h->Ubase + h->xa : nullptr, rows_raw(h, h->V, h->pv), rows_raw(h, h->V2, h->pv),
                      rows_raw(h, h->Sa, h->pa), rows_raw(h, h->phi, h->pa), cr(h->W), cr(h->W2), cr(h->Sc),
                      cr(h->phiT), cols_raw(h, h->Sb), h->Sd ? h->Sd + h->xa : nullptr})
      dfree(q);
    for (double* q : h->tsend) if (q) cudaFree(q);
    for (double* q : h->trecv) if (q) cudaFree(q);
    for (void* q : h->ipc_open) cudaIpcCloseMemHandle(q);
    if (h->dbar) cudaFree(h->dbar);
  } else {
    for (double* q : {rows_raw(h, h->Ubase, h->pu), rows_raw(h, h->V, h->pv), rows_raw(h, h->V2, h->pv),
                      rows_raw(h, h->Sa, h->pa), rows_raw(h, h->phi, h->pa), rows_raw(h, h->Ca, h->pa),
                      cols_raw(h, h->W), cols_raw(h, h->W2), cols_raw(h, h->W3), cols_raw(h, h->Sb),
                      cols_raw(h, h->phiT), cols_raw(h, h->Cb)})
      dfree(q);
  }
  for (void* q : {(void*)h->edges, (void*)h->flag, (void*)h->d_norms, (void*)h->d_k, (void*)h->d_taper})
    if (q) cudaFree(q);
  for (adi::Axis* A : {&h->ax, &h->ay})
    for (void* q : {(void*)A->d_segs, (void*)A->d_fsegs, (void*)A->d_tabU, (void*)A->d_tabX, (void*)A->d_ptl,
                    (void*)A->d_ptp})
      if (q) cudaFree(q);
}

// band cuts of y positions [0, npos) over nranks (as dist.band_partition, align 4): interior
// cuts b with (b - 1) % 4 == 0, so each band's row sweep starts on a 4-line group
void dist_bands(int npos, int nranks, int* cuts) {
  cuts[0] = 0;
  for (int k = 1; k < nranks; ++k) {
    const double b = (double)k * npos / nranks;
    const int q = std::max(1, (int)std::nearbyint((b - 1.0) / 4.0));   // ties to even, as Python round
    cuts[k] = 1 + 4 * q;
  }
  cuts[nranks] = npos;
}

// ---- heterogeneous media (NEXT row f3) ------------------------------------------
// Ca[y][x] = (kappa(y, x) at u positions x = 1..nxi, rho^-1 of V̄ row y-1 at x = 0..nxv-1)
__global__ void pack_media_rows(float2* Ca, int pa, int y_lo, int y_hi, int nxi, int nxu, int nxv, const float* kap,
                                const float* rv) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = y_lo + blockIdx.y;
  if (x >= pa || y > y_hi) return;
  float2 e;
  e.x = (x >= 1 && x <= nxi) ? kap[(size_t)y * nxu + x] : 0.f;
  e.y = (x < nxv) ? rv[(size_t)(y - 1) * nxv + x] : 0.f;
  Ca[(size_t)y * pa + x] = e;
}
// Cb[x][y] = (kappa(y, x) at u positions y = 1..nyi, rho^-1 of W̄ (row y, column x-1) at y = 0..nyv-1)
__global__ void pack_media_cols(float2* Cb, int pb, int y_lo, int nxi, int nyi, int nyv, int nxu, const float* kap,
                                const float* rw) {
  const int y = y_lo + blockIdx.x * blockDim.x + threadIdx.x, x = blockIdx.y + 1;
  if (y >= y_lo + pb || x > nxi) return;
  float2 e;
  e.x = (y >= 1 && y <= nyi) ? kap[(size_t)y * nxu + x] : 0.f;
  e.y = (y < nyv) ? rw[(size_t)y * nxi + (x - 1)] : 0.f;
  Cb[(size_t)x * pb + y] = e;
}

}  // namespace

extern "C" {

const char* adi_version(void) { return kVersion; }

}  // extern "C"

// The y extent of a band's arrays: its positions [y0, y1) plus `halo` on each side
// (field_rows with the halo; even start).  A whole grid: [0, nyu).
static void band_extent(const adi_ctx* h, int y0, int y1, int halo, int* ya, int* yb) {
  const int npos = h->ay.n + 1;
  if (y0 <= 0 && y1 >= npos) { *ya = 0; *yb = h->nyu; return; }
  // (32 positions of margin below the halo: a band tile holding the halo may start up
  // to one chunk below it, and its TMA coordinates stay non-negative)
  *ya = std::max(y0 - halo - 32, 0) & ~1;
  *yb = (y1 >= npos) ? h->nyu : std::min(y1 + halo, h->nyu);
}

// create a handle whose arrays hold the band [y0, y1) of y positions (plus halo) only,
// or the whole grid (y0 = 0, y1 >= number of positions)
static int create_impl(int nx, int ny, double hh, double dt, double c, int method, int batch, int y0, int y1,
                       adi_handle* out) {
  if (!out) return ADI_EINVAL;
  *out = nullptr;
  if (method != ADI_CFD && method != ADI_MFD && method != ADI_CFD_FULL) return ADI_EINVAL;
  if (nx < 9 || ny < 9 || batch < 1) return ADI_EINVAL;
  if (!(hh > 0) || !(dt > 0) || !(c > 0) || !std::isfinite(hh) || !std::isfinite(dt) ||
      !std::isfinite(c))
    return ADI_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return ADI_ECUDA;
  }
  adi_ctx* h = new adi_ctx();
  if (cudaGetDevice(&h->dev) != cudaSuccess) {
    cudaGetLastError();
    delete h;
    return ADI_ECUDA;
  }
  h->full = (method == ADI_CFD_FULL);
  h->off = h->full ? 0 : 1;
  if (h->full) method = ADI_CFD;   // the CFD operators; every node unknown
  h->method = method; h->nx = nx; h->ny = ny; h->batch = batch;
  h->h = hh; h->dt = dt; h->c = c; h->rho = 1.0;
  if (method == ADI_CFD) {
    h->nxu = nx; h->nyu = ny; h->nxi = nx - 2; h->nyi = ny - 2;
  } else {
    h->nxu = nx + 1; h->nyu = ny + 1; h->nxi = nx - 1; h->nyi = ny - 1;
  }
  if (h->full) { h->nxi = nx; h->nyi = ny; }   // U, V, W, F: all ny x nx
  h->nxv = nx; h->nyv = ny;
  h->nU = (size_t)h->nyu * h->nxu;
  h->nV = (size_t)h->nyi * h->nxv;
  h->nW = (size_t)h->nyv * h->nxi;
  h->nS = (size_t)h->nyi * h->nxi;
  h->pu = padp(h->nxu);
  h->pa = padp(h->nxu);
  h->pv = padp(h->nxu);
  h->ay.n = ny - 1;   // (setup_axis sets it again) band_extent needs the position count
  {
    int ya, yb;
    band_extent(h, y0, y1, adi::plan_halo(method), &ya, &yb);
    set_extent(h, ya, yb);
  }
  int rc = init_constants(h);
  auto bail = [&](int code) {
    free_ctx(h);
    delete h;
    return code;
  };
  if (rc) return bail(rc);
  const size_t B = (size_t)batch;
  {
    double *U = halloc(h, B * h->aU), *V = halloc(h, B * h->aV), *V2 = halloc(h, B * h->aV);
    double *W = halloc(h, B * h->aW), *W2 = halloc(h, B * h->aW);
    double *Sa = halloc(h, B * h->aS), *Sb = halloc(h, B * h->aS);
    h->Ubase = rows_in(h, U, h->pu);
    h->V = rows_in(h, V, h->pv);
    h->V2 = rows_in(h, V2, h->pv);
    h->Sa = rows_in(h, Sa, h->pa);
    h->W = cols_in(h, W);
    h->W2 = cols_in(h, W2);
    h->Sb = cols_in(h, Sb);
    if (!U || !V || !V2 || !W || !W2 || !Sa || !Sb || cudaMalloc(&h->flag, sizeof(int))) {
      cudaGetLastError();
      return bail(ADI_ENOMEM);
    }
  }
  h->U = h->Ubase;
  cudaMemset(h->flag, 0, sizeof(int));
  if ((rc = setup_axis(h, h->ax, nx - 1, h->nyi, 1))) return bail(rc);
  if ((rc = setup_axis(h, h->ay, ny - 1, h->nxi, 4))) return bail(rc);
  if (cudaDeviceSynchronize() != cudaSuccess) return bail(ADI_ECUDA);
  h->fields_set = true;  // zero fields are a valid state
  if (y0 > 0 || y1 < h->ay.n + 1) {
    // the band's lines and output positions (adi_set_band on arrays already band-local)
    const int ny_pos = h->ay.n + 1;
    if (y0 < 0 || y1 > ny_pos || y0 >= y1) return bail(ADI_EINVAL);
    const int hl = h->ay.halo;
    if ((y0 > 0 && y1 - y0 < hl) || (y1 < ny_pos && y1 - y0 < hl)) return bail(ADI_EINVAL);
    h->band_y0 = y0;
    h->band_y1 = y1;
    h->ax.l0 = std::max(y0, 1);
    h->ax.l1 = std::min(y1, h->nyi + 1);
    h->ay.o0 = y0;
    h->ay.o1 = y1;
    if ((rc = setup_axis(h, h->ay, ny - 1, h->nxi, 4))) return bail(rc);
  }
  *out = h;
  const double cfl = c * dt / hh;
  const double lim = (method == ADI_MFD) ? 2.0 / std::sqrt(6.0) : 2.0 / std::sqrt(3.0);
  if (cfl > lim) {
    h->err = "c*dt/h above the inner-iteration limit";
    return ADI_WUNSTABLE;
  }
  return ADI_OK;
}

extern "C" {

int adi_create_batch(int nx, int ny, double hh, double dt, double c, int method, int batch,
                     adi_handle* out) {
  return create_impl(nx, ny, hh, dt, c, method, batch, 0, 1 << 30, out);
}

int adi_create(int nx, int ny, double hh, double dt, double c, int method, adi_handle* out) {
  return adi_create_batch(nx, ny, hh, dt, c, method, 1, out);
}

int adi_set_param(adi_handle h, int key, double v) {
  DevGuard dg_(h);
  if (!h) return ADI_EINVAL;
  h->err.clear();
  // keys that size or plan work already enqueued by adi_step_begin (the stopping rule's
  // norm buffer, the tile plan, the carry buffer) cannot change inside a call
  if (h->in_call && (key == ADI_K_SWEEPS || key == ADI_EPS || key == ADI_K_MIN || key == ADI_TILE_CHUNKS ||
                     key == ADI_CARRY || key == ADI_RHO || key == ADI_THREAD_LINES || key == ADI_DIST_FUSED ||
                     key == ADI_STEP_INDEX))
    return fail(h, ADI_ESTATE, "call in progress");
  if (key == ADI_K_SWEEPS) {
    if (!(v >= 1) || v != std::floor(v) || v > 1000) return fail(h, ADI_EINVAL, "K must be an integer >= 1");
    h->K = (int)v;
  } else if (key == ADI_RHO) {
    if (!(v > 0) || !std::isfinite(v)) return fail(h, ADI_EINVAL, "rho must be > 0");
    h->rho = v;
    h->carry_valid = false;   // alpha, beta of the carried a2 change
  } else if (key == ADI_CHECK_FINITE) {
    h->check_finite = (v != 0);
  } else if (key == ADI_TIMING) {
    h->timing = (v != 0);
  } else if (key == ADI_EPS) {
    if (!(v >= 0) || !std::isfinite(v)) return fail(h, ADI_EINVAL, "eps must be finite and >= 0");
    h->eps = v;
  } else if (key == ADI_K_MIN) {
    if (!(v >= 2) || v != std::floor(v) || v > 1000) return fail(h, ADI_EINVAL, "k_min must be an integer >= 2");
    h->kmin = (int)v;
  } else if (key == ADI_ABSORB_WIDTH || key == ADI_ABSORB_RATE) {
    if (!h->full) return fail(h, ADI_EINVAL, "the absorbing layer belongs to the full-matrix variant");
    if (h->in_call) return fail(h, ADI_ESTATE, "call in progress");
    int nb = h->absorb_nb;
    double a = h->absorb_a;
    if (key == ADI_ABSORB_WIDTH) {
      if (!(v >= 0) || v != std::floor(v) || 2 * v > std::min(h->nx, h->ny))
        return fail(h, ADI_EINVAL, "absorbing width must be an integer in [0, min(nx, ny)/2]");
      nb = (int)v;
    } else {
      if (!(v > 0) || !std::isfinite(v)) return fail(h, ADI_EINVAL, "absorbing rate must be > 0");
      a = v;
    }
    // Cerjan taper G(d) = exp(-(a (nb - d))^2), d = distance (points) from the nearest edge
    std::vector<double> g((size_t)std::max(nb, 1));
    for (int d = 0; d < nb; ++d) g[d] = std::exp(-(a * (nb - d)) * (a * (nb - d)));
    if (h->d_taper) { cudaFree(h->d_taper); h->d_taper = nullptr; }
    CUDA_TRY(h, cudaMalloc(&h->d_taper, g.size() * sizeof(double)));
    H2D_SYNC(h, h->d_taper, g.data(), g.size() * sizeof(double));
    h->absorb_nb = nb;
    h->absorb_a = a;
  } else if (key == ADI_CARRY) {
    if (v != 0.0 && v != 1.0) return fail(h, ADI_EINVAL, "carry must be 0 or 1");
    h->carry_on = (int)v;
    if (!h->carry_on) h->carry_valid = false;
  } else if (key == ADI_THREAD_LINES) {
    if (v != 0.0 && v != 1.0 && v != -1.0) return fail(h, ADI_EINVAL, "thread lines must be -1, 0 or 1");
    h->small = (int)v;
    h->carry_valid = false;
  } else if (key == ADI_DIST_FUSED) {
    if (v != 0.0 && v != 1.0) return fail(h, ADI_EINVAL, "dist fused must be 0 or 1");
    if (v == 1.0 && (!h->tmode || (int)h->tpeer.size() != h->nranks))
      return fail(h, ADI_EINVAL, "no fused transpose on this handle (transpose mode, <= 8 ranks, peer mappings)");
    h->tfused = (v == 1.0);
  } else if (key == ADI_STEP_INDEX) {
    if (!(v >= 0) || v != std::floor(v) || v > 1e15) return fail(h, ADI_EINVAL, "step index must be an integer >= 0");
    h->m = (long long)v;
    h->carry_valid = false;   // the carried explicit half belongs to the old time level
  } else if (key == ADI_WARP_LINES) {
    if (v != 0.0 && v != 1.0) return fail(h, ADI_EINVAL, "warp lines must be 0 or 1");
    h->warp_lines = (int)v;
  } else if (key == ADI_FRAG_TILES) {
    if (v != 0.0 && v != 1.0) return fail(h, ADI_EINVAL, "fragment tiles must be 0 or 1");
    h->frag_on = (int)v;
  } else if (key == ADI_ASYNC_STORE) {
    if (v != 0.0 && v != 1.0) return fail(h, ADI_EINVAL, "async store must be 0 or 1");
    h->async_store = (int)v;
  } else if (key == ADI_GRAPH) {
    if (v != 0.0 && v != 1.0) return fail(h, ADI_EINVAL, "graph must be 0 or 1");
    h->graph_on = (int)v;
  } else if (key == ADI_PREFETCH) {
    if (!(v >= 0) || v != std::floor(v) || v > 8) return fail(h, ADI_EINVAL, "prefetch must be an integer in [0, 8]");
    h->prefetch = (int)v;
  } else if (key == ADI_TILE_CHUNKS) {
    if (!(v >= 0) || v != std::floor(v)) return fail(h, ADI_EINVAL, "tile chunks must be >= 0");
    h->tile_chunks = (int)v;
    int rc = setup_axis(h, h->ax, h->nx - 1, h->nyi, 1);
    if (!rc) rc = setup_axis(h, h->ay, h->ny - 1, h->nxi, 4);
    if (rc) return rc;
  } else {
    return fail(h, ADI_EINVAL, "unknown parameter");
  }
  return ADI_OK;
}

int adi_set_stream(adi_handle h, void* s) {
  DevGuard dg_(h);
  if (!h) return ADI_EINVAL;
  h->err.clear();
  if (h->in_call) return fail(h, ADI_ESTATE, "call in progress");
  // work already enqueued on the previous stream finishes first
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  h->stream = (cudaStream_t)s;
  return ADI_OK;
}

// Rows moved by adi_set/get_fields: all of them, or, with a band set (§7), the y
// positions this handle uses: [y0 - halo, y1 + halo) on set (the first half-step
// of a call reads the halo rows of U and W̄), [y0, y1) on get.  Rows of the U block
// beyond the last band position (MFD: position n+1) belong to the top band.
static void field_rows(adi_ctx* h, bool with_halo, int* ya, int* yb) {
  const int npos = h->ay.n + 1;
  const bool banded = h->band_y0 > 0 || h->band_y1 < npos;
  if (!banded) { *ya = 0; *yb = h->nyu; return; }
  const int hl = with_halo ? h->ay.halo : 0;
  *ya = std::max(h->band_y0 - hl, 0);
  *yb = (h->band_y1 >= npos) ? h->nyu : std::min(h->band_y1 + hl, h->nyu);
}

// ---- fields of a transpose-mode rank (adi_ctx::tmode): U and W̄ on the column side (all
// rows, the columns [xa, xb)), V̄ on the row side (the rows [ya, yb)); a get returns the
// owned rows Y_r of V̄ and the owned columns X_r of U and W̄
static int tm_fields(adi_ctx* h, double* U, double* V, double* W, cudaMemcpyKind kind, bool set) {
  const int off = h->off;
  const int x0 = set ? h->xa : h->tx0, x1 = set ? h->xb : (h->tx1 >= h->ax.n + 1 ? h->nxu : h->tx1);
  const int y0 = set ? h->ya : h->ty0, y1 = set ? h->yb : (h->ty1 >= h->ay.n + 1 ? h->nyu : h->ty1);
  const int ja = std::max(y0 - off, 0), jb = std::min(y1 - off, h->nyi);
  const int ia = std::max(x0 - off, 0), ib = std::min(x1 - off, h->nxi);
  double* scratch = h->W2 + (ptrdiff_t)h->xa * h->pc;   // W2's allocation as a dense buffer
  for (int b = 0; b < h->batch; ++b) {
    double* Ui = h->U + b * h->aU + x0;
    double* Uu = U + b * h->nU + x0;
    if (set) CUDA_TRY(h, cudaMemcpy2DAsync(Ui, h->pd * 8, Uu, h->nxu * 8, (x1 - x0) * 8, h->nyu, kind, h->stream));
    else CUDA_TRY(h, cudaMemcpy2DAsync(Uu, h->nxu * 8, Ui, h->pd * 8, (x1 - x0) * 8, h->nyu, kind, h->stream));
    if (jb > ja) {
      double* Vi = h->V + b * h->aV + (size_t)(ja + off) * h->pv;
      double* Vu = V + b * h->nV + (size_t)ja * h->nxv;
      if (set) CUDA_TRY(h, cudaMemcpy2DAsync(Vi, h->pv * 8, Vu, h->nxv * 8, h->nxv * 8, jb - ja, kind, h->stream));
      else CUDA_TRY(h, cudaMemcpy2DAsync(Vu, h->nxv * 8, Vi, h->pv * 8, h->nxv * 8, jb - ja, kind, h->stream));
    }
    if (ib > ia) {   // W̄ columns [ia, ib) (dense user rows y) <-> W̄^T rows x = i + off
      double* Wi = h->W + b * h->aW + (size_t)(ia + off) * h->pc;
      double* Wu = W + b * h->nW + ia;
      if (set) {
        CUDA_TRY(h, cudaMemcpy2DAsync(scratch, (ib - ia) * 8, Wu, h->nxi * 8, (ib - ia) * 8, h->nyv, kind, h->stream));
        int rc = transpose(h, scratch, Wi, h->nyv, ib - ia, ib - ia, h->pc, 1, 0, 0);
        if (rc) return rc;
      } else {
        int rc = transpose(h, Wi, scratch, ib - ia, h->nyv, h->pc, ib - ia, 1, 0, 0);
        if (rc) return rc;
        CUDA_TRY(h, cudaMemcpy2DAsync(Wu, h->nxi * 8, scratch, (ib - ia) * 8, (ib - ia) * 8, h->nyv, kind, h->stream));
      }
    }
  }
  return ADI_OK;
}
static int tm_set_fields(adi_ctx* h, const double* U, const double* V, const double* W, cudaMemcpyKind kind,
                         bool sync) {
  int rc = tm_fields(h, const_cast<double*>(U), const_cast<double*>(V), const_cast<double*>(W), kind, true);
  if (rc) return rc;
  if (kind == cudaMemcpyHostToDevice && sync) CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  h->fields_set = true;
  return ADI_OK;
}
static int tm_get_fields(adi_ctx* h, double* U, double* V, double* W, cudaMemcpyKind kind, bool sync) {
  int rc = tm_fields(h, U, V, W, kind, false);
  if (rc) return rc;
  if (kind == cudaMemcpyDeviceToHost && sync) CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  return ADI_OK;
}

static int set_fields_impl(adi_handle h, const double* U, const double* V, const double* W,
                           cudaMemcpyKind kind, bool sync = true) {
  DevGuard dg_(h);
  if (!h) return ADI_EINVAL;
  h->carry_valid = false;   // the next call recomputes its a2 (prologue)
  h->err.clear();
  if (!U || !V || !W) return fail(h, ADI_EINVAL, "null field pointer");
  if (h->in_call) return fail(h, ADI_ESTATE, "call in progress");
  const size_t B = (size_t)h->batch;
  if (h->tmode) return tm_set_fields(h, U, V, W, kind, sync);
  int ya, yb;
  field_rows(h, true, &ya, &yb);
  const int off = h->off;   // V̄ row j = y position j + off
  const int ja = std::max(ya - off, 0), jb = std::min(yb - off, h->nyi);
  const int wa = std::min(ya, h->nyv), wb = std::min(yb, h->nyv);      // W̄ rows are y positions
  // user layouts are dense; internal rows are pitched (batch strides aU, aV, aW)
  for (size_t b = 0; b < B; ++b) {
    CUDA_TRY(h, cudaMemcpy2DAsync(h->U + b * h->aU + (size_t)ya * h->pu, h->pu * 8,
                                  U + b * h->nU + (size_t)ya * h->nxu, h->nxu * 8, h->nxu * 8, yb - ya, kind,
                                  h->stream));
    if (jb > ja)
      CUDA_TRY(h, cudaMemcpy2DAsync(h->V + b * h->aV + (size_t)(ja + off) * h->pv, h->pv * 8,
                                    V + b * h->nV + (size_t)ja * h->nxv, h->nxv * 8, h->nxv * 8, jb - ja, kind,
                                    h->stream));
    // W̄ rows [wa, wb) (dense) -> internal W̄^T (row = x position i + 1, column = y)
    // via the W2 scratch buffer
    if (wb > wa) {
      double* scratch = cols_raw(h, h->W2);   // the allocation of W2 as a dense buffer
      CUDA_TRY(h, cudaMemcpyAsync(scratch, W + b * h->nW + (size_t)wa * h->nxi, (size_t)(wb - wa) * h->nxi * 8,
                                  kind, h->stream));
      int rc = transpose(h, scratch, h->W + b * h->aW + (size_t)off * h->pw + wa, wb - wa, h->nxi, h->nxi, h->pw,
                         1, 0, 0);
      if (rc) return rc;
    }
  }
  if (kind == cudaMemcpyHostToDevice && sync) CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  h->fields_set = true;
  h->fresh = true;   // the band and its halo rows hold the state: no call-start exchange
  return ADI_OK;
}

int adi_set_fields(adi_handle h, const double* U, const double* V, const double* W) {
  DevGuard dg_(h);
  return set_fields_impl(h, U, V, W, cudaMemcpyHostToDevice);
}
int adi_set_fields_device(adi_handle h, const double* U, const double* V, const double* W) {
  DevGuard dg_(h);
  return set_fields_impl(h, U, V, W, cudaMemcpyDeviceToDevice);
}
int adi_set_fields_async(adi_handle h, const double* U, const double* V, const double* W) {
  DevGuard dg_(h);
  return set_fields_impl(h, U, V, W, cudaMemcpyHostToDevice, false);
}

static int set_points(adi_handle h, const int* ix, const int* iy) {
  // x-direction lines are interior rows (line = iy-1, pos = ix); y-direction: line = ix-1, pos = iy
  const int B = h->batch;
  std::vector<int> xl(B), xp(B), yl(B), yp(B);
  const int uhx = (h->method == ADI_CFD && !h->full) ? h->nx - 2 : h->nx - 1;
  const int uhy = (h->method == ADI_CFD && !h->full) ? h->ny - 2 : h->ny - 1;
  for (int b = 0; b < B; ++b) {
    if (ix[b] < h->off || ix[b] > uhx || iy[b] < h->off || iy[b] > uhy)
      return fail(h, ADI_EINVAL, "point source outside the pressure interior");
    xl[b] = iy[b]; xp[b] = ix[b];   // row sweep: line = y position, pos = x position
    yl[b] = ix[b]; yp[b] = iy[b];
  }
  for (adi::Axis* A : {&h->ax, &h->ay}) {
    if (!A->d_ptl) {
      CUDA_TRY(h, cudaMalloc(&A->d_ptl, B * sizeof(int)));
      CUDA_TRY(h, cudaMalloc(&A->d_ptp, B * sizeof(int)));
    }
  }
  H2D_SYNC(h, h->ax.d_ptl, xl.data(), B * sizeof(int));
  H2D_SYNC(h, h->ax.d_ptp, xp.data(), B * sizeof(int));
  H2D_SYNC(h, h->ay.d_ptl, yl.data(), B * sizeof(int));
  H2D_SYNC(h, h->ay.d_ptp, yp.data(), B * sizeof(int));
  h->has_pt = true;
  return ADI_OK;
}

int adi_set_source(adi_handle h, const double* phi, int ix, int iy, const double* g, int ng) {
  DevGuard dg_(h);
  if (!h) return ADI_EINVAL;
  h->carry_valid = false;   // the next call recomputes its a2 (prologue)
  h->err.clear();
  if (g && ng < 1) return fail(h, ADI_EINVAL, "empty source table");
  const bool has_pt = ix >= h->off;   // (the full variant: every node, ix >= 0)
  if (has_pt && h->batch != 1) return fail(h, ADI_EINVAL, "use adi_set_point_sources for a batch");
  if (phi) {
    if (!h->phi || !h->phiT) {
      h->tmaps.clear();
    h->smaps.clear();
      // (the line kernels read the pattern directly, a whole tile of 1026 positions from a
      // segment start: a band-local phiT gets that much slack behind its last row)
      if (!h->phi) {
        double* r = halloc(h, h->aS + kSrcSlack);
        if (!r) return fail(h, ADI_ENOMEM, "source pattern");
        h->phi = rows_in(h, r, h->pa);
      }
      if (!h->phiT) {
        const size_t n = (h->tmode ? h->aC : h->aS) + kSrcSlack;
        double* r = halloc(h, n);
        if (!r) return fail(h, ADI_ENOMEM, "source pattern");
        h->phiT = h->tmode ? r - (ptrdiff_t)h->xa * h->pc : cols_in(h, r);
      }
    }
    CUDA_TRY(h, cudaMemsetAsync(rows_raw(h, h->phi, h->pa), 0, (h->aS + kSrcSlack) * 8, h->stream));
    if (h->tmode) {
      // the column side: phiT rows x in [xa, xb) (all y), from the user's columns
      CUDA_TRY(h, cudaMemsetAsync(h->phiT + (ptrdiff_t)h->xa * h->pc, 0, (h->aC + kSrcSlack) * 8, h->stream));
      const int off = h->off;
      const int ia = std::max(h->xa - off, 0), ib = std::min(h->xb - off, h->nxi);
      if (ib > ia) {
        double* tmp = nullptr;
        CUDA_TRY(h, cudaMalloc(&tmp, (size_t)h->nyi * (ib - ia) * 8));
        cudaError_t e = cudaMemcpy2DAsync(tmp, (ib - ia) * 8, phi + ia, h->nxi * 8, (ib - ia) * 8, h->nyi,
                                          cudaMemcpyHostToDevice, h->stream);
        int rc = e == cudaSuccess ? transpose(h, tmp, h->phiT + (size_t)(ia + off) * h->pc + off, h->nyi, ib - ia,
                                              ib - ia, h->pc, 1, 0, 0)
                                  : fail(h, ADI_ECUDA, "source copy");
        cudaStreamSynchronize(h->stream);
        cudaFree(tmp);
        if (rc) return rc;
      }
    } else {
      CUDA_TRY(h, cudaMemsetAsync(cols_raw(h, h->phiT), 0, (h->aS + kSrcSlack) * 8, h->stream));
    }
    // interior point (j, i) of the user's block is position (y, x) = (j + off, i + off);
    // a band-local handle keeps the rows y in [ya, yb)
    const int off = h->off;
    const int y0 = std::max(h->ya, off), y1 = std::min(h->yb, off + h->nyi);
    if (y1 > y0) {
      CUDA_TRY(h, cudaMemcpy2DAsync(h->phi + (size_t)y0 * h->pa + off, h->pa * 8, phi + (size_t)(y0 - off) * h->nxi,
                                    h->nxi * 8, h->nxi * 8, y1 - y0, cudaMemcpyHostToDevice, h->stream));
      if (!h->tmode) {
        int rc = transpose(h, h->phi + (size_t)y0 * h->pa + off, h->phiT + (size_t)off * h->pb + y0, y1 - y0,
                           h->nxi, h->pa, h->pb, 1, 0, 0);
        if (rc) return rc;
      }
    }
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  } else if (h->phi) {
    h->tmaps.clear();
    h->smaps.clear();
    hfree(h, rows_raw(h, h->phi, h->pa), h->aS + kSrcSlack);
    if (h->tmode) hfree(h, h->phiT + (ptrdiff_t)h->xa * h->pc, h->aC + kSrcSlack);
    else hfree(h, cols_raw(h, h->phiT), h->aS + kSrcSlack);
    h->phi = nullptr;
    h->phiT = nullptr;
  }
  h->has_pt = false;
  if (has_pt) {
    int rc = set_points(h, &ix, &iy);
    if (rc) return rc;
  }
  h->gf.assign(g ? g : nullptr, g ? g + ng : nullptr);
  return ADI_OK;
}

int adi_set_point_sources(adi_handle h, const int* ix, const int* iy, const double* g, int ng) {
  DevGuard dg_(h);
  if (!h || !ix || !iy) return ADI_EINVAL;
  h->carry_valid = false;   // the next call recomputes its a2 (prologue)
  h->err.clear();
  if (g && ng < 1) return fail(h, ADI_EINVAL, "empty source table");
  int rc = set_points(h, ix, iy);
  if (rc) return rc;
  h->gf.assign(g ? g : nullptr, g ? g + ng : nullptr);
  return ADI_OK;
}

int adi_set_boundary(adi_handle h, const double* edges, const double* g, int ng) {
  DevGuard dg_(h);
  if (!h) return ADI_EINVAL;
  h->carry_valid = false;   // the next call recomputes its a2 (prologue)
  h->err.clear();
  if (g && ng < 1) return fail(h, ADI_EINVAL, "empty boundary table");
  if (h->full && edges) return fail(h, ADI_EINVAL, "the full-matrix variant has no Dirichlet data");
  const size_t ne = 2 * (size_t)h->nxu + 2 * (size_t)h->nyu;
  if (edges) {
    if (!h->edges) CUDA_TRY(h, cudaMalloc(&h->edges, ne * 8));
    H2D_SYNC(h, h->edges, edges, ne * 8);
  } else if (h->edges) {
    cudaFree(h->edges);
    h->edges = nullptr;
  }
  h->gb.assign(g ? g : nullptr, g ? g + ng : nullptr);
  return ADI_OK;
}

int adi_set_media(adi_handle h, const float* kappa, const float* rinv_v, const float* rinv_w) {
  DevGuard dg_(h);
  if (!h) return ADI_EINVAL;
  h->carry_valid = false;   // the next call recomputes its a2 (prologue)
  h->err.clear();
  if (h->in_call) return fail(h, ADI_ESTATE, "call in progress");
  if (!kappa && !rinv_v && !rinv_w) {   // back to the scalar medium
    h->tmaps.clear();
    h->smaps.clear();
    hfree(h, rows_raw(h, h->Ca, h->pa), h->aS);
    hfree(h, cols_raw(h, h->Cb), h->aS);
    h->Ca = h->Cb = nullptr;
    h->het = false;
    return ADI_OK;
  }
  if (!kappa || !rinv_v || !rinv_w) return fail(h, ADI_EINVAL, "kappa, rinv_v, rinv_w: all or none");
  if (h->tmode) return fail(h, ADI_EINVAL, "media fields are not available in the transpose decomposition");
  if (h->full) return fail(h, ADI_EINVAL, "media fields are not available for the full-matrix variant");
  // values: finite and > 0; the CFL bound uses max kappa * max rho^-1 >= c_max^2
  double kmax = 0, rmax = 0;
  auto scan = [&](const float* a, size_t n, size_t r0, size_t r1, size_t rowlen, size_t c0, size_t c1,
                  double& mx) -> bool {
    (void)n;
    for (size_t r = r0; r < r1; ++r)
      for (size_t c = c0; c < c1; ++c) {
        const float v = a[r * rowlen + c];
        if (!(v >= FLT_MIN) || !std::isfinite(v)) return false;   // normal, > 0 (exact in-kernel widening)
        mx = std::max(mx, (double)v);
      }
    return true;
  };
  if (!scan(kappa, h->nU, 1, h->nyu - 1, h->nxu, 1, h->nxu - 1, kmax) ||
      !scan(rinv_v, h->nV, 0, h->nyi, h->nxv, 0, h->nxv, rmax) ||
      !scan(rinv_w, h->nW, 0, h->nyv, h->nxi, 0, h->nxi, rmax))
    return fail(h, ADI_EINVAL, "media values must be finite normal floats > 0");
  if (!h->Ca) {
    h->tmaps.clear();
    h->smaps.clear();
    double* ra = halloc(h, h->aS);
    double* rb = ra ? halloc(h, h->aS) : nullptr;
    if (!ra || !rb) {
      hfree(h, ra, h->aS);
      return fail(h, ADI_ENOMEM, "media arrays");
    }
    h->Ca = rows_in(h, ra, h->pa);
    h->Cb = cols_in(h, rb);
  }
  float* tmp = nullptr;
  const size_t nk = h->nU, nv = h->nV, nw = h->nW;
  CUDA_TRY(h, cudaMalloc(&tmp, (nk + nv + nw) * sizeof(float)));
  auto done = [&](int rc) { cudaStreamSynchronize(h->stream); cudaFree(tmp); return rc; };
  if (cudaMemcpyAsync(tmp, kappa, nk * 4, cudaMemcpyHostToDevice, h->stream) != cudaSuccess ||
      cudaMemcpyAsync(tmp + nk, rinv_v, nv * 4, cudaMemcpyHostToDevice, h->stream) != cudaSuccess ||
      cudaMemcpyAsync(tmp + nk + nv, rinv_w, nw * 4, cudaMemcpyHostToDevice, h->stream) != cudaSuccess)
    return done(fail(h, ADI_ECUDA, "media copy"));
  {
    // the rows y of the band-local arrays: [ya, yb) (row sweep lines 1..nyi among them)
    const int ylo = std::max(h->ya, 1), yhi = std::min(h->yb - 1, h->nyi);
    if (yhi >= ylo)
      pack_media_rows<<<dim3((h->pa + 255) / 256, yhi - ylo + 1), 256, 0, h->stream>>>(
          reinterpret_cast<float2*>(h->Ca), h->pa, ylo, yhi, h->nxi, h->nxu, h->nxv, tmp, tmp + nk);
    pack_media_cols<<<dim3((h->pb + 255) / 256, h->nxi), 256, 0, h->stream>>>(
        reinterpret_cast<float2*>(h->Cb), h->pb, h->ya, h->nxi, h->nyi, h->nyv, h->nxu, tmp, tmp + nk + nv);
  }
  if (cudaGetLastError() != cudaSuccess) return done(fail(h, ADI_ECUDA, "media pack"));
  int rc = done(ADI_OK);
  h->het = true;
  const double cfl = std::sqrt(kmax * rmax) * h->dt / h->h;
  const double lim = (h->method == ADI_MFD) ? 2.0 / std::sqrt(6.0) : 2.0 / std::sqrt(3.0);
  if (rc == ADI_OK && cfl > lim) {
    h->err = "c_max*dt/h above the inner-iteration limit";
    return ADI_WUNSTABLE;
  }
  return rc;
}

// carry mode: the last column kernel of a call also writes the next
// step's S1 and W* (the fused a2 of a regular column kernel), so that the next call can
// skip its prologue.  Plain handles only: no band or dist (halo rows of S1 would be
// stale), no stopping rule, no media, not the full-matrix variant.
static bool carry_ok(const adi_ctx* h) {
  return h->carry_on && !h->full && !h->het && h->eps <= 0.0 && !h->dist && h->band_y0 <= 0 &&
         h->band_y1 >= h->ay.n + 1 && !thread_mode(h);
}

// ---- one call = begin (prologue), n x {rows, cols}, end.  The phases are public so
// that a multi-GPU driver can exchange halos between the row and column sweeps.
int adi_step_begin(adi_handle h, int nsteps) {
  DevGuard dg_(h);
  if (!h) return ADI_EINVAL;
  h->err.clear();
  if (h->in_call) return fail(h, ADI_ESTATE, "a call is already in progress");
  if (nsteps < 1) return fail(h, ADI_EINVAL, "n < 1");
  if (!h->fields_set) return fail(h, ADI_ESTATE, "fields not set");
  const long long m0 = h->m, m1 = h->m + nsteps;
  if (!h->gf.empty() && (long long)h->gf.size() < 2 * m1 + 1)
    return fail(h, ADI_EINVAL, "source table too short for the requested steps");
  if (!h->gb.empty() && (long long)h->gb.size() < 2 * m1 + 1)
    return fail(h, ADI_EINVAL, "boundary table too short for the requested steps");
  if (h->eps > 0.0 && h->full)
    return fail(h, ADI_EINVAL, "the stopping rule (ADI_EPS > 0) is not available for the full-matrix variant");
  if (h->eps > 0.0 && h->het)
    return fail(h, ADI_EINVAL, "the stopping rule (ADI_EPS > 0) is not available with media fields");
  if (h->eps > 0.0 && h->dist && h->nranks > 1)
    return fail(h, ADI_EINVAL, "the stopping rule (ADI_EPS > 0) needs the whole grid on one handle");
  if (h->eps > 0.0) {
    // the stopping rule tests norms of the whole grid: no band decomposition
    if (h->band_y0 > 0 || h->band_y1 < h->ay.n + 1)
      return fail(h, ADI_EINVAL, "the stopping rule (ADI_EPS > 0) needs the whole grid on one handle");
    if (h->kmin > h->K) return fail(h, ADI_EINVAL, "ADI_K_MIN exceeds ADI_K_SWEEPS");
    if (h->d_norms_cap < h->K + 1) {
      if (h->d_norms) cudaFree(h->d_norms);
      h->d_norms = nullptr;
      h->d_norms_cap = 0;
      CUDA_TRY(h, cudaMalloc(&h->d_norms, sizeof(double) * 4 * (h->K + 1)));
      h->d_norms_cap = h->K + 1;
    }
    if (!h->d_k) CUDA_TRY(h, cudaMalloc(&h->d_k, 4 * sizeof(int)));
  }
  int rc;
  // carry mode: the buffer the last column kernel writes the next step's W* into is
  // allocated here, before any launch of the call; without it the call ends with the
  // plain FINAL kernel (call_carry = false) instead of failing half way
  h->call_carry = carry_ok(h);
  if (h->call_carry && !h->W3) {
    double* r = halloc(h, (size_t)h->batch * h->aW);
    if (r) h->W3 = cols_in(h, r);
    else {
      h->call_carry = false;
      h->carry_valid = false;
    }
  }
  h->call_K = h->K;
  if (h->carry_valid && carry_ok(h)) {
    // the previous call's last column kernel left S1 in Sa and W* in W3
    h->carry_valid = false;
    h->Vcur = h->V; h->Valt = h->V2;
    h->Wcur = h->W3; h->Walt = h->W2;
  } else {
    h->carry_valid = false;
    // a2 (standalone once per call): S1 = U - alpha D̄_y W + dt/2 F(t^m), W* = W - beta D_y U
    adi::KParams p = base_params(h, h->ay, true);
    p.U_in = h->U;
    p.X_in = h->W; p.X_out = h->W2;
    p.S_out = h->tmode ? h->Sd : h->Sa;
    p.gf = tabv(h->gf, 2 * m0);
    if ((rc = launch(h, adi::KM_PROLOGUE, h->ay, p, ADI_KK_PROLOGUE))) return rc;
    h->Vcur = h->V; h->Valt = h->V2;
    h->Wcur = h->W2; h->Walt = h->W;
  }
  h->call_m1 = m1;
  h->in_call = true;
  return ADI_OK;
}

int adi_step_rows(adi_handle h) {
  DevGuard dg_(h);
  if (!h) return ADI_EINVAL;
  if (!h->in_call || h->m >= h->call_m1) return fail(h, ADI_ESTATE, "no step pending");
  const long long m = h->m;
  adi::KParams p = base_params(h, h->ax, false);
  p.S_in = h->Sa; p.S_out = h->Sb;
  p.X_in = h->Vcur; p.X_out = h->Valt;
  p.gb = tabv(h->gb, 2 * m + 1);   // boundary values of the intermediate U* at t^m + dt/2 [G9]
  p.gf = tabv(h->gf, 2 * m + 2);
  int rc;
  if (h->eps > 0.0) rc = stage_with_rule(h, adi::KM_SWEEP_T, h->ax, p, ADI_KK_ROW, 0);
  else rc = launch(h, adi::KM_SWEEP, h->ax, p, ADI_KK_ROW);
  if (rc) return rc;
  std::swap(h->Vcur, h->Valt);
  return ADI_OK;
}

int adi_step_cols(adi_handle h) {
  DevGuard dg_(h);
  if (!h) return ADI_EINVAL;
  if (!h->in_call || h->m >= h->call_m1) return fail(h, ADI_ESTATE, "no step pending");
  const long long m = h->m;
  const bool last = (m + 1 == h->call_m1);
  adi::KParams p = base_params(h, h->ay, true);
  p.S_in = h->tmode ? h->Sc : h->Sb;
  p.X_in = h->Wcur;
  p.gb = tabv(h->gb, 2 * m + 2);
  p.gf = tabv(h->gf, 2 * m + 2);
  int rc;
  // a band whose halo exchange is in flight (split_wait): the segments that
  // read no halo position run first, the others after the exchange has landed
  auto cols = [&](int mode, int kind) -> int {
    if (!h->split_wait) return launch(h, mode, h->ay, p, kind);
    TimeScope ts(h, kind);          // one record for both launches (one logical kernel)
    const int timing = h->timing;
    h->timing = 0;
    h->cols_phase = 1;
    int r = launch(h, mode, h->ay, p, kind);
    h->cols_phase = 2;
    if (!r && cudaStreamWaitEvent(h->stream, h->split_wait, 0) != cudaSuccess)
      r = fail(h, ADI_ECUDA, "stream wait on the halo exchange");
    if (!r) r = launch(h, mode, h->ay, p, kind);
    h->cols_phase = 0;
    h->split_wait = nullptr;
    h->timing = timing;
    return r;
  };
  if (last && h->call_carry) {
    // a regular column kernel (S1, W* of step m+1 into Sa, W3) that also writes
    // U^{m+1} and W̄^{m+1}; the three W buffers rotate: W = W̄^{m+1}, W3 = W*, W2 = free
    // (W3 was allocated by adi_step_begin)
    double* in = h->Wcur;
    double* outW = nullptr;
    double* outC = nullptr;
    for (double* q : {h->W, h->W2, h->W3}) {
      if (q == in) continue;
      if (!outW) outW = q;
      else if (!outC) outC = q;
    }
    p.S_out = h->Sa;
    p.X_out = outC;
    p.U_out = h->U;
    p.X_out2 = outW;
    p.carry = 1;
    rc = launch(h, adi::KM_SWEEP, h->ay, p, ADI_KK_FINAL);
    if (rc) return rc;
    h->W = outW; h->W3 = outC; h->W2 = in;
    h->Wcur = h->W; h->Walt = h->W2;
    h->carry_valid = true;
  } else if (last) {  // write U^{m+1} and W̄^{m+1} into the canonical buffers
    p.U_out = h->U;
    p.X_out = (h->Wcur == h->W) ? h->W2 : h->W;
    rc = (h->eps > 0.0) ? stage_with_rule(h, adi::KM_FINAL_T, h->ay, p, ADI_KK_FINAL, 1)
                        : cols(adi::KM_FINAL, ADI_KK_FINAL);
    if (rc) return rc;
    if (h->Wcur == h->W) std::swap(h->W, h->W2);
  } else {
    p.S_out = h->tmode ? h->Sd : h->Sa;
    p.X_out = h->Walt;
    rc = (h->eps > 0.0) ? stage_with_rule(h, adi::KM_SWEEP_T, h->ay, p, ADI_KK_COL, 1)
                        : cols(adi::KM_SWEEP, ADI_KK_COL);
    if (rc) return rc;
    std::swap(h->Wcur, h->Walt);
  }
  h->m = m + 1;
  return ADI_OK;
}

int adi_step_end(adi_handle h) {
  DevGuard dg_(h);
  if (!h) return ADI_EINVAL;
  if (!h->in_call || h->m != h->call_m1) return fail(h, ADI_ESTATE, "steps of the call not finished");
  if (h->Vcur != h->V) std::swap(h->V, h->V2);
  if (!h->full) {  // Dirichlet columns of U^{m1}
    dim3 g(((h->tmode ? h->nyu : h->yb - h->ya) + 255) / 256, h->batch);
    const double* ex0 = h->edges ? h->edges + 2 * h->nxu : nullptr;
    const double* ex1 = h->edges ? h->edges + 2 * h->nxu + h->nyu : nullptr;
    TimeScope ts(h, ADI_KK_EDGE);
    // (the transpose decomposition: U holds all rows, the columns [xa, xb))
    const int r0 = h->tmode ? 0 : h->ya, r1 = h->tmode ? h->nyu : h->yb;
    const int lo = h->tmode ? (h->xa == 0) : 1, hi = h->tmode ? (h->xb == h->nxu) : 1;
    edge_cols_kernel<<<g, 256, 0, h->stream>>>(h->U, r0, r1, h->nxu, h->pu, (long long)h->aU, ex0, ex1,
                                                tabv(h->gb, 2 * h->m), lo, hi);
    CUDA_TRY(h, cudaGetLastError());
    h->launches++;
    if (!h->capturing) h->host_launches++;
  }
  h->in_call = false;
  if (h->check_finite && !h->capturing) {   // (a captured call checks after its graph launch)
    int f = 0;
    CUDA_TRY(h, cudaMemcpyAsync(&f, h->flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    if (f) {
      h->nonfinite = 1;
      return fail(h, ADI_ENONFINITE, "non-finite value in the fields");
    }
  }
  return ADI_OK;
}

static int dist_exchange(adi_ctx* h, int kind);
static int tm_exchange(adi_ctx* h, int kind);
static int tm_barrier(adi_ctx* h);

// ADI_GRAPH: capture the call's launches on the capture stream, then launch the graph on
// the handle's stream (kernel parameters differ from call to call -- time factors, the
// rotating buffers -- so the kept executable graph is updated with the new capture)
static int step_graph(adi_ctx* h, int nsteps) {
  // everything that allocates or synchronizes happens before the capture
  if (carry_ok(h) && !h->W3) {
    double* r = halloc(h, (size_t)h->batch * h->aW);
    if (!r) return fail(h, ADI_ENOMEM, "carry buffer");
    h->W3 = cols_in(h, r);
  }
  if (!h->gstream && cudaStreamCreateWithFlags(&h->gstream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(h, ADI_ECUDA, "capture stream");
  cudaStream_t user = h->stream;
  cudaStream_t cap = user ? user : h->gstream;
  CUDA_TRY(h, cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed));
  h->stream = cap;
  h->capturing = true;
  const long long m0 = h->m;
  const bool carry0 = h->carry_valid;
  int rc = adi_step(h, nsteps);
  h->capturing = false;
  h->stream = user;
  cudaGraph_t g = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(cap, &g);
  if (rc || ec != cudaSuccess) {
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    // nothing ran: the host state goes back to the start of the call
    h->m = m0;
    h->in_call = false;
    h->carry_valid = carry0 && !rc ? carry0 : false;
    return rc ? rc : fail(h, ADI_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ec));
  }
  bool ok = false;
  if (h->gexec) {
    cudaGraphExecUpdateResultInfo info;
    ok = cudaGraphExecUpdate(h->gexec, g, &info) == cudaSuccess;
    if (!ok) { cudaGetLastError(); cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; }
  }
  if (!ok && cudaGraphInstantiate(&h->gexec, g, 0) != cudaSuccess) {
    cudaGetLastError();
    cudaGraphDestroy(g);
    h->gexec = nullptr;
    return fail(h, ADI_ECUDA, "graph instantiate");
  }
  cudaGraphDestroy(g);
  CUDA_TRY(h, cudaGraphLaunch(h->gexec, h->stream));
  h->host_launches++;
  if (h->check_finite) {
    int f = 0;
    CUDA_TRY(h, cudaMemcpyAsync(&f, h->flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    if (f) {
      h->nonfinite = 1;
      return fail(h, ADI_ENONFINITE, "non-finite value in the fields");
    }
  }
  return ADI_OK;
}

int adi_step(adi_handle h, int nsteps) {
  DevGuard dg_(h);
  if (!h) return ADI_EINVAL;
  if (nsteps < 0) return fail(h, ADI_EINVAL, "n < 0");
  if (nsteps == 0) return ADI_OK;
  // a handle of adi_create_dist: the halo exchanges of DESIGN.md §7 happen here (U and W̄
  // before the call's prologue unless the fields were just set; S and W* after every
  // row sweep), NCCL grouped send/recv on the handle's stream
  if (h->loop && h->nranks > 1)
    return fail(h, ADI_ESTATE, "a rank of adi_create_dist_local steps with adi_step_dist_local");
  if (h->graph_on && !h->capturing && !(h->dist && h->nranks > 1) && h->eps <= 0.0) return step_graph(h, nsteps);
  const bool ex = h->dist && h->nranks > 1;
  int rc = ADI_OK;
  if (ex && h->tmode) {   // the transpose decomposition (NCCL all-to-all of S)
    // fused: the kernels stored S into the owners' arrays; a barrier replaces the exchange
    const bool fz = tm_fused_now(h);
    auto xchg = [&](int kind) { return fz ? tm_barrier(h) : tm_exchange(h, kind); };
    rc = adi_step_begin(h, nsteps);
    if (!rc) rc = xchg(1);
    for (int k = 0; k < nsteps && !rc; ++k) {
      rc = adi_step_rows(h);
      if (!rc) rc = xchg(0);
      if (!rc) rc = adi_step_cols(h);
      if (!rc && k + 1 < nsteps) rc = xchg(1);
    }
    if (rc) { h->in_call = false; return rc; }
    return adi_step_end(h);
  }
  if (ex && !h->fresh) rc = dist_exchange(h, 1);
  if (rc == ADI_OK) rc = adi_step_begin(h, nsteps);
  for (int k = 0; k < nsteps && rc == ADI_OK; ++k) {
    rc = adi_step_rows(h);
    if (rc == ADI_OK && ex) rc = dist_exchange(h, 0);
    if (rc == ADI_OK) rc = adi_step_cols(h);
  }
  if (rc == ADI_OK) h->fresh = false;
  if (rc != ADI_OK) { h->in_call = false; h->split_wait = nullptr; return rc; }
  return adi_step_end(h);
}

// ---- band decomposition --------------------------------------------------
// Re-lay the arrays out for the y extent [nya, nyb): the state (U, V̄, W̄)
// and the static inputs (phi, media) keep their rows inside both extents; the scratch
// arrays are new.  Rows of the new extent outside the old one are zero.
static int relayout(adi_ctx* h, int nya, int nyb) {
  const int oya = h->ya, oyb = h->yb, opb = h->pb, opw = h->pw;
  const size_t oaU = h->aU, oaS = h->aS, oaV = h->aV, oaW = h->aW;
  const size_t B = (size_t)h->batch;
  struct Arr { double** p; bool rows; int pitch_old; size_t a_old; size_t nb; bool live; };
  double* oraw[12];
  Arr arrs[12] = {
      {&h->Ubase, true, h->pu, oaU, B, true},   {&h->V, true, h->pv, oaV, B, true},
      {&h->V2, true, h->pv, oaV, B, false},     {&h->Sa, true, h->pa, oaS, B, false},
      {&h->phi, true, h->pa, oaS, 1, true},     {&h->Ca, true, h->pa, oaS, 1, true},
      {&h->W, false, opw, oaW, B, true},        {&h->W2, false, opw, oaW, B, false},
      {&h->W3, false, opw, oaW, B, false},      {&h->Sb, false, opb, oaS, B, false},
      {&h->phiT, false, opb, oaS, 1, true},     {&h->Cb, false, opb, oaS, 1, true}};
  for (int k = 0; k < 12; ++k)
    oraw[k] = arrs[k].rows ? rows_raw(h, *arrs[k].p, arrs[k].pitch_old) : cols_raw(h, *arrs[k].p);
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  set_extent(h, nya, nyb);
  const int ylo = std::max(oya, nya), yhi = std::min(oyb, nyb);
  double* nraw[12] = {};
  bool ok = true;
  for (int k = 0; k < 12 && ok; ++k) {
    if (!oraw[k] || (k == 8)) continue;   // absent, or the carry buffer W3 (bands do not carry)
    const Arr& A = arrs[k];
    const bool isS = (A.p == &h->Sa || A.p == &h->Sb || A.p == &h->phi || A.p == &h->phiT || A.p == &h->Ca ||
                      A.p == &h->Cb);
    const bool isPhi = (A.p == &h->phi || A.p == &h->phiT);
    const size_t an = (isS ? h->aS : A.rows ? (A.p == &h->Ubase ? h->aU : h->aV) : h->aW) + (isPhi ? kSrcSlack : 0);
    nraw[k] = halloc(h, A.nb * an);
    if (!nraw[k]) { ok = false; break; }
    if (!A.live || yhi <= ylo) continue;
    for (size_t b = 0; b < A.nb; ++b) {
      cudaError_t e;
      if (A.rows)
        e = cudaMemcpyAsync(nraw[k] + b * an + (size_t)(ylo - nya) * A.pitch_old,
                            oraw[k] + b * A.a_old + (size_t)(ylo - oya) * A.pitch_old,
                            (size_t)(yhi - ylo) * A.pitch_old * 8, cudaMemcpyDeviceToDevice, h->stream);
      else
        e = cudaMemcpy2DAsync(nraw[k] + b * an + (ylo - nya), (A.p == &h->W ? h->pw : h->pb) * 8,
                              oraw[k] + b * A.a_old + (ylo - oya), A.pitch_old * 8, (size_t)(yhi - ylo) * 8,
                              h->nxu, cudaMemcpyDeviceToDevice, h->stream);
      if (e != cudaSuccess) { cudaGetLastError(); ok = false; break; }
    }
  }
  if (ok && cudaStreamSynchronize(h->stream) != cudaSuccess) ok = false;
  if (!ok) {   // undo: keep the old layout
    for (int k = 0; k < 12; ++k)
      if (nraw[k]) hfree(h, nraw[k], 0);
    h->ya = oya; h->yb = oyb; h->pb = opb; h->pw = opw;
    h->aU = oaU; h->aS = oaS; h->aV = oaV; h->aW = oaW;
    return fail(h, ADI_ENOMEM, "band re-layout");
  }
  for (int k = 0; k < 12; ++k) {
    const Arr& A = arrs[k];
    const size_t an_old = A.a_old * A.nb;
    if (oraw[k]) hfree(h, oraw[k], an_old);
    *A.p = nraw[k] ? (A.rows ? rows_in(h, nraw[k], A.pitch_old) : cols_in(h, nraw[k])) : nullptr;
  }
  h->U = h->Ubase;
  h->tmaps.clear();
    h->smaps.clear();
  h->carry_valid = false;
  return ADI_OK;
}

int adi_set_band(adi_handle h, int y0, int y1) {
  DevGuard dg_(h);
  if (!h) return ADI_EINVAL;
  h->carry_valid = false;   // the next call recomputes its a2 (prologue)
  h->err.clear();
  if (h->in_call) return fail(h, ADI_ESTATE, "call in progress");
  const int ny_pos = h->ay.n + 1;  // y positions 0..n_y
  if (y0 < 0 || y1 > ny_pos || y0 >= y1) return fail(h, ADI_EINVAL, "band out of range");
  if (h->full) return fail(h, ADI_EINVAL, "no band decomposition for the full-matrix variant");
  if (h->dist && h->nranks > 1)
    return fail(h, ADI_EINVAL, "the band of an adi_create_dist handle is fixed at creation");
  // validated before any state changes (a refused band leaves the handle as it was)
  const int hl = h->ay.halo;
  if ((y0 > 0 && y1 - y0 < hl) || (y1 < ny_pos && y1 - y0 < hl))
    return fail(h, ADI_EINVAL, "band thinner than the halo");
  const adi::Axis ax_old = h->ax, ay_old = h->ay;
  const int b0_old = h->band_y0, b1_old = h->band_y1;
  h->band_y0 = y0;
  h->band_y1 = y1;
  // row sweep: interior rows (lines = y positions 1..nyi) inside [y0, y1)
  h->ax.l0 = std::max(y0, 1);
  h->ax.l1 = std::min(y1, h->nyi + 1);
  // column sweep: outputs at y positions [y0, y1)
  h->ay.o0 = y0;
  h->ay.o1 = y1;
  h->ay.d_segs = nullptr;   // setup_axis allocates a new plan; the old one is kept until it succeeds
  h->ay.d_tabU = h->ay.d_tabX = nullptr;
  int rc = setup_axis(h, h->ay, h->ny - 1, h->nxi, 4);
  if (!rc) {
    // band-local arrays: the band and its halo rows only (memory per handle ~ 1/P)
    int nya, nyb;
    band_extent(h, y0, y1, hl, &nya, &nyb);
    if (nya != h->ya || nyb != h->yb) rc = relayout(h, nya, nyb);
  }
  if (rc) {
    for (void* q : {(void*)h->ay.d_segs, (void*)h->ay.d_tabU, (void*)h->ay.d_tabX})
      if (q) cudaFree(q);
    h->ax = ax_old;
    h->ay = ay_old;
    h->band_y0 = b0_old;
    h->band_y1 = b1_old;
    return rc;
  }
  for (void* q : {(void*)ay_old.d_segs, (void*)ay_old.d_tabU, (void*)ay_old.d_tabX})
    if (q) cudaFree(q);
  return ADI_OK;
}

// halo rows [a, b) (y positions) exchanged on one side of the band
static void halo_range(adi_ctx* h, int side, int own, int* a, int* b) {
  const int hl = h->ay.halo, npos = h->ay.n + 1;
  if (side == 0) {  // low side
    if (own) { *a = h->band_y0; *b = std::min(h->band_y0 + hl, h->band_y1); }
    else { *a = std::max(h->band_y0 - hl, 0); *b = h->band_y0; }
  } else {
    if (own) { *a = std::max(h->band_y1 - hl, h->band_y0); *b = h->band_y1; }
    else { *a = h->band_y1; *b = std::min(h->band_y1 + hl, npos); }
  }
}

// layout of one halo message: kind 0 (after the row sweep): S (S^T layout) then W* (W̄^T);
// kind 1 (before the prologue): U rows then W̄ (W̄^T layout).  Per grid of the batch.
static size_t halo_elems(adi_ctx* h, int kind, int rows) {
  if (kind == 0) return (size_t)h->batch * ((size_t)h->nxi * rows * 2);
  return (size_t)h->batch * ((size_t)h->nxu * rows + (size_t)h->nxi * rows);
}

int adi_halo_bytes(adi_handle h, int kind, int side, size_t* bytes) {
  DevGuard dg_(h);
  if (!h || !bytes || kind < 0 || kind > 1 || side < 0 || side > 1 || h->tmode) return ADI_EINVAL;
  int a, b, c, d;
  halo_range(h, side, 1, &a, &b);
  halo_range(h, side, 0, &c, &d);
  *bytes = 8 * halo_elems(h, kind, std::max(b - a, d - c));
  return ADI_OK;
}

// copy y positions [a, b) of the halo fields between the internal arrays and a
// contiguous device buffer (pack: dir = 0, unpack: dir = 1)
static int halo_copy(adi_ctx* h, int kind, int a, int b, double* buf, int dir, cudaStream_t st) {
  const int rows = b - a;
  if (rows <= 0) return ADI_OK;
  double* q = buf;
  auto cp = [&](double* arr, size_t pitch, int nr, int col0, size_t bstride) -> int {
    for (int bb = 0; bb < h->batch; ++bb) {
      double* base = arr + bb * bstride + col0;
      cudaError_t e = dir == 0
          ? cudaMemcpy2DAsync(q, rows * 8, base, pitch * 8, rows * 8, nr, cudaMemcpyDeviceToDevice, st)
          : cudaMemcpy2DAsync(base, pitch * 8, q, rows * 8, rows * 8, nr, cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return fail(h, ADI_ECUDA, std::string("halo copy: ") + cudaGetErrorString(e));
      q += (size_t)nr * rows;
    }
    return ADI_OK;
  };
  int rc;
  if (kind == 0) {
    // S (S^T layout, row = x position, index = y) and W* (W̄^T, same indexing), rows 1..nxi
    if ((rc = cp(h->Sb + h->pb, h->pb, h->nxi, a, h->aS))) return rc;
    if ((rc = cp(h->Wcur + h->pw, h->pw, h->nxi, a, h->aW))) return rc;
  } else {
    // U rows a..b-1 (all columns, contiguous per row) and W̄ (W̄^T layout)
    for (int bb = 0; bb < h->batch; ++bb) {
      double* base = h->U + bb * h->aU + (size_t)a * h->pu;
      cudaError_t e = dir == 0
          ? cudaMemcpy2DAsync(q, h->nxu * 8, base, h->pu * 8, h->nxu * 8, rows, cudaMemcpyDeviceToDevice, st)
          : cudaMemcpy2DAsync(base, h->pu * 8, q, h->nxu * 8, h->nxu * 8, rows, cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return fail(h, ADI_ECUDA, std::string("halo copy: ") + cudaGetErrorString(e));
      q += (size_t)h->nxu * rows;
    }
    if ((rc = cp(h->W + h->pw, h->pw, h->nxi, a, h->aW))) return rc;
  }
  return ADI_OK;
}

int adi_halo_pack(adi_handle h, int kind, int side, void* dev_buf) {
  DevGuard dg_(h);
  if (!h || !dev_buf || kind < 0 || kind > 1 || side < 0 || side > 1 || h->tmode) return ADI_EINVAL;
  h->err.clear();
  int a, b;
  halo_range(h, side, 1, &a, &b);
  return halo_copy(h, kind, a, b, (double*)dev_buf, 0, h->stream);
}

int adi_halo_unpack(adi_handle h, int kind, int side, const void* dev_buf) {
  DevGuard dg_(h);
  if (!h || !dev_buf || kind < 0 || kind > 1 || side < 0 || side > 1 || h->tmode) return ADI_EINVAL;
  h->carry_valid = false;   // the next call recomputes its a2 (prologue)
  h->err.clear();
  int a, b;
  halo_range(h, side, 0, &a, &b);
  return halo_copy(h, kind, a, b, (double*)dev_buf, 1, h->stream);
}

// ---- adi_create_dist: the band decomposition with the exchange inside the library ----
// One exchange = pack this band's edge rows (main stream) -> transfer
// (exchange stream cs: NCCL grouped send/recv with the two neighbours, or loopback copies
// from the neighbour handles' send buffers) -> unpack into the halo rows (cs).  ev_recv
// marks the landed halo: kind 0 (S2, W*, after the row sweep) only gates the column
// segments that read the halo (adi_step_cols, split_wait), so the transfer overlaps the
// others; kind 1 (U, W̄, before a call's prologue) is waited for at once.
static int nbr(const adi_ctx* h, int side) { return side == 0 ? h->rank - 1 : h->rank + 1; }
static bool has_nbr(const adi_ctx* h, int side) { const int q = nbr(h, side); return q >= 0 && q < h->nranks; }

static int dist_pack(adi_ctx* h, int kind) {
  if (h->loop)   // a neighbour may still be copying our previous message
    for (adi_ctx* q : h->peer)
      if (q && q->ev_recv) CUDA_TRY(h, cudaStreamWaitEvent(h->stream, q->ev_recv, 0));
  for (int side = 0; side < 2; ++side) {
    if (!has_nbr(h, side)) continue;
    int a, b;
    halo_range(h, side, 1, &a, &b);
    int rc = halo_copy(h, kind, a, b, h->hbuf[kind][side][0], 0, h->stream);
    if (rc) return rc;
  }
  CUDA_TRY(h, cudaEventRecord(h->ev_pack, h->stream));
  return ADI_OK;
}

static int dist_transfer(adi_ctx* h, int kind) {
  CUDA_TRY(h, cudaStreamWaitEvent(h->cs, h->ev_pack, 0));
  if (h->loop) {
    for (int side = 0; side < 2; ++side) {
      adi_ctx* q = h->peer[side];
      if (!has_nbr(h, side)) continue;
      if (!q) return fail(h, ADI_ESTATE, "loopback neighbour destroyed");
      if (q->hcount[kind][1 - side][0] != h->hcount[kind][side][1])
        return fail(h, ADI_EINVAL, "internal: halo message sizes differ");
      CUDA_TRY(h, cudaStreamWaitEvent(h->cs, q->ev_pack, 0));
      CUDA_TRY(h, cudaMemcpyAsync(h->hbuf[kind][side][1], q->hbuf[kind][1 - side][0],
                                  h->hcount[kind][side][1] * sizeof(double), cudaMemcpyDeviceToDevice, h->cs));
    }
    return ADI_OK;
  }
  NCCL_TRY(h, g_nccl.groupStart());
  for (int side = 0; side < 2; ++side) {
    if (!has_nbr(h, side)) continue;
    NCCL_TRY(h, g_nccl.send(h->hbuf[kind][side][0], h->hcount[kind][side][0], ncclFloat64, nbr(h, side), h->comm,
                            h->cs));
    NCCL_TRY(h, g_nccl.recv(h->hbuf[kind][side][1], h->hcount[kind][side][1], ncclFloat64, nbr(h, side), h->comm,
                            h->cs));
  }
  NCCL_TRY(h, g_nccl.groupEnd());
  return ADI_OK;
}

static int dist_unpack(adi_ctx* h, int kind) {
  for (int side = 0; side < 2; ++side) {
    if (!has_nbr(h, side)) continue;
    int a, b;
    halo_range(h, side, 0, &a, &b);
    int rc = halo_copy(h, kind, a, b, h->hbuf[kind][side][1], 1, h->cs);
    if (rc) return rc;
  }
  CUDA_TRY(h, cudaEventRecord(h->ev_recv, h->cs));
  if (kind == 0) h->split_wait = h->ev_recv;      // the column sweep waits per segment class
  else CUDA_TRY(h, cudaStreamWaitEvent(h->stream, h->ev_recv, 0));
  return ADI_OK;
}

static int dist_exchange(adi_ctx* h, int kind) {
  int rc = dist_pack(h, kind);
  if (!rc) rc = dist_transfer(h, kind);
  if (!rc) rc = dist_unpack(h, kind);
  return rc;
}

// halo buffers, exchange stream and events of a dist handle (band already set)
static int dist_init(adi_ctx* h) {
  for (int kind = 0; kind < 2; ++kind)
    for (int side = 0; side < 2; ++side) {
      if (!has_nbr(h, side)) continue;
      for (int own = 1; own >= 0; --own) {   // send = own rows, recv = the neighbour's
        int a, b;
        halo_range(h, side, own, &a, &b);
        const size_t n = halo_elems(h, kind, b - a);
        double*& buf = h->hbuf[kind][side][own ? 0 : 1];
        h->hcount[kind][side][own ? 0 : 1] = n;
        if (cudaMalloc(&buf, std::max<size_t>(n, 1) * sizeof(double)) != cudaSuccess) {
          cudaGetLastError();
          return ADI_ENOMEM;
        }
        h->dev_bytes += (long long)(std::max<size_t>(n, 1) * sizeof(double));
      }
    }
  if (cudaStreamCreateWithFlags(&h->cs, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_pack, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_recv, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    return ADI_ECUDA;
  }
  return ADI_OK;
}

int adi_plan_halo(int method, int* halo) {
  if (!halo || (method != ADI_CFD && method != ADI_MFD)) return ADI_EINVAL;
  *halo = adi::plan_halo(method);
  return ADI_OK;
}

int adi_dist_bands(int npos, int nranks, int* cuts) {
  if (npos < 1 || nranks < 1 || !cuts) return ADI_EINVAL;
  dist_bands(npos, nranks, cuts);
  return ADI_OK;
}

int adi_nccl_unique_id(void* out) {
  if (!out) return ADI_EINVAL;
  if (!nccl_load()) return ADI_ENCCL;
  ncclUniqueId id;
  if (g_nccl.getUniqueId(&id) != ncclSuccess) return ADI_ENCCL;
  std::memcpy(out, &id, sizeof id);
  return ADI_OK;
}

// ---- ADI_DIST_TRANSPOSE: the all-to-all decomposition ---------------
// Re-shape a band handle (rows Y_r) into a transpose-mode rank: the column sweep takes the
// whole lines x in X_r, and the column-side arrays are allocated for those lines only.
static int trank_setup(adi_ctx* h, const std::vector<int>& cy, const std::vector<int>& cx) {
  const int r = h->rank;
  h->tmode = true;
  h->cut_y = cy;
  h->cut_x = cx;
  h->ty0 = cy[r]; h->ty1 = cy[r + 1];
  h->tx0 = cx[r]; h->tx1 = cx[r + 1];
  const int npx = h->ax.n + 1;
  h->xa = std::max(h->tx0 - 4, 0) & ~3;   // (16-byte pairs of lines in the transposed stores)
  h->xb = (h->tx1 >= npx) ? h->nxu : h->tx1;
  // the column sweep: lines x in X_r (interior), every position of each line
  h->ay.o0 = 0;
  h->ay.o1 = 1 << 30;
  h->ay.l0 = std::max(h->tx0, h->off);
  h->ay.l1 = std::min(h->tx1, h->nxi + h->off);
  h->band_y0 = 0;                 // (no halo exchange: the band machinery is off)
  h->band_y1 = 1 << 30;
  int rc = setup_axis(h, h->ay, h->ny - 1, h->nxi, 4);
  if (rc) return rc;
  // column-side arrays: drop the band-shaped ones, allocate [xa, xb) x all y
  const size_t B = (size_t)h->batch;
  hfree(h, cols_raw(h, h->W), B * h->aW);
  hfree(h, cols_raw(h, h->W2), B * h->aW);
  hfree(h, rows_raw(h, h->Ubase, h->pu), B * h->aU);
  h->W = h->W2 = h->Ubase = h->U = nullptr;
  const int nxl = h->xb - h->xa;
  h->pc = padp(h->nyu);
  h->pd = padp(nxl);
  h->pu = h->pd;
  h->aU = (size_t)h->nyu * h->pd;
  h->aC = std::max((size_t)nxl * h->pc, (size_t)h->nyu * h->pd);
  h->aW = std::max((size_t)nxl * h->pc, (size_t)h->nyv * nxl);
  double *W = halloc(h, B * h->aW), *W2 = halloc(h, B * h->aW), *U = halloc(h, B * h->aU);
  double *Sc = halloc(h, B * h->aC), *Sd = halloc(h, B * h->aC);
  if (!W || !W2 || !U || !Sc || !Sd) {
    for (double* q : {W, W2, U, Sc, Sd}) hfree(h, q, 0);
    return fail(h, ADI_ENOMEM, "transpose-mode arrays");
  }
  h->W = W - (ptrdiff_t)h->xa * h->pc;
  h->W2 = W2 - (ptrdiff_t)h->xa * h->pc;
  h->Sc = Sc - (ptrdiff_t)h->xa * h->pc;
  h->Sd = Sd - h->xa;
  h->Ubase = h->U = U - h->xa;
  h->tmaps.clear();
    h->smaps.clear();
  return ADI_OK;
}

// one all-to-all of the transpose decomposition.  kind 0 (after the row sweep): the block
// Sb[x in X_q][y in Y_r] of S2^T goes from rank r to rank q's Sc; kind 1 (after the column
// sweep or the prologue): Sd[y in Y_q][x in X_r] of S1'^T goes from rank r to q's Sa.
struct TRange { int a0, a1, c0, c1; };   // rows [a0, a1) x columns [c0, c1) of the block
static TRange trange(const adi_ctx* g, int q, int r, int kind) {
  auto clip = [](int v, int hi) { return std::min(v, hi); };
  if (kind == 0)
    return {g->cut_x[q], clip(g->cut_x[q + 1], g->nxu), g->cut_y[r], clip(g->cut_y[r + 1], g->nyu)};
  return {g->cut_y[q], clip(g->cut_y[q + 1], g->nyu), g->cut_x[r], clip(g->cut_x[r + 1], g->nxu)};
}
static size_t trange_n(const TRange& t) {
  return (size_t)std::max(t.a1 - t.a0, 0) * (size_t)std::max(t.c1 - t.c0, 0);
}
// the block's start and row pitch in the producing (src) or receiving (dst) rank's array
static double* tsrc(const adi_ctx* h, const TRange& t, int kind, int b, size_t* pitch) {
  if (kind == 0) { *pitch = h->pb; return h->Sb + b * h->aS + (size_t)t.a0 * h->pb + t.c0; }
  *pitch = h->pd;
  return h->Sd + b * h->aC + (size_t)t.a0 * h->pd + t.c0;
}
static double* tdst(const adi_ctx* h, const TRange& t, int kind, int b, size_t* pitch) {
  if (kind == 0) { *pitch = h->pc; return h->Sc + b * h->aC + (size_t)t.a0 * h->pc + t.c0; }
  *pitch = h->pa;
  return h->Sa + b * h->aS + (size_t)t.a0 * h->pa + t.c0;
}

static int tm_exchange(adi_ctx* h, int kind) {
  const int P = h->nranks, r = h->rank;
  auto copy2d = [&](double* d, size_t dp, const double* s, size_t sp, const TRange& t) -> int {
    const size_t w = (size_t)std::max(t.c1 - t.c0, 0), hg = (size_t)std::max(t.a1 - t.a0, 0);
    if (!w || !hg) return ADI_OK;
    CUDA_TRY(h, cudaMemcpy2DAsync(d, dp * 8, s, sp * 8, w * 8, hg, cudaMemcpyDeviceToDevice, h->stream));
    return ADI_OK;
  };
  if (h->loop) {
    // every rank's producing kernel precedes any rank's copy (adi_step_dist_local)
    for (int q = 0; q < P; ++q)
      if (q != r) CUDA_TRY(h, cudaStreamWaitEvent(h->stream, h->group[q]->ev_pack, 0));
    for (int q = 0; q < P; ++q) {   // the block rank q produced for me
      const TRange t = trange(h, r, q, kind);
      for (int b = 0; b < h->batch; ++b) {
        size_t sp, dp;
        const double* sptr = tsrc(h->group[q], t, kind, b, &sp);
        double* dptr = tdst(h, t, kind, b, &dp);
        int rc = copy2d(dptr, dp, sptr, sp, t);
        if (rc) return rc;
      }
    }
    return ADI_OK;
  }
  // NCCL: pack every peer's block, one grouped send/recv, unpack; the own block is a copy
  for (int q = 0; q < P; ++q) {
    const TRange t = trange(h, q, r, kind);   // what I produce for q
    size_t off = 0;
    for (int b = 0; b < h->batch; ++b) {
      size_t sp, dp;
      const double* sptr = tsrc(h, t, kind, b, &sp);
      int rc;
      if (q == r) {
        double* dptr = tdst(h, t, kind, b, &dp);
        rc = copy2d(dptr, dp, sptr, sp, t);
      } else {
        rc = copy2d(h->tsend[q] + off, (size_t)std::max(t.c1 - t.c0, 1), sptr, sp, t);
        off += trange_n(t);
      }
      if (rc) return rc;
    }
  }
  NCCL_TRY(h, g_nccl.groupStart());
  for (int q = 0; q < P; ++q) {
    if (q == r) continue;
    const size_t ns = h->batch * trange_n(trange(h, q, r, kind));
    const size_t nr = h->batch * trange_n(trange(h, r, q, kind));
    if (ns) NCCL_TRY(h, g_nccl.send(h->tsend[q], ns, ncclFloat64, q, h->comm, h->stream));
    if (nr) NCCL_TRY(h, g_nccl.recv(h->trecv[q], nr, ncclFloat64, q, h->comm, h->stream));
  }
  NCCL_TRY(h, g_nccl.groupEnd());
  for (int q = 0; q < P; ++q) {
    if (q == r) continue;
    const TRange t = trange(h, r, q, kind);   // what q produced for me
    size_t off = 0;
    for (int b = 0; b < h->batch; ++b) {
      size_t dp;
      double* dptr = tdst(h, t, kind, b, &dp);
      int rc = copy2d(dptr, dp, h->trecv[q] + off, (size_t)std::max(t.c1 - t.c0, 1), t);
      if (rc) return rc;
      off += trange_n(t);
    }
  }
  return ADI_OK;
}

// the fused transpose's half-step barrier: every rank's kernels before it (which stored S
// into the owners' arrays) complete before any rank's kernels after it (which read S, or
// overwrite what the others still read).  A local group: each rank's stream waits for the
// others' marks (adi_step_dist_local records them); NCCL: a one-element all-reduce, which
// no rank passes before every rank has reached it in stream order
static int tm_barrier(adi_ctx* h) {
  if (h->loop) {
    for (int q = 0; q < h->nranks; ++q)
      if (q != h->rank) CUDA_TRY(h, cudaStreamWaitEvent(h->stream, h->group[q]->ev_pack, 0));
    return ADI_OK;
  }
  NCCL_TRY(h, g_nccl.allReduce(h->dbar, h->dbar, 1, ncclFloat64, ncclSum, h->comm, h->stream));
  return ADI_OK;
}

// the fused transpose's peer table of a local group: the ranks' own arrays
static void tm_fuse_local(adi_ctx** g, int P) {
  for (int r = 0; r < P; ++r) {
    g[r]->tpeer.clear();
    for (int q = 0; q < P; ++q)
      g[r]->tpeer.push_back({g[q]->Sc, g[q]->Sa, g[q]->pc, g[q]->pa, (long long)g[q]->aC, (long long)g[q]->aS});
    g[r]->tfused = P <= adi::MAX_TRANKS;
    if (!g[r]->tfused) g[r]->tpeer.clear();
  }
}

// the fused transpose across processes: every rank's Sc and Sa allocations as CUDA IPC
// handles, with the offsets of the absolute-index views, all-gathered over NCCL (grouped
// send/recv of the records) and mapped with cudaIpcOpenMemHandle (peer access over
// NVLink).  All ranks fuse or none: the outcome is agreed by an all-reduce, so the
// protocols (barrier or all-to-all) match.  Failure of any step leaves the handle unfused
static int tm_fuse_init(adi_ctx* h) {
  const int P = h->nranks, r = h->rank;
  if (P > adi::MAX_TRANKS || !g_nccl.allReduce) return ADI_OK;
  struct Rec { cudaIpcMemHandle_t hc, ha; long long oc, oa, pc, pa, aC, aS; };
  std::vector<Rec> recs(P);
  double* Sc_raw = h->Sc + (ptrdiff_t)h->xa * h->pc;
  double* Sa_raw = rows_raw(h, h->Sa, h->pa);
  char* bc = reinterpret_cast<char*>(Sc_raw - adi::BUF_GUARD_FRONT);   // the cudaMalloc'd bases
  char* ba = reinterpret_cast<char*>(Sa_raw - adi::BUF_GUARD_FRONT);
  bool ok = cudaIpcGetMemHandle(&recs[r].hc, bc) == cudaSuccess && cudaIpcGetMemHandle(&recs[r].ha, ba) == cudaSuccess;
  if (!ok) cudaGetLastError();
  recs[r].oc = (long long)(reinterpret_cast<char*>(h->Sc) - bc);
  recs[r].oa = (long long)(reinterpret_cast<char*>(h->Sa) - ba);
  recs[r].pc = h->pc; recs[r].pa = h->pa; recs[r].aC = (long long)h->aC; recs[r].aS = (long long)h->aS;
  CUDA_TRY(h, cudaMalloc(&h->dbar, 2 * sizeof(double)));
  char* dbuf = nullptr;
  CUDA_TRY(h, cudaMalloc(&dbuf, P * sizeof(Rec)));
  int rc = ADI_OK;
  const size_t sz = sizeof(Rec);
  if (cudaMemcpy(dbuf + r * sz, &recs[r], sz, cudaMemcpyHostToDevice) != cudaSuccess) rc = ADI_ECUDA;
  if (!rc) {
    if (g_nccl.groupStart() != ncclSuccess) {
      rc = ADI_ENCCL;
    } else {
      for (int q = 0; q < P && !rc; ++q) {
        if (q == r) continue;
        if (g_nccl.send(dbuf + r * sz, sz, ncclChar, q, h->comm, h->stream) != ncclSuccess ||
            g_nccl.recv(dbuf + q * sz, sz, ncclChar, q, h->comm, h->stream) != ncclSuccess)
          rc = ADI_ENCCL;
      }
      if (g_nccl.groupEnd() != ncclSuccess && !rc) rc = ADI_ENCCL;
    }
  }
  if (!rc && (cudaStreamSynchronize(h->stream) != cudaSuccess ||
              cudaMemcpy(recs.data(), dbuf, P * sz, cudaMemcpyDeviceToHost) != cudaSuccess))
    rc = ADI_ECUDA;
  cudaFree(dbuf);
  if (rc) return fail(h, rc, "fused transpose: exchange of the IPC handles");
  std::vector<adi_ctx::TPeer> tp(P);
  for (int q = 0; q < P && ok; ++q) {
    if (q == r) {
      tp[q] = {h->Sc, h->Sa, h->pc, h->pa, (long long)h->aC, (long long)h->aS};
      continue;
    }
    void *mc = nullptr, *ma = nullptr;
    if (cudaIpcOpenMemHandle(&mc, recs[q].hc, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
        cudaIpcOpenMemHandle(&ma, recs[q].ha, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      if (mc) cudaIpcCloseMemHandle(mc);
      ok = false;
      break;
    }
    h->ipc_open.push_back(mc);
    h->ipc_open.push_back(ma);
    tp[q] = {reinterpret_cast<double*>(static_cast<char*>(mc) + recs[q].oc),
             reinterpret_cast<double*>(static_cast<char*>(ma) + recs[q].oa), recs[q].pc, recs[q].pa, recs[q].aC,
             recs[q].aS};
  }
  // agree: fused only if every rank mapped every peer (sum of failures == 0)
  const double mine = ok ? 0.0 : 1.0;
  double tot = 0.0;
  if (cudaMemcpy(h->dbar, &mine, sizeof mine, cudaMemcpyHostToDevice) != cudaSuccess) return fail(h, ADI_ECUDA, "fused transpose");
  NCCL_TRY(h, g_nccl.allReduce(h->dbar, h->dbar, 1, ncclFloat64, ncclSum, h->comm, h->stream));
  if (cudaStreamSynchronize(h->stream) != cudaSuccess ||
      cudaMemcpy(&tot, h->dbar, sizeof tot, cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(h, ADI_ECUDA, "fused transpose: agreement");
  if (tot == 0.0) {
    h->tpeer = tp;
    h->tfused = true;
  } else {
    for (void* q : h->ipc_open) cudaIpcCloseMemHandle(q);
    h->ipc_open.clear();
  }
  return ADI_OK;
}

// NCCL staging of the transpose mode (per peer, both directions and kinds)
static int tm_init(adi_ctx* h) {
  const int P = h->nranks;
  h->tsend.assign(P, nullptr);
  h->trecv.assign(P, nullptr);
  for (int q = 0; q < P; ++q) {
    if (q == h->rank) continue;
    const size_t yq = h->cut_y[q + 1] - h->cut_y[q] + 1, xq = h->cut_x[q + 1] - h->cut_x[q] + 1;
    const size_t yr = h->cut_y[h->rank + 1] - h->cut_y[h->rank] + 1, xr = h->cut_x[h->rank + 1] - h->cut_x[h->rank] + 1;
    const size_t n = (size_t)h->batch * std::max(xq * yr, xr * yq) + 8;
    if (cudaMalloc(&h->tsend[q], n * 8) != cudaSuccess || cudaMalloc(&h->trecv[q], n * 8) != cudaSuccess) {
      cudaGetLastError();
      return ADI_ENOMEM;
    }
    h->dev_bytes += (long long)(2 * n * 8);
  }
  if (cudaEventCreateWithFlags(&h->ev_pack, cudaEventDisableTiming) != cudaSuccess) return ADI_ECUDA;
  return ADI_OK;
}

// one rank's handle: its band's arrays only (band + halo rows), dist state set
static int create_rank(int nx, int ny, double hh, double dt, double c, int method, int batch, int rank, int nranks,
                       adi_handle* out, int mode = ADI_DIST_HALO) {
  *out = nullptr;
  const int npos = ny;   // y positions 0..ny-1 (the planner's positions of both reduced variants)
  std::vector<int> cuts(nranks + 1);
  dist_bands(npos, nranks, cuts.data());
  adi_handle h = nullptr;
  int rc = create_impl(nx, ny, hh, dt, c, method, batch, nranks > 1 ? cuts[rank] : 0,
                       nranks > 1 ? cuts[rank + 1] : 1 << 30, &h);
  if (rc < 0) return rc;
  h->dist = true;
  h->rank = rank;
  h->nranks = nranks;
  if (mode == ADI_DIST_TRANSPOSE && nranks > 1) {
    std::vector<int> cx(nranks + 1);
    dist_bands(nx, nranks, cx.data());
    const int e = trank_setup(h, cuts, cx);
    if (e) { adi_destroy(h); return e; }
  }
  *out = h;
  return rc;
}

int adi_create_dist(int nx, int ny, double hh, double dt, double c, int method, int batch,
                    const void* nccl_unique_id, int rank, int nranks, adi_handle* out) {
  return adi_create_dist_ex(nx, ny, hh, dt, c, method, batch, nccl_unique_id, rank, nranks, ADI_DIST_HALO, out);
}

int adi_create_dist_ex(int nx, int ny, double hh, double dt, double c, int method, int batch,
                       const void* nccl_unique_id, int rank, int nranks, int mode, adi_handle* out) {
  if (!out) return ADI_EINVAL;
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !nccl_unique_id)) return ADI_EINVAL;
  if (method == ADI_CFD_FULL && nranks > 1) return ADI_EINVAL;   // no band decomposition
  if (mode != ADI_DIST_HALO && mode != ADI_DIST_TRANSPOSE) return ADI_EINVAL;
  adi_handle h = nullptr;
  int rc = create_rank(nx, ny, hh, dt, c, method, batch, rank, nranks, &h, mode);
  if (rc < 0) return rc;
  const int warn = rc;
  if (nranks > 1) {
    DevGuard dg_(h);
    if (!nccl_load()) { adi_destroy(h); return ADI_ENCCL; }
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof id);
    if (g_nccl.commInitRank(&h->comm, nranks, id, rank) != ncclSuccess) {
      h->comm = nullptr;
      adi_destroy(h);
      return ADI_ENCCL;
    }
    if ((rc = h->tmode ? tm_init(h) : dist_init(h))) { adi_destroy(h); return rc; }
    if (h->tmode && (rc = tm_fuse_init(h))) { adi_destroy(h); return rc; }
  }
  *out = h;
  return warn;
}

int adi_create_dist_local(int nx, int ny, double hh, double dt, double c, int method, int batch, int nranks,
                          adi_handle* out) {
  return adi_create_dist_local_ex(nx, ny, hh, dt, c, method, batch, nranks, ADI_DIST_HALO, out);
}

int adi_create_dist_local_ex(int nx, int ny, double hh, double dt, double c, int method, int batch, int nranks,
                             int mode, adi_handle* out) {
  if (!out || nranks < 1) return ADI_EINVAL;
  for (int r = 0; r < nranks; ++r) out[r] = nullptr;
  if (method == ADI_CFD_FULL && nranks > 1) return ADI_EINVAL;
  if (mode != ADI_DIST_HALO && mode != ADI_DIST_TRANSPOSE) return ADI_EINVAL;
  int warn = ADI_OK;
  for (int r = 0; r < nranks; ++r) {
    int rc = create_rank(nx, ny, hh, dt, c, method, batch, r, nranks, &out[r], mode);
    if (rc < 0) {
      for (int q = 0; q < r; ++q) { adi_destroy(out[q]); out[q] = nullptr; }
      return rc;
    }
    warn = rc;
    out[r]->loop = true;
  }
  for (int r = 0; r < nranks && nranks > 1; ++r) {
    out[r]->peer[0] = r > 0 ? out[r - 1] : nullptr;
    out[r]->peer[1] = r + 1 < nranks ? out[r + 1] : nullptr;
    DevGuard dg_(out[r]);
    int rc;
    if (out[r]->tmode) {
      out[r]->group = new adi_ctx*[nranks];
      for (int q = 0; q < nranks; ++q) out[r]->group[q] = out[q];
      rc = cudaEventCreateWithFlags(&out[r]->ev_pack, cudaEventDisableTiming) == cudaSuccess ? ADI_OK : ADI_ECUDA;
    } else {
      rc = dist_init(out[r]);
    }
    if (rc) {
      for (int q = 0; q < nranks; ++q) { adi_destroy(out[q]); out[q] = nullptr; }
      return rc;
    }
  }
  if (nranks > 1 && out[0]->tmode) tm_fuse_local(out, nranks);
  return warn;
}

int adi_step_dist_local(adi_handle* hs, int nranks, int nsteps) {
  if (!hs || nranks < 1 || nsteps < 0) return ADI_EINVAL;
  for (int r = 0; r < nranks; ++r)
    if (!hs[r] || !hs[r]->loop || hs[r]->nranks != nranks || hs[r]->rank != r) return ADI_EINVAL;
  if (nsteps == 0) return ADI_OK;
  // the collective protocol of adi_step, rank by rank in one thread:
  // every rank's phase runs before any rank's next phase, so no rank waits on another
  const bool ex = nranks > 1;
  auto all = [&](auto fn) -> int {
    for (int r = 0; r < nranks; ++r) {
      DevGuard dg_(hs[r]);
      int rc = fn(hs[r]);
      if (rc) return rc;
    }
    return ADI_OK;
  };
  int rc = ADI_OK;
  if (ex && hs[0]->tmode) {
    // the transpose decomposition: an all-to-all of S after the prologue, every row sweep
    // and every column sweep but the last (each producer records ev_pack first)
    // (fused: the kernels stored S into the owners' arrays; every rank's stream then waits
    // for every other rank's phase -- a barrier -- instead of copying)
    auto mark = [](adi_ctx* h) { return cudaEventRecord(h->ev_pack, h->stream) == cudaSuccess ? ADI_OK : ADI_ECUDA; };
    auto xchg = [](adi_ctx* h, int kind) { return tm_fused_now(h) ? tm_barrier(h) : tm_exchange(h, kind); };
    rc = all([&](adi_ctx* h) { return adi_step_begin(h, nsteps); });
    if (!rc) rc = all(mark);
    if (!rc) rc = all([&](adi_ctx* h) { return xchg(h, 1); });
    for (int k = 0; k < nsteps && !rc; ++k) {
      rc = all([](adi_ctx* h) { return adi_step_rows(h); });
      if (!rc) rc = all(mark);
      if (!rc) rc = all([&](adi_ctx* h) { return xchg(h, 0); });
      if (!rc) rc = all([](adi_ctx* h) { return adi_step_cols(h); });
      if (!rc && k + 1 < nsteps) rc = all(mark);
      if (!rc && k + 1 < nsteps) rc = all([&](adi_ctx* h) { return xchg(h, 1); });
    }
    if (rc) {
      for (int r = 0; r < nranks; ++r) hs[r]->in_call = false;
      return rc;
    }
    return all([](adi_ctx* h) { return adi_step_end(h); });
  }
  if (ex && !hs[0]->fresh) {
    rc = all([](adi_ctx* h) { return dist_pack(h, 1); });
    if (!rc) rc = all([](adi_ctx* h) { return dist_transfer(h, 1); });
    if (!rc) rc = all([](adi_ctx* h) { return dist_unpack(h, 1); });
  }
  if (!rc) rc = all([&](adi_ctx* h) { return adi_step_begin(h, nsteps); });
  for (int k = 0; k < nsteps && !rc; ++k) {
    rc = all([](adi_ctx* h) { return adi_step_rows(h); });
    if (!rc && ex) rc = all([](adi_ctx* h) { return dist_pack(h, 0); });
    if (!rc && ex) rc = all([](adi_ctx* h) { return dist_transfer(h, 0); });
    if (!rc && ex) rc = all([](adi_ctx* h) { return dist_unpack(h, 0); });
    if (!rc) rc = all([](adi_ctx* h) { return adi_step_cols(h); });
  }
  if (rc) {
    for (int r = 0; r < nranks; ++r) { hs[r]->in_call = false; hs[r]->split_wait = nullptr; }
    return rc;
  }
  for (int r = 0; r < nranks; ++r) hs[r]->fresh = false;
  return all([](adi_ctx* h) { return adi_step_end(h); });
}

int adi_dist_info(adi_handle h, int* mode, int* rows0, int* rows1, int* cols0, int* cols1) {
  DevGuard dg_(h);
  if (!h) return ADI_EINVAL;
  const int npy = h->ay.n + 1, npx = h->ax.n + 1;
  if (mode) *mode = h->tmode ? ADI_DIST_TRANSPOSE : ADI_DIST_HALO;
  if (h->tmode) {
    if (rows0) *rows0 = h->ty0;
    if (rows1) *rows1 = std::min(h->ty1, npy);
    if (cols0) *cols0 = h->tx0;
    if (cols1) *cols1 = std::min(h->tx1, npx);
  } else {
    if (rows0) *rows0 = h->band_y0 > h->ay.n ? 0 : h->band_y0;
    if (rows1) *rows1 = std::min(h->band_y1, npy);
    if (cols0) *cols0 = 0;
    if (cols1) *cols1 = npx;
  }
  return ADI_OK;
}

int adi_check_guards(adi_handle h, long long* bad) {
  DevGuard dg_(h);
  if (!h || !bad) return ADI_EINVAL;
  *bad = 0;
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  std::vector<unsigned char> buf(std::max(adi::BUF_GUARD_FRONT, adi::BUF_GUARD_TAIL) * sizeof(double));
  for (auto& a : h->allocs) {
    const char* raw = reinterpret_cast<const char*>(a.first - adi::BUF_GUARD_FRONT);
    const size_t front = adi::BUF_GUARD_FRONT * sizeof(double), tail = adi::BUF_GUARD_TAIL * sizeof(double);
    const char* tailp = reinterpret_cast<const char*>(a.first + a.second);
    for (int part = 0; part < 2; ++part) {
      const size_t nb = part ? tail : front;
      CUDA_TRY(h, cudaMemcpy(buf.data(), part ? tailp : raw, nb, cudaMemcpyDeviceToHost));
      for (size_t k = 0; k < nb; k += 8) {
        bool ok = true;
        for (int j = 0; j < 8; ++j) ok = ok && buf[k + j] == kCanary;
        *bad += !ok;
      }
    }
  }
  return ADI_OK;
}

int adi_band_info(adi_handle h, int* y0, int* y1, int* halo, int* npos) {
  DevGuard dg_(h);
  if (!h) return ADI_EINVAL;
  if (y0) *y0 = h->band_y0 > h->ay.n ? 0 : h->band_y0;
  if (y1) *y1 = std::min(h->band_y1, h->ay.n + 1);
  if (halo) *halo = h->ay.halo;
  if (npos) *npos = h->ay.n + 1;
  return ADI_OK;
}

static int get_fields_impl(adi_handle h, double* U, double* V, double* W, cudaMemcpyKind kind,
                           bool sync = true) {
  DevGuard dg_(h);
  if (!h) return ADI_EINVAL;
  h->err.clear();
  if (!U || !V || !W) return fail(h, ADI_EINVAL, "null field pointer");
  if (h->in_call) return fail(h, ADI_ESTATE, "call in progress");
  const size_t B = (size_t)h->batch;
  if (h->tmode) return tm_get_fields(h, U, V, W, kind, sync);
  int ya, yb;
  field_rows(h, false, &ya, &yb);
  const int off = h->off;
  const int ja = std::max(ya - off, 0), jb = std::min(yb - off, h->nyi);
  const int wa = std::min(ya, h->nyv), wb = std::min(yb, h->nyv);
  for (size_t b = 0; b < B; ++b) {
    CUDA_TRY(h, cudaMemcpy2DAsync(U + b * h->nU + (size_t)ya * h->nxu, h->nxu * 8,
                                  h->U + b * h->aU + (size_t)ya * h->pu, h->pu * 8, h->nxu * 8, yb - ya, kind,
                                  h->stream));
    if (jb > ja)
      CUDA_TRY(h, cudaMemcpy2DAsync(V + b * h->nV + (size_t)ja * h->nxv, h->nxv * 8,
                                    h->V + b * h->aV + (size_t)(ja + off) * h->pv, h->pv * 8, h->nxv * 8, jb - ja,
                                    kind, h->stream));
    // internal W̄^T (columns [wa, wb)) -> W̄ rows via the W2 scratch buffer
    if (wb > wa) {
      double* scratch = cols_raw(h, h->W2);
      int rc = transpose(h, h->W + b * h->aW + (size_t)off * h->pw + wa, scratch, h->nxi, wb - wa, h->pw, h->nxi, 1,
                         0, 0);
      if (rc) return rc;
      CUDA_TRY(h, cudaMemcpyAsync(W + b * h->nW + (size_t)wa * h->nxi, scratch, (size_t)(wb - wa) * h->nxi * 8,
                                  kind, h->stream));
    }
  }
  if (kind == cudaMemcpyDeviceToHost && sync) CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  return ADI_OK;
}

int adi_get_fields(adi_handle h, double* U, double* V, double* W) {
  DevGuard dg_(h);
  return get_fields_impl(h, U, V, W, cudaMemcpyDeviceToHost);
}
int adi_get_fields_async(adi_handle h, double* U, double* V, double* W) {
  DevGuard dg_(h);
  return get_fields_impl(h, U, V, W, cudaMemcpyDeviceToHost, false);
}
int adi_get_fields_device(adi_handle h, double* U, double* V, double* W) {
  DevGuard dg_(h);
  return get_fields_impl(h, U, V, W, cudaMemcpyDeviceToDevice);
}

int adi_get_last_sweeps(adi_handle h, int* k_rows, int* k_cols) {
  DevGuard dg_(h);
  if (!h) return ADI_EINVAL;
  h->err.clear();
  int k[2] = {h->K, h->K};
  if (h->eps > 0.0 && h->d_k && h->m > 0) {
    CUDA_TRY(h, cudaMemcpyAsync(k, h->d_k, sizeof k, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  }
  if (k_rows) *k_rows = k[0];
  if (k_cols) *k_cols = k[1];
  return ADI_OK;
}

int adi_get_stats(adi_handle h, adi_stats* s) {
  DevGuard dg_(h);
  if (!h || !s) return ADI_EINVAL;
  h->err.clear();
  s->steps = h->m;
  s->t = h->m * h->dt;
  s->nonfinite = h->nonfinite;
  s->k_sweeps = h->K;
  s->kernel_launches = h->launches;
  s->device_bytes = h->dev_bytes;
  s->host_launches = h->host_launches;
  s->last_test[0] = s->last_test[1] = -1.0;
  s->last_k[0] = s->last_k[1] = h->K;
  // the stopping rule's test value (Alg. 3/4) at the chosen sweep of the last row and
  // column stage; this synchronizes the handle's stream
  if (h->eps > 0.0 && h->d_norms && h->d_k && h->m > 0 && !h->in_call && h->d_norms_cap >= h->K + 1) {
    std::vector<double> n(4 * (size_t)(h->K + 1));
    int k[2];
    CUDA_TRY(h, cudaMemcpyAsync(n.data(), h->d_norms, n.size() * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaMemcpyAsync(k, h->d_k, sizeof k, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    for (int st = 0; st < 2; ++st) {
      const double* q = n.data() + (size_t)st * 2 * (h->K + 1) + 2 * k[st];
      s->last_k[st] = k[st];
      s->last_test[st] = std::sqrt(q[0]) + std::sqrt(q[1]);
    }
  }
  return ADI_OK;
}

int adi_get_kernel_times(adi_handle h, double* ms, long long* launches, int nkinds) {
  DevGuard dg_(h);
  if (!h || nkinds < 0) return ADI_EINVAL;
  h->err.clear();
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  for (int k = 0; k < nkinds; ++k) {
    if (ms) ms[k] = 0.0;
    if (launches) launches[k] = 0;
  }
  for (auto& r : h->recs) {
    float t = 0.f;
    CUDA_TRY(h, cudaEventElapsedTime(&t, r.a, r.b));
    if (r.kind < nkinds) {
      if (ms) ms[r.kind] += t;
      if (launches) launches[r.kind] += 1;
    }
    h->pool.push_back(r.a);
    h->pool.push_back(r.b);
  }
  h->recs.clear();
  return ADI_OK;
}

int adi_set_trace(adi_handle h, void* dev_buf, long long cap, int kind) {
  DevGuard dg_(h);
  if (!h) return ADI_EINVAL;
  h->err.clear();
  if (dev_buf && (cap < 0 || kind < 0 || kind >= ADI_NKINDS)) return fail(h, ADI_EINVAL, "bad trace arguments");
  if (dev_buf && !ADI_TILE_TRACE)
    return fail(h, ADI_EINVAL, "tile tracing needs a library built with -DADI_TILE_TRACE=1 (tools/build_variant.sh)");
  h->trace = (unsigned long long*)dev_buf;
  h->trace_cap = dev_buf ? cap : 0;
  h->trace_kind = dev_buf ? kind : -1;
  return ADI_OK;
}

const char* adi_last_error(adi_handle h) { return h ? h->err.c_str() : "null handle"; }

void adi_destroy(adi_handle h) {
  DevGuard dg_(h);
  if (!h) return;
  free_ctx(h);
  delete h;
}

}  // extern "C"
