// Does cuTensorMapEncodeTiled accept an overlapping-row view, and does a TMA
// tensor load of it produce the padded (34-double rows) staging layout?
//   view: d0 = 34 doubles (inner), d1 = pair offset (stride 16 B),
//         d2 = 32-position chunk (stride 256 B), d3 = line, d4 = batch
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_overlap tma_overlap.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct Params {
  CUtensorMap tm;
  int c1, c2, c3, c4;
  double* out;
};

__global__ void load_kernel(const __grid_constant__ Params P) {
  __shared__ alignas(128) double sm[32 * 34];
  __shared__ alignas(8) unsigned long long bar;
  const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
  const unsigned sd = (unsigned)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(32 * 34 * 8));
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4, %5, %6}], [%7];" ::"r"(sd),
        "l"((uint64_t)&P.tm), "r"(0), "r"(P.c1), "r"(P.c2), "r"(P.c3), "r"(P.c4), "r"(sb)
        : "memory");
  }
  __syncwarp();
  unsigned ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(sb));
  }
  for (int i = threadIdx.x; i < 32 * 34; i += 32) P.out[i] = sm[i];
}

int main() {
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
  const int P0 = 1024, pitch = 2048 + 64, nl = 4, guard = 2048;
  const size_t total = guard + (size_t)nl * pitch + guard;
  std::vector<double> h(total, -1.0);
  for (int l = 0; l < nl; ++l)
    for (int p = 0; p < pitch; ++p) h[guard + (size_t)l * pitch + p] = l * 1e5 + p;
  double *d, *o;
  cudaMalloc(&d, total * 8);
  cudaMalloc(&o, 32 * 34 * 8);
  cudaMemcpy(d, h.data(), total * 8, cudaMemcpyHostToDevice);
  double* base = d + guard - P0;  // position -P0 of line 0
  CUtensorMap tm;
  cuuint64_t dims[5] = {34, 16, (cuuint64_t)((pitch + P0) / 32), (cuuint64_t)nl, 1};
  cuuint64_t strides[4] = {16, 256, (cuuint64_t)pitch * 8, (cuuint64_t)nl * pitch * 8};
  cuuint32_t box[5] = {34, 1, 32, 1, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode overlapping view: %d\n", (int)r);
  if (r) return 2;
  int bad = 0, tests = 0;
  const int starts[] = {0, 2, 30, 34, 96, 1000, -4, -30, -64};
  for (int line = 0; line < nl + 1; ++line)
    for (int s0 : starts) {
      Params P;
      P.tm = tm;
      const int sh = s0 + P0;
      P.c1 = (sh & 31) >> 1; P.c2 = sh >> 5; P.c3 = line; P.c4 = 0; P.out = o;
      load_kernel<<<1, 32>>>(P);
      std::vector<double> g(32 * 34);
      cudaError_t e = cudaMemcpy(g.data(), o, g.size() * 8, cudaMemcpyDeviceToHost);
      if (e) { printf("cuda error %s\n", cudaGetErrorString(e)); return 3; }
      for (int j = 0; j < 32; ++j)
        for (int k = 0; k < 34; ++k) {
          const long long pos = (long long)s0 + 32 * j + k;
          double want;
          if (line >= nl) want = 0.0;  // OOB line: zero fill
          else {
            const long long off = guard + (long long)line * pitch + pos;
            want = (off >= 0 && off < (long long)total) ? h[off] : 0.0;
          }
          ++tests;
          if (g[j * 34 + k] != want) {
            if (bad < 10) printf("line %d s0 %d row %d k %d: got %g want %g\n", line, s0, j, k, g[j * 34 + k], want);
            ++bad;
          }
        }
    }
  printf("overlap TMA view: %d / %d mismatches\n", bad, tests);
  return bad ? 4 : 0;
}
