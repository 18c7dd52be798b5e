// FP64 probe for B200 (sm_100a): DFMA latency, peak DFMA throughput, and the
// issue rate of dependent DFMA chains versus resident warps per SM.
// Used to size the ADI line kernels. Not on the product path.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void lat_kernel(double* out, long long* cyc, int iters, double a, double b) {
  double x = out[0];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = fma(x, a, b);
  }
  long long t1 = clock64();
  out[0] = x; cyc[0] = t1 - t0;
}

// CH independent chains per thread
template <int CH>
__global__ void tput_kernel(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#pragma unroll
      for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678) out[blockIdx.x] = s;
}

template <int CH>
double run_tput(int blocks, int threads, int iters, double* d) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  tput_kernel<CH><<<blocks, threads>>>(d, 10, 0.999999, 1e-7);
  cudaEventRecord(e0);
  tput_kernel<CH><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * blocks * threads * (double)iters * 8 * CH;
  return flops / (ms * 1e-3) / 1e12;
}

int main() {
  double* d; long long* c; CK(cudaMalloc(&d, 1 << 20)); CK(cudaMalloc(&c, 64));
  CK(cudaMemset(d, 0, 1 << 20));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  lat_kernel<<<1, 1>>>(d, c, 1000, 0.999, 1e-9); CK(cudaDeviceSynchronize());
  long long h; CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost));
  printf("DFMA dependent latency: %.2f cycles\n", h / 16000.0);
  int iters = 20000;
  printf("peak tput CH=8 blocks=%d x 256: %.2f TFLOP/s\n", sms * 8, run_tput<8>(sms * 8, 256, iters, d));
  printf("peak tput CH=4 blocks=%d x 512: %.2f TFLOP/s\n", sms * 4, run_tput<4>(sms * 4, 512, iters, d));
  // dependent chains: one chain per thread, vary warps per SM (1 block per SM)
  for (int w : {4, 8, 12, 16, 24, 32}) {
    printf("1 chain/thread, %2d warps/SM: %.2f TFLOP/s\n", w, run_tput<1>(sms, w * 32, iters * 4, d));
  }
  for (int w : {4, 8, 16}) {
    printf("2 chains/thread, %2d warps/SM: %.2f TFLOP/s\n", w, run_tput<2>(sms, w * 32, iters * 2, d));
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
