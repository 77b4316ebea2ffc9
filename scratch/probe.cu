#include <cstdio>
#include <cuda_runtime.h>
__global__ void ddiv_k(const double* a, double* out, int iters, double b) {
  double x = a[threadIdx.x + blockIdx.x*blockDim.x];
  double acc = 0;
  for (int i = 0; i < iters; ++i) { acc += x / b; x += 1.0; }
  out[threadIdx.x + blockIdx.x*blockDim.x] = acc;
}
__global__ void dsqrt_k(const double* a, double* out, int iters) {
  double x = a[threadIdx.x + blockIdx.x*blockDim.x];
  double acc = 0;
  for (int i = 0; i < iters; ++i) { acc += sqrt(x); x += 1.0; }
  out[threadIdx.x + blockIdx.x*blockDim.x] = acc;
}
__global__ void dfma_k(const double* a, double* out, int iters) {
  double x = a[threadIdx.x + blockIdx.x*blockDim.x], y = x*0.5, z = x*0.25, w = x*0.125;
  for (int i = 0; i < iters; ++i) { x = fma(x, 1.0000001, 0.5); y = fma(y, 1.0000001, 0.5); z = fma(z, 1.0000001, 0.5); w = fma(w, 1.0000001, 0.5);}
  out[threadIdx.x + blockIdx.x*blockDim.x] = x+y+z+w;
}
__global__ void i2f_k(const long long* a, double* out, int iters) {
  long long x = a[threadIdx.x + blockIdx.x*blockDim.x];
  double acc = 0;
  for (int i = 0; i < iters; ++i) { acc += (double)x; x += 3; }
  out[threadIdx.x + blockIdx.x*blockDim.x] = acc;
}
int main() {
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("%s SMs=%d cc=%d.%d l2=%d smem/blk optin=%zu clock=%d memclk=%d busw=%d\n", p.name, p.multiProcessorCount, p.major, p.minor, p.l2CacheSize, p.sharedMemPerBlockOptin, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  int n = 148*8*256; double *a, *o; long long* ai;
  cudaMalloc(&a, n*8); cudaMalloc(&o, n*8); cudaMalloc(&ai, n*8); cudaMemset(a, 0, n*8); cudaMemset(ai, 0, n*8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int it = 4096;
  for (int rep = 0; rep < 2; ++rep) {
  cudaEventRecord(e0); ddiv_k<<<148*8,256>>>(a,o,it,3.7); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
  printf("ddiv: %.3f G/s\n", (double)n*it/ms/1e6);
  cudaEventRecord(e0); dsqrt_k<<<148*8,256>>>(a,o,it); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
  printf("dsqrt: %.3f G/s\n", (double)n*it/ms/1e6);
  cudaEventRecord(e0); dfma_k<<<148*8,256>>>(a,o,it); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
  printf("dfma: %.3f G/s (x4)\n", 4.0*n*it/ms/1e6);
  cudaEventRecord(e0); i2f_k<<<148*8,256>>>(ai,o,it); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
  printf("i2f64: %.3f G/s\n", (double)n*it/ms/1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
