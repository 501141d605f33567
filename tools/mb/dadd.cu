#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, double x, int n, long long* cyc) {
  double r = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    r = __dadd_rn(r, x);
    r = __dadd_rn(r, -x * 0.5);
    r = __dadd_rn(r, x * 0.25);
    r = __dadd_rn(r, -x * 0.125);
  }
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = r;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
__global__ void fchain(float* out, float x, int n, long long* cyc) {
  float r = threadIdx.x * 1e-3f;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    r = __fadd_rn(r, x);
    r = __fadd_rn(r, -x * 0.5f);
    r = __fadd_rn(r, x * 0.25f);
    r = __fadd_rn(r, -x * 0.125f);
  }
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = r;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* o; float* fo; long long* c; long long h;
  cudaMalloc(&o, 1 << 20); cudaMalloc(&fo, 1 << 20); cudaMalloc(&c, 8);
  int n = 100000;
  for (int warps : {1, 4, 16}) {
    chain<<<1, 32 * warps>>>(o, 1.5, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("dadd chain, %d warps/CTA: %.2f cycles per dependent DADD\n", warps, double(h) / (4.0 * n));
  }
  fchain<<<1, 32>>>(fo, 1.5f, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("fadd chain: %.2f cycles per dependent FADD\n", double(h) / (4.0 * n));
  return 0;
}
