// microbenchmark (diagnostic): issue rate of FFMA vs FFMA2 (packed f32x2) per SM sub-partition
#include <cstdio>
#include <cuda_runtime.h>
template <int V>
__global__ void k(float* out, int iters, long long* cyc) {
  float a[8], b = 1.0000001f, c = 1e-7f;
  float2 a2[8], b2 = make_float2(b, b), c2 = make_float2(c, c);
  for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x + j; a2[j] = make_float2(a[j], a[j] + 1); }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (V == 0) a[j] = fmaf(a[j], b, c);
      else a2[j] = __ffma2_rn(a2[j], b2, c2);
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 8; ++j) s += (V == 0 ? a[j] : a2[j].x + a2[j].y);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 1 << 24); cudaMalloc(&c, 8);
  for (int nw : {4, 8, 16, 32}) {
    for (int v = 0; v < 2; ++v) {
      int it = 4096;
      if (v == 0) k<0><<<148, nw * 32>>>(o, it, c); else k<1><<<148, nw * 32>>>(o, it, c);
      cudaDeviceSynchronize();
      if (v == 0) k<0><<<148, nw * 32>>>(o, it, c); else k<1><<<148, nw * 32>>>(o, it, c);
      long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      double winst = (double)it * 8 * nw / 4;  // warp-instructions per SMSP
      printf("warps/SM %2d %s: %.2f cycles per warp-instruction per SMSP (%.2f fp32 lanes-op/cyc/SMSP)\n", nw,
             v ? "FFMA2" : "FFMA ", h / winst, 32.0 * (v ? 2 : 1) * winst / h);
    }
  }
  return 0;
}
