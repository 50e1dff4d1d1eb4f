// Microbenchmark: fp64 DMMA (mma.sync .f64) vs DFMA throughput on sm_100a.
// Measurement tool only (not on the product path). Prints TFLOP/s per variant.
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[ACC][2];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ACC>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
  double c[ACC][4];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ACC>
__global__ void dfma_loop(double* out, int iters) {
  double x[ACC];
  double m = 1.0000001, a = 1e-9 * threadIdx.x;
#pragma unroll
  for (int i = 0; i < ACC; ++i) x[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) x[i] = fma(x[i], m, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * 148 * 64 * 1024);
  const int iters = 4096;
  for (int bpsm : {1, 2, 4}) {
    for (int threads : {128, 256, 512}) {
      int grid = sms * bpsm;
      float ms = timeit([&] { dmma_m8n8k4<8><<<grid, threads>>>(out, iters); });
      double fl = double(grid) * (threads / 32) * iters * 8 * 512.0;
      printf("dmma m8n8k4   grid=%d thr=%d : %.2f TFLOP/s\n", grid, threads, fl / ms / 1e9);
      ms = timeit([&] { dmma_m16n8k16<4><<<grid, threads>>>(out, iters / 4); });
      fl = double(grid) * (threads / 32) * (iters / 4) * 4 * (16 * 8 * 16 * 2.0);
      printf("dmma m16n8k16 grid=%d thr=%d : %.2f TFLOP/s\n", grid, threads, fl / ms / 1e9);
      ms = timeit([&] { dfma_loop<8><<<grid, threads>>>(out, iters); });
      fl = double(grid) * threads * iters * 8 * 2.0;
      printf("dfma          grid=%d thr=%d : %.2f TFLOP/s\n", grid, threads, fl / ms / 1e9);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
