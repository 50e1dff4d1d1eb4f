// Microbenchmark: legacy-path tensor throughput on sm_100a (HMMA via mma.sync) for tf32 and
// bf16, and fp32 SIMT (FFMA / FFMA2).  Measurement tool only (not on the product path): it
// decides whether a per-matrix fp32 kernel can run its products on mma.sync instead of
// tcgen05.  Prints TFLOP/s per variant.
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void hmma_tf32_m16n8k8(float* out, int iters) {
  unsigned a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
#pragma unroll
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(1.0f + threadIdx.x * 1e-4f + i);
  float c[ACC][4];
#pragma unroll
  for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};\n"
          : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ACC>
__global__ void hmma_bf16_m16n8k16(float* out, int iters) {
  unsigned a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = 0x3f803f80u + threadIdx.x + i;
#pragma unroll
  for (int i = 0; i < 2; ++i) b[i] = 0x3f803f80u + threadIdx.x * 3 + i;
  float c[ACC][4];
#pragma unroll
  for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};\n"
          : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ACC>
__global__ void ffma2_loop(float* out, int iters) {
  float2 x[ACC];
  const float2 m = make_float2(1.0000001f, 0.9999999f), a = make_float2(1e-9f * threadIdx.x, 2e-9f);
#pragma unroll
  for (int i = 0; i < ACC; ++i) x[i] = make_float2(i, i + 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) {
      unsigned long long xv = *reinterpret_cast<unsigned long long*>(&x[i]);
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;\n"
                   : "+l"(xv)
                   : "l"(*reinterpret_cast<const unsigned long long*>(&m)),
                     "l"(*reinterpret_cast<const unsigned long long*>(&a)));
      x[i] = *reinterpret_cast<float2*>(&xv);
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += x[i].x + x[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * 148 * 64 * 1024);
  const int iters = 4096;
  for (int bpsm : {1, 2}) {
    for (int threads : {128, 256, 512}) {
      const int grid = sms * bpsm;
      float ms = timeit([&] { hmma_tf32_m16n8k8<8><<<grid, threads>>>(out, iters); });
      double fl = double(grid) * (threads / 32) * iters * 8 * (16 * 8 * 8 * 2.0);
      printf("hmma tf32 m16n8k8   grid=%d thr=%d : %.1f TFLOP/s\n", grid, threads, fl / ms / 1e9);
      ms = timeit([&] { hmma_bf16_m16n8k16<8><<<grid, threads>>>(out, iters); });
      fl = double(grid) * (threads / 32) * iters * 8 * (16 * 8 * 16 * 2.0);
      printf("hmma bf16 m16n8k16  grid=%d thr=%d : %.1f TFLOP/s\n", grid, threads, fl / ms / 1e9);
      ms = timeit([&] { ffma2_loop<8><<<grid, threads>>>(out, iters); });
      fl = double(grid) * threads * iters * 8 * 4.0;
      printf("ffma2               grid=%d thr=%d : %.1f TFLOP/s\n", grid, threads, fl / ms / 1e9);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
