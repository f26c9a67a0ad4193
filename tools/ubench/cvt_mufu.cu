// Pipe-sharing microbenchmark for the ring-attention softmax on sm_100a: does
// the fp32 -> bf16x2 pack (cvt.rn.bf16x2.f32, SASS F2FP) issue to the same
// pipe as ex2.approx (MUFU.EX2)? Times, per SM, loops of
//   ex2 only | cvt only | ex2 + cvt (softmax ratio: 1 pack per 2 ex2)
//   | ex2 + integer-rounded pack (IADD + PRMT, no F2FP)
//   | pack + ex2.approx.ftz.bf16x2 (one MUFU op per pair?) + unpack
//   | the same with ex2.approx.f16x2
// with 8 warps per SM (the two softmax warpgroups). If F2FP rides the MUFU
// pipe the mixed loop costs the sum of the two alone.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cvt_mufu cvt_mufu.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

constexpr int kIters = 4096;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t cvt_pack(float lo, float hi) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// round-half-up on the bit pattern, then take the two high halves
__device__ __forceinline__ uint32_t int_pack(float lo, float hi) {
  const uint32_t a = __float_as_uint(lo) + 0x8000u, b = __float_as_uint(hi) + 0x8000u;
  uint32_t r;
  asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

__device__ __forceinline__ uint32_t ex2_bf16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

__device__ __forceinline__ uint32_t ex2_f16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) bench(float* out, long long* cyc, float seed) {
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = seed * (threadIdx.x + i) * 1e-3f;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      float a = v[i], b = v[i + 1];
      if (MODE == 0 || MODE == 2 || MODE == 3) {
        a = ex2(a);
        b = ex2(b);
      }
      if (MODE == 1 || MODE == 2) acc ^= cvt_pack(a, b);
      if (MODE == 3) acc ^= int_pack(a, b);
      if (MODE == 5) {  // f16x2 pack, one f16x2 ex2 for the pair, unpack
        __half2 h = __floats2half2_rn(a, b);
        const uint32_t p = ex2_f16x2(*reinterpret_cast<uint32_t*>(&h));
        const __half2 q = *reinterpret_cast<const __half2*>(&p);
        a = __low2float(q);
        b = __high2float(q);
      }
      if (MODE == 4) {  // pack, one bf16x2 ex2 for the pair, unpack
        const uint32_t p = ex2_bf16x2(cvt_pack(a, b));
        a = __uint_as_float(p << 16);
        b = __uint_as_float(p & 0xffff0000u);
      }
      v[i] = a * -0.5f;
      v[i + 1] = b * -0.5f;
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int sms, float* out, long long* cyc) {
  bench<MODE><<<sms, 256>>>(out, cyc, 1.f);
  bench<MODE><<<sms, 256>>>(out, cyc, 1.f);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double pairs = 256.0 * kIters * 8;  // value pairs per SM
  printf("%-28s %7.0f cycles  %6.2f pairs/clk/SM  %s\n", name, double(c), pairs / c,
         cudaGetErrorString(e));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* cyc;
  cudaMalloc(&out, sms * 256 * 4);
  cudaMalloc(&cyc, sms * 8);
  run<0>("ex2 x2", sms, out, cyc);
  run<1>("cvt.rn.bf16x2 (F2FP)", sms, out, cyc);
  run<2>("ex2 x2 + F2FP", sms, out, cyc);
  run<3>("ex2 x2 + IADD/PRMT pack", sms, out, cyc);
  run<4>("F2FP + ex2.bf16x2 + unpack", sms, out, cyc);
  run<5>("F2FP + ex2.f16x2 + unpack", sms, out, cyc);
  return 0;
}
