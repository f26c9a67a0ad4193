// Issue-throughput microbenchmark of the softmax instruction mix on sm_100a:
// ops per clock per SM for MUFU.EX2, FFMA2, FFMA, FADD2, F2FP (bf16x2 pack),
// FMNMX3 and the attention softmax's per-pair mix, at 4/8/16 warps per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

__device__ __forceinline__ uint64_t pk(float a, float b) {
  uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r;
}

template <int OP>
__global__ void bench(float* out, long long* cyc, float seed) {
  float v[kChains];
  uint64_t w[kChains];
  uint32_t u[kChains];
  for (int i = 0; i < kChains; ++i) {
    v[i] = seed * (threadIdx.x + i) * 1e-3f;
    w[i] = pk(v[i], v[i] + 1.f);
    u[i] = 0;
  }
  const uint64_t m2 = pk(0.999f, 0.999f), a2 = pk(1e-3f, 1e-3f);
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
      if (OP == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(w[i]) : "l"(m2), "l"(a2));
      if (OP == 2) asm volatile("fma.rn.f32 %0, %0, 0f3F7FBE77, 0f3A83126F;" : "+f"(v[i]));
      if (OP == 3) asm volatile("add.f32x2 %0, %0, %1;" : "+l"(w[i]) : "l"(a2));
      if (OP == 4) {
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v[i]), "f"(v[(i + 1) % kChains]));
        u[i] ^= r;
        asm volatile("" : "+f"(v[i]) : "r"(u[i]));
      }
      if (OP == 5) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(v[(i + 3) % kChains]), "f"(v[(i + 5) % kChains]));
      if (OP == 7) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u[i]));
      if (OP == 8) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u[i]));
      if (OP == 6) {  // softmax pair: FFMA2, 2x MUFU, FADD2, F2FP
        uint64_t x;
        asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(x) : "l"(w[i]), "l"(m2), "l"(a2));
        float x0, x1;
        asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(x0), "=f"(x1) : "l"(x));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x1), "f"(x0));
        u[i] ^= r;
        asm volatile("add.f32x2 %0, %0, %1;" : "+l"(w[i]) : "l"(pk(x0, x1)));
      }
    }
  }
  const long long t1 = clock64();
  float acc = 0.f;
  for (int i = 0; i < kChains; ++i) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(w[i]));
    acc += v[i] + a + b + __uint_as_float(u[i]);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int ops_per_chain_iter, int sms) {
  float* out; long long* cyc;
  cudaMalloc(&out, sms * 1024 * 4);
  cudaMalloc(&cyc, sms * 8);
  for (int warps : {4, 8, 16, 32}) {
    bench<OP><<<sms, warps * 32>>>(out, cyc, 1.0f);
    bench<OP><<<sms, warps * 32>>>(out, cyc, 1.0f);
    cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double ops = double(kIters) * kChains * ops_per_chain_iter * warps * 32;
    printf("%-8s warps/SM=%2d  %7.2f ops/clk/SM  (%lld cycles)\n", name, warps, ops / c, c);
  }
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("ex2", 1, sms);
  run<1>("ffma2", 2, sms);
  run<2>("ffma", 1, sms);
  run<3>("fadd2", 2, sms);
  run<4>("f2fp", 2, sms);
  run<5>("fmnmx3", 1, sms);
  run<6>("sm_pair", 2, sms);  // values (exp) per clock
  run<7>("ex2bf16x2", 2, sms);
  run<8>("ex2f16x2", 2, sms);
  return 0;
}
