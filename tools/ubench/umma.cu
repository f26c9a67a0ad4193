// tcgen05.mma issue-throughput microbenchmark on sm_100a: FLOP/clk/SM of
// back-to-back kind::f16 MMAs (M=128, K=16) for N = 64/128/256 with both
// operands in shared memory (SS) and with A in tensor memory (TS). Operand
// contents are irrelevant (zeros). One CTA per SM, one elected issuing thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2404_09526_b200/csrc/kernels -o umma umma.cu
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"

using namespace esp;

template <int N, bool kTS>
__global__ void __launch_bounds__(128, 1) bench(long long* cyc, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc<512>(&slot);
  ptx::fence_async_shared();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  long long t0 = 0, t1 = 0;
  if (threadIdx.x < 32) {
    const bool leader = ptx::elect_one();
    constexpr uint32_t idesc = ptx::make_idesc_bf16(128, N, false, false);
    const uint32_t a0 = ptx::smem_u32(smem), b0 = ptx::smem_u32(smem + 32768);
    uint32_t phase = 0;
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 64; ++k) {
        const uint64_t db = ptx::make_sdesc_sw128(b0 + (k & 3) * 32, 16, 1024);
        if (kTS) {
          if (leader) ptx::umma_f16_ts(tmem + 256, tmem + 384 + (k & 3) * 8, db, idesc, 1);
        } else {
          const uint64_t da = ptx::make_sdesc_sw128(a0 + (k & 3) * 32, 16, 1024);
          if (leader) ptx::umma_f16_ss(tmem, da, db, idesc, 1);
        }
      }
      if (leader) ptx::tc_commit(&bar);
      __syncwarp();
      ptx::mbar_wait(&bar, phase);
      phase ^= 1;
    }
    t1 = clock64();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int N, bool kTS>
void run(int sms, long long* cyc) {
  const int iters = 2000;
  cudaFuncSetAttribute(bench<N, kTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  bench<N, kTS><<<sms, 128, 70000>>>(cyc, 10);
  bench<N, kTS><<<sms, 128, 70000>>>(cyc, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double flop = 2.0 * 128 * N * 16 * 64.0 * iters;
  printf("%s N=%3d  %8.1f FLOP/clk/SM  (%.1f cycles per MMA) %s\n", kTS ? "TS" : "SS", N, flop / c,
         double(c) / (64.0 * iters), cudaGetErrorString(e));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  cudaMalloc(&cyc, sms * 8);
  run<64, false>(sms, cyc);
  run<128, false>(sms, cyc);
  run<256, false>(sms, cyc);
  run<64, true>(sms, cyc);
  run<128, true>(sms, cyc);
  return 0;
}
