// Contention microbenchmark for the ring-attention MMA mix on sm_100a: the
// tensor-core rate of the K1 step pattern (per step and query tile: 8 SS
// MMAs M=128 N=128 K=16 for S = Q.K^T, 8 TS MMAs N=128 for O += P.V) alone,
// and with the other traffic of the real kernel running on other warps:
//   tmem : 4 warps re-reading 128 S columns and storing 64 P columns per step
//          (tcgen05.ld/st, the softmax's TMEM traffic),
//   smem : one warp streaming 16-byte st.shared (64 KB per step, the TMA
//          K/V writes' shared-memory bandwidth),
//   tma  : real TMA loads of 2 x 32 KB tiles per step from global memory.
// Prints FLOP/clk/SM of the MMAs. One CTA per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2404_09526_b200/csrc/kernels -o umma_mix umma_mix.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"

using namespace esp;

constexpr int kSteps = 400;

template <bool kTmem, bool kSmem, bool kTma>
__global__ void __launch_bounds__(256, 1)
    bench(long long* cyc, const __grid_constant__ CUtensorMap tm) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t bar, tbar;
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < (160 * 1024) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::mbar_init(&tbar, 1);
    ptx::fence_barrier_init();
    stop = 0;
  }
  if (threadIdx.x < 32) ptx::tmem_alloc<512>(&slot);
  ptx::fence_async_shared();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    const bool leader = ptx::elect_one();
    constexpr uint32_t idesc_s = ptx::make_idesc_bf16(128, 128, false, false);
    constexpr uint32_t idesc_o = ptx::make_idesc_bf16(128, 128, false, true);
    const uint32_t q0 = ptx::smem_u32(smem), k0 = ptx::smem_u32(smem + 32768),
                   v0 = ptx::smem_u32(smem + 65536);
    uint32_t phase = 0;
    const long long t0 = clock64();
    for (int st = 0; st < kSteps; ++st) {
#pragma unroll
      for (int t = 0; t < 2; ++t) {  // two query tiles per step, as in K1 v2
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // O_t += P_t V
          const uint64_t dv = ptx::make_sdesc_sw128(v0 + k * 2048, 128 * 128, 1024);
          if (leader) ptx::umma_f16_ts(tmem + 256 + t * 128, tmem + t * 128 + k * 8, dv, idesc_o, 1);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // S_t = Q_t K^T
          const uint32_t off = (k >> 2) * (128 * 128) + (k & 3) * 32;
          const uint64_t da = ptx::make_sdesc_sw128(q0 + off, 16, 1024);
          const uint64_t db = ptx::make_sdesc_sw128(k0 + off, 16, 1024);
          if (leader) ptx::umma_f16_ss(tmem + t * 128, da, db, idesc_s, k != 0);
        }
      }
      if (leader) ptx::tc_commit(&bar);
      __syncwarp();
      ptx::mbar_wait(&bar, phase);
      phase ^= 1;
    }
    const long long t1 = clock64();
    if (lane == 0) {
      cyc[blockIdx.x] = t1 - t0;
      stop = 1;
    }
  } else if (warp == 1 && kTma) {
    if (lane == 0) {
      uint32_t ph = 0;
      uint8_t* dst = smem + 98304;
      int row = blockIdx.x * 256;
      while (!stop) {
        ptx::mbar_expect_tx(&tbar, 2 * 32768);
        for (int b = 0; b < 2; ++b) {
          for (int h = 0; h < 2; ++h) {
            ptx::tma_load_2d(dst + b * 32768 + h * 16384, &tm, &tbar, h * 64, row);
          }
        }
        ptx::mbar_wait(&tbar, ph);
        ph ^= 1;
        row = (row + 128) % (148 * 1024);
      }
    }
  } else if (warp == 1 && kSmem) {
    uint4* dst = reinterpret_cast<uint4*>(smem + 98304);
    int i = 0;
    while (!stop) {
#pragma unroll 8
      for (int k = 0; k < 64; ++k) {
        dst[(i + k * 32 + lane) & 4095] = make_uint4(k, i, 0, 0);
      }
      i += 2048;
    }
  } else if (warp >= 4 && kTmem) {
    const uint32_t lane_off = ((warp & 3) * 32) << 16;
    int t = 0;
    while (!stop) {
      uint32_t s[32];
      for (int c = 0; c < 128; c += 32) {
        ptx::tmem_ld_32x32b_x32(tmem + 448 + lane_off, s);  // S-like reads (unused cols)
        ptx::tmem_wait_ld();
      }
      for (int c = 0; c < 2; ++c) {
        ptx::tmem_st_32x32b_x32(tmem + 480 + lane_off, s);  // P-like stores
        ptx::tmem_wait_st();
      }
      ++t;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

template <bool A, bool B, bool C>
void run(const char* name, int sms, long long* cyc, const CUtensorMap& tm) {
  cudaFuncSetAttribute(bench<A, B, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, 170000);
  bench<A, B, C><<<sms, 256, 170000>>>(cyc, tm);
  bench<A, B, C><<<sms, 256, 170000>>>(cyc, tm);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double flop = 2.0 * 128 * 128 * 16 * 32.0 * kSteps;
  printf("%-22s %8.1f FLOP/clk/SM (%5.1f%% of 8070; %.0f cycles per 2-tile step) %s\n", name,
         flop / c, 100.0 * flop / c / 8070.0, double(c) / kSteps, cudaGetErrorString(e));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  cudaMalloc(&cyc, sms * 8);
  void* g;
  const size_t rows = 148 * 1024 + 256;
  cudaMalloc(&g, rows * 128 * 2);
  cudaMemset(g, 0, rows * 128 * 2);
  CUtensorMap tm;
  const cuuint64_t dims[2] = {128, rows};
  const cuuint64_t strides[1] = {256};
  const cuuint32_t box[2] = {64, 128};
  const cuuint32_t es[2] = {1, 1};
  cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  run<false, false, false>("mma mix alone", sms, cyc, tm);
  run<true, false, false>("+ softmax TMEM ld/st", sms, cyc, tm);
  run<false, true, false>("+ smem stores", sms, cyc, tm);
  run<false, false, true>("+ TMA loads", sms, cyc, tm);
  run<true, false, true>("+ TMEM + TMA", sms, cyc, tm);
  return 0;
}
