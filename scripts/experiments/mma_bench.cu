// Microbenchmark: issue rate of tcgen05.mma (cta_group::1, M=128) per kind,
// operand source and N -- the tile-shape decision of k_conv_tc rests on it.
// One CTA per SM; thread 0 issues ITERS MMAs into two alternating TMEM
// accumulators over K-offsets of a 32 KB swizzled operand buffer, commits,
// waits, and reports clock64 cycles per MMA.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_bench scripts/mma_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

template <int KIND>  // 0 tf32 SS, 1 tf32 TS (A in TMEM), 2 bf16 SS
__device__ __forceinline__ void mma(uint32_t d, uint64_t da, uint32_t ta, uint64_t db, uint32_t idesc,
                                    uint32_t acc) {
  if constexpr (KIND == 0) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(da), "l"(db), "r"(idesc), "r"(acc));
  } else if constexpr (KIND == 1) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(ta), "l"(db), "r"(idesc), "r"(acc));
  } else {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(da), "l"(db), "r"(idesc), "r"(acc));
  }
}

template <int KIND, int N, int ALT = 0, int CONT = 0>
__global__ void __launch_bounds__(256, 1) k_bench(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(buf)[i] = 0x3f800000u ^ (i * 2654435761u & 0x007fffffu);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (CONT && threadIdx.x >= 128) {
    // contention warps 4..7 (TMEM lanes 32*(w-4)..): until the MMA thread is done
    const int w = threadIdx.x / 32 - 4;
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(1.0f + i);
    const uint32_t ta = tmem + (uint32_t(w * 32) << 16) + 320u;
    uint32_t acc = 0;
    while (!stop) {
      if (CONT == 1) {
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
            "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
            "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(ta),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
            "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
            "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
            "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
            "r"(v[29]), "r"(v[30]), "r"(v[31])
            : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      } else if (CONT == 3) {
        // the 3xTF32 split: cvt.rna.tf32.f32 + fsub
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          uint32_t h;
          asm volatile("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(__uint_as_float(v[i])));
          v[i] = __float_as_uint(__uint_as_float(v[i]) - __uint_as_float(h)) + 0x3f800000u;
        }
      } else if (CONT == 4) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(fmaf(__uint_as_float(v[i]), 1.0001f, 0.5f));
      } else {
        const uint32_t row = smem_u32(buf + 49152 + (threadIdx.x - 128) * 128);
        for (int c = 0; c < 8; ++c) {
          uint32_t x0, x1, x2, x3;
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3) : "r"(row + uint32_t(c << 4)));
          acc += x0 ^ x1 ^ x2 ^ x3;
        }
      }
    }
    if (acc == 12345 || v[3] == 12345u) out[0] = acc;
  }
  if (threadIdx.x == 0) {
    constexpr uint32_t afmt = KIND == 2 ? 1u : 2u;  // bf16 = 1, tf32 = 2
    constexpr uint32_t idesc = (1u << 4) | (afmt << 7) | (afmt << 10) |
                               (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint64_t da = sw128_desc(smem_u32(buf));
    const uint64_t db = sw128_desc(smem_u32(buf + 16384));
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      // one accumulator at columns [0, N), as a conv tile's K loop; the TS
      // A operand at columns [256, 288)
      const uint64_t koff = uint64_t((i & 3) * 32) >> 4;
      // ALT: alternate two accumulators (columns 0 / 128) and two A tiles,
      // as two M tiles sharing one B
      const uint32_t dcol = ALT ? uint32_t(i & 1) * 128u : 0u;
      const uint64_t aoff = ALT ? uint64_t((i & 1) * 8192) >> 4 : 0;
      mma<KIND>(tmem + dcol, da + koff + aoff, tmem + 256u + 8u * uint32_t(i & 3) + (ALT ? 32u * (i & 1) : 0u),
                db + koff, idesc, i > 1);
    }
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&bar))
        : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
        "@!P1 bra W;\n\t}" ::"r"(smem_u32(&bar))
        : "memory");
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int KIND, int N, int ALT = 0, int CONT = 0>
void run(const char* name, int ctas) {
  const int iters = 4096;
  long long* d;
  cudaMalloc(&d, ctas * sizeof(long long));
  const size_t smem = 97 * 1024;
  cudaFuncSetAttribute(k_bench<KIND, N, ALT, CONT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k_bench<KIND, N, ALT, CONT><<<ctas, 256, smem>>>(iters, d);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_bench<KIND, N, ALT, CONT><<<ctas, 256, smem>>>(iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, d, ctas * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < ctas; ++i) avg += double(h[i]) / ctas;
  const int kk = KIND == 2 ? 16 : 8;
  const double macs = 128.0 * N * kk;
  const double flops = 2.0 * macs * iters * ctas;
  printf("%-10s%s%s N=%3d ctas=%3d  %6.1f cyc/MMA  %6.0f MAC/clk/SM  %7.1f TFLOP/s  %s\n", name, ALT ? " alt" : "    ", CONT == 1 ? " +tmem.st" : CONT == 2 ? " +ld.shr " : CONT == 3 ? " +cvt.tf32" : CONT == 4 ? " +ffma   " : "         ", N,
         ctas, avg / iters, macs / (avg / iters), flops / (ms * 1e-3) / 1e12,
         err == cudaSuccess ? "" : cudaGetErrorString(err));
  cudaFree(d);
}

// cta_group::2 pair: M=256 (128 rows per CTA), N total, A in TMEM (TS) or
// smem (SS), B halves of N/2 rows in each CTA's smem at the same offset.
template <int N, bool TS, int CONT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) k_pair(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int stop;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(buf)[i] = 0x3f800000u ^ (i * 2654435761u & 0x007fffffu);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  if (CONT && threadIdx.x >= 128) {
    uint32_t acc = 0;
    while (!stop) {
      const uint32_t row = smem_u32(buf + 65536 + (threadIdx.x - 128) * 128);
      for (int c = 0; c < 8; ++c) {
        uint32_t x0, x1, x2, x3;
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3) : "r"(row + uint32_t(c << 4)));
        acc += x0 ^ x1 ^ x2 ^ x3;
      }
    }
    if (acc == 12345) out[0] = acc;
  }
  if (threadIdx.x == 0 && rank == 0) {
    constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) |
                               (uint32_t(256 >> 4) << 24);
    const uint64_t da = sw128_desc(smem_u32(buf));
    const uint64_t db = sw128_desc(smem_u32(buf + 16384));
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t koff = uint64_t((i & 3) * 32) >> 4;
      const uint32_t acc = i > 0;
      if (TS) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                     "r"(tmem + 256u + 8u * uint32_t(i & 3)), "l"(db + koff), "r"(idesc), "r"(acc));
      } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(da + koff), "l"(db + koff), "r"(idesc), "r"(acc));
      }
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)), "h"(uint16_t(3))
        : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
        "@!P1 bra W;\n\t}" ::"r"(smem_u32(&bar))
        : "memory");
    out[blockIdx.x / 2] = clock64() - t0;
  }
  if (threadIdx.x == 0 && rank == 1) {
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
        "@!P1 bra W;\n\t}" ::"r"(smem_u32(&bar))
        : "memory");
  }
  if (threadIdx.x == 0) stop = 1;
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, bool TS, int CONT>
void run_pair(int ctas) {
  const int iters = 4096;
  long long* d;
  cudaMalloc(&d, ctas * sizeof(long long));
  const size_t smem = 97 * 1024;
  cudaFuncSetAttribute(k_pair<N, TS, CONT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k_pair<N, TS, CONT><<<ctas, 256, smem>>>(iters, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_pair<N, TS, CONT><<<ctas, 256, smem>>>(iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, d, ctas / 2 * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < ctas / 2; ++i) avg += double(h[i]) / (ctas / 2);
  const double macs = 256.0 * N * 8;
  printf("pair tf32 %s%s N=%3d ctas=%3d  %6.1f cyc/MMA  %6.0f MAC/clk/SM  %7.1f TFLOP/s  %s\n",
         TS ? "TS" : "SS", CONT ? " +ld.shr" : "        ", N, ctas, avg / iters,
         macs / 2 / (avg / iters), 2.0 * macs * iters * (ctas / 2) / (ms * 1e-3) / 1e12,
         err == cudaSuccess ? "" : cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  run_pair<64, true, 0>(148);
  run_pair<64, false, 0>(148);
  run_pair<128, true, 0>(148);
  run_pair<256, true, 0>(148);
  run_pair<128, false, 0>(148);
  run_pair<256, false, 0>(148);
  run_pair<128, true, 1>(148);
  run_pair<256, true, 1>(148);
  run<1, 128, 0, 2>("tf32 TS", 148);
  return 0;
  for (int ctas : {148}) {
    run<1, 128, 0, 3>("tf32 TS", ctas);
    run<1, 128, 0, 4>("tf32 TS", ctas);
    run<1, 128, 0, 1>("tf32 TS", ctas);
    run<1, 128, 0, 2>("tf32 TS", ctas);
    run<1, 64, 0, 1>("tf32 TS", ctas);
    run<0, 128, 0, 2>("tf32 SS", ctas);
    run<0, 128, 0, 1>("tf32 SS", ctas);
    run<0, 64>("tf32 SS", ctas);
    run<0, 128>("tf32 SS", ctas);
    run<0, 256>("tf32 SS", ctas);
    run<1, 64>("tf32 TS", ctas);
    run<1, 128>("tf32 TS", ctas);
    run<1, 256>("tf32 TS", ctas);
    run<2, 64>("bf16 SS", ctas);
    run<2, 128>("bf16 SS", ctas);
    run<2, 256>("bf16 SS", ctas);
  }
  return 0;
}
