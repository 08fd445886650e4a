// HBM direction probe (harness, not product): read-only, write-only and copy
// bandwidth of one B200 with plain 16-byte LDG/STG and with TMA bulk copies,
// to see how much of the copy peak is lost to read/write mixing.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_probe scripts/hbm_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void rd_kernel(const int4* __restrict__ a, size_t n, int4* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a + i));
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678) sink[0] = acc;
}
__global__ void wr_kernel(int4* a, size_t n) {
  const int4 v = make_int4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(a + i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__global__ void cp_kernel(const int4* __restrict__ a, int4* b, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a + i));
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(b + i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  }
}

__device__ __forceinline__ uint32_t s32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mwait(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}\n" ::"r"(s32(bar)), "r"(ph) : "memory");
}
// TMA read-only: a ring of ST stages of PIECE bytes, loads only.
__global__ void tma_rd_kernel(const uint8_t* a, size_t bytes, int piece, int st) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + size_t(st) * piece);
  if (threadIdx.x) return;
  for (int s = 0; s < st; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bars[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t np = bytes / piece, p0 = np * blockIdx.x / gridDim.x, p1 = np * (blockIdx.x + 1) / gridDim.x;
  uint32_t ph[32] = {0};
  size_t k = 0;
  for (size_t i = p0; i < p1; ++i, ++k) {
    const int s = k % st;
    if (k >= (size_t)st) { mwait(&bars[s], ph[s]); ph[s] ^= 1; }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bars[s])), "r"(piece) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(s32(sm + size_t(s) * piece)), "l"(a + i * piece), "r"(piece), "r"(s32(&bars[s])) : "memory");
  }
  for (size_t j = (k > (size_t)st ? k - st : 0); j < k; ++j) { const int s = j % st; mwait(&bars[s], ph[s]); ph[s] ^= 1; }
}
// TMA write-only: bulk stores of one smem stage, up to ST groups in flight.
__global__ void tma_wr_kernel(uint8_t* a, size_t bytes, int piece, int st) {
  extern __shared__ __align__(128) uint8_t sm[];
  if (threadIdx.x) return;
  const size_t np = bytes / piece, p0 = np * blockIdx.x / gridDim.x, p1 = np * (blockIdx.x + 1) / gridDim.x;
  for (size_t i = p0; i < p1; ++i) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a + i * piece), "r"(s32(sm)), "r"(piece) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t bytes = size_t(4) << 30;
  uint8_t *a, *b;
  int4* sink;
  CK(cudaMalloc(&a, bytes));
  CK(cudaMalloc(&b, bytes));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMemset(a, 1, bytes));
  CK(cudaMemset(b, 2, bytes));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t n = bytes / 16;
  CK(cudaFuncSetAttribute(tma_rd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  CK(cudaFuncSetAttribute(tma_wr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  auto run = [&](const char* name, double mult, auto f) {
    float best = 1e9;
    for (int r = 0; r < 12; ++r) {
      cudaEventRecord(e0);
      f();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 2 && ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("{\"probe\": \"%s\", \"ms\": %.4f, \"GBps\": %.1f, \"err\": \"%s\"}\n", name, best,
           mult * bytes / best / 1e6, cudaGetErrorString(err));
  };
  for (int cps : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, 64, "ldg_read_%dcta", cps);
    run(nm, 1, [&] { rd_kernel<<<sms * cps, 256>>>((const int4*)a, n, sink); });
    snprintf(nm, 64, "stg_write_%dcta", cps);
    run(nm, 1, [&] { wr_kernel<<<sms * cps, 256>>>((int4*)b, n); });
    snprintf(nm, 64, "ldst_copy_%dcta", cps);
    run(nm, 2, [&] { cp_kernel<<<sms * cps, 256>>>((const int4*)a, (int4*)b, n); });
  }
  run("memcpy_d2d", 2, [&] { cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice); });
  for (int st : {2, 3, 4, 6}) {
    char nm[64];
    snprintf(nm, 64, "tma_read_32k_x%d", st);
    run(nm, 1, [&] { tma_rd_kernel<<<sms, 32, st * 32768 + 8 * st>>>(a, bytes, 32768, st); });
  }
  run("tma_write_32k", 1, [&] { tma_wr_kernel<<<sms, 32, 32768>>>(b, bytes, 32768, 0); });
  run("tma_write_32k_2cta", 1, [&] { tma_wr_kernel<<<sms * 2, 32, 32768>>>(b, bytes, 32768, 0); });
  // per-SM rates: a few CTAs (one per SM), 256 MiB, deep rings
  const size_t small = size_t(256) << 20;
  auto runs = [&](const char* name, double mult, auto f) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      f();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 1 && ms < best) best = ms;
    }
    printf("{\"probe\": \"%s\", \"ms\": %.4f, \"GBps\": %.1f}\n", name, best, mult * small / best / 1e6);
  };
  for (int g : {1, 8, 16}) {
    for (int st : {4, 6}) {
      char nm[64];
      snprintf(nm, 64, "tma_read_%dsm_x%d", g, st);
      runs(nm, 1, [&] { tma_rd_kernel<<<g, 32, st * 32768 + 8 * st>>>(a, small, 32768, st); });
    }
    char nm[64];
    snprintf(nm, 64, "tma_write_%dsm", g);
    runs(nm, 1, [&] { tma_wr_kernel<<<g, 32, 32768>>>(b, small, 32768, 0); });
    snprintf(nm, 64, "ldg_read_%dsm_1024thr", g);
    runs(nm, 1, [&] { rd_kernel<<<g, 1024>>>((const int4*)a, small / 16, sink); });
    snprintf(nm, 64, "stg_write_%dsm_1024thr", g);
    runs(nm, 1, [&] { wr_kernel<<<g, 1024>>>((int4*)b, small / 16); });
    snprintf(nm, 64, "ldst_copy_%dsm_1024thr", g);
    runs(nm, 2, [&] { cp_kernel<<<g, 1024>>>((const int4*)a, (int4*)b, small / 16); });
  }
  return 0;
}
