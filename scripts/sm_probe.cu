// Per-SM memory throughput ceiling: what one SM (one CTA of 1024 threads,
// each with UNROLL 16-byte accesses in flight) can read, write and copy
// through HBM, with the launch confined to `ctas` CTAs (= SMs).  Tells
// whether the ~100 GB/s of read + write per SM that the capped swap kernels
// reach (profiles/r01_hybrid3.jsonl: ring, hybrid and LDST alike) is the
// SM's own limit.  One JSON line per (kind, ctas).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sm_probe scripts/sm_probe.cu
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include <cuda_runtime.h>

constexpr int UNROLL = 8;

__device__ __forceinline__ int4 ldnc(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void stna(void* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}

// kind 0 read, 1 write, 2 copy; grid-stride over 16 KiB tiles (1024 threads x 16 B)
template <int KIND>
__global__ void __launch_bounds__(1024) probe(const int4* __restrict__ a, int4* __restrict__ b, int64_t n16,
                                              int4* sink) {
  const int64_t tid = threadIdx.x, step = int64_t(gridDim.x) * blockDim.x * UNROLL;
  int4 acc = make_int4(0, 0, 0, 0);
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x * UNROLL; base < n16; base += step) {
    int4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t i = base + u * blockDim.x + tid;
      if (KIND != 1 && i < n16) v[u] = ldnc(a + i);
      else v[u] = make_int4(int(i), 1, 2, 3);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t i = base + u * blockDim.x + tid;
      if (i >= n16) continue;
      if (KIND == 0) acc.x ^= v[u].x, acc.y ^= v[u].y;
      else stna(b + i, v[u]);
    }
  }
  if (KIND == 0 && (acc.x ^ acc.y) == 0x5eed) sink[0] = acc;
}

template <int KIND>
float run(const int4* a, int4* b, int64_t n16, int ctas, int4* sink) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe<KIND><<<ctas, 1024>>>(a, b, n16, sink);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    probe<KIND><<<ctas, 1024>>>(a, b, n16, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best;
}

int main() {
  const size_t bytes = size_t(1) << 30;
  int4 *a, *b, *sink;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMalloc(&sink, 64);
  cudaMemset(a, 1, bytes);
  cudaMemset(b, 0, bytes);
  const int caps[] = {1, 2, 4, 8, 16, 32, 64, 148};
  for (int ctas : caps) {
    // scale the bytes with the SM count so each run lasts a few ms
    const int64_t n16 = int64_t(std::min<size_t>(bytes, size_t(ctas) * (64u << 20))) / 16;
    const double gb = n16 * 16.0 / 1e9;
    const float r = run<0>(a, b, n16, ctas, sink), w = run<1>(a, b, n16, ctas, sink), c = run<2>(a, b, n16, ctas, sink);
    std::printf("{\"ctas\": %d, \"bytes\": %lld, \"read_GBps\": %.1f, \"write_GBps\": %.1f, \"copy_rw_GBps\": %.1f, "
                "\"per_sm\": {\"read\": %.1f, \"write\": %.1f, \"copy_rw\": %.1f}}\n",
                ctas, (long long)(n16 * 16), gb / r * 1e3, gb / w * 1e3, 2 * gb / c * 1e3, gb / r * 1e3 / ctas,
                gb / w * 1e3 / ctas, 2 * gb / c * 1e3 / ctas);
  }
  return cudaGetLastError() != cudaSuccess;
}
