// Host cost of one aqua_swap_out / aqua_swap_in call through the C ABI, by
// the number of blocks in the call: the library's bookkeeping, descriptor
// build / upload and the launch, without Python.  `host_cost dry` runs the
// bookkeeping alone (AQUA_DRYRUN: no CUDA, runs on a CPU-only box);
// `host_cost gpu` a real context on device 0 (self-lender arena) and also
// times a bare empty-kernel launch and an event record for scale.
// One JSON line per block count: microseconds per call (median of reps).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -Iinclude
//        scripts/host_cost.cu -Lpaper_2407_21255_b200 -laqua
//        -Xlinker -rpath,$PWD/paper_2407_21255_b200 -o /tmp/host_cost
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "aqua.h"

#define CHECK(x)                                                                       \
  do {                                                                                 \
    aqua_status _s = (x);                                                              \
    if (_s != AQUA_OK) {                                                               \
      std::fprintf(stderr, "%s:%d %s -> %d (%s)\n", __FILE__, __LINE__, #x, int(_s),   \
                   aqua_last_error(nullptr));                                          \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

__global__ void empty_kernel() {}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

int main(int argc, char** argv) {
  const bool dry = argc > 1 && std::strcmp(argv[1], "dry") == 0;
  // Llama-3-8B-shaped chunks with few layers, so 32K-block pools stay small:
  // L = 2, H = 1, D = 16, bs = 16, bf16 -> S = 512 B, U = 2 KiB
  const int L = 2, bs = 16, H = 1, D = 16, e = 2;
  const int NB = 65536 + 64;
  const int64_t S = int64_t(bs) * H * D * e, U = 2 * L * S;
  std::vector<void*> bases(L);
  void* arena = nullptr;
  cudaStream_t st = nullptr;
  if (dry) {
    for (int l = 0; l < L; ++l) bases[l] = reinterpret_cast<void*>(uintptr_t((uint64_t(l) + 1) << 40));
    arena = reinterpret_cast<void*>(uintptr_t(uint64_t(8) << 40));
  } else {
    for (int l = 0; l < L; ++l)
      if (cudaMalloc(&bases[l], 2 * int64_t(NB) * S) != cudaSuccess) return 2;
    if (cudaMalloc(&arena, int64_t(NB) * U) != cudaSuccess) return 2;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  }
  aqua_kv_layout lay;
  std::memset(&lay, 0, sizeof lay);
  lay.num_layers = L;
  lay.block_tokens = bs;
  lay.num_kv_heads = H;
  lay.head_dim = D;
  lay.elem_bytes = e;
  lay.num_blocks = NB;
  lay.layer_base = bases.data();
  aqua_ctx* ctx = nullptr;
  CHECK(aqua_create(dry ? AQUA_DRYRUN : 0, &lay, &ctx));
  int32_t nslots = 0;
  CHECK(aqua_lend(ctx, dry ? 0 : AQUA_MAPPED, arena, uint64_t(NB) * U, &nslots));
  std::vector<int32_t> ids(NB), counts(4);

  if (!dry) {   // scale: a bare launch and an event record on the same stream
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    std::vector<double> tl, te;
    for (int r = 0; r < 2000; ++r) {
      double t0 = now_us();
      empty_kernel<<<148, 32, 0, st>>>();
      double t1 = now_us();
      cudaEventRecord(ev, st);
      double t2 = now_us();
      if (r >= 100) tl.push_back(t1 - t0), te.push_back(t2 - t1);
    }
    cudaStreamSynchronize(st);
    std::printf("{\"what\": \"scale\", \"empty_launch_us\": %.2f, \"event_record_us\": %.2f}\n", median(tl),
                median(te));
    cudaEventDestroy(ev);
  }

  const int ns[] = {1, 8, 64, 512, 4096, 32768};
  for (int n : ns) {
    const uint64_t pid = 1;
    CHECK(aqua_alloc_blocks(ctx, pid, n, st, ids.data()));
    const int reps = n >= 4096 ? 200 : 2000;
    std::vector<double> to, ti;
    for (int r = 0; r < reps; ++r) {
      uint64_t t = 0;
      double t0 = now_us();
      CHECK(aqua_swap_out(ctx, 1, &pid, st, &t));
      double t1 = now_us();
      CHECK(aqua_swap_in(ctx, 1, &pid, st, ids.data(), NB, counts.data(), &t));
      double t2 = now_us();
      if (r >= reps / 10) to.push_back(t1 - t0), ti.push_back(t2 - t1);
      if (!dry && (r % 16) == 15) cudaStreamSynchronize(st);   // keep the queue short
    }
    if (!dry) cudaStreamSynchronize(st);
    CHECK(aqua_free(ctx, pid, st));
    std::printf("{\"mode\": \"%s\", \"blocks\": %d, \"chunk_bytes\": %lld, \"swap_out_us\": %.2f, \"swap_in_us\": %.2f,"
                " \"per_block_ns\": %.1f}\n",
                dry ? "dry" : "gpu", n, (long long)S, median(to), median(ti),
                1e3 * (median(to) + median(ti)) / (2.0 * n));
    std::fflush(stdout);
  }
  CHECK(aqua_destroy(ctx));
  return 0;
}
