/* Plain-C client of libaqua (no torch, no C++): exercises the C ABI in
 * AQUA_DRYRUN mode -- bookkeeping and descriptors only, so it runs without
 * a GPU.  Prints "ok" and exits 0 on success.  Expected values follow the
 * C1 golden script (tests/golden/c1_script.json). */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "aqua.h"

#define CHECK(x)                                                           \
  do {                                                                     \
    aqua_status _s = (x);                                                  \
    if (_s != AQUA_OK) {                                                   \
      fprintf(stderr, "%s:%d %s -> %d (%s)\n", __FILE__, __LINE__, #x, _s, \
              aqua_strerror(_s));                                          \
      return 1;                                                            \
    }                                                                      \
  } while (0)
#define EXPECT(c)                                               \
  do {                                                          \
    if (!(c)) {                                                 \
      fprintf(stderr, "%s:%d expected %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                 \
    }                                                           \
  } while (0)

int main(void) {
  void* bases[2] = {(void*)(uintptr_t)(1ull << 40), (void*)(uintptr_t)((1ull << 40) + (1ull << 32))};
  aqua_kv_layout lay;
  memset(&lay, 0, sizeof lay);
  lay.num_layers = 2;
  lay.block_tokens = 16;
  lay.num_kv_heads = 2;
  lay.head_dim = 64;
  lay.elem_bytes = 2;
  lay.num_blocks = 40;
  lay.layer_base = bases;
  aqua_ctx* ctx = NULL;
  CHECK(aqua_create(AQUA_DRYRUN, &lay, &ctx));
  const uint64_t U = 2ull * 2 * 16 * 2 * 64 * 2;
  int32_t nslots = 0;
  CHECK(aqua_lend(ctx, 0, (void*)(uintptr_t)(2ull << 40), 8 * U, &nslots));
  EXPECT(nslots == 8);
  CHECK(aqua_lend(ctx, AQUA_HOST, (void*)(uintptr_t)(3ull << 40), 8 * U, &nslots));
  int32_t ids[64];
  for (uint64_t p = 0; p < 8; ++p) {
    CHECK(aqua_alloc_blocks(ctx, p, 4, NULL, ids));
    EXPECT(ids[0] == (int32_t)(4 * p) && ids[3] == (int32_t)(4 * p + 3));
  }
  const uint64_t out[3] = {1, 4, 6};
  uint64_t ticket = 0;
  CHECK(aqua_swap_out(ctx, 3, out, NULL, &ticket));
  int32_t st, loc, n, slots[8];
  CHECK(aqua_query(ctx, 6, &st, &loc, &n, slots, 8));
  EXPECT(st == AQUA_ST_SWAPPED && loc == AQUA_LOC_HOST && n == 4 && slots[0] == 0);
  CHECK(aqua_alloc_blocks(ctx, 100, 6, NULL, ids));
  EXPECT(ids[0] == 4 && ids[4] == 16 && ids[5] == 17);
  const uint64_t in[3] = {6, 1, 4};
  int32_t counts[3];
  CHECK(aqua_swap_in(ctx, 3, in, NULL, ids, 64, counts, &ticket));
  EXPECT(counts[0] == 4 && ids[0] == 18 && ids[4] == 26 && ids[11] == 37);
  EXPECT(aqua_swap_in(ctx, 1, in, NULL, ids, 64, counts, &ticket) == AQUA_E_STATE);
  CHECK(aqua_free(ctx, 100, NULL));
  int32_t fb, pf, hf;
  CHECK(aqua_counts(ctx, &fb, &pf, &hf));
  EXPECT(fb == 8 && pf == 8 && hf == 8);
  /* options and the launch report through the C ABI */
  int64_t v = 0;
  CHECK(aqua_get_option(ctx, AQUA_OPT_TMA_SCHED, &v));
  EXPECT(v == AQUA_TMA_SCHED_AUTO);
  CHECK(aqua_get_option(ctx, AQUA_OPT_INLINE_MAX, &v));
  EXPECT(v == 4064);
  EXPECT(aqua_set_option(ctx, AQUA_OPT_INLINE_MAX, 4065) == AQUA_E_INVAL);
  CHECK(aqua_set_option(ctx, AQUA_OPT_TMA_VARIANT, 3));
  int32_t grid = -1;
  EXPECT(aqua_last_launch(ctx, &grid, NULL, NULL, NULL, NULL, NULL, NULL) == AQUA_E_STATE); /* dry: no launch */
  CHECK(aqua_destroy(ctx));
  printf("ok %s\n", aqua_version());
  return 0;
}
