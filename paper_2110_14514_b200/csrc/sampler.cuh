#pragma once
#include "common.cuh"

namespace ogcp {

struct DrawScratch {
  DevBuf tmaps, bagg, bstart, scal, cand, miss, zcount, zoff;
};

// Merged nonzero stratum of a draw: the distinct drawn ordinals in ascending
// order with their multiplicities (uint8; callers keep p <= 8*eta so a count
// cannot reach 256 with any realistic probability) and the distinct count on
// the device.
struct MergedDraw {
  DevBuf hist, ord, cnt, bcount, boff;
  long long* count = nullptr;
};

void init_jump_table();
void draw_enqueue(Ctx* ctx, const Slice* X, const Pcg64& g, int64_t p, int64_t q, int64_t budget,
                  int32_t* ordinals, int32_t* zero_subs, long long code, DrawScratch& scr,
                  MergedDraw* merged = nullptr);

}  // namespace ogcp
