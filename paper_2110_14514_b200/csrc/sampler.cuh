#pragma once
#include "common.cuh"

namespace ogcp {

struct DrawScratch {
  DevBuf tmaps, bagg, bstart, scal, cand, miss, zcount, zoff;
};

void init_jump_table();
void draw_enqueue(Ctx* ctx, const Slice* X, const Pcg64& g, int64_t p, int64_t q, int64_t budget,
                  int32_t* ordinals, int32_t* zero_subs, long long code, DrawScratch& scr);

}  // namespace ogcp
