#pragma once
#include "common.cuh"

namespace ogcp {

struct DrawScratch {
  DevBuf tmaps, bagg, bstart, scal, cand, miss, zcount, zoff;
  DevBuf zkey, zkey_s, zval, zval_s, zsorted, ztmp;  // sorted zero rows (bucketed merged solves)
};

// Merged nonzero stratum of a draw: the distinct drawn ordinals in ascending
// order with their multiplicities (uint8; callers keep p <= 8*eta so a count
// cannot reach 256 with any realistic probability) and the distinct count on
// the device.
// perm (nullable): the slice's bucketed order (Slice::perm); the set is then
// emitted in position order -- ord holds positions into Slice::rec_b.
// [olo, ohi) (ohi = 0: the whole slice): the ordinal range this rank owns in a
// multi-GPU solve; only draws landing there are counted (the RNG words are
// still generated in full, so the counts are exactly the reference's).
struct MergedDraw {
  DevBuf hist, ord, cnt, bcount, boff, pnib;
  long long* count = nullptr;
  const int32_t* perm = nullptr;
  uint32_t olo = 0, ohi = 0;
};

void init_jump_table();
// Where a draw left its zero stratum: zsub points at [rows x ndim] int32
// coordinates -- zero_subs, or the candidate scratch of `scr` (valid until the
// next draw with the same scratch).  Lazy layout (q_dev != nullptr): the rows
// are candidate rows [0, *q_dev) and rows whose first coordinate is -1 are
// rejected candidates to skip; otherwise exactly q accepted rows.
struct DrawOut {
  const int32_t* zsub;
  const long long* q_dev;
};

// semi = true: the semi-stratified extension -- the q zero-stratum rows are the
// first q uniform cells of the box (no rejection), exactly q rows at zsub.
DrawOut draw_enqueue(Ctx* ctx, const Slice* X, const Pcg64& g, int64_t p, int64_t q, int64_t budget,
                     int32_t* ordinals, int32_t* zero_subs, long long code, DrawScratch& scr,
                     MergedDraw* merged = nullptr, bool lazy = false, bool semi = false);

// Word-range sharded merged draw (multi-GPU).  Rank r
// generates only its 1/N of the stream's 32-bit words: the per-tile aggregate
// maps are all-gathered so every rank scans the whole stream (tile start column
// and element offset, the nonzero stratum's end word), its draws are histogrammed
// into nibble counters over all ordinals that are reduce-scattered to the
// ordinal owners (uint32 sums of packed nibbles are nibble sums while no counter
// wraps: the owners' counter sums must add up to p), and its zero candidate rows
// (the rows that start in its element range) are probed locally; an all-gather
// of the per-rank (misses, rows, counter sum) locates the q-th miss.  One rank's device state:
struct ShardScratch {
  DevBuf tm_z;             // own zero-stream tiles' chunk maps
  DevBuf bagg_nz, bagg_z;  // per-tile aggregate maps, world x slot tiles (all-gathered)
  DevBuf bst_nz, bst_z;    // per-tile start (column, element) of every tile
  DevBuf hist;             // world x cw nibble words (chunk r: owner r's ordinals after the reduce-scatter)
  DevBuf zrec;             // world x 3 int64: (zero-row misses, zero rows, counter sum) per rank (all-gathered)
  DevBuf scal;             // 16 int64 scalars
  DevBuf cand, miss, zcount, zoff;  // this rank's zero candidate rows [rows x ndim], hit bits, miss scan
};
// Owner ranges of a sharded merged draw: chunks of 8 * ceil(ceil(eta / 8) / world)
// ordinals (whole nibble words).
void shard_owner_range(int64_t eta, int rank, int world, int64_t* olo, int64_t* ohi);
bool shard_draw_eligible(const Ctx* ctx, const Slice* X, int64_t p, int64_t q, bool semi);
// The draw as rank ctx->rank of ctx->world: md receives this rank's merged nonzeros
// (ordinals [olo, ohi) of shard_owner_range), the result's zsub / q_dev this rank's
// zero rows in the lazy layout (local rows [0, *q_dev), -1-flagged hits skipped).
// With a draw communicator the exchanges are NCCL collectives on ctx->stream; in
// shard simulation (no communicator) every rank's part runs on this GPU in lock
// step with device-side exchanges -- exact -- or, with ctx->shard_sim_timing, only
// this rank's part with its own slots standing in for the others' (timing only).
DrawOut shard_draw_enqueue(Ctx* ctx, const Slice* X, const Pcg64& g, int64_t p, int64_t q, int64_t budget,
                           long long code, MergedDraw& md, ShardScratch& sh);

// Every draw of a solver epoch made up front (small draws only, see
// draw_batch_eligible): draw b's nonzero ordinals at ord + b p, its zero stratum
// in the lazy layout at cand + b rows_max ndim with the row count at
// scal + 16 b + 8.
struct DrawBatchSet {
  DevBuf ord, cand, scal, specs, zspecs;
  int n = 0;
  int64_t p = 0, q = 0, rows_max = 0;
};
bool draw_batch_eligible(const Ctx* ctx, const Slice* X, int64_t p, int64_t q, int64_t budget, bool semi);
void draw_batch_enqueue(Ctx* ctx, const Slice* X, const Pcg64* gens, int n, int64_t p, int64_t q, int64_t budget,
                        long long code0, long long code_stride, DrawBatchSet& B);

}  // namespace ogcp
