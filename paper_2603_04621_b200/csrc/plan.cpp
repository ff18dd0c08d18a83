// Host-side planners: length buckets -> tiles, shard split.
//
// blocks grouped by length into buckets [2^(t-1), 2^t).  Here the
// buckets are laid out contiguously in HBM (bucket descending, source ascending) and
// cut into tiles: one block per tile for t >= kBigBucket (multi-warp groups), greedy
// packing up to tile_cap entries otherwise; every tile starts 16-byte aligned.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace dl {

Plan make_plan(const int64_t* row_ptr, int64_t I, int32_t tile_cap) {
  Plan P;
  // counting sort of nonempty blocks by bucket (descending), stable in source id
  std::vector<int64_t> count(65, 0);
  for (int64_t i = 0; i < I; ++i) {
    int64_t s = row_ptr[i + 1] - row_ptr[i];
    if (s > 0) count[bucket_of(s)]++;
  }
  std::vector<int64_t> start(65, 0);
  int64_t acc = 0;
  for (int t = 64; t >= 1; --t) {
    start[t] = acc;
    acc += count[t];
    if (count[t]) P.num_buckets++;
  }
  P.perm.assign(acc, 0);
  {
    std::vector<int64_t> pos(start);
    for (int64_t i = 0; i < I; ++i) {
      int64_t s = row_ptr[i + 1] - row_ptr[i];
      if (s > 0) P.perm[pos[bucket_of(s)]++] = i;
    }
  }
  P.blk_off.assign(acc, 0);
  int64_t off = 0;
  int64_t b = 0;
  auto open_tile = [&](int t) {
    off = (off + kAlign - 1) / kAlign * kAlign;
    Tile tl{};
    tl.rel_off = -1;
    tl.off = off;
    tl.b0 = (int32_t)b;
    tl.bucket = t;
    P.tiles.push_back(tl);
  };
  for (int t = 64; t >= 1; --t) {
    const int64_t end = start[t] + count[t];
    const bool big = t >= kBigBucket;
    while (b < end) {
      // longest run of whole blocks from b that fits tile_cap (one block per tile when big), trimmed
      // to whole warp rounds (round_blocks(t) blocks) when it exceeds one round and blocks remain
      int64_t n = 0, tot = 0;
      while (b + n < end) {
        const int64_t i = P.perm[b + n];
        const int64_t s = stored_len(row_ptr[i + 1] - row_ptr[i]);
        if (n > 0 && (big || tot + s > tile_cap)) break;
        tot += s;
        ++n;
      }
      if (!big) {
        const int64_t R = round_blocks(t, tile_cap);
        if (n > R && b + n < end) n -= n % R;
      }
      open_tile(t);
      Tile& tl = P.tiles.back();
      for (int64_t q = 0; q < n; ++q, ++b) {
        const int64_t i = P.perm[b];
        P.max_len = std::max<int32_t>(P.max_len, (int32_t)(row_ptr[i + 1] - row_ptr[i]));
        const int64_t s = stored_len(row_ptr[i + 1] - row_ptr[i]);
        P.blk_off[b] = off;
        off += s;
        tl.nnz += (int32_t)s;
        tl.nb += 1;
      }
    }
  }
  P.total = off;
  // phase ranges over the tile list (tiles are bucket-descending)
  int32_t nt = (int32_t)P.tiles.size();
  int32_t q = 0;
  for (int ph = 0; ph < kNumBigPhases; ++ph) {
    P.ph_begin[ph] = q;
    while (q < nt && P.tiles[q].bucket >= kBigBucket && big_phase_of(P.tiles[q].bucket) == ph) ++q;
  }
  P.ph_begin[kNumBigPhases] = q;
  P.ph_begin[kNumBigPhases + 1] = nt;
  return P;
}

// Shared memory of the fused kernel: barriers + reduction scratch + cached duals +
// 16 warps x (2 stages x tile_cap x (4 B dest + 4 B c + 4 B per family) + per-warp metadata).
static constexpr size_t kSmemFixed = 2048 + 1024;  // head + tail pad for over-reads past a tile
static constexpr size_t kSmemMax = 232448;  // 227 KB opt-in per CTA on sm_100
static constexpr int kMinTileCap = 256;      // every small block (< 256 entries) fits one tile
static constexpr int kHotTileCap = 384;      // tiles when only the hot duals are staged (r02 sweep at J = 100k:
                                             // 256 -> 3.57 ms, 320 -> 3.57, 384 -> 3.23, 448 -> 3.43, 512 -> 3.90)

size_t fused_smem_bytes(int32_t m, int32_t kind, int32_t tile_cap, int32_t hot) {
  const size_t lam = ((size_t)m * hot * 4 + 127) / 128 * 128;
  return kSmemFixed + lam + (size_t)kWarps * (2 * (size_t)tile_cap * (8 + 4 * (size_t)m) + meta_bytes(kind));
}

// lambda placement and tile capacity: all m*J duals in shared memory if
// that still leaves tiles of >= 256 entries (largest tile 2048); otherwise 256-entry tiles and as
// many duals of the most popular destination labels as the rest of the 227 KB holds (R15).
SmemRule smem_rule(int32_t m, int32_t J, int32_t kind) {
  const int64_t per_entry = (int64_t)kWarps * 2 * (8 + 4 * (int64_t)m);
  const int64_t fixed = (int64_t)kSmemFixed + (int64_t)kWarps * meta_bytes(kind);
  SmemRule r{};
  const int64_t lam_all = ((int64_t)m * J * 4 + 127) / 128 * 128;
  int64_t cap = ((int64_t)kSmemMax - fixed - lam_all) / per_entry / kAlign * kAlign;
  if (cap >= kMinTileCap) {
    r.lam_mode = kLamSmem;
    r.hot = J;
    r.tile_cap = (int32_t)std::min<int64_t>(cap, 2048);
    return r;
  }
  // tiles of kHotTileCap entries and the rest of shared memory for hot duals; DUALIP_TILE_CAP (a
  // multiple of 4 in [256, 2048]) trades hot duals for longer tiles (tuning experiments)
  int64_t tc = kHotTileCap;
  if ((int64_t)kSmemMax - fixed - tc * per_entry < (32 << 10)) tc = kMinTileCap;  // keep >= 32 KB of hot duals
  if (const char* e = std::getenv("DUALIP_TILE_CAP")) {
    const int64_t v = std::atoll(e);
    if (v >= kMinTileCap && v <= 2048 && v % kAlign == 0 && (int64_t)kSmemMax - fixed - v * per_entry >= 0) tc = v;
  }
  r.tile_cap = (int32_t)tc;
  const int64_t budget = (int64_t)kSmemMax - fixed - tc * per_entry;
  int64_t hot = budget / (4 * (int64_t)m) / 32 * 32;
  hot = std::max<int64_t>(0, std::min<int64_t>(hot, J));
  r.hot = (int32_t)hot;
  r.lam_mode = hot > 0 ? kLamHot : kLamGlobal;
  return r;
}

int32_t tile_cap_rule(int32_t m, int32_t J, int* lambda_in_smem) {
  SmemRule r = smem_rule(m, J, DL_PROJ_SIMPLEX);
  if (lambda_in_smem) *lambda_in_smem = r.lam_mode == kLamSmem;
  return r.tile_cap;
}

}  // namespace dl

using namespace dl;

extern "C" dl_status dl_plan_tiles(const int64_t* row_ptr, int64_t I, int32_t tile_cap, int64_t* perm,
                                   int64_t* blk_off, int64_t* tiles, int64_t* num_blocks, int64_t* num_tiles,
                                   int64_t* total) {
  if (!row_ptr || I < 0 || tile_cap < 256 || tile_cap % kAlign) {
    set_error("dl_plan_tiles: bad arguments (row_ptr NULL, I < 0, or tile_cap not a multiple of 4 >= 256)");
    return DL_ERR_INVALID;
  }
  for (int64_t i = 0; i < I; ++i)
    if (row_ptr[i + 1] < row_ptr[i]) {
      set_error("dl_plan_tiles: row_ptr decreasing");
      return DL_ERR_INVALID;
    }
  Plan P = make_plan(row_ptr, I, tile_cap);
  if (num_blocks) *num_blocks = (int64_t)P.perm.size();
  if (num_tiles) *num_tiles = (int64_t)P.tiles.size();
  if (total) *total = P.total;
  if (perm) std::memcpy(perm, P.perm.data(), P.perm.size() * sizeof(int64_t));
  if (blk_off) std::memcpy(blk_off, P.blk_off.data(), P.blk_off.size() * sizeof(int64_t));
  if (tiles)
    for (size_t q = 0; q < P.tiles.size(); ++q) {
      tiles[5 * q + 0] = P.tiles[q].b0;
      tiles[5 * q + 1] = P.tiles[q].nb;
      tiles[5 * q + 2] = P.tiles[q].off;
      tiles[5 * q + 3] = P.tiles[q].nnz;
      tiles[5 * q + 4] = P.tiles[q].bucket;
    }
  return DL_OK;
}

extern "C" dl_status dl_plan_shards(const int64_t* row_ptr, int64_t I, int32_t world, int64_t* bounds) {
  if (!row_ptr || !bounds || I < 0 || world < 1) {
    set_error("dl_plan_shards: bad arguments");
    return DL_ERR_INVALID;
  }
  const int64_t nnz = row_ptr[I];
  bounds[0] = 0;
  for (int32_t w = 1; w < world; ++w) {
    // floor(w*nnz/world) without overflow for nnz < 2^62 / world
    int64_t target = (int64_t)(((__int128)w * nnz) / world);
    int64_t lo = std::lower_bound(row_ptr, row_ptr + I + 1, target) - row_ptr;
    bounds[w] = std::max(std::min(lo, I), bounds[w - 1]);
  }
  bounds[world] = I;
  return DL_OK;
}

extern "C" int32_t dl_tile_cap(int32_t m, int32_t J) { return tile_cap_rule(m, J, nullptr); }
