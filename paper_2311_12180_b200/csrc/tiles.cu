// tiles.cu — host-side tile planner (see tiles.h).
#include <algorithm>
#include <stdexcept>
#include <string>

#include "tiles.h"

namespace pdlp {

template <class Off>
TilePlan plan_tiles(int64_t rows, const Off* rp, bool parity, int stream_max_row,
                    int warp_max_row, int chunk_nnz, int stream_nnz, int stream_rows, int threads,
                    int lane_nnz, const std::vector<int64_t>& breaks,
                    const std::vector<uint8_t>* contig) {
  // rows whose columns are mostly consecutive (contig[r] != 0) get
  // element-interleaved WARP tiles; others quad-strided ones
  auto cflag = [&](int64_t i) { return contig ? int((*contig)[size_t(i)]) : 0; };
  TilePlan plan;
  int64_t r = 0;
  size_t bi = 0;
  auto len = [&](int64_t i) { return int64_t(rp[i + 1] - rp[i]); };
  while (r < rows) {
    while (bi < breaks.size() && breaks[bi] <= r) ++bi;
    const int64_t brk = bi < breaks.size() ? breaks[bi] : rows;  // next forced tile start
    const int64_t l = len(r);
    if (l <= stream_max_row) {
      const int64_t r0 = r, k0 = rp[r];
      while (r < brk && r - r0 < stream_rows && len(r) <= stream_max_row &&
             int64_t(rp[r + 1]) - k0 <= stream_nnz)
        ++r;
      // end interior tiles on a multiple of 4 rows so the 4-row groups of the
      // next tile stay 32-byte aligned for vector epilogues
      if (r < brk && r - r0 > 4 && (r & 3) && len(r) <= stream_max_row) r -= (r & 3);
      // uniform row length L (every row of the tile): the kernels index rows as
      // k0 + (r - row0) * L and skip the row offsets (Tile::part = L, else 0)
      int32_t uni = r > r0 ? int32_t(len(r0)) : 0;
      for (int64_t i = r0 + 1; i < r && uni > 0; ++i)
        if (len(i) != uni) uni = 0;
      plan.tiles.push_back({kTileStream, int32_t(r0), int32_t(r), int32_t(k0), int32_t(rp[r]), uni, 1, 0});
      ++plan.stream_tiles;
    } else if (!parity && l <= warp_max_row && contig && (*contig)[size_t(r)] == 2 && r + 4 <= brk) {
      // four column-shifted rows in one interleaved tile (contig flag 2 marks
      // the first row of such a group; spmv_engine.cuh)
      plan.tiles.push_back({kTileWarp, int32_t(r), int32_t(r + 4), int32_t(rp[r]), int32_t(rp[r + 4]),
                            threads / 4, 1, 2});
      ++plan.warp_tiles;
      r += 4;
    } else if (!parity && l <= warp_max_row) {
      // lanes per row: ~lane_nnz per lane, a power of two in [8, threads]
      auto lanes = [&](int64_t L) {
        int64_t g = 8;
        while (g < threads && g * lane_nnz < L) g *= 2;
        return int(g);
      };
      const int g = lanes(l);
      const int64_t r0 = r;
      const int cf = cflag(r);
      while (r < brk && r - r0 < threads / g && len(r) > stream_max_row && len(r) <= warp_max_row &&
             lanes(len(r)) == g && cflag(r) == cf)
        ++r;
      plan.tiles.push_back({kTileWarp, int32_t(r0), int32_t(r), int32_t(rp[r0]), int32_t(rp[r]), g, 1,
                            cf == 1 ? 1 : 0});
      ++plan.warp_tiles;
    } else {
      const int64_t k0 = rp[r], k1 = rp[r + 1];
      const int64_t parts = parity ? 1 : std::max<int64_t>(1, (l + chunk_nnz - 1) / chunk_nnz);
      const int32_t ctr = parts > 1 ? plan.split_rows++ : -1;
      for (int64_t p = 0; p < parts; ++p) {
        const int64_t a = k0 + p * chunk_nnz;
        const int64_t b = parts == 1 ? k1 : std::min<int64_t>(k1, a + chunk_nnz);
        plan.tiles.push_back({kTileChunk, int32_t(r), ctr, int32_t(a), int32_t(b), int32_t(p),
                              int32_t(parts), plan.chunk_slots});
        ++plan.chunk_tiles;
      }
      if (parts > 1) plan.chunk_slots += int32_t(parts);
      ++r;
    }
  }
  // Degenerate operators (no rows) still get one empty tile, so every fused
  // kernel has a CTA to run its reductions and step decision.
  if (plan.tiles.empty()) {
    plan.tiles.push_back({kTileStream, 0, 0, 0, 0, 0, 1, 0});
    ++plan.stream_tiles;
  }
  return plan;
}

template <class Off>
std::vector<int64_t> shard_cuts(int64_t rows, const Off* rp, int world) {
  if (world < 1) throw std::invalid_argument("shards: world size must be >= 1");
  std::vector<int64_t> cuts(size_t(world) + 1, 0);
  cuts[size_t(world)] = rows;
  const double total = double(rp[rows]) + double(rows);  // nnz + row work
  int64_t r = 0;
  for (int p = 1; p < world; ++p) {
    const double target = total * double(p) / double(world);
    // first row whose prefix weight reaches the target (binary search)
    int64_t lo = r, hi = rows;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (double(rp[mid]) + double(mid) < target)
        lo = mid + 1;
      else
        hi = mid;
    }
    int64_t c = lo & ~int64_t(3);
    if (c <= cuts[size_t(p) - 1]) c = cuts[size_t(p) - 1] + 4;
    if (c >= rows)
      throw std::invalid_argument("shards: " + std::to_string(rows) + " rows cannot be split " +
                                  std::to_string(world) + " ways");
    cuts[size_t(p)] = c;
    r = c;
  }
  return cuts;
}

std::pair<int, int> tile_range(const TilePlan& plan, int64_t r0, int64_t r1, int64_t rows) {
  // the last shard also takes the empty tile of an operator without rows
  int a = 0;
  const int n = int(plan.tiles.size());
  while (a < n && plan.tiles[size_t(a)].row0 < r0) ++a;
  int b = a;
  while (b < n && (r1 >= rows || plan.tiles[size_t(b)].row0 < r1)) ++b;
  return {a, b};
}

template TilePlan plan_tiles<int>(int64_t, const int*, bool, int, int, int, int, int, int, int,
                                  const std::vector<int64_t>&, const std::vector<uint8_t>*);
template TilePlan plan_tiles<int64_t>(int64_t, const int64_t*, bool, int, int, int, int, int, int,
                                      int, const std::vector<int64_t>&, const std::vector<uint8_t>*);
template std::vector<int64_t> shard_cuts<int>(int64_t, const int*, int);
template std::vector<int64_t> shard_cuts<int64_t>(int64_t, const int64_t*, int);

}  // namespace pdlp
