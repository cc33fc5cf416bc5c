// tiles.h — load-balanced row tiling of a CSR operator (host-side planner).
//
// The SpMV of every fused kernel walks a list of tiles, one CTA per tile:
//   STREAM  consecutive short rows (len <= kStreamMaxRow), <= kStreamNnz nnz and
//           <= kThreads rows: the nnz block is loaded with 128-bit coalesced loads,
//           the gathered products are staged in shared memory, and each row is then
//           summed by one thread in index order — the reference's sequential order
//           (sparse_matrix.hpp:123-131), so STREAM rows are bitwise equal to it;
//   WARP    medium rows, G lanes per row (G = 8..256 chosen for ~lane_nnz per lane,
//           stored in Tile::part), kThreads/G rows per tile, fixed-order reduction;
//   CHUNK   one long row or a kChunkNnz slice of it (merge-path style split for
//           skewed rows, e.g. the multicommodity budget rows); slices combine their
//           partials in slice order in whichever CTA finishes last (deterministic).
// In parity mode WARP/CHUNK rows are summed sequentially by one thread instead,
// and rows are never split, so every row sum equals the reference bitwise.
#pragma once

#include <stdint.h>

#include <utility>
#include <vector>

namespace pdlp {

enum TileKind : int32_t { kTileStream = 0, kTileWarp = 1, kTileChunk = 2 };

struct Tile {
  int32_t kind;
  int32_t row0;
  int32_t row1;   // STREAM/WARP: end row; CHUNK: counter index of a split row (-1 if unsplit)
  int32_t k0;
  int32_t k1;
  int32_t part;   // WARP: lanes per row; CHUNK: slice index; STREAM: uniform row length (0 = mixed)
  int32_t nparts;
  int32_t slot;   // CHUNK: first partial slot of the row; WARP: 1 = element-interleaved lanes
};
static_assert(sizeof(Tile) == 32, "tile descriptor is 32 bytes");

struct TilePlan {
  std::vector<Tile> tiles;
  int32_t chunk_slots = 0;     // partial slots needed by split rows
  int32_t split_rows = 0;      // counters needed by split rows
  int32_t stream_tiles = 0, warp_tiles = 0, chunk_tiles = 0;
};

// Builds the tile list for a CSR with `rows` rows and offsets `rp` (rows+1).
// `parity` disables WARP tiles and row splitting. `breaks` (sorted, may be
// empty) are rows where a tile must start: the shard boundaries, so every
// rank's rows are a contiguous run of whole tiles of the one global plan.
template <class Off>
TilePlan plan_tiles(int64_t rows, const Off* rp, bool parity, int stream_max_row,
                    int warp_max_row, int chunk_nnz, int stream_nnz, int stream_rows, int threads,
                    int lane_nnz, const std::vector<int64_t>& breaks = {},
                    const std::vector<uint8_t>* contig = nullptr);

// Shard boundaries: world + 1 rows 0 = c_0 < c_1 < ... < c_world = rows,
// balancing nnz + rows per shard, interior cuts on multiples of 4 rows.
// Throws std::invalid_argument when the operator is too small to split.
template <class Off>
std::vector<int64_t> shard_cuts(int64_t rows, const Off* rp, int world);

// [first, last) indices of the tiles whose first row lies in [r0, r1) (the
// shard ending at `rows` takes every remaining tile).
std::pair<int, int> tile_range(const TilePlan& plan, int64_t r0, int64_t r1, int64_t rows);

}  // namespace pdlp
