// plan.h — the block plan shared by the host builder (builder.cpp), the
// C-ABI layer (api.cpp) and the kernels (kernels.cu).  Product code only.
//
// Layout in HBM.  Internal numbering: communities contiguous
// in label order (the permutation P of P:644-650), inside a community rows
// sorted by decreasing list length.  Rows are cut into community-aligned
// TILES of rows_per_tile = 512*rpt rows; one CTA (16 warps) owns a tile and
// lane l of warp w owns rows (w + 16 r)*32 + l, r < rpt ("chunk" = 32 rows).
//
// Per row j the stored list is the complement list Z_j of its dense blocks
// (subtracted) and the non-zero list NZ_j of its sparse blocks (added)
// (P:538-570).  The column space is cut into WINDOWS of WZ = 4096 columns
// (64 KB of z).  For each tile the windows that hold at least hot_min of the
// tile's entries are HOT: the CTA stages z[window] in shared memory and the
// entries are stored as 16-bit window-local indices.  All other entries are
// REMOTE, stored as 32-bit column ids and gathered from global memory.  A
// PART is one (hot window | remote, sign) pair of a tile, so the sign is
// uniform inside a part and costs nothing per entry.
//
// A part's data is a list of 16-byte units; for chunk c of the tile it is
// ng groups of 32 units, unit (g, lane) holding the entries 8g..8g+7 (hot)
// or 4g..4g+3 (remote) of the lane's row, padded with a sentinel that points
// at a zero z entry.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "kur.h"

namespace kur {

constexpr int WZ_SHIFT = 12;
constexpr int WZ = 1 << WZ_SHIFT;  // columns per shared-memory window (64 KB of double2)
constexpr int NWARPS = 16;         // warps per CTA
constexpr int NTHREADS = NWARPS * 32;
constexpr int MAX_RPT = 4;         // rows per thread (tile rows = 512 * rpt)
constexpr uint32_t HOT_SENT = WZ;  // window-local sentinel slot (always zero)
constexpr int DEFAULT_HOT_MIN = 1024;

struct TileDesc {   // 32 bytes; device array
  int32_t row0;     // first internal row (global numbering)
  int32_t nrows;    // rows in this tile (<= rows_per_tile)
  int32_t comm;     // community of every row of the tile
  int32_t part0;    // first part of the tile
  int32_t nhot;     // hot parts (part0 .. part0+nhot-1)
  int32_t nremote;  // 0..2 remote parts (after the hot parts)
  int32_t pad0, pad1;
};

struct ChunkDesc {  // 8 bytes; device array [n_parts * chunks_per_tile]
  uint32_t ofs;     // offset of the chunk's first unit (16-byte units) in the pool
  uint32_t ng;      // groups (each group = 32 units)
};

struct Unit {       // 16 bytes of the pool
  uint32_t w[4];
};

struct HostPlan {
  int64_t n = 0;
  int32_t C = 0;
  int rpt = 1, rows_per_tile = NTHREADS, chunks_per_tile = NWARPS;
  int32_t rank = 0, world = 1;
  int64_t row_begin = 0, row_end = 0;     // this rank's internal rows
  int32_t tile_begin = 0, tile_end = 0;   // this rank's tiles (global ids)
  int32_t comm_begin = 0, comm_end = 0;   // this rank's communities
  std::vector<int32_t> perm;        // [n] internal -> user
  std::vector<int32_t> comm_off;    // [C+1] internal row offsets
  std::vector<int32_t> comm_tile0;  // [C+1] tile offsets (global tile ids)
  std::vector<int32_t> D_ptr, D_idx;  // dense column communities of each row community
  std::vector<TileDesc> tiles;      // this rank's tiles (parts renumbered locally)
  std::vector<int32_t> part_window; // [n_parts] window id (-1 = remote)
  std::vector<int32_t> part_neg;    // [n_parts] 1 = complement entries (subtracted)
  std::vector<ChunkDesc> chunks;    // [n_parts * chunks_per_tile]
  std::vector<Unit> pool;           // index data
  std::vector<int32_t> tile_order;  // launch order (local tile ids, decreasing work)
  std::vector<int32_t> shard_row0;  // [world+1] internal row ranges of all ranks
  std::vector<int32_t> shard_tile0; // [world+1]
  // statistics (this rank)
  int64_t nnz = 0, n_idx_hot = 0, n_idx_remote = 0, n_slots_hot = 0, n_slots_remote = 0;
  int64_t n_dense_blocks = 0, n_sparse_blocks = 0, n_hot_parts = 0;
};

// Builds the plan on the host.  `sm_count` steers the tile size choice.
kur_status build_plan(const kur_graph_desc* d, int32_t rank, int32_t world, int sm_count,
                      HostPlan& P, std::string& err);

}  // namespace kur
