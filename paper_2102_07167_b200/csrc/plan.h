// plan.h — the block plan shared by the host builder (builder.cpp), the
// C-ABI layer (api.cpp) and the kernels (kernels.cu).  Product code only.
//
// Layout in HBM.  Internal numbering: communities contiguous
// in label order (the permutation P of P:644-650), inside a community rows
// sorted by decreasing list length.  Rows are cut into community-aligned
// TILES of at most 2048 rows; one CTA (16 warps) owns a tile and keeps the
// row sums W_j of the tile in shared memory.
//
// Per row j the stored list is the complement list Z_j of its dense blocks
// (subtracted) and the non-zero list NZ_j of its sparse blocks (added)
// (P:538-570).  The column space is cut into WINDOWS of WZ = 4096 columns
// (64 KB of z).  For each tile the windows that hold at least hot_min of the
// tile's entries are HOT: the CTA stages z[window] in shared memory (TMA bulk
// copy) and the entries are 16-bit window-local slots.  All other entries are
// REMOTE: 32-bit column ids gathered from global memory.  A PART is one
// (hot window | remote, sign) pair of a tile, so the sign is uniform inside a
// part and costs nothing per entry.
//
// Inside a part the rows that have entries are sorted by their entry count
// (longest first) and cut into CHUNKS of 32 rows, one row per lane, so the
// rows of a chunk have nearly equal lengths (little padding).  A chunk is a
// 64-byte header (32 x uint16 local row ids, 0xFFFF = empty lane) followed by
// the lane-interleaved entries.  Remote chunks: ng groups of 32 16-byte units,
// unit (g, lane) = the lane's 32-bit columns at positions 4g..4g+3.  Hot chunks:
// ng = (G << 1) | tail; G full groups of 32 16-byte units (unit (g, lane) = nine
// 13-bit slots at positions 9g..9g+8, slot e in bits 13e..13e+12), then, if tail
// is set, one trailing group of 32 8-byte units (four 16-bit slots at positions
// 9G..9G+3), so a chunk's length is rounded up to 9G or 9G + 4 positions.  In hot parts the entries of
// every quarter-warp (lanes 8q..8q+7) at one position have pairwise distinct
// slot residues mod 8, i.e. they hit distinct 16-byte shared-memory bank
// groups: every LDS.128 of the gather loop is bank-conflict free.  Padding
// slots point at zero sentinels WZ + rho (one per residue rho), remote padding
// at z[n] = 0.
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
constexpr uint32_t HOT_SENT = WZ;  // first of the 8 zero sentinel slots WZ..WZ+7
constexpr int DEFAULT_HOT_MIN = 2048;

constexpr int MAX_TILE_ROWS = 2048;  // W_j of a tile live in shared memory (32 KB)
constexpr int MAX_TILE_ROWS_NOPARTS = 4096;  // plans without stored entries keep no W_j in shared memory
constexpr int HDR_UNITS = 4;         // 64-byte chunk header
constexpr uint16_t EMPTY_LANE = 0xFFFF;

struct TileDesc {   // 32 bytes; device array
  int32_t row0;     // first internal row (global numbering)
  int32_t nrows;    // rows in this tile (<= rows_per_tile)
  int32_t comm;     // community of every row of the tile
  int32_t part0;    // first part of the tile
  int32_t nparts;   // hot parts first (by window), then remote parts
  int32_t nhot;     // number of hot parts
  int32_t nown;     // of which the first nown lie wholly inside the tile's own community
  int32_t nloc;     // of which the first nloc also lie inside this rank's rows (phase A, world > 1)
};

struct PartDesc {   // 16 bytes; device array
  int32_t window;   // window id (hot) or -1 (remote)
  int32_t neg;      // hot: 1 complement entries (subtracted), 0 non-zero entries (added), bits 8+: row
                    // pieces; remote (one part per tile): 0, the sign is per entry (bit 31 of the id)
  uint32_t chunk0;  // first chunk in the chunk table
  uint32_t nchunks;
};

struct ChunkDesc {  // 8 bytes; device array
  uint32_t ofs;     // pool offset (16-byte units) of the chunk header
  uint32_t ng;      // remote: groups of 4 positions; hot: half-groups of 4 positions (see above)
};

struct Unit {       // 16 bytes of the pool
  uint32_t w[4];
};

struct HostPlan {
  int64_t n = 0;
  int32_t C = 0;
  int rows_per_tile = NTHREADS;
  bool small = false;                     // world 1, n <= 8192, few entries: single-CTA kur_step
  bool split_remote = false;              // remote parts summed by a separate k_remote pass (see builder)
  int32_t rank = 0, world = 1;
  int64_t row_begin = 0, row_end = 0;     // this rank's internal rows
  int32_t tile_begin = 0, tile_end = 0;   // this rank's tiles (global ids)
  std::vector<int32_t> perm;        // [n] internal -> user
  std::vector<int32_t> comm_off;    // [C+1] internal row offsets
  std::vector<int32_t> comm_tile0;  // [C+1] tile offsets (global tile ids)
  std::vector<int32_t> D_ptr, D_idx;  // dense column communities of each row community
  std::vector<TileDesc> tiles;      // this rank's tiles (parts renumbered locally)
  std::vector<PartDesc> parts;      // this rank's parts
  std::vector<ChunkDesc> chunks;    // this rank's chunks
  std::vector<Unit> pool;           // index data
  std::vector<int32_t> tile_order;  // launch order (local tile ids, decreasing work)
  std::vector<uint32_t> rchunks;    // remote pass: [2k] chunk id, [2k+1] local row of the chunk's tile row 0,
                                    // all tiles' remote chunks, longest first
  std::vector<uint8_t> rem_lp;      // remote pass: row-piece shift (PartDesc.neg >> 8) per listed chunk
  std::vector<double> rowscale;     // [local rows] 1/M_m (degree scaling only; empty = uniform K/N)
  std::vector<double> potc;         // [local rows] off-diagonal ones + [z_m inside W_m] (kur_potential)
  std::vector<int32_t> shard_row0;  // [world+1] internal row ranges of all ranks
  std::vector<int32_t> shard_tile0; // [world+1]
  // statistics (this rank)
  int64_t nnz = 0, n_idx_hot = 0, n_idx_remote = 0, n_slots_hot = 0, n_slots_remote = 0;
  int64_t n_dense_blocks = 0, n_sparse_blocks = 0, n_hot_parts = 0;
  int64_t n_window_loads = 0;       // hot windows staged per RHS (all tiles)
};

// Builds the plan on the host.  `sm_count` steers the tile size choice.
kur_status build_plan(const kur_graph_desc* d, int32_t rank, int32_t world, int sm_count,
                      HostPlan& P, std::string& err);

}  // namespace kur
