// kde_tiles.cuh — the triangular tile map shared by every pair kernel (row a4 of SURVEY §8(a)).
#pragma once
#include <math.h>
#include <stdint.h>

namespace kde {

// Linear tile id bx -> (l, q), q <= l, of the upper-triangular tile grid numbered column by
// column (Eq. 42-43).
__host__ __device__ inline void tile_coords(int64_t bx, int64_t& l, int64_t& q) {
  // Eq. 42: l = ceil((sqrt(8 bx + 9) - 3) / 2);  Eq. 43: q = bx - l(l+1)/2.  The fp64 sqrt is
  // exact enough to land within +-1 of l for bx < 2^62; the loops make it exact (reading Z13).
  double s = sqrt(8.0 * (double)bx + 9.0);
  int64_t L = (int64_t)ceil((s - 3.0) * 0.5);
  if (L < 0) L = 0;
  while (L > 0 && L * (L + 1) / 2 > bx) --L;
  while ((L + 1) * (L + 2) / 2 <= bx) ++L;
  l = L;
  q = bx - L * (L + 1) / 2;
}

// The multi-GPU partition: rank r of P evaluates every P-th chunk of kShardChunk
// consecutive tile ids (round-robin), so every rank gets the same mix of diagonal, near and
// exactly-zero (skipped) tiles; a contiguous split loaded the ranks unevenly once far tiles were
// skipped on sorted data (C4 Psi4 pass at P = 8: heaviest rank 11% above the mean; 1.7% round-robin).
// A rank addresses its tiles by a local index i in [0, shard_count): global id shard_tile(i).
constexpr int kShardChunk = 16;
__host__ __device__ inline int64_t shard_tile(int64_t i, int rank, int world) {
  if (world <= 1) return i;
  const int64_t c = i / kShardChunk;
  return (c * world + rank) * kShardChunk + (i - c * kShardChunk);
}
__host__ __device__ inline int64_t shard_count(int64_t tiles, int rank, int world) {
  if (world <= 1) return tiles;
  const int64_t per = (int64_t)kShardChunk * world, full = tiles / per, rem = tiles - full * per;
  int64_t extra = rem - (int64_t)rank * kShardChunk;
  extra = extra < 0 ? 0 : (extra > kShardChunk ? kShardChunk : extra);
  return full * kShardChunk + extra;
}

}  // namespace kde
