// archive.cu — whole-slide tile archive assembly on the device.
//
// A whole slide (BASELINE configs[3]: 65536^2 RGB) is 256 independent 4096^2 tile containers
// (each exactly encode_image's output, container.py:167-206).  Tiles are sharded contiguously
// over the GPUs of one box; a rank encodes its tiles in batches (wbpc_encode, containers packed
// back to back per batch region, offsets on the device), then:
//   k_tile_sizes    per-tile container byte counts of this rank (the all-gather payload)
//   (NCCL all_gather of those counts over NVLink -- the path's only collective)
//   k_archive_index exclusive scan of all tiles' sizes -> archive offsets; writes the archive
//                   header + index (paper_2005_08713_b200/archive.py layout) and this rank's
//                   offsets relative to its first tile
//   k_gather_tiles  moves each tile's container from its batch region to its archive offset
// so the archive assembles without a host round trip (the device-side counterpart of the
// reference's `offset += len(blob)` index loop, container.py:199-206).
#include <algorithm>

#include "common.cuh"

namespace wb {

// enc_off: per batch k, (B+1) u64 container offsets within batch region k (stride B+1).
__global__ void k_tile_sizes(const u64* enc_off, int B, int n_local, int per, u64* sizes) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= per) return;
  u64 v = 0;
  if (i < n_local) {
    const int k = i / B, j = i - k * B;
    const u64* o = enc_off + (u64)k * (B + 1);
    v = o[j + 1] - o[j];
  }
  sizes[i] = v;
}

// Archive layout (archive.py): "WBPA" u8 1, u32 tiles_x, u32 tiles_y, (u64 off, u64 len) per
// tile in row-major tile order, then the tile containers.  One CTA: block-wide exclusive scan.
__global__ void __launch_bounds__(1024) k_archive_index(const u64* sizes_all, int n_tiles, int tiles_x,
                                                        int tiles_y, int first, int n_local, uint8_t* hdr,
                                                        u64* local_off, u64* base_total) {
  __shared__ u64 warp_sum[32];
  __shared__ u64 carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u64 hbytes = 13ull + 16ull * (u64)n_tiles;
  if (tid == 0) carry = hbytes;
  if (hdr && tid == 0) {
    hdr[0] = 'W'; hdr[1] = 'B'; hdr[2] = 'P'; hdr[3] = 'A'; hdr[4] = 1;
    for (int b = 0; b < 4; ++b) {
      hdr[5 + b] = (uint8_t)((unsigned)tiles_x >> (8 * b));
      hdr[9 + b] = (uint8_t)((unsigned)tiles_y >> (8 * b));
    }
  }
  __syncthreads();
  for (int c0 = 0; c0 < n_tiles; c0 += 1024) {
    const int i = c0 + tid;
    const u64 v = i < n_tiles ? sizes_all[i] : 0;
    u64 incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const u64 t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_sum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      u64 ws = warp_sum[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const u64 t = __shfl_up_sync(0xffffffffu, ws, o);
        if (lane >= o) ws += t;
      }
      warp_sum[lane] = ws;  // inclusive over warps
    }
    __syncthreads();
    const u64 off = carry + (warp ? warp_sum[warp - 1] : 0) + incl - v;
    if (i < n_tiles) {
      if (hdr) {
        uint8_t* e = hdr + 13 + 16ull * i;
        for (int b = 0; b < 8; ++b) {
          e[b] = (uint8_t)(off >> (8 * b));
          e[8 + b] = (uint8_t)(v >> (8 * b));
        }
      }
      if (i == first && base_total) base_total[0] = off;  // archive offset of this rank's first tile
    }
    __syncthreads();
    if (tid == 0) carry += warp_sum[31];
    __syncthreads();
  }
  if (tid == 0 && base_total) {
    base_total[1] = carry;  // total archive bytes
    if (first >= n_tiles) base_total[0] = carry;  // a rank without tiles starts at the end
  }
  // second pass over this rank's tiles: offsets relative to its first tile (n_local + 1 entries)
  __syncthreads();
  if (local_off) {
    __shared__ u64 run;
    if (tid == 0) run = 0;
    __syncthreads();
    for (int c0 = 0; c0 <= n_local; c0 += 1024) {
      const int j = c0 + tid;
      const u64 v = j < n_local ? sizes_all[first + j] : 0;
      u64 incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const u64 t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) warp_sum[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        u64 ws = warp_sum[lane];
        for (int o = 1; o < 32; o <<= 1) {
          const u64 t = __shfl_up_sync(0xffffffffu, ws, o);
          if (lane >= o) ws += t;
        }
        warp_sum[lane] = ws;
      }
      __syncthreads();
      if (j <= n_local) local_off[j] = run + (warp ? warp_sum[warp - 1] : 0) + incl - v;
      __syncthreads();
      if (tid == 0) run += warp_sum[31];
      __syncthreads();
    }
  }
}

// Copy tile i (blockIdx.y) from its batch region to dst + local_off[i].  Offsets are arbitrary
// bytes; the CTA's 16-byte destination chunks are aligned and whole (vector stores), their
// source bytes assembled from aligned 32-bit loads with funnel shifts.  The head / tail bytes
// outside whole aligned chunks (shared with the neighbouring tiles' ranges) are written bytewise.
constexpr int GATHER_CHUNK = 1 << 16;  // destination bytes per CTA

__device__ __forceinline__ uint32_t ld_src_word(const uint32_t* s, u64 byte) {
  // 4 bytes starting at an arbitrary source byte
  const u64 w = byte >> 2;
  const uint32_t sh = (uint32_t)(byte & 3) * 8;
  const uint32_t a = __ldg(s + w);
  return sh ? __funnelshift_r(a, __ldg(s + w + 1), sh) : a;
}

__global__ void __launch_bounds__(256) k_gather_tiles(const uint8_t* store, u64 region, const u64* enc_off, int B,
                                                      uint8_t* dst, const u64* local_off) {
  const int i = blockIdx.y;
  const int k = i / B, j = i - k * B;
  const u64* o = enc_off + (u64)k * (B + 1);
  const u64 so = (u64)k * region + o[j];
  const u64 n = o[j + 1] - o[j];
  const u64 d0 = local_off[i];
  const uint32_t* s32 = reinterpret_cast<const uint32_t*>(store);
  // CTA x takes chunks x, x + gridDim.x, ... of the tile's bytes
  for (u64 c0 = (u64)blockIdx.x * GATHER_CHUNK; c0 < n; c0 += (u64)gridDim.x * GATHER_CHUNK) {
    const u64 c1 = min(n, c0 + (u64)GATHER_CHUNK);
    // aligned 16-byte destination chunks inside [d0 + c0, d0 + c1)
    const u64 a0 = (d0 + c0 + 15) & ~15ull, a1 = (d0 + c1) & ~15ull;
    for (u64 d = a0 + 16ull * threadIdx.x; d < a1; d += 16ull * blockDim.x) {
      const u64 sb = so + (d - d0);
      uint4 v;
      v.x = ld_src_word(s32, sb);
      v.y = ld_src_word(s32, sb + 4);
      v.z = ld_src_word(s32, sb + 8);
      v.w = ld_src_word(s32, sb + 12);
      *reinterpret_cast<uint4*>(dst + d) = v;
    }
    // head [d0+c0, min(a0, d0+c1)) and tail [max(a1, head end), d0+c1): bytewise
    const u64 h1 = min(a0, d0 + c1);
    for (u64 d = d0 + c0 + threadIdx.x; d < h1; d += blockDim.x) dst[d] = store[so + (d - d0)];
    for (u64 d = max(a1, h1) + threadIdx.x; d < d0 + c1; d += blockDim.x) dst[d] = store[so + (d - d0)];
  }
}

// Streaming assembly: batch k's tiles get rank-local archive offsets as soon as batch k is encoded.
// local_off[k*B] (this batch's base) was written by batch k-1's launch (0 for batch 0); this
// launch writes local_off[k*B + 1 .. k*B + b], the last being batch k+1's base.
__global__ void k_batch_offsets(const u64* enc_off_k, int b, u64* local_off_k) {
  const int j = threadIdx.x;
  const u64 base = local_off_k[0];
  if (j >= 1 && j <= b) local_off_k[j] = base + (enc_off_k[j] - enc_off_k[0]);
}

cudaError_t launch_batch_offsets(const u64* enc_off_k, int b, u64* local_off_k, cudaStream_t s) {
  k_batch_offsets<<<1, 1024, 0, s>>>(enc_off_k, b, local_off_k);
  return cudaGetLastError();
}

cudaError_t launch_tile_sizes(const u64* enc_off, int B, int n_local, int per, u64* sizes, cudaStream_t s) {
  prof_mark("archive_sizes", s);
  k_tile_sizes<<<(per + 255) / 256, 256, 0, s>>>(enc_off, B, n_local, per, sizes);
  return cudaGetLastError();
}

cudaError_t launch_archive_index(const u64* sizes_all, int n_tiles, int tiles_x, int tiles_y, int first, int n_local,
                                 uint8_t* hdr, u64* local_off, u64* base_total, cudaStream_t s) {
  prof_mark("archive_index", s);
  k_archive_index<<<1, 1024, 0, s>>>(sizes_all, n_tiles, tiles_x, tiles_y, first, n_local, hdr, local_off,
                                     base_total);
  return cudaGetLastError();
}

cudaError_t launch_gather_tiles(const uint8_t* store, u64 region, const u64* enc_off, int B, int n_local,
                                uint8_t* dst, const u64* local_off, cudaStream_t s) {
  if (n_local <= 0) return cudaSuccess;
  prof_mark("archive_gather", s);
  // ~4 CTAs of 256 threads per SM over all tiles of the rank
  const unsigned per_tile = (unsigned)std::max(1, (148 * 4 + n_local - 1) / n_local);
  k_gather_tiles<<<dim3(per_tile, (unsigned)n_local), 256, 0, s>>>(store, region, enc_off, B, dst, local_off);
  return cudaGetLastError();
}

}  // namespace wb
