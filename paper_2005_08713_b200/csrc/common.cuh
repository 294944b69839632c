// common.cuh — shared geometry, status recording and bit helpers for the sm_100a codec kernels.
//
// Geometry follows the reference container layout (pkg/src/wbpc/container.py:1-22, 111-137):
// per channel the LL grid of the deepest level, then the high-pass (LH,HL,HH) grids for levels
// L..1, each row major, 128x128 tiles, grid dims from the LL dims at that level.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/wbpc_b200.h"

#define WB_DIM 128          // container.py:54 BLOCK_DIM
#define WB_PP 2048          // areas per plane of a 128x128 block (bitplanes.py:182-185)
#define WB_MAXL 30          // transforms.py:21 MAX_LEVELS
#define WB_MAX_DEPTH 32     // int32 coefficients: |c| < 2^31 -> depth <= 32
#define WB_MAX_SLOTS (3 * WB_MAX_DEPTH)

typedef long long i64;
typedef unsigned long long u64;

struct LevelGeom {
  int w, h;      // LL dims after `l` splits (level_dims, transforms.py:227-232)
  int gw, gh;    // block grid at this level (ceil(w/128), ceil(h/128))
  int pw, ph;    // padded plane dims (gw*128, gh*128)
  int sw[4], sh[4];  // true dims of LL, LH, HL, HH produced by the split at this level (l>=1)
  i64 off[4];    // element offsets (within one channel's coefficient area) of LL, LH, HL, HH planes
  int slot0;     // first slot (within a channel) of the HP3 grid of this level
  int depth_bound[2];  // static max depth for LL / HP3 blocks of this level
  int swar;      // encode: every value of this level's split stays inside +-8000 (packed 16-bit lifting allowed)
  u64 md_gw;     // division magic for gw (fdiv)
};

struct Geom {
  int W, H, C, L, bd, rct;
  int slots_per_channel;
  int slots_per_image;
  i64 chan_stride;  // int32 elements per channel
  i64 img_stride;   // int32 elements per image (C * chan_stride)
  int sym_stride_ll, sym_stride_hp;  // bytes of symbol workspace per LL / HP3 block
  int raw_kind;     // -1: image container; 0/1: raw LL / HP3 coefficient blocks (block API)
  int coef16;       // encode coefficients stored as int16 (static bound < 2^15), else int32
  int keep;         // raw decode: planes_to_keep (-1 = None)
  u64 md_spc, md_spi;  // division magics for slots_per_channel / slots_per_image (fdiv)
  LevelGeom lv[WB_MAXL + 1];
};

// n / d for 0 <= n < 2^32 and d >= 1, with m = floor((2^64 - 1) / d) (host: div_magic):
// floor((n + 1) * m / 2^64) -- one 64-bit high multiply instead of a ~25-instruction integer
// division (whose reciprocal step also occupies the MUFU pipe).  Exact: (n+1) m / 2^64 is
// (n+1)/d minus less than 2^-32 < 1/d.
__device__ __forceinline__ int fdiv(int n, u64 m) { return (int)__umul64hi((u64)(uint32_t)n + 1ull, m); }

// decode_region per-level boxes (rows [r0, r1), cols [c0, c1)) in LL coordinates of each level
struct RegionBoxes {
  int r0[WB_MAXL + 1], r1[WB_MAXL + 1], c0[WB_MAXL + 1], c1[WB_MAXL + 1];
};

// ---- device status word (first bytes of every workspace) -----------------------------------
struct DevStatus {
  unsigned long long key;  // (priority<<56 | slot<<8 | code), atomicMin; ~0 = ok
  unsigned long long total;
  unsigned long long aux;
  unsigned long long pad;
};

__device__ __forceinline__ void record_error(DevStatus* st, int code, u64 slot, int priority = 1) {
  u64 key = ((u64)priority << 56) | ((slot & 0xFFFFFFFFFFFull) << 8) | (u64)(code & 0xFF);
  atomicMin(&st->key, key);
}

// Whole-sample symmetric extension (transforms.py:117-133,145-158): mirror about 0 and n-1.
__device__ __forceinline__ int reflect_pos(int p, int n) {
  if ((unsigned)p < (unsigned)n) return p;
  if (n == 1) return 0;
  int period = 2 * (n - 1);
  p %= period;
  if (p < 0) p += period;
  return p < n ? p : period - p;
}

__device__ __forceinline__ unsigned bswap32(unsigned x) { return __byte_perm(x, 0, 0x0123); }

// Locate (channel, kind, level, grid row, grid col) of a slot within one image (iter_slots,
// container.py:115-129).  kind 0 = LL, 1 = HP3.
struct SlotInfo {
  int c, kind, lev, r, col;
};

__device__ __forceinline__ SlotInfo slot_info(const Geom& g, int slot) {
  SlotInfo s;
  if (g.raw_kind >= 0) {  // block API: block i is tile row i of a 128-wide plane (LL: level 0, HP3: level 1)
    s.c = 0;
    s.kind = g.raw_kind;
    s.lev = g.raw_kind;
    s.r = slot;
    s.col = 0;
    return s;
  }
  s.c = fdiv(slot, g.md_spc);
  int k = slot - s.c * g.slots_per_channel;
  const LevelGeom& top = g.lv[g.L];
  int nll = top.gw * top.gh;
  if (k < nll) {
    s.kind = 0;
    s.lev = g.L;
    s.r = fdiv(k, top.md_gw);
    s.col = k - s.r * top.gw;
    return s;
  }
  int lev = g.L;
  while (lev > 1 && k >= g.lv[lev - 1].slot0) --lev;
  const LevelGeom& lg = g.lv[lev];
  int j = k - lg.slot0;
  s.kind = 1;
  s.lev = lev;
  s.r = fdiv(j, lg.md_gw);
  s.col = j - s.r * lg.gw;
  return s;
}

// Optional per-kernel CUDA-event timing (wbpc_profile_*): a mark before every kernel launch;
// the time between consecutive marks on the stream is the kernel's device time.
namespace wb {
void prof_mark(const char* name, cudaStream_t s);
}
