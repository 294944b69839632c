// decode.cu — container index check, per-block header/tree parse, Huffman + zero-run decode of
// every stored plane in parallel, and coefficient reconstruction into subband planes (sm_100a).
//
// Replaces (reference /root/reference/pkg/src/wbpc):
//   ContainerReader index validation        container.py:212-229
//   decode_slot (planes_dropped -> keep)    container.py:235-244
//   parse_header, decode_block              blocks.py:150-250
//   read_tree, HuffmanCode._assign_codes    entropy.py:272-310, 88-100
//   decode_tokens (numba)                   _kernels.py:33-89
//   deserialize_block/_planes_to_values     bitplanes.py:268-291,125-130
//   _stitch                                 container.py:247-298
//
// The reference decodes the stored planes of a block sequentially and afterwards checks that each
// plane started at its seek entry (blocks.py:241-242).  Here every stored plane is decoded by its
// own lane starting at its seek entry; when all planes decode cleanly and each one ends exactly
// where the next one's seek entry points, the result is identical to the sequential decode.  Any
// other outcome (corrupt stream) re-runs the reference's sequential algorithm on lane 0 so the
// raised error class is the reference's.
#include <cstdlib>

#include "coder.cuh"

namespace wb {

constexpr int LUT_BITS = 10;
constexpr int LUT_SIZE = 1 << LUT_BITS;

struct DecMeta {
  uint32_t decoded[3];  // bit (b*nsub + s): slot symbols present in the workspace
  uint8_t depth, nsub, needed, pad;
};

// ---- index validation -------------------------------------------------------------------------
struct IndexParams {
  Geom g;
  int batch;
  const uint8_t* data;
  const u64* img_off;   // [batch+1] container start offsets within data, [batch] = end
  u64* blk_off;         // absolute byte offset of each block
  uint32_t* blk_len;
  DevStatus* st;
};

static __device__ __forceinline__ u64 rd_le(const uint8_t* p, int n) {
  u64 v = 0;
  for (int i = n - 1; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

__global__ void k_index_check(IndexParams P) {
  const int spi = P.g.slots_per_image;
  const i64 gi = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= (i64)P.batch * spi) return;
  const int b = (int)(gi / spi), slot = (int)(gi - (i64)b * spi);
  const u64 base = P.img_off[b], clen = P.img_off[b + 1] - base;
  const u64 need = 19 + 12ull * spi;
  const uint8_t* c = P.data + base;
  if (clen < need) {  // container.py:217-219
    if (slot == 0) record_error(P.st, WBPC_ERR_CONTAINER_PARSE, (u64)b * spi, 0);
    P.blk_off[gi] = base;
    P.blk_len[gi] = 0;
    return;
  }
  if (slot == 0 && b > 0) {
    // batch members must share the geometry of image 0 (header bytes 0..18)
    for (int i = 0; i < 19; ++i)
      if (c[i] != P.data[P.img_off[0] + i]) { record_error(P.st, WBPC_ERR_CONTAINER_PARSE, (u64)b * spi, 0); break; }
  }
  const uint8_t* e = c + 19 + 12ull * slot;
  u64 off = rd_le(e, 8), len = rd_le(e + 8, 4);
  u64 prev_end = need;
  if (slot > 0) prev_end = rd_le(e - 12, 8) + rd_le(e - 4, 4);
  if (off < prev_end || off + len > clen || off + len < off) {  // container.py:226-227
    record_error(P.st, WBPC_ERR_CORRUPTION, (u64)gi, 0);
    P.blk_off[gi] = base;
    P.blk_len[gi] = 0;
    return;
  }
  P.blk_off[gi] = base + off;
  P.blk_len[gi] = (uint32_t)len;
}

// Block API: block i spans bytes [offsets[i], offsets[i+1]) of the packed buffer.
__global__ void k_raw_index(const u64* offsets, int n, u64* blk_off, uint32_t* blk_len) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  blk_off[i] = offsets[i];
  blk_len[i] = (uint32_t)(offsets[i + 1] - offsets[i]);
}

cudaError_t launch_raw_index(const u64* offsets, int n, u64* blk_off, uint32_t* blk_len, cudaStream_t s) {
  k_raw_index<<<(n + 255) / 256, 256, 0, s>>>(offsets, n, blk_off, blk_len);
  return cudaGetLastError();
}

// ---- bit reader over the container buffer ------------------------------------------------------
struct BitSrc {
  const uint8_t* data;
  u64 nbytes;  // bytes valid in `data` (whole buffer)
  // optional shared-memory copy of words [sw_lo, sw_lo + sw_n) (raw little-endian bytes)
  const uint32_t* sw = nullptr;
  u64 sw_lo = 0;
  uint32_t sw_n = 0;
  __device__ __forceinline__ uint32_t word(u64 k) const {  // big-endian word k (bytes 4k..4k+3)
    if (k - sw_lo < sw_n) return bswap32(sw[k - sw_lo]);
    if (4 * k + 3 < nbytes) return bswap32(__ldg(reinterpret_cast<const uint32_t*>(data) + k));
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) {
      u64 bi = 4 * k + i;
      v = (v << 8) | (bi < nbytes ? data[bi] : 0u);
    }
    return v;
  }
  // read n (<= 32) bits at absolute bit position p
  __device__ __forceinline__ uint32_t bits(u64 p, int n) const {
    if (n == 0) return 0;
    u64 k = p >> 5;
    u64 w = ((u64)word(k) << 32) | word(k + 1);
    return (uint32_t)((w << (p & 31)) >> (64 - n));
  }
};


// Decode tables of one block: built by k_block_header (global), copied to smem by k_block_planes.
struct __align__(16) BlockTab {
  uint32_t lut[LUT_SIZE];  // leaf: (sym << 8) | len ; long code: 0x80000000 | node
  int16_t left[512], right[512], sym[512];
  uint32_t seek[WB_MAX_SLOTS];
  uint8_t slot_of[WB_MAX_SLOTS];
  u64 pstart;              // absolute payload start bit
  int rc, depth, cw, zr, nst, dn, ntree, nsub;
};

struct DecodeParams {
  Geom g;
  int batch;
  int level;            // output level: blocks of levels <= level are not needed
  int drop_global;
  int drop_ll;
  int drop_hp[WB_MAXL + 1];
  int per_level;
  BitSrc src;
  const u64* blk_off;
  const uint32_t* blk_len;
  BlockTab* tabs;
  const uint8_t* need;  // optional per-block mask (decode_region): 0 = block not decoded
  uint32_t* flags;      // per block: a plane failed (error path)
  uint8_t* syms;        // stride g.sym_stride_hp per block
  DecMeta* dmeta;
  DevStatus* st;
  uint32_t stage_bytes; // shared-memory staging window per block (multiple of 16)
};

// Register bit buffer (header parse): `buf` holds `nb` valid bits, MSB first.
struct BitBuf {
  const BitSrc* src;
  uint64_t buf;
  int nb;
  u64 next;
  u64 pos;
  __device__ __forceinline__ void init(const BitSrc& s, u64 p) {
    src = &s;
    u64 k = p >> 5;
    buf = (((uint64_t)s.word(k) << 32) | s.word(k + 1)) << (p & 31);
    nb = 64 - (int)(p & 31);
    next = k + 2;
    pos = p;
  }
  __device__ __forceinline__ void refill() {
    if (nb <= 32) {
      buf |= (uint64_t)src->word(next++) << (32 - nb);
      nb += 32;
    }
  }
  __device__ __forceinline__ uint32_t get(int n) {
    if (n == 0) return 0;
    if (nb < n) refill();
    uint32_t v = (uint32_t)(buf >> (64 - n));
    buf <<= n;
    nb -= n;
    pos += (u64)n;
    refill();
    return v;
  }
};

// Header parse of blocks.py:150-192 (+ read_tree entropy.py:272-310) into the smem scratch `T`
// (fields depth, cw, zr, nst, ntree, pstart, left/right/sym, seek, pending, seen); node depths and
// codes go to ndepth/ncode.  Register bit buffer over a word source (staged smem words with a
// global fallback).  Returns 0 or the reference's error class.
template <typename Tab>
static __device__ int parse_block_header(const BitSrc src, u64 bstart, u64 bend, int nsub, Tab& T,
                                         uint8_t* ndepth, uint32_t* ncode, uint32_t* mask3) {
  // 64-bit buffer: `buf` holds `nb` valid bits (MSB first) starting at absolute bit `pos`
  u64 k = bstart >> 5;
  uint64_t buf = (((uint64_t)src.word(k) << 32) | src.word(k + 1)) << (bstart & 31);
  int nb = 64 - (int)(bstart & 31);
  u64 nextw = k + 2;
  u64 pos = bstart;
  auto refill = [&]() {
    if (nb <= 32) {
      buf |= (uint64_t)src.word(nextw++) << (32 - nb);
      nb += 32;
    }
  };
  auto get = [&](int n) -> uint32_t {  // n <= 32
    if (n == 0) return 0u;
    refill();
    const uint32_t v = (uint32_t)(buf >> (64 - n));
    buf <<= n;
    nb -= n;
    pos += (u64)n;
    return v;
  };
#define NEED(n)                    \
  if (pos + (u64)(n) > bend) return WBPC_ERR_BLOCK_PARSE;
  NEED(6);
  const int depth = (int)get(6);
  if (depth < 1) return WBPC_ERR_BLOCK_PARSE;
  NEED(5);
  const int cw = (int)get(5);
  NEED(8);
  const int zr = (int)get(8);
  mask3[0] = mask3[1] = mask3[2] = 0;
  int cnt = 0;
  uint64_t mk[3] = {0, 0, 0};
  for (int s = 0; s < nsub; ++s) {
    NEED(depth);
    u64 v;
    if (depth > 32) {
      v = (u64)get(depth - 32) << 32;
      v |= get(32);
    } else {
      v = get(depth);
    }
    mk[s] = v;  // MSB = plane 0
    cnt += __popcll(v);
  }
  T.depth = depth;
  T.cw = cw;
  T.zr = zr;
  T.nst = cnt;
  int ntree = 0;
  if (cnt) {
    for (int i = 0; i < 8; ++i) T.seen[i] = 0;
    int np = 0;
    bool first = true;
    while (first || np) {
      first = false;
      if (pos + 1 > bend) return WBPC_ERR_MALFORMED_TREE;
      refill();
      const uint32_t bit = (uint32_t)(buf >> 63);
      const int idx = ntree;
      if (idx > 511) return WBPC_ERR_MALFORMED_TREE;
      if (bit) {
        if (pos + 9 > bend) return WBPC_ERR_MALFORMED_TREE;
        const int sy = (int)((buf >> 55) & 255u);
        buf <<= 9;
        nb -= 9;
        pos += 9;
        const uint32_t m = 1u << (sy & 31);
        if (T.seen[sy >> 5] & m) return WBPC_ERR_MALFORMED_TREE;
        T.seen[sy >> 5] |= m;
        T.left[idx] = -1; T.right[idx] = -1; T.sym[idx] = (int16_t)sy;
      } else {
        buf <<= 1;
        nb -= 1;
        pos += 1;
        T.left[idx] = -2; T.right[idx] = -2; T.sym[idx] = -1;
      }
      ++ntree;
      if (idx > 0) {
        const int parent = T.pending[np - 1];
        if (T.left[parent] == -2) T.left[parent] = (int16_t)idx;
        else { T.right[parent] = (int16_t)idx; --np; }
      }
      if (!bit) T.pending[np++] = (int16_t)idx;
    }
    // depths/codes in preorder (parents precede children); CodeLengthError (entropy.py:97-98)
    ndepth[0] = 0;
    ncode[0] = 0;
    for (int i = 0; i < ntree; ++i) {
      const int l = T.left[i];
      if (l == -1) continue;
      if (ndepth[i] >= 32) return WBPC_ERR_CODE_LENGTH;
      const int r = T.right[i];
      ndepth[l] = ndepth[r] = (uint8_t)(ndepth[i] + 1);
      ncode[l] = ncode[i] << 1;
      ncode[r] = (ncode[i] << 1) | 1u;
    }
  }
  T.ntree = ntree;
  NEED(16);
  const int seek_count = (int)get(16);
  if (seek_count != cnt) return WBPC_ERR_CORRUPTION;
  const int t = seek_bits(nsub, depth);
  uint32_t prev = 0;
  bool decreasing = false;
  for (int i = 0; i < cnt; ++i) {
    NEED(t);
    const uint32_t v = get(t);
    if (i < WB_MAX_SLOTS) T.seek[i] = v;
    if (i && v < prev) decreasing = true;
    prev = v;
  }
  if (decreasing) return WBPC_ERR_CORRUPTION;  // blocks.py:177-178
  T.pstart = pos;
  for (int s = 0; s < nsub; ++s)
    for (int b = 0; b < depth; ++b)
      if ((mk[s] >> (depth - 1 - b)) & 1ull) {
        const int kk = b * nsub + s;
        if (kk < WB_MAX_SLOTS) mask3[kk >> 5] |= 1u << (kk & 31);
      }
  return 0;
#undef NEED
}

// K1: one warp per block -- lane 0 parses header + tree (scratch in smem), the warp builds the
// decode LUT; results (BlockTab, DecMeta) go to global memory for K2 / reconstruction.
constexpr int HW = 4;  // warps (blocks) per K1 CTA
struct HdrScratch {        // shared-memory image of the BlockTab fields lane 0 parses
  uint32_t hw[256];         // first 1 KB of the block (header), raw little-endian words
  int16_t left[512], right[512], sym[512], pending[512];
  uint32_t seen[8];
  uint32_t seek[WB_MAX_SLOTS];
  uint8_t ndepth[512];
  uint32_t ncode[512];
  uint32_t m3[3];
  u64 pstart;
  int rc, depth, cw, zr, nst, ntree, dn;
  uint8_t slot_of[WB_MAX_SLOTS];
};

__global__ void __launch_bounds__(HW * 32) k_block_header(DecodeParams P) {
  __shared__ HdrScratch HS[HW];
  const Geom& g = P.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = blockIdx.x * HW + warp;
  if (gid >= P.batch * g.slots_per_image) return;
  const int b = gid / g.slots_per_image;
  const SlotInfo si = slot_info(g, gid - b * g.slots_per_image);
  DecMeta* DM = P.dmeta + gid;
  BlockTab& T = P.tabs[gid];
  HdrScratch& H = HS[warp];
  // not needed for this output level, or outside decode_region's per-level boxes: its
  // coefficients are never read by the requested output pixels
  if (!(si.kind == 0 || si.lev > P.level) || (P.need && !P.need[gid])) {
    if (lane == 0) { DM->needed = 0; T.rc = -1; T.dn = 0; }
    return;
  }
  const int nsub = si.kind ? 3 : 1;
  // stage the first 1 KB of the block (the whole header for <= ~8 Kbit headers) into smem
  const u64 w0 = P.blk_off[gid] >> 2;
  const u64 nw = P.src.nbytes >> 2;
  for (int i = lane; i < 256; i += 32) H.hw[i] = w0 + i < nw ? __ldg(reinterpret_cast<const uint32_t*>(P.src.data) + w0 + i) : 0u;
  __syncwarp();
  BitSrc hsrc = P.src;
  hsrc.sw = H.hw;
  hsrc.sw_lo = w0;
  hsrc.sw_n = nw > w0 ? (uint32_t)(nw - w0 < 256 ? nw - w0 : 256) : 0u;
  if (lane == 0) {
    const u64 bstart = 8ull * P.blk_off[gid];
    const u64 bend = bstart + 8ull * P.blk_len[gid];
    int rc = parse_block_header(hsrc, bstart, bend, nsub, H, H.ndepth, H.ncode, H.m3);
    if (!rc && H.depth > WB_MAX_DEPTH) rc = WBPC_ERR_UNSUPPORTED;  // magnitudes beyond int32
    H.rc = rc;
    H.dn = 0;
    if (rc) {
      record_error(P.st, rc, (u64)gid);
      DM->needed = 0;
    } else {
      const int depth = H.depth;
      const int drop = P.per_level ? (si.kind ? P.drop_hp[si.lev] : P.drop_ll) : P.drop_global;
      int q = depth - drop;
      if (g.raw_kind >= 0 && g.keep >= 0) q = g.keep;  // decode_block(planes_to_keep=...) (blocks.py:210)
      if (q < 0) q = 0;
      if (q > depth) q = depth;
      int dn = 0;
      uint32_t d3[3] = {0, 0, 0};
      for (int pb = 0; pb < q; ++pb)
        for (int s = 0; s < nsub; ++s) {
          const int k = pb * nsub + s;
          if ((H.m3[k >> 5] >> (k & 31)) & 1u) {
            H.slot_of[dn++] = (uint8_t)k;
            d3[k >> 5] |= 1u << (k & 31);
          }
        }
      H.dn = dn;
      DM->decoded[0] = d3[0];
      DM->decoded[1] = d3[1];
      DM->decoded[2] = d3[2];
      DM->depth = (uint8_t)depth;
      DM->nsub = (uint8_t)nsub;
      DM->needed = 1;
    }
  }
  __syncwarp();
  // warp copies the parsed tables to global and builds the decode LUT
  if (lane == 0) {
    T.rc = H.rc;
    T.nsub = nsub;
    T.dn = H.dn;
    T.depth = H.depth;
    T.cw = H.cw;
    T.zr = H.zr;
    T.nst = H.nst;
    T.ntree = H.ntree;
    T.pstart = H.pstart;
  }
  if (H.rc) return;
  const int ntree = H.ntree;
  for (int i = lane; i < ntree; i += 32) {
    T.left[i] = H.left[i];
    T.right[i] = H.right[i];
    T.sym[i] = H.sym[i];
  }
  const int nseek = min(H.nst, WB_MAX_SLOTS);
  for (int i = lane; i < nseek; i += 32) T.seek[i] = H.seek[i];
  for (int i = lane; i < H.dn; i += 32) T.slot_of[i] = H.slot_of[i];
  if (H.dn == 0) return;
  // decode LUT: leaves with len <= LUT_BITS replicated, internal nodes at LUT_BITS marked
  for (int i = lane; i < ntree; i += 32) {
    const int d = H.ndepth[i];
    if (H.left[i] == -1) {
      if (d <= LUT_BITS) {
        const uint32_t first = d ? H.ncode[i] << (LUT_BITS - d) : 0u, cnt = 1u << (LUT_BITS - d);
        const uint32_t e = ((uint32_t)H.sym[i] << 8) | (uint32_t)d;
        for (uint32_t k = 0; k < cnt; ++k) T.lut[first + k] = e;
      }
    } else if (d == LUT_BITS) {
      T.lut[H.ncode[i]] = 0x80000000u | (uint32_t)i;
    }
  }
}

// Serial decode of one plane (2048 symbols) from absolute bit `pos_abs` (_kernels.py:50-88);
// returns status (0 ok, 1 truncated, 2 overrun) and the end position.  Fallback / error path.
static __device__ int decode_plane(const BitSrc& src, const BlockTab& T, u64 pos_abs, u64 end_abs, int zr, int cw,
                                   uint8_t* out, u64* end_out) {
  u64 pos = pos_abs;
  int o = 0;
  auto bit_at = [&](u64 q) -> uint32_t { return (src.word(q >> 5) >> (31 - (q & 31))) & 1u; };
  while (o < WB_PP) {
    const u64 k = pos >> 5;
    const uint32_t bits = __funnelshift_l(src.word(k + 1), src.word(k), (uint32_t)(pos & 31));
    const uint32_t e = T.lut[bits >> (32 - LUT_BITS)];
    int sym;
    u64 len;
    if (!(e & 0x80000000u)) {
      sym = (int)(e >> 8);
      len = e & 255u;
      if (pos + len > end_abs) { *end_out = pos; return 1; }
    } else {
      if (pos + LUT_BITS > end_abs) { *end_out = pos; return 1; }
      int node = (int)(e & 0xFFFFu);
      len = LUT_BITS;
      while (T.left[node] != -1) {
        if (pos + len >= end_abs) { *end_out = pos + len; return 1; }
        node = bit_at(pos + len) ? T.right[node] : T.left[node];
        ++len;
      }
      sym = T.sym[node];
    }
    pos += len;
    if (sym == zr) {
      if (pos + (u64)cw > end_abs) { *end_out = pos; return 1; }
      uint32_t counter = 0;
      for (int i = 0; i < cw; ++i) counter = (counter << 1) | bit_at(pos + i);
      pos += (u64)cw;
      if (counter == 0) {
        out[o++] = (uint8_t)sym;
      } else {
        if ((int)counter > WB_PP - o) { *end_out = pos; return 2; }
        o += (int)counter;  // zeros (buffer pre-zeroed)
      }
    } else {
      out[o++] = (uint8_t)sym;
    }
  }
  *end_out = pos;
  return 0;
}

// Faithful sequential decode_tokens (tree walk) used only on the error path.
static __device__ int decode_tokens_seq(const BitSrc& src, const int16_t* left, const int16_t* right,
                                        const int16_t* leaf, u64 start, u64 end, int zr, int cw, int nseg, u64* end_out) {
  u64 pos = start;
  for (int s = 0; s < nseg; ++s) {
    int remaining = WB_PP;
    while (remaining > 0) {
      int node = 0;
      while (left[node] != -1) {
        if (pos >= end) { *end_out = pos; return 1; }
        const uint32_t bit = (src.word(pos >> 5) >> (31 - (pos & 31))) & 1u;
        ++pos;
        node = bit ? right[node] : left[node];
      }
      const int value = leaf[node];
      if (value == zr) {
        if (pos + (u64)cw > end) { *end_out = pos; return 1; }
        uint32_t counter = 0;
        for (int i = 0; i < cw; ++i) {
          counter = (counter << 1) | ((src.word(pos >> 5) >> (31 - (pos & 31))) & 1u);
          ++pos;
        }
        if (counter == 0) --remaining;
        else {
          if ((int)counter > remaining) { *end_out = pos; return 2; }
          remaining -= (int)counter;
        }
      } else {
        --remaining;
      }
    }
  }
  *end_out = pos;
  return 0;
}

// ---- warp-parallel plane decode (self-synchronising Huffman) ------------------------------------
// Huffman codewords + fixed-width counters form a prefix-free token stream, which re-synchronises
// a few tokens after decoding starts at an arbitrary bit.  A warp decodes one plane:
//  pass 1  lane i decodes speculatively from the start of its chunk [iS, (i+1)S) and records its
//          first KREC token starts with the symbol count before each;
//  pass 2  lane i continues past its chunk until it lands on a token start recorded by a later
//          lane (sync point) -- from there that lane's speculative decode is the true one;
//  chain   lane 0 links the sync points from the plane start; chain lanes own the true token
//          sequence in [q_v, p_v); a warp scan of their symbol counts gives output offsets;
//  pass 3  chain lanes decode [q_v, p_v) again and write their symbols.
// Any inconsistency (corrupt stream) falls back to the serial decoder; a failing serial decode
// re-runs the reference's sequential algorithm to raise its exact error class.
constexpr int NWD = 4;   // warps (planes) per decode CTA
constexpr int KREC = 32; // token starts recorded per lane

struct __align__(16) PlaneScratch {
  uint8_t out[WB_PP];
  uint16_t lpos[32][KREC];
  uint16_t lcnt[32][KREC];
  uint32_t p[32], q[32], cb[32], bef[32];
  int n[32], extra[32], nrec[32], valid[32], fail[32], ok;
};

// Decode tables in shared memory (copied per CTA from the block's BlockTab).
struct TabSmem {
  uint32_t lut[LUT_SIZE];
  int16_t left[512], right[512], sym[512];
};
struct TabView {
  const TabSmem* t;
  __device__ __forceinline__ uint32_t lut(uint32_t i) const { return t->lut[i]; }
  __device__ __forceinline__ int left(int i) const { return t->left[i]; }
  __device__ __forceinline__ int right(int i) const { return t->right[i]; }
  __device__ __forceinline__ int sym(int i) const { return t->sym[i]; }
};

// Payload words: the warp's staged window in shared memory, else the container in global memory.
constexpr int PSTAGE = 512;   // staged words per warp (16 Kbit)
struct WordSrc {
  const uint32_t* w;
  u64 nfull;
  const BitSrc* src;
  const uint32_t* sw;
  u64 sw_lo;
  uint32_t sw_n;
  __device__ __forceinline__ uint32_t word(u64 k) const {
    if (k - sw_lo < sw_n) return bswap32(sw[k - sw_lo]);
    return k < nfull ? bswap32(__ldg(w + k)) : src->word(k);
  }
};

// Plane fully staged in smem (words already byte-swapped): 32-bit addressing, no bounds checks.
struct StagedSrc {
  const uint32_t* sw;   // sw[i] = big-endian word i of the window
  uint32_t base;        // bit offset of the plane start inside the window
  __device__ __forceinline__ uint32_t wrd(uint32_t i) const { return sw[i]; }
};

// Token decode from a staged plane (see dec_tok for the contract).
static __device__ __forceinline__ int dec_tok_s(const StagedSrc& src, const TabView& T, uint32_t pos, uint32_t end,
                                                int zr, int cw, uint32_t* np, uint32_t* val) {
  const uint32_t a = src.base + pos;
  const uint32_t k = a >> 5;
  const uint32_t bits = __funnelshift_l(src.wrd(k + 1), src.wrd(k), a & 31u);
  const uint32_t e = T.lut(bits >> (32 - LUT_BITS));
  int sym;
  uint32_t len;
  if (!(e & 0x80000000u)) {
    sym = (int)(e >> 8);
    len = e & 255u;
  } else {
    int node = (int)(e & 0xFFFFu);
    len = LUT_BITS;
    while (T.left(node) != -1) {
      if (len > 40) return 0;
      const uint32_t bp = a + len;
      node = ((src.wrd(bp >> 5) >> (31 - (bp & 31))) & 1u) ? T.right(node) : T.left(node);
      ++len;
    }
    sym = T.sym(node);
  }
  uint32_t count = 1, value = (uint32_t)sym, used = len;
  if (sym == zr) {
    uint32_t ctr = 0;
    if (cw) {
      if (len + cw <= 32) {
        ctr = (bits << len) >> 1 >> (31 - cw);
      } else {
        const uint32_t c0 = a + len;
        ctr = __funnelshift_l(src.wrd((c0 >> 5) + 1), src.wrd(c0 >> 5), c0 & 31u) >> (32 - cw);
      }
    }
    used += (uint32_t)cw;
    if (ctr) { count = ctr; value = 0; }
  }
  if (pos + used > end) return 0;
  *np = pos + used;
  *val = value;
  return (int)count;
}

// Uniform token-decoder front ends for decode_plane_warp.
struct GenDec {
  const WordSrc* src;
  u64 base;
  __device__ __forceinline__ int operator()(const TabView& T, uint32_t pos, uint32_t end, int zr, int cw, uint32_t* np,
                                            uint32_t* val) const;
};
struct StgDec {
  StagedSrc src;
  __device__ __forceinline__ int operator()(const TabView& T, uint32_t pos, uint32_t end, int zr, int cw, uint32_t* np,
                                            uint32_t* val) const {
    return dec_tok_s(src, T, pos, end, zr, cw, np, val);
  }
};

// One token at relative bit `pos` (absolute base + pos): returns its symbol count (>= 1) and sets
// *np / *val (0 for a zero run), or returns 0 if the token does not fit before `end`.
static __device__ __forceinline__ int dec_tok(const WordSrc& src, const TabView& T, u64 base, uint32_t pos,
                                              uint32_t end, int zr, int cw, uint32_t* np, uint32_t* val) {
  const u64 a = base + pos;
  const u64 k = a >> 5;
  const uint32_t w0 = src.word(k), w1 = src.word(k + 1);
  const uint32_t bits = __funnelshift_l(w1, w0, (uint32_t)(a & 31));
  const uint32_t e = T.lut(bits >> (32 - LUT_BITS));
  int sym;
  uint32_t len;
  if (!(e & 0x80000000u)) {
    sym = (int)(e >> 8);
    len = e & 255u;
  } else {
    int node = (int)(e & 0xFFFFu);
    len = LUT_BITS;
    while (T.left(node) != -1) {
      if (len > 40) return 0;
      const u64 bp = a + len;
      node = ((src.word(bp >> 5) >> (31 - (bp & 31))) & 1u) ? T.right(node) : T.left(node);
      ++len;
    }
    sym = T.sym(node);
  }
  uint32_t count = 1, value = (uint32_t)sym, used = len;
  if (sym == zr) {
    uint32_t ctr = 0;
    if (cw) {
      if (len + cw <= 32) {
        ctr = (bits << len) >> 1 >> (31 - cw);
      } else {
        const u64 c0 = a + len;
        const u64 kc = c0 >> 5;
        ctr = __funnelshift_l(src.word(kc + 1), src.word(kc), (uint32_t)(c0 & 31)) >> (32 - cw);
      }
    }
    used += (uint32_t)cw;
    if (ctr) { count = ctr; value = 0; }
  }
  if (pos + used > end) return 0;
  *np = pos + used;
  *val = value;
  return (int)count;
}

__device__ __forceinline__ int GenDec::operator()(const TabView& T, uint32_t pos, uint32_t end, int zr, int cw,
                                                  uint32_t* np, uint32_t* val) const {
  return dec_tok(*src, T, base, pos, end, zr, cw, np, val);
}

// Returns true if the plane [s, s+E) was decoded into W.out (symbols 0..2047).
// last: the plane's end is unknown (E = rest of the block); tokens after the 2048th symbol ignored.
template <typename Dec>
static __device__ bool decode_plane_warp(const Dec& dec, const TabView& T, PlaneScratch& W, uint32_t E, bool last,
                                         int zr, int cw) {
  const int lane = threadIdx.x & 31;
  if (E >= 65535u) return false;  // positions are kept in 16 bits
  const uint32_t S = E >= 32 ? (E + 31) / 32 : 1u;
  const uint32_t lo = min((uint32_t)lane * S, E), hi = min(lo + S, E);
  // pass 1: speculative decode of the own chunk, first KREC token starts recorded
  uint32_t pos = lo, n = 0;
  int failed = 0, nr = 0;
  while (pos < hi) {
    if (nr < KREC) {
      W.lpos[lane][nr] = (uint16_t)pos;
      W.lcnt[lane][nr] = (uint16_t)min(n, 65535u);
      ++nr;
    }
    uint32_t np, v;
    const int c = dec(T, pos, E, zr, cw, &np, &v);
    if (!c) { failed = 1; break; }
    n += (uint32_t)min(c, WB_PP);
    pos = np;
  }
  W.nrec[lane] = nr;
  W.n[lane] = (int)n;
  __syncwarp();
  // pass 2: continue into later chunks until a token start recorded by that chunk's lane
  uint32_t extra = 0, cbv = 0;
  if (!failed && pos < E) {
    uint32_t k = pos / S;
    uint32_t kend = (k + 1) * S;
    int r = 0;
    while (pos < E) {
      while (pos >= kend) { ++k; kend += S; r = 0; }
      if (k < 32) {
        const int nk = W.nrec[k];
        // advance the merge pointer through lane k's (increasing) token starts
        while (r < nk && W.lpos[k][r] < pos) ++r;
        if (r < nk && W.lpos[k][r] == pos) { cbv = W.lcnt[k][r]; break; }
      }
      uint32_t np, v;
      const int c = dec(T, pos, E, zr, cw, &np, &v);
      if (!c) { failed = 1; break; }
      extra += (uint32_t)min(c, WB_PP);
      pos = np;
    }
  }
  W.p[lane] = pos;
  W.cb[lane] = cbv;
  W.extra[lane] = (int)extra;
  W.fail[lane] = failed;
  W.valid[lane] = 0;
  __syncwarp();
  // chain from the plane start
  if (lane == 0) {
    int ok = 1, v = 0;
    W.valid[0] = 1;
    W.q[0] = 0;
    W.bef[0] = 0;
    for (int guard = 0; guard < 33; ++guard) {
      if (W.fail[v]) { ok = last ? 2 : 0; break; }  // truncated: fine only past the 2048th symbol (last plane)
      const uint32_t pv = W.p[v];
      if (pv >= E) { if (pv != E && !last) ok = 0; break; }
      const int k = (int)(pv / S);
      if (k <= v || k >= 32) { ok = 0; break; }
      W.valid[k] = 1;
      W.q[k] = pv;
      W.bef[k] = W.cb[v];
      v = k;
    }
    W.ok = ok;
  }
  __syncwarp();
  if (!W.ok) return false;
  const int cnt = W.valid[lane] ? W.n[lane] - (int)W.bef[lane] + W.extra[lane] : 0;
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (last ? total < WB_PP : total != WB_PP) return false;
  // pass 3: chain lanes write their symbols
  for (int i = lane; i < WB_PP / 16; i += 32) reinterpret_cast<uint4*>(W.out)[i] = make_uint4(0, 0, 0, 0);
  __syncwarp();
  bool ok3 = true;
  if (W.valid[lane]) {
    int o = incl - cnt;
    uint32_t pp = W.q[lane];
    const uint32_t pe = W.p[lane];
    while (pp < pe && o < WB_PP) {
      uint32_t np, v;
      const int c = dec(T, pp, E, zr, cw, &np, &v);
      if (!c || c > WB_PP - o) { ok3 = false; break; }  // truncated / run overruns the plane
      if (v) W.out[o] = (uint8_t)v;
      o += c;
      pp = np;
    }
  }
  return __all_sync(0xffffffffu, ok3);
}

// K2: grid (block, plane group); each warp decodes one plane of its block.
__global__ void __launch_bounds__(NWD * 32) k_block_planes(DecodeParams P) {
  __shared__ TabSmem TS;
  __shared__ PlaneScratch PS[NWD];
  __shared__ __align__(16) uint32_t STG[NWD][PSTAGE];
  const Geom& g = P.g;
  const int gid = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const BlockTab& G = P.tabs[gid];
  const int dn = G.dn;
  if (G.rc != 0 || (int)blockIdx.y * NWD >= dn) return;  // error recorded by K1 / not needed / no planes here
  {  // LUT + tree -> smem (16-B copies)
    const uint4* a = reinterpret_cast<const uint4*>(G.lut);
    uint4* d = reinterpret_cast<uint4*>(TS.lut);
    for (int i = tid; i < LUT_SIZE / 4; i += NWD * 32) d[i] = a[i];
    const int nt = G.ntree;
    for (int i = tid; i < nt; i += NWD * 32) { TS.left[i] = G.left[i]; TS.right[i] = G.right[i]; TS.sym[i] = G.sym[i]; }
  }
  __syncthreads();
  const int j = blockIdx.y * NWD + warp;
  if (j >= dn) return;
  const TabView T{&TS};
  const u64 boff = P.blk_off[gid];
  const u64 bend = 8ull * (boff + P.blk_len[gid]);
  const int cw = G.cw, zr = G.zr, nst = G.nst;
  const u64 pstart = G.pstart;
  const u64 s = pstart + G.seek[j];
  // The reference checks the start of every decoded plane (blocks.py:241-242), i.e. the ends of
  // planes 0..dn-2; the last decoded plane just stops after 2048 symbols.  Its work range uses
  // the next seek entry as a hint when there is one (the serial fallback reads to the block end).
  const bool last = j + 1 >= dn;
  u64 e;
  if (!last) e = pstart + G.seek[j + 1];
  else if (j + 1 < nst) e = min(bend, pstart + (u64)G.seek[j + 1] + 64);
  else e = bend;
  // stage the plane's payload words [s/32, e/32] (16-B aligned window) into smem
  const u64 nfull = P.src.nbytes >> 2;
  const u64 wlo = (s >> 5) & ~3ull;
  u64 whi = ((e >> 5) + 2 + 3) & ~3ull;
  if (whi > wlo + PSTAGE) whi = wlo + PSTAGE;
  if (whi > (nfull & ~3ull)) whi = nfull & ~3ull;
  const uint32_t nst4 = whi > wlo ? (uint32_t)((whi - wlo) / 4) : 0u;
  const uint4* gsrc = reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(P.src.data) + wlo);
  for (uint32_t i = lane; i < nst4; i += 32) {  // byte-swapped once here: smem holds big-endian words
    uint4 v = __ldg(gsrc + i);
    v.x = bswap32(v.x); v.y = bswap32(v.y); v.z = bswap32(v.z); v.w = bswap32(v.w);
    reinterpret_cast<uint4*>(STG[warp])[i] = v;
  }
  __syncwarp();
  PlaneScratch& W = PS[warp];
  bool ok = G.seek[0] == 0 && e >= s && e - s < 0xFFFFFFF0ull;
  if (ok) {
    const uint32_t E = (uint32_t)(e - s);
    // staged window covers words [wlo, wlo + 4*nst4); the plane needs up to word (e>>5) + 2
    if ((e >> 5) + 2 < wlo + 4ull * nst4) {
      StgDec d{{STG[warp], (uint32_t)(s - 32 * wlo)}};
      ok = decode_plane_warp(d, T, W, E, last, zr, cw);
    } else {
      WordSrc src{reinterpret_cast<const uint32_t*>(P.src.data), nfull, &P.src, nullptr, 0, 0};
      GenDec d{&src, s};
      ok = decode_plane_warp(d, T, W, E, last, zr, cw);
    }
  }
  uint8_t* dst = P.syms + (i64)gid * g.sym_stride_hp + (i64)G.slot_of[j] * WB_PP;
  __syncwarp();
  if (ok) {
    for (int i = lane; i < WB_PP / 16; i += 32)
      reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(W.out)[i];
  } else if (lane == 0) {
    atomicAdd(&P.st->pad, 1ull);  // fallback counter (diagnostics)
    uint4* zp = reinterpret_cast<uint4*>(dst);
    for (int i = 0; i < WB_PP / 16; ++i) zp[i] = make_uint4(0, 0, 0, 0);
    u64 endp = 0;
    const int st = decode_plane(P.src, G, s, bend, zr, cw, dst, &endp);
    if (st || (!last && endp != e) || G.seek[0] != 0) atomicOr(&P.flags[gid], 1u);
  }
}

// K2b: blocks whose planes did not decode consistently re-run the reference's sequential
// decode (blocks.py:224-242) to raise its exact error class.
__global__ void k_block_errors(DecodeParams P) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= P.batch * P.g.slots_per_image) return;
  if (!P.flags[gid]) return;
  const BlockTab& G = P.tabs[gid];
  const u64 bend = 8ull * (P.blk_off[gid] + P.blk_len[gid]);
  u64 e = 0;
  const int st = decode_tokens_seq(P.src, G.left, G.right, G.sym, G.pstart, bend, G.zr, G.cw, G.dn, &e);
  record_error(P.st, st == 1 ? WBPC_ERR_TRUNCATION : WBPC_ERR_CORRUPTION, (u64)gid);
  P.dmeta[gid].needed = 0;
}

// ---- coefficient reconstruction: symbols -> signed magnitudes in the padded subband planes ----
struct ReconParams {
  Geom g;
  const uint8_t* syms;
  const DecMeta* dmeta;
  int32_t* coef;
};

__global__ void __launch_bounds__(256) k_block_reconstruct(ReconParams P) {
  const Geom& g = P.g;
  const int gid = blockIdx.x;
  const DecMeta dm = P.dmeta[gid];
  if (!dm.needed) return;
  const int b = gid / g.slots_per_image;
  const int slot = gid - b * g.slots_per_image;
  const SlotInfo si = slot_info(g, slot);
  const LevelGeom& lg = g.lv[si.lev];
  const int nsub = dm.nsub, depth = dm.depth;
  const uint8_t* symbase = P.syms + (i64)gid * g.sym_stride_hp;
  int32_t* cbase = P.coef + (i64)b * g.img_stride + (i64)si.c * g.chan_stride;
  const int y0 = si.r * WB_DIM, x0 = si.col * WB_DIM;
  for (int s = 0; s < nsub; ++s) {
    int32_t* plane = cbase + lg.off[si.kind ? 1 + s : 0];
    auto symb = [&](int pb, int k) -> uint32_t {  // symbol of plane pb (0 if not decoded / past depth)
      if (pb >= depth) return 0u;
      const int sl = pb * nsub + s;
      if (!((dm.decoded[sl >> 5] >> (sl & 31)) & 1u)) return 0u;
      return symbase[(i64)sl * WB_PP + k];
    };
    for (int k = threadIdx.x; k < WB_PP; k += 256) {
      // stream position k -> area (r, c) (bitplanes.py:159-166 for 128x128)
      const int r = 2 * (k >> 6) + (k & 1), c = (k >> 1) & 31;
      uint32_t mag[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      const uint32_t sign = symb(0, k);
      // magnitude planes 1..depth-1, four at a time: byte p of x = symbol of plane pb+p; for bit i,
      // ((x >> i) & 0x01010101) * 0x08040201 >> 24 packs the 4 plane bits MSB first
      for (int pb = 1; pb < depth; pb += 4) {
        const uint32_t x = symb(pb, k) | (symb(pb + 1, k) << 8) | (symb(pb + 2, k) << 16) | (symb(pb + 3, k) << 24);
        if (!x) continue;
        const int shl = depth - 4 - pb;  // weight of the 4th plane of the group (may be < 0)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t nib = (((x >> i) & 0x01010101u) * 0x08040201u) >> 24;
          mag[i] |= shl >= 0 ? nib << shl : nib >> (-shl);
        }
      }
      int v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = ((sign >> i) & 1u) ? -(int)mag[i] : (int)mag[i];
      int32_t* pp = plane + (i64)(y0 + 2 * r) * lg.pw + x0 + 4 * c;
      *reinterpret_cast<int4*>(pp) = make_int4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<int4*>(pp + lg.pw) = make_int4(v[4], v[5], v[6], v[7]);
    }
  }
}

// ---- ABI mirror of _kernels.decode_tokens (single thread, reference tree walk) ---------------
__global__ void k_decode_tokens(const uint8_t* payload, u64 nbytes, i64 start_bit, i64 end_bit, const int32_t* left,
                                const int32_t* right, const int32_t* leaf, int zr, int cw, const i64* seg_len, int nseg,
                                uint8_t* out, i64* seg_starts, i64* result) {
  if (threadIdx.x || blockIdx.x) return;
  BitSrc src{payload, nbytes};
  i64 bitpos = start_bit, oi = 0;
  for (int s = 0; s < nseg; ++s) {
    seg_starts[s] = bitpos - start_bit;
    i64 remaining = seg_len[s];
    while (remaining > 0) {
      int node = 0;
      while (left[node] != -1) {
        if (bitpos >= end_bit) { result[0] = 1; result[1] = bitpos; return; }
        uint32_t bit = src.bits((u64)bitpos, 1);
        ++bitpos;
        node = bit ? right[node] : left[node];
      }
      int value = leaf[node];
      if (value == zr) {
        if (bitpos + cw > end_bit) { result[0] = 1; result[1] = bitpos; return; }
        i64 counter = 0;
        for (int i = 0; i < cw; ++i) { counter = (counter << 1) | src.bits((u64)bitpos, 1); ++bitpos; }
        if (counter == 0) { out[oi++] = (uint8_t)value; --remaining; }
        else {
          if (counter > remaining) { result[0] = 2; result[1] = bitpos; return; }
          for (i64 i = 0; i < counter; ++i) out[oi++] = 0;
          remaining -= counter;
        }
      } else { out[oi++] = (uint8_t)value; --remaining; }
    }
  }
  result[0] = 0;
  result[1] = bitpos;
}

// ------------------------------------------------------------------------------------ launch
size_t block_tab_bytes() { return sizeof(BlockTab); }

cudaError_t launch_index_check(const Geom& g, int batch, const uint8_t* data, const u64* img_off, u64* blk_off,
                               uint32_t* blk_len, DevStatus* st, cudaStream_t s) {
  IndexParams P;
  P.g = g;
  P.batch = batch;
  P.data = data;
  P.img_off = img_off;
  P.blk_off = blk_off;
  P.blk_len = blk_len;
  P.st = st;
  i64 n = (i64)batch * g.slots_per_image;
  prof_mark("index_check", s);
  k_index_check<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_decode_blocks(const Geom& g, int batch, int level, int drop_global, const int* drop_hp,
                                 int drop_ll, int per_level, const uint8_t* data, u64 nbytes, const u64* blk_off,
                                 const uint32_t* blk_len, BlockTab* tabs, uint32_t* flags, uint8_t* syms,
                                 DecMeta* dmeta, int32_t* coef, DevStatus* st, cudaStream_t s,
                                 const uint8_t* need) {
  DecodeParams P;
  P.need = need;
  P.stage_bytes = 0;
  P.g = g;
  P.batch = batch;
  P.level = level;
  P.drop_global = drop_global;
  P.drop_ll = drop_ll;
  for (int i = 0; i <= WB_MAXL; ++i) P.drop_hp[i] = (per_level && i >= 1 && drop_hp) ? drop_hp[i - 1] : 0;
  P.per_level = per_level;
  P.src.data = data;
  P.src.nbytes = nbytes;
  P.blk_off = blk_off;
  P.blk_len = blk_len;
  P.tabs = tabs;
  P.flags = flags;
  P.syms = syms;
  P.dmeta = dmeta;
  P.st = st;
  const int nblocks = batch * g.slots_per_image;
  cudaMemsetAsync(flags, 0, 4ull * nblocks, s);
  prof_mark("block_header", s);
  k_block_header<<<(nblocks + HW - 1) / HW, HW * 32, 0, s>>>(P);
  prof_mark("block_decode", s);
  dim3 grid(nblocks, (3 * WB_MAX_DEPTH + NWD - 1) / NWD);
  k_block_planes<<<grid, NWD * 32, 0, s>>>(P);
  prof_mark("block_errors", s);
  k_block_errors<<<(nblocks + 127) / 128, 128, 0, s>>>(P);
  ReconParams R;
  R.g = g;
  R.syms = syms;
  R.dmeta = dmeta;
  R.coef = coef;
  prof_mark("block_reconstruct", s);
  k_block_reconstruct<<<nblocks, 256, 0, s>>>(R);
  return cudaGetLastError();
}

// decode_region (container.py:338-390): a block is decoded iff its tile intersects the per-level
// box of its level (_stitch's tile ranges, container.py:261-275, with the box clamped to the LL
// dims of that level).  Everything else is skipped, so corrupt blocks outside raise nothing.
__global__ void k_region_need(Geom g, int level, RegionBoxes B, uint8_t* need) {
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= g.slots_per_image) return;
  const SlotInfo si = slot_info(g, slot);
  uint8_t n = 0;
  if (si.kind == 0 || si.lev > level) {
    const LevelGeom& lg = g.lv[si.lev];
    const int r1 = min(B.r1[si.lev], lg.h), c1 = min(B.c1[si.lev], lg.w);
    const int tr0 = B.r0[si.lev] / WB_DIM, tr1 = (r1 + WB_DIM - 1) / WB_DIM;
    const int tc0 = B.c0[si.lev] / WB_DIM, tc1 = (c1 + WB_DIM - 1) / WB_DIM;
    n = si.r >= tr0 && si.r < tr1 && si.col >= tc0 && si.col < tc1;
  }
  need[slot] = n;
}

cudaError_t launch_region_need(const Geom& g, int level, const RegionBoxes& B, uint8_t* need, cudaStream_t s) {
  k_region_need<<<(g.slots_per_image + 127) / 128, 128, 0, s>>>(g, level, B, need);
  return cudaGetLastError();
}

// Header parse only (K1), every block (container_info parses all slots, container.py:435-437).
cudaError_t launch_block_headers(const Geom& g, int batch, const uint8_t* data, u64 nbytes, const u64* blk_off,
                                 const uint32_t* blk_len, BlockTab* tabs, DecMeta* dmeta, DevStatus* st,
                                 cudaStream_t s) {
  DecodeParams P;
  memset(&P, 0, sizeof P);
  P.g = g;
  P.batch = batch;
  P.level = 0;
  P.src.data = data;
  P.src.nbytes = nbytes;
  P.blk_off = blk_off;
  P.blk_len = blk_len;
  P.tabs = tabs;
  P.dmeta = dmeta;
  P.st = st;
  const int nblocks = batch * g.slots_per_image;
  prof_mark("block_header", s);
  k_block_header<<<(nblocks + HW - 1) / HW, HW * 32, 0, s>>>(P);
  return cudaGetLastError();
}

// container_info (container.py:435-440): per-block depth and header bits (payload_start).
__global__ void k_block_summary(const BlockTab* tabs, const u64* blk_off, int n, int32_t* depth, uint32_t* hbits) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  depth[i] = tabs[i].depth;
  hbits[i] = (uint32_t)(tabs[i].pstart - 8ull * blk_off[i]);
}

cudaError_t launch_block_summary(const BlockTab* tabs, const u64* blk_off, int n, int32_t* depth, uint32_t* hbits,
                                 cudaStream_t s) {
  k_block_summary<<<(n + 127) / 128, 128, 0, s>>>(tabs, blk_off, n, depth, hbits);
  return cudaGetLastError();
}

cudaError_t launch_decode_tokens(const uint8_t* payload, u64 nbytes, i64 start_bit, i64 end_bit, const int32_t* left,
                                 const int32_t* right, const int32_t* leaf, int zr, int cw, const i64* seg_len,
                                 int nseg, uint8_t* out, i64* seg_starts, i64* result, cudaStream_t s) {
  k_decode_tokens<<<1, 1, 0, s>>>(payload, nbytes, start_bit, end_bit, left, right, leaf, zr, cw, seg_len, nseg, out,
                                  seg_starts, result);
  return cudaGetLastError();
}

}  // namespace wb
