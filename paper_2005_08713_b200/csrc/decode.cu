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
    return;
  }
  P.blk_off[gi] = base + off;
  P.blk_len[gi] = (uint32_t)len;
}

// ---- bit reader over the container buffer ------------------------------------------------------
struct BitSrc {
  const uint8_t* data;
  u64 nbytes;  // bytes valid in `data` (whole buffer)
  __device__ __forceinline__ uint32_t word(u64 k) const {  // big-endian word k (bytes 4k..4k+3)
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

struct TreeSmem {
  int16_t left[512], right[512], sym[512];
  uint8_t depth[512];
  uint32_t code[512];
  uint32_t lut[LUT_SIZE];  // leaf: (sym << 8) | len ; long code: 0x80000000 | node
  uint32_t seek[WB_MAX_SLOTS];
  uint64_t ends[WB_MAX_SLOTS];
  int stat[WB_MAX_SLOTS];
  int slot_of[WB_MAX_SLOTS];
  int hdr[12];
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
  uint8_t* syms;        // stride g.sym_stride_hp per block
  DecMeta* dmeta;
  DevStatus* st;
};

// Emit helper: buffered 4-byte stores of decoded symbols (slot buffers are 2048-aligned)
struct SymOut {
  uint8_t* p;
  uint32_t acc;
  int na;
  int o;
  __device__ __forceinline__ void put(uint32_t s) {
    acc |= s << (8 * na);
    if (++na == 4) {
      *reinterpret_cast<uint32_t*>(p + o) = acc;
      o += 4;
      na = 0;
      acc = 0;
    }
  }
  __device__ __forceinline__ void zeros(int n) {
    while (n > 0 && na) { put(0); --n; }
    while (n >= 16 && (o & 15) == 0) {
      *reinterpret_cast<uint4*>(p + o) = make_uint4(0, 0, 0, 0);
      o += 16;
      n -= 16;
    }
    while (n >= 4) {
      *reinterpret_cast<uint32_t*>(p + o) = 0;
      o += 4;
      n -= 4;
    }
    while (n > 0) { put(0); --n; }
  }
};

// Decode `nsym` symbols of one plane from bit `pos` (absolute) with the LUT; returns status
// (0 ok, 1 truncated, 2 overrun) and the end position.  Mirrors _kernels.py:50-88.
static __device__ int decode_plane(const BitSrc& src, const TreeSmem& T, u64 pos, u64 end, int zr, int cw, uint8_t* out,
                            bool write, u64* end_out) {
  SymOut so{out, 0u, 0, 0};
  int remaining = WB_PP;
  while (remaining > 0) {
    uint32_t peek = src.bits(pos, LUT_BITS);
    uint32_t e = T.lut[peek];
    int sym, len;
    if (!(e & 0x80000000u)) {
      sym = (int)(e >> 8);
      len = (int)(e & 0xFFu);
      if (pos + (u64)len > end) { *end_out = pos; return 1; }
      pos += (u64)len;
    } else {
      if (pos + LUT_BITS > end) { *end_out = pos; return 1; }
      int node = (int)(e & 0xFFFFu);
      pos += LUT_BITS;
      while (T.left[node] != -1) {
        if (pos >= end) { *end_out = pos; return 1; }
        uint32_t bit = src.bits(pos, 1);
        ++pos;
        node = bit ? T.right[node] : T.left[node];
      }
      sym = T.sym[node];
    }
    if (sym == zr) {
      if (pos + (u64)cw > end) { *end_out = pos; return 1; }
      uint32_t counter = src.bits(pos, cw);
      pos += (u64)cw;
      if (counter == 0) {
        if (write) so.put((uint32_t)sym);
        --remaining;
      } else {
        if ((int)counter > remaining) { *end_out = pos; return 2; }
        if (write) so.zeros((int)counter);
        remaining -= (int)counter;
      }
    } else {
      if (write) so.put((uint32_t)sym);
      --remaining;
    }
  }
  *end_out = pos;
  return 0;
}

// Faithful sequential decode_tokens (tree walk) used only on the error path and by the ABI mirror.
static __device__ int decode_tokens_seq(const BitSrc& src, const int16_t* left, const int16_t* right, const int16_t* leaf,
                                 u64 start, u64 end, int zr, int cw, int nseg, const u64* seek_rel, u64* end_out,
                                 int* bad_seek) {
  u64 pos = start;
  *bad_seek = 0;
  for (int s = 0; s < nseg; ++s) {
    if (seek_rel && pos - start != seek_rel[s]) *bad_seek = 1;
    int remaining = WB_PP;
    while (remaining > 0) {
      int node = 0;
      while (left[node] != -1) {
        if (pos >= end) { *end_out = pos; return 1; }
        uint32_t bit = src.bits(pos, 1);
        ++pos;
        node = bit ? right[node] : left[node];
      }
      int value = leaf[node];
      if (value == zr) {
        if (pos + (u64)cw > end) { *end_out = pos; return 1; }
        uint32_t counter = src.bits(pos, cw);
        pos += (u64)cw;
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

// Header parse of blocks.py:150-192 (+ read_tree entropy.py:272-310). Lane 0 only.
// Returns 0 or an error status; fills T and hdr fields.
static __device__ int parse_block_header(const BitSrc& src, u64 bstart, u64 bend, int nsub, TreeSmem& T, int* depth_o,
                                  int* cw_o, int* zr_o, uint32_t* mask3, int* nstored_o, u64* payload_o,
                                  int* ntree_o) {
  u64 pos = bstart;
#define NEED(n)                      \
  if (pos + (u64)(n) > bend) return WBPC_ERR_BLOCK_PARSE;
  NEED(6);
  int depth = (int)src.bits(pos, 6);
  pos += 6;
  if (depth < 1) return WBPC_ERR_BLOCK_PARSE;
  NEED(5);
  int cw = (int)src.bits(pos, 5);
  pos += 5;
  NEED(8);
  int zr = (int)src.bits(pos, 8);
  pos += 8;
  mask3[0] = mask3[1] = mask3[2] = 0;
  // masks in (s, b) order; keep them as bit (b*nsub + s).  depth <= 63 from 6 bits.
  int cnt = 0;
  uint64_t mk[3] = {0, 0, 0};
  for (int s = 0; s < nsub; ++s) {
    NEED(depth);
    u64 v = 0;
    if (depth > 32) {
      v = ((u64)src.bits(pos, depth - 32) << 32) | src.bits(pos + depth - 32, 32);
    } else {
      v = src.bits(pos, depth);
    }
    pos += depth;
    mk[s] = v;  // MSB = plane 0
    cnt += __popcll(v);
  }
  *depth_o = depth;
  *cw_o = cw;
  *zr_o = zr;
  *nstored_o = cnt;
  int ntree = 0;
  if (cnt) {
    // read_tree
    int pending[512];
    int np = 0;
    bool first = true;
    unsigned seen[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    while (first || np) {
      first = false;
      if (pos + 1 > bend) return WBPC_ERR_MALFORMED_TREE;
      uint32_t bit = src.bits(pos, 1);
      pos += 1;
      int idx = ntree;
      if (idx > 511) return WBPC_ERR_MALFORMED_TREE;
      if (bit) {
        if (pos + 8 > bend) return WBPC_ERR_MALFORMED_TREE;
        int s = (int)src.bits(pos, 8);
        pos += 8;
        if ((seen[s >> 5] >> (s & 31)) & 1) return WBPC_ERR_MALFORMED_TREE;
        seen[s >> 5] |= 1u << (s & 31);
        T.left[idx] = -1; T.right[idx] = -1; T.sym[idx] = (int16_t)s;
      } else {
        T.left[idx] = -2; T.right[idx] = -2; T.sym[idx] = -1;
      }
      ++ntree;
      if (idx > 0) {
        int parent = pending[np - 1];
        if (T.left[parent] == -2) T.left[parent] = (int16_t)idx;
        else { T.right[parent] = (int16_t)idx; --np; }
      }
      if (!bit) pending[np++] = idx;
    }
    // depths/codes in preorder (parents precede children); CodeLengthError (entropy.py:97-98)
    T.depth[0] = 0;
    T.code[0] = 0;
    for (int i = 0; i < ntree; ++i) {
      if (T.left[i] == -1) continue;
      if (T.depth[i] >= 32) return WBPC_ERR_CODE_LENGTH;
      int l = T.left[i], r = T.right[i];
      T.depth[l] = T.depth[r] = (uint8_t)(T.depth[i] + 1);
      T.code[l] = T.code[i] << 1;
      T.code[r] = (T.code[i] << 1) | 1u;
    }
  }
  *ntree_o = ntree;
  NEED(16);
  int seek_count = (int)src.bits(pos, 16);
  pos += 16;
  if (seek_count != cnt) return WBPC_ERR_CORRUPTION;
  int t = seek_bits(nsub, depth);
  uint32_t prev = 0;
  bool decreasing = false;
  for (int i = 0; i < cnt; ++i) {
    NEED(t);
    uint32_t v = src.bits(pos, t);
    pos += t;
    if (i < WB_MAX_SLOTS) T.seek[i] = v;
    if (i && v < prev) decreasing = true;
    prev = v;
  }
  if (decreasing) return WBPC_ERR_CORRUPTION;  // blocks.py:177-178
  *payload_o = pos;
  T.hdr[11] = (int)(pos - bstart);
  // convert masks to bit (b*nsub+s)
  for (int s = 0; s < nsub; ++s)
    for (int b = 0; b < depth; ++b)
      if ((mk[s] >> (depth - 1 - b)) & 1ull) {
        int k = b * nsub + s;
        if (k < WB_MAX_SLOTS) mask3[k >> 5] |= 1u << (k & 31);
      }
  return 0;
#undef NEED
}

__global__ void __launch_bounds__(32) k_block_decode(DecodeParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TreeSmem& T = *reinterpret_cast<TreeSmem*>(smem_raw);
  const Geom& g = P.g;
  const int gid = blockIdx.x;
  const int b = gid / g.slots_per_image;
  const int slot = gid - b * g.slots_per_image;
  const SlotInfo si = slot_info(g, slot);
  const int lane = threadIdx.x;
  DecMeta* DM = P.dmeta + gid;
  const bool needed = si.kind == 0 || si.lev > P.level;
  if (!needed) {
    if (lane == 0) DM->needed = 0;
    return;
  }
  const int nsub = si.kind ? 3 : 1;
  const u64 bstart = 8ull * P.blk_off[gid];
  const u64 bend = bstart + 8ull * P.blk_len[gid];
  if (lane == 0) {
    int depth = 0, cw = 0, zr = 0, nst = 0, ntree = 0;
    u64 pstart = 0;
    uint32_t m3[3];
    int rc = parse_block_header(P.src, bstart, bend, nsub, T, &depth, &cw, &zr, m3, &nst, &pstart, &ntree);
    if (!rc && depth > WB_MAX_DEPTH) rc = WBPC_ERR_UNSUPPORTED;  // magnitudes beyond int32
    T.hdr[0] = rc;
    T.hdr[1] = depth;
    T.hdr[2] = cw;
    T.hdr[3] = zr;
    T.hdr[4] = nst;
    T.hdr[5] = ntree;
    T.hdr[6] = (int)(pstart - bstart);
    T.hdr[7] = (int)m3[0];
    T.hdr[8] = (int)m3[1];
    T.hdr[9] = (int)m3[2];
    if (!rc) {
      int drop = P.per_level ? (si.kind ? P.drop_hp[si.lev] : P.drop_ll) : P.drop_global;
      int q = depth - drop;
      if (q < 0) q = 0;
      if (q > depth) q = depth;
      int n = 0, dn = 0;
      for (int pb = 0; pb < depth; ++pb)
        for (int s = 0; s < nsub; ++s) {
          int k = pb * nsub + s;
          if ((m3[k >> 5] >> (k & 31)) & 1u) {
            if (pb < q) { T.slot_of[dn] = k; ++dn; }
            ++n;
          }
        }
      T.hdr[10] = dn;
    }
  }
  __syncwarp();
  const int rc0 = T.hdr[0];
  if (rc0) {
    if (lane == 0) {
      record_error(P.st, rc0, (u64)gid);
      DM->needed = 0;
    }
    return;
  }
  const int depth = T.hdr[1], cw = T.hdr[2], zr = T.hdr[3], ntree = T.hdr[5], dn = T.hdr[10];
  const u64 pstart = bstart + (u64)T.hdr[6];
  uint8_t* symbase = P.syms + (i64)gid * g.sym_stride_hp;
  if (dn) {
    // LUT (leaf len <= LUT_BITS: replicate; internal node at depth LUT_BITS: long-code marker)
    for (int i = lane; i < ntree; i += 32) {
      int d = T.depth[i];
      if (T.left[i] == -1) {
        if (d <= LUT_BITS) {
          uint32_t first = T.code[i] << (LUT_BITS - d), cnt = 1u << (LUT_BITS - d);
          if (d == 0) first = 0;
          uint32_t e = ((uint32_t)T.sym[i] << 8) | (uint32_t)d;
          for (uint32_t k = 0; k < cnt; ++k) T.lut[first + k] = e;
        }
      } else if (d == LUT_BITS) {
        T.lut[T.code[i]] = 0x80000000u | (uint32_t)i;
      }
    }
    __syncwarp();
    for (int j = lane; j < dn; j += 32) {
      u64 endp = 0;
      int st = decode_plane(P.src, T, pstart + T.seek[j], bend, zr, cw, symbase + (i64)T.slot_of[j] * WB_PP, true,
                            &endp);
      T.stat[j] = st;
      T.ends[j] = endp;
    }
    __syncwarp();
    if (lane == 0) {
      bool ok = T.seek[0] == 0;
      for (int j = 0; j < dn && ok; ++j) {
        if (T.stat[j]) ok = false;
        if (j + 1 < dn && T.ends[j] != pstart + T.seek[j + 1]) ok = false;
      }
      if (!ok) {
        // reference order: sequential decode first (status -> Truncation/Corruption), then seek check
        u64 sr[WB_MAX_SLOTS];
        for (int j = 0; j < dn; ++j) sr[j] = T.seek[j];
        u64 e = 0;
        int bad = 0;
        int st = decode_tokens_seq(P.src, T.left, T.right, T.sym, pstart, bend, zr, cw, dn, sr, &e, &bad);
        int code = st == 1 ? WBPC_ERR_TRUNCATION : st == 2 ? WBPC_ERR_CORRUPTION : WBPC_ERR_CORRUPTION;
        record_error(P.st, code, (u64)gid);
        DM->needed = 0;
      } else {
        DM->needed = 1;
      }
    }
  } else if (lane == 0) {
    DM->needed = 1;
  }
  if (lane == 0) {
    uint32_t d3[3] = {0, 0, 0};
    for (int j = 0; j < dn; ++j) d3[T.slot_of[j] >> 5] |= 1u << (T.slot_of[j] & 31);
    DM->decoded[0] = d3[0];
    DM->decoded[1] = d3[1];
    DM->decoded[2] = d3[2];
    DM->depth = (uint8_t)depth;
    DM->nsub = (uint8_t)nsub;
  }
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
    for (int k = threadIdx.x; k < WB_PP; k += 256) {
      // stream position k -> area (r, c) (bitplanes.py:159-166 for 128x128)
      const int r = 2 * (k >> 6) + (k & 1), c = (k >> 1) & 31;
      uint32_t mag[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      uint32_t sign = 0;
      for (int pb = 0; pb < depth; ++pb) {
        const int sl = pb * nsub + s;
        if (!((dm.decoded[sl >> 5] >> (sl & 31)) & 1u)) continue;
        uint32_t sym = symbase[(i64)sl * WB_PP + k];
        if (!sym) continue;
        if (pb == 0) { sign = sym; continue; }
        const int sh = depth - 1 - pb;
#pragma unroll
        for (int i = 0; i < 8; ++i) mag[i] |= ((sym >> i) & 1u) << sh;
      }
      int4 top, bot;
      int v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = ((sign >> i) & 1u) ? -(int)mag[i] : (int)mag[i];
      top = make_int4(v[0], v[1], v[2], v[3]);
      bot = make_int4(v[4], v[5], v[6], v[7]);
      int32_t* p = plane + (i64)(y0 + 2 * r) * lg.pw + x0 + 4 * c;
      *reinterpret_cast<int4*>(p) = top;
      *reinterpret_cast<int4*>(p + lg.pw) = bot;
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
size_t decode_smem_bytes() { return sizeof(TreeSmem); }

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
                                 const uint32_t* blk_len, uint8_t* syms, DecMeta* dmeta, int32_t* coef,
                                 DevStatus* st, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_block_decode, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TreeSmem));
    attr = true;
  }
  DecodeParams P;
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
  P.syms = syms;
  P.dmeta = dmeta;
  P.st = st;
  const int nblocks = batch * g.slots_per_image;
  prof_mark("block_decode", s);
  k_block_decode<<<nblocks, 32, sizeof(TreeSmem), s>>>(P);
  ReconParams R;
  R.g = g;
  R.syms = syms;
  R.dmeta = dmeta;
  R.coef = coef;
  prof_mark("block_reconstruct", s);
  k_block_reconstruct<<<nblocks, 256, 0, s>>>(R);
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
