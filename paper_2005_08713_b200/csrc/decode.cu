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


// ---- TMA bulk copy global -> shared with an mbarrier (sm_90+/sm_100a) -------------------------
static __device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
static __device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
static __device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
static __device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
static __device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(phase) : "memory");
  }
}

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
  uint64_t bar;
  uint32_t stage_lo_word, stage_nwords;
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
  uint32_t stage_bytes; // shared-memory staging window per block (multiple of 16)
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

// Register bit buffer over the container: `buf` holds `nb` valid bits, MSB first; refills
// one big-endian word at a time (one global load per 32 bits consumed).
struct BitBuf {
  const BitSrc* src;
  uint64_t buf;
  int nb;
  u64 next;  // next word index to load
  u64 pos;   // absolute bit position of the first bit in buf
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
  __device__ __forceinline__ uint32_t peek(int n) const { return (uint32_t)(buf >> (64 - n)); }
  __device__ __forceinline__ void skip(int n) {
    buf <<= n;
    nb -= n;
    pos += (u64)n;
  }
  // read n <= 32 bits (refills as needed)
  __device__ __forceinline__ uint32_t get(int n) {
    if (n == 0) return 0;
    if (nb < n) refill();
    uint32_t v = peek(n);
    skip(n);
    refill();
    return v;
  }
};

// Decode one plane (2048 symbols) starting at absolute bit `pos`, with `end` the block's end bit;
// returns status (0 ok, 1 truncated, 2 overrun) and the end position (_kernels.py:50-88).
// Hot loop is 32-bit only: a 3-word window (w0:w1 funnel-shifted by the bit offset gives the next
// 32 stream bits), the zero-run counter is read predicated from the same 32 bits (code <= LUT_BITS
// and counter <= 22 bits), runs only advance the output position (plane buffer zeroed by the
// caller), and one 4-byte word is stored per 4 output positions.
static __device__ int decode_plane(const BitSrc& src, const TreeSmem& T, u64 pos_abs, u64 end_abs, int zr, int cw,
                                   uint8_t* out, u64* end_out) {
  auto ld = [&](u64 k) -> uint32_t { return src.word(k); };
  const u64 base = pos_abs & ~31ull;         // window origin (word aligned)
  const u64 end64 = end_abs - base;
  const uint32_t end = end64 > 0xFFFFFFF0ull ? 0xFFFFFFF0u : (uint32_t)end64;
  uint32_t pos = (uint32_t)(pos_abs - base);  // bit position relative to `base`
  u64 wk = base >> 5;                          // word index of w0
  uint32_t w0 = ld(wk), w1 = ld(wk + 1), w2 = ld(wk + 2);
  uint32_t wsh = 0;                            // bits of `pos` already shifted out of the window (multiple of 32)
  const bool fast_cw = cw <= 22;
  const uint32_t cwmask = cw ? (0xFFFFFFFFu >> (32 - cw)) : 0u;
  uint32_t* ow = reinterpret_cast<uint32_t*>(out);
  uint32_t acc = 0;
  int o = 0;
  while (o < WB_PP) {
    const uint32_t off = pos - wsh;            // 0..31
    const uint32_t bits = __funnelshift_l(w1, w0, off);
    uint32_t e = T.lut[bits >> (32 - LUT_BITS)];
    int sym, len;
    uint32_t counter;
    if (!(e & 0x80000000u) && fast_cw) {
      sym = (int)(e >> 8);
      len = (int)(e & 0xFFu);
      const bool isz = sym == zr;
      const uint32_t used = (uint32_t)len + (isz ? (uint32_t)cw : 0u);
      if (pos + used > end) { *end_out = base + pos; return 1; }
      counter = isz ? ((bits << len) >> 1 >> (31 - cw)) & cwmask : 0u;
      pos += used;
    } else {
      // slow path: long codeword (tree walk from the LUT node) and/or wide counter
      auto bit_at = [&](uint32_t p) -> uint32_t {
        u64 q = base + p;
        return (src.word(q >> 5) >> (31 - (q & 31))) & 1u;
      };
      if (e & 0x80000000u) {
        if (pos + LUT_BITS > end) { *end_out = base + pos; return 1; }
        int node = (int)(e & 0xFFFFu);
        len = LUT_BITS;
        while (T.left[node] != -1) {
          if (pos + (uint32_t)len >= end) { *end_out = base + pos + len; return 1; }
          node = bit_at(pos + (uint32_t)len) ? T.right[node] : T.left[node];
          ++len;
        }
        sym = T.sym[node];
      } else {
        sym = (int)(e >> 8);
        len = (int)(e & 0xFFu);
        if (pos + (uint32_t)len > end) { *end_out = base + pos; return 1; }
      }
      pos += (uint32_t)len;
      counter = 0;
      if (sym == zr) {
        if (pos + (uint32_t)cw > end) { *end_out = base + pos; return 1; }
        for (int i = 0; i < cw; ++i) counter = (counter << 1) | bit_at(pos + i);
        pos += (uint32_t)cw;
      }
    }
    // advance the window (at most one word per fast-path symbol; loop for the slow path)
    while (pos - wsh >= 32) {
      w0 = w1;
      w1 = w2;
      wsh += 32;
      w2 = ld(wk + 3 + (wsh >> 5) - 1);
    }
    const int count = counter ? (int)counter : 1;
    if (count > WB_PP - o) { *end_out = base + pos; return 2; }
    const uint32_t value = counter ? 0u : (uint32_t)sym;
    const int q0 = o >> 2;
    acc |= value << (8 * (o & 3));
    o += count;
    if ((o >> 2) != q0) {
      ow[q0] = acc;
      acc = 0;
    }
  }
  *end_out = base + pos;
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
static __device__ int parse_block_header(const BitSrc& src, u64 bstart, u64 bend, int nsub, TreeSmem& T,
                                         int* depth_o, int* cw_o, int* zr_o, uint32_t* mask3, int* nstored_o,
                                         u64* payload_o, int* ntree_o) {
  BitBuf bb;
  bb.init(src, bstart);
#define NEED(n)                         \
  if (bb.pos + (u64)(n) > bend) return WBPC_ERR_BLOCK_PARSE;
  NEED(6);
  int depth = (int)bb.get(6);
  if (depth < 1) return WBPC_ERR_BLOCK_PARSE;
  NEED(5);
  int cw = (int)bb.get(5);
  NEED(8);
  int zr = (int)bb.get(8);
  mask3[0] = mask3[1] = mask3[2] = 0;
  // masks in (s, b) order; kept as bit (b*nsub + s).  depth <= 63 from 6 bits.
  int cnt = 0;
  uint64_t mk[3] = {0, 0, 0};
  for (int s = 0; s < nsub; ++s) {
    NEED(depth);
    u64 v;
    if (depth > 32) {
      v = (u64)bb.get(depth - 32) << 32;
      v |= bb.get(32);
    } else {
      v = bb.get(depth);
    }
    mk[s] = v;  // MSB = plane 0
    cnt += __popcll(v);
  }
  *depth_o = depth;
  *cw_o = cw;
  *zr_o = zr;
  *nstored_o = cnt;
  int ntree = 0;
  if (cnt) {
    // read_tree (entropy.py:272-310)
    int16_t pending[512];
    int np = 0;
    bool first = true;
    unsigned seen[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    while (first || np) {
      first = false;
      if (bb.pos + 1 > bend) return WBPC_ERR_MALFORMED_TREE;
      uint32_t bit = bb.get(1);
      int idx = ntree;
      if (idx > 511) return WBPC_ERR_MALFORMED_TREE;
      if (bit) {
        if (bb.pos + 8 > bend) return WBPC_ERR_MALFORMED_TREE;
        int s = (int)bb.get(8);
        if ((seen[s >> 5] >> (s & 31)) & 1u) return WBPC_ERR_MALFORMED_TREE;
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
      if (!bit) pending[np++] = (int16_t)idx;
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
  int seek_count = (int)bb.get(16);
  if (seek_count != cnt) return WBPC_ERR_CORRUPTION;
  int t = seek_bits(nsub, depth);
  uint32_t prev = 0;
  bool decreasing = false;
  for (int i = 0; i < cnt; ++i) {
    NEED(t);
    uint32_t v = bb.get(t);
    if (i < WB_MAX_SLOTS) T.seek[i] = v;
    if (i && v < prev) decreasing = true;
    prev = v;
  }
  if (decreasing) return WBPC_ERR_CORRUPTION;  // blocks.py:177-178
  *payload_o = bb.pos;
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
  const u64 boff = P.blk_off[gid];
  const u64 bstart = 8ull * boff;
  const u64 bend = bstart + 8ull * P.blk_len[gid];
  // stage the block's bytes into shared memory with one TMA bulk copy (16-B aligned interior)
  uint32_t* stage = reinterpret_cast<uint32_t*>(smem_raw + ((sizeof(TreeSmem) + 127) & ~(size_t)127));
  {
    const u64 a0 = boff & ~15ull;
    u64 a1 = boff + P.blk_len[gid];
    if (a1 > a0 + P.stage_bytes) a1 = a0 + P.stage_bytes;
    if (a1 > P.src.nbytes) a1 = P.src.nbytes;
    a1 &= ~15ull;
    const uint32_t nbytes = a1 > a0 ? (uint32_t)(a1 - a0) : 0u;
    if (lane == 0) {
      T.stage_lo_word = (uint32_t)0;
      T.stage_nwords = nbytes / 4;
      if (nbytes) {
        mbar_init(&T.bar, 1);
        mbar_expect_tx(&T.bar, nbytes);
        tma_bulk_g2s(stage, P.src.data + a0, nbytes, &T.bar);
      }
    }
    __syncwarp();
    if (nbytes) mbar_wait(&T.bar, 0);
    __syncwarp();
  }
  BitSrc src = P.src;
  src.sw = stage;
  src.sw_lo = (boff & ~15ull) >> 2;
  src.sw_n = T.stage_nwords;
  if (lane == 0) {
    int depth = 0, cw = 0, zr = 0, nst = 0, ntree = 0;
    u64 pstart = 0;
    uint32_t m3[3];
    int rc = parse_block_header(src, bstart, bend, nsub, T, &depth, &cw, &zr, m3, &nst, &pstart, &ntree);
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
      uint4* zp = reinterpret_cast<uint4*>(symbase + (i64)T.slot_of[j] * WB_PP);
      for (int i = 0; i < WB_PP / 16; ++i) zp[i] = make_uint4(0, 0, 0, 0);
      int st = decode_plane(src, T, pstart + T.seek[j], bend, zr, cw, symbase + (i64)T.slot_of[j] * WB_PP, &endp);
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
        int st = decode_tokens_seq(src, T.left, T.right, T.sym, pstart, bend, zr, cw, dn, sr, &e, &bad);
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
  const int max_stage = 96 * 1024;
  const int tree_bytes = (int)((sizeof(TreeSmem) + 127) & ~(size_t)127);
  if (!attr) {
    cudaFuncSetAttribute(k_block_decode, cudaFuncAttributeMaxDynamicSharedMemorySize, tree_bytes + max_stage);
    attr = true;
  }
  // staging window: ~2x the average block, 16 KB..96 KB (larger blocks read their tail from HBM)
  const u64 nblk = (u64)batch * g.slots_per_image;
  u64 avg = nblk ? nbytes / nblk : 0;
  const u64 raw = (u64)g.W * g.H * g.C * (g.bd > 8 ? 2 : 1) * (u64)batch;  // compressed <= raw, typically
  u64 stage = avg * 2;
  if (nblk && raw / nblk < stage) stage = raw / nblk;
  stage += 1024;
  if (stage < 16 * 1024) stage = 16 * 1024;
  static int cap_env = -1;
  if (cap_env < 0) {
    const char* e = getenv("WBPC_DECODE_STAGE_MAX");
    cap_env = e ? atoi(e) : 16 * 1024;
  }
  if (stage > (u64)cap_env) stage = (u64)cap_env;
  if (stage > (u64)max_stage) stage = max_stage;
  stage = (stage + 15) & ~15ull;
  DecodeParams P;
  P.stage_bytes = (uint32_t)stage;
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
  k_block_decode<<<nblocks, 32, tree_bytes + (int)stage, s>>>(P);
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
