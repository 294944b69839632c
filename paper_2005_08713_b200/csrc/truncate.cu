// truncate.cu — lossy plane truncation of a container without re-encoding (sm_100a).
//
// Replaces (reference /root/reference/pkg/src/wbpc):
//   truncate_block   blocks.py:264-304   (keep planes b < depth-n; same depth/cw/zr/tree; masks for
//                                         b >= q cleared; count = keep_n; payload cut at seek[keep_n])
//   truncate_stream  container.py:393-417
//
// Every rewritten block is a concatenation of bit ranges of the original block (fields, the kept
// prefix of each subband mask, the tree, the first keep_n seek entries, the payload prefix) plus
// zero bits and the new 16-bit count, so the emit kernel assembles each output word from at most
// a handful of source ranges with funnel shifts; unchanged blocks are copied byte for byte.
#include "coder.cuh"

namespace wb {

struct BitSrcT {
  const uint8_t* data;
  u64 nbytes;
  __device__ __forceinline__ uint32_t word(u64 k) const {
    if (4 * k + 3 < nbytes) return bswap32(__ldg(reinterpret_cast<const uint32_t*>(data) + k));
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) {
      u64 bi = 4 * k + i;
      v = (v << 8) | (bi < nbytes ? data[bi] : 0u);
    }
    return v;
  }
  __device__ __forceinline__ uint32_t bits(u64 p, int n) const {
    if (n == 0) return 0;
    u64 k = p >> 5;
    u64 w = ((u64)word(k) << 32) | word(k + 1);
    return (uint32_t)((w << (p & 31)) >> (64 - n));
  }
};

// Sequential reader over BitSrcT: a 64-bit register window refilled 32 bits at a time, the next 32
// bits always requested one refill ahead (the load's latency overlaps the parsing of the bits in
// hand instead of stalling the walk at every refill).
constexpr int TSTAGE = 264;  // staged words per block (every header fits: <= 870 bytes)
struct SeqBits {
  const BitSrcT* S;
  const uint32_t* st;  // the block's first TSTAGE container words (big-endian values) in shared memory
  u64 k0;              // container word index of st[0]
  u64 pos;   // absolute position of the next unread bit
  u64 buf;   // bits [pos, pos + nb), MSB aligned
  uint32_t pf;  // bits [pos + nb, pos + nb + 32), loaded ahead
  int nb;
  __device__ __forceinline__ uint32_t bits32(u64 p) const {
    const u64 k = (p >> 5) - k0;
    if (k + 1 < (u64)TSTAGE) return __funnelshift_l(st[k + 1], st[k], (uint32_t)(p & 31));
    return S->bits(p, 32);
  }
  __device__ __forceinline__ void init(const BitSrcT* s, const uint32_t* stage, u64 kbase, u64 p) {
    S = s; st = stage; k0 = kbase; pos = p; buf = 0; nb = 0;
    pf = bits32(pos);
  }
  __device__ __forceinline__ void fill(int n) {  // make n <= 32 bits available
    if (nb < n) {
      buf |= (u64)pf << (32 - nb);
      nb += 32;
      pf = bits32(pos + nb);
    }
  }
  __device__ __forceinline__ uint32_t peek32() {  // the next 32 bits (not consumed)
    fill(32);
    return (uint32_t)(buf >> 32);
  }
  __device__ __forceinline__ void skip(int n) {  // n <= nb
    buf <<= n;
    nb -= n;
    pos += n;
  }
  __device__ __forceinline__ uint32_t take(int n) {  // 1 <= n <= 32
    fill(n);
    const uint32_t v = (uint32_t)(buf >> (64 - n));
    skip(n);
    return v;
  }
};

constexpr int MAX_SEG = 12;  // 19-bit fields + 2 per subband mask + tree + count + seek + payload = 11
struct TruncMeta {
  uint32_t new_len;
  uint32_t mode;        // 0 = copy verbatim, 1 = rewrite
  uint32_t nseg;
  uint32_t pad;
  // segment k: dest bit start, length, source absolute bit start (or ~0 = literal), literal
  uint32_t dst[MAX_SEG], len[MAX_SEG];
  u64 src[MAX_SEG];
  uint32_t lit[MAX_SEG];
};

struct TruncParams {
  Geom g;
  int per_level, drop_global, drop_ll;
  int drop_hp[WB_MAXL + 1];
  BitSrcT src;
  const u64* blk_off;
  const uint32_t* blk_len;
  TruncMeta* tm;
  uint32_t* sizes;
  DevStatus* st;
};

// One warp per block: the lanes stage the block's first TSTAGE words in shared memory, lane 0
// walks the header from there (blocks.py:150-192 + read_tree entropy.py:272-310, error classes
// identical; a walk over global memory paid a load latency per 32 bits) and writes the segment
// plan of truncate_block.
constexpr int TPW = 4;  // warps (blocks) per CTA
__global__ void __launch_bounds__(TPW * 32) k_trunc_plan(TruncParams P) {
  __shared__ uint32_t stage[TPW][TSTAGE];
  __shared__ unsigned seen_s[TPW][8];
  const Geom& g = P.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = blockIdx.x * TPW + warp;
  const int nblocks = g.slots_per_image;  // single container
  if (gid >= nblocks) return;
  {
    const u64 kb = (8ull * P.blk_off[gid]) >> 5;
    for (int i = lane; i < TSTAGE; i += 32) stage[warp][i] = P.src.word(kb + i);
    if (lane < 8) seen_s[warp][lane] = 0u;
    __syncwarp();
    if (lane) return;
  }
  unsigned* const seen = seen_s[warp];
  const SlotInfo si = slot_info(g, gid);
  const int nsub = si.kind ? 3 : 1;
  TruncMeta* T = P.tm + gid;
  const uint32_t olen = P.blk_len[gid];
  const u64 bstart = 8ull * P.blk_off[gid];
  const u64 bend = bstart + 8ull * olen;
  const int n = P.per_level ? (si.kind ? P.drop_hp[si.lev] : P.drop_ll) : P.drop_global;
  T->mode = 0;
  T->new_len = olen;
  P.sizes[gid] = olen;
  if (n == 0) return;  // blocks.py:274-275
  SeqBits R;
  R.init(&P.src, stage[warp], bstart >> 5, bstart);
  int err = 0;
#define NEED(k)                    \
  if (R.pos + (u64)(k) > bend) {   \
    err = WBPC_ERR_BLOCK_PARSE;    \
    goto fail;                     \
  }
  {
    NEED(19);
    const int depth = (int)R.take(6);
    if (depth < 1) { err = WBPC_ERR_BLOCK_PARSE; goto fail; }
    R.take(13);
    const u64 mask_pos = R.pos;
    int cnt = 0;
    int q = depth - n;
    if (q < 0) q = 0;
    int keep_n = 0;
    // masks (s-major); count stored per plane order: keep_n = #stored with b < q
    for (int s = 0; s < nsub; ++s) {
      NEED(depth);
      for (int bb = 0; bb < depth; ++bb) {
        const uint32_t bit = R.take(1);
        cnt += bit;
        if (bit && bb < q) ++keep_n;
      }
    }
    const u64 tree_pos = R.pos;
    if (cnt) {
      // read_tree (entropy.py:272-310): `open` = unfilled child slots of pending internal nodes.
      // Node depths, for the CodeLengthError the HuffmanCode constructor raises after the read
      // completes (entropy.py:86,97-98: an internal node at depth >= 32), come from a bit mask of
      // the ancestors whose right child is still to come: an internal node at depth d sets bit d
      // and is followed by its left child at d + 1; after a leaf the next node is the right child
      // of the deepest marked ancestor.  A run of k internal nodes (k zero bits: each the left
      // child of the one before) is consumed at once; the checks the reference makes per node
      // (bits left in the block, more than 512 nodes) bound k, so the first failing node raises
      // the same class.
      int nodes = 0, open = 0, d = 0;
      u64 pend = 0;
      bool first = true, toolong = false;
      while (first || open) {
        if (R.pos + 1 > bend || nodes > 511) { err = WBPC_ERR_MALFORMED_TREE; goto fail; }
        const uint32_t w = R.peek32();
        if (!(w >> 31)) {  // internal nodes
          int k = w ? __clz(w) : 32;
          const u64 room = bend - R.pos;
          if ((u64)k > room) k = (int)room;
          if (k > 512 - nodes) k = 512 - nodes;
          R.skip(k);
          if (!toolong) {
            if (d + k - 1 >= 32) toolong = true;
            else { pend |= ((1ull << k) - 1ull) << d; d += k; }
          }
          open += k + (first ? 1 : 0);
          nodes += k;
        } else {  // leaf: 1 + 8-bit symbol
          R.skip(1);
          if (R.pos + 8 > bend) { err = WBPC_ERR_MALFORMED_TREE; goto fail; }
          const int sy = (int)R.take(8);
          if ((seen[sy >> 5] >> (sy & 31)) & 1u) { err = WBPC_ERR_MALFORMED_TREE; goto fail; }
          seen[sy >> 5] |= 1u << (sy & 31);
          if (!first) --open;
          if (!toolong && pend) {
            const int h = 63 - __clzll((long long)pend);
            pend &= ~(1ull << h);
            d = h + 1;
          }
          ++nodes;
        }
        first = false;
      }
      if (toolong) { err = WBPC_ERR_CODE_LENGTH; goto fail; }
    }
    const u64 tree_bits = R.pos - tree_pos;
    NEED(16);
    const int seek_count = (int)R.take(16);
    if (seek_count != cnt) { err = WBPC_ERR_CORRUPTION; goto fail; }
    const int t = seek_bits(nsub, depth);
    const u64 seek_pos = R.pos;
    uint32_t prev = 0, cut = 0;
    bool dec = false;
    for (int i = 0; i < cnt; ++i) {
      NEED(t);
      const uint32_t v = R.take(t);
      if (i && v < prev) dec = true;
      if (i == keep_n) cut = v;
      prev = v;
    }
    if (dec) { err = WBPC_ERR_CORRUPTION; goto fail; }
    const u64 payload_pos = R.pos;
    if (keep_n == cnt) return;  // blocks.py:279-281: unchanged
    if (payload_pos + cut > bend) { err = WBPC_ERR_TRUNCATION; goto fail; }  // bitio.py:95-97
    // segment plan (blocks.py:288-304)
    uint32_t d = 0;
    int k = 0;
    auto add = [&](u64 src, uint32_t len, uint32_t lit) {
      if (!len) return;
      T->dst[k] = d; T->len[k] = len; T->src[k] = src; T->lit[k] = lit;
      d += len;
      ++k;
    };
    add(bstart, 19, 0);                                       // depth, counter width, zr
    for (int s = 0; s < nsub; ++s) {                          // masks, planes >= q cleared
      int keepb = q < depth ? q : depth;
      add(mask_pos + (u64)s * depth, (uint32_t)keepb, 0);
      add(~0ull, (uint32_t)(depth - keepb), 0);
    }
    if (keep_n) add(tree_pos, (uint32_t)tree_bits, 0);       // tree only if planes remain
    add(~0ull, 16, (uint32_t)keep_n);                          // seek count
    add(seek_pos, (uint32_t)(keep_n * t), 0);                  // first keep_n seek entries
    add(payload_pos, cut, 0);                                  // payload prefix
    T->nseg = k;
    T->mode = 1;
    T->new_len = (d + 7) >> 3;
    P.sizes[gid] = T->new_len;
  }
  return;
fail:
  record_error(P.st, err, (u64)gid);
#undef NEED
}

struct TruncEmitParams {
  Geom g;
  BitSrcT src;
  const u64* blk_off;
  const uint32_t* blk_len;
  const TruncMeta* tm;
  const u64* new_off;
  const u64* img_off;
  uint8_t* out;
  u64 cap;
};

__global__ void __launch_bounds__(128) k_trunc_emit(TruncEmitParams P) {
  const int gid = blockIdx.x;
  const TruncMeta& T = P.tm[gid];
  const u64 O = P.new_off[gid];
  const uint32_t nl = T.new_len;
  if (O + nl > P.cap) return;
  const u64 img0 = P.img_off[0];
  if (threadIdx.x == 0 && P.g.raw_kind < 0) {
    uint8_t* ie = P.out + img0 + 19 + 12ull * gid;
    u64 rel = O - img0;
    for (int i = 0; i < 8; ++i) ie[i] = (uint8_t)(rel >> (8 * i));
    for (int i = 0; i < 4; ++i) ie[8 + i] = (uint8_t)(nl >> (8 * i));
    if (gid == 0)  // container.py:417 header.pack(): same 19 bytes as the source
      for (int i = 0; i < 19; ++i) P.out[img0 + i] = P.src.data[i];
  }
  const uint8_t* sb = P.src.data + P.blk_off[gid];
  uint8_t* db = P.out + O;
  if (T.mode == 0) {
    for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) db[i] = sb[i];
    return;
  }
  const uint32_t nwords = (nl + 3) / 4;
  for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x) {
    const uint32_t lo = 32 * w, hi = lo + 32;
    uint32_t v = 0;
    for (uint32_t k = 0; k < T.nseg; ++k) {
      uint32_t a = max(lo, T.dst[k]), e = min(hi, T.dst[k] + T.len[k]);
      if (a >= e) continue;
      uint32_t n = e - a;
      uint32_t bits;
      if (T.src[k] == ~0ull) {
        // literal (right-aligned in len bits)
        uint32_t off = a - T.dst[k];
        u64 lit = T.lit[k];
        bits = (uint32_t)((lit >> (T.len[k] - off - n)) & ((n == 32) ? 0xFFFFFFFFull : ((1ull << n) - 1)));
      } else {
        bits = P.src.bits(T.src[k] + (a - T.dst[k]), (int)n);
      }
      v |= (n == 32) ? bits : (bits << (hi - e));
    }
    for (int i = 0; i < 4; ++i) {
      uint32_t bi = 4 * w + i;
      if (bi < nl) db[bi] = (uint8_t)(v >> (24 - 8 * i));
    }
  }
}

size_t trunc_meta_bytes() { return sizeof(TruncMeta); }

cudaError_t launch_offsets(int nblocks, int spi, int batch, const uint32_t* sizes, u64* block_off, u64* img_off,
                           u64 cap, DevStatus* st, cudaStream_t s, int raw, uint32_t* outw);

cudaError_t launch_truncate(const Geom& g, int per_level, int drop_global, const int* drop_hp, int drop_ll,
                            const uint8_t* data, u64 nbytes, const u64* blk_off, const uint32_t* blk_len,
                            TruncMeta* tm, uint32_t* sizes, u64* new_off, u64* img_off, uint8_t* out, u64 cap,
                            DevStatus* st, cudaStream_t s) {
  TruncParams P;
  P.g = g;
  P.per_level = per_level;
  P.drop_global = drop_global;
  P.drop_ll = drop_ll;
  for (int i = 0; i <= WB_MAXL; ++i) P.drop_hp[i] = (per_level && i >= 1 && drop_hp) ? drop_hp[i - 1] : 0;
  P.src.data = data;
  P.src.nbytes = nbytes;
  P.blk_off = blk_off;
  P.blk_len = blk_len;
  P.tm = tm;
  P.sizes = sizes;
  P.st = st;
  const int n = g.slots_per_image;
  prof_mark("trunc_plan", s);
  k_trunc_plan<<<(n + TPW - 1) / TPW, TPW * 32, 0, s>>>(P);
  launch_offsets(n, n, 1, sizes, new_off, img_off, cap, st, s, g.raw_kind >= 0, nullptr);
  TruncEmitParams E;
  E.g = g;
  E.src = P.src;
  E.blk_off = blk_off;
  E.blk_len = blk_len;
  E.tm = tm;
  E.new_off = new_off;
  E.img_off = img_off;
  E.out = out;
  E.cap = cap;
  prof_mark("trunc_emit", s);
  k_trunc_emit<<<n, 128, 0, s>>>(E);
  return cudaGetLastError();
}

}  // namespace wb
