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

constexpr int LUT_BITS = 11;                 // first-level decode table index bits
constexpr int LUT_SIZE = 1 << LUT_BITS;
constexpr int L2_BITS = 5;                   // second level: codes of LUT_BITS+1 .. LUT_BITS+L2_BITS bits
constexpr int L2_CAP = 2048;                 // second-level entries (64 subtables of 2^L2_BITS)
constexpr int LUT_ALL = LUT_SIZE + L2_CAP;

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
  // two-level decode table.  Entry: leaf (len << 8) | sym (len <= 16); 0x8000 | base: second
  // level at lut[LUT_SIZE + base + next L2_BITS bits]; 0xC000 | node: tree walk from node
  uint16_t lut[LUT_ALL];
  int16_t left[512], right[512], sym[512];
  uint32_t seek[WB_MAX_SLOTS];
  uint8_t slot_of[WB_MAX_SLOTS];
  u64 pstart;              // absolute payload start bit
  int rc, depth, cw, zr, nst, dn, ntree, nsub;
  int two_level;           // 0: every code fits the first level (no subtables, no long codes)
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

// Header parse of blocks.py:150-192 (+ read_tree entropy.py:272-310), in three parts so the tree
// structure can be built by the whole warp:
//   part A (lane 0): depth, cw, zr, masks, then a scan of the preorder tree tokens ('0' internal,
//                    '1' + 8-bit symbol) into tok[] with the reference's MalformedTree checks;
//   tree_structure (warp): parents, children, depths and codes from the token list;
//   part C (lane 0): seek count and entries.
// The bit reader is a 64-bit register buffer over a word source (staged smem words with a global
// fallback); its state lives in lane 0 between parts A and C.
struct HdrBits {
  BitSrc src;
  uint64_t buf;
  int nb;
  u64 nextw, pos, bend;
  __device__ __forceinline__ void init(const BitSrc& s, u64 bstart, u64 bend_) {
    src = s;
    const u64 k = bstart >> 5;
    buf = (((uint64_t)s.word(k) << 32) | s.word(k + 1)) << (bstart & 31);
    nb = 64 - (int)(bstart & 31);
    nextw = k + 2;
    pos = bstart;
    bend = bend_;
  }
  __device__ __forceinline__ void refill() {
    if (nb <= 32) {
      buf |= (uint64_t)src.word(nextw++) << (32 - nb);
      nb += 32;
    }
  }
  __device__ __forceinline__ uint32_t get(int n) {  // n <= 32
    if (n == 0) return 0u;
    refill();
    const uint32_t v = (uint32_t)(buf >> (64 - n));
    buf <<= n;
    nb -= n;
    pos += (u64)n;
    return v;
  }
  __device__ __forceinline__ bool need(u64 n) const { return pos + n <= bend; }
};

// Part A.  Returns 0 or the error class; on success *ntok tokens are in tok[] (0 = internal,
// 0x100 | symbol = leaf) and *maxopen is the largest open-slot count seen (> 33 implies an
// internal node at depth >= 32, i.e. CodeLengthError, see tree_structure).
template <typename Tab>
static __device__ int parse_header_a(HdrBits& R, int nsub, Tab& T, uint64_t* mk, uint16_t* tok, int* ntok,
                                     int* maxopen) {
  if (!R.need(6)) return WBPC_ERR_BLOCK_PARSE;
  const int depth = (int)R.get(6);
  if (depth < 1) return WBPC_ERR_BLOCK_PARSE;
  if (!R.need(5)) return WBPC_ERR_BLOCK_PARSE;
  const int cw = (int)R.get(5);
  if (!R.need(8)) return WBPC_ERR_BLOCK_PARSE;
  const int zr = (int)R.get(8);
  int cnt = 0;
  for (int s = 0; s < nsub; ++s) {
    if (!R.need((u64)depth)) return WBPC_ERR_BLOCK_PARSE;
    u64 v;
    if (depth > 32) {
      v = (u64)R.get(depth - 32) << 32;
      v |= R.get(32);
    } else {
      v = R.get(depth);
    }
    mk[s] = v;  // MSB = plane 0
    cnt += __popcll(v);
  }
  T.depth = depth;
  T.cw = cw;
  T.zr = zr;
  T.nst = cnt;
  *ntok = 0;
  *maxopen = 1;
  if (!cnt) return 0;
  // token scan (tok[] is pre-zeroed): a run of internal nodes ('0' bits) is consumed at once
  // with a leading-zero count; only leaves are stored.  Duplicate leaves are checked by the
  // warp afterwards (also MalformedTreeError, before CodeLengthError).
  const u64 rem64 = R.bend > R.pos ? R.bend - R.pos : 0;
  uint32_t rem = rem64 > 0xFFFFFFF0ull ? 0xFFFFFFF0u : (uint32_t)rem64;
  const uint32_t rem0 = rem;
  int n = 0, open = 1, mo = 1;
  // Fast path: the scan reads at most 512 nodes (<= 512 * 9 bits) before it ends or fails; when
  // that span lies inside the shared-memory copy of the block, the window is formed straight
  // from the staged words (two loads and a funnel shift per step) instead of the bit buffer.
  {
    const u64 wlo = R.src.sw_lo * 32ull;
    const u64 whi = (R.src.sw_lo + R.src.sw_n) * 32ull;
    if (R.src.sw && R.pos >= wlo && R.pos + 512 * 9 + 64 <= whi) {
      const uint32_t* sw = R.src.sw;
      uint32_t q = (uint32_t)(R.pos - wlo);  // bit offset in the staged words
      auto window = [&](uint32_t qq) {
        const uint32_t hi = bswap32(sw[qq >> 5]), lo = bswap32(sw[(qq >> 5) + 1]);
        return __funnelshift_l(lo, hi, qq & 31);
      };
      while (true) {
        const uint32_t win = window(q);
        const int z = __clz(win);  // a run of internal nodes ('0' bits), 32 if the window is all zero
        if ((uint32_t)z > rem || n + z > 512) return WBPC_ERR_MALFORMED_TREE;  // out of bits / > 512 nodes
        q += (uint32_t)z;
        rem -= (uint32_t)z;
        n += z;
        open += z;
        mo = max(mo, open);
        if (z == 32) continue;
        // a leaf: '1' + 8-bit symbol
        if (rem < 9 || n > 511) return WBPC_ERR_MALFORMED_TREE;
        const uint32_t sym = z + 9 <= 32 ? (win << (z + 1)) >> 24 : (window(q) << 1) >> 24;
        tok[n] = (uint16_t)(0x100u | sym);
        q += 9;
        rem -= 9;
        ++n;
        if (--open == 0) break;
      }
      R.init(R.src, R.pos + (rem0 - rem), R.bend);  // the bit buffer resumes after the tree
      *ntok = n;
      *maxopen = mo;
      return 0;
    }
  }
  while (true) {
    R.refill();
    int z = __clzll(R.buf);
    const bool allzero = z >= R.nb;  // every valid buffered bit is an internal node
    if (allzero) z = R.nb;
    if ((uint32_t)z > rem || n + z > 512) return WBPC_ERR_MALFORMED_TREE;  // out of bits / > 512 nodes
    if (z) {
      R.buf = z < 64 ? R.buf << z : 0ull;
      R.nb -= z;
      rem -= (uint32_t)z;
      n += z;
      open += z;
      mo = max(mo, open);
    }
    if (allzero) continue;
    // a leaf: '1' + 8-bit symbol
    if (rem < 9 || n > 511) return WBPC_ERR_MALFORMED_TREE;
    R.refill();
    tok[n] = (uint16_t)(0x100u | (uint32_t)((R.buf >> 55) & 255u));
    R.buf <<= 9;
    R.nb -= 9;
    rem -= 9;
    ++n;
    if (--open == 0) break;
  }
  R.pos += rem0 - rem;
  *ntok = n;
  *maxopen = mo;
  return 0;
}

// Part C: seek count and entries (blocks.py:172-178); payload start.
template <typename Tab>
static __device__ int parse_header_c(HdrBits& R, int nsub, Tab& T, const uint64_t* mk, uint32_t* mask3) {
  const int cnt = T.nst, depth = T.depth;
  if (!R.need(16)) return WBPC_ERR_BLOCK_PARSE;
  const int seek_count = (int)R.get(16);
  if (seek_count != cnt) return WBPC_ERR_CORRUPTION;
  const int t = seek_bits(nsub, depth);
  uint32_t prev = 0;
  bool decreasing = false;
  const u64 wlo = R.src.sw_lo * 32ull, whi = (R.src.sw_lo + R.src.sw_n) * 32ull;
  if (R.src.sw && t <= 32 && R.pos >= wlo && R.pos + (u64)cnt * t + 64 <= whi && R.need((u64)cnt * t)) {
    // every entry inside the staged words: independent fixed-width reads (no bit-buffer chain)
    const uint32_t* sw = R.src.sw;
    const uint32_t q0 = (uint32_t)(R.pos - wlo);
    for (int i = 0; i < cnt; ++i) {
      const uint32_t q = q0 + (uint32_t)(i * t);
      const uint32_t hi = bswap32(sw[q >> 5]), lo = bswap32(sw[(q >> 5) + 1]);
      const uint32_t v = __funnelshift_l(lo, hi, q & 31) >> (32 - t);
      if (i < WB_MAX_SLOTS) T.seek[i] = v;
      if (i && v < prev) decreasing = true;
      prev = v;
    }
    R.init(R.src, R.pos + (u64)cnt * t, R.bend);
  } else {
    for (int i = 0; i < cnt; ++i) {
      if (!R.need((u64)t)) return WBPC_ERR_BLOCK_PARSE;
      const uint32_t v = R.get(t);
      if (i < WB_MAX_SLOTS) T.seek[i] = v;
      if (i && v < prev) decreasing = true;
      prev = v;
    }
  }
  if (decreasing) return WBPC_ERR_CORRUPTION;  // blocks.py:177-178
  T.pstart = R.pos;
  mask3[0] = mask3[1] = mask3[2] = 0;
  for (int s = 0; s < nsub; ++s)
    for (int b = 0; b < depth; ++b)
      if ((mk[s] >> (depth - 1 - b)) & 1ull) {
        const int kk = b * nsub + s;
        if (kk < WB_MAX_SLOTS) mask3[kk >> 5] |= 1u << (kk & 31);
      }
  return 0;
}

// K1: one warp per block -- lane 0 parses header + tree (scratch in smem), the warp builds the
// decode LUT; results (BlockTab, DecMeta) go to global memory for K2 / reconstruction.
constexpr int HW = 2;  // warps (blocks) per K1 CTA
struct HdrScratch {        // shared-memory image of the BlockTab fields of the block being finished
  int16_t left[512], right[512], sym[512], pending[512];  // pending: parent / jump pointer
  uint16_t tok[512];        // preorder tree tokens: 0 internal, 0x100 | symbol leaf
  uint8_t oprev[512], isr[512];
  int16_t last[40];
  int16_t anc2[512];
  uint8_t dist2[512];
  uint32_t bits2[512];
  uint32_t seen[8];
  uint32_t seek[WB_MAX_SLOTS];
  uint8_t ndepth[512];
  uint32_t ncode[512];
  uint32_t m3[3];
  u64 pstart;
  int rc, depth, cw, zr, nst, ntree, dn;
  uint8_t slot_of[WB_MAX_SLOTS];
};

// Warp-parallel tree structure from the preorder token list (n tokens, a complete full binary
// tree).  With O(t) = open slots before token t (1 + #internal - #leaf before t): token t is
// the left child of t-1 if t-1 is internal, otherwise the right child of the last u < t with
// O(u) = O(t) (the slot it fills was opened by u).  Depths and codes follow by pointer
// jumping.  Returns 0 or CodeLengthError (an internal node at depth >= 32, entropy.py:97-98).
template <typename Tab>
static __device__ int tree_structure(Tab& H, int n, int lane) {
  // A. open slots before each token (exclusive scan, 16 tokens per lane)
  const int t0 = 16 * lane;
  int loc = 0;
  for (int i = 0; i < 16; ++i)
    if (t0 + i < n) loc += H.tok[t0 + i] ? -1 : 1;
  int incl = loc;
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  int run = 1 + incl - loc;
  for (int i = 0; i < 16; ++i)
    if (t0 + i < n) {
      H.oprev[t0 + i] = (uint8_t)run;
      run += H.tok[t0 + i] ? -1 : 1;
    }
  for (int i = lane; i < 40; i += 32) H.last[i] = -1;
  __syncwarp();
  // B. parents, 32 tokens at a time; `last` keeps the latest token of each open-slot count
  for (int k = 0; k < n; k += 32) {
    const int t = k + lane;
    const bool valid = t < n;
    const int v = valid ? H.oprev[t] : 39;
    const unsigned mask = __match_any_sync(0xffffffffu, v);
    int par = -1, isr = 0;
    if (valid && t > 0) {
      if (H.tok[t - 1] == 0) {
        par = t - 1;
      } else {
        const unsigned m = mask & ((1u << lane) - 1u);
        par = m ? k + 31 - __clz(m) : H.last[v];
        isr = 1;
      }
    }
    __syncwarp();
    if (valid && (lane == 31 || (mask >> (lane + 1)) == 0)) H.last[v] = (int16_t)t;
    if (valid) {
      H.pending[t] = (int16_t)par;
      H.isr[t] = (uint8_t)isr;
    }
    __syncwarp();
  }
  // C. children and symbols
  for (int t = lane; t < n; t += 32) {
    if (H.tok[t]) {
      H.left[t] = -1;
      H.right[t] = -1;
      H.sym[t] = (int16_t)(H.tok[t] & 255);
    } else {
      H.sym[t] = -1;
    }
  }
  __syncwarp();
  for (int t = lane; t < n; t += 32) {
    if (t == 0) continue;
    const int p = H.pending[t];
    if (H.isr[t]) H.right[p] = (int16_t)t;
    else H.left[p] = (int16_t)t;
  }
  // D. depth (dist to the root) and code by pointer jumping: buffer 1 = (pending, ndepth,
  //    ncode), buffer 2 = (anc2, dist2, bits2)
  for (int t = lane; t < n; t += 32) {
    H.ndepth[t] = (uint8_t)(t ? 1 : 0);
    H.ncode[t] = H.isr[t];
  }
  __syncwarp();
  bool in1 = true;
  for (int round = 0; round < 10; ++round) {
    bool any = false;
    for (int t = lane; t < n; t += 32) {
      const int a = in1 ? H.pending[t] : H.anc2[t];
      const int d = in1 ? H.ndepth[t] : H.dist2[t];
      const uint32_t bt = in1 ? H.ncode[t] : H.bits2[t];
      int na = -1, nd = d;
      uint32_t nbt = bt;
      if (a >= 0) {
        na = in1 ? H.pending[a] : H.anc2[a];
        const int da = in1 ? H.ndepth[a] : H.dist2[a];
        const uint32_t ba = in1 ? H.ncode[a] : H.bits2[a];
        nd = min(255, d + da);
        nbt = (d < 32 ? ba << d : 0u) | bt;
        any = true;
      }
      if (in1) { H.anc2[t] = (int16_t)na; H.dist2[t] = (uint8_t)nd; H.bits2[t] = nbt; }
      else { H.pending[t] = (int16_t)na; H.ndepth[t] = (uint8_t)nd; H.ncode[t] = nbt; }
    }
    __syncwarp();
    in1 = !in1;
    if (!__any_sync(0xffffffffu, any)) break;
  }
  if (!in1) {  // results are in buffer 2: copy back
    for (int t = lane; t < n; t += 32) {
      H.ndepth[t] = H.dist2[t];
      H.ncode[t] = H.bits2[t];
    }
  }
  __syncwarp();
  bool bad = false;
  for (int t = lane; t < n; t += 32) bad |= H.tok[t] == 0 && H.ndepth[t] >= 32;
  return __any_sync(0xffffffffu, bad) ? WBPC_ERR_CODE_LENGTH : 0;
}

// Several blocks per warp: their serial header/tree scans (part A, the bulk of this kernel's
// instructions) run side by side, lane bi on block bi, so one warp instruction advances HBW
// scans; the warp then finishes the blocks one after another (duplicate leaves, tree structure,
// part C on the owning lane, tables, decode LUT).
struct HdrStage {
  uint32_t hw[256];      // first 1 KB of the block (header), raw little-endian words
  uint16_t tok[512];     // preorder tree tokens from part A
};
struct HdrA {            // part A results of one block (the fields parse_header_a writes)
  int depth, cw, zr, nst;
};

__device__ void header_block(const DecodeParams& P, HdrScratch& H, HdrStage& Sg, const HdrA& A,
                                              int rcA, int ntok, int maxopen, int gid, int owner, HdrBits& R,
                                              const uint64_t* mk) {
  const Geom& g = P.g;
  const int lane = threadIdx.x & 31;
  const int b = fdiv(gid, g.md_spi);
  const SlotInfo si = slot_info(g, gid - b * g.slots_per_image);
  DecMeta* DM = P.dmeta + gid;
  BlockTab& T = P.tabs[gid];
  const int nsub = si.kind ? 3 : 1;
  if (lane == 0) {
    H.rc = rcA;
    H.ntree = rcA ? 0 : ntok;
    H.depth = A.depth;
    H.cw = A.cw;
    H.zr = A.zr;
    H.nst = A.nst;
  }
  if (lane < 8) H.seen[lane] = 0u;
  for (int i = lane; i < 256; i += 32) reinterpret_cast<uint32_t*>(H.tok)[i] = reinterpret_cast<const uint32_t*>(Sg.tok)[i];
  __syncwarp();
  if (H.rc == 0 && H.ntree > 0) {
    const int n = H.ntree;
    bool dup = false;  // a symbol in two leaves (read_tree, entropy.py:300-303)
    for (int t = lane; t < n; t += 32)
      if (H.tok[t]) {
        const uint32_t sy = H.tok[t] & 255u, m = 1u << (sy & 31);
        dup |= (atomicOr(&H.seen[sy >> 5], m) & m) != 0;
      }
    int rs;
    if (__any_sync(0xffffffffu, dup)) rs = WBPC_ERR_MALFORMED_TREE;
    // more than 33 open slots: some node is 33+ deep below an internal node at depth >= 32
    else if (maxopen > 33) rs = WBPC_ERR_CODE_LENGTH;
    else rs = tree_structure(H, n, lane);
    if (lane == 0 && rs) H.rc = rs;
  }
  __syncwarp();
  if (lane == owner) {  // the lane whose bit reader stopped after this block's tree
    int rc = H.rc;
    if (!rc) rc = parse_header_c(R, nsub, H, mk, H.m3);
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
        for (int s2 = 0; s2 < nsub; ++s2) {
          const int k = pb * nsub + s2;
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
      // the largest detail-block depth of the call decides the detail coefficient width of the
      // reconstruction and the inverse transform (|c| < 2^(depth-1): int16 when depth <= 16)
      if (si.kind) atomicMax(&P.st->pad, (u64)depth);
    }
  }
  __syncwarp();
  // warp copies the parsed tables to global and builds the decode LUT
  if (lane == owner) {
    T.rc = H.rc;
    T.nsub = nsub;
    T.dn = H.dn;
    T.depth = H.depth;
    T.cw = H.cw;
    T.zr = H.zr;
    T.nst = H.nst;
    T.ntree = H.ntree;
    T.pstart = H.pstart;
    T.two_level = 1;
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
  // decode tables.  Level 1: leaves with len <= LUT_BITS replicated over their aligned
  // 2^(LUT_BITS-len) range; internal nodes at depth LUT_BITS get a 2^L2_BITS second-level
  // subtable (in preorder, while capacity lasts; else a tree-walk marker).
  auto fill = [&](uint16_t* t, uint32_t first, uint32_t cnt, uint16_t e) {
    if (cnt >= 8) {
      const uint32_t e2 = (uint32_t)e * 0x10001u;
      const uint4 v = make_uint4(e2, e2, e2, e2);
      uint4* q = reinterpret_cast<uint4*>(t + first);
      for (uint32_t k = 0; k < cnt / 8; ++k) q[k] = v;
    } else {
      for (uint32_t k = 0; k < cnt; ++k) t[first + k] = e;
    }
  };
  int nsubt = 0;
  for (int i0 = 0; i0 < ntree; i0 += 32) {
    const int i = i0 + lane;
    const bool in = i < ntree;
    const int d = in ? H.ndepth[i] : 0;
    const bool leaf = in && H.left[i] == -1;
    const bool sub = in && !leaf && d == LUT_BITS;
    const unsigned bal = __ballot_sync(0xffffffffu, sub);
    if (leaf && d <= LUT_BITS) {
      const uint32_t first = d ? H.ncode[i] << (LUT_BITS - d) : 0u;
      fill(T.lut, first, 1u << (LUT_BITS - d), (uint16_t)((d << 8) | H.sym[i]));
    } else if (sub) {
      const int k = nsubt + __popc(bal & ((1u << lane) - 1u));
      T.lut[H.ncode[i]] = k < L2_CAP >> L2_BITS ? (uint16_t)(0x8000u | (k << L2_BITS)) : (uint16_t)(0xC000u | i);
    }
    nsubt += __popc(bal);
  }
  __syncwarp();
  // no internal node at depth LUT_BITS <=> every code is at most LUT_BITS bits long
  if (lane == 0) T.two_level = nsubt > 0 ? 1 : 0;
  if (nsubt == 0) return;
  // level 2: nodes of depth LUT_BITS+1 .. LUT_BITS+L2_BITS under a subtabled prefix
  constexpr int DMAX = LUT_BITS + L2_BITS;
  for (int i = lane; i < ntree; i += 32) {
    const int d = H.ndepth[i];
    const bool leaf = H.left[i] == -1;
    if (d <= LUT_BITS || d > DMAX || (!leaf && d != DMAX)) continue;
    const uint32_t code = H.ncode[i];
    const uint16_t e1 = T.lut[code >> (d - LUT_BITS)];
    if ((e1 & 0xC000u) != 0x8000u) continue;  // prefix without a subtable
    const uint32_t rel = code & ((1u << (d - LUT_BITS)) - 1u);
    uint16_t* t2 = T.lut + LUT_SIZE + (e1 & 0x3FFFu);
    if (leaf) fill(t2, rel << (DMAX - d), 1u << (DMAX - d), (uint16_t)((d << 8) | H.sym[i]));
    else t2[rel] = (uint16_t)(0xC000u | i);
  }
}


// HBW blocks per warp: 4 for large batches (the serial scans run side by side), 1 when the batch
// has too few blocks to fill the GPU with 4 per warp (single images, small batches)
template <int HBW>
__global__ void __launch_bounds__(HW * 32) k_block_header(DecodeParams P) {
  __shared__ HdrScratch HS[HW];
  __shared__ HdrStage ST[HW][HBW];
  const Geom& g = P.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nblocks = P.batch * g.slots_per_image;
  const int gid0 = (blockIdx.x * HW + warp) * HBW;
  HdrScratch& H = HS[warp];
  // which of the warp's blocks are decoded: blocks not needed for this output level, or outside
  // decode_region's per-level boxes, are never read by the requested output pixels
  unsigned act = 0;
  for (int bi = 0; bi < HBW; ++bi) {
    const int gid = gid0 + bi;
    if (gid >= nblocks) break;
    const int b = fdiv(gid, g.md_spi);
    const SlotInfo si = slot_info(g, gid - b * g.slots_per_image);
    if (!(si.kind == 0 || si.lev > P.level) || (P.need && !P.need[gid])) {
      if (lane == 0) { P.dmeta[gid].needed = 0; P.tabs[gid].rc = -1; P.tabs[gid].dn = 0; }
      continue;
    }
    act |= 1u << bi;
    // stage the first 1 KB of the block (the whole header for <= ~8 Kbit headers)
    const u64 w0 = P.blk_off[gid] >> 2;
    const u64 nw = P.src.nbytes >> 2;
    for (int i = lane; i < 256; i += 32)
      ST[warp][bi].hw[i] = w0 + i < nw ? __ldg(reinterpret_cast<const uint32_t*>(P.src.data) + w0 + i) : 0u;
    for (int i = lane; i < 256; i += 32) reinterpret_cast<uint32_t*>(ST[warp][bi].tok)[i] = 0u;
  }
  if (!act) return;
  __syncwarp();
  // part A, lane bi on block bi (serial token scans side by side)
  HdrBits R;
  uint64_t mk[3] = {0, 0, 0};
  int rcA = 0, ntok = 0, maxopen = 1;
  HdrA A{0, 0, 0, 0};
  if (lane < HBW && ((act >> lane) & 1u)) {
    const int gid = gid0 + lane;
    const int b = fdiv(gid, g.md_spi);
    const SlotInfo si = slot_info(g, gid - b * g.slots_per_image);
    const u64 w0 = P.blk_off[gid] >> 2;
    const u64 nw = P.src.nbytes >> 2;
    BitSrc hsrc = P.src;
    hsrc.sw = ST[warp][lane].hw;
    hsrc.sw_lo = w0;
    hsrc.sw_n = nw > w0 ? (uint32_t)(nw - w0 < 256 ? nw - w0 : 256) : 0u;
    const u64 bstart = 8ull * P.blk_off[gid];
    const u64 bend = bstart + 8ull * P.blk_len[gid];
    R.init(hsrc, bstart, bend);
    rcA = parse_header_a(R, si.kind ? 3 : 1, A, mk, ST[warp][lane].tok, &ntok, &maxopen);
  }
  __syncwarp();
  for (int bi = 0; bi < HBW; ++bi) {
    if (!((act >> bi) & 1u)) continue;
    const int gid = gid0 + bi;
    const int rc_b = __shfl_sync(0xffffffffu, rcA, bi);
    const int nt_b = __shfl_sync(0xffffffffu, ntok, bi);
    const int mo_b = __shfl_sync(0xffffffffu, maxopen, bi);
    HdrA Ab;
    Ab.depth = __shfl_sync(0xffffffffu, A.depth, bi);
    Ab.cw = __shfl_sync(0xffffffffu, A.cw, bi);
    Ab.zr = __shfl_sync(0xffffffffu, A.zr, bi);
    Ab.nst = __shfl_sync(0xffffffffu, A.nst, bi);
    header_block(P, H, ST[warp][bi], Ab, rc_b, nt_b, mo_b, gid, bi, R, mk);
    __syncwarp();
  }
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

// ---- plane decode ----------------------------------------------------------------------------
// Every decoded plane starts at a seek-table entry, so the planes of a block decode
// independently.  A group of LPB lanes owns one block (two-level decode table in shared
// memory); the block's planes are ranked by bit length and snake-assigned to the lanes so their
// loads balance.  The lanes of a warp run different planes in lockstep, so the token loop is
// branch-free (predicated) -- any per-lane branch would be paid by the whole warp on almost
// every iteration:
//  * the 32 bits at the position come from one funnel shift of two payload words (wa, wb);
//  * payload words stream through a per-lane shared-memory ring of 8 x 16-byte chunks filled
//    by predicated cp.async seven chunks ahead (no registers wait on the loads);
//  * codes up to 16 bits resolve in one or two table lookups (longer: a rare tree walk);
//  * the plane is pre-zeroed; symbols are OR-ed into a register word at their byte position (a
//    zero run only advances the position) and the word is stored, predicated, when left.
// Any inconsistency (truncation, run overrun, plane end != next seek) flags the block; K2b then
// re-runs the reference's sequential algorithm for the exact error class.
constexpr int PT = 64;   // threads per decode CTA
constexpr int RING = 8;  // 16-byte chunks per lane ring
constexpr int TOK = 8;   // tokens per group (one warp vote, one ring refill)

// Only the first-level table (4 KB) is staged in shared memory; the second level (codes longer
// than LUT_BITS, rare) is read from the block's global table through L1.  Halving the staged
// bytes raises the resident decode CTAs per SM from 5 to 8 (the kernel is latency bound).
struct __align__(16) TabSmem {
  uint16_t lut[LUT_SIZE];
};

__device__ __forceinline__ uint32_t ldg_u16_if(bool p, const uint16_t* a) {
  uint32_t v;
  asm volatile(
      "{\n .reg .pred q;\n .reg .b16 h;\n setp.ne.b32 q, %2, 0;\n mov.b16 h, 0;\n @q ld.global.nc.u16 h, [%1];\n"
      " cvt.u32.u16 %0, h;\n}\n"
      : "=r"(v)
      : "l"(a), "r"((int)p));
  return v;
}

__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
// 16-byte async copy of `nsrc` (0..16) source bytes, zero-filling the rest; committed as one group
__device__ __forceinline__ void cp16_commit_if(bool p, uint32_t sdst, const void* gsrc, uint32_t nsrc) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n"
      " @q cp.async.ca.shared.global [%0], [%1], 16, %3;\n @q cp.async.commit_group;\n}\n" ::"r"(sdst),
      "l"(gsrc), "r"((int)p), "r"(nsrc)
      : "memory");
}
__device__ __forceinline__ void st_u32_if(bool p, uint32_t* a, uint32_t v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q st.global.u32 [%1], %2;\n}\n" ::"r"((int)p), "l"(a),
               "r"(v)
               : "memory");
}
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct DecCtx {
  const uint8_t* abase;  // this lane's block start rounded down to 16 bytes
  uint32_t nab;          // container bytes from abase (the copies zero-fill past them), capped
  u64 bitoff;            // 8 * (data - abase) mod 2^64: absolute bit -> bit relative to abase
  uint32_t lut_s;        // shared address of the decode table
  uint32_t ring_s;       // shared address of this lane's ring
  uint32_t zrs;          // zero-run symbol (~0 when counters are absent)
  int cw, csh;           // counter width, 32 - max(cw, 1)
  const BlockTab* G;     // tree (long-code fallback)
  const uint8_t* data;
  u64 nbytes;
};

// source of chunk c and its valid byte count (0 past the container: pure zero fill)
__device__ __forceinline__ void chunk_src(const DecCtx& C, uint32_t c, const void** src, uint32_t* n) {
  const uint32_t off = 16u * c;
  const uint32_t rem = C.nab > off ? C.nab - off : 0u;
  *n = rem < 16u ? rem : 16u;
  *src = C.abase + (rem ? off : 0u);
}

// Fill the ring with chunks c0 .. c0+RING-1 (slot = chunk & 7) and wait for them.
__device__ __forceinline__ void ring_load(const DecCtx& C, uint32_t c0) {
#pragma unroll
  for (int k = 0; k < RING; ++k) {
    const uint32_t c = c0 + k;
    const void* src;
    uint32_t n;
    chunk_src(C, c, &src, &n);
    cp16_commit_if(true, C.ring_s + 16 * (c & (RING - 1)), src, n);
  }
  cp_wait<0>();
}

__device__ __forceinline__ uint32_t ring_word(const DecCtx& C, uint32_t w) {
  return bswap32(lds_u32(C.ring_s + 4 * (w & (4 * RING - 1))));
}

// Code longer than the tables resolve: tree walk from `node`, the node at depth L0 the table
// entry names (L0 = LUT_BITS + L2_BITS for a second-level marker, LUT_BITS for a first-level
// prefix past the subtable capacity), over the bits after absolute position abs_code + L0.
__device__ __noinline__ int dec_long(const DecCtx& C, u64 abs_code, uint32_t room, int node, uint32_t L0) {
  BitSrc src{C.data, C.nbytes};
  const BlockTab& G = *C.G;
  uint32_t L = L0;
  while (G.left[node] != -1) {
    if (L >= room || L > 48) return -1;
    const u64 bp = abs_code + L;
    node = ((src.word(bp >> 5) >> (31 - (bp & 31))) & 1u) ? G.right[node] : G.left[node];
    ++L;
  }
  return (int)((L << 16) | (uint32_t)(G.sym[node] & 255));
}

__device__ __forceinline__ uint32_t lds_u16_if(bool p, uint32_t a) {
  uint32_t v;
  asm volatile(
      "{\n .reg .pred q;\n .reg .b16 h;\n setp.ne.b32 q, %2, 0;\n mov.b16 h, 0;\n @q ld.shared.u16 h, [%1];\n"
      " cvt.u32.u16 %0, h;\n}\n"
      : "=r"(v)
      : "r"(a), "r"((int)p));
  return v;
}

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp16_if(bool p, uint32_t sdst, const void* gsrc, uint32_t nsrc) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q cp.async.ca.shared.global [%0], [%1], 16, %3;\n}\n" ::"r"(sdst),
      "l"(gsrc), "r"((int)p), "r"(nsrc)
      : "memory");
}

// Decode the plane starting at absolute bit s (stream order): 2048 symbols into dst (512
// words).  Returns true if complete within the block; *endp = absolute end bit.  Truncation
// and run overrun are checked once at the end: the loop is bounded by the symbol count, stores
// stay inside the plane, and reads past the container are zero-filled by the ring copies.
// The token loop is branch-free: lanes that finished their plane or met a code longer than 16
// bits freeze (act = false).  TOK = 8 tokens run per warp vote; the loop leaves when every lane
// is done or any lane froze on a long code, which is then resolved by a tree walk outside the
// loop.  The payload ring is refilled once per group: a token advances the window by at most
// one word, so a group moves at most two 16-byte chunks; chunks up to RING-1 ahead of the
// current one are requested at the group's end and committed as one copy group, and every
// chunk a group can touch was requested at least two groups earlier, so waiting for all but
// the most recent group at the group's start never stalls on data in flight.  (Measured: a
// 4-chunk ring with 4-token groups fits 10 CTAs per SM instead of 9 but is 5% slower -- the
// requests are then only ~8 tokens ahead of their use, less than a DRAM round trip.)
// TWO = false: the warp's blocks have every code within the first-level table (no second
// level lookups, no long codes).
template <bool TWO>
__device__ __forceinline__ bool dec_plane(const DecCtx& C, bool have, u64 s, u64 bend, uint32_t* __restrict__ dst,
                                          u64* endp) {
  if (have) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll 8
    for (int i = 0; i < WB_PP / 16; ++i) d4[i] = make_uint4(0, 0, 0, 0);
  }
  // positions are relative to the aligned word space of abase (the lane's block)
  const u64 sa = s + C.bitoff;
  const uint32_t w0 = (uint32_t)(sa >> 5), p0 = (uint32_t)(sa & 31);
  uint32_t wi = w0;   // word index of wa
  uint32_t pos = p0;  // bit position within wa (< 32 between tokens)
  const u64 lim64 = bend > s ? bend - s : 0;
  const uint32_t lim = (uint32_t)(lim64 > 0x7FFFFFFFull ? 0x7FFFFFFFull : lim64);
  ring_load(C, wi >> 2);
  uint32_t wa = ring_word(C, wi), wb = ring_word(C, wi + 1);
  int o = have ? 0 : WB_PP;  // a lane without a plane runs frozen
  uint32_t acc = 0;
  bool fail = false;
  constexpr uint32_t wm = 0xFFFFFFFFu;
  // consume a decoded symbol whose code ends at `pos` (bits = window at the code start, len =
  // code length within it): zero-run counter, window advance, symbol/run output
  auto consume = [&](bool act, uint32_t sym, uint32_t len, uint32_t bits, uint32_t nx) {
    // zero-run counter: cw bits after the zr code (len + cw <= 32 bits of the window)
    const bool z = act && sym == C.zrs;
    const uint32_t ctr = z ? (bits << len) >> C.csh : 0u;
    pos += len + (z ? (uint32_t)C.cw : 0u);
    // advance the window by one word when the position leaves wa (<= 32 bits per token)
    const bool adv = pos >= 32;
    const uint32_t wn = wi + 1;
    wa = adv ? wb : wa;
    wb = adv ? nx : wb;
    wi = adv ? wn : wi;
    pos = adv ? pos - 32 : pos;
    const int o2 = act ? o + (ctr ? (int)ctr : 1) : o;
    acc |= (act && !ctr ? sym : 0u) << (8 * (o & 3));
    const bool st = act && ((o ^ o2) >= 4 || o2 >= WB_PP);
    st_u32_if(st, dst + (o >> 2), acc);
    acc = st ? 0u : acc;
    o = o2;
  };
  uint32_t nf = (wi >> 2) + RING;  // next chunk to request
  for (;;) {
    bool lng = false;
    cp_wait<1>();  // every chunk this group can read (see above)
#pragma unroll
    for (int u = 0; u < TOK; ++u) {
      // the word after wb (needed if this token leaves wa)
      const uint32_t nx = ring_word(C, wi + 2);
      const uint32_t bits = __funnelshift_l(wb, wa, pos);
      const uint32_t e1 = lds_u16(C.lut_s + ((bits >> (32 - LUT_BITS)) << 1));
      uint32_t e = e1;
      if constexpr (TWO) {
        const bool is2 = (e1 & 0xC000u) == 0x8000u;
        const uint32_t i2 = LUT_SIZE + (e1 & 0x3FFFu) + ((bits << LUT_BITS) >> (32 - L2_BITS));
        const uint32_t e2 = ldg_u16_if(is2, C.G->lut + i2);
        e = is2 ? e2 : e1;
      }
      const bool live = o < WB_PP;
      lng = TWO && live && (e & 0x8000u);
      const bool act = live && (!TWO || !(e & 0x8000u));
      consume(act, e & 255u, act ? (e >> 8) & 31u : 0u, bits, nx);
    }
    {  // refill: chunks up to RING-1 ahead of the current one (the slot of the one before it)
      const uint32_t last = (wi >> 2) + RING - 1;
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const bool p = nf <= last;
        const void* src;
        uint32_t n;
        chunk_src(C, nf, &src, &n);
        cp16_if(p, C.ring_s + 16 * (nf & (RING - 1)), src, n);
        nf += p ? 1u : 0u;
      }
      cp_commit();
    }
    // warp OR of (live | long << 1), once per group
    const uint32_t vote = __reduce_or_sync(wm, (o < WB_PP ? 1u : 0u) | (lng ? 2u : 0u));
    if (vote == 1u) continue;
    if (!(vote & 2u)) break;
    if (TWO && lng) {  // code longer than 16 bits (rare): tree walk, then re-position
      const uint32_t bits = __funnelshift_l(wb, wa, pos);
      const uint32_t e1 = lds_u16(C.lut_s + ((bits >> (32 - LUT_BITS)) << 1));
      const bool is2 = (e1 & 0xC000u) == 0x8000u;
      const uint32_t e = is2 ? (uint32_t)C.G->lut[LUT_SIZE + (e1 & 0x3FFFu) + ((bits << LUT_BITS) >> (32 - L2_BITS))]
                             : e1;
      const uint32_t used = (wi - w0) * 32 + pos - p0;
      const int r = dec_long(C, s + used, lim > used ? lim - used : 0u, (int)(e & 0x3FFFu),
                             is2 ? (uint32_t)(LUT_BITS + L2_BITS) : (uint32_t)LUT_BITS);
      if (r < 0) {
        fail = true;
        o = WB_PP;  // stop this lane
      } else {
        const u64 na = s + used + ((uint32_t)r >> 16) + C.bitoff;
        wi = (uint32_t)(na >> 5);
        pos = (uint32_t)(na & 31);
        cp_wait<0>();
        ring_load(C, wi >> 2);
        nf = (wi >> 2) + RING;
        wa = ring_word(C, wi);
        wb = ring_word(C, wi + 1);
        consume(true, (uint32_t)r & 255u, 0u, __funnelshift_l(wb, wa, pos), ring_word(C, wi + 2));
      }
    }
  }
  cp_wait<0>();
  const uint32_t used = (wi - w0) * 32 + pos - p0;
  *endp = s + used;
  return !fail && o == WB_PP && used <= lim;
}

// K2: LPB lanes per block, PT / LPB blocks per CTA.
template <int LPB>
__global__ void __launch_bounds__(PT) k_block_planes(DecodeParams P) {
  constexpr int BPC = PT / LPB;
  constexpr int MAXP = (WB_MAX_SLOTS + LPB - 1) / LPB;  // planes per lane
  static_assert(MAXP <= 8, "a lane's plane list fits one 64-bit register");
  __shared__ TabSmem TS[BPC];
  // the payload rings; before the planes are decoded they hold the plane bit lengths and the
  // lanes' plane lists (9 instead of 8 CTAs per SM)
  __shared__ __align__(16) uint32_t RB[PT][4 * RING];
  static_assert(sizeof(RB) >= BPC * WB_MAX_SLOTS * sizeof(uint32_t) + BPC * LPB * MAXP, "overlay fits the rings");
  uint32_t (*plen)[WB_MAX_SLOTS] = reinterpret_cast<uint32_t (*)[WB_MAX_SLOTS]>(&RB[0][0]);
  uint8_t (*plist)[LPB][MAXP] = reinterpret_cast<uint8_t (*)[LPB][MAXP]>(&RB[0][0] + BPC * WB_MAX_SLOTS);
  const int tid = threadIdx.x;
  const int sub = tid / LPB, l = tid % LPB;
  const int gid = blockIdx.x * BPC + sub;
  const int nblocks = P.batch * P.g.slots_per_image;
  const BlockTab* Gp = gid < nblocks ? &P.tabs[gid] : nullptr;
  const int dn = Gp && Gp->rc == 0 ? Gp->dn : 0;
  u64 bend = 0, pstart = 0;
  if (dn) {
    const BlockTab& G = *Gp;
    {  // decode tables -> smem (16-B copies)
      const uint4* a = reinterpret_cast<const uint4*>(G.lut);
      uint4* d = reinterpret_cast<uint4*>(TS[sub].lut);
      for (int i = l; i < LUT_SIZE / 8; i += LPB) d[i] = a[i];
    }
    bend = 8ull * (P.blk_off[gid] + P.blk_len[gid]);
    pstart = G.pstart;
    // plane bit lengths (the last plane: to the block end)
    const int nst = G.nst;
    for (int j = l; j < dn; j += LPB) {
      const u64 a = pstart + G.seek[j];
      const u64 b = j + 1 < nst ? pstart + G.seek[j + 1] : bend;
      plen[sub][j] = b > a ? (uint32_t)min(b - a, (u64)0xFFFFFFFFull) : 0u;
    }
  }
  __syncthreads();
  if (dn) {
    // rank planes by length (desc) and snake-assign ranks to lanes
    for (int j = l; j < dn; j += LPB) {
      const uint32_t lj = plen[sub][j];
      int r = 0;
      for (int k = 0; k < dn; ++k) {
        const uint32_t lk = plen[sub][k];
        r += (lk > lj) || (lk == lj && k < j);
      }
      const int row = r / LPB, col = r % LPB;
      plist[sub][(row & 1) ? LPB - 1 - col : col][row] = (uint8_t)j;
    }
  }
  __syncthreads();
  // Every lane of the warp runs the same number of dec_plane calls (the warp maximum) so the
  // token loop can vote with a full mask; lanes without a plane run frozen.
  bool work = dn > 0;
  if (work && Gp->seek[0] != 0) {
    if (l == 0) atomicOr(&P.flags[gid], 1u);
    work = false;
  }
  // my planes: rows 0..rows-2 are full; the last row may skip this lane -> plist[sub][l][0..np)
  int np = 0;
  if (work) {
    const int rows = (dn + LPB - 1) / LPB;
    const int lastcol = ((rows - 1) & 1) ? LPB - 1 - l : l;
    np = rows - 1 + ((rows - 1) * LPB + lastcol < dn ? 1 : 0);
  }
  u64 mine = 0;  // this lane's plane list, one byte per plane
  for (int k = 0; k < np; ++k) mine |= (u64)plist[sub][l][k] << (8 * k);
  __syncthreads();  // the rings are free from here on
  const int npw = __reduce_max_sync(0xFFFFFFFFu, np);
  if (npw == 0) return;
  DecCtx C;
  // word positions are 32-bit relative to the lane's own block (rounded down to 16 bytes), so a
  // call may span any number of bytes; only a single block must stay below 512 MB
  const uintptr_t da = reinterpret_cast<uintptr_t>(P.src.data);
  const uintptr_t ab = (da + (work ? P.blk_off[gid] : 0)) & ~(uintptr_t)15;
  C.abase = reinterpret_cast<const uint8_t*>(ab);
  C.bitoff = 8ull * (u64)(da - ab);  // wraps: relative = absolute - 8 * (abase - data)
  {
    const u64 rem = (u64)(da + P.src.nbytes - ab);
    C.nab = (uint32_t)(rem > 0xFFFFFF00ull ? 0xFFFFFF00ull : rem);
  }
  C.data = P.src.data;
  C.nbytes = P.src.nbytes;
  C.lut_s = (uint32_t)__cvta_generic_to_shared(TS[sub].lut);
  C.ring_s = (uint32_t)__cvta_generic_to_shared(RB[tid]);
  const int cw = work ? Gp->cw : 0;
  C.cw = cw;
  C.zrs = cw ? (uint32_t)Gp->zr : 0xFFFFFFFFu;  // no counters: zr never matches
  C.csh = 32 - (cw ? cw : 1);
  C.G = Gp ? Gp : P.tabs;  // lanes without a block still form (never use) second-level addresses
  uint8_t* symbase = P.syms + (i64)gid * P.g.sym_stride_hp;
  uint32_t bad = 0;
  const bool two = __any_sync(0xFFFFFFFFu, work && Gp->two_level);  // warp-uniform table mode
  for (int k = 0; k < npw; ++k) {
    const bool have = k < np;
    const int j = have ? (int)((mine >> (8 * k)) & 255u) : 0;
    const u64 ps = have ? pstart + Gp->seek[j] : 0;
    u64 endp = 0;
    uint32_t* dstp = reinterpret_cast<uint32_t*>(symbase + (have ? (i64)Gp->slot_of[j] * WB_PP : 0));
    const bool ok = two ? dec_plane<true>(C, have, ps, bend, dstp, &endp) : dec_plane<false>(C, have, ps, bend, dstp, &endp);
    // The reference checks the start of every decoded plane (blocks.py:241-242), i.e. the ends
    // of planes 0..dn-2; the last decoded plane just stops after 2048 symbols.
    if (have) bad |= (ok && (j + 1 >= dn || endp == pstart + Gp->seek[j + 1])) ? 0u : 1u;
  }
  if (bad) atomicOr(&P.flags[gid], 1u);
}

// ---- plane decode, continuous lists -----------------------------------------------------------
// k_block_planes runs the lanes' planes in lockstep rounds: round r costs the warp its longest
// plane of that round, so a block of 23 planes on 16 lanes pays longest + 17th-longest (measured
// on the cfg4 generator: 73% of the lane steps decode a token).  Here every lane walks its own
// list: a lane that finishes a plane switches to its next one at the following group boundary
// while the other lanes carry on, so the warp's cost is the heaviest lane's token sum, and the
// lists are built by longest-first greedy assignment (LPT) instead of the snake.  A lane keeps two
// payload rings: the next plane's first chunks are requested into the idle ring when the current
// plane starts, long before the switch reads them, so a switch waits for nothing.
__device__ __forceinline__ void ring_request(const DecCtx& C, uint32_t rs, uint32_t c0) {
#pragma unroll
  for (int k = 0; k < RING; ++k) {
    const uint32_t c = c0 + k;
    const void* src;
    uint32_t n;
    chunk_src(C, c, &src, &n);
    cp16_commit_if(true, rs + 16 * (c & (RING - 1)), src, n);
  }
}
__device__ __forceinline__ uint32_t ring_word_at(uint32_t rs, uint32_t w) {
  return bswap32(lds_u32(rs + 4 * (w & (4 * RING - 1))));
}

template <bool TWO>
__device__ __forceinline__ uint32_t dec_list(const DecCtx& C, int np, u64 mine, const BlockTab* Gp, u64 pstart,
                                             u64 bend, uint8_t* symbase, int dn, uint32_t ring2_s) {
  // pre-zero every plane of the list (zero runs only advance the position)
  for (int k = 0; k < np; ++k) {
    const int j = (int)((mine >> (8 * k)) & 255u);
    uint4* d4 = reinterpret_cast<uint4*>(symbase + (i64)Gp->slot_of[j] * WB_PP);
#pragma unroll 8
    for (int i = 0; i < WB_PP / 16; ++i) d4[i] = make_uint4(0, 0, 0, 0);
  }
  uint32_t rs = C.ring_s, rs2 = ring2_s;
  int ci = 0, j = 0;
  u64 s = 0;
  uint32_t w0 = 0, p0 = 0, lim = 0;
  uint32_t* dst = reinterpret_cast<uint32_t*>(symbase);
  // start of plane k of the list: absolute bit, word / bit position relative to abase, bit budget
  auto setup = [&](int k) {
    j = (int)((mine >> (8 * k)) & 255u);
    s = pstart + Gp->seek[j];
    const u64 sa = s + C.bitoff;
    w0 = (uint32_t)(sa >> 5);
    p0 = (uint32_t)(sa & 31);
    const u64 lim64 = bend > s ? bend - s : 0;
    lim = (uint32_t)(lim64 > 0x7FFFFFFFull ? 0x7FFFFFFFull : lim64);
    dst = reinterpret_cast<uint32_t*>(symbase + (i64)Gp->slot_of[j] * WB_PP);
  };
  auto first_chunk = [&](int k) {
    const int jj = (int)((mine >> (8 * k)) & 255u);
    return (uint32_t)((pstart + Gp->seek[jj] + C.bitoff) >> 7);
  };
  const bool have = np > 0;
  if (have) setup(0);
  uint32_t wi = w0, pos = p0;
  ring_request(C, rs, wi >> 2);
  if (np > 1) ring_request(C, rs2, first_chunk(1));
  cp_wait<0>();
  uint32_t wa = ring_word_at(rs, wi), wb = ring_word_at(rs, wi + 1);
  int o = have ? 0 : WB_PP;  // a lane without a plane runs frozen
  uint32_t acc = 0;
  bool fail = false;
  uint32_t bad = 0;
  constexpr uint32_t wm = 0xFFFFFFFFu;
  auto consume = [&](bool act, uint32_t sym, uint32_t len, uint32_t bits, uint32_t nx) {
    const bool z = act && sym == C.zrs;
    const uint32_t ctr = z ? (bits << len) >> C.csh : 0u;
    pos += len + (z ? (uint32_t)C.cw : 0u);
    const bool adv = pos >= 32;
    const uint32_t wn = wi + 1;
    wa = adv ? wb : wa;
    wb = adv ? nx : wb;
    wi = adv ? wn : wi;
    pos = adv ? pos - 32 : pos;
    const int o2 = act ? o + (ctr ? (int)ctr : 1) : o;
    acc |= (act && !ctr ? sym : 0u) << (8 * (o & 3));
    const bool st = act && ((o ^ o2) >= 4 || o2 >= WB_PP);
    st_u32_if(st, dst + (o >> 2), acc);
    acc = st ? 0u : acc;
    o = o2;
  };
  // the plane just finished (or failed): the reference checks the start of every decoded plane
  // (blocks.py:241-242), i.e. the ends of planes 0..dn-2; the last one just stops after 2048
  auto finish = [&]() {
    const uint32_t used = (wi - w0) * 32 + pos - p0;
    const bool ok = !fail && o == WB_PP && used <= lim;
    bad |= (ok && (j + 1 >= dn || s + used == pstart + Gp->seek[j + 1])) ? 0u : 1u;
  };
  uint32_t nf = (wi >> 2) + RING;  // next chunk to request
  for (;;) {
    bool lng = false;
    cp_wait<1>();
#pragma unroll
    for (int u = 0; u < TOK; ++u) {
      const uint32_t nx = ring_word_at(rs, wi + 2);
      const uint32_t bits = __funnelshift_l(wb, wa, pos);
      const uint32_t e1 = lds_u16(C.lut_s + ((bits >> (32 - LUT_BITS)) << 1));
      uint32_t e = e1;
      if constexpr (TWO) {
        const bool is2 = (e1 & 0xC000u) == 0x8000u;
        const uint32_t i2 = LUT_SIZE + (e1 & 0x3FFFu) + ((bits << LUT_BITS) >> (32 - L2_BITS));
        const uint32_t e2 = ldg_u16_if(is2, C.G->lut + i2);
        e = is2 ? e2 : e1;
      }
      const bool live = o < WB_PP;
      lng = TWO && live && (e & 0x8000u);
      const bool act = live && (!TWO || !(e & 0x8000u));
      consume(act, e & 255u, act ? (e >> 8) & 31u : 0u, bits, nx);
    }
    {  // refill (live lanes only: a finished lane leaves nothing in flight for its switch to wait on)
      const uint32_t last = (wi >> 2) + RING - 1;
      const bool livep = o < WB_PP;
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const bool p = livep && nf <= last;
        const void* src;
        uint32_t n;
        chunk_src(C, nf, &src, &n);
        cp16_if(p, rs + 16 * (nf & (RING - 1)), src, n);
        nf += p ? 1u : 0u;
      }
      cp_commit();
    }
    const bool next = o >= WB_PP && !lng && ci + 1 < np;  // this lane switches planes
    uint32_t vote = __reduce_or_sync(wm, (o < WB_PP ? 1u : 0u) | (lng ? 2u : 0u) | (next ? 4u : 0u));
    if (vote & 4u) {
      if (next) {
        finish();
        ++ci;
        setup(ci);
        wi = w0;
        pos = p0;
        const uint32_t t = rs; rs = rs2; rs2 = t;
        cp_wait<1>();  // this plane's first chunks were requested a whole plane ago
        wa = ring_word_at(rs, wi);
        wb = ring_word_at(rs, wi + 1);
        nf = (wi >> 2) + RING;
        o = 0;
        acc = 0;
        fail = false;
        if (ci + 1 < np) {  // third and later planes of a list (more than 32 planes in the block)
          cp_wait<0>();
          ring_request(C, rs2, first_chunk(ci + 1));
        }
      }
      vote = __reduce_or_sync(wm, (o < WB_PP ? 1u : 0u) | (lng ? 2u : 0u));
    }
    if (vote == 1u) continue;
    if (!(vote & 2u)) break;
    if (TWO && lng) {  // code longer than 16 bits (rare): tree walk, then re-position
      const uint32_t bits = __funnelshift_l(wb, wa, pos);
      const uint32_t e1 = lds_u16(C.lut_s + ((bits >> (32 - LUT_BITS)) << 1));
      const bool is2 = (e1 & 0xC000u) == 0x8000u;
      const uint32_t e = is2 ? (uint32_t)C.G->lut[LUT_SIZE + (e1 & 0x3FFFu) + ((bits << LUT_BITS) >> (32 - L2_BITS))]
                             : e1;
      const uint32_t used = (wi - w0) * 32 + pos - p0;
      const int r = dec_long(C, s + used, lim > used ? lim - used : 0u, (int)(e & 0x3FFFu),
                             is2 ? (uint32_t)(LUT_BITS + L2_BITS) : (uint32_t)LUT_BITS);
      if (r < 0) {
        fail = true;
        o = WB_PP;  // stop this plane (the block is flagged; its later planes are still decoded)
      } else {
        const u64 na = s + used + ((uint32_t)r >> 16) + C.bitoff;
        wi = (uint32_t)(na >> 5);
        pos = (uint32_t)(na & 31);
        cp_wait<0>();
        ring_request(C, rs, wi >> 2);
        cp_wait<0>();
        nf = (wi >> 2) + RING;
        wa = ring_word_at(rs, wi);
        wb = ring_word_at(rs, wi + 1);
        consume(true, (uint32_t)r & 255u, 0u, __funnelshift_l(wb, wa, pos), ring_word_at(rs, wi + 2));
      }
    }
  }
  cp_wait<0>();
  if (have) finish();
  return bad;
}

// LPB lanes per block, PT / LPB blocks per CTA; two rings per lane.
template <int LPB>
__global__ void __launch_bounds__(PT) k_block_planes_c(DecodeParams P) {
  constexpr int BPC = PT / LPB;
  __shared__ TabSmem TS[BPC];
  // the payload rings (two per lane); before the planes are decoded they hold the plane bit
  // lengths and the planes in descending length order
  __shared__ __align__(16) uint32_t RB[PT][2 * 4 * RING];
  static_assert(sizeof(RB) >= BPC * WB_MAX_SLOTS * sizeof(uint32_t) + BPC * WB_MAX_SLOTS, "overlay fits the rings");
  uint32_t (*plen)[WB_MAX_SLOTS] = reinterpret_cast<uint32_t (*)[WB_MAX_SLOTS]>(&RB[0][0]);
  uint8_t (*ord)[WB_MAX_SLOTS] = reinterpret_cast<uint8_t (*)[WB_MAX_SLOTS]>(&RB[0][0] + BPC * WB_MAX_SLOTS);
  const int tid = threadIdx.x;
  const int sub = tid / LPB, l = tid % LPB;
  const int gid = blockIdx.x * BPC + sub;
  const int nblocks = P.batch * P.g.slots_per_image;
  const BlockTab* Gp = gid < nblocks ? &P.tabs[gid] : nullptr;
  int dn = Gp && Gp->rc == 0 ? Gp->dn : 0;
  u64 bend = 0, pstart = 0;
  if (dn) {
    const BlockTab& G = *Gp;
    {
      const uint4* a = reinterpret_cast<const uint4*>(G.lut);
      uint4* d = reinterpret_cast<uint4*>(TS[sub].lut);
      for (int i = l; i < LUT_SIZE / 8; i += LPB) d[i] = a[i];
    }
    bend = 8ull * (P.blk_off[gid] + P.blk_len[gid]);
    pstart = G.pstart;
    const int nst = G.nst;
    for (int jj = l; jj < dn; jj += LPB) {
      const u64 a = pstart + G.seek[jj];
      const u64 b = jj + 1 < nst ? pstart + G.seek[jj + 1] : bend;
      plen[sub][jj] = b > a ? (uint32_t)min(b - a, (u64)0x07FFFFFFull) : 0u;
    }
  }
  __syncthreads();
  if (dn) {  // planes in descending length order
    for (int jj = l; jj < dn; jj += LPB) {
      const uint32_t lj = plen[sub][jj];
      int r = 0;
      for (int k = 0; k < dn; ++k) {
        const uint32_t lk = plen[sub][k];
        r += (lk > lj) || (lk == lj && k < jj);
      }
      ord[sub][r] = (uint8_t)jj;
    }
  }
  __syncthreads();
  if (dn && Gp->seek[0] != 0) {
    if (l == 0) atomicOr(&P.flags[gid], 1u);
    dn = 0;
  }
  // longest-first greedy assignment: every plane, longest first, goes to the lane of the block
  // with the smallest bit load so far (at most 8 planes per lane: one byte each in `mine`)
  u64 mine = 0;
  int np = 0;
  {
    uint32_t load = 0;
    const int dmax = __reduce_max_sync(0xFFFFFFFFu, dn);
    for (int r = 0; r < dmax; ++r) {
      const bool in = r < dn;
      const int jj = in ? ord[sub][r] : 0;
      uint32_t key = np >= 8 ? 0xFFFFFFFFu : ((load << 4) | (uint32_t)l);
#pragma unroll
      for (int d = LPB / 2; d > 0; d >>= 1) key = min(key, __shfl_xor_sync(0xFFFFFFFFu, key, d));
      if (in && (int)(key & 15u) == l && key != 0xFFFFFFFFu) {
        mine |= (u64)jj << (8 * np);
        ++np;
        load = min(load + plen[sub][jj], 0x07FFFFFFu);
      }
    }
    // planes no lane could take (more than 8 per lane: impossible for <= 96 planes on 16 lanes
    // unless the loads are degenerate) would be lost: flag the block instead
    int taken = np;
#pragma unroll
    for (int d = LPB / 2; d > 0; d >>= 1) taken += __shfl_xor_sync(0xFFFFFFFFu, taken, d);
    if (taken != dn && l == 0 && gid < nblocks) atomicOr(&P.flags[gid], 1u);
  }
  __syncthreads();  // the rings are free from here on
  const int npw = __reduce_max_sync(0xFFFFFFFFu, np);
  if (npw == 0) return;
  const bool work = dn > 0;
  DecCtx C;
  const uintptr_t da = reinterpret_cast<uintptr_t>(P.src.data);
  const uintptr_t ab = (da + (work ? P.blk_off[gid] : 0)) & ~(uintptr_t)15;
  C.abase = reinterpret_cast<const uint8_t*>(ab);
  C.bitoff = 8ull * (u64)(da - ab);
  {
    const u64 rem = (u64)(da + P.src.nbytes - ab);
    C.nab = (uint32_t)(rem > 0xFFFFFF00ull ? 0xFFFFFF00ull : rem);
  }
  C.data = P.src.data;
  C.nbytes = P.src.nbytes;
  C.lut_s = (uint32_t)__cvta_generic_to_shared(TS[sub].lut);
  C.ring_s = (uint32_t)__cvta_generic_to_shared(RB[tid]);
  const int cw = work ? Gp->cw : 0;
  C.cw = cw;
  C.zrs = cw ? (uint32_t)Gp->zr : 0xFFFFFFFFu;
  C.csh = 32 - (cw ? cw : 1);
  C.G = Gp ? Gp : P.tabs;  // lanes without a block still form (never use) second-level addresses
  uint8_t* symbase = P.syms + (i64)gid * P.g.sym_stride_hp;
  const bool two = __any_sync(0xFFFFFFFFu, work && Gp->two_level);
  const uint32_t bad = two ? dec_list<true>(C, np, mine, Gp, pstart, bend, symbase, dn, C.ring_s + 16 * RING)
                           : dec_list<false>(C, np, mine, Gp, pstart, bend, symbase, dn, C.ring_s + 16 * RING);
  if (bad) atomicOr(&P.flags[gid], 1u);
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
  const u64* hpdepth;  // max detail-block depth of the call (DevStatus::pad, set by k_block_header)
  int allow16;         // detail planes may be stored as int16 (image decode; not the block API)
};

// Detail planes (LH, HL, HH) hold int16 coefficients when every decoded detail block of the call
// has depth <= 16; LL planes are always int32.  Both instantiations are launched and the one
// that does not apply returns at once (no host round trip to choose).
__device__ __forceinline__ bool detail16(const u64* hpdepth, int allow16) { return allow16 && *hpdepth <= 16; }

// Thread = 4 consecutive stream positions k0..k0+3 (k0 % 4 == 0) of one subband, i.e. the 2x2
// areas (R, C), (R+1, C), (R, C+1), (R+1, C+1) with R = 2*(k0>>6), C = (k0>>1)&31 -- an 8x4
// coefficient patch (bitplanes.py:159-166 for 128x128).  Per plane one coalesced u32 load
// gives the 4 positions' symbols; 4 planes are byte-transposed per position and every
// coefficient's 4 magnitude bits are gathered with one multiply.
template <typename CT>
__device__ __forceinline__ void reconstruct_body(const ReconParams& P, const DecMeta& dm, const SlotInfo& si, int b) {
  const Geom& g = P.g;
  const int gid = blockIdx.x;
  constexpr bool I16 = sizeof(CT) == 2;
  const LevelGeom& lg = g.lv[si.lev];
  const int nsub = dm.nsub, depth = dm.depth;
  const uint8_t* symbase = P.syms + (i64)gid * g.sym_stride_hp;
  int32_t* cbase = P.coef + (i64)b * g.img_stride + (i64)si.c * g.chan_stride;
  const int y0 = si.r * WB_DIM, x0 = si.col * WB_DIM;
  const int s = blockIdx.y;
  if (s >= nsub) return;
  CT* plane = reinterpret_cast<CT*>(cbase + lg.off[si.kind ? 1 + s : 0]);
  auto word = [&](int pb, int k0) -> uint32_t {  // symbols k0..k0+3 of plane pb (0 if absent)
    if (pb >= depth) return 0u;
    const int sl = pb * nsub + s;
    if (!((dm.decoded[sl >> 5] >> (sl & 31)) & 1u)) return 0u;
    return *reinterpret_cast<const uint32_t*>(symbase + (i64)sl * WB_PP + k0);
  };
  for (int k0 = 4 * threadIdx.x; k0 < WB_PP; k0 += 4 * 256) {
    uint32_t mag[4][8];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 8; ++i) mag[j][i] = 0;
    const uint32_t sign = word(0, k0);
    for (int pb = 1; pb < depth; pb += 4) {
      const uint32_t x0w = word(pb, k0), x1w = word(pb + 1, k0), x2w = word(pb + 2, k0), x3w = word(pb + 3, k0);
      if (!(x0w | x1w | x2w | x3w)) continue;
      // y[j] byte p = symbol of position j in plane pb+p
      const uint32_t lo01 = __byte_perm(x0w, x1w, 0x5140), lo23 = __byte_perm(x2w, x3w, 0x5140);
      const uint32_t hi01 = __byte_perm(x0w, x1w, 0x7362), hi23 = __byte_perm(x2w, x3w, 0x7362);
      const uint32_t y[4] = {__byte_perm(lo01, lo23, 0x5410), __byte_perm(lo01, lo23, 0x7632),
                             __byte_perm(hi01, hi23, 0x5410), __byte_perm(hi01, hi23, 0x7632)};
      const int shl = depth - 4 - pb;  // weight of the 4th plane of the group (may be < 0)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t nib = (((y[j] >> i) & 0x01010101u) * 0x08040201u) >> 24;
          mag[j][i] |= shl >= 0 ? nib << shl : nib >> (-shl);
        }
    }
    int v[4][8];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 8; ++i) v[j][i] = ((sign >> (8 * j + i)) & 1u) ? -(int)mag[j][i] : (int)mag[j][i];
    const int R = 2 * (k0 >> 6), C = (k0 >> 1) & 31;
    CT* pp = plane + (i64)(y0 + 2 * R) * lg.pw + x0 + 4 * C;
    // rows 2R, 2R+1: positions 0 (cols 4C..) and 2 (cols 4C+4..); rows 2R+2, 2R+3: positions 1, 3
    auto st4 = [&](CT* q, int a, int b2, int c, int d) {
      if constexpr (I16)
        *reinterpret_cast<uint2*>(q) = make_uint2((uint32_t)(a & 0xFFFF) | ((uint32_t)b2 << 16),
                                                  (uint32_t)(c & 0xFFFF) | ((uint32_t)d << 16));
      else
        *reinterpret_cast<int4*>(q) = make_int4(a, b2, c, d);
    };
    st4(pp, v[0][0], v[0][1], v[0][2], v[0][3]);
    st4(pp + 4, v[2][0], v[2][1], v[2][2], v[2][3]);
    st4(pp + lg.pw, v[0][4], v[0][5], v[0][6], v[0][7]);
    st4(pp + lg.pw + 4, v[2][4], v[2][5], v[2][6], v[2][7]);
    st4(pp + 2 * lg.pw, v[1][0], v[1][1], v[1][2], v[1][3]);
    st4(pp + 2 * lg.pw + 4, v[3][0], v[3][1], v[3][2], v[3][3]);
    st4(pp + 3 * lg.pw, v[1][4], v[1][5], v[1][6], v[1][7]);
    st4(pp + 3 * lg.pw + 4, v[3][4], v[3][5], v[3][6], v[3][7]);
  }
}

// 8x8 bit transpose: byte j of the result holds bit j of each of the 8 input bytes
// (bit i of result byte j = bit j of input byte i).
__device__ __forceinline__ uint64_t tr8x8(uint64_t x) {
  uint64_t t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull;
  x = x ^ t ^ (t << 7);
  t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull;
  x = x ^ t ^ (t << 14);
  t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull;
  return x ^ t ^ (t << 28);
}

// Detail blocks of an int16 decode (depth <= 16).  Per 8 magnitude planes and area position, one
// 8x8 bit transpose of the planes' symbol bytes yields every pixel's 8 magnitude bits at once
// (byte i = pixel i, planes ordered so bit p carries weight 2^(depth-1-top+p)); pixel pairs are
// packed into int16x2 words with byte permutes, shifted into place, signed per 16-bit field and
// stored as 16-byte rows.  All symbol words of a position group are loaded before any is used.
__device__ __forceinline__ void reconstruct_body16(const ReconParams& P, const DecMeta& dm, const SlotInfo& si,
                                                   int b) {
  const Geom& g = P.g;
  const int gid = blockIdx.x;
  const LevelGeom& lg = g.lv[si.lev];
  const int depth = dm.depth;  // <= 16 here
  const int s = blockIdx.y;
  if (s >= 3) return;
  const uint8_t* symbase = P.syms + (i64)gid * g.sym_stride_hp + (i64)s * WB_PP;
  int32_t* cbase = P.coef + (i64)b * g.img_stride + (i64)si.c * g.chan_stride;
  int16_t* plane = reinterpret_cast<int16_t*>(cbase + lg.off[1 + s]);
  const int y0 = si.r * WB_DIM, x0 = si.col * WB_DIM;
  uint32_t pm = 0;  // bit pb: plane pb of this subband decoded
  for (int pb = 0; pb < depth; ++pb) {
    const int sl = pb * 3 + s;
    pm |= ((dm.decoded[sl >> 5] >> (sl & 31)) & 1u) << pb;
  }
  const bool two = depth > 9;  // a second group of 8 magnitude planes (planes 9..15)
#pragma unroll 1
  for (int k0 = 4 * threadIdx.x; k0 < WB_PP; k0 += 4 * 256) {
    uint32_t w[16];
#pragma unroll
    for (int pb = 0; pb < 16; ++pb)
      w[pb] = ((pm >> pb) & 1u) ? __ldg(reinterpret_cast<const uint32_t*>(symbase + (i64)pb * 3 * WB_PP + k0)) : 0u;
    uint32_t M[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) M[j][q] = 0;
#pragma unroll
    for (int grp = 0; grp < 2; ++grp) {
      if (grp == 1 && !two) break;
      const int top = 8 * grp + 8;  // byte p of the transpose input = plane top - p
      uint32_t a[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) a[p] = (top - p) < 16 ? w[(top - p) & 15] : 0u;
      // 4x4 byte transposes: lo[j] = (a0_j, a1_j, a2_j, a3_j), hi[j] = (a4_j .. a7_j)
      uint32_t lo[4], hi[4];
      {
        const uint32_t l01 = __byte_perm(a[0], a[1], 0x5140), l23 = __byte_perm(a[2], a[3], 0x5140);
        const uint32_t h01 = __byte_perm(a[0], a[1], 0x7362), h23 = __byte_perm(a[2], a[3], 0x7362);
        lo[0] = __byte_perm(l01, l23, 0x5410); lo[1] = __byte_perm(l01, l23, 0x7632);
        lo[2] = __byte_perm(h01, h23, 0x5410); lo[3] = __byte_perm(h01, h23, 0x7632);
      }
      {
        const uint32_t l01 = __byte_perm(a[4], a[5], 0x5140), l23 = __byte_perm(a[6], a[7], 0x5140);
        const uint32_t h01 = __byte_perm(a[4], a[5], 0x7362), h23 = __byte_perm(a[6], a[7], 0x7362);
        hi[0] = __byte_perm(l01, l23, 0x5410); hi[1] = __byte_perm(l01, l23, 0x7632);
        hi[2] = __byte_perm(h01, h23, 0x5410); hi[3] = __byte_perm(h01, h23, 0x7632);
      }
      const int sh = depth - 1 - top;  // weight exponent of bit 0
      const uint32_t rmask = sh < 0 ? (0xFFu >> (-sh)) * 0x10001u : 0xFFFFFFFFu;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t T = tr8x8(((uint64_t)hi[j] << 32) | lo[j]);
        const uint32_t tl = (uint32_t)T, th = (uint32_t)(T >> 32);
        const uint32_t pr[4] = {__byte_perm(tl, 0u, 0x4140), __byte_perm(tl, 0u, 0x4342),
                                __byte_perm(th, 0u, 0x4140), __byte_perm(th, 0u, 0x4342)};
#pragma unroll
        for (int q = 0; q < 4; ++q) M[j][q] |= sh >= 0 ? pr[q] << sh : (pr[q] >> (-sh)) & rmask;
      }
    }
    // signs (plane 0 byte j = pixels 0..7 of position j): v = sign ? -m : m per 16-bit field
    // (m < 2^15; a zero field with its sign set stays zero: the sign mask is cleared there)
    uint32_t V[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t sb = (w[0] >> (8 * j)) & 0xFFu;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t m = M[j][q];
        const uint32_t f = ((sb >> (2 * q)) & 1u) | (((sb >> (2 * q + 1)) & 1u) << 16);
        const uint32_t nz = ((m + 0x7FFF7FFFu) & 0x80008000u) >> 15;
        const uint32_t sm = (f & nz) * 0xFFFFu;
        V[j][q] = (m ^ sm) + (sm & 0x00010001u);
      }
    }
    const int R = 2 * (k0 >> 6), C = (k0 >> 1) & 31;
    int16_t* pp = plane + (i64)(y0 + 2 * R) * lg.pw + x0 + 4 * C;
    // rows 2R, 2R+1: positions 0 (cols 4C..) and 2 (cols 4C+4..); rows 2R+2, 2R+3: positions 1, 3
    *reinterpret_cast<uint4*>(pp) = make_uint4(V[0][0], V[0][1], V[2][0], V[2][1]);
    *reinterpret_cast<uint4*>(pp + lg.pw) = make_uint4(V[0][2], V[0][3], V[2][2], V[2][3]);
    *reinterpret_cast<uint4*>(pp + 2 * lg.pw) = make_uint4(V[1][0], V[1][1], V[3][0], V[3][1]);
    *reinterpret_cast<uint4*>(pp + 3 * lg.pw) = make_uint4(V[1][2], V[1][3], V[3][2], V[3][3]);
  }
}

__global__ void __launch_bounds__(256, 5) k_block_reconstruct(ReconParams P) {  // 5 CTAs/SM: 138 -> 132 us
  const Geom& g = P.g;
  const int gid = blockIdx.x;
  const DecMeta dm = P.dmeta[gid];
  if (!dm.needed) return;
  const int b = fdiv(gid, g.md_spi);
  const int slot = gid - b * g.slots_per_image;
  const SlotInfo si = slot_info(g, slot);
  // LL planes are int32; detail planes take the call's width (one uniform branch per block)
  if (si.kind && detail16(P.hpdepth, P.allow16)) reconstruct_body16(P, dm, si, b);
  else reconstruct_body<int32_t>(P, dm, si, b);
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
  if (nblocks >= 4096)
    k_block_header<4><<<(nblocks + HW * 4 - 1) / (HW * 4), HW * 32, 0, s>>>(P);
  else
    k_block_header<1><<<(nblocks + HW - 1) / HW, HW * 32, 0, s>>>(P);
  prof_mark("block_decode", s);
  // 16 lanes per block for batches of >= 2 cfg2-sized images (throughput: twice the planes per
  // lane, half the CTAs), else 32 (latency of a single image)
  // large batches: continuous per-lane plane lists (throughput); small ones keep the lockstep
  // rounds with 32 lanes per block (latency of a single image)
  static const int use_cont = [] {
    const char* e = getenv("WBPC_DEC_CONT");
    return e ? atoi(e) : 1;
  }();
  if (nblocks >= 512 && use_cont)
    k_block_planes_c<16><<<(nblocks + PT / 16 - 1) / (PT / 16), PT, 0, s>>>(P);
  else if (nblocks >= 512)
    k_block_planes<16><<<(nblocks + PT / 16 - 1) / (PT / 16), PT, 0, s>>>(P);
  else
    k_block_planes<32><<<(nblocks + PT / 32 - 1) / (PT / 32), PT, 0, s>>>(P);
  prof_mark("block_errors", s);
  k_block_errors<<<(nblocks + 127) / 128, 128, 0, s>>>(P);
  ReconParams R;
  R.g = g;
  R.syms = syms;
  R.dmeta = dmeta;
  R.coef = coef;
  R.hpdepth = &st->pad;
  R.allow16 = g.raw_kind < 0;
  prof_mark("block_reconstruct", s);
  k_block_reconstruct<<<dim3(nblocks, 3), 256, 0, s>>>(R);
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
  if (nblocks >= 4096)
    k_block_header<4><<<(nblocks + HW * 4 - 1) / (HW * 4), HW * 32, 0, s>>>(P);
  else
    k_block_header<1><<<(nblocks + HW - 1) / HW, HW * 32, 0, s>>>(P);
  return cudaGetLastError();
}

// plane_offsets (blocks.py:253-261): stored slots (b*nsub + s) and their seek entries.
__global__ void k_plane_offsets(const BlockTab* tab, int32_t* slots, uint32_t* offs, int32_t* count) {
  const BlockTab& T = *tab;
  if (threadIdx.x == 0) *count = T.rc == 0 ? T.dn : 0;
  if (T.rc) return;
  for (int i = threadIdx.x; i < T.dn; i += blockDim.x) {
    slots[i] = T.slot_of[i];
    offs[i] = T.seek[i];
  }
}

cudaError_t launch_plane_offsets(const BlockTab* tab, int32_t* slots, uint32_t* offs, int32_t* count, cudaStream_t s) {
  k_plane_offsets<<<1, 128, 0, s>>>(tab, slots, offs, count);
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
