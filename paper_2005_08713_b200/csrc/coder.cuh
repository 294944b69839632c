// coder.cuh — per-block metadata and Huffman helpers shared by the encode / truncate kernels.
#pragma once
#include "common.cuh"

namespace wb {

constexpr int CT = 256;  // threads per block-coder CTA

// Everything the emit pass needs about one coded block (written by k_block_analyze).
struct __align__(16) BlockMeta {
  uint32_t bytes;         // block byte length (padded to a byte, blocks.py:119 / bitio.py:47-50)
  uint32_t hdr_bits;      // bits before the payload
  uint32_t payload_bits;
  uint32_t tree_bits;
  uint16_t depth, nstored;
  uint8_t w, zr, kind, nsub;
  uint32_t stored[3];     // bit (b*nsub + s) = slot stored (blocks.py:89-90)
  uint32_t seek[WB_MAX_SLOTS];
  uint8_t code_len[256];  // 0xFF = absent
  uint32_t code_val[256];
  uint32_t tree_words[80];  // preorder tree bits, MSB-first big-endian words (entropy.py:259-269)
  uint32_t pad[5];
};

// Scratch for one Huffman build (shared memory).
struct HuffScratch {
  uint32_t key[512];     // (freq << 8) | min symbol; leaves 0..n-1 sorted, internal n..2n-2
  int16_t left[512];
  int16_t par[512];      // parent node
  uint16_t lc[512];      // leaves in the subtree
  uint8_t isr[512];      // 1 = right child of its parent
  int16_t leafsym[256];
  int n;
  int err;
};

// seek_entry_bits, blocks.py:45-50 (128x128 blocks): floor(log2(nsub*depth*2048)) + 5
__device__ __forceinline__ int seek_bits(int nsub, int depth) {
  unsigned total = (unsigned)(nsub * depth * WB_PP);
  return (31 - __clz(total)) + 5;
}

// Deterministic Huffman build of entropy.py:194-248 (heap on (frequency, min symbol), first popped
// = left child = bit 0) as a two-queue merge: leaves sorted by (f, sym), internal nodes appear in
// non-decreasing (f, min sym) order, so comparing the two queue heads reproduces every heappop.
// Code lengths/values and the preorder tree offsets come from one walk per leaf to the root:
//   depth = #edges, code bit d = 1 if the d-th edge from the leaf is a right edge,
//   preorder offset = sum over edges of 1 (+ bits of the left sibling subtree = 10*lc - 1 on a
//   right edge)  (write_tree, entropy.py:259-269: internal '0', leaf '1' + 8 bits).
// A single symbol gets a 0-bit code; CodeLengthError when an internal node is at depth >= 32.

// The build runs in three phases for many blocks per CTA: the two parallel phases run warp per block,
// the serial merge runs lane per block, so one warp instruction of the merge advances up to 32
// blocks' merges at once (the merge is instruction-issue bound when every block spends a warp on it).
// Phase A (warp): rank-sort the present symbols of `freq` into hs (keys, leaf symbols); returns n.
static __device__ int huff_rank_warp(const int* freq, HuffScratch* hs) {
  // full bitonic sort of the 256 keys in registers: element e = 8 * lane + i; absent symbols
  // carry the key ~0 and sort to the end, so position r < n is the leaf of rank r (keys are
  // distinct: the low byte is the symbol, which is also how the leaf symbol is recovered)
  const int lane = threadIdx.x & 31;
  constexpr uint32_t FULLM = 0xffffffffu;
  uint32_t v[8];
  int n = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int s = 8 * lane + i;
    const int f = freq[s];
    v[i] = f > 0 ? (((uint32_t)f << 8) | (uint32_t)s) : 0xFFFFFFFFu;
    n += __popc(__ballot_sync(FULLM, f > 0));
  }
#pragma unroll
  for (int k = 2; k <= 256; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 8) {  // partner in lane ^ (j / 8), same slot
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int e = 8 * lane + i;
          const uint32_t o = __shfl_xor_sync(FULLM, v[i], j >> 3);
          const bool asc = (e & k) == 0, lower = (e & j) == 0;
          v[i] = (lower == asc) ? min(v[i], o) : max(v[i], o);
        }
      } else {  // partner in this lane: slot i ^ j
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i & j) continue;
          const int e = 8 * lane + i;
          const bool asc = (e & k) == 0;
          const uint32_t a = v[i], b = v[i | j];
          v[i] = asc ? min(a, b) : max(a, b);
          v[i | j] = asc ? max(a, b) : min(a, b);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = 8 * lane + i;
    if (r < n) {
      hs->key[r] = v[i];
      hs->leafsym[r] = (int16_t)(v[i] & 255u);
      hs->lc[r] = 1;
    }
  }
  if (lane == 0) {
    hs->n = n;
    hs->err = n == 0 ? WBPC_ERR_EMPTY_ALPHABET : 0;  // entropy.py:210-211
  }
  __syncwarp();
  return n;
}

// Phase B (one thread per block): the serial two-queue merge.  Each step takes the two smallest
// of the first two sorted leaves (l0 < l1) and the first two internal nodes (q0 < q1) in one
// comparison network -- two leaves, two internal nodes, or one of each (entropy.py:219-222: the
// internal node only when strictly smaller; keys are distinct) -- and the four head refills for
// the next step are loaded together while the new node is formed.  Only keys and children are
// kept; parents, right-child flags and subtree leaf counts are derived in parallel afterwards (the
// right child is parked in par[k] meanwhile).
static __device__ void huff_merge_thread(HuffScratch* hs) {
  const int n = hs->n;
  const uint32_t INF = 0xFFFFFFFFu;
  int i = 0, j = n;
  uint32_t l0 = n > 0 ? hs->key[0] : INF, l1 = n > 1 ? hs->key[1] : INF, q0 = INF, q1 = INF;
  for (int k = n; k < 2 * n - 1; ++k) {
    const bool two_leaves = l1 < q0;
    const bool two_nodes = !two_leaves && q1 < l0;
    const bool lf = l0 < q0;
    const uint32_t ka = two_leaves ? l0 : (two_nodes ? q0 : (lf ? l0 : q0));
    const uint32_t kb = two_leaves ? l1 : (two_nodes ? q1 : (lf ? q0 : l0));
    const int a = two_leaves ? i : (two_nodes ? j : (lf ? i : j));
    const int b = two_leaves ? i + 1 : (two_nodes ? j + 1 : (lf ? j : i));
    i += two_leaves ? 2 : (two_nodes ? 0 : 1);
    j += two_nodes ? 2 : (two_leaves ? 0 : 1);
    const uint32_t nl0 = hs->key[min(i, 511)], nl1 = hs->key[min(i + 1, 511)];
    const uint32_t nq0 = hs->key[min(j, 511)], nq1 = hs->key[min(j + 1, 511)];
    const uint32_t kk = ((ka & ~255u) + (kb & ~255u)) | min(ka & 255u, kb & 255u);
    hs->key[k] = kk;
    hs->left[k] = (int16_t)a;
    hs->par[k] = (int16_t)b;
    l0 = i < n ? nl0 : INF;
    l1 = i + 1 < n ? nl1 : INF;
    q0 = j < k ? nq0 : (j == k ? kk : INF);
    q1 = j + 1 < k ? nq1 : (j + 1 == k ? kk : INF);
  }
}

// Phase C (warp): parents, subtree leaf counts (tree only), per-leaf walks -> code lengths
// (all 256 entries written, 0xFF = absent), optional code values and preorder tree bits.
static __device__ void huff_codes_warp(HuffScratch* hs, uint8_t* code_len, uint32_t* code_val, uint32_t* tree_out) {
  const int lane = threadIdx.x & 31;
  const int n = hs->n;
  for (int s = lane; s < 256; s += 32) {
    code_len[s] = 0xFF;
    if (code_val) code_val[s] = 0;
  }
  int ra[8], rb[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int kc = n + lane + 32 * r;
    ra[r] = rb[r] = -1;
    if (kc < 2 * n - 1) { ra[r] = hs->left[kc]; rb[r] = hs->par[kc]; }
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int kc = n + lane + 32 * r;
    if (kc < 2 * n - 1) {
      hs->par[ra[r]] = (int16_t)kc;
      hs->par[rb[r]] = (int16_t)kc;
      hs->isr[ra[r]] = 0;
      hs->isr[rb[r]] = 1;
      hs->lc[kc] = 0;
    }
  }
  if (lane == 0 && n > 0) hs->par[2 * n - 2] = -1;
  __syncwarp();
  // the lane's (up to) 8 leaves walk to the root side by side: one level of all eight per
  // iteration, so their dependent shared loads overlap
  if (tree_out) {
    uint32_t* lc32 = reinterpret_cast<uint32_t*>(hs->lc);
    int p[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) p[r] = lane + 32 * r < n ? hs->par[lane + 32 * r] : -1;
    for (;;) {
      bool any = false;
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (p[r] >= 0) {
          atomicAdd(&lc32[p[r] >> 1], 1u << (16 * (p[r] & 1)));
          p[r] = hs->par[p[r]];
          any = true;
        }
      if (!any) break;
    }
    __syncwarp();
  }
  if (hs->err) {
    __syncwarp();
    return;
  }
  int node[8], d[8];
  uint32_t code[8], toff[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    node[r] = lane + 32 * r < n ? lane + 32 * r : -1;
    d[r] = 0;
    code[r] = toff[r] = 0;
  }
  for (;;) {
    bool any = false;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (node[r] < 0) continue;
      const int p = hs->par[node[r]];
      if (p < 0) continue;
      if (hs->isr[node[r]]) {
        if (d[r] < 32) code[r] |= 1u << d[r];
        if (tree_out) toff[r] += 10u * hs->lc[hs->left[p]];
      } else {
        toff[r] += 1u;
      }
      ++d[r];
      node[r] = p;
      any = true;
    }
    if (!any) break;
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int t = lane + 32 * r;
    if (t >= n) continue;
    if (d[r] > 32) hs->err = WBPC_ERR_CODE_LENGTH;  // an internal node at depth >= 32 (entropy.py:97-98)
    const int s = hs->leafsym[t];
    code_len[s] = (uint8_t)min(d[r], 255);
    if (code_val) code_val[s] = code[r];
    if (tree_out) {
      const uint64_t v = (uint64_t)(0x100u | (uint32_t)s) << (64 - 9 - (toff[r] & 31));
      atomicOr(&tree_out[toff[r] >> 5], (uint32_t)(v >> 32));
      const uint32_t lo = (uint32_t)v;
      if (lo) atomicOr(&tree_out[(toff[r] >> 5) + 1], lo);
    }
  }
  __syncwarp();
}

// OR `nbits` (<= 57) bits of `value` MSB-first into big-endian word buffer at bit `pos`.
__device__ __forceinline__ void put_bits_smem(uint32_t* buf, uint32_t pos, uint64_t value, int nbits) {
  if (nbits <= 0) return;
  uint64_t v = value << (64 - nbits);  // MSB aligned
  uint32_t w = pos >> 5, sh = pos & 31;
  uint32_t w0 = (uint32_t)(v >> (32 + sh));
  uint64_t rest = v << (32 - sh);
  uint32_t w1 = (uint32_t)(rest >> 32);
  uint32_t w2 = (uint32_t)rest;
  if (w0) atomicOr(&buf[w], w0);
  if (w1) atomicOr(&buf[w + 1], w1);
  if (w2) atomicOr(&buf[w + 2], w2);
}

}  // namespace wb
