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
  int16_t left[512], right[512];
  uint16_t size[512];    // serialized subtree bits
  uint16_t toff[512];    // preorder bit offset
  uint8_t depth[512];
  uint32_t code[512];
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
// Whole CTA calls this.  Outputs code_len/code_val (per symbol, 0xFF = absent) and, if tree_out
// != nullptr, the preorder tree bits (zeroed by the caller) + returns their count.
static __device__ int huff_build(const int* freq, HuffScratch* hs, uint8_t* code_len, uint32_t* code_val,
                          uint32_t* tree_out) {
  const int tid = threadIdx.x;
  // 1. rank-sort present symbols by key (parallel)
  uint32_t mykey = 0xFFFFFFFFu;
  if (tid < 256) {
    int f = freq[tid];
    if (f > 0) mykey = ((uint32_t)f << 8) | (uint32_t)tid;
    hs->key[256 + tid] = mykey;  // temp area
    code_len[tid] = 0xFF;
    code_val[tid] = 0;
  }
  int n = __syncthreads_count(tid < 256 && mykey != 0xFFFFFFFFu);
  if (tid < 256 && mykey != 0xFFFFFFFFu) {
    int rank = 0;
    for (int s = 0; s < 256; ++s) rank += hs->key[256 + s] < mykey;
    hs->leafsym[rank] = (int16_t)tid;
    hs->key[rank] = mykey;  // ranks < n <= 256, temp area starts at 256: no overlap
  }
  __syncthreads();
  // 2. serial two-queue merge (thread 0)
  if (tid == 0) {
    hs->n = n;
    hs->err = 0;
    for (int i = 0; i < n; ++i) { hs->size[i] = 9; hs->left[i] = -1; }
    int i = 0, j = n;
    uint32_t ki = n > 0 ? hs->key[0] : 0xFFFFFFFFu;
    for (int k = n; k < 2 * n - 1; ++k) {
      int a, b;
      uint32_t ka, kb;
      uint32_t kj = j < k ? hs->key[j] : 0xFFFFFFFFu;
      if (j < k && (i >= n || kj < ki)) { a = j++; ka = kj; }
      else { a = i++; ka = ki; ki = i < n ? hs->key[i] : 0xFFFFFFFFu; }
      kj = j < k ? hs->key[j] : 0xFFFFFFFFu;
      if (j < k && (i >= n || kj < ki)) { b = j++; kb = kj; }
      else { b = i++; kb = ki; ki = i < n ? hs->key[i] : 0xFFFFFFFFu; }
      hs->key[k] = ((ka & ~255u) + (kb & ~255u)) | min(ka & 255u, kb & 255u);
      hs->left[k] = (int16_t)a;
      hs->right[k] = (int16_t)b;
      hs->size[k] = (uint16_t)(1 + hs->size[a] + hs->size[b]);
    }
    // 3. downward pass: depth, code, preorder offsets (HuffmanCode._assign_codes, entropy.py:88-100)
    if (n == 0) hs->err = WBPC_ERR_EMPTY_ALPHABET;  // entropy.py:210-211
    int root = n > 0 ? 2 * n - 2 : 0;
    hs->depth[root] = 0;
    hs->code[root] = 0;
    hs->toff[root] = 0;
    for (int k = root; n > 0 && k >= n; --k) {
      int d = hs->depth[k];
      if (d >= 32) { hs->err = WBPC_ERR_CODE_LENGTH; break; }
      uint32_t c = hs->code[k];
      int a = hs->left[k], b = hs->right[k];
      hs->depth[a] = (uint8_t)(d + 1);
      hs->depth[b] = (uint8_t)(d + 1);
      hs->code[a] = c << 1;
      hs->code[b] = (c << 1) | 1u;
      hs->toff[a] = (uint16_t)(hs->toff[k] + 1);
      hs->toff[b] = (uint16_t)(hs->toff[k] + 1 + hs->size[a]);
    }
  }
  __syncthreads();
  // 4. per-leaf outputs (parallel)
  if (tid < n && !hs->err) {
    int s = hs->leafsym[tid];
    code_len[s] = hs->depth[tid];
    code_val[s] = hs->depth[tid] ? hs->code[tid] : 0u;
    if (tree_out) {
      // leaf: '1' + 8-bit symbol at its preorder offset (internal nodes are '0' = untouched)
      uint32_t pos = hs->toff[tid];
      uint64_t v = (uint64_t)(0x100u | (uint32_t)s) << (64 - 9 - (pos & 31));
      atomicOr(&tree_out[pos >> 5], (uint32_t)(v >> 32));
      uint32_t lo = (uint32_t)v;
      if (lo) atomicOr(&tree_out[(pos >> 5) + 1], lo);
    }
  }
  __syncthreads();
  return n;
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
