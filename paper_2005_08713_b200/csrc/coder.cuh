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
// Only the merge is serial (thread 0); code lengths/values and the preorder tree offsets are then
// computed by one thread per leaf walking to the root:
//   depth = #edges, code bit d = 1 if the d-th edge from the leaf is a right edge,
//   preorder offset = sum over edges of 1 (+ bits of the left sibling subtree = 10*lc - 1 on a
//   right edge)  (write_tree, entropy.py:259-269: internal '0', leaf '1' + 8 bits).
// Whole CTA calls this.  Outputs code_len/code_val (0xFF = absent) and, if tree_out != nullptr,
// the preorder tree bits (zeroed by the caller).  Returns the number of leaves.
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
    if (code_val) code_val[tid] = 0;
  }
  // rank = #keys below mine (keys are distinct): each warp bitonic-sorts its 32 keys with
  // shuffles into key[256 + 32 w ..]; a key's rank is the sum of its lower bounds in the 8 lists
  if (tid < 256) {
    const int lane = tid & 31;
    uint32_t v = mykey;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        const uint32_t o = __shfl_xor_sync(0xffffffffu, v, j);
        const bool up = (lane & k) == 0, lower = (lane & j) == 0;
        v = (lower == up) ? min(v, o) : max(v, o);
      }
    hs->key[256 + tid] = v;
  }
  const int n = __syncthreads_count(tid < 256 && mykey != 0xFFFFFFFFu);
  int rank = 0;
  if (tid < 256 && mykey != 0xFFFFFFFFu) {
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint32_t* L = hs->key + 256 + 32 * w;
      int lo = 0;  // lower bound: number of entries < mykey
#pragma unroll
      for (int step = 16; step > 0; step >>= 1)
        if (L[lo + step - 1] < mykey) lo += step;
      lo += L[lo] < mykey ? 1 : 0;
      rank += lo;
    }
  }
  __syncthreads();  // the sorted lists are read before key[0..n) is overwritten
  if (tid < 256 && mykey != 0xFFFFFFFFu) {
    hs->leafsym[rank] = (int16_t)tid;
    hs->key[rank] = mykey;  // ranks < n <= 256
    hs->lc[rank] = 1;
  }
  __syncthreads();
  // 2. serial two-queue merge (thread 0).  Each step takes the two smallest of the first two
  // sorted leaves (l0 < l1) and the first two internal nodes (q0 < q1) in one comparison network
  // -- two leaves, two internal nodes, or one of each (entropy.py:219-222: the internal node
  // only when strictly smaller; keys are distinct) -- and the four head refills for the next
  // step are loaded together while the new node is formed.  The serial step keeps only what
  // the merge itself needs (keys, children); parents, right-child flags and subtree leaf counts
  // are derived in parallel afterwards (the right child is parked in par[k] meanwhile).
  if (tid == 0) {
    hs->n = n;
    hs->err = n == 0 ? WBPC_ERR_EMPTY_ALPHABET : 0;  // entropy.py:210-211
    const uint32_t INF = 0xFFFFFFFFu;
    int i = 0, j = n;
    uint32_t l0 = n > 0 ? hs->key[0] : INF, l1 = n > 1 ? hs->key[1] : INF, q0 = INF, q1 = INF;
    for (int k = n; k < 2 * n - 1; ++k) {
      const bool two_leaves = l1 < q0;
      const bool two_nodes = !two_leaves && q1 < l0;
      const bool lf = l0 < q0;  // mixed case: the leaf is popped first
      const uint32_t ka = two_leaves ? l0 : (two_nodes ? q0 : (lf ? l0 : q0));
      const uint32_t kb = two_leaves ? l1 : (two_nodes ? q1 : (lf ? q0 : l0));
      const int a = two_leaves ? i : (two_nodes ? j : (lf ? i : j));
      const int b = two_leaves ? i + 1 : (two_nodes ? j + 1 : (lf ? j : i));
      i += two_leaves ? 2 : (two_nodes ? 0 : 1);
      j += two_nodes ? 2 : (two_leaves ? 0 : 1);
      // refills for the next step, issued together (indices clamped; invalid heads become INF)
      const uint32_t nl0 = hs->key[min(i, 511)], nl1 = hs->key[min(i + 1, 511)];
      const uint32_t nq0 = hs->key[min(j, 511)], nq1 = hs->key[min(j + 1, 511)];
      const uint32_t kk = ((ka & ~255u) + (kb & ~255u)) | min(ka & 255u, kb & 255u);
      hs->key[k] = kk;
      hs->left[k] = (int16_t)a;
      hs->par[k] = (int16_t)b;  // right child, until the parent pass below
      l0 = i < n ? nl0 : INF;
      l1 = i + 1 < n ? nl1 : INF;
      // internal queue [j, k]: node k was just formed (its smem entry is not in the refill)
      q0 = j < k ? nq0 : (j == k ? kk : INF);
      q1 = j + 1 < k ? nq1 : (j + 1 == k ? kk : INF);
    }
  }
  __syncthreads();
  {  // parents and right-child flags (every right child is read before any parent is written)
    const int nn = hs->n;
    int kc[2], ra[2], rb[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      kc[r] = nn + tid + r * (int)blockDim.x;
      ra[r] = rb[r] = -1;
      if (kc[r] < 2 * nn - 1) { ra[r] = hs->left[kc[r]]; rb[r] = hs->par[kc[r]]; }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 2; ++r)
      if (kc[r] < 2 * nn - 1) {
        hs->par[ra[r]] = (int16_t)kc[r];
        hs->par[rb[r]] = (int16_t)kc[r];
        hs->isr[ra[r]] = 0;
        hs->isr[rb[r]] = 1;
        hs->lc[kc[r]] = 0;
      }
    if (tid == 0 && nn > 0) hs->par[2 * nn - 2] = -1;
    __syncthreads();
    // subtree leaf counts (only the serialised tree needs them): every leaf adds 1 to each
    // ancestor (16-bit halves of 32-bit words; counts <= 256 never carry into the other half)
    if (tree_out) {
      if (tid < nn) {
        uint32_t* lc32 = reinterpret_cast<uint32_t*>(hs->lc);
        for (int p = hs->par[tid]; p >= 0; p = hs->par[p]) atomicAdd(&lc32[p >> 1], 1u << (16 * (p & 1)));
      }
      __syncthreads();
    }
  }
  // 3. per-leaf walk to the root: depth, code, preorder offset (parallel)
  if (tid < n && !hs->err) {
    int node = tid, d = 0;
    uint32_t code = 0, toff = 0;
    bool toolong = false;
    while (hs->par[node] >= 0) {
      const int p = hs->par[node];
      if (hs->isr[node]) {
        if (d < 32) code |= 1u << d;
        if (tree_out) toff += 10u * hs->lc[hs->left[p]];  // 1 + (10*lc - 1)
      } else {
        toff += 1u;
      }
      ++d;
      node = p;
    }
    if (d > 32) toolong = true;  // an internal node at depth >= 32 (entropy.py:97-98)
    if (toolong) hs->err = WBPC_ERR_CODE_LENGTH;
    const int s = hs->leafsym[tid];
    code_len[s] = (uint8_t)min(d, 255);
    if (code_val) code_val[s] = code;
    if (tree_out) {
      // leaf: '1' + 8-bit symbol at its preorder offset (internal nodes are '0' = untouched)
      const uint64_t v = (uint64_t)(0x100u | (uint32_t)s) << (64 - 9 - (toff & 31));
      atomicOr(&tree_out[toff >> 5], (uint32_t)(v >> 32));
      const uint32_t lo = (uint32_t)v;
      if (lo) atomicOr(&tree_out[(toff >> 5) + 1], lo);
    }
  }
  __syncthreads();
  return n;
}

// Warp version of huff_build (same algorithm, same outputs): one warp builds one block's code, so
// the serial merge of lane 0 costs only its own warp -- the other warps of the SM are other
// blocks' builds, and the merge latency of one overlaps the others'.  Lane l handles symbols
// l, l + 32, ... (eight bitonic-sorted lists of 32 keys); internal nodes and leaves are strided
// over the lanes likewise.
static __device__ int huff_build_warp(const int* freq, HuffScratch* hs, uint8_t* code_len, uint32_t* code_val,
                                      uint32_t* tree_out) {
  const int lane = threadIdx.x & 31;
  constexpr uint32_t FULLM = 0xffffffffu;
  uint32_t mykey[8];
  int n = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int s = 32 * i + lane;
    const int f = freq[s];
    const uint32_t key = f > 0 ? (((uint32_t)f << 8) | (uint32_t)s) : 0xFFFFFFFFu;
    mykey[i] = key;
    code_len[s] = 0xFF;
    if (code_val) code_val[s] = 0;
    uint32_t v = key;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        const uint32_t o = __shfl_xor_sync(FULLM, v, j);
        const bool up = (lane & k) == 0, lower = (lane & j) == 0;
        v = (lower == up) ? min(v, o) : max(v, o);
      }
    hs->key[256 + 32 * i + lane] = v;
    n += __popc(__ballot_sync(FULLM, key != 0xFFFFFFFFu));
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t key = mykey[i];
    if (key == 0xFFFFFFFFu) continue;
    int rank = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint32_t* L = hs->key + 256 + 32 * w;
      int lo = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1)
        if (L[lo + step - 1] < key) lo += step;
      lo += L[lo] < key ? 1 : 0;
      rank += lo;
    }
    hs->leafsym[rank] = (int16_t)(32 * i + lane);  // ranks < n <= 256: the lists stay intact
    hs->key[rank] = key;
    hs->lc[rank] = 1;
  }
  __syncwarp();
  if (lane == 0) {  // serial two-queue merge (see huff_build)
    hs->n = n;
    hs->err = n == 0 ? WBPC_ERR_EMPTY_ALPHABET : 0;
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
  __syncwarp();
  {
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
    if (tree_out) {
      uint32_t* lc32 = reinterpret_cast<uint32_t*>(hs->lc);
      for (int t = lane; t < n; t += 32)
        for (int p = hs->par[t]; p >= 0; p = hs->par[p]) atomicAdd(&lc32[p >> 1], 1u << (16 * (p & 1)));
      __syncwarp();
    }
  }
  const int err0 = hs->err;
  for (int t = lane; t < n && !err0; t += 32) {
    int node = t, d = 0;
    uint32_t code = 0, toff = 0;
    while (hs->par[node] >= 0) {
      const int p = hs->par[node];
      if (hs->isr[node]) {
        if (d < 32) code |= 1u << d;
        if (tree_out) toff += 10u * hs->lc[hs->left[p]];
      } else {
        toff += 1u;
      }
      ++d;
      node = p;
    }
    if (d > 32) hs->err = WBPC_ERR_CODE_LENGTH;
    const int s = hs->leafsym[t];
    code_len[s] = (uint8_t)min(d, 255);
    if (code_val) code_val[s] = code;
    if (tree_out) {
      const uint64_t v = (uint64_t)(0x100u | (uint32_t)s) << (64 - 9 - (toff & 31));
      atomicOr(&tree_out[toff >> 5], (uint32_t)(v >> 32));
      const uint32_t lo = (uint32_t)v;
      if (lo) atomicOr(&tree_out[(toff >> 5) + 1], lo);
    }
  }
  __syncwarp();
  return n;
}

// huff_build in three phases for many blocks per CTA: the two parallel phases run warp per block,
// the serial merge runs lane per block, so one warp instruction of the merge advances up to 32
// blocks' merges at once (the merge is instruction-issue bound when every block spends a warp on it).
// Phase A (warp): rank-sort the present symbols of `freq` into hs (keys, leaf symbols); returns n.
static __device__ int huff_rank_warp(const int* freq, HuffScratch* hs) {
  const int lane = threadIdx.x & 31;
  constexpr uint32_t FULLM = 0xffffffffu;
  uint32_t mykey[8];
  int n = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int s = 32 * i + lane;
    const int f = freq[s];
    const uint32_t key = f > 0 ? (((uint32_t)f << 8) | (uint32_t)s) : 0xFFFFFFFFu;
    mykey[i] = key;
    uint32_t v = key;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        const uint32_t o = __shfl_xor_sync(FULLM, v, j);
        const bool up = (lane & k) == 0, lower = (lane & j) == 0;
        v = (lower == up) ? min(v, o) : max(v, o);
      }
    hs->key[256 + 32 * i + lane] = v;
    n += __popc(__ballot_sync(FULLM, key != 0xFFFFFFFFu));
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t key = mykey[i];
    int rank = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint32_t* L = hs->key + 256 + 32 * w;
      int lo = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1)
        if (L[lo + step - 1] < key) lo += step;
      lo += L[lo] < key ? 1 : 0;
      rank += lo;
    }
    if (key != 0xFFFFFFFFu) {
      hs->leafsym[rank] = (int16_t)(32 * i + lane);  // ranks < n <= 256: the lists stay intact
      hs->key[rank] = key;
      hs->lc[rank] = 1;
    }
  }
  if (lane == 0) {
    hs->n = n;
    hs->err = n == 0 ? WBPC_ERR_EMPTY_ALPHABET : 0;  // entropy.py:210-211
  }
  __syncwarp();
  return n;
}

// Phase B (one thread per block): the serial two-queue merge of huff_build.
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
