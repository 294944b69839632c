// encode.cu — per-128x128-block coefficient coder (sm_100a): bit-plane symbols, empty-plane
// masks, zero-run + deterministic Huffman planning, bit-exact block emission, container assembly.
//
// Replaces (reference /root/reference/pkg/src/wbpc):
//   CoefficientBlock.build depth            bitplanes.py:72-81
//   _smr_planes/_plane_symbols/_area_order  bitplanes.py:112-122,224-229,148-170
//   serialize_block, plane_slot_order       bitplanes.py:243-265
//   stored masks                            blocks.py:89-90
//   _plan_stream                            blocks.py:53-81
//   select_zr_symbol/_segment_runs          entropy.py:131-159
//   optimize_counter_width                  entropy.py:171-191
//   build_huffman (x2), write_tree          entropy.py:194-269
//   tokenize + pack_tokens                  entropy.py:324-421
//   encode_block writer                     blocks.py:84-120
//   encode_image index/header assembly      container.py:185-206
//
// Kernels (one CTA per block unless noted):
//   k_block_analyze  coefficients -> symbols (workspace) + stats + two Huffman builds + per-slot
//                    payload sizes (seek table) -> BlockMeta
//   k_offsets        single CTA: exclusive scan of block sizes -> container offsets (no host sync)
//   k_block_emit     header + tree + seek table + payload bits, written at the final offset,
//                    plus this block's index entry (and the container header for slot 0)
#include <atomic>
#include <climits>
#include <type_traits>

#include "coder.cuh"

namespace wb {

// Per-block statistics of the symbol pass (k_block_symbols -> k_block_huffman / k_block_sizes).
struct BlockStats {
  int hist[256];    // histogram of the kept stream (stored slots; bin 0 = their zero count)
  int chunks[15];   // sum over zero runs of ceil(L / (2^w - 1)), w = 2..16
  int sum_len, nruns, nstored, depth, zr;
  uint32_t stored[3];
  int pad[7];
};

struct SymSmem {
  int hist[256];
  int shortrun[33];              // zero runs of length 2..32 (chunk sums formed per length)
  uint8_t stored[WB_MAX_SLOTS];
  int order[WB_MAX_SLOTS];       // stored slot indices in serialization order
  int acc[20];                   // [0] sum run len, [1] #runs, [2..16] chunks(w), [17] zeros
  int misc[8];
  unsigned red[CT / 32];
};

struct AnalyzeParams {
  Geom g;
  int nblocks;
  const void* coef;       // int16 elements when g.coef16, else int32
  const unsigned* bmax;
  uint8_t* syms;          // symbol workspace, stride g.sym_stride_hp per block
  uint16_t* wbits;        // token bits per (stored slot, 32-symbol word), 64 * max_slots per block
  BlockMeta* meta;
  BlockStats* stats;
  uint32_t* zmask;        // zero-symbol masks, 64 words per slot row, max_slots rows per block
  uint32_t* sizes;
  DevStatus* st;
  int max_slots;          // zero-mask rows (3 x static depth bound)
};

// ceil(L / (2^w - 1)) for L <= 2048
static __device__ __forceinline__ int chunk_count(int L, int w) {
  int cap = (1 << w) - 1;
  return (L + cap - 1) / cap;
}
// Same without an integer division for 1 <= L <= 2048: floor((L-1)/cap) + 1 with the magic
// m = ceil(2^32 / cap) (chunk_magic; cap >= 2): (L-1) m / 2^32 exceeds (L-1)/cap by less than
// (L-1)/2^32 < 1/cap, so the high multiply is exact.
static __host__ __device__ __forceinline__ uint32_t chunk_magic(int cap) {
  return cap >= 2 ? (uint32_t)((0x100000000ull + (unsigned)cap - 1) / (unsigned)cap) : 0u;
}
static __device__ __forceinline__ int chunk_count_m(int L, uint32_t m) { return (int)__umulhi((uint32_t)(L - 1), m) + 1; }

__global__ void __launch_bounds__(CT, 8) k_block_symbols(AnalyzeParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SymSmem& S = *reinterpret_cast<SymSmem*>(smem_raw);
  // per-warp histograms of the symbol pass (no cross-warp contention); static shared memory so
  // the per-plane update addresses them with a constant base
  __shared__ int whist[CT / 32][256];
  // zero-symbol bitmask per slot (2048 bits), LSB = lower position; rows = 3 * static depth bound
  uint16_t (*zm)[128] = reinterpret_cast<uint16_t (*)[128]>(smem_raw + ((sizeof(SymSmem) + 15) & ~(size_t)15));
  const Geom& g = P.g;
  const int gid = blockIdx.x;
  const int b = fdiv(gid, g.md_spi);
  const int slot = gid - b * g.slots_per_image;
  const SlotInfo si = slot_info(g, slot);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned peak = P.bmax[gid];
  const int depth = 1 + (peak ? 32 - __clz(peak) : 0);  // bitplanes.py:77-79
  const int nsub = si.kind ? 3 : 1;
  const int nslots = nsub * depth;
  uint8_t* symbase = P.syms + (i64)gid * g.sym_stride_hp;
  if (depth > WB_MAX_DEPTH || (i64)nslots * WB_PP > g.sym_stride_hp || nslots > P.max_slots) {
    if (tid == 0) {
      record_error(P.st, WBPC_ERR_UNSUPPORTED, (u64)gid);
      P.stats[gid].nstored = 0;  // the later passes see an empty block
      P.stats[gid].depth = 1;
    }
    return;
  }
  for (int i = tid; i < 256; i += CT) S.hist[i] = 0;
  for (int i = tid; i < (CT / 32) * 256; i += CT) (&whist[0][0])[i] = 0;
  for (int i = tid; i < 33; i += CT) S.shortrun[i] = 0;
  for (int i = tid; i < WB_MAX_SLOTS; i += CT) S.stored[i] = 0;
  for (int i = tid; i < 20; i += CT) S.acc[i] = 0;
  __syncthreads();

  // ---- 1. symbols: lane per 4x2 area.  A warp takes 32 consecutive stream positions k of one
  //         subband (area row r = 2*(k>>6) + (k&1), col c = (k>>1)&31, bitplanes.py:159-166);
  //         each lane loads its 8 coefficients and forms every plane's symbol at once with 8x8
  //         bit transposes of the magnitudes (byte j of the transpose = bit j of the 8 values).
  //         Per plane: one coalesced 32-byte store, one ballot for the zero mask / stored flag.
  const LevelGeom& lg = g.lv[si.lev];
  const i64 cbase = (i64)b * g.img_stride + (i64)si.c * g.chan_stride;
  const int y0 = si.r * WB_DIM, x0 = si.col * WB_DIM;
  const int ngroups = nsub * (WB_PP / 32);
  uint32_t* zm32 = reinterpret_cast<uint32_t*>(zm);  // 64 words (2048 bits) per slot row
  // this warp's histogram as an opaque 32-bit shared address (kept in a register by the
  // 32-register symbol loop instead of being re-derived for every plane)
  uint32_t wh_s;
  asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(wh_s) : "l"(&whist[warp][0]));
  auto tr8 = [](uint64_t x) -> uint64_t {
    uint64_t t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull;
    x = x ^ t ^ (t << 7);
    t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull;
    x = x ^ t ^ (t << 14);
    t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull;
    return x ^ t ^ (t << 28);
  };
  // The group loop is instantiated per subband count so the plane stride of the symbol
  // workspace is a constant: every plane's store is an immediate offset from one base pointer.
  auto sym_groups = [&](auto nsub_c) {
  constexpr int NSUB = decltype(nsub_c)::value;
  constexpr int pstride = NSUB * WB_PP;  // bytes between planes of one subband in the symbol workspace
  for (int gi = warp; gi < NSUB * (WB_PP / 32); gi += CT / 32) {
    const int s = gi >> 6, g32 = gi & 63;
    const int k = 32 * g32 + lane;
    const int r = 2 * (k >> 6) + (k & 1), c = (k >> 1) & 31;
    const i64 pi = cbase + lg.off[si.kind ? 1 + s : 0] + (i64)(y0 + 2 * r) * lg.pw + x0 + 4 * c;
    // AREA_WEIGHTS (bitplanes.py:31): row 2r -> bits 0..3, row 2r+1 -> bits 4..7
    int v[8];
    if (g.coef16) {  // 4 int16 per row: one 8-byte load each
      const int16_t* p = reinterpret_cast<const int16_t*>(P.coef) + pi;
      const uint2 a = *reinterpret_cast<const uint2*>(p), bq = *reinterpret_cast<const uint2*>(p + lg.pw);
      v[0] = (int)(int16_t)(a.x & 0xFFFFu); v[1] = (int)(int16_t)(a.x >> 16);
      v[2] = (int)(int16_t)(a.y & 0xFFFFu); v[3] = (int)(int16_t)(a.y >> 16);
      v[4] = (int)(int16_t)(bq.x & 0xFFFFu); v[5] = (int)(int16_t)(bq.x >> 16);
      v[6] = (int)(int16_t)(bq.y & 0xFFFFu); v[7] = (int)(int16_t)(bq.y >> 16);
    } else {
      const int32_t* p = reinterpret_cast<const int32_t*>(P.coef) + pi;
      const int4 q0 = *reinterpret_cast<const int4*>(p);
      const int4 q1 = *reinterpret_cast<const int4*>(p + lg.pw);
      v[0] = q0.x; v[1] = q0.y; v[2] = q0.z; v[3] = q0.w;
      v[4] = q1.x; v[5] = q1.y; v[6] = q1.z; v[7] = q1.w;
    }
    unsigned sgn = 0;
    unsigned mg[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      sgn |= ((unsigned)v[i] >> 31) << i;
      mg[i] = (unsigned)abs(v[i]);
    }
    // lane p keeps plane p's non-zero ballot and writes its mask word / stored flag once below
    unsigned mynz = 0;
    int lane_o;  // opaque copy of the lane index (not re-read from the thread index per plane)
    asm volatile("mov.b32 %0, %1;" : "=r"(lane_o) : "r"(lane));
    uint8_t* const sp = symbase + s * WB_PP + k;  // plane pb of this position: sp[pb * pstride]
    auto emit = [&](int pb, uint8_t* dst, unsigned sym) {  // plane-major slot (bitplanes.py:243-246)
      *dst = (uint8_t)sym;
      const unsigned nzb = __ballot_sync(0xffffffffu, sym != 0);
      mynz = lane_o == pb ? nzb : mynz;
      // every symbol counts, zeros included (bin 0 is replaced by the zero count of the stored
      // slots before it is used); same-address increments are aggregated by the hardware
      asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(wh_s + 4u * sym) : "memory");
    };
    emit(0, sp, sgn);
    // magnitude plane pb (1..depth-1) = bit depth-1-pb; planes are visited top down, so the
    // destination walks down one plane stride per plane.  The byte transposes of the first two
    // 8-bit groups are formed up front (depth <= 17: every 8/9/10/12-bit image), so the
    // magnitudes are dead during the emission.
    uint8_t* const dtop = sp + (i64)(depth - 1) * pstride;  // plane 1 = magnitude bit depth-2
    auto group = [&](int q) {
      uint32_t b0 = 0, b1 = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        b0 |= ((mg[i] >> (8 * q)) & 0xFFu) << (8 * i);
        b1 |= ((mg[4 + i] >> (8 * q)) & 0xFFu) << (8 * i);
      }
      return tr8(((uint64_t)b1 << 32) | b0);
    };
    auto emit8 = [&](int q, uint64_t t) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int bit = 8 * q + j;
        if (bit <= depth - 2) emit(depth - 1 - bit, dtop - bit * pstride, (unsigned)(t >> (8 * j)) & 0xFFu);
      }
    };
    if (depth <= 17) {
      const uint64_t t0 = group(0);
      const uint64_t t1 = depth > 9 ? group(1) : 0ull;
      emit8(0, t0);
      if (depth > 9) emit8(1, t1);
    } else {
      for (int q = 0; 8 * q <= depth - 2; ++q) emit8(q, group(q));
    }
    if (lane < depth) {
      const int sl = lane * NSUB + s;
      zm32[sl * 64 + g32] = ~mynz;
      if (mynz) S.stored[sl] = 1;
    }
  }
  };
  if (nsub == 3) sym_groups(std::integral_constant<int, 3>{});
  else sym_groups(std::integral_constant<int, 1>{});
  __syncthreads();

  for (int i = tid; i < 256; i += CT) {
    int v = 0;
#pragma unroll
    for (int w = 0; w < CT / 32; ++w) v += whist[w][i];
    S.hist[i] = v;
  }
  // ---- 2. stored slots, zero runs (entropy.py:131-153) restricted to stored slots
  if (tid == 0) {
    int n = 0;
    for (int k = 0; k < nslots; ++k)
      if (S.stored[k]) S.order[n++] = k;
    S.misc[0] = n;
  }
  __syncthreads();
  const int nstored = S.misc[0];
  {
    // warp per stored slot row: lane l owns positions 64l .. 64l+63 of the row's 2048-bit zero
    // mask; run ends come from the lane's own non-zero bits or, past its segment, from the first
    // non-zero position of the lanes above (suffix-min scan), so every run costs O(1) whatever
    // its length (runs never cross a slot, entropy.py:131-153)
    int acc_len = 0, acc_runs = 0, acc_zero = 0, nlong = 0;
    int acc_ch[10];  // ceil(L / (2^w - 1)) for w = 2..11; w >= 12 gives one chunk per long run
    for (int i = 0; i < 10; ++i) acc_ch[i] = 0;
    for (int j = warp; j < nstored; j += CT / 32) {
      const uint32_t* zr32 = zm32 + S.order[j] * 64;
      const uint64_t z = (uint64_t)zr32[2 * lane] | ((uint64_t)zr32[2 * lane + 1] << 32);  // bit i: zero
      acc_zero += __popcll(z);
      const uint64_t nz = ~z;
      const uint64_t prevbit = (uint64_t)(__shfl_up_sync(0xffffffffu, (unsigned)(z >> 63), 1) & (lane ? 1u : 0u));
      const uint64_t nextbit = (uint64_t)(__shfl_down_sync(0xffffffffu, (unsigned)(z & 1ull), 1) & (lane < 31 ? 1u : 0u));
      const uint64_t zprev = (z << 1) | prevbit;
      const uint64_t znext = (z >> 1) | (nextbit << 63);
      uint64_t starts = z & (zprev | znext) & ~zprev;  // first positions of runs of length >= 2
      int v = nz ? 64 * lane + __ffsll((long long)nz) - 1 : WB_PP;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_down_sync(0xffffffffu, v, o);
        if (lane + o < 32) v = min(v, t);
      }
      const int nxt = __shfl_down_sync(0xffffffffu, v, 1);
      const int after = lane < 31 ? nxt : WB_PP;  // first non-zero position in lanes > lane
      while (starts) {
        const int i = __ffsll((long long)starts) - 1;
        starts &= starts - 1;
        const uint64_t m = nz & (~0ull << i);
        const int end = m ? 64 * lane + __ffsll((long long)m) - 1 : after;
        const int L = end - (64 * lane + i);
        acc_len += L;
        acc_runs += 1;
        if (L <= 32) {
          atomicAdd(&S.shortrun[L], 1);
        } else {
          // a float estimate corrected exactly; a run never exceeds 2048 symbols
#pragma unroll
          for (int ww = 2; ww <= 11; ++ww) acc_ch[ww - 2] += chunk_count_m(L, chunk_magic((1 << ww) - 1));
          ++nlong;
        }
      }
    }
    // reduce
    for (int o = 16; o > 0; o >>= 1) {
      acc_len += __shfl_xor_sync(0xffffffffu, acc_len, o);
      acc_runs += __shfl_xor_sync(0xffffffffu, acc_runs, o);
      acc_zero += __shfl_xor_sync(0xffffffffu, acc_zero, o);
      nlong += __shfl_xor_sync(0xffffffffu, nlong, o);
#pragma unroll
      for (int i = 0; i < 10; ++i) acc_ch[i] += __shfl_xor_sync(0xffffffffu, acc_ch[i], o);
    }
    if (lane == 0) {
      atomicAdd(&S.acc[0], acc_len);
      atomicAdd(&S.acc[1], acc_runs);
      atomicAdd(&S.acc[17], acc_zero);
      for (int i = 0; i < 10; ++i) atomicAdd(&S.acc[2 + i], acc_ch[i]);
      for (int i = 10; i < 15; ++i) atomicAdd(&S.acc[2 + i], nlong);
    }
  }
  __syncthreads();
  // chunk sums of the short runs: thread (w, L) adds count[L] * ceil(L / (2^w - 1))
  for (int it = tid; it < 15 * 31; it += CT) {
    const int ww = 2 + it / 31, L = 2 + it % 31;
    const int c = S.shortrun[L];
    if (c) atomicAdd(&S.acc[ww], c * chunk_count(L, ww));
  }
  __syncthreads();

  int zr = 0;
  if (nstored) {
    // hist over the kept stream (blocks.py:93): nonzero symbols only come from stored slots
    if (tid == 0) S.hist[0] = S.acc[17];
    __syncthreads();
    // select_zr_symbol (entropy.py:156-159): argmin, ties -> smallest symbol
    {
      unsigned key = 0xFFFFFFFFu;
      if (tid < 256) key = ((unsigned)S.hist[tid] << 8) | (unsigned)tid;
      for (int o = 16; o > 0; o >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, o));
      if (lane == 0) S.red[warp] = key;
      __syncthreads();
      if (tid == 0) {
        unsigned k = 0xFFFFFFFFu;
        for (int w = 0; w < CT / 32; ++w) k = min(k, S.red[w]);
        S.misc[1] = (int)(k & 255u);
      }
      __syncthreads();
      zr = S.misc[1];
    }
  }
  // ---- stats + zero masks of the stored slots to global for the Huffman / size kernels
  BlockStats* T = P.stats + gid;
  for (int i = tid; i < 256; i += CT) T->hist[i] = S.hist[i];
  if (tid < 15) T->chunks[tid] = S.acc[2 + tid];
  if (tid == 0) {
    T->sum_len = S.acc[0];
    T->nruns = S.acc[1];
    T->nstored = nstored;
    T->depth = depth;
    T->zr = zr;
    uint32_t st3[3] = {0, 0, 0};
    for (int k = 0; k < nslots; ++k)
      if (S.stored[k]) st3[k >> 5] |= 1u << (k & 31);
    T->stored[0] = st3[0];
    T->stored[1] = st3[1];
    T->stored[2] = st3[2];
  }
  uint32_t* zg = P.zmask + (i64)gid * P.max_slots * 64;
  for (int it = tid; it < nstored * 64; it += CT) {
    const int j = it >> 6, w = it & 63;
    zg[j * 64 + w] = zm32[S.order[j] * 64 + w];  // row j = j-th stored slot
  }
}

// K_h: both Huffman builds of a block (blocks.py:53-81: provisional code -> counter width ->
// final code on the token frequencies, entropy.py:171-248) and the preorder tree bits
// (entropy.py:259-269), HB blocks per CTA.  The rank sort and the code assignment run warp per
// block; the serial two-queue merge runs lane per block, so one warp instruction advances HB
// merges at once (per block the merge is ~500 dependent steps; issued once per block it would
// dominate the kernel's instruction count).
constexpr int HB = 14;      // blocks per Huffman CTA (2 CTAs of ~102 KB smem per SM)
constexpr int HWARPS = 8;   // warps per Huffman CTA
struct HuffBlockSmem {
  HuffScratch hs;
  uint8_t code_len[256];
  uint32_t tree[80];
  int width;
};

size_t huffman_smem_bytes() { return HB * sizeof(HuffBlockSmem) + HWARPS * 256 * sizeof(int); }

__global__ void __launch_bounds__(HWARPS * 32, 2) k_block_huffman(AnalyzeParams P) {
  extern __shared__ __align__(16) unsigned char hsm[];
  HuffBlockSmem* HBS = reinterpret_cast<HuffBlockSmem*>(hsm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* freq = reinterpret_cast<int*>(hsm + HB * sizeof(HuffBlockSmem)) + 256 * warp;
  const int g0 = blockIdx.x * HB;
  const int nb = min(HB, P.nblocks - g0);
  // ---- provisional code (blocks.py:67-75): [0] -= zeros in runs, [zr] += #runs
  for (int bi = warp; bi < nb; bi += HWARPS) {
    const BlockStats* T = P.stats + g0 + bi;
    HuffBlockSmem& H = HBS[bi];
    if (T->nstored && T->nruns > 0) {
      const int sum_len = T->sum_len, nruns = T->nruns, zr = T->zr;
      for (int i = lane; i < 256; i += 32) freq[i] = T->hist[i] - (i == 0 ? sum_len : 0) + (i == zr ? nruns : 0);
      __syncwarp();
      huff_rank_warp(freq, &H.hs);
    } else if (lane == 0) {
      H.hs.n = 0;
      H.hs.err = 0;
    }
    if (lane == 0) H.width = 2;
  }
  __syncthreads();
  if (threadIdx.x < nb) huff_merge_thread(&HBS[threadIdx.x].hs);
  __syncthreads();
  for (int bi = warp; bi < nb; bi += HWARPS) {
    const BlockStats* T = P.stats + g0 + bi;
    HuffBlockSmem& H = HBS[bi];
    if (T->nstored && T->nruns > 0) {
      huff_codes_warp(&H.hs, H.code_len, nullptr, nullptr);  // only len(code[zr]) is used
      if (lane == 0 && H.hs.err) record_error(P.st, H.hs.err, (u64)(g0 + bi));
      // optimize_counter_width (entropy.py:171-191): argmin over w = 2..16, ties -> smaller w
      const int zb = H.code_len[T->zr];
      unsigned long long key = ~0ull;
      if (lane < 15) key = ((unsigned long long)((long long)T->chunks[lane] * (lane + 2 + zb)) << 8) | (unsigned)(lane + 2);
      for (int o = 16; o > 0; o >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, o));
      if (lane == 0) H.width = (int)(key & 255u);
    }
  }
  __syncthreads();
  // ---- final code on the token frequencies (blocks.py:79-80; entropy.py:381-382)
  for (int bi = warp; bi < nb; bi += HWARPS) {
    const BlockStats* T = P.stats + g0 + bi;
    HuffBlockSmem& H = HBS[bi];
    if (T->nstored) {
      const int sum_len = T->sum_len, zr = T->zr;
      const int nch = T->nruns > 0 ? T->chunks[H.width - 2] : 0;
      for (int i = lane; i < 256; i += 32) freq[i] = T->hist[i] - (i == 0 ? sum_len : 0) + (i == zr ? nch : 0);
      for (int i = lane; i < 80; i += 32) H.tree[i] = 0;
      __syncwarp();
      huff_rank_warp(freq, &H.hs);
    } else if (lane == 0) {
      H.hs.n = 0;
      H.hs.err = 0;
    }
  }
  __syncthreads();
  if (threadIdx.x < nb) huff_merge_thread(&HBS[threadIdx.x].hs);
  __syncthreads();
  for (int bi = warp; bi < nb; bi += HWARPS) {
    const int gid = g0 + bi;
    const BlockStats* T = P.stats + gid;
    BlockMeta* M = P.meta + gid;
    HuffBlockSmem& H = HBS[bi];
    const int nstored = T->nstored;
    if (nstored) {
      huff_codes_warp(&H.hs, H.code_len, M->code_val, H.tree);  // code values straight to the block meta
      if (lane == 0 && H.hs.err) record_error(P.st, H.hs.err, (u64)gid);
      for (int i = lane; i < 256; i += 32) M->code_len[i] = H.code_len[i];
      for (int i = lane; i < 80; i += 32) M->tree_words[i] = H.tree[i];
    }
    if (lane == 0) {
      M->tree_bits = nstored ? 10u * (uint32_t)H.hs.n - 1 : 0u;  // preorder bits: (n-1) '0' + n * 9
      M->w = (uint8_t)H.width;
      M->zr = (uint8_t)T->zr;
    }
  }
}

// K_s: per-slot payload bits (tokenize + pack_tokens sizes, entropy.py:324-421) and their per-word
// counts for emit, the seek table and the block's header geometry (blocks.py:104-120); CTA per block.
struct SizeSmem {
  uint8_t code_len[256];
  int slot_bits[WB_MAX_SLOTS];
  int order[WB_MAX_SLOTS];  // stored slot indices in serialization order
};

__global__ void __launch_bounds__(CT, 6) k_block_sizes(AnalyzeParams P) {
  __shared__ SizeSmem S;
  extern __shared__ __align__(16) uint32_t zsm[];  // zero masks of the stored slots, 64 words each
  const Geom& g = P.g;
  const int gid = blockIdx.x;
  const int b = fdiv(gid, g.md_spi);
  const int slot = gid - b * g.slots_per_image;
  const SlotInfo si = slot_info(g, slot);
  const int tid = threadIdx.x;
  const BlockStats* T = P.stats + gid;
  BlockMeta* M = P.meta + gid;
  const int nsub = si.kind ? 3 : 1;
  const int depth = T->depth, nstored = T->nstored;
  const int nslots = nsub * depth;
  if (nstored) {
    // token bits of an ordinary symbol: its code length, plus the zero counter for a literal zr
    // (entropy.py:346); absent symbols never occur outside runs
    const int zr0 = M->zr, w0 = M->w;
    for (int i = tid; i < 256; i += CT) {
      const uint32_t cl = M->code_len[i];
      S.code_len[i] = (uint8_t)(cl == 0xFFu ? 0u : cl + (i == zr0 ? (uint32_t)w0 : 0u));
    }
    for (int i = tid; i < nstored; i += CT) S.slot_bits[i] = 0;
    const uint4* zg = reinterpret_cast<const uint4*>(P.zmask + (i64)gid * P.max_slots * 64);
    for (int i = tid; i < nstored * 16; i += CT) reinterpret_cast<uint4*>(zsm)[i] = zg[i];
    if (tid == 0) {
      int n = 0;
      for (int k = 0; k < nslots; ++k)
        if ((T->stored[k >> 5] >> (k & 31)) & 1u) S.order[n++] = k;
    }
  }
  __syncthreads();
  const uint32_t st0 = T->stored[0], st1 = T->stored[1], st2 = T->stored[2];
  if (nstored) {
    const int zr = M->zr, width = M->w;
    const uint8_t* symbase = P.syms + (i64)gid * g.sym_stride_hp;
    const int lzr = S.code_len[zr] - width;  // the zr code alone
    const int capw = (1 << width) - 1;
    const uint32_t mcap = chunk_magic(capw);
    // warp per stored slot row, lane l = words 2l, 2l+1 (positions 64l .. 64l+63); a run's
    // chunks count in the word where it starts, its end comes from the lane's own non-zero bits
    // or the first non-zero position of the lanes above (suffix-min scan)
    const int lane = tid & 31, warp = tid >> 5;
    for (int j = warp; j < nstored; j += CT / 32) {
      const int sl = S.order[j];
      const uint32_t* zm32 = zsm + j * 64;
      const uint64_t z = (uint64_t)zm32[2 * lane] | ((uint64_t)zm32[2 * lane + 1] << 32);
      const uint64_t nz = ~z;
      const uint64_t prevbit = (uint64_t)(__shfl_up_sync(0xffffffffu, (unsigned)(z >> 63), 1) & (lane ? 1u : 0u));
      const uint64_t nextbit = (uint64_t)(__shfl_down_sync(0xffffffffu, (unsigned)(z & 1ull), 1) & (lane < 31 ? 1u : 0u));
      const uint64_t zprev = (z << 1) | prevbit;
      const uint64_t znext = (z >> 1) | (nextbit << 63);
      const uint64_t inrun = z & (zprev | znext);
      uint64_t starts = inrun & ~zprev;
      int v = nz ? 64 * lane + __ffsll((long long)nz) - 1 : WB_PP;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_down_sync(0xffffffffu, v, o);
        if (lane + o < 32) v = min(v, t);
      }
      const int nxt = __shfl_down_sync(0xffffffffu, v, 1);
      const int after = lane < 31 ? nxt : WB_PP;
      const uint4* sp = reinterpret_cast<const uint4*>(symbase + (i64)sl * WB_PP + 64 * lane);
      int bits[2];  // (indexed with constants only: stays in registers)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint4 q0 = sp[2 * h], q1 = sp[2 * h + 1];
        const unsigned wd[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
        const uint32_t ir = (uint32_t)(inrun >> (32 * h));
        int b2 = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const unsigned sym = (wd[i >> 2] >> (8 * (i & 3))) & 0xFFu;
          b2 += ((ir >> i) & 1u) ? 0 : (int)S.code_len[sym];
        }
        bits[h] = b2;
      }
      while (starts) {
        const int i = __ffsll((long long)starts) - 1;
        starts &= starts - 1;
        const uint64_t m = nz & (~0ull << i);
        const int end = m ? 64 * lane + __ffsll((long long)m) - 1 : after;
        const int L = end - (64 * lane + i);
        const int cb = chunk_count_m(L, mcap) * (lzr + width);
        bits[0] += i < 32 ? cb : 0;
        bits[1] += i < 32 ? 0 : cb;
      }
      *reinterpret_cast<uint32_t*>(P.wbits + ((i64)gid * P.max_slots + j) * 64 + 2 * lane) =
          (uint32_t)(bits[0] & 0xFFFF) | ((uint32_t)bits[1] << 16);
      int tot = bits[0] + bits[1];
      for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
      if (lane == 0) S.slot_bits[j] = tot;
    }
    __syncthreads();
  }
  // ---- header geometry + seek table (blocks.py:104-120)
  if (tid == 0) {
    const int t = seek_bits(nsub, depth);
    const uint32_t tb = nstored ? M->tree_bits : 0u;
    int hdr = 6 + 5 + 8 + nsub * depth + (int)tb + 16 + nstored * t;
    uint32_t acc = 0;
    for (int j = 0; j < nstored; ++j) {
      if (t < 32 && (acc >> t) != 0) record_error(P.st, WBPC_ERR_DOMAIN, (u64)gid);  // bitio.py:30-31
      M->seek[j] = acc;
      acc += (uint32_t)S.slot_bits[j];
    }
    M->hdr_bits = (uint32_t)hdr;
    M->payload_bits = acc;
    M->bytes = (uint32_t)(((u64)hdr + acc + 7) >> 3);
    P.sizes[gid] = M->bytes;
    M->depth = (uint16_t)depth;
    M->nstored = (uint16_t)nstored;
    M->kind = (uint8_t)si.kind;
    M->nsub = (uint8_t)nsub;
    M->stored[0] = st0;
    M->stored[1] = st1;
    M->stored[2] = st2;
  }
}

// ---- container offsets: one CTA, exclusive scan over (image header + index) + block bytes ----
struct OffsetsParams {
  int nblocks, spi, batch;
  int raw;                // block API: no container header / index
  const uint32_t* sizes;  // byte length of every block
  u64* block_off;     // absolute byte offset of each block in the output buffer
  u64* img_off;       // [batch + 1] image start offsets, [batch] = total
  u64 cap;
  DevStatus* st;
  uint32_t* outw;     // encode: clear each block's first and last output word (shared with the
                      // neighbouring block / index and OR-ed by k_block_emit); null otherwise
};

static __device__ __forceinline__ u64 block_scan_u64(u64 v, u64* red) {
  // inclusive scan over CT threads
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    u64 t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    u64 x = lane < (int)(blockDim.x >> 5) ? red[lane] : 0ull;
    for (int o = 1; o < 32; o <<= 1) {
      u64 t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    red[lane] = x;
  }
  __syncthreads();
  if (warp) v += red[warp - 1];
  return v;
}

__global__ void __launch_bounds__(1024) k_offsets(OffsetsParams P) {
  __shared__ u64 red[32];
  __shared__ u64 carry;
  const u64 hdr = P.raw ? 0ull : 19 + 12ull * (u64)P.spi;  // container.py:58-59,202
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  constexpr int PER = 4;
  for (int base = 0; base < P.nblocks; base += 1024 * PER) {
    u64 v[PER], tot = 0;
    for (int k = 0; k < PER; ++k) {
      int gidx = base + threadIdx.x * PER + k;
      u64 x = 0;
      if (gidx < P.nblocks) {
        x = P.sizes[gidx];
        if (gidx % P.spi == 0) x += hdr;
      }
      v[k] = x;
      tot += x;
    }
    u64 incl = block_scan_u64(tot, red);
    u64 excl = carry + incl - tot;
    for (int k = 0; k < PER; ++k) {
      int gidx = base + threadIdx.x * PER + k;
      if (gidx < P.nblocks) {
        bool first = gidx % P.spi == 0;
        if (first) P.img_off[gidx / P.spi] = excl;
        const u64 bo = excl + (first ? hdr : 0);
        P.block_off[gidx] = bo;
        const u64 nbl = P.sizes[gidx];
        if (P.outw && nbl && bo + nbl <= P.cap) {
          P.outw[bo >> 2] = 0u;
          P.outw[(bo + nbl - 1) >> 2] = 0u;
        }
      }
      excl += v[k];
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    P.img_off[P.batch] = carry;
    P.st->total = carry;
    if (carry > P.cap) {
      P.st->aux = carry;
      record_error(P.st, WBPC_ERR_OUT_CAPACITY, 0, 2);
    }
  }
}

// ---- emit -------------------------------------------------------------------------------------
// Warp per stored slot: the slot's bit range in the block is known from the seek table, so slots
// are emitted independently.  Lane l owns symbols [64l, 64l+64): zero runs are found from the
// 2048-bit zero mask (neighbour bits and the next non-zero position come by shuffles), token bit
// costs are prefix-summed across the warp, and codewords/counters are OR-ed into a per-warp smem
// window aligned to the container's 32-bit word grid.  Full words are stored directly; partial
// words (shared with the neighbouring slot / header / block) are atomicOr-ed into the output:
// k_offsets clears each block's first and last word, the emitting CTA its internal shared words.
constexpr int EW = 8;        // warps per emit CTA
constexpr int CAPW = 768;    // window words per warp

struct EmitParams {
  Geom g;
  const uint8_t* syms;
  const uint16_t* wbits;  // analyze's token bits per (stored slot, 32-symbol word)
  int max_slots;
  const BlockMeta* meta;
  const u64* block_off;
  const u64* img_off;
  uint8_t* out;
  u64 cap;
  DevStatus* st;
};

struct EmitSmem {
  uint32_t win[EW][CAPW];
  uint8_t sym[EW][WB_PP];
  uint8_t code_len[256];
  uint32_t code_val[256];
  uint2 tok[256];          // x: codeword (with the literal-zr zero counter appended for zr);
                           // y: its length (may exceed 32 only for zr) -- one 8-byte load
  int order[WB_MAX_SLOTS];
};

__device__ __forceinline__ void store_word_bytes(uint8_t* dst, uint32_t w, int nbytes) {
  for (int i = 0; i < nbytes; ++i) dst[i] = (uint8_t)(w >> (24 - 8 * i));
}

// OR `nbits` (<= 57) bits of `value` at window bit `pos` (may be < 0 or past the window: clipped).
__device__ __forceinline__ void put_bits_clip(uint32_t* win, long long pos, uint64_t value, int nbits, int capw) {
  if (nbits <= 0) return;
  long long w = pos >> 5;  // floor
  const int sh = (int)(pos & 31);
  const uint64_t v = value << (64 - nbits);
  const uint32_t w0 = (uint32_t)(v >> (32 + sh));
  const uint64_t rest = v << (32 - sh);
  const uint32_t w1 = (uint32_t)(rest >> 32), w2 = (uint32_t)rest;
  if (w0 && w >= 0 && w < capw) atomicOr(&win[w], w0);
  if (w1 && w + 1 >= 0 && w + 1 < capw) atomicOr(&win[w + 1], w1);
  if (w2 && w + 2 >= 0 && w + 2 < capw) atomicOr(&win[w + 2], w2);
}

// Flush window words [0, nw) to the output word grid starting at global word gw0.
__device__ __forceinline__ void flush_window(uint32_t* outw, u64 gw0, const uint32_t* win, int nw, bool first_partial,
                                             bool last_partial) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < nw; i += 32) {
    const uint32_t v = bswap32(win[i]);
    const bool partial = (i == 0 && first_partial) || (i == nw - 1 && last_partial);
    if (partial) { if (v) atomicOr(&outw[gw0 + i], v); }
    else outw[gw0 + i] = v;
  }
}

__global__ void __launch_bounds__(EW * 32, 5) k_block_emit(EmitParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  EmitSmem& S = *reinterpret_cast<EmitSmem*>(smem_raw);
  const Geom& g = P.g;
  const int gid = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const BlockMeta* M = P.meta + gid;
  const u64 O = P.block_off[gid];
  const uint32_t nbytes = M->bytes;
  if (O + nbytes > P.cap) return;
  const int b = fdiv(gid, g.md_spi);
  const int slot = gid - b * g.slots_per_image;
  const u64 img0 = P.img_off[b];
  uint32_t* outw = reinterpret_cast<uint32_t*>(P.out);
  // index entry (container.py:202-205) and, for slot 0, the container header (:76-87)
  if (tid == 0 && g.raw_kind < 0) {
    uint8_t* ie = P.out + img0 + 19 + 12ull * slot;
    const u64 rel = O - img0;
    for (int i = 0; i < 8; ++i) ie[i] = (uint8_t)(rel >> (8 * i));
    for (int i = 0; i < 4; ++i) ie[8 + i] = (uint8_t)(nbytes >> (8 * i));
    if (slot == 0) {
      uint8_t* h = P.out + img0;
      h[0] = 'W'; h[1] = 'B'; h[2] = 'P'; h[3] = 'C'; h[4] = 1;
      for (int i = 0; i < 4; ++i) { h[5 + i] = (uint8_t)((unsigned)g.W >> (8 * i)); h[9 + i] = (uint8_t)((unsigned)g.H >> (8 * i)); }
      h[13] = (uint8_t)g.C; h[14] = (uint8_t)g.bd; h[15] = (uint8_t)(g.rct ? 1 : 0); h[16] = (uint8_t)g.L;
      h[17] = WB_DIM & 255; h[18] = WB_DIM >> 8;
    }
  }
  const int depth = M->depth, nsub = M->nsub, nstored = M->nstored, width = M->w, zr = M->zr;
  const int nslots = depth * nsub;
  if (tid < 256) {
    const uint32_t cl = M->code_len[tid], cv = M->code_val[tid];
    S.code_len[tid] = (uint8_t)cl;
    S.code_val[tid] = cv;
    const bool zrs = tid == M->zr;  // literal escape: zero counter after the zr code (entropy.py:346)
    const uint32_t tl = (cl == 0xFF ? 0u : cl) + (zrs ? M->w : 0u);
    S.tok[tid] = make_uint2(zrs ? (tl <= 32 ? cv << M->w : cv) : cv, cl == 0xFF ? 0u : (tl > 255u ? 255u : tl));
  }
  if (tid == 0) {
    int n = 0;
    for (int k = 0; k < nslots; ++k)
      if ((M->stored[k >> 5] >> (k & 31)) & 1u) S.order[n++] = k;
  }
  const u64 gb = 8ull * O;           // global bit of the block start
  const uint32_t hdr_bits = M->hdr_bits;
  {  // output words OR-ed by two of this block's windows (header end, slot starts) start at zero;
     // the block's first / last word were cleared by k_offsets (shared with other blocks)
    const u64 fw = gb >> 5, lw = (gb + 8ull * nbytes - 1) >> 5;
    for (int j = tid; j < (nstored > 0 ? nstored : 1); j += EW * 32) {
      u64 w;
      bool part;
      if (j == 0) {  // the header window's last word is always OR-ed
        w = (gb + hdr_bits - 1) >> 5;
        part = true;
      } else {       // slot j's first word, when it does not start on a word boundary
        const u64 bit = gb + hdr_bits + M->seek[j];
        w = bit >> 5;
        part = (bit & 31) != 0;
      }
      if (part && w > fw && w < lw) outw[w] = 0u;
    }
  }
  __syncthreads();
  // ---- header (warp 0): depth, cw, zr, masks, tree, count, seek table (blocks.py:104-118)
  if (warp == 0) {
    uint32_t* win = S.win[0];
    const int sh = (int)(gb & 31);
    const int nw = (int)((sh + hdr_bits + 31) >> 5);
    for (int i = lane; i < nw + 1; i += 32) win[i] = 0;
    __syncwarp();
    if (lane == 0) {
      put_bits_smem(win, sh + 0, (u64)depth, 6);
      put_bits_smem(win, sh + 6, (u64)width, 5);
      put_bits_smem(win, sh + 11, (u64)zr, 8);
    }
    for (int i = lane; i < nslots; i += 32) {  // masks: for s: for b: stored[b*nsub+s]
      const int s = i / depth, pb = i - s * depth;
      const int k = pb * nsub + s;
      if ((M->stored[k >> 5] >> (k & 31)) & 1u) put_bits_smem(win, sh + 19 + i, 1, 1);
    }
    uint32_t pos = sh + 19 + nslots;
    if (nstored) {
      const int tb = M->tree_bits;
      for (int i = lane; i < (tb + 31) / 32; i += 32) {
        const uint32_t wv = M->tree_words[i];
        const int nb = min(32, tb - 32 * i);
        put_bits_smem(win, pos + 32 * i, (u64)(wv >> (32 - nb)), nb);
      }
      pos += tb;
    }
    if (lane == 0) put_bits_smem(win, pos, (u64)nstored, 16);
    pos += 16;
    const int t = seek_bits(nsub, depth);
    for (int j = lane; j < nstored; j += 32) put_bits_smem(win, pos + j * t, (u64)M->seek[j], t);
    __syncwarp();
    // first word shared with the previous block / index, last word with slot 0 (or the next block)
    flush_window(outw, gb >> 5, win, nw, true, true);
    __syncwarp();
  }
  // ---- payload: warp per stored slot
  const uint8_t* symbase = P.syms + (i64)gid * g.sym_stride_hp;
  const int lzr = nstored ? S.code_len[zr] : 0;
  const uint32_t czr = nstored ? S.code_val[zr] : 0;
  const int cap = (1 << width) - 1;
  const uint32_t mcap = chunk_magic(cap);
  uint8_t* ssym = S.sym[warp];
  uint32_t* win = S.win[warp];
  // Each lane reads only its own 64 staged symbols (zero mask, token scan), so it copies exactly
  // those with cp.async and requests the next slot's as soon as it has finished with the current
  // one: the staging latency overlaps the window flush and the next slot's prologue.
  const uint32_t seg_s = (uint32_t)__cvta_generic_to_shared(ssym + 64 * lane);
  auto stage = [&](int jj) {
    const uint8_t* src = symbase + (i64)S.order[jj] * WB_PP + 64 * lane;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(seg_s + 16 * q), "l"(src + 16 * q) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int j0 = (warp + 1) % EW;
  if (j0 < nstored) stage(j0);
  for (int j = j0; j < nstored; j += EW) {
    const uint32_t sbeg = M->seek[j];
    const uint32_t send = j + 1 < nstored ? M->seek[j + 1] : M->payload_bits;
    const u64 g0 = gb + hdr_bits + sbeg;  // global bit of this slot's first token
    asm volatile("cp.async.wait_all;" ::: "memory");  // this lane's 64 symbols of slot j
    const uint8_t* my = ssym + 64 * lane;
    uint64_t z = 0;  // bit i: symbol 64*lane+i is zero
#pragma unroll
    for (int i = 0; i < 64; i += 16) {
      const uint4 q = *reinterpret_cast<const uint4*>(my + i);
      const uint32_t ww[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        z |= (uint64_t)((((__vcmpeq4(ww[k], 0u) & 0x08040201u) * 0x01010101u) >> 24)) << (i + 4 * k);
    }
    const uint64_t prevbit = (uint64_t)(__shfl_up_sync(0xffffffffu, (unsigned)(z >> 63), 1) & (lane ? 1u : 0u));
    const uint64_t nextbit = (uint64_t)(__shfl_down_sync(0xffffffffu, (unsigned)(z & 1ull), 1) & (lane < 31 ? 1u : 0u));
    const uint64_t zprev = (z << 1) | prevbit;
    const uint64_t znext = (z >> 1) | (nextbit << 63);
    const uint64_t inrun = z & (zprev | znext);
    const uint64_t starts = inrun & ~zprev;
    const uint64_t nz = ~z;
    const int first_nz = nz ? 64 * lane + __ffsll((long long)nz) - 1 : WB_PP;
    int after;  // first non-zero position in lanes > lane
    {
      int v = first_nz;
      for (int o = 1; o < 32; o <<= 1) {
        const int t2 = __shfl_down_sync(0xffffffffu, v, o);
        if (lane + o < 32) v = min(v, t2);
      }
      const int nxt = __shfl_down_sync(0xffffffffu, v, 1);
      after = lane < 31 ? nxt : WB_PP;
    }
    // token bit costs of this lane's 64 symbols (tokenize + pack_tokens, entropy.py:324-421),
    // counted per 32-symbol word by k_block_analyze (a run counts where it starts)
    const uint32_t wb2 = *reinterpret_cast<const uint32_t*>(P.wbits + ((i64)gid * P.max_slots + j) * 64 + 2 * lane);
    uint32_t tot = (wb2 & 0xFFFFu) + (wb2 >> 16);
    uint32_t incl = tot;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t2 = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t2;
    }
    const uint32_t slot_bits = __shfl_sync(0xffffffffu, incl, 31);
    if (lane == 0 && slot_bits != send - sbeg) record_error(P.st, WBPC_ERR_CORRUPTION, (u64)gid, 3);  // internal
    const int sh = (int)(g0 & 31);
    const uint32_t lane_off = incl - tot;
    if (slot_bits + 64 <= (uint32_t)(CAPW * 32)) {
      // fast path: whole slot in the window; each lane packs its segment in a register word
      const int nw = (int)((sh + slot_bits + 31) >> 5);
      const uint32_t ws = sh + lane_off, we = ws + tot;  // window bits of this lane's segment
      // only the words a lane shares with a neighbour (or with bits outside the slot) are OR-ed;
      // every other window word is written whole, so just the segment's end words are cleared
      if (tot) {
        win[ws >> 5] = 0u;
        win[(we - 1) >> 5] = 0u;
      }
      if (lane == 0) win[0] = 0u;  // a slot of 0-bit codes has no segment but may share word 0
      __syncwarp();
      uint32_t wi = ws >> 5;
      // 32-bit accumulator: `fill` pending bits at the top of `hi` (fill < 32 between tokens);
      // each append is <= 32 bits, a full 32-bit word is written out as soon as it exists and
      // the bits that did not fit start the next one
      int fill = (int)(ws & 31);
      uint32_t hi = 0;
      // shared addresses of the staged symbols, the token table and the window, made opaque so the
      // register-capped loop keeps them instead of re-deriving them per token
      uint32_t my_s, tok_s, win_s;
      asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(my_s) : "l"(my));
      asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(tok_s) : "l"(S.tok));
      asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(win_s) : "l"(win));
      // append nb (1..32) bits, branch free: the word that fills up is stored (or OR-ed when it is
      // shared with the previous lane's segment) under a predicate, so lanes never diverge here
      auto put = [&](uint32_t v, int nb) {
        const uint32_t top = v << (32 - nb);  // MSB-aligned code
        hi |= top >> fill;
        const int tot = fill + nb;
        const bool full = tot >= 32;
        const bool shared_w = (wi << 5) < ws;
        asm volatile(
            "{\n .reg .pred p, q;\n setp.ne.b32 p, %2, 0;\n setp.ne.b32 q, %3, 0;\n"
            " @p red.shared.or.b32 [%0], %1;\n @q st.shared.u32 [%0], %1;\n}\n" ::"r"(win_s + 4u * wi),
            "r"(hi), "r"((int)(full && shared_w)), "r"((int)(full && !shared_w))
            : "memory");
        // bits of this code that did not fit the stored word (0 when fill == 0: clamped shift)
        const uint32_t spill = __funnelshift_l(0u, top, 32 - fill);
        hi = full ? spill : hi;
        wi += full ? 1u : 0u;
        fill = full ? tot - 32 : tot;
      };
      const int zrw = lzr + width;                       // bits of a zr code + its counter
      const uint32_t zrc = lzr ? czr << width : 0u;       // zr code shifted above the counter
      // positions that emit something: symbols outside runs and run starts (bit scan).  Symbols
      // and single-chunk runs share one append (no divergence between the two kinds of token);
      // multi-chunk runs and zr codes too long to carry their counter take the slow path.
      const uint64_t todo64 = ~inrun | starts;
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {  // 32-bit halves: cheaper scan than 64-bit ops
        uint32_t todo = (uint32_t)(todo64 >> (32 * half));
        const uint32_t st32 = (uint32_t)(starts >> (32 * half));
        const uint32_t nzhalf = (uint32_t)(nz >> (32 * half));
        const uint32_t nzu = half ? 0u : (uint32_t)(nz >> 32);
        const int nzu_end = nzu ? 64 * lane + 32 + __ffs(nzu) - 1 : after;
        while (todo) {
          const int i = 32 * half + __ffs(todo) - 1;
          todo &= todo - 1;
          const bool isrun = (st32 >> (i & 31)) & 1u;
          unsigned sym;  // my[i] through an opaque shared address (a run start reads its zero symbol)
          asm("ld.shared.u8 %0, [%1];" : "=r"(sym) : "r"(my_s + (uint32_t)i));
          uint2 tk;
          asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(tk.x), "=r"(tk.y) : "r"(tok_s + 8u * sym));
          // run end: the next non-zero position (this half, the upper half, or a later lane)
          const uint32_t nzh = nzhalf & (~0u << (i & 31));
          const int end = nzh ? 64 * lane + 32 * half + __ffs(nzh) - 1 : nzu_end;
          const int L = end - (64 * lane + i);
          const uint32_t v = isrun ? (zrc | (uint32_t)L) : tk.x;
          const int nb = isrun ? zrw : (int)tk.y;
          const bool simple = isrun ? (L <= cap && zrw <= 32) : nb <= 32;
          if (simple) {
            if (nb) put(v, nb);
          } else if (isrun) {
            // all but the last chunk carry `cap`, the last the remainder (entropy.py:349-358)
            const int nch = L <= cap ? 1 : chunk_count_m(L, mcap);
            for (int c = 0; c < nch; ++c) {
              const int vv = c == nch - 1 ? L - cap * (nch - 1) : cap;
              if (zrw <= 32) {
                put(zrc | (uint32_t)vv, zrw);
              } else {
                put(czr, lzr);
                put((uint32_t)vv, width);
              }
            }
          } else {  // a zr code too long to carry its counter in one append
            put(S.code_val[sym], S.code_len[sym]);
            put(0u, width);
          }
        }
      }
      if (j + EW < nstored) stage(j + EW);  // this lane is done with its symbols of slot j
      const uint32_t cur = hi;
      if (fill > 0 && (wi << 5) < we) atomicOr(&win[wi], cur);
      __syncwarp();
      flush_window(outw, g0 >> 5, win, nw, sh != 0, ((sh + slot_bits) & 31) != 0);
      __syncwarp();
    } else {
      // large slot: windows of (CAPW-2)*32 bits, tokens clipped to the window
      for (uint32_t wlo = 0; wlo < slot_bits; wlo += (CAPW - 2) * 32) {
        const uint32_t whi = min(slot_bits, wlo + (CAPW - 2) * 32);
        const u64 gstart = g0 + wlo;
        const int shw = (int)(gstart & 31);
        const int nw = (int)((shw + (whi - wlo) + 31) >> 5);
        for (int i = lane; i < nw + 1; i += 32) win[i] = 0;
        __syncwarp();
        long long off = (long long)shw - (long long)wlo + lane_off;
        for (int i = 0; i < 64; ++i) {
          if ((starts >> i) & 1ull) {
            const uint64_t m = nz & (~0ull << i);
            const int end = m ? 64 * lane + __ffsll((long long)m) - 1 : after;
            const int L = end - (64 * lane + i);
            const int nch = chunk_count_m(L, mcap);
            for (int c = 0; c < nch; ++c) {
              const int vv = c == nch - 1 ? L - cap * (nch - 1) : cap;
              if (off + lzr + width > 0 && off < (long long)nw * 32)
                put_bits_clip(win, off, ((u64)czr << width) | (u64)vv, lzr + width, nw);
              off += lzr + width;
            }
          } else if (!((inrun >> i) & 1ull)) {
            const unsigned sym = my[i];
            const int len = S.code_len[sym];
            if (off + len > 0 && off < (long long)nw * 32) put_bits_clip(win, off, (u64)S.code_val[sym], len, nw);
            off += len + (sym == (unsigned)zr ? width : 0);
          }
        }
        __syncwarp();
        // The word where two windows meet belongs to this slot only: the earlier window stores it
        // whole (its low bits zero) and the next window ORs into it, so no stale output bits
        // survive.  Only the slot's own last word is shared with the next slot / block.
        const bool last_win = whi == slot_bits;
        flush_window(outw, gstart >> 5, win, nw, shw != 0, last_win && ((shw + (whi - wlo)) & 31) != 0);
        __syncwarp();
      }
      if (j + EW < nstored) stage(j + EW);
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// Block API: max |c| per raw 128x128 block (CoefficientBlock.build depth, bitplanes.py:77-79).
__global__ void k_raw_bmax(const Geom g, const int32_t* coef, unsigned* bmax, DevStatus* st) {
  const int gid = blockIdx.x;
  const LevelGeom& lg = g.lv[g.raw_kind];
  const int nsub = g.raw_kind ? 3 : 1;
  unsigned m = 0;
  bool bad = false;
  for (int s = 0; s < nsub; ++s) {
    const int32_t* p = coef + lg.off[g.raw_kind ? 1 + s : 0] + (i64)gid * WB_DIM * WB_DIM;
    for (int i = threadIdx.x; i < WB_DIM * WB_DIM; i += blockDim.x) {
      const int v = p[i];
      bad |= v == INT_MIN;
      m = max(m, (unsigned)abs(v));
    }
  }
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ unsigned red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  if (bad) record_error(st, WBPC_ERR_UNSUPPORTED, (u64)gid, 0);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned a = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a = max(a, red[w]);
    bmax[gid] = a;
  }
}

cudaError_t launch_raw_bmax(const Geom& g, int nblocks, const int32_t* coef, unsigned* bmax, DevStatus* st,
                            cudaStream_t s) {
  k_raw_bmax<<<nblocks, 256, 0, s>>>(g, coef, bmax, st);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------ launch
size_t emit_smem_bytes() { return sizeof(EmitSmem); }

cudaError_t launch_offsets(int nblocks, int spi, int batch, const uint32_t* sizes, u64* block_off, u64* img_off,
                           u64 cap, DevStatus* st, cudaStream_t s, int raw = 0, uint32_t* outw = nullptr) {
  OffsetsParams O;
  O.raw = raw;
  O.outw = outw;
  O.nblocks = nblocks;
  O.spi = spi;
  O.batch = batch;
  O.sizes = sizes;
  O.block_off = block_off;
  O.img_off = img_off;
  O.cap = cap;
  O.st = st;
  prof_mark("offsets", s);
  k_offsets<<<1, 1024, 0, s>>>(O);
  return cudaGetLastError();
}

cudaError_t launch_encode_blocks(const Geom& g, int batch, const void* coef, const unsigned* bmax, uint8_t* syms,
                                 uint16_t* wbits, BlockMeta* meta, void* stats, uint32_t* zmask, uint32_t* sizes,
                                 u64* block_off, u64* img_off, uint8_t* out, u64 cap, DevStatus* st, cudaStream_t s) {
  // dynamic smem opt-in is a per-device function attribute: set once per device
  static std::atomic<bool> attr[64];
  int dev = 0;
  cudaGetDevice(&dev);
  const int max_slots = g.sym_stride_hp / WB_PP;
  const int sym_smem = (int)((sizeof(SymSmem) + 15) & ~(size_t)15) + max_slots * 256;
  if (dev < 0 || dev >= 64 || !attr[dev].load(std::memory_order_acquire)) {
    cudaFuncSetAttribute(k_block_symbols, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)((sizeof(SymSmem) + 15) & ~(size_t)15) + WB_MAX_SLOTS * 256);
    cudaFuncSetAttribute(k_block_sizes, cudaFuncAttributeMaxDynamicSharedMemorySize, WB_MAX_SLOTS * 256);
    cudaFuncSetAttribute(k_block_huffman, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)huffman_smem_bytes());
    cudaFuncSetAttribute(k_block_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(EmitSmem));
    if (dev >= 0 && dev < 64) attr[dev].store(true, std::memory_order_release);
  }
  const int nblocks = batch * g.slots_per_image;
  AnalyzeParams A;
  A.g = g;
  A.nblocks = nblocks;
  A.coef = coef;
  A.bmax = bmax;
  A.syms = syms;
  A.wbits = wbits;
  A.meta = meta;
  A.stats = reinterpret_cast<BlockStats*>(stats);
  A.zmask = zmask;
  A.sizes = sizes;
  A.st = st;
  A.max_slots = max_slots;
  prof_mark("block_symbols", s);
  k_block_symbols<<<nblocks, CT, sym_smem, s>>>(A);
  prof_mark("block_huffman", s);
  k_block_huffman<<<(nblocks + HB - 1) / HB, HWARPS * 32, huffman_smem_bytes(), s>>>(A);
  prof_mark("block_sizes", s);
  k_block_sizes<<<nblocks, CT, max_slots * 256, s>>>(A);
  // block-boundary output words are cleared by k_offsets, block-internal shared words by the
  // emitting CTA itself; every other output word is written whole
  launch_offsets(nblocks, g.slots_per_image, batch, sizes, block_off, img_off, cap, st, s, g.raw_kind >= 0,
                 reinterpret_cast<uint32_t*>(out));
  EmitParams E;
  E.g = g;
  E.syms = syms;
  E.wbits = wbits;
  E.max_slots = max_slots;
  E.meta = meta;
  E.block_off = block_off;
  E.img_off = img_off;
  E.out = out;
  E.cap = cap;
  E.st = st;
  prof_mark("block_emit", s);
  k_block_emit<<<nblocks, EW * 32, sizeof(EmitSmem), s>>>(E);
  return cudaGetLastError();
}

size_t block_stats_bytes() { return sizeof(BlockStats); }

}  // namespace wb
