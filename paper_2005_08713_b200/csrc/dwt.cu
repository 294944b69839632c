// dwt.cu — reversible colour transform + 5/3 integer lifting DWT, forward and inverse (sm_100a).
//
// Replaces (reference /root/reference/pkg/src/wbpc):
//   rct_forward / rct_inverse          transforms.py:79-104
//   _split_axis0 / _merge_axis0        transforms.py:107-162
//   _split_plane / _merge_plane        transforms.py:184-199
//   dwt2d_forward (recursion on LL)    transforms.py:202-216
//   decode_image level loop            container.py:324-335, _finish_image :301-306
//
// Register-streaming design: one warp owns a strip of 32 subband columns x SR subband rows.
// Lane l holds the input column pair (2n, 2n+1) of subband column n; the horizontal lifting
// neighbours come from warp shuffles (edge lanes load their 1-2 halo samples themselves), and the
// vertical lifting streams down the strip keeping the previous even row and the previous high
// coefficient in registers - every input sample is read once from HBM and every coefficient
// written once, coalesced (32 lanes x 4 B per subband row).  Image edges use whole-sample
// symmetric extension by reflecting the per-lane column / per-row index (exactly the reference's
// mirroring for even/odd lengths and n == 1).  Forward lifts rows then columns, inverse merges
// columns then rows, which pins the reference's H-then-V order.  int32 arithmetic with floor
// shifts; the host's static coefficient bound guarantees no overflow.  The forward pass also
// records max |c| per 128x128 block (the coder's plane depth) and zero-pads the block grid.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace wb {

constexpr int WPB = 8;   // warps per CTA
constexpr unsigned FULL = 0xffffffffu;

struct FwdParams {
  Geom g;
  int level;               // producing level l (1..L)
  const void* src;         // level 1: image; level >1: unused (coefficients)
  int src_dtype, src_layout;
  i64 src_img_stride;      // bytes between images (level 1)
  void* coef;              // coefficient base (image-major: img_stride elements per image);
                           // int16 elements when g.coef16, else int32
  unsigned* bmax;          // per (image, slot) max |c|
  DevStatus* st;
  int sr;                  // strip height (subband rows), divides 128
  int fast_rgb8;           // level 1: interior strips handled by k_fwd_rgb8
};

// Coefficient element store; CT = int16_t when the static bound allows (g.coef16), else int32_t.
template <typename CT>
static __device__ __forceinline__ void stc(const FwdParams& P, i64 idx, int v) {
  reinterpret_cast<CT*>(P.coef)[idx] = (CT)v;
}

// Strip height: the largest of 32/16/8 that still gives >= ~4 warps per SM.
static int pick_sr(i64 strips_x, i64 rows, i64 z) {
  for (int sr = 32; sr > 8; sr >>= 1)
    if (strips_x * ((rows + sr - 1) / sr) * z >= 148 * 4 * 8) return sr;
  return 8;
}

// ---------------------------------------------------------------------------- forward
// Horizontal 5/3 split of one row (transforms.py:125,133) for the lane's column pair.
// xa, xb: x[2n0-2], x[2n0-1] (lane 0 halo); xr: x[2n0+64] (lane 31 halo).
static __device__ __forceinline__ void hsplit(int lane, int xe, int xo, int xa, int xb, int xr, int& lo, int& hi) {
  int xn = __shfl_down_sync(FULL, xe, 1);
  if (lane == 31) xn = xr;
  hi = xo - ((xe + xn) >> 1);
  const int hm1 = xb - ((xa + xe) >> 1);  // meaningful on lane 0 only: high[n0-1]
  int hp = __shfl_up_sync(FULL, hi, 1);
  if (lane == 0) hp = hm1;
  lo = xe + ((hp + hi + 2) >> 2);
}

// Row sources: `row_ptr(y)` is uniform per row; per-lane element offsets are precomputed once.
template <typename T, bool HWC>
struct PixSrc {
  const T* p;
  int W, H, C;
  __device__ __forceinline__ const T* row_ptr(int y, int c) const {
    return HWC ? p + (i64)y * W * C + c : p + ((i64)c * H + y) * W;
  }
  __device__ __forceinline__ int col_off(int x) const { return HWC ? x * C : x; }
};

template <typename E>
struct CoefSrc {
  const E* p;
  int pitch;
  __device__ __forceinline__ const E* row_ptr(int y, int) const { return p + (i64)y * pitch; }
  __device__ __forceinline__ int col_off(int x) const { return x; }
};

template <typename T>
static __device__ __forceinline__ int ldv(const T* p) { return (int)__ldg(p); }

// NCH channels handled by the warp (3 with the fused RCT, else 1).  Strip: 32 subband columns
// x `sr` subband rows (sr divides 128, so a strip never crosses a block boundary).
template <int NCH, bool RCT, typename T, typename CT, typename Src>
static __device__ void fwd_strip(const FwdParams& P, const Src& S, int b, int ch0, int n0, int m0, int sr) {
  const Geom& g = P.g;
  const int lev = P.level;
  const LevelGeom& lg = g.lv[lev];
  const LevelGeom& pg = g.lv[lev - 1];
  const int lane = threadIdx.x & 31;
  const int NX = pg.w, NY = pg.h;
  const int n = n0 + lane;
  // per-lane column offsets; every lane loads the halo slots too (its own columns on lanes
  // 1..30) so the row loads are branch free
  const int oe = S.col_off(reflect_pos(2 * n, NX)), oo = S.col_off(reflect_pos(2 * n + 1, NX));
  const int oa = lane == 0 ? S.col_off(reflect_pos(2 * n0 - 2, NX)) : oe;
  const int ob = lane == 0 ? S.col_off(reflect_pos(2 * n0 - 1, NX)) : oo;
  const int orr = lane == 31 ? S.col_off(reflect_pos(2 * n0 + 64, NX)) : oe;
  const int lim = 1 << g.bd;
  unsigned badacc = 0;
  const i64 img0 = (i64)b * g.img_stride;

  // raw loads of one input row (halo slots only on the edge lanes) ...
  struct Raw { int e[NCH], o[NCH], a[NCH], b[NCH], r[NCH]; };
  auto load = [&](int y, Raw& R) {
    const int yy = reflect_pos(y, NY);
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const T* rp = (const T*)S.row_ptr(yy, RCT ? c : ch0);
      R.e[c] = ldv(rp + oe);
      R.o[c] = ldv(rp + oo);
      R.a[c] = lane == 0 ? ldv(rp + oa) : 0;
      R.b[c] = lane == 0 ? ldv(rp + ob) : 0;
      R.r[c] = lane == 31 ? ldv(rp + orr) : 0;
    }
  };
  // ... then colour transform + horizontal split
  auto split = [&](Raw& R, int* L, int* Hh) {
    if (lev == 1) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) badacc |= (unsigned)(R.e[c] | R.o[c] | R.a[c] | R.b[c] | R.r[c]);
    }
    if (RCT) {  // rct_forward (transforms.py:86-88): Y=(R+2G+B)>>2, Cb=B-G, Cr=R-G
      auto rct = [](int* v) {
        int Rr = v[0], G = v[1], B = v[2];
        v[0] = (Rr + 2 * G + B) >> 2;
        v[1] = B - G;
        v[2] = Rr - G;
      };
      rct(R.e); rct(R.o); rct(R.a); rct(R.b); rct(R.r);
    }
#pragma unroll
    for (int c = 0; c < NCH; ++c) hsplit(lane, R.e[c], R.o[c], R.a[c], R.b[c], R.r[c], L[c], Hh[c]);
  };
  auto row = [&](int y, int* L, int* Hh) {
    Raw R;
    load(y, R);
    split(R, L, Hh);
  };

  // vertical prologue: rows 2m0-2, 2m0-1, 2m0 -> high[m0-1] and the even row 2m0
  int La[NCH], Ha[NCH], Lb[NCH], Hb[NCH], Lc[NCH], Hc[NCH];
  row(2 * m0 - 2, La, Ha);
  row(2 * m0 - 1, Lb, Hb);
  row(2 * m0, Lc, Hc);
  int eL[NCH], eH[NCH], vL[NCH], vH[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    vL[c] = Lb[c] - ((La[c] + Lc[c]) >> 1);
    vH[c] = Hb[c] - ((Ha[c] + Hc[c]) >> 1);
    eL[c] = Lc[c];
    eH[c] = Hc[c];
  }
  const bool cLL = n < lg.sw[0], cLH = n < lg.sw[1], cHL = n < lg.sw[2], cHH = n < lg.sw[3];
  const bool top = lev == g.L;
  unsigned mhp[NCH], mll[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) { mhp[c] = 0; mll[c] = 0; }
  i64 outi[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) outi[c] = img0 + (i64)(ch0 + c) * g.chan_stride + (i64)m0 * lg.pw + n;
  const i64 o1 = lg.off[1] - lg.off[0], o2 = lg.off[2] - lg.off[0], o3 = lg.off[3] - lg.off[0];
  // software pipeline: the two input rows of output row m+1 are loaded before row m is lifted
  // (two row pairs in flight per warp), the loop unrolled by two so buffers swap roles
  auto lift = [&](int m, Raw& R1, Raw& R2) {
    int L1[NCH], H1[NCH], L2[NCH], H2[NCH];
    split(R1, L1, H1);
    split(R2, L2, H2);
    const bool rLL = m < lg.sh[0], rLH = m < lg.sh[1], rHL = m < lg.sh[2], rHH = m < lg.sh[3];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int vhL = L1[c] - ((eL[c] + L2[c]) >> 1);
      const int vlL = eL[c] + ((vL[c] + vhL + 2) >> 2);
      const int vhH = H1[c] - ((eH[c] + H2[c]) >> 1);
      const int vlH = eH[c] + ((vH[c] + vhH + 2) >> 2);
      eL[c] = L2[c]; vL[c] = vhL;
      eH[c] = H2[c]; vH[c] = vhH;
      // zero padding outside the true subband dims (container.py:132-145)
      const int ll = (cLL && rLL) ? vlL : 0;
      const int lh = (cLH && rLH) ? vhL : 0;
      const int hl = (cHL && rHL) ? vlH : 0;
      const int hh = (cHH && rHH) ? vhH : 0;
      const i64 q = outi[c] + lg.off[0];
      stc<CT>(P, q, ll);
      stc<CT>(P, q + o1, lh);
      stc<CT>(P, q + o2, hl);
      stc<CT>(P, q + o3, hh);
      outi[c] += lg.pw;
      mhp[c] = max(mhp[c], max((unsigned)abs(lh), max((unsigned)abs(hl), (unsigned)abs(hh))));
      mll[c] = max(mll[c], (unsigned)abs(ll));
    }
  };
  Raw A1, A2, B1, B2;
  load(2 * m0 + 1, A1);
  load(2 * m0 + 2, A2);
  for (int m = m0; m < m0 + sr; m += 2) {
    const bool more = m + 1 < m0 + sr;
    if (more) {
      load(2 * m + 3, B1);
      load(2 * m + 4, B2);
    }
    lift(m, A1, A2);
    if (!more) break;
    if (m + 2 < m0 + sr) {
      load(2 * m + 5, A1);
      load(2 * m + 6, A2);
    }
    lift(m + 1, B1, B2);
  }
  if (lev == 1 && __any_sync(FULL, badacc >= (unsigned)lim) && lane == 0)
    record_error(P.st, WBPC_ERR_DOMAIN, 0, 0);  // validate_source, transforms.py:57-62
  const int by = m0 / WB_DIM, bx = n0 / WB_DIM;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    unsigned a = __reduce_max_sync(FULL, mhp[c]);
    unsigned l = __reduce_max_sync(FULL, mll[c]);
    if (lane == 0) {
      unsigned* bm = P.bmax + (i64)b * g.slots_per_image + (i64)(ch0 + c) * g.slots_per_channel;
      atomicMax(&bm[lg.slot0 + by * lg.gw + bx], a);
      if (top) atomicMax(&bm[by * lg.gw + bx], l);
    }
  }
}


// Fast path for interior strips of 8-bit interleaved RGB with the RCT (cfg 2/3/4 layout): the
// warp loads each input row segment (pixels 2n0-2 .. 2n0+64 = bytes [6n0-8, 6n0+200)) as 52
// coalesced 32-bit words (2 per lane), and every lane gathers its 6 bytes (+ halo bytes) with
// shuffles.  Raw state is 2 registers per row, so two row pairs are kept in flight.
static __device__ __forceinline__ void rgb_from_words(int lane, uint32_t w0, uint32_t w1, int* e, int* o, int* a,
                                                      int* b, int* r) {
  const int ia = (6 * lane + 8) >> 2;  // 2..48
  const uint32_t a0 = __shfl_sync(FULL, w0, ia & 31), a1 = __shfl_sync(FULL, w1, ia & 31);
  const uint32_t b0 = __shfl_sync(FULL, w0, (ia + 1) & 31), b1 = __shfl_sync(FULL, w1, (ia + 1) & 31);
  const uint32_t A = ia < 32 ? a0 : a1, B = ia + 1 < 32 ? b0 : b1;
  const uint64_t X = ((((uint64_t)B) << 32) | A) >> ((lane & 1) ? 16 : 0);
  e[0] = (int)(X & 255); e[1] = (int)((X >> 8) & 255); e[2] = (int)((X >> 16) & 255);
  o[0] = (int)((X >> 24) & 255); o[1] = (int)((X >> 32) & 255); o[2] = (int)((X >> 40) & 255);
  // lane-0 halo: pixels 2n0-2, 2n0-1 = bytes [2, 8) -> words 0, 1
  const uint32_t h0 = __shfl_sync(FULL, w0, 0), h1 = __shfl_sync(FULL, w0, 1);
  const uint64_t Y = ((((uint64_t)h1) << 32) | h0) >> 16;
  a[0] = (int)(Y & 255); a[1] = (int)((Y >> 8) & 255); a[2] = (int)((Y >> 16) & 255);
  b[0] = (int)((Y >> 24) & 255); b[1] = (int)((Y >> 32) & 255); b[2] = (int)((Y >> 40) & 255);
  // lane-31 halo: pixel 2n0+64 = bytes [200, 203) -> word 50 (lane 18 of w1)
  const uint32_t z = __shfl_sync(FULL, w1, 18);
  r[0] = (int)(z & 255); r[1] = (int)((z >> 8) & 255); r[2] = (int)((z >> 16) & 255);
}

template <typename CT>
static __device__ void fwd_strip_rgb8(const FwdParams& P, const uint8_t* img, int b, int n0, int m0, int sr) {
  const Geom& g = P.g;
  const LevelGeom& lg = g.lv[1];
  const int lane = threadIdx.x & 31;
  const int NY = g.H;
  const int n = n0 + lane;
  const i64 rowbytes = (i64)g.W * 3;
  const uint8_t* seg = img + 6 * (i64)n0 - 8;
  const i64 img0 = (i64)b * g.img_stride;
  auto load = [&](int y, uint32_t& w0, uint32_t& w1) {
    const uint32_t* rp = reinterpret_cast<const uint32_t*>(seg + (i64)reflect_pos(y, NY) * rowbytes);
    w0 = __ldg(rp + lane);
    w1 = lane < 20 ? __ldg(rp + 32 + lane) : 0u;
  };
  auto split = [&](uint32_t w0, uint32_t w1, int* L, int* Hh) {
    int e[3], o[3], a[3], bb[3], r[3];
    rgb_from_words(lane, w0, w1, e, o, a, bb, r);
    auto rct = [](int* v) {  // rct_forward (transforms.py:86-88)
      int R = v[0], G = v[1], B = v[2];
      v[0] = (R + 2 * G + B) >> 2;
      v[1] = B - G;
      v[2] = R - G;
    };
    rct(e); rct(o); rct(a); rct(bb); rct(r);
#pragma unroll
    for (int c = 0; c < 3; ++c) hsplit(lane, e[c], o[c], a[c], bb[c], r[c], L[c], Hh[c]);
  };
  uint32_t p0, p1;
  int La[3], Ha[3], Lb[3], Hb[3], Lc[3], Hc[3];
  load(2 * m0 - 2, p0, p1); split(p0, p1, La, Ha);
  load(2 * m0 - 1, p0, p1); split(p0, p1, Lb, Hb);
  load(2 * m0, p0, p1); split(p0, p1, Lc, Hc);
  int eL[3], eH[3], vL[3], vH[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    vL[c] = Lb[c] - ((La[c] + Lc[c]) >> 1);
    vH[c] = Hb[c] - ((Ha[c] + Hc[c]) >> 1);
    eL[c] = Lc[c];
    eH[c] = Hc[c];
  }
  const bool cLL = n < lg.sw[0], cLH = n < lg.sw[1], cHL = n < lg.sw[2], cHH = n < lg.sw[3];
  const bool top = g.L == 1;
  unsigned mhp[3] = {0, 0, 0}, mll[3] = {0, 0, 0};
  const i64 o1 = lg.off[1] - lg.off[0], o2 = lg.off[2] - lg.off[0], o3 = lg.off[3] - lg.off[0];
  i64 q = img0 + lg.off[0] + (i64)m0 * lg.pw + n;
  // two row pairs in flight: (p0,p1)/(q0,q1) hold rows 2m+1, 2m+2; (s0..t1) the next pair
  uint32_t q0, q1, s0, s1, t0, t1;
  load(2 * m0 + 1, p0, p1);
  load(2 * m0 + 2, q0, q1);
  load(2 * m0 + 3, s0, s1);
  load(2 * m0 + 4, t0, t1);
  for (int m = m0; m < m0 + sr; ++m) {
    const uint32_t c0 = p0, c1 = p1, d0 = q0, d1 = q1;
    p0 = s0; p1 = s1; q0 = t0; q1 = t1;
    if (m + 2 < m0 + sr) {
      load(2 * m + 5, s0, s1);
      load(2 * m + 6, t0, t1);
    }
    int L1[3], H1[3], L2[3], H2[3];
    split(c0, c1, L1, H1);
    split(d0, d1, L2, H2);
    const bool rLL = m < lg.sh[0], rLH = m < lg.sh[1], rHL = m < lg.sh[2], rHH = m < lg.sh[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int vhL = L1[c] - ((eL[c] + L2[c]) >> 1);
      const int vlL = eL[c] + ((vL[c] + vhL + 2) >> 2);
      const int vhH = H1[c] - ((eH[c] + H2[c]) >> 1);
      const int vlH = eH[c] + ((vH[c] + vhH + 2) >> 2);
      eL[c] = L2[c]; vL[c] = vhL;
      eH[c] = H2[c]; vH[c] = vhH;
      const int ll = (cLL && rLL) ? vlL : 0;
      const int lh = (cLH && rLH) ? vhL : 0;
      const int hl = (cHL && rHL) ? vlH : 0;
      const int hh = (cHH && rHH) ? vhH : 0;
      const i64 qc = q + (i64)c * g.chan_stride;
      stc<CT>(P, qc, ll);
      stc<CT>(P, qc + o1, lh);
      stc<CT>(P, qc + o2, hl);
      stc<CT>(P, qc + o3, hh);
      mhp[c] = max(mhp[c], max((unsigned)abs(lh), max((unsigned)abs(hl), (unsigned)abs(hh))));
      mll[c] = max(mll[c], (unsigned)abs(ll));
    }
    q += lg.pw;
  }
  // 8-bit samples are always < 2^bd for bd == 8 (validate_source): nothing to record
  const int by = m0 / WB_DIM, bx = n0 / WB_DIM;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    unsigned a = __reduce_max_sync(FULL, mhp[c]);
    unsigned l = __reduce_max_sync(FULL, mll[c]);
    if (lane == 0) {
      unsigned* bm = P.bmax + (i64)b * g.slots_per_image + (i64)c * g.slots_per_channel;
      atomicMax(&bm[lg.slot0 + by * lg.gw + bx], a);
      if (top) atomicMax(&bm[by * lg.gw + bx], l);
    }
  }
}

// ---- TMA-pipelined level 1 for 8-bit interleaved RGB + RCT (cfg 2/3/4 layout) ------------------
// CTA = TW consumer warps + 1 producer warp; consumer warp w owns 64 subband columns
// (n0 = N0 + 64w), lane k the two columns n0+2k, n0+2k+1 = pixels p = 2n0+4k .. +3.  The producer
// streams the input rows the CTA needs, two per ring slot (an odd row and the even row after it),
// into NST shared-memory slots with cp.async.bulk; full/empty mbarriers pace producer and
// consumers.  A slot row holds image row bytes [6*N0 - 16, 6*N0 + 384*TW + 16); pixels outside the
// image row (left/right image edges) are written into the slot by the producer warp already
// reflected (whole-sample symmetric extension, transforms.py:117-133), so every consumer lane reads
// the same 24-byte window -- pixels p-2 .. p+4 -- as six aligned 32-bit words and lifts its two
// column pairs with no shuffles and no edge cases.  Consumers probe the next slot's barrier
// (non-blocking test_wait) before lifting the current one, so its latency hides behind the math.
// Requires W*3 % 16 == 0 (16-B aligned rows) and an aligned source.
constexpr int TW = 4;                          // consumer warps
#ifndef WBPC_FWD_MINB
#define WBPC_FWD_MINB 4                        // resident CTAs per SM (register cap)
#endif
constexpr int NST = 8;                         // ring slots (row pairs in flight)
constexpr int ROWB = 16 + 6 * 64 * TW + 16;    // bytes per staged row
constexpr int SEGB = 2 * ROWB;                 // slot: odd row, then even row

static __device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
static __device__ __forceinline__ void bar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(n));
}
static __device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(b)), "r"(bytes) : "memory");
}
static __device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(b)) : "memory");
}
static __device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(s_u32(b)), "r"(parity) : "memory");
}
static __device__ __forceinline__ uint32_t bar_test(uint64_t* b, uint32_t parity) {
  uint32_t done;
  asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(done) : "r"(s_u32(b)), "r"(parity) : "memory");
  return done;
}
// 32-bit shared address through an opaque conversion: the compiler keeps the result in a register
// instead of re-deriving the address (CTA window base + offset) at every use
static __device__ __forceinline__ uint32_t s_u32_keep(const void* p) {
  uint32_t a;
  asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(a) : "l"(p));
  return a;
}
// the same on 32-bit shared addresses the caller keeps in registers (a generic pointer would be
// converted, through the CTA's shared window, at every use)
static __device__ __forceinline__ void bar_arrive_a(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
static __device__ __forceinline__ void bar_wait_a(uint32_t a, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(a), "r"(parity) : "memory");
}
static __device__ __forceinline__ uint32_t bar_test_a(uint32_t a, uint32_t parity) {
  uint32_t done;
  asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(done) : "r"(a), "r"(parity) : "memory");
  return done;
}
static __device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(s_u32(dst)), "l"(src), "r"(bytes), "r"(s_u32(b)) : "memory");
}
static __device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
static __device__ __forceinline__ int byte_of(uint32_t w, int k) { return (int)__byte_perm(w, 0u, 0x4440u + k); }

// Vertical lifting runs SWAR on the lane's two columns: each 32-bit word holds the two columns'
// values as 16-bit fields biased by SB = 2^14.  Level-1 values of 8-bit RGB stay within +-2^12
// and every intermediate below keeps each field inside [0, 2^16), so a plain 32-bit add or
// subtract of packed words is exact per field, and a logical shift followed by masking off the
// bits the high field spills into the low field is an exact per-field floor division.
constexpr uint32_t SB = 0x4000u, SB2 = 0x40004000u;

// high = odd - floor((even_prev + even_next) / 2)  (transforms.py:125), biased in and out
static __device__ __forceinline__ uint32_t swar_high(uint32_t O, uint32_t E0, uint32_t E1) {
  return O - (((E0 + E1) >> 1) & 0x7FFF7FFFu) + SB2;
}
// low = even + floor((high_prev + high + 2) / 4)  (transforms.py:133), biased in and out
static __device__ __forceinline__ uint32_t swar_low(uint32_t E, uint32_t Hp, uint32_t H) {
  return E + (((Hp + H + 0x00020002u) >> 2) & 0x3FFF3FFFu) - 0x20002000u;
}

// colour transform + horizontal split of one staged row window (pixels p-2 .. p+4 in six words):
// per channel the lane's two low (Lp) and two high (Hp) coefficients, packed and biased
static __device__ __forceinline__ void rgb_hsplit(const uint32_t* w, uint32_t* Lp, uint32_t* Hp) {
  int x[7][3];
  x[0][0] = byte_of(w[0], 2); x[0][1] = byte_of(w[0], 3); x[0][2] = byte_of(w[1], 0);
  x[1][0] = byte_of(w[1], 1); x[1][1] = byte_of(w[1], 2); x[1][2] = byte_of(w[1], 3);
  x[2][0] = byte_of(w[2], 0); x[2][1] = byte_of(w[2], 1); x[2][2] = byte_of(w[2], 2);
  x[3][0] = byte_of(w[2], 3); x[3][1] = byte_of(w[3], 0); x[3][2] = byte_of(w[3], 1);
  x[4][0] = byte_of(w[3], 2); x[4][1] = byte_of(w[3], 3); x[4][2] = byte_of(w[4], 0);
  x[5][0] = byte_of(w[4], 1); x[5][1] = byte_of(w[4], 2); x[5][2] = byte_of(w[4], 3);
  x[6][0] = byte_of(w[5], 0); x[6][1] = byte_of(w[5], 1); x[6][2] = byte_of(w[5], 2);
#pragma unroll
  for (int i = 0; i < 7; ++i) {  // rct_forward (transforms.py:86-88): Y=(R+2G+B)>>2, Cb=B-G, Cr=R-G
    const int R = x[i][0], G = x[i][1], B = x[i][2];
    x[i][0] = (R + 2 * G + B) >> 2;
    x[i][1] = B - G;
    x[i][2] = R - G;
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {  // _split_axis0 (transforms.py:125,133) on columns p-2 .. p+4
    const int hm1 = x[1][c] - ((x[0][c] + x[2][c]) >> 1);
    const int h0 = x[3][c] - ((x[2][c] + x[4][c]) >> 1);
    const int h1 = x[5][c] - ((x[4][c] + x[6][c]) >> 1);
    const int l0 = x[2][c] + ((hm1 + h0 + 2) >> 2);
    const int l1 = x[4][c] + ((h0 + h1 + 2) >> 2);
    Lp[c] = __byte_perm((uint32_t)(l0 + (int)SB), (uint32_t)(l1 + (int)SB), 0x5410u);
    Hp[c] = __byte_perm((uint32_t)(h0 + (int)SB), (uint32_t)(h1 + (int)SB), 0x5410u);
  }
}

// store the lane's two coefficients (a biased packed word) as int16 x2 or int32 x2
template <typename CT>
static __device__ __forceinline__ void st_packed(char* p, uint32_t s16) {
  if constexpr (sizeof(CT) == 2) *reinterpret_cast<uint32_t*>(p) = s16;
  else *reinterpret_cast<int2*>(p) = make_int2((int)(int16_t)(s16 & 0xFFFFu), (int)(int16_t)(s16 >> 16));
}

// Persistent: CTA i handles tiles i, i + gridDim.x, ... (tile = 256 subband columns x sr rows of
// one image); the ring's slot counter runs on across tiles, so the producer streams the next
// tile's rows while the consumers finish the current one.
template <typename CT>
__global__ void __launch_bounds__((TW + 1) * 32, WBPC_FWD_MINB) k_fwd_rgb8_tma(FwdParams P, int tiles_x, int tiles_y, int ntiles) {
  __shared__ __align__(128) uint8_t ring[NST][SEGB];
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  const Geom& g = P.g;
  const LevelGeom& lg = g.lv[1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sr = P.sr;
  const int NX = g.W, NY = g.H;
  const i64 rowbytes = (i64)NX * 3;
  // slot k of a tile holds input rows 2m0-3+2k (odd; slot 0 leaves it out) and 2m0-2+2k (even),
  // k = 0..sr+1
  const int nslots = sr + 2;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) { bar_init(&full[i], 1); bar_init(&empty[i], TW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto tile_of = [&](int t, int& N0, int& m0, int& b) {
    N0 = (t % tiles_x) * (TW * 64);
    m0 = ((t / tiles_x) % tiles_y) * sr;
    b = t / (tiles_x * tiles_y);
  };
  if (warp == TW) {  // ---- producer warp
    uint32_t q = 0;  // running slot counter
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int N0, m0, b;
      tile_of(t, N0, m0, b);
      const uint8_t* img = (const uint8_t*)P.src + (i64)b * P.src_img_stride;
      const i64 s0 = 6 * (i64)N0 - 16;            // image row byte of staged row byte 0
      const i64 c0 = s0 < 0 ? 0 : s0;             // in-row bytes [c0, c1): one bulk copy per row
      const i64 c1 = s0 + ROWB < rowbytes ? s0 + ROWB : rowbytes;
      const uint32_t nb = c1 > c0 ? (uint32_t)(c1 - c0) : 0u;
      auto row_y = [&](int k, int h) { return reflect_pos(2 * m0 - 3 + 2 * k + h, NY); };
      for (int k = 0; k < nslots; ++k, ++q) {
        const int sl = q % NST;
        if (q >= NST) bar_wait(&empty[sl], ((q / NST) - 1) & 1);
        if (lane == 0) {
          bar_expect(&full[sl], (k == 0 ? 1u : 2u) * nb);
          if (nb)
            for (int h = (k == 0); h < 2; ++h)
              bulk_g2s(ring[sl] + h * ROWB + (c0 - s0), img + (i64)row_y(k, h) * rowbytes + c0, nb, &full[sl]);
        }
      }
    }
    return;
  }
  // ---- consumers
  const uint32_t win0 = s_u32_keep(ring[0]) + 16 + 384 * warp + 12 * lane - 8;  // pixel p-2 .. p+4
  const uint32_t full0 = s_u32_keep(full), empty0 = s_u32_keep(empty);
  const bool top = g.L == 1;
  constexpr int SZ = (int)sizeof(CT);
  const i64 cs = SZ * g.chan_stride, o1 = SZ * (lg.off[1] - lg.off[0]), o2 = SZ * (lg.off[2] - lg.off[0]),
            o3 = SZ * (lg.off[3] - lg.off[0]);
  const i64 pitch = SZ * (i64)lg.pw;
  uint32_t q = 0;  // running slot counter (same sequence as the producer's)
  bool fixl = false, fixr = false;  // per tile: the lane's window crosses the left / right row end
  // Whole-sample symmetric extension at the image row ends (transforms.py:117-133) from the lane's
  // own window (pixel p+j sits at window bytes 3j+8 .. 3j+10): pixels -2, -1 = pixels 2, 1 on the
  // lane with p = 0, pixel W = pixel W-2 on the lane with p = W-4 (W is a multiple of 16, so
  // pixel W+1 never feeds a stored coefficient).
  auto reflect_fix = [&](uint32_t* w) {
    if (fixl) {
      w[0] = w[3];
      w[1] = __byte_perm(__byte_perm(w[4], w[2], 0x3270u), w[3], 0x5410u);
    }
    if (fixr) w[5] = __byte_perm(w[3], w[4], 0x0432u);
  };
  auto load_slot = [&](uint32_t qq, uint32_t* wo, uint32_t* we) {
    const uint32_t a = win0 + (qq % NST) * SEGB;
#pragma unroll
    for (int i = 0; i < 6; ++i) { wo[i] = lds32(a + 4 * i); we[i] = lds32(a + ROWB + 4 * i); }
    reflect_fix(wo);
    reflect_fix(we);
  };
  auto release = [&](uint32_t qq) {
    __syncwarp();
    if (lane == 0) bar_arrive_a(empty0 + 8u * (qq % NST));
  };
  auto wait_slot = [&](uint32_t qq) { bar_wait_a(full0 + 8u * (qq % NST), (qq / NST) & 1); };
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int N0, m0, b;
    tile_of(t, N0, m0, b);
    const int n0 = N0 + 64 * warp;
    const int na = n0 + 2 * lane;                  // the lane's columns na, na + 1
    const bool active = n0 < lg.pw;                // the tile may extend past the padded plane
    fixl = na == 0;
    fixr = 2 * na == NX - 4;
    // zero padding outside the true subband dims (container.py:132-145); `fullc` tiles need none.
    // Column masks per subband (both 16-bit halves), row masks per output row.
    const bool fullc = N0 + 64 * TW <= min(min(lg.sw[0], lg.sw[1]), min(lg.sw[2], lg.sw[3])) &&
                       m0 + sr <= min(min(lg.sh[0], lg.sh[1]), min(lg.sh[2], lg.sh[3]));
    uint32_t cm[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) cm[k] = (na < lg.sw[k] ? 0xFFFFu : 0u) | (na + 1 < lg.sw[k] ? 0xFFFF0000u : 0u);
    // slot 0: even row 2m0-2;  slot 1: rows 2m0-1, 2m0 -> high[m0-1]
    uint32_t eL[3], eH[3], vL[3], vH[3];  // previous even row (L, H parts), previous vertical highs
    uint32_t wo[6], we[6];
    wait_slot(q);
    load_slot(q, wo, we);
    {
      uint32_t t0[3], t1[3];
      rgb_hsplit(wo, t0, t1);  // (slot 0 has no odd row: result unused)
      rgb_hsplit(we, eL, eH);
    }
    release(q);  // after the words are consumed
    ++q;
    wait_slot(q);
    load_slot(q, wo, we);
    {
      uint32_t Lo[3], Ho[3], Le[3], He[3];
      rgb_hsplit(wo, Lo, Ho);
      rgb_hsplit(we, Le, He);
      release(q);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        vL[c] = swar_high(Lo[c], eL[c], Le[c]);
        vH[c] = swar_high(Ho[c], eH[c], He[c]);
        eL[c] = Le[c];
        eH[c] = He[c];
      }
    }
    ++q;
    wait_slot(q);
    load_slot(q, wo, we);
    // block max |c| trackers (only the bit length matters: bitplanes.py:77-79): packed signed
    // int16 max / min of the stored values
    uint32_t mxh[3], mnh[3], mxl[3], mnl[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) { mxh[c] = mxl[c] = mnh[c] = mnl[c] = 0u; }
    char* rp = (char*)P.coef + SZ * ((i64)b * g.img_stride + lg.off[0] + (i64)m0 * lg.pw + na);
    // the row loop, specialised on whether the tile needs zero padding
    auto rows = [&](auto padc) {
      constexpr bool PAD = decltype(padc)::value;
      for (int k = 2; k < nslots; ++k, ++q) {  // output row m = m0 + k - 2 from rows 2m+1 (odd), 2m+2 (even)
        const int m = m0 + k - 2;
        const bool nxt = k + 1 < nslots;
        // probe the next slot now; its wait (if any) happens after the math below
        const uint32_t ready = nxt ? bar_test_a(full0 + 8u * ((q + 1) % NST), ((q + 1) / NST) & 1) : 1u;
        uint32_t L1[3], H1[3], L2[3], H2[3];
        rgb_hsplit(wo, L1, H1);
        rgb_hsplit(we, L2, H2);
        release(q);
        uint32_t rm[4];
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2) rm[s2] = PAD ? (m < lg.sh[s2] ? cm[s2] : 0u) : 0xFFFFFFFFu;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const uint32_t vhL = swar_high(L1[c], eL[c], L2[c]);
          const uint32_t vlL = swar_low(eL[c], vL[c], vhL);
          const uint32_t vhH = swar_high(H1[c], eH[c], H2[c]);
          const uint32_t vlH = swar_low(eH[c], vH[c], vhH);
          eL[c] = L2[c]; vL[c] = vhL;
          eH[c] = H2[c]; vH[c] = vhH;
          // unbias to two int16 per word (per-field add of -SB)
          uint32_t ll = __vadd2(vlL, 0xC000C000u), lh = __vadd2(vhL, 0xC000C000u);
          uint32_t hl = __vadd2(vlH, 0xC000C000u), hh = __vadd2(vhH, 0xC000C000u);
          if constexpr (PAD) { ll &= rm[0]; lh &= rm[1]; hl &= rm[2]; hh &= rm[3]; }
          if (active) {
            char* qc = rp + c * cs;
            st_packed<CT>(qc, ll);
            st_packed<CT>(qc + o1, lh);
            st_packed<CT>(qc + o2, hl);
            st_packed<CT>(qc + o3, hh);
          }
          mxh[c] = __vmaxs2(mxh[c], __vmaxs2(lh, __vmaxs2(hl, hh)));
          mnh[c] = __vmins2(mnh[c], __vmins2(lh, __vmins2(hl, hh)));
          mxl[c] = __vmaxs2(mxl[c], ll);
          mnl[c] = __vmins2(mnl[c], ll);
        }
        rp += pitch;
        if (nxt) {
          if (!ready) wait_slot(q + 1);
          load_slot(q + 1, wo, we);
        }
      }
    };
    if (fullc) rows(std::false_type{});
    else rows(std::true_type{});
    if (active) {
      const int by = m0 / WB_DIM, bx = n0 / WB_DIM;
      // max |c| of the packed signed extremes (zero initialised: |.| >= 0)
      auto amax = [](uint32_t mx, uint32_t mn) {
        const int a = max(max((int)(int16_t)(mx & 0xFFFFu), (int)(int16_t)(mx >> 16)),
                          -min((int)(int16_t)(mn & 0xFFFFu), (int)(int16_t)(mn >> 16)));
        return (uint32_t)a;
      };
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const unsigned a = __reduce_max_sync(FULL, amax(mxh[c], mnh[c]));
        const unsigned l = __reduce_max_sync(FULL, amax(mxl[c], mnl[c]));
        if (lane == 0) {
          unsigned* bm = P.bmax + (i64)b * g.slots_per_image + (i64)c * g.slots_per_channel;
          atomicMax(&bm[lg.slot0 + by * lg.gw + bx], a);
          if (top) atomicMax(&bm[by * lg.gw + bx], l);
        }
      }
    }
  }
}

// ---- TMA-pipelined levels >= 2 on int16 planes -------------------------------------------------
// Same pipeline as k_fwd_rgb8_tma, for one channel's LL plane of the level below (int16, row pitch
// pg.pw): the producer warp streams row pairs into the ring with cp.async.bulk and patches the
// samples outside the plane row (already reflected); consumer lane k of warp w owns the two
// subband columns na = N0 + 64w + 2k, na + 1, i.e. input samples p = 2 na .. p + 3, and reads the
// window p-2 .. p+5 of both rows of a slot.  The horizontal split runs packed too: one word holds
// the same column of the slot's odd row (low field) and even row (high field), biased by 2^14, so
// each swar_high / swar_low lifts both rows at once; the results are re-paired by column for the
// vertical pass.  Host gate: lv[level].swar (every value of the level within +-8000), int16
// coefficients, plane width a multiple of 8 samples (16-byte row segments for the bulk copies).
constexpr int ROWB2 = 16 + 4 * 64 * TW + 16;   // staged row: samples [2 N0 - 8, 2 N0 + 128 TW + 8)
constexpr int SEGB2 = 2 * ROWB2;
#ifndef WBPC_FWD2_MINB
#define WBPC_FWD2_MINB 6
#endif

// bias two int16 fields by 2^14 each: x ^ 0x8000 is x + 2^15 per field, then subtract 2^14
// (no borrow: the fields are >= 2^14 for |x| < 2^14)
static __device__ __forceinline__ uint32_t swar_bias(uint32_t w) { return (w ^ 0x80008000u) - SB2; }

// wo / we: words (p-2,p-1) (p,p+1) (p+2,p+3) (p+4,p+5) of the slot's odd / even row.  Outputs per
// row the lane's two low and two high coefficients, packed by column and biased.
static __device__ __forceinline__ void i16_hsplit(const uint32_t* wo, const uint32_t* we, uint32_t& Lo, uint32_t& Ho,
                                                  uint32_t& Le, uint32_t& He) {
  uint32_t x[7];  // column p-2+i: (odd row, even row)
#pragma unroll
  for (int i = 0; i < 7; ++i) x[i] = swar_bias(__byte_perm(wo[i >> 1], we[i >> 1], (i & 1) ? 0x7632u : 0x5410u));
  const uint32_t hm1 = swar_high(x[1], x[0], x[2]);  // _split_axis0 (transforms.py:125,133)
  const uint32_t h0 = swar_high(x[3], x[2], x[4]);
  const uint32_t h1 = swar_high(x[5], x[4], x[6]);
  const uint32_t l0 = swar_low(x[2], hm1, h0);
  const uint32_t l1 = swar_low(x[4], h0, h1);
  Lo = __byte_perm(l0, l1, 0x5410u); Le = __byte_perm(l0, l1, 0x7632u);
  Ho = __byte_perm(h0, h1, 0x5410u); He = __byte_perm(h0, h1, 0x7632u);
}

__global__ void __launch_bounds__((TW + 1) * 32, WBPC_FWD2_MINB) k_fwd_i16_tma(FwdParams P, int tiles_x, int tiles_y, int ntiles) {
  __shared__ __align__(128) uint8_t ring[NST][SEGB2];
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  const Geom& g = P.g;
  const LevelGeom& lg = g.lv[P.level];
  const LevelGeom& pg = g.lv[P.level - 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sr = P.sr;
  const int NX = pg.w, NY = pg.h;
  const i64 rowbytes = 2 * (i64)NX;      // true row bytes (NX % 8 == 0)
  const i64 pitchb = 2 * (i64)pg.pw;     // source row pitch
  const int nslots = sr + 2;  // slot k: input rows 2m0-3+2k (odd; slot 0 leaves it out), 2m0-2+2k (even)
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) { bar_init(&full[i], 1); bar_init(&empty[i], TW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto tile_of = [&](int t, int& N0, int& m0, int& z) {
    N0 = (t % tiles_x) * (TW * 64);
    m0 = ((t / tiles_x) % tiles_y) * sr;
    z = t / (tiles_x * tiles_y);
  };
  auto plane_of = [&](int z) {  // (image, channel) z -> element offset of its coefficient area
    const int b = z / g.C, ch = z - b * g.C;
    return (i64)b * g.img_stride + (i64)ch * g.chan_stride;
  };
  if (warp == TW) {  // ---- producer warp
    uint32_t q = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int N0, m0, z;
      tile_of(t, N0, m0, z);
      const uint8_t* src = (const uint8_t*)(reinterpret_cast<const int16_t*>(P.coef) + plane_of(z) + pg.off[0]);
      const i64 s0 = 4 * (i64)N0 - 16;            // plane row byte of staged row byte 0
      const i64 c0 = s0 < 0 ? 0 : s0;
      const i64 c1 = s0 + ROWB2 < rowbytes ? s0 + ROWB2 : rowbytes;
      const uint32_t nb = c1 > c0 ? (uint32_t)(c1 - c0) : 0u;
      auto row_y = [&](int k, int h) { return reflect_pos(2 * m0 - 3 + 2 * k + h, NY); };
      for (int k = 0; k < nslots; ++k, ++q) {
        const int sl = q % NST;
        if (q >= NST) bar_wait(&empty[sl], ((q / NST) - 1) & 1);
        if (lane == 0) {
          bar_expect(&full[sl], (k == 0 ? 1u : 2u) * nb);
          if (nb)
            for (int h = (k == 0); h < 2; ++h)
              bulk_g2s(ring[sl] + h * ROWB2 + (c0 - s0), src + (i64)row_y(k, h) * pitchb + c0, nb, &full[sl]);
        }
      }
    }
    return;
  }
  // ---- consumers
  const uint32_t win0 = s_u32_keep(ring[0]) + 16 + 256 * warp + 8 * lane - 4;  // sample p-2
  const uint32_t full0 = s_u32_keep(full), empty0 = s_u32_keep(empty);
  const bool top = P.level == g.L;
  const i64 o1 = 2 * (lg.off[1] - lg.off[0]), o2 = 2 * (lg.off[2] - lg.off[0]), o3 = 2 * (lg.off[3] - lg.off[0]);
  const i64 pitch = 2 * (i64)lg.pw;
  uint32_t q = 0;
  bool fixl = false, fixr = false;  // per tile: the lane's window crosses the left / right row end
  auto load_slot = [&](uint32_t qq, uint32_t* wo, uint32_t* we) {
    const uint32_t a = win0 + (qq % NST) * SEGB2;
#pragma unroll
    for (int i = 0; i < 4; ++i) { wo[i] = lds32(a + 4 * i); we[i] = lds32(a + ROWB2 + 4 * i); }
    // whole-sample symmetric extension at the plane's row ends (transforms.py:117-133), from the
    // lane's own window: x[-2], x[-1] = x[2], x[1];  x[NX] = x[NX-2] (NX even; x[NX+1] is unused)
    if (fixl) { wo[0] = __byte_perm(wo[1], wo[2], 0x3254u); we[0] = __byte_perm(we[1], we[2], 0x3254u); }
    if (fixr) { wo[3] = wo[2]; we[3] = we[2]; }
  };
  auto release = [&](uint32_t qq) {
    __syncwarp();
    if (lane == 0) bar_arrive_a(empty0 + 8u * (qq % NST));
  };
  auto wait_slot = [&](uint32_t qq) { bar_wait_a(full0 + 8u * (qq % NST), (qq / NST) & 1); };
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int N0, m0, z;
    tile_of(t, N0, m0, z);
    const int n0 = N0 + 64 * warp;
    const int na = n0 + 2 * lane;
    const bool active = n0 < lg.pw;
    const bool fullc = N0 + 64 * TW <= min(min(lg.sw[0], lg.sw[1]), min(lg.sw[2], lg.sw[3])) &&
                       m0 + sr <= min(min(lg.sh[0], lg.sh[1]), min(lg.sh[2], lg.sh[3]));
    uint32_t cm[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) cm[k] = (na < lg.sw[k] ? 0xFFFFu : 0u) | (na + 1 < lg.sw[k] ? 0xFFFF0000u : 0u);
    fixl = na == 0;
    fixr = 2 * na == NX - 4;
    uint32_t eL, eH, vL, vH;  // previous even row (L, H parts), previous vertical highs
    uint32_t wo[4], we[4];
    wait_slot(q);
    load_slot(q, wo, we);
    {
      // slot 0 has no odd row: its (low) fields must still be in range, stale shared memory
      // there would carry into the even row's fields
      const uint32_t zero[4] = {0u, 0u, 0u, 0u};
      uint32_t t0, t1;
      i16_hsplit(zero, we, t0, t1, eL, eH);
    }
    release(q);
    ++q;
    wait_slot(q);
    load_slot(q, wo, we);
    {
      uint32_t Lo, Ho, Le, He;
      i16_hsplit(wo, we, Lo, Ho, Le, He);
      release(q);
      vL = swar_high(Lo, eL, Le);
      vH = swar_high(Ho, eH, He);
      eL = Le;
      eH = He;
    }
    ++q;
    wait_slot(q);
    load_slot(q, wo, we);
    uint32_t mxh = 0u, mnh = 0u, mxl = 0u, mnl = 0u;  // packed signed extremes of the stored values
    const i64 pl = plane_of(z);
    char* rp = (char*)P.coef + 2 * (pl + lg.off[0] + (i64)m0 * lg.pw + na);
    auto rows = [&](auto padc) {
      constexpr bool PAD = decltype(padc)::value;
      for (int k = 2; k < nslots; ++k, ++q) {  // output row m = m0 + k - 2
        const int m = m0 + k - 2;
        const bool nxt = k + 1 < nslots;
        const uint32_t ready = nxt ? bar_test_a(full0 + 8u * ((q + 1) % NST), ((q + 1) / NST) & 1) : 1u;
        uint32_t L1, H1, L2, H2;
        i16_hsplit(wo, we, L1, H1, L2, H2);
        release(q);
        const uint32_t vhL = swar_high(L1, eL, L2);
        const uint32_t vlL = swar_low(eL, vL, vhL);
        const uint32_t vhH = swar_high(H1, eH, H2);
        const uint32_t vlH = swar_low(eH, vH, vhH);
        eL = L2; vL = vhL;
        eH = H2; vH = vhH;
        uint32_t ll = __vadd2(vlL, 0xC000C000u), lh = __vadd2(vhL, 0xC000C000u);
        uint32_t hl = __vadd2(vlH, 0xC000C000u), hh = __vadd2(vhH, 0xC000C000u);
        if constexpr (PAD) {  // zero padding outside the true subband dims (container.py:132-145)
          ll &= m < lg.sh[0] ? cm[0] : 0u; lh &= m < lg.sh[1] ? cm[1] : 0u;
          hl &= m < lg.sh[2] ? cm[2] : 0u; hh &= m < lg.sh[3] ? cm[3] : 0u;
        }
        if (active) {
          *reinterpret_cast<uint32_t*>(rp) = ll;
          *reinterpret_cast<uint32_t*>(rp + o1) = lh;
          *reinterpret_cast<uint32_t*>(rp + o2) = hl;
          *reinterpret_cast<uint32_t*>(rp + o3) = hh;
        }
        mxh = __vmaxs2(mxh, __vmaxs2(lh, __vmaxs2(hl, hh)));
        mnh = __vmins2(mnh, __vmins2(lh, __vmins2(hl, hh)));
        mxl = __vmaxs2(mxl, ll);
        mnl = __vmins2(mnl, ll);
        rp += pitch;
        if (nxt) {
          if (!ready) wait_slot(q + 1);
          load_slot(q + 1, wo, we);
        }
      }
    };
    if (fullc) rows(std::false_type{});
    else rows(std::true_type{});
    if (active) {
      const int by = m0 / WB_DIM, bx = n0 / WB_DIM;
      auto amax = [](uint32_t mx, uint32_t mn) {
        const int a = max(max((int)(int16_t)(mx & 0xFFFFu), (int)(int16_t)(mx >> 16)),
                          -min((int)(int16_t)(mn & 0xFFFFu), (int)(int16_t)(mn >> 16)));
        return (uint32_t)a;
      };
      const unsigned a = __reduce_max_sync(FULL, amax(mxh, mnh));
      const unsigned l = __reduce_max_sync(FULL, amax(mxl, mnl));
      if (lane == 0) {
        const int b = z / g.C, ch = z - b * g.C;
        unsigned* bm = P.bmax + (i64)b * g.slots_per_image + (i64)ch * g.slots_per_channel;
        atomicMax(&bm[lg.slot0 + by * lg.gw + bx], a);
        if (top) atomicMax(&bm[by * lg.gw + bx], l);
      }
    }
  }
}

// grid: x = ceil(strips / WPB), z = batch (RCT) or batch*C
template <typename T, bool HWC, bool RCT, typename CT>
__global__ void __launch_bounds__(WPB * 32) k_fwd_l1(FwdParams P) {
  const Geom& g = P.g;
  const LevelGeom& lg = g.lv[1];
  const int sxn = lg.pw / 32;
  const int strip = blockIdx.x * WPB + (threadIdx.x >> 5);
  const int sx = strip % sxn, sy = strip / sxn;
  if (sy * P.sr >= lg.ph) return;
  const int b = RCT ? blockIdx.z : blockIdx.z / g.C;
  const int ch = RCT ? 0 : blockIdx.z % g.C;
  PixSrc<T, HWC> S{(const T*)((const char*)P.src + (i64)b * P.src_img_stride), g.W, g.H, g.C};
  if (P.fast_rgb8) {
    const int n0 = sx * 32;
    if (n0 >= 32 && 2 * n0 + 68 <= g.W) {  // interior strip: word loads never leave the row
      fwd_strip_rgb8<CT>(P, (const uint8_t*)S.p, b, n0, sy * P.sr, P.sr);
      return;
    }
  }
  if (RCT) fwd_strip<3, true, T, CT>(P, S, b, 0, sx * 32, sy * P.sr, P.sr);
  else fwd_strip<1, false, T, CT>(P, S, b, ch, sx * 32, sy * P.sr, P.sr);
}


// Levels >= 2: the LL plane of the level below -> the four subbands of this level.  CTA = one
// 32 x 32 subband tile of one channel: the 67 x 67 input window (64 x 64 samples + the lifting
// halo, reflected at the plane edges) is loaded into shared memory with every load in flight at
// once, then the 5/3 split runs in parallel phases -- row highs, row lows, column highs, column
// lows -- so the kernel is bound by memory, not by a per-row dependency chain.
constexpr int FT = 32;              // output tile (subband coefficients per side)
constexpr int FI = 2 * FT + 3;      // input window per side: samples 2n0-2 .. 2n0+2FT
template <typename CT>
__global__ void __launch_bounds__(256) k_fwd_tile(FwdParams P) {
  constexpr int NE = FT + 2, NO = FT + 1;  // even / odd window columns (local 2k / 2k+1)
  __shared__ int Xe[FI][NE], Xo[FI][NO];  // input window, de-interleaved by column parity
  __shared__ int Lr[FI][FT], Hr[FI][FT];  // row lows / highs (columns n0 .. n0+FT-1)
  __shared__ unsigned red[2];
  const Geom& g = P.g;
  const LevelGeom& lg = g.lv[P.level];
  const LevelGeom& pg = g.lv[P.level - 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = blockIdx.x * FT, m0 = blockIdx.y * FT;
  const int b = blockIdx.z / g.C, ch = blockIdx.z % g.C;
  const int NX = pg.w, NY = pg.h;
  const i64 cbase = (i64)b * g.img_stride + (i64)ch * g.chan_stride;
  const CT* src = reinterpret_cast<const CT*>(P.coef) + cbase + pg.off[0];
  if (tid < 2) red[tid] = 0;
  // 1. window load (whole-sample symmetric extension, transforms.py:117-133).  Every load of a
  // thread is issued before any is consumed (unrolled into registers): warp w takes window rows
  // w, w+8, ...; interior-column tiles read each (even, odd) sample pair as one word per lane.
  constexpr int RPW = (FI + 7) / 8;  // window rows per warp
  {
    const bool colin = 2 * n0 - 2 >= 0 && 2 * n0 - 2 + FI + 1 <= NX;  // CTA-uniform
    if (colin) {  // 68 samples per row = 34 pairs: lanes 0..31 + lanes 0..1 again
      using P2 = typename std::conditional<sizeof(CT) == 2, uint32_t, int2>::type;
      P2 v[RPW][2];
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr) {
        const int r = warp + 8 * rr;
        const P2* rowp = reinterpret_cast<const P2*>(src + (i64)reflect_pos(2 * m0 - 2 + min(r, FI - 1), NY) * pg.pw +
                                                     (2 * n0 - 2));
        v[rr][0] = rowp[lane];
        v[rr][1] = lane < 2 ? rowp[32 + lane] : v[rr][0];
      }
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr) {
        const int r = warp + 8 * rr;
        if (r < FI) {
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int w = lane + 32 * k;
            if (k == 0 || lane < 2) {
              int a, bb;
              if constexpr (sizeof(CT) == 2) {
                a = (int)(int16_t)(v[rr][k] & 0xFFFFu);
                bb = (int)(int16_t)(v[rr][k] >> 16);
              } else {
                a = v[rr][k].x;
                bb = v[rr][k].y;
              }
              Xe[r][w] = a;
              if (w < NO) Xo[r][w] = bb;
            }
          }
        }
      }
    } else {  // plane-edge tiles: reflected columns, one sample per load
      int xs[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) xs[k] = reflect_pos(2 * n0 - 2 + min(lane + 32 * k, FI - 1), NX);
      int v[RPW][3];
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr) {
        const int r = warp + 8 * rr;
        const CT* rowp = src + (i64)reflect_pos(2 * m0 - 2 + min(r, FI - 1), NY) * pg.pw;
#pragma unroll
        for (int k = 0; k < 3; ++k) v[rr][k] = (int)rowp[xs[k]];
      }
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr) {
        const int r = warp + 8 * rr;
        if (r < FI) {
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const int c = lane + 32 * k;
            if (c < FI) {
              if (c & 1) Xo[r][c >> 1] = v[rr][k];
              else Xe[r][c >> 1] = v[rr][k];
            }
          }
        }
      }
    }
  }
  __syncthreads();
  // 2. horizontal split of every window row (transforms.py:125,133): warp per row, lane j owns
  // column n0+j: h_{j-1} and h_j (even column 2j+2 sits at Xe[j+1]) then l_j
#pragma unroll
  for (int rr = 0; rr < RPW; ++rr) {
    const int r = warp + 8 * rr;
    if (r < FI) {
      const int e0 = Xe[r][lane], e1 = Xe[r][lane + 1], e2 = Xe[r][lane + 2];
      const int hA = Xo[r][lane] - ((e0 + e1) >> 1);
      const int hB = Xo[r][lane + 1] - ((e1 + e2) >> 1);
      Hr[r][lane] = hB;
      Lr[r][lane] = e1 + ((hA + hB + 2) >> 2);
    }
  }
  __syncthreads();
  // 3. vertical split of the 2FT columns (Lr: LL/LH, Hr: HL/HH) and the outputs.  Thread = one
  // column x 8 consecutive output rows i (input rows 2i .. 2i+4 of the window), sliding down.
  const int col = tid & 63, grp = tid >> 6;  // warps 0,2,4,6: Lr columns; 1,3,5,7: Hr columns
  const bool hcol = col >= FT;
  const int cj = hcol ? col - FT : col;
  int (*A)[FT] = hcol ? Hr : Lr;
  const int n = n0 + cj;
  const int kl = hcol ? 2 : 0, kh = hcol ? 3 : 1;  // subband index of the low / high output
  const bool cl = n < lg.sw[kl], chh = n < lg.sw[kh];
  CT* dl = reinterpret_cast<CT*>(P.coef) + cbase + lg.off[kl] + n;
  CT* dh = reinterpret_cast<CT*>(P.coef) + cbase + lg.off[kh] + n;
  unsigned mh = 0, ml = 0;  // OR of |c| (only the bit length matters: bitplanes.py:77-79)
  const int i0 = 8 * grp;
  int a0 = A[2 * i0][cj], a1 = A[2 * i0 + 1][cj], a2 = A[2 * i0 + 2][cj];
  int vprev = a1 - ((a0 + a2) >> 1);  // vertical high of output row i0-1
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = i0 + k, m = m0 + i;
    const int a3 = A[2 * i + 3][cj], a4 = A[2 * i + 4][cj];
    const int vh = a3 - ((a2 + a4) >> 1);
    const int vl = a2 + ((vprev + vh + 2) >> 2);
    const int lo = (cl && m < lg.sh[kl]) ? vl : 0;  // zero padding (container.py:132-145)
    const int hi = (chh && m < lg.sh[kh]) ? vh : 0;
    dl[(i64)m * lg.pw] = (CT)lo;
    dh[(i64)m * lg.pw] = (CT)hi;
    mh |= (unsigned)abs(hi) | (hcol ? (unsigned)abs(lo) : 0u);
    ml |= hcol ? 0u : (unsigned)abs(lo);
    vprev = vh;
    a2 = a4;
  }
  mh = __reduce_or_sync(FULL, mh);
  ml = __reduce_or_sync(FULL, ml);
  if (lane == 0) {
    atomicOr(&red[0], mh);
    atomicOr(&red[1], ml);
  }
  __syncthreads();
  if (tid == 0) {
    const int by = m0 / WB_DIM, bx = n0 / WB_DIM;
    unsigned* bm = P.bmax + (i64)b * g.slots_per_image + (i64)ch * g.slots_per_channel;
    atomicMax(&bm[lg.slot0 + by * lg.gw + bx], red[0]);
    if (P.level == g.L) atomicMax(&bm[by * lg.gw + bx], red[1]);
  }
}

// L == 0: the LL grid is the (colour transformed) image itself, zero padded to 128 multiples.
template <typename T>
static __device__ __forceinline__ int ld_any(const void* base, int dt, i64 idx) {
  switch (dt) {
    case WBPC_DTYPE_U8: return ((const uint8_t*)base)[idx];
    case WBPC_DTYPE_U16: return ((const uint16_t*)base)[idx];
    case WBPC_DTYPE_I16: return ((const int16_t*)base)[idx];
    default: return ((const int32_t*)base)[idx];
  }
}

template <typename CT>
__global__ void __launch_bounds__(256) k_level0(FwdParams P) {
  const Geom& g = P.g;
  const LevelGeom& lg = g.lv[0];
  const int b = blockIdx.z;
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
  const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
  __shared__ unsigned red[4][8];
  unsigned m[4] = {0, 0, 0, 0};
  const bool in = x < g.W && y < g.H;
  int v[4] = {0, 0, 0, 0};
  if (in) {
    const int lim = 1 << g.bd;
    bool bad = false;
    const char* base = (const char*)P.src + (i64)b * P.src_img_stride;
    for (int ch = 0; ch < g.C; ++ch) {
      i64 idx = P.src_layout == WBPC_LAYOUT_HWC ? ((i64)y * g.W + x) * g.C + ch : ((i64)ch * g.H + y) * g.W + x;
      v[ch] = ld_any<int>(base, P.src_dtype, idx);
      bad |= (unsigned)v[ch] >= (unsigned)lim;
    }
    if (bad) record_error(P.st, WBPC_ERR_DOMAIN, 0, 0);
    if (g.rct) {
      int R = v[0], G = v[1], B = v[2];
      v[0] = (R + 2 * G + B) >> 2;
      v[1] = B - G;
      v[2] = R - G;
    }
  }
  const i64 img0 = (i64)b * g.img_stride;
  for (int ch = 0; ch < g.C; ++ch) {
    stc<CT>(P, img0 + (i64)ch * g.chan_stride + lg.off[0] + (i64)y * lg.pw + x, v[ch]);
    m[ch] = (unsigned)abs(v[ch]);
  }
  for (int ch = 0; ch < 4; ++ch)
    for (int o = 16; o > 0; o >>= 1) m[ch] = max(m[ch], __shfl_xor_sync(FULL, m[ch], o));
  if ((threadIdx.x & 31) == 0)
    for (int ch = 0; ch < 4; ++ch) red[ch][threadIdx.x >> 5] = m[ch];
  __syncthreads();
  if (threadIdx.x < g.C) {
    unsigned a = 0;
    for (int w = 0; w < 8; ++w) a = max(a, red[threadIdx.x][w]);
    unsigned* bm = P.bmax + (i64)b * g.slots_per_image + (i64)threadIdx.x * g.slots_per_channel;
    atomicMax(&bm[(y / WB_DIM) * lg.gw + x / WB_DIM], a);
  }
}

// ---------------------------------------------------------------------------- inverse
struct InvParams {
  Geom g;
  int level;           // merging level l (LL_l + details_l -> LL_{l-1})
  int32_t* coef;
  void* out;           // final output (fused last level / finish), else null
  int out_dtype, out_layout;
  i64 out_img_stride;  // bytes
  int out_channels;    // channels written (3 for RCT containers claiming 4)
  int sr;              // strip height (subband rows)
  int ox, oy, ow, oh;  // output window (decode_region crop); full image by default
  const u64* hpdepth;  // max detail-block depth of the decode (DevStatus::pad)
  int allow16;         // detail planes may hold int16 (see k_block_reconstruct)
};

// Detail-plane element type of this decode: int16 when every decoded detail block has depth <= 16
// (set on the device by the header pass).  Both instantiations are launched; the other returns.
template <typename HT>
__device__ __forceinline__ bool inv_variant_active(const InvParams& P) {
  const bool d16 = P.allow16 && *P.hpdepth <= 16;
  return (sizeof(HT) == 2) == d16;
}

static __device__ __forceinline__ void store_sample(void* base, int dtype, i64 idx, int v, int bd) {
  switch (dtype) {
    case WBPC_DTYPE_U8_DISPLAY: {  // clip + 8-bit display scale (service.py:72-78)
      const int maxval = (1 << bd) - 1;
      v = v < 0 ? 0 : (v > maxval ? maxval : v);
      if (bd > 8) v = (v * 255 + maxval / 2) / maxval;
      ((uint8_t*)base)[idx] = (uint8_t)v;
      break;
    }
    case WBPC_DTYPE_U8: ((uint8_t*)base)[idx] = (uint8_t)v; break;
    case WBPC_DTYPE_U16: ((uint16_t*)base)[idx] = (uint16_t)v; break;
    case WBPC_DTYPE_I16: ((int16_t*)base)[idx] = (int16_t)v; break;
    default: ((int32_t*)base)[idx] = v; break;
  }
}

// Reflected subband index of position 2k+h of a length-N signal (transforms.py:145-158).
static __device__ __forceinline__ int sb_idx(int k, int h, int N) { return reflect_pos(2 * k + h, N) >> 1; }

// Final-level output of one parent pixel pair (px0, px0+1) of row py.  WIN = crop window
// (decode_region); the full-image instantiation keeps only the image-bounds checks.
template <int NC, bool WIN>
static __device__ __forceinline__ void store_final(const InvParams& P, int b, int py, int px0, int NX, int NY,
                                                   bool out_lane, const int* ve, const int* vo) {
  const int ox = WIN ? P.ox : 0, oy = WIN ? P.oy : 0;
  const int ow = WIN ? P.ow : NX, oh = WIN ? P.oh : NY;
  bool rowok = out_lane && py < NY;
  if (WIN) rowok = rowok && py >= oy && py < oy + oh;
  if (!rowok) return;
  const int OC = P.out_channels;
  char* ob = (char*)P.out + (i64)b * P.out_img_stride;
  const int qy = py - oy;
  bool in0 = px0 < NX, in1 = px0 + 1 < NX;
  if (WIN) {
    in0 = in0 && px0 >= ox && px0 < ox + ow;
    in1 = in1 && px0 + 1 >= ox && px0 + 1 < ox + ow;
  }
  const int qx = px0 - ox;
  const i64 pix = (i64)qy * ow + qx;
  if (in0 && in1 && P.out_layout == WBPC_LAYOUT_HWC && P.out_dtype == WBPC_DTYPE_U8 && OC == 3 &&
      (((unsigned)qy * (unsigned)ow + (unsigned)qx) & 1u) == 0) {
    // 2 RGB pixels = 6 bytes at an even offset: three 16-bit stores
    uint16_t* q = reinterpret_cast<uint16_t*>(ob + pix * 3);
    q[0] = (uint16_t)((ve[0] & 255) | ((ve[1] & 255) << 8));
    q[1] = (uint16_t)((ve[2] & 255) | ((vo[0] & 255) << 8));
    q[2] = (uint16_t)((vo[1] & 255) | ((vo[2] & 255) << 8));
  } else if (in0 || in1) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (c >= OC) break;
      const i64 i0 = P.out_layout == WBPC_LAYOUT_HWC ? pix * OC + c : ((i64)c * oh + qy) * ow + qx;
      if (in0) store_sample(ob, P.out_dtype, i0, ve[c], P.g.bd);
      if (in1) store_sample(ob, P.out_dtype, i0 + (P.out_layout == WBPC_LAYOUT_HWC ? OC : 1), vo[c], P.g.bd);
    }
  }
}

// Lanes 0..31 own subband columns n0-1 .. n0+30; lanes 1..30 produce parent columns 2n, 2n+1.
// NC channels per warp (all channels for the fused final level, else 1).  The next row pair's
// 4*NC loads are issued before the current pair is lifted (one iteration of prefetch).
template <int NC, bool FINAL, bool WIN, typename HT>
static __device__ void inv_strip(const InvParams& P, int b, int ch0, int n0, int m0, int sr) {
  const Geom& g = P.g;
  const int lev = P.level;
  const LevelGeom& lg = g.lv[lev];
  const LevelGeom& pg = g.lv[lev - 1];
  const int lane = threadIdx.x & 31;
  const int NX = pg.w, NY = pg.h;
  const int n = n0 - 1 + lane;
  const int32_t* img_coef = P.coef + (i64)b * g.img_stride;
  const int pitch = lg.pw;
  // per-lane column index of the low (LL, LH) and high (HL, HH) subbands; empty high band -> 0
  const int cl = sb_idx(n, 0, NX);
  const int chh = NX == 1 ? 0 : sb_idx(n, 1, NX);
  const bool hx_empty = NX == 1, hy_empty = NY == 1;
  const int32_t* base[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) base[c] = img_coef + (i64)(ch0 + c) * g.chan_stride;
  // detail-plane offsets in HT elements from the channel base (plane starts are int32 offsets)
  constexpr i64 PW = (i64)(sizeof(int32_t) / sizeof(HT));
  const i64 offLL = lg.off[0] + cl, offLH = PW * lg.off[1] + cl, offHL = PW * lg.off[2] + chh,
            offHH = PW * lg.off[3] + chh;
  // loads of subband row pair (low row k, high row k) for all channels
  auto load4 = [&](int k, int* vLL, int* vLH, int* vHL, int* vHH) {
    const i64 rl = (i64)sb_idx(k, 0, NY) * pitch;
    const i64 rh = hy_empty ? 0 : (i64)sb_idx(k, 1, NY) * pitch;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      vLL[c] = __ldg(base[c] + offLL + rl);
      const HT* hb = reinterpret_cast<const HT*>(base[c]);
      vLH[c] = hy_empty ? 0 : (int)__ldg(hb + offLH + rh);
      vHL[c] = hx_empty ? 0 : (int)__ldg(hb + offHL + rl);
      vHH[c] = (hx_empty || hy_empty) ? 0 : (int)__ldg(hb + offHH + rh);
    }
  };
  int xeL[NC], hL[NC], xeH[NC], hH[NC];
  {
    int aLL[NC], aLH[NC], aHL[NC], aHH[NC], bLL[NC], bLH[NC], bHL[NC], bHH[NC];
    load4(m0 - 1, aLL, aLH, aHL, aHH);
    load4(m0, bLL, bLH, bHL, bHH);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      hL[c] = bLH[c];
      xeL[c] = bLL[c] - ((aLH[c] + hL[c] + 2) >> 2);
      hH[c] = bHH[c];
      xeH[c] = bHL[c] - ((aHH[c] + hH[c] + 2) >> 2);
    }
  }
  if constexpr (NC == 1) {
  const bool out_lane = lane >= 1 && lane <= 30;
  const int px0 = 2 * n;
  // output row pair m consumes subband row m+1; two buffers (unrolled by two) keep the loads of
  // the next two row pairs in flight without register moves
  auto merge_rows = [&](int m, const int* cLL, const int* cLH, const int* cHL, const int* cHH) {
    int lx[2][NC], hx[2][NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int hL1 = cLH[c];
      const int xeL1 = cLL[c] - ((hL[c] + hL1 + 2) >> 2);
      lx[0][c] = xeL[c];
      lx[1][c] = hL[c] + ((xeL[c] + xeL1) >> 1);
      xeL[c] = xeL1; hL[c] = hL1;
      const int hH1 = cHH[c];
      const int xeH1 = cHL[c] - ((hH[c] + hH1 + 2) >> 2);
      hx[0][c] = xeH[c];
      hx[1][c] = hH[c] + ((xeH[c] + xeH1) >> 1);
      xeH[c] = xeH1; hH[c] = hH1;
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int py = 2 * m + r;
      int ve[4], vo[4];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int hl = __shfl_up_sync(FULL, hx[r][c], 1);
        const int xe = lx[r][c] - ((hl + hx[r][c] + 2) >> 2);
        const int xr = __shfl_down_sync(FULL, xe, 1);
        ve[c] = xe;
        vo[c] = hx[r][c] + ((xe + xr) >> 1);
      }
      if (!FINAL) {
        if (out_lane && py < pg.ph && px0 < pg.pw) {
          int32_t* dst = P.coef + (i64)b * g.img_stride + (i64)ch0 * g.chan_stride + pg.off[0] + (i64)py * pg.pw + px0;
          *reinterpret_cast<int2*>(dst) = make_int2(ve[0], vo[0]);
        }
      } else {
        if (g.rct) {  // rct_inverse (transforms.py:101-103), no clamp (container.py:313-316)
          int G = ve[0] - ((ve[1] + ve[2]) >> 2);
          int R = ve[2] + G, B = ve[1] + G;
          ve[0] = R; ve[1] = G; ve[2] = B;
          G = vo[0] - ((vo[1] + vo[2]) >> 2);
          R = vo[2] + G; B = vo[1] + G;
          vo[0] = R; vo[1] = G; vo[2] = B;
        }
        store_final<NC, WIN>(P, b, py, px0, NX, NY, out_lane, ve, vo);
      }
    }
  };
  int aLL[NC], aLH[NC], aHL[NC], aHH[NC], bLL[NC], bLH[NC], bHL[NC], bHH[NC];
  load4(m0 + 1, aLL, aLH, aHL, aHH);
  if (sr > 1) load4(m0 + 2, bLL, bLH, bHL, bHH);
  for (int m = m0; m < m0 + sr; m += 2) {
    merge_rows(m, aLL, aLH, aHL, aHH);
    if (m + 2 < m0 + sr) load4(m + 3, aLL, aLH, aHL, aHH);
    if (m + 1 >= m0 + sr) break;
    merge_rows(m + 1, bLL, bLH, bHL, bHH);
    if (m + 3 < m0 + sr) load4(m + 4, bLL, bLH, bHL, bHH);
  }
  } else {
  int nLL[NC], nLH[NC], nHL[NC], nHH[NC];
  load4(m0 + 1, nLL, nLH, nHL, nHH);
  const bool out_lane = lane >= 1 && lane <= 30;
  const int px0 = 2 * n;
  // 8-bit interleaved RGB output of a whole even-width image: the lane's two pixels of every row
  // are three 16-bit words at a fixed offset from the row start (row pointer hoisted; the general
  // store_final handles every other case)
  const bool rgb8 = FINAL && !WIN && NC == 3 && P.out_dtype == WBPC_DTYPE_U8 && P.out_layout == WBPC_LAYOUT_HWC &&
                    P.out_channels == 3 && (NX & 1) == 0;
  const bool rgb8_lane = rgb8 && out_lane && px0 + 1 < NX;
  char* const orow0 = FINAL ? (char*)P.out + (i64)b * P.out_img_stride + (i64)px0 * 3 : nullptr;
  const i64 rowbytes = (i64)NX * 3;
  for (int m = m0; m < m0 + sr; ++m) {
    int cLL[NC], cLH[NC], cHL[NC], cHH[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) { cLL[c] = nLL[c]; cLH[c] = nLH[c]; cHL[c] = nHL[c]; cHH[c] = nHH[c]; }
    if (m + 1 < m0 + sr) load4(m + 2, nLL, nLH, nHL, nHH);  // prefetch the next pair
    int lx[2][NC], hx[2][NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int hL1 = cLH[c];
      const int xeL1 = cLL[c] - ((hL[c] + hL1 + 2) >> 2);
      lx[0][c] = xeL[c];
      lx[1][c] = hL[c] + ((xeL[c] + xeL1) >> 1);
      xeL[c] = xeL1; hL[c] = hL1;
      const int hH1 = cHH[c];
      const int xeH1 = cHL[c] - ((hH[c] + hH1 + 2) >> 2);
      hx[0][c] = xeH[c];
      hx[1][c] = hH[c] + ((xeH[c] + xeH1) >> 1);
      xeH[c] = xeH1; hH[c] = hH1;
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int py = 2 * m + r;
      int ve[4], vo[4];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int hl = __shfl_up_sync(FULL, hx[r][c], 1);
        const int xe = lx[r][c] - ((hl + hx[r][c] + 2) >> 2);
        const int xr = __shfl_down_sync(FULL, xe, 1);
        ve[c] = xe;
        vo[c] = hx[r][c] + ((xe + xr) >> 1);
      }
      if (!FINAL) {
        if (out_lane && py < pg.ph && px0 < pg.pw) {
          int32_t* dst = P.coef + (i64)b * g.img_stride + (i64)ch0 * g.chan_stride + pg.off[0] + (i64)py * pg.pw + px0;
          *reinterpret_cast<int2*>(dst) = make_int2(ve[0], vo[0]);
        }
      } else {
        if (g.rct) {  // rct_inverse (transforms.py:101-103), no clamp (container.py:313-316)
          int G = ve[0] - ((ve[1] + ve[2]) >> 2);
          int R = ve[2] + G, B = ve[1] + G;
          ve[0] = R; ve[1] = G; ve[2] = B;
          G = vo[0] - ((vo[1] + vo[2]) >> 2);
          R = vo[2] + G; B = vo[1] + G;
          vo[0] = R; vo[1] = G; vo[2] = B;
        }
        if (rgb8) {
          if (rgb8_lane && py < NY) {
            uint16_t* q = reinterpret_cast<uint16_t*>(orow0 + (i64)py * rowbytes);
            q[0] = (uint16_t)((ve[0] & 255) | ((ve[1] & 255) << 8));
            q[1] = (uint16_t)((ve[2] & 255) | ((vo[0] & 255) << 8));
            q[2] = (uint16_t)((vo[1] & 255) | ((vo[2] & 255) << 8));
          }
        } else {
          store_final<NC, WIN>(P, b, py, px0, NX, NY, out_lane, ve, vo);
        }
      }
    }
  }
  }
}

// Two subband columns per lane (int16 detail planes, whole-image output): lanes 0..31 own the
// column pairs (n0-2+2l, n0-1+2l), lanes 1..30 produce the parent columns 4 per lane -- every
// subband row is read as one word per lane and plane (the int32 LL pair as 8 bytes), the merged
// rows leave as one 16-byte store (intermediate levels) or as the 12 bytes of four RGB pixels
// (final level), and a row needs two shuffles per channel for 60 subband columns instead of 30.
// Only strips that touch no plane edge take this path (no column reflection, both columns of a
// pair adjacent in memory); edge strips run inv_strip on their two 30-column halves.
template <int NC, bool FINAL>
static __device__ void inv_strip2(const InvParams& P, int b, int ch0, int n0, int m0, int sr) {
  const Geom& g = P.g;
  const LevelGeom& lg = g.lv[P.level];
  const LevelGeom& pg = g.lv[P.level - 1];
  const int lane = threadIdx.x & 31;
  const int NX = pg.w, NY = pg.h;
  const int n = n0 - 2 + 2 * lane;  // the lane's columns n, n + 1
  const int pitch = lg.pw;
  const int32_t* base[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) base[c] = P.coef + (i64)b * g.img_stride + (i64)(ch0 + c) * g.chan_stride;
  // plane offsets: LL in int32 elements, details in int16 elements (plane starts are int32 offsets)
  const i64 offLL = lg.off[0] + n, offLH = 2 * lg.off[1] + n, offHL = 2 * lg.off[2] + n, offHH = 2 * lg.off[3] + n;
  struct Raw { int2 ll[NC]; uint32_t lh[NC], hl[NC], hh[NC]; };
  auto load4 = [&](int k, Raw& R) {  // subband row pair (low row k, high row k), mirrored at the ends
    const i64 rl = (i64)sb_idx(k, 0, NY) * pitch;
    const i64 rh = (i64)sb_idx(k, 1, NY) * pitch;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int16_t* hb = reinterpret_cast<const int16_t*>(base[c]);
      R.ll[c] = __ldg(reinterpret_cast<const int2*>(base[c] + offLL + rl));
      R.lh[c] = __ldg(reinterpret_cast<const uint32_t*>(hb + offLH + rh));
      R.hl[c] = __ldg(reinterpret_cast<const uint32_t*>(hb + offHL + rl));
      R.hh[c] = __ldg(reinterpret_cast<const uint32_t*>(hb + offHH + rh));
    }
  };
  auto lo16 = [](uint32_t w) { return (int)(int16_t)(w & 0xFFFFu); };
  auto hi16 = [](uint32_t w) { return (int)w >> 16; };
  // vertical state per channel and column: previous even row / previous high of the L and H halves
  int xeL[NC][2], hL[NC][2], xeH[NC][2], hH[NC][2];
  {
    Raw A, B;
    load4(m0 - 1, A);
    load4(m0, B);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int aLH[2] = {lo16(A.lh[c]), hi16(A.lh[c])}, aHH[2] = {lo16(A.hh[c]), hi16(A.hh[c])};
      const int bLL[2] = {B.ll[c].x, B.ll[c].y}, bLH[2] = {lo16(B.lh[c]), hi16(B.lh[c])};
      const int bHL[2] = {lo16(B.hl[c]), hi16(B.hl[c])}, bHH[2] = {lo16(B.hh[c]), hi16(B.hh[c])};
#pragma unroll
      for (int j = 0; j < 2; ++j) {  // _merge_axis0 on columns (transforms.py:137-162)
        hL[c][j] = bLH[j];
        xeL[c][j] = bLL[j] - ((aLH[j] + hL[c][j] + 2) >> 2);
        hH[c][j] = bHH[j];
        xeH[c][j] = bHL[j] - ((aHH[j] + hH[c][j] + 2) >> 2);
      }
    }
  }
  const bool out_lane = lane >= 1 && lane <= 30;
  const int px0 = 2 * n;  // parent columns px0 .. px0 + 3
  char* const orow0 = FINAL ? (char*)P.out + (i64)b * P.out_img_stride + (i64)px0 * 3 : nullptr;
  const i64 rowbytes = (i64)NX * 3;
  int32_t* const drow0 = FINAL ? nullptr : P.coef + (i64)b * g.img_stride + (i64)ch0 * g.chan_stride + pg.off[0] + px0;
  // output row pair m consumes subband row m+1; two buffers (the loop unrolled by two) keep the
  // loads of the next two row pairs in flight
  auto merge_rows = [&](int m, const Raw& cur) {
    int lx[2][NC][2], hx[2][NC][2];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int cLL[2] = {cur.ll[c].x, cur.ll[c].y}, cLH[2] = {lo16(cur.lh[c]), hi16(cur.lh[c])};
      const int cHL[2] = {lo16(cur.hl[c]), hi16(cur.hl[c])}, cHH[2] = {lo16(cur.hh[c]), hi16(cur.hh[c])};
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int hL1 = cLH[j];
        const int xeL1 = cLL[j] - ((hL[c][j] + hL1 + 2) >> 2);
        lx[0][c][j] = xeL[c][j];
        lx[1][c][j] = hL[c][j] + ((xeL[c][j] + xeL1) >> 1);
        xeL[c][j] = xeL1; hL[c][j] = hL1;
        const int hH1 = cHH[j];
        const int xeH1 = cHL[j] - ((hH[c][j] + hH1 + 2) >> 2);
        hx[0][c][j] = xeH[c][j];
        hx[1][c][j] = hH[c][j] + ((xeH[c][j] + xeH1) >> 1);
        xeH[c][j] = xeH1; hH[c][j] = hH1;
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int py = 2 * m + r;
      int v[4][NC];  // parent pixels px0 .. px0+3
#pragma unroll
      for (int c = 0; c < NC; ++c) {  // _merge_axis0 on rows: even samples, then odd ones
        const int hprev = __shfl_up_sync(FULL, hx[r][c][1], 1);
        const int xe0 = lx[r][c][0] - ((hprev + hx[r][c][0] + 2) >> 2);
        const int xe1 = lx[r][c][1] - ((hx[r][c][0] + hx[r][c][1] + 2) >> 2);
        const int xnext = __shfl_down_sync(FULL, xe0, 1);
        v[0][c] = xe0;
        v[1][c] = hx[r][c][0] + ((xe0 + xe1) >> 1);
        v[2][c] = xe1;
        v[3][c] = hx[r][c][1] + ((xe1 + xnext) >> 1);
      }
      if constexpr (!FINAL) {
        if (out_lane && py < pg.ph)
          *reinterpret_cast<int4*>(drow0 + (i64)py * pg.pw) = make_int4(v[0][0], v[1][0], v[2][0], v[3][0]);
      } else {
        // rct_inverse (transforms.py:101-103), 8-bit interleaved RGB: four pixels = three words
        uint32_t px[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int G = v[i][0] - ((v[i][1] + v[i][2]) >> 2);
          const int R = v[i][2] + G, B = v[i][1] + G;
          px[i] = (uint32_t)(R & 255) | ((uint32_t)(G & 255) << 8) | ((uint32_t)(B & 255) << 16);
        }
        if (out_lane && py < NY) {
          uint32_t* q = reinterpret_cast<uint32_t*>(orow0 + (i64)py * rowbytes);
          q[0] = px[0] | (px[1] << 24);
          q[1] = (px[1] >> 8) | (px[2] << 16);
          q[2] = (px[2] >> 16) | (px[3] << 8);
        }
      }
    }
  };
  Raw ra, rb;
  load4(m0 + 1, ra);
  if (sr > 1) load4(m0 + 2, rb);
  for (int m = m0; m < m0 + sr; m += 2) {
    merge_rows(m, ra);
    if (m + 2 < m0 + sr) load4(m + 3, ra);
    if (m + 1 >= m0 + sr) break;
    merge_rows(m + 1, rb);
    if (m + 3 < m0 + sr) load4(m + 4, rb);
  }
}

// grid.x covers 60-column strips; a strip away from the plane edges runs inv_strip2, an edge
// strip the reflecting one-column-per-lane inv_strip on its two halves.
template <int NC, bool FINAL>
__global__ void __launch_bounds__(WPB * 32) k_inv2(InvParams P) {
  const Geom& g = P.g;
  const LevelGeom& lg = g.lv[P.level];
  const int sxn = (lg.w + 59) / 60;
  const int syn = (lg.h + P.sr - 1) / P.sr;
  const int strip = blockIdx.x * WPB + (threadIdx.x >> 5);
  if (strip >= sxn * syn) return;
  const int sx = strip % sxn, sy = strip / sxn;
  const int b = FINAL ? blockIdx.z : blockIdx.z / g.C;
  const int ch = FINAL ? 0 : blockIdx.z % g.C;
  const int n0 = sx * 60, m0 = sy * P.sr;
  const bool v16 = inv_variant_active<int16_t>(P);  // detail planes hold int16 in this decode
  auto halves = [&](int nn0) {
    if (v16) inv_strip<NC, FINAL, false, int16_t>(P, b, ch, nn0, m0, P.sr);
    else inv_strip<NC, FINAL, false, int32_t>(P, b, ch, nn0, m0, P.sr);
  };
  if (v16 && n0 >= 2 && n0 + 62 <= min(lg.sw[2], lg.sw[0])) {
    inv_strip2<NC, FINAL>(P, b, ch, n0, m0, P.sr);
  } else {
    halves(n0);
    if (n0 + 30 < lg.w) halves(n0 + 30);
  }
}

template <int NC, bool FINAL, bool WIN>
__global__ void __launch_bounds__(WPB * 32) k_inv(InvParams P) {
  const Geom& g = P.g;
  const LevelGeom& lg = g.lv[P.level];
  const int sxn = (lg.w + 29) / 30;
  const int syn = (lg.h + P.sr - 1) / P.sr;
  const int strip = blockIdx.x * WPB + (threadIdx.x >> 5);
  if (strip >= sxn * syn) return;
  const int sx = strip % sxn, sy = strip / sxn;
  const int b = FINAL ? blockIdx.z : blockIdx.z / g.C;
  const int ch = FINAL ? 0 : blockIdx.z % g.C;
  // detail-plane width: one uniform branch per kernel into two fully typed bodies
  if (inv_variant_active<int16_t>(P)) inv_strip<NC, FINAL, WIN, int16_t>(P, b, ch, sx * 30, sy * P.sr, P.sr);
  else inv_strip<NC, FINAL, WIN, int32_t>(P, b, ch, sx * 30, sy * P.sr, P.sr);
}

// Intermediate inverse levels (LL_l + details_l -> LL_{l-1}, not the output level): CTA = one
// 64 x 64 tile of LL_{l-1} from the 34 x 34 windows (32 x 32 + the lifting halo, subband indices
// mirrored by sb_idx) of the four subbands, staged in shared memory with every load in flight at
// once; the column merge (_merge_axis0 on columns, transforms.py:137-162,194-199) then the row merge
// run as parallel phases.
constexpr int IT = 32;            // subband tile per side
constexpr int IW = IT + 2;        // window: subband indices n0-1 .. n0+IT
struct InvTileSmem {
  int S[4][IW][IW];          // LL, LH, HL, HH windows
  int Lc[2 * IT][IW + 1];    // column-merged low (from LL, LH)
  int Hc[2 * IT][IW + 1];    // column-merged high (from HL, HH)
};

template <typename HT>
__device__ __forceinline__ void inv_tile_body(const InvParams& P, InvTileSmem& T) {
  auto& S = T.S;
  auto& Lc = T.Lc;
  auto& Hc = T.Hc;
  const Geom& g = P.g;
  const LevelGeom& lg = g.lv[P.level];
  const LevelGeom& pg = g.lv[P.level - 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = blockIdx.x * IT, m0 = blockIdx.y * IT;
  const int b = blockIdx.z / g.C, ch = blockIdx.z % g.C;
  const int NX = pg.w, NY = pg.h;
  const bool hx_empty = NX == 1, hy_empty = NY == 1;  // the empty high band reads as 0
  const int32_t* base = P.coef + (i64)b * g.img_stride + (i64)ch * g.chan_stride;
  // 1. window loads: warp w takes window rows w, w+8, ...; lanes 0..31 (+ 0..1) the columns
  {
    constexpr int RPW = (IW + 7) / 8;
    int cl[2], chh[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int c = n0 - 1 + min(lane + 32 * k, IW - 1);
      cl[k] = sb_idx(c, 0, NX);
      chh[k] = hx_empty ? 0 : sb_idx(c, 1, NX);
    }
#pragma unroll
    for (int half = 0; half < 2; ++half) {  // (LL, HL) rows from the low row index, (LH, HH) high
      int v[RPW][2][2];
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr) {
        const int r = min(warp + 8 * rr, IW - 1);
        const int k = m0 - 1 + r;
        const bool zero_row = half == 1 && hy_empty;
        const i64 row = (i64)(half == 0 ? sb_idx(k, 0, NY) : (hy_empty ? 0 : sb_idx(k, 1, NY))) * lg.pw;
        const int32_t* pl = base + lg.off[0] + row;                                       // LL (int32)
        const HT* plh = reinterpret_cast<const HT*>(base + lg.off[1]) + row;              // LH
        const HT* ph = reinterpret_cast<const HT*>(base + lg.off[half == 0 ? 2 : 3]) + row;  // HL or HH
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const bool on = kk == 0 || lane < IW - 32;
          v[rr][kk][0] = (on && !zero_row) ? (half == 0 ? __ldg(pl + cl[kk]) : (int)__ldg(plh + cl[kk])) : 0;
          v[rr][kk][1] = (on && !zero_row && !hx_empty) ? (int)__ldg(ph + chh[kk]) : 0;
        }
      }
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr) {
        const int r = warp + 8 * rr;
        if (r < IW) {
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const int c = lane + 32 * kk;
            if (c < IW) {
              S[half == 0 ? 0 : 1][r][c] = v[rr][kk][0];
              S[half == 0 ? 2 : 3][r][c] = v[rr][kk][1];
            }
          }
        }
      }
    }
  }
  __syncthreads();
  // 2. column merge: task = (window column, low/high pair, group of 8 output row pairs)
  for (int t = tid; t < 2 * IW * 4; t += 256) {
    const int c = t % IW, rest = t / IW;
    const int pair = rest & 1, grp = rest >> 1;   // pair 0: (LL, LH) -> Lc;  1: (HL, HH) -> Hc
    const int (*Lw)[IW] = S[pair == 0 ? 0 : 2];
    const int (*Hw)[IW] = S[pair == 0 ? 1 : 3];
    int (*O)[IW + 1] = pair == 0 ? Lc : Hc;
    // subband row m0+i sits at window row i+1; even output row 2i: L[i] - ((H[i-1] + H[i] + 2) >> 2)
    const int i0 = 8 * grp;
    int xe = Lw[i0 + 1][c] - ((Hw[i0][c] + Hw[i0 + 1][c] + 2) >> 2);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = i0 + k;
      const int xn = Lw[i + 2][c] - ((Hw[i + 1][c] + Hw[i + 2][c] + 2) >> 2);
      O[2 * i][c] = xe;
      O[2 * i + 1][c] = Hw[i + 1][c] + ((xe + xn) >> 1);
      xe = xn;
    }
  }
  __syncthreads();
  // 3. row merge + store: warp per output row, lane j -> columns 2(n0+j), 2(n0+j)+1
  int32_t* dst = P.coef + (i64)b * g.img_stride + (i64)ch * g.chan_stride + pg.off[0];
  const int px = 2 * (n0 + lane);
#pragma unroll
  for (int rr = 0; rr < 2 * IT / 8; ++rr) {
    const int r = warp + 8 * rr;
    const int xe0 = Lc[r][lane + 1] - ((Hc[r][lane] + Hc[r][lane + 1] + 2) >> 2);
    const int xe1 = Lc[r][lane + 2] - ((Hc[r][lane + 1] + Hc[r][lane + 2] + 2) >> 2);
    const int xo = Hc[r][lane + 1] + ((xe0 + xe1) >> 1);
    const int py = 2 * m0 + r;
    if (py < pg.ph && px < pg.pw) *reinterpret_cast<int2*>(dst + (i64)py * pg.pw + px) = make_int2(xe0, xo);
  }
}

__global__ void __launch_bounds__(256) k_inv_tile(InvParams P) {
  __shared__ InvTileSmem T;
  if (inv_variant_active<int16_t>(P)) inv_tile_body<int16_t>(P, T);
  else inv_tile_body<int32_t>(P, T);
}

// Output from the LL planes at `level` (decode_image(level>0) or L == 0), window aware.
__global__ void k_finish(InvParams P) {
  const Geom& g = P.g;
  const LevelGeom& lg = g.lv[P.level];
  const int b = blockIdx.z;
  const int qx = blockIdx.x * 32 + (threadIdx.x & 31);
  const int qy = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (qx >= P.ow || qy >= P.oh) return;
  const int x = P.ox + qx, y = P.oy + qy;
  const int32_t* ic = P.coef + (i64)b * g.img_stride;
  int v[4];
  for (int c = 0; c < g.C; ++c) v[c] = ic[(i64)c * g.chan_stride + lg.off[0] + (i64)y * lg.pw + x];
  if (g.rct) {
    int Y = v[0], Cb = v[1], Cr = v[2];
    int G = Y - ((Cb + Cr) >> 2);
    v[0] = Cr + G;
    v[1] = G;
    v[2] = Cb + G;
  }
  char* ob = (char*)P.out + (i64)b * P.out_img_stride;
  const int OC = P.out_channels;
  for (int c = 0; c < OC; ++c) {
    i64 idx = P.out_layout == WBPC_LAYOUT_HWC ? ((i64)qy * P.ow + qx) * OC + c : ((i64)c * P.oh + qy) * P.ow + qx;
    store_sample(ob, P.out_dtype, idx, v[c], g.bd);
  }
}

// ------------------------------------------------------------------------------ launchers
template <typename T, bool HWC, bool RCT, typename CT>
static void launch_l1_ct(FwdParams P, int batch, cudaStream_t s) {
  const LevelGeom& lg = P.g.lv[1];
  const int z = RCT ? batch : batch * P.g.C;
  P.sr = pick_sr(lg.pw / 32, lg.ph, z);
  const Geom& g = P.g;
  // developer switches, read once (thread-safe static initialisation)
  static const int use_tma = [] {
    const char* e = getenv("WBPC_FWD_TMA");
    return e ? atoi(e) : 1;
  }();
  if (use_tma && sizeof(T) == 1 && HWC && RCT && g.bd == 8 && ((i64)g.W * 3) % 16 == 0 &&
      (((uintptr_t)P.src) & 15) == 0 && (P.src_img_stride & 15) == 0) {
    // validation of 8-bit samples against 2^8 is vacuous (validate_source): nothing to check
    static const int fsr = [] {
      const char* e = getenv("WBPC_FWD_SR");
      const int v = e ? atoi(e) : 16;
      return (v == 8 || v == 16 || v == 32 || v == 64) ? v : 16;
    }();
    P.sr = fsr;
    const int tx = (lg.pw + TW * 64 - 1) / (TW * 64), ty = lg.ph / P.sr;
    const int ntiles = tx * ty * batch;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::min(ntiles, 4 * nsm);  // persistent: 4 CTAs per SM
    k_fwd_rgb8_tma<CT><<<grid, (TW + 1) * 32, 0, s>>>(P, tx, ty, ntiles);
    return;
  }
  P.fast_rgb8 = sizeof(T) == 1 && HWC && RCT && g.bd == 8 && (g.W & 3) == 0 && (((uintptr_t)P.src) & 3) == 0 &&
                (P.src_img_stride & 3) == 0 && (g.W - 68) / 64 >= 1 && (P.sr % 4) == 0;
  const int strips = (lg.pw / 32) * ((lg.ph + P.sr - 1) / P.sr);
  dim3 grid((strips + WPB - 1) / WPB, 1, z);
  k_fwd_l1<T, HWC, RCT, CT><<<grid, WPB * 32, 0, s>>>(P);
}

template <typename T, bool HWC, bool RCT>
static void launch_l1(FwdParams P, int batch, cudaStream_t s) {
  if (P.g.coef16) launch_l1_ct<T, HWC, RCT, int16_t>(P, batch, s);
  else launch_l1_ct<T, HWC, RCT, int32_t>(P, batch, s);
}

cudaError_t launch_dwt_forward(const Geom& g, int batch, const void* src, int dtype, int layout, i64 img_stride,
                               void* coef, unsigned* bmax, DevStatus* st, cudaStream_t s) {
  FwdParams P;
  P.g = g;
  P.src = src;
  P.src_dtype = dtype;
  P.src_layout = layout;
  P.src_img_stride = img_stride;
  P.coef = coef;
  P.bmax = bmax;
  P.st = st;
  P.fast_rgb8 = 0;
  if (g.L == 0) {
    P.level = 0;
    const LevelGeom& lg = g.lv[0];
    dim3 grid(lg.pw / 32, lg.ph / 8, batch);
    prof_mark("level0", s);
    if (g.coef16) k_level0<int16_t><<<grid, 256, 0, s>>>(P);
    else k_level0<int32_t><<<grid, 256, 0, s>>>(P);
    return cudaGetLastError();
  }
  P.level = 1;
  prof_mark("dwt_fwd_l1", s);
  const bool hwc = layout == WBPC_LAYOUT_HWC;
  const bool rct = g.rct != 0;
  switch (dtype) {
    case WBPC_DTYPE_U8:
      if (rct) { if (hwc) launch_l1<uint8_t, true, true>(P, batch, s); else launch_l1<uint8_t, false, true>(P, batch, s); }
      else { if (hwc) launch_l1<uint8_t, true, false>(P, batch, s); else launch_l1<uint8_t, false, false>(P, batch, s); }
      break;
    case WBPC_DTYPE_U16:
      if (rct) { if (hwc) launch_l1<uint16_t, true, true>(P, batch, s); else launch_l1<uint16_t, false, true>(P, batch, s); }
      else { if (hwc) launch_l1<uint16_t, true, false>(P, batch, s); else launch_l1<uint16_t, false, false>(P, batch, s); }
      break;
    case WBPC_DTYPE_I16:
      if (rct) { if (hwc) launch_l1<int16_t, true, true>(P, batch, s); else launch_l1<int16_t, false, true>(P, batch, s); }
      else { if (hwc) launch_l1<int16_t, true, false>(P, batch, s); else launch_l1<int16_t, false, false>(P, batch, s); }
      break;
    default:
      if (rct) { if (hwc) launch_l1<int32_t, true, true>(P, batch, s); else launch_l1<int32_t, false, true>(P, batch, s); }
      else { if (hwc) launch_l1<int32_t, true, false>(P, batch, s); else launch_l1<int32_t, false, false>(P, batch, s); }
      break;
  }
  // levels >= 2: the shared-memory tile kernel (measured faster than the level-1 strip design
  // on these planes, unlike the inverse direction)
  static const int use_tma2 = [] {
    const char* e = getenv("WBPC_FWD2_TMA");
    return e ? atoi(e) : 1;
  }();
  for (int l = 2; l <= g.L; ++l) {
    P.level = l;
    const LevelGeom& lg = g.lv[l];
    const LevelGeom& pg = g.lv[l - 1];
    prof_mark("dwt_fwd", s);
    // wide int16 planes within the packed-lifting range: the TMA row-ring kernel
    if (use_tma2 && g.coef16 && lg.swar && (pg.w & 7) == 0 && pg.w >= 2 * 64 * TW && pg.h >= 2 * 16 &&
        (((uintptr_t)coef) & 15) == 0 && (g.chan_stride & 7) == 0 && (pg.off[0] & 7) == 0) {
      P.sr = 16;
      const int tx = (lg.pw + TW * 64 - 1) / (TW * 64), ty = lg.ph / P.sr;
      const int ntiles = tx * ty * batch * g.C;
      int dev = 0, nsm = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      const int grid = std::min(ntiles, WBPC_FWD2_MINB * nsm);
      k_fwd_i16_tma<<<grid, (TW + 1) * 32, 0, s>>>(P, tx, ty, ntiles);
      continue;
    }
    dim3 grid(lg.pw / FT, lg.ph / FT, batch * g.C);
    if (g.coef16) k_fwd_tile<int16_t><<<grid, 256, 0, s>>>(P);
    else k_fwd_tile<int32_t><<<grid, 256, 0, s>>>(P);
  }
  return cudaGetLastError();
}

cudaError_t launch_dwt_inverse(const Geom& g, int batch, int out_level, int32_t* coef, void* out, int out_dtype,
                               int out_layout, i64 out_img_stride, int out_channels, cudaStream_t s,
                               const int* window, const u64* hpdepth, int allow16) {
  InvParams P;
  P.g = g;
  P.hpdepth = hpdepth;
  P.allow16 = allow16;
  const LevelGeom& lo = g.lv[out_level];
  P.ox = window ? window[0] : 0;
  P.oy = window ? window[1] : 0;
  P.ow = window ? window[2] : lo.w;
  P.oh = window ? window[3] : lo.h;
  P.coef = coef;
  P.out_dtype = out_dtype;
  P.out_layout = out_layout;
  P.out_img_stride = out_img_stride;
  P.out_channels = out_channels;
  for (int l = g.L; l > out_level; --l) {
    P.level = l;
    const LevelGeom& lg = g.lv[l];
    const bool fuse = (l == out_level + 1) && out_level == 0;
    P.out = fuse ? out : nullptr;
    P.sr = pick_sr((lg.w + 29) / 30, lg.h, fuse ? batch : batch * g.C);
    const int strips = ((lg.w + 29) / 30) * ((lg.h + P.sr - 1) / P.sr);
    dim3 grid((strips + WPB - 1) / WPB, 1, fuse ? batch : batch * g.C);
    prof_mark(fuse ? "dwt_inv_l1" : "dwt_inv", s);
    // intermediate levels: the register-streaming strip kernel for wide levels (measured on the
    // 4096^2 tiles: 22% faster than the shared-memory tile kernel), the tile kernel for narrow
    // ones (few strips per level)
    static const int use_inv2 = [] {
      const char* e = getenv("WBPC_INV2");
      return e ? atoi(e) : 1;
    }();
    const LevelGeom& pgl = g.lv[l - 1];
    const bool full = !(window && !(P.ox == 0 && P.oy == 0 && P.ow == lo.w && P.oh == lo.h));
    // two columns per lane: wide levels whose detail planes may hold int16 (the kernel falls back
    // per strip otherwise); the final level only as 8-bit interleaved RGB with the colour transform
    const bool inv2 = use_inv2 && allow16 && lg.w >= 512 && pgl.h >= 2 &&
                      (!fuse || (full && g.C == 3 && g.rct && out_channels == 3 && out_dtype == WBPC_DTYPE_U8 &&
                                 out_layout == WBPC_LAYOUT_HWC && (pgl.w & 3) == 0 && (((uintptr_t)out) & 3) == 0 &&
                                 (out_img_stride & 3) == 0));
    if (inv2) {
      // 16-row strips: shorter walks keep more strips in flight (measured on 4096^2 tiles: level 2
      // 86 -> 77 us, level 1 210 -> 197 us against 32-row strips)
      P.sr = std::min(16, pick_sr((lg.w + 59) / 60, lg.h, fuse ? batch : batch * g.C));
      const int strips2 = ((lg.w + 59) / 60) * ((lg.h + P.sr - 1) / P.sr);
      dim3 grid2((strips2 + WPB - 1) / WPB, 1, fuse ? batch : batch * g.C);
      if (fuse) k_inv2<3, true><<<grid2, WPB * 32, 0, s>>>(P);
      else k_inv2<1, false><<<grid2, WPB * 32, 0, s>>>(P);
    } else if (!fuse && lg.w >= 256) {
      k_inv<1, false, false><<<grid, WPB * 32, 0, s>>>(P);
    } else if (!fuse) {
      dim3 tg((lg.w + IT - 1) / IT, (lg.h + IT - 1) / IT, batch * g.C);
      k_inv_tile<<<tg, 256, 0, s>>>(P);
    } else if (window && !(P.ox == 0 && P.oy == 0 && P.ow == lo.w && P.oh == lo.h)) {
      switch (g.C) {
        case 1: k_inv<1, true, true><<<grid, WPB * 32, 0, s>>>(P); break;
        case 2: k_inv<2, true, true><<<grid, WPB * 32, 0, s>>>(P); break;
        case 3: k_inv<3, true, true><<<grid, WPB * 32, 0, s>>>(P); break;
        default: k_inv<4, true, true><<<grid, WPB * 32, 0, s>>>(P); break;
      }
    } else {
      switch (g.C) {
        case 1: k_inv<1, true, false><<<grid, WPB * 32, 0, s>>>(P); break;
        case 2: k_inv<2, true, false><<<grid, WPB * 32, 0, s>>>(P); break;
        case 3: k_inv<3, true, false><<<grid, WPB * 32, 0, s>>>(P); break;
        default: k_inv<4, true, false><<<grid, WPB * 32, 0, s>>>(P); break;
      }
    }
  }
  if (out_level > 0 || g.L == 0) {
    P.level = out_level;
    P.out = out;
    dim3 grid((P.ow + 31) / 32, (P.oh + 7) / 8, batch);
    prof_mark("finish", s);
    k_finish<<<grid, 256, 0, s>>>(P);
  }
  return cudaGetLastError();
}

}  // namespace wb
