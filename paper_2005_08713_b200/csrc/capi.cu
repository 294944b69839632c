// capi.cu — extern "C" entry points (include/wbpc_b200.h): host-side geometry planning,
// workspace carving and kernel sequencing.  No device memory is allocated here; every call is
// stream ordered and the only host synchronisation is wbpc_query_status().
#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "coder.cuh"

namespace wb {
struct DecMeta;
struct TruncMeta;
struct BlockTab;
size_t block_tab_bytes();
cudaError_t launch_dwt_forward(const Geom& g, int batch, const void* src, int dtype, int layout, i64 img_stride,
                               void* coef, unsigned* bmax, DevStatus* st, cudaStream_t s);
cudaError_t launch_dwt_inverse(const Geom& g, int batch, int out_level, int32_t* coef, void* out, int out_dtype,
                               int out_layout, i64 out_img_stride, int out_channels, cudaStream_t s,
                               const int* window, const u64* hpdepth, int allow16);
cudaError_t launch_encode_blocks(const Geom& g, int batch, const void* coef, const unsigned* bmax, uint8_t* syms,
                                 uint16_t* wbits, BlockMeta* meta, void* stats, uint32_t* zmask, uint32_t* sizes,
                                 u64* block_off, u64* img_off, uint8_t* out, u64 cap, DevStatus* st, cudaStream_t s);
size_t block_stats_bytes();
cudaError_t launch_index_check(const Geom& g, int batch, const uint8_t* data, const u64* img_off, u64* blk_off,
                               uint32_t* blk_len, DevStatus* st, cudaStream_t s);
cudaError_t launch_decode_blocks(const Geom& g, int batch, int level, int drop_global, const int* drop_hp,
                                 int drop_ll, int per_level, const uint8_t* data, u64 nbytes, const u64* blk_off,
                                 const uint32_t* blk_len, BlockTab* tabs, uint32_t* flags, uint8_t* syms,
                                 DecMeta* dmeta, int32_t* coef, DevStatus* st, cudaStream_t s,
                                 const uint8_t* need);
cudaError_t launch_block_headers(const Geom& g, int batch, const uint8_t* data, u64 nbytes, const u64* blk_off,
                                 const uint32_t* blk_len, BlockTab* tabs, DecMeta* dmeta, DevStatus* st,
                                 cudaStream_t s);
cudaError_t launch_plane_offsets(const BlockTab* tab, int32_t* slots, uint32_t* offs, int32_t* count, cudaStream_t s);
cudaError_t launch_region_need(const Geom& g, int level, const RegionBoxes& B, uint8_t* need, cudaStream_t s);
cudaError_t launch_block_summary(const BlockTab* tabs, const u64* blk_off, int n, int32_t* depth, uint32_t* hbits,
                                 cudaStream_t s);
cudaError_t launch_truncate(const Geom& g, int per_level, int drop_global, const int* drop_hp, int drop_ll,
                            const uint8_t* data, u64 nbytes, const u64* blk_off, const uint32_t* blk_len,
                            TruncMeta* tm, uint32_t* sizes, u64* new_off, u64* img_off, uint8_t* out, u64 cap,
                            DevStatus* st, cudaStream_t s);
cudaError_t launch_decode_tokens(const uint8_t* payload, u64 nbytes, i64 start_bit, i64 end_bit, const int32_t* left,
                                 const int32_t* right, const int32_t* leaf, int zr, int cw, const i64* seg_len,
                                 int nseg, uint8_t* out, i64* seg_starts, i64* result, cudaStream_t s);
size_t trunc_meta_bytes();
cudaError_t launch_raw_bmax(const Geom& g, int nblocks, const int32_t* coef, unsigned* bmax, DevStatus* st,
                            cudaStream_t s);
cudaError_t launch_raw_index(const u64* offsets, int n, u64* blk_off, uint32_t* blk_len, cudaStream_t s);
cudaError_t launch_tile_sizes(const u64* enc_off, int B, int n_local, int per, u64* sizes, cudaStream_t s);
cudaError_t launch_archive_index(const u64* sizes_all, int n_tiles, int tiles_x, int tiles_y, int first, int n_local,
                                 uint8_t* hdr, u64* local_off, u64* base_total, cudaStream_t s);
cudaError_t launch_gather_tiles(const uint8_t* store, u64 region, const u64* enc_off, int B, int n_local,
                                uint8_t* dst, const u64* local_off, cudaStream_t s);
cudaError_t launch_batch_offsets(const u64* enc_off_k, int b, u64* local_off_k, cudaStream_t s);
}  // namespace wb

using namespace wb;

// ---------------------------------------------------------------------------- profiling
namespace {
struct Mark {
  std::string name;
  cudaEvent_t ev;
  cudaStream_t s;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<Mark> g_marks;
std::vector<cudaEvent_t> g_pool;
}  // namespace

void wb::prof_mark(const char* name, cudaStream_t s) {
  if (!g_prof_on) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEvent_t ev;
  if (g_pool.empty()) cudaEventCreate(&ev);
  else { ev = g_pool.back(); g_pool.pop_back(); }
  cudaEventRecord(ev, s);
  g_marks.push_back({name, ev, s});
}

static thread_local std::string g_msg;
static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_msg = buf;
  return code;
}
#define CUDA_TRY(x)                                                          \
  do {                                                                       \
    cudaError_t e_ = (x);                                                    \
    if (e_ != cudaSuccess) return fail(WBPC_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
  } while (0)

static inline u64 align_up(u64 v, u64 a) { return (v + a - 1) / a * a; }

// ---------------------------------------------------------------------------- geometry
static void level_dims(u64 w, u64 h, int l, u64* lw, u64* lh) {
  if (l >= 63) { *lw = 1; *lh = 1; return; }
  *lw = (w + (1ull << l) - 1) >> l;
  *lh = (h + (1ull << l) - 1) >> l;
}

struct Interval { i64 lo, hi; };
// Conservative bounds of one 1-D 5/3 split (transforms.py:125,133) of a signal in [lo, hi].
static void lift_bound(Interval x, int n, Interval* low, Interval* high) {
  if (n <= 1) { *low = x; *high = {0, 0}; return; }
  Interval h{x.lo - x.hi, x.hi - x.lo};
  auto fdiv4 = [](i64 a) { return a >= 0 ? a / 4 : -((-a + 3) / 4); };
  *high = h;
  *low = {x.lo + fdiv4(2 * h.lo + 2), x.hi + fdiv4(2 * h.hi + 2)};
}
static i64 mag(Interval v) { return std::max(v.lo < 0 ? -v.lo : v.lo, v.hi < 0 ? -v.hi : v.hi); }
static int depth_of(i64 m) {
  int b = 0;
  while (m) { ++b; m >>= 1; }
  return 1 + b;
}

// Exact max-row L1 norms of the linear part (the floors dropped) of the 1-D 5/3 analysis
// cascade on a signal of length N: lo[l] / hi[l] for the level-l lowpass / highpass outputs
// (lo[0] = 1), l = 1..L, splits and boundary mirroring as transforms.py:107-133.  Every output
// is a linear functional of the input samples, carried as a dense window (offset + taps) and
// combined by the lifting steps.  Rows near an edge depend only on the per-level length
// parities, i.e. on N mod 2^(L+1), and interior rows are the cascaded filter, so a long signal
// is replaced by one of length N mod 2^(L+1) + 16 * 2^(L+1).  Returns false when that is still
// too long to evaluate (the caller then keeps the per-pass bound).
static bool cascade_norms_eval(u64 n, int L, double* lo, double* hi);
static bool cascade_norms(u64 N, int L, double* lo, double* hi) {
  const u64 P = L + 1 < 40 ? 1ull << (L + 1) : ~0ull;
  u64 n = N;
  if (P != ~0ull && N > 24 * P) n = N % P + 16 * P;
  if (n > (1u << 16)) return false;
  // memoised: geometry is planned on every encode call
  struct Row { bool ok; double lo[WB_MAXL + 1], hi[WB_MAXL + 1]; };
  static std::mutex mu;
  static std::map<std::pair<u64, int>, Row> memo;
  std::lock_guard<std::mutex> lk(mu);
  auto it = memo.find({n, L});
  if (it == memo.end()) {
    Row r{};
    r.ok = cascade_norms_eval(n, L, r.lo, r.hi);
    if (memo.size() > 4096) memo.clear();
    it = memo.emplace(std::make_pair(n, L), r).first;
  }
  std::copy(it->second.lo, it->second.lo + L + 1, lo);
  std::copy(it->second.hi, it->second.hi + L + 1, hi);
  return it->second.ok;
}
static bool cascade_norms_eval(u64 n, int L, double* lo, double* hi) {
  struct Fn { i64 off; std::vector<double> c; };
  auto comb = [](const Fn* f, const double* w, int k) {
    i64 a = f[0].off, b = f[0].off + (i64)f[0].c.size();
    for (int i = 1; i < k; ++i) { a = std::min(a, f[i].off); b = std::max(b, f[i].off + (i64)f[i].c.size()); }
    Fn r{a, std::vector<double>((size_t)(b - a), 0.0)};
    for (int i = 0; i < k; ++i)
      for (size_t j = 0; j < f[i].c.size(); ++j) r.c[(size_t)(f[i].off - a) + j] += w[i] * f[i].c[j];
    return r;
  };
  auto norm = [](const Fn& f) { double t = 0; for (double v : f.c) t += v < 0 ? -v : v; return t; };
  std::vector<Fn> x((size_t)n);
  for (u64 i = 0; i < n; ++i) x[i] = Fn{(i64)i, {1.0}};
  lo[0] = 1.0;
  hi[0] = 0.0;
  for (int l = 1; l <= L; ++l) {
    const size_t m = x.size();
    if (m <= 1) { lo[l] = lo[l - 1]; hi[l] = 0; continue; }  // a length-1 split is the identity
    const size_t mh = m / 2, ml = m - mh;
    std::vector<Fn> h(mh), lw(ml);
    const double wh[3] = {1.0, -0.5, -0.5}, wl[3] = {1.0, 0.25, 0.25};
    for (size_t k = 0; k < mh; ++k) {
      size_t r = 2 * k + 2 < m ? 2 * k + 2 : 2 * k;  // x[m] mirrors to x[m-2]
      Fn f[3] = {x[2 * k + 1], x[2 * k], x[r]};
      h[k] = comb(f, wh, 3);
    }
    for (size_t k = 0; k < ml; ++k) {
      Fn f[3] = {x[2 * k], h[k ? k - 1 : 0], h[std::min(k, mh - 1)]};  // high[-1]=high[0], high[mh]=high[mh-1]
      lw[k] = comb(f, wl, 3);
    }
    double a = 0, b = 0;
    for (auto& f : lw) a = std::max(a, norm(f));
    for (auto& f : h) b = std::max(b, norm(f));
    lo[l] = a; hi[l] = b;
    x.swap(lw);
  }
  return true;
}

static u64 div_magic(int d) { return d >= 1 ? ~0ull / (u64)d : 0ull; }
static void geom_magics(Geom* g) {
  g->md_spc = div_magic(g->slots_per_channel);
  g->md_spi = div_magic(g->slots_per_image);
  for (int l = 0; l <= WB_MAXL; ++l) g->lv[l].md_gw = div_magic(g->lv[l].gw);
}

// Returns 0 or a wbpc_status.  Builds every offset the kernels use.
static int make_geom(u64 W, u64 H, int C, int bd, int L, int rct, Geom* g) {
  memset(g, 0, sizeof *g);
  g->raw_kind = -1;
  g->keep = -1;
  if (W < 1 || H < 1 || W > (1u << 30) || H > (1u << 30)) return fail(WBPC_ERR_DOMAIN, "image dimensions");
  if (C < 1 || C > 4) return fail(WBPC_ERR_UNSUPPORTED_LAYOUT, "channels must be 1..4, got %d", C);
  if (L < 0 || L > WB_MAXL) return fail(WBPC_ERR_LEVEL_RANGE, "levels must be in [0, %d]", WB_MAXL);
  g->W = (int)W; g->H = (int)H; g->C = C; g->L = L; g->bd = bd; g->rct = rct;
  i64 off = 0;
  for (int l = 0; l <= L; ++l) {
    LevelGeom& lg = g->lv[l];
    u64 w, h;
    level_dims(W, H, l, &w, &h);
    lg.w = (int)w; lg.h = (int)h;
    lg.gw = (int)((w + WB_DIM - 1) / WB_DIM);
    lg.gh = (int)((h + WB_DIM - 1) / WB_DIM);
    lg.pw = lg.gw * WB_DIM;
    lg.ph = lg.gh * WB_DIM;
    if (l >= 1) {
      u64 pw, ph;
      level_dims(W, H, l - 1, &pw, &ph);
      int cw = (int)((pw + 1) / 2), fw = (int)(pw / 2), ch = (int)((ph + 1) / 2), fh = (int)(ph / 2);
      lg.sw[0] = cw; lg.sh[0] = ch;  // LL
      lg.sw[1] = cw; lg.sh[1] = fh;  // LH (container.py:132-137)
      lg.sw[2] = fw; lg.sh[2] = ch;  // HL
      lg.sw[3] = fw; lg.sh[3] = fh;  // HH
      i64 psz = (i64)lg.pw * lg.ph;
      for (int k = 0; k < 4; ++k) { lg.off[k] = off; off += psz; }
    } else if (L == 0) {
      lg.off[0] = off;
      off += (i64)lg.pw * lg.ph;
    }
  }
  g->chan_stride = (i64)align_up((u64)off, 64);
  g->img_stride = g->chan_stride * C;
  // slots (iter_slots, container.py:115-129)
  int nll = g->lv[L].gw * g->lv[L].gh;
  int acc = nll;
  for (int l = L; l >= 1; --l) { g->lv[l].slot0 = acc; acc += g->lv[l].gw * g->lv[l].gh; }
  g->slots_per_channel = acc;
  g->slots_per_image = acc * C;
  geom_magics(g);
  // static coefficient bounds -> depth bounds and int32 safety
  const i64 mx = (1ll << bd) - 1;
  Interval x = rct ? Interval{-mx, mx} : Interval{0, mx};
  int dmax = 1;
  const i64 SAFE = 1ll << 30;
  const i64 SAFE16 = (1ll << 15) - 1;  // int16 storage when every bound stays inside +-32767
  bool fits16 = mag(x) <= SAFE16;
  i64 m16 = mag(x);  // filter-norm bound of the current LL (see below)
  if (mag(x) >= SAFE) return fail(WBPC_ERR_UNSUPPORTED, "coefficient range exceeds int32 path");
  // Exact separable bound for int16 storage: |coef| <= norm(band) * M + rounding error, with the
  // band norm the product of the two axes' cascade norms and the floors' error propagated pass
  // by pass (a pass turns an input error E into <= 1.5E + 1 on low outputs, <= 2E + 1 on high
  // ones).  Row-pass intermediates are covered for either axis order.
  double aw[WB_MAXL + 1], bw[WB_MAXL + 1], ah[WB_MAXL + 1], bh[WB_MAXL + 1];
  bool exact16 = mag(x) <= SAFE16 && cascade_norms(W, L, aw, bw) && cascade_norms(H, L, ah, bh);
  if (exact16) {
    const double M = (double)mag(x);
    const double SWAR_MAX = 8000.0;
    bool swar_in = M <= SWAR_MAX;  // the level's input (LL of the level below) is in range too
    double E = 0;
    for (int l = 1; l <= L && exact16; ++l) {
      const double eL = 1.5 * E + 1, eH = 2 * E + 1, eHH = 2 * eH + 1, eLL = 1.5 * eL + 1;
      const double nrm = std::max({aw[l] * ah[l], aw[l] * bh[l], bw[l] * ah[l], bw[l] * bh[l],
                                   aw[l] * ah[l - 1], bw[l] * ah[l - 1], aw[l - 1] * ah[l], aw[l - 1] * bh[l]});
      const double bnd = nrm * M * (1 + 1e-9) + eHH + 1;  // every value of level l, row-pass ones included
      exact16 = bnd <= (double)SAFE16;
      // packed 16-bit lifting (dwt.cu k_fwd_i16_tma): inputs, intermediates and outputs of the
      // level inside +-SWAR_MAX (fields biased by 2^14 must stay below 2^15 with headroom)
      swar_in = swar_in && bnd <= SWAR_MAX;
      g->lv[l].swar = swar_in ? 1 : 0;
      E = eLL;
    }
  }
  for (int l = 1; l <= L; ++l) {
    u64 pw, ph;
    level_dims(W, H, l - 1, &pw, &ph);
    Interval lr, hr, ll, lh, hl, hh;
    lift_bound(x, (int)pw, &lr, &hr);
    lift_bound(lr, (int)ph, &ll, &lh);
    lift_bound(hr, (int)ph, &hl, &hh);
    i64 mh = std::max(mag(lh), std::max(mag(hl), mag(hh)));
    // int16 storage uses the filter-norm bound, far tighter than the interval one: a 1-D 5/3
    // lifting pass over |x| <= M gives |low| <= 1.5M + 2 (taps -1/8 1/4 3/4 1/4 -1/8 plus the
    // floor roundings) and |high| <= 2M + 1 (taps -1/2 1 -1/2); mirroring repeats samples
    {
      auto lo1 = [](i64 m) { return (3 * m + 1) / 2 + 2; };
      auto hi1 = [](i64 m) { return 2 * m + 1; };
      const i64 nLL = lo1(lo1(m16)), nLH = hi1(lo1(m16)), nHL = lo1(hi1(m16)), nHH = hi1(hi1(m16));
      fits16 = fits16 && std::max(std::max(nLL, nLH), std::max(nHL, nHH)) <= SAFE16;
      m16 = std::min(nLL, mag(ll));  // the next level's input (never above the interval bound)
    }
    if (mag(ll) >= SAFE || mh >= SAFE || mag(lr) >= SAFE || mag(hr) >= SAFE)
      return fail(WBPC_ERR_UNSUPPORTED, "static coefficient bound exceeds the int32 path at level %d", l);
    g->lv[l].depth_bound[1] = depth_of(mh);
    dmax = std::max(dmax, g->lv[l].depth_bound[1]);
    x = ll;
  }
  g->lv[L].depth_bound[0] = depth_of(mag(x));
  dmax = std::max(dmax, g->lv[L].depth_bound[0]);
  if (dmax > WB_MAX_DEPTH) dmax = WB_MAX_DEPTH;
  g->sym_stride_hp = 3 * dmax * WB_PP;
  g->sym_stride_ll = dmax * WB_PP;
  g->coef16 = (fits16 || exact16) && getenv("WBPC_COEF32") == nullptr ? 1 : 0;
  return 0;
}


// Block API geometry: n raw 128x128 blocks of one kind.  Coefficients are channel planar per
// subband: LL -> [n][128][128] (level-0 plane), HP3 -> [3][n][128][128] (LH, HL, HH planes of
// "level 1"); block i is tile row i.
static int make_geom_raw(int kind, u64 n, Geom* g) {
  memset(g, 0, sizeof *g);
  if (kind != 0 && kind != 1) return fail(WBPC_ERR_DOMAIN, "unknown block kind %d", kind);
  if (n < 1 || n > (1u << 20)) return fail(WBPC_ERR_INVALID_ARG, "block count");
  g->raw_kind = kind;
  g->keep = -1;
  g->W = WB_DIM;
  g->H = (int)(WB_DIM * n);
  g->C = 1;
  g->L = kind;
  g->bd = 16;
  LevelGeom& lg = g->lv[kind];
  lg.w = WB_DIM; lg.h = (int)(WB_DIM * n);
  lg.gw = 1; lg.gh = (int)n;
  lg.pw = WB_DIM; lg.ph = (int)(WB_DIM * n);
  const i64 plane = (i64)WB_DIM * WB_DIM * (i64)n;
  for (int k = 0; k < 4; ++k) { lg.sw[k] = WB_DIM; lg.sh[k] = (int)(WB_DIM * n); }
  if (kind == 0) lg.off[0] = 0;
  else { lg.off[1] = 0; lg.off[2] = plane; lg.off[3] = 2 * plane; lg.off[0] = 0; }
  g->chan_stride = (kind ? 3 : 1) * plane;
  g->img_stride = g->chan_stride;
  g->slots_per_channel = (int)n;
  g->slots_per_image = (int)n;
  geom_magics(g);
  g->sym_stride_hp = 3 * WB_MAX_DEPTH * WB_PP;
  g->sym_stride_ll = WB_MAX_DEPTH * WB_PP;
  return 0;
}

// Decode geometry: depth in the stream can be anything <= 32 (larger is unsupported).
static int make_geom_decode(const wbpc_header* h, Geom* g) {
  int rc = make_geom(h->width, h->height, (int)h->channels, 16, (int)h->levels, h->color_transform == 1 && h->channels >= 3, g);
  if (rc == WBPC_ERR_UNSUPPORTED) rc = 0;  // bounds are for the encoder only
  if (rc) return rc;
  g->bd = (int)h->bit_depth;
  g->coef16 = 0;  // decode kernels use int32 coefficients
  g->sym_stride_hp = 3 * WB_MAX_DEPTH * WB_PP;
  g->sym_stride_ll = WB_MAX_DEPTH * WB_PP;
  return 0;
}

// ---------------------------------------------------------------------------- workspace
struct Carver {
  u64 off = 0;
  char* base;
  explicit Carver(void* b) : base((char*)b) {}
  template <typename T>
  T* take(u64 bytes) {
    off = align_up(off, 256);
    T* p = base ? (T*)(base + off) : nullptr;
    off += bytes;
    return p;
  }
};

struct EncWs {
  DevStatus* st;
  int32_t* coef;
  unsigned* bmax;
  uint8_t* syms;
  uint16_t* wbits;  // token bits per (block, stored slot, 32-symbol word): sizes -> emit
  void* stats;      // per-block symbol statistics: symbols -> huffman / sizes
  uint32_t* zmask;  // zero masks of the stored slots: symbols -> sizes
  BlockMeta* meta;
  uint32_t* sizes;
  u64* block_off;
  u64* img_off;
  u64 total;
};

static EncWs carve_encode(void* base, const Geom& g, u64 batch) {
  Carver c(base);
  EncWs w;
  const u64 nb = batch * (u64)g.slots_per_image;
  w.st = c.take<DevStatus>(sizeof(DevStatus));
  w.coef = c.take<int32_t>(4ull * g.img_stride * batch);
  w.bmax = c.take<unsigned>(4ull * nb);
  w.syms = c.take<uint8_t>((u64)g.sym_stride_hp * nb);
  w.wbits = c.take<uint16_t>(2ull * 64 * (g.sym_stride_hp / WB_PP) * nb);
  w.stats = c.take<char>(block_stats_bytes() * nb);
  w.zmask = c.take<uint32_t>(256ull * (g.sym_stride_hp / WB_PP) * nb);
  w.meta = c.take<BlockMeta>(sizeof(BlockMeta) * nb);
  w.sizes = c.take<uint32_t>(4ull * nb);
  w.block_off = c.take<u64>(8ull * nb);
  w.img_off = c.take<u64>(8ull * (batch + 1));
  w.total = align_up(c.off, 256);
  return w;
}

struct DecWs {
  DevStatus* st;
  int32_t* coef;
  BlockTab* tabs;
  uint32_t* flags;
  uint8_t* syms;
  DecMeta* dmeta;
  u64* blk_off;
  uint32_t* blk_len;
  u64* img_off;
  uint8_t* need;
  u64 total;
};

static DecWs carve_decode(void* base, const Geom& g, u64 batch) {
  Carver c(base);
  DecWs w;
  const u64 nb = batch * (u64)g.slots_per_image;
  w.st = c.take<DevStatus>(sizeof(DevStatus));
  w.coef = c.take<int32_t>(4ull * g.img_stride * batch);
  w.tabs = c.take<BlockTab>(block_tab_bytes() * nb);
  w.flags = c.take<uint32_t>(4ull * nb);
  w.syms = c.take<uint8_t>((u64)g.sym_stride_hp * nb);
  w.dmeta = c.take<DecMeta>(32ull * nb);
  w.blk_off = c.take<u64>(8ull * nb);
  w.blk_len = c.take<uint32_t>(4ull * nb);
  w.img_off = c.take<u64>(8ull * (batch + 1));
  w.need = c.take<uint8_t>(nb);
  w.total = align_up(c.off, 256);
  return w;
}

struct TrWs {
  DevStatus* st;
  TruncMeta* tm;
  uint32_t* sizes;
  u64* blk_off;
  uint32_t* blk_len;
  u64* new_off;
  u64* img_off;
  u64 total;
};

static TrWs carve_trunc(void* base, const Geom& g) {
  Carver c(base);
  TrWs w;
  const u64 nb = (u64)g.slots_per_image;
  w.st = c.take<DevStatus>(sizeof(DevStatus));
  w.tm = c.take<TruncMeta>(trunc_meta_bytes() * nb);
  w.sizes = c.take<uint32_t>(4ull * nb);
  w.blk_off = c.take<u64>(8ull * nb);
  w.blk_len = c.take<uint32_t>(4ull * nb);
  w.new_off = c.take<u64>(8ull * nb);
  w.img_off = c.take<u64>(16);
  w.total = align_up(c.off, 256);
  return w;
}

__global__ void k_set_offsets(u64* img_off, u64 len) {
  img_off[0] = 0;
  img_off[1] = len;
}

static int dtype_size(int dt) {
  switch (dt) {
    case WBPC_DTYPE_U8: case WBPC_DTYPE_U8_DISPLAY: return 1;
    case WBPC_DTYPE_U16: case WBPC_DTYPE_I16: return 2;
    case WBPC_DTYPE_I32: return 4;
    default: return 0;
  }
}

// ---------------------------------------------------------------------------- extern "C"
extern "C" {

int wbpc_abi_version(void) { return 1; }
const char* wbpc_last_error(void) { return g_msg.c_str(); }

int wbpc_parse_header(const uint8_t* d, size_t len, wbpc_header* out) {
  if (!d || !out) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  if (len < 19) return fail(WBPC_ERR_CONTAINER_PARSE, "container shorter than its header");
  if (memcmp(d, "WBPC", 4)) return fail(WBPC_ERR_CONTAINER_PARSE, "bad magic");
  if (d[4] != 1) return fail(WBPC_ERR_CONTAINER_PARSE, "unsupported version %d", d[4]);
  auto le = [&](int o, int n) { u64 v = 0; for (int i = n - 1; i >= 0; --i) v = (v << 8) | d[o + i]; return v; };
  out->width = (uint32_t)le(5, 4);
  out->height = (uint32_t)le(9, 4);
  out->channels = d[13];
  out->bit_depth = d[14];
  out->color_transform = d[15];
  out->levels = d[16];
  out->block_dim = (uint32_t)le(17, 2);
  if (out->width < 1 || out->height < 1 || out->channels < 1 || out->channels > 4 || out->block_dim < 8)
    return fail(WBPC_ERR_CONTAINER_PARSE, "invalid header geometry");
  return 0;
}

int wbpc_slot_count(const wbpc_header* h, uint64_t* n) {
  if (!h || !n) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  u64 total = 0;
  int L = (int)h->levels;
  for (int pass = 0; pass <= L; ++pass) {
    int l = pass == 0 ? L : L - pass + 1;
    u64 w, hh;
    level_dims(h->width, h->height, l, &w, &hh);
    u64 dim = h->block_dim ? h->block_dim : 128;
    total += ((w + dim - 1) / dim) * ((hh + dim - 1) / dim);
  }
  *n = total * h->channels;
  return 0;
}

int wbpc_encode_plan_size(const wbpc_image_desc* d, uint32_t batch, int levels, int use_rct, size_t* ws,
                          size_t* cap) {
  if (!d || !ws) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  if (use_rct && d->channels != 3) return fail(WBPC_ERR_UNSUPPORTED_LAYOUT, "color transform needs exactly 3 channels");
  if (d->bit_depth < 1 || d->bit_depth > 16) return fail(WBPC_ERR_DOMAIN, "bit depth must be 1..16, got %u", d->bit_depth);
  Geom g;
  int rc = make_geom(d->width, d->height, (int)d->channels, (int)d->bit_depth, levels, use_rct ? 1 : 0, &g);
  if (rc) return rc;
  EncWs w = carve_encode(nullptr, g, batch ? batch : 1);
  *ws = (size_t)w.total;
  if (cap) {
    // generous first guess: raw samples x 1.25 + index/header + per-block header slack
    u64 raw = (u64)d->width * d->height * d->channels * 2;
    u64 per = 19 + 12ull * g.slots_per_image + 1200ull * g.slots_per_image + raw + raw / 4;
    *cap = (size_t)(per * (batch ? batch : 1));
  }
  return 0;
}

int wbpc_encode_coef_bytes(const wbpc_image_desc* d, int levels, int use_rct, int* out) {
  if (!d || !out) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  if (use_rct && d->channels != 3) return fail(WBPC_ERR_UNSUPPORTED_LAYOUT, "color transform needs exactly 3 channels");
  if (d->bit_depth < 1 || d->bit_depth > 16) return fail(WBPC_ERR_DOMAIN, "bit depth must be 1..16, got %u", d->bit_depth);
  Geom g;
  int rc = make_geom(d->width, d->height, (int)d->channels, (int)d->bit_depth, levels, use_rct ? 1 : 0, &g);
  if (rc) return rc;
  *out = g.coef16 ? 2 : 4;
  return 0;
}

int wbpc_encode(const wbpc_image_desc* d, const void* d_pixels, uint32_t batch, int levels, int use_rct, void* d_ws,
                size_t ws_bytes, uint8_t* d_out, size_t out_cap, uint64_t* d_out_offsets, void* stream) {
  if (!d || !d_pixels || !d_ws || !d_out) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  if (batch < 1) return fail(WBPC_ERR_INVALID_ARG, "batch must be >= 1");
  if (d->channels < 1 || d->channels > 4) return fail(WBPC_ERR_UNSUPPORTED_LAYOUT, "channels must be 1..4, got %u", d->channels);
  if (d->bit_depth < 1 || d->bit_depth > 16) return fail(WBPC_ERR_DOMAIN, "bit depth must be 1..16, got %u", d->bit_depth);
  if (use_rct && d->channels != 3) return fail(WBPC_ERR_UNSUPPORTED_LAYOUT, "color transform needs exactly 3 channels");
  if (!dtype_size(d->dtype)) return fail(WBPC_ERR_INVALID_ARG, "unsupported dtype %d", d->dtype);
  Geom g;
  int rc = make_geom(d->width, d->height, (int)d->channels, (int)d->bit_depth, levels, use_rct ? 1 : 0, &g);
  if (rc) return rc;
  EncWs w = carve_encode(d_ws, g, batch);
  if (w.total > ws_bytes) return fail(WBPC_ERR_WORKSPACE, "workspace %zu < %llu", ws_bytes, (unsigned long long)w.total);
  cudaStream_t s = (cudaStream_t)stream;
  const u64 nb = (u64)batch * g.slots_per_image;
  CUDA_TRY(cudaMemsetAsync(w.st, 0xFF, sizeof(u64), s));
  CUDA_TRY(cudaMemsetAsync(&w.st->total, 0, 3 * sizeof(u64), s));
  CUDA_TRY(cudaMemsetAsync(w.bmax, 0, 4 * nb, s));
  u64 stride = d->image_stride_bytes ? d->image_stride_bytes
                                     : (u64)d->width * d->height * d->channels * dtype_size(d->dtype);
  CUDA_TRY(launch_dwt_forward(g, (int)batch, d_pixels, d->dtype, d->layout, (i64)stride, w.coef, w.bmax, w.st, s));
  CUDA_TRY(launch_encode_blocks(g, (int)batch, w.coef, w.bmax, w.syms, w.wbits, w.meta, w.stats, w.zmask, w.sizes, w.block_off, w.img_off, d_out,
                                out_cap, w.st, s));
  prof_mark("", s);
  if (d_out_offsets)
    CUDA_TRY(cudaMemcpyAsync(d_out_offsets, w.img_off, 8ull * (batch + 1), cudaMemcpyDeviceToDevice, s));
  return 0;
}

int wbpc_decode_plan_size(const wbpc_header* h, int level, size_t* ws) {
  (void)level;
  if (!h || !ws) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  Geom g;
  int rc = make_geom_decode(h, &g);
  if (rc) return rc;
  *ws = (size_t)carve_decode(nullptr, g, 1).total;
  return 0;
}

int wbpc_decode_batch_plan_size(const wbpc_header* h, uint32_t batch, size_t* ws) {
  if (!h || !ws) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  Geom g;
  int rc = make_geom_decode(h, &g);
  if (rc) return rc;
  *ws = (size_t)carve_decode(nullptr, g, batch ? batch : 1).total;
  return 0;
}

static int decode_impl(const wbpc_header* h, const uint8_t* d_data, u64 nbytes, const u64* d_img_off, uint32_t batch,
                       int level, int planes_dropped, const int32_t* drop_hp, int32_t drop_ll, void* d_out,
                       int out_dtype, int out_layout, void* d_ws, size_t ws_bytes, void* stream,
                       const int* region = nullptr) {
  if (!h || !d_data || !d_out || !d_ws) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  if (h->block_dim != WB_DIM) return fail(WBPC_ERR_UNSUPPORTED, "block_dim %u (only 128 is supported)", h->block_dim);
  if (level < 0 || level > (int)h->levels) return fail(WBPC_ERR_LEVEL_RANGE, "level must be in [0, %u]", h->levels);
  if (planes_dropped < 0) return fail(WBPC_ERR_DOMAIN, "planes_dropped must be >= 0");
  if (!dtype_size(out_dtype)) return fail(WBPC_ERR_INVALID_ARG, "unsupported dtype %d", out_dtype);
  if (h->levels > WB_MAXL) return fail(WBPC_ERR_UNSUPPORTED, "levels %u > %d", h->levels, WB_MAXL);
  Geom g;
  int rc = make_geom_decode(h, &g);
  if (rc) return rc;
  DecWs w = carve_decode(d_ws, g, batch);
  if (w.total > ws_bytes) return fail(WBPC_ERR_WORKSPACE, "workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(w.st, 0xFF, sizeof(u64), s));
  CUDA_TRY(cudaMemsetAsync(&w.st->total, 0, 3 * sizeof(u64), s));
  const u64* img_off = d_img_off;
  if (!img_off) {
    k_set_offsets<<<1, 1, 0, s>>>(w.img_off, nbytes);
    img_off = w.img_off;
  }
  CUDA_TRY(launch_index_check(g, (int)batch, d_data, img_off, w.blk_off, w.blk_len, w.st, s));
  int dh[WB_MAXL + 1] = {0};
  int per_level = drop_hp != nullptr;
  if (per_level)
    for (int i = 0; i < (int)h->levels; ++i) dh[i] = drop_hp[i];
  const uint8_t* need = nullptr;
  if (region) {
    // per-level boxes, even starts, 4-coefficient margin (container.py:365-375)
    const int margin = 4;
    RegionBoxes B;
    std::memset(&B, 0, sizeof B);
    B.r0[level] = region[1];
    B.r1[level] = region[1] + region[3];
    B.c0[level] = region[0];
    B.c1[level] = region[0] + region[2];
    for (int lev = level + 1; lev <= (int)h->levels; ++lev) {
      const int pr0 = B.r0[lev - 1], pr1 = B.r1[lev - 1], pc0 = B.c0[lev - 1], pc1 = B.c1[lev - 1];
      B.r0[lev] = std::max(pr0 / 2 - margin, 0) & ~1;
      B.c0[lev] = std::max(pc0 / 2 - margin, 0) & ~1;
      B.r1[lev] = std::min((pr1 + 1) / 2 + margin, g.lv[lev].h);
      B.c1[lev] = std::min((pc1 + 1) / 2 + margin, g.lv[lev].w);
    }
    CUDA_TRY(launch_region_need(g, level, B, w.need, s));
    need = w.need;
  }
  CUDA_TRY(launch_decode_blocks(g, (int)batch, level, planes_dropped, dh, per_level ? drop_ll : 0, per_level, d_data,
                                nbytes, w.blk_off, w.blk_len, w.tabs, w.flags, w.syms, w.dmeta, w.coef, w.st, s, need));
  const int oc = (h->color_transform == 1 && h->channels == 4) ? 3 : (int)h->channels;
  const LevelGeom& lo = g.lv[level];
  const i64 npix = region ? (i64)region[2] * region[3] : (i64)lo.w * lo.h;
  i64 ostride = npix * oc * dtype_size(out_dtype);
  CUDA_TRY(launch_dwt_inverse(g, (int)batch, level, w.coef, d_out, out_dtype, out_layout, ostride, oc, s, region,
                              &w.st->pad, 1));
  prof_mark("", s);
  return 0;
}

int wbpc_decode(const wbpc_header* h, const uint8_t* d_container, size_t len, int level, int planes_dropped,
                const int32_t* drop_hp, int32_t drop_ll, void* d_out, int out_dtype, int out_layout, void* d_ws,
                size_t ws_bytes, void* stream) {
  return decode_impl(h, d_container, len, nullptr, 1, level, planes_dropped, drop_hp, drop_ll, d_out, out_dtype,
                     out_layout, d_ws, ws_bytes, stream);
}

int wbpc_decode_batch(const wbpc_header* h, const uint8_t* d_data, size_t total_len, const uint64_t* d_img_offsets,
                      uint32_t batch, int level, int planes_dropped, void* d_out, int out_dtype, int out_layout,
                      void* d_ws, size_t ws_bytes, void* stream) {
  if (!d_img_offsets) return fail(WBPC_ERR_INVALID_ARG, "null offsets");
  return decode_impl(h, d_data, total_len, reinterpret_cast<const u64*>(d_img_offsets), batch, level, planes_dropped, nullptr, 0, d_out, out_dtype,
                     out_layout, d_ws, ws_bytes, stream);
}

int wbpc_decode_region(const wbpc_header* h, const uint8_t* d_container, size_t len, int32_t x, int32_t y,
                       int32_t width, int32_t height, int level, int planes_dropped, void* d_out, int out_dtype,
                       int out_layout, void* d_ws, size_t ws_bytes, void* stream) {
  if (!h) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  if (level < 0 || level > (int)h->levels) return fail(WBPC_ERR_LEVEL_RANGE, "level must be in [0, %u]", h->levels);
  if (planes_dropped < 0) return fail(WBPC_ERR_DOMAIN, "planes_dropped must be >= 0");
  int lw = (int)h->width, lh = (int)h->height;
  for (int i = 0; i < level; ++i) {  // level_dims (transforms.py:227-232)
    lw = (lw + 1) / 2;
    lh = (lh + 1) / 2;
  }
  if (width < 1 || height < 1) return fail(WBPC_ERR_DOMAIN, "empty region");
  if (x < 0 || y < 0 || (i64)x + width > lw || (i64)y + height > lh)
    return fail(WBPC_ERR_DOMAIN, "region outside level dimensions");
  const int region[4] = {x, y, width, height};
  return decode_impl(h, d_container, len, nullptr, 1, level, planes_dropped, nullptr, 0, d_out, out_dtype, out_layout,
                     d_ws, ws_bytes, stream, region);
}

int wbpc_block_summary(const wbpc_header* h, const uint8_t* d_container, size_t len, int32_t* d_depth,
                       uint32_t* d_header_bits, void* d_ws, size_t ws_bytes, void* stream) {
  if (!h || !d_container || !d_depth || !d_header_bits || !d_ws) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  if (h->block_dim != WB_DIM) return fail(WBPC_ERR_UNSUPPORTED, "block_dim %u (only 128 is supported)", h->block_dim);
  if (h->levels > WB_MAXL) return fail(WBPC_ERR_UNSUPPORTED, "levels %u > %d", h->levels, WB_MAXL);
  Geom g;
  int rc = make_geom_decode(h, &g);
  if (rc) return rc;
  DecWs w = carve_decode(d_ws, g, 1);
  if (w.total > ws_bytes) return fail(WBPC_ERR_WORKSPACE, "workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(w.st, 0xFF, sizeof(u64), s));
  CUDA_TRY(cudaMemsetAsync(&w.st->total, 0, 3 * sizeof(u64), s));
  k_set_offsets<<<1, 1, 0, s>>>(w.img_off, len);
  CUDA_TRY(launch_index_check(g, 1, d_container, w.img_off, w.blk_off, w.blk_len, w.st, s));
  CUDA_TRY(launch_block_headers(g, 1, d_container, len, w.blk_off, w.blk_len, w.tabs, w.dmeta, w.st, s));
  CUDA_TRY(launch_block_summary(w.tabs, w.blk_off, g.slots_per_image, d_depth, d_header_bits, s));
  prof_mark("", s);
  return 0;
}

int wbpc_truncate_plan_size(const wbpc_header* h, size_t len, size_t* ws, size_t* cap) {
  if (!h || !ws) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  Geom g;
  int rc = make_geom_decode(h, &g);
  if (rc) return rc;
  *ws = (size_t)carve_trunc(nullptr, g).total;
  if (cap) *cap = len;
  return 0;
}

int wbpc_truncate(const wbpc_header* h, const uint8_t* d_container, size_t len, int planes_dropped,
                  const int32_t* drop_hp, int32_t drop_ll, void* d_ws, size_t ws_bytes, uint8_t* d_out,
                  size_t out_cap, uint64_t* d_out_len, void* stream) {
  if (!h || !d_container || !d_ws || !d_out) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  if (planes_dropped < 0) return fail(WBPC_ERR_DOMAIN, "planes_dropped must be >= 0");
  if (h->block_dim != WB_DIM) return fail(WBPC_ERR_UNSUPPORTED, "block_dim %u (only 128 is supported)", h->block_dim);
  if (h->levels > WB_MAXL) return fail(WBPC_ERR_UNSUPPORTED, "levels %u > %d", h->levels, WB_MAXL);
  Geom g;
  int rc = make_geom_decode(h, &g);
  if (rc) return rc;
  TrWs w = carve_trunc(d_ws, g);
  if (w.total > ws_bytes) return fail(WBPC_ERR_WORKSPACE, "workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(w.st, 0xFF, sizeof(u64), s));
  CUDA_TRY(cudaMemsetAsync(&w.st->total, 0, 3 * sizeof(u64), s));
  k_set_offsets<<<1, 1, 0, s>>>(w.img_off, len);
  CUDA_TRY(launch_index_check(g, 1, d_container, w.img_off, w.blk_off, w.blk_len, w.st, s));
  int dh[WB_MAXL + 1] = {0};
  int per_level = drop_hp != nullptr;
  if (per_level)
    for (int i = 0; i < (int)h->levels; ++i) dh[i] = drop_hp[i];
  CUDA_TRY(launch_truncate(g, per_level, planes_dropped, dh, per_level ? drop_ll : 0, d_container, len, w.blk_off,
                           w.blk_len, w.tm, w.sizes, w.new_off, w.img_off, d_out, out_cap, w.st, s));
  prof_mark("", s);
  if (d_out_len) CUDA_TRY(cudaMemcpyAsync(d_out_len, w.img_off + 1, 8, cudaMemcpyDeviceToDevice, s));
  return 0;
}

// Per-kernel device time: every library call ends with an "" mark; the time between a kernel's
// mark and the next mark on the same stream is that kernel's duration.
int wbpc_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_on = on != 0;
  return 0;
}

// Writes up to max_entries aggregated (name, total ms, launches) rows; names '\n'-separated.
int wbpc_profile_collect(char* names, size_t names_len, double* ms, int* counts, int max_entries, int* n_out) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  std::map<std::string, std::pair<double, int>> agg;
  std::vector<std::string> order;
  for (size_t i = 0; i + 1 < g_marks.size(); ++i) {
    if (g_marks[i].name.empty()) continue;
    size_t j = i + 1;
    while (j < g_marks.size() && g_marks[j].s != g_marks[i].s) ++j;
    if (j >= g_marks.size()) break;
    cudaEventSynchronize(g_marks[j].ev);
    float t = 0.f;
    cudaEventElapsedTime(&t, g_marks[i].ev, g_marks[j].ev);
    auto it = agg.find(g_marks[i].name);
    if (it == agg.end()) { order.push_back(g_marks[i].name); agg[g_marks[i].name] = {t, 1}; }
    else { it->second.first += t; it->second.second += 1; }
  }
  for (auto& m : g_marks) g_pool.push_back(m.ev);
  g_marks.clear();
  std::string all;
  int n = 0;
  for (auto& k : order) {
    if (n >= max_entries) break;
    ms[n] = agg[k].first;
    counts[n] = agg[k].second;
    all += k;
    all += "\n";
    ++n;
  }
  if (names && names_len) {
    size_t c = std::min(names_len - 1, all.size());
    memcpy(names, all.data(), c);
    names[c] = 0;
  }
  if (n_out) *n_out = n;
  return 0;
}


// ---- block API (encode_block / decode_block / truncate_block, blocks.py:84-304) -----------------
__global__ void k_depth_to_bmax(const int32_t* depth, unsigned* bmax, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int d = depth[i];
  bmax[i] = d <= 1 ? 0u : (1u << (d - 2));  // 1 + bit_length(bmax) == d
}

int wbpc_block_plan_size(int kind, uint32_t n, size_t* ws, size_t* cap) {
  if (!ws) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  Geom g;
  int rc = make_geom_raw(kind, n, &g);
  if (rc) return rc;
  const EncWs e = carve_encode(nullptr, g, 1);
  const DecWs d = carve_decode(nullptr, g, 1);
  const TrWs t = carve_trunc(nullptr, g);
  *ws = (size_t)std::max(e.total, std::max(d.total, t.total));
  if (cap) *cap = (size_t)n * ((kind ? 3 : 1) * 128ull * 128 * 8 + 1024);
  return 0;
}

int wbpc_encode_blocks(int kind, uint32_t n, const int32_t* d_coeffs, const int32_t* d_depth, void* d_ws,
                       size_t ws_bytes, uint8_t* d_out, size_t out_cap, uint64_t* d_offsets, void* stream) {
  if (!d_coeffs || !d_ws || !d_out || !d_offsets) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  Geom g;
  int rc = make_geom_raw(kind, n, &g);
  if (rc) return rc;
  EncWs w = carve_encode(d_ws, g, 1);
  if (w.total > ws_bytes) return fail(WBPC_ERR_WORKSPACE, "workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(w.st, 0xFF, sizeof(u64), s));
  CUDA_TRY(cudaMemsetAsync(&w.st->total, 0, 3 * sizeof(u64), s));
  CUDA_TRY(launch_raw_bmax(g, (int)n, d_coeffs, w.bmax, w.st, s));
  if (d_depth) k_depth_to_bmax<<<(n + 255) / 256, 256, 0, s>>>(d_depth, w.bmax, (int)n);
  CUDA_TRY(launch_encode_blocks(g, 1, d_coeffs, w.bmax, w.syms, w.wbits, w.meta, w.stats, w.zmask, w.sizes, w.block_off, w.img_off, d_out, out_cap,
                                w.st, s));
  prof_mark("", s);
  CUDA_TRY(cudaMemcpyAsync(d_offsets, w.block_off, 8ull * n, cudaMemcpyDeviceToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(d_offsets + n, w.img_off + 1, 8, cudaMemcpyDeviceToDevice, s));
  return 0;
}

int wbpc_decode_blocks(int kind, uint32_t n, const uint8_t* d_data, size_t len, const uint64_t* d_offsets,
                       int planes_to_keep, int32_t* d_coeffs_out, void* d_ws, size_t ws_bytes, void* stream) {
  if (!d_data || !d_offsets || !d_coeffs_out || !d_ws) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  if (len >= (1ull << 32) - 64) return fail(WBPC_ERR_UNSUPPORTED, "block data >= 4 GiB per call");
  Geom g;
  int rc = make_geom_raw(kind, n, &g);
  if (rc) return rc;
  g.keep = planes_to_keep < 0 ? -1 : planes_to_keep;
  DecWs w = carve_decode(d_ws, g, 1);
  if (w.total > ws_bytes) return fail(WBPC_ERR_WORKSPACE, "workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(w.st, 0xFF, sizeof(u64), s));
  CUDA_TRY(cudaMemsetAsync(&w.st->total, 0, 3 * sizeof(u64), s));
  CUDA_TRY(launch_raw_index(reinterpret_cast<const u64*>(d_offsets), (int)n, w.blk_off, w.blk_len, s));
  int dh[WB_MAXL + 1] = {0};
  CUDA_TRY(launch_decode_blocks(g, 1, 0, 0, dh, 0, 0, d_data, len, w.blk_off, w.blk_len, w.tabs, w.flags, w.syms,
                                w.dmeta, d_coeffs_out, w.st, s, nullptr));
  prof_mark("", s);
  return 0;
}

int wbpc_plane_offsets(int kind, const uint8_t* d_block, size_t len, int32_t* d_slots, uint32_t* d_offsets,
                       int32_t* d_count, void* d_ws, size_t ws_bytes, void* stream) {
  if (!d_block || !d_slots || !d_offsets || !d_count || !d_ws) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  Geom g;
  int rc = make_geom_raw(kind, 1, &g);
  if (rc) return rc;
  DecWs w = carve_decode(d_ws, g, 1);
  if (w.total > ws_bytes) return fail(WBPC_ERR_WORKSPACE, "workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(w.st, 0xFF, sizeof(u64), s));
  CUDA_TRY(cudaMemsetAsync(&w.st->total, 0, 3 * sizeof(u64), s));
  k_set_offsets<<<1, 1, 0, s>>>(w.img_off, len);
  CUDA_TRY(launch_raw_index(w.img_off, 1, w.blk_off, w.blk_len, s));
  CUDA_TRY(launch_block_headers(g, 1, d_block, len, w.blk_off, w.blk_len, w.tabs, w.dmeta, w.st, s));
  CUDA_TRY(launch_plane_offsets(w.tabs, d_slots, d_offsets, d_count, s));
  prof_mark("", s);
  return 0;
}

int wbpc_truncate_blocks(int kind, uint32_t n, const uint8_t* d_data, size_t len, const uint64_t* d_offsets,
                         int planes_dropped, void* d_ws, size_t ws_bytes, uint8_t* d_out, size_t out_cap,
                         uint64_t* d_out_offsets, void* stream) {
  if (!d_data || !d_offsets || !d_out || !d_out_offsets || !d_ws) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  if (planes_dropped < 0) return fail(WBPC_ERR_DOMAIN, "planes_dropped must be >= 0");
  Geom g;
  int rc = make_geom_raw(kind, n, &g);
  if (rc) return rc;
  TrWs w = carve_trunc(d_ws, g);
  if (w.total > ws_bytes) return fail(WBPC_ERR_WORKSPACE, "workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(w.st, 0xFF, sizeof(u64), s));
  CUDA_TRY(cudaMemsetAsync(&w.st->total, 0, 3 * sizeof(u64), s));
  CUDA_TRY(launch_raw_index(reinterpret_cast<const u64*>(d_offsets), (int)n, w.blk_off, w.blk_len, s));
  int dh[WB_MAXL + 1] = {0};
  CUDA_TRY(launch_truncate(g, 0, planes_dropped, dh, 0, d_data, len, w.blk_off, w.blk_len, w.tm, w.sizes, w.new_off,
                           w.img_off, d_out, out_cap, w.st, s));
  prof_mark("", s);
  CUDA_TRY(cudaMemcpyAsync(d_out_offsets, w.new_off, 8ull * n, cudaMemcpyDeviceToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(d_out_offsets + n, w.img_off + 1, 8, cudaMemcpyDeviceToDevice, s));
  return 0;
}

// Sized copy: *d_nbytes (device resident) bytes from src to dst, any device-accessible
// pointers -- device memory or pinned host memory (unified addressing).  Lets a host-buffer
// pipeline move a container whose length is known only on the device without a host round
// trip; PCIe transfers issued by SMs also do not queue behind copy-engine transfers.
// A small grid (PCIe latency x bandwidth ~ 100 KB in flight: 64 CTAs x 128 threads x 2 x 16 B)
// so that the copy leaves the SMs to concurrently running codec kernels.
__global__ void __launch_bounds__(128) k_copy_sized(uint8_t* dst, const uint8_t* src, const u64* d_nbytes) {
  const u64 n = *d_nbytes;
  const u64 tid = (u64)blockIdx.x * blockDim.x + threadIdx.x, nth = (u64)gridDim.x * blockDim.x;
  const bool al = (((uintptr_t)dst | (uintptr_t)src) & 15) == 0;
  const u64 n16 = al ? n / 16 : 0;
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  u64 i = tid;
  for (; i + nth < n16; i += 2 * nth) {
    const uint4 a = s4[i], b = s4[i + nth];
    d4[i] = a;
    d4[i + nth] = b;
  }
  for (; i < n16; i += nth) d4[i] = s4[i];
  for (u64 j = 16 * n16 + tid; j < n; j += nth) dst[j] = src[j];
}

int wbpc_copy_sized(void* dst, const void* src, const uint64_t* d_nbytes, void* stream) {
  if (!dst || !src || !d_nbytes) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  k_copy_sized<<<64, 128, 0, s>>>(reinterpret_cast<uint8_t*>(dst), reinterpret_cast<const uint8_t*>(src),
                                      reinterpret_cast<const u64*>(d_nbytes));
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// ---------------------------------------------------------------------------- tile archive
int wbpc_archive_tile_sizes(const uint64_t* d_enc_offsets, uint32_t batch, uint32_t n_local, uint32_t per,
                            uint64_t* d_sizes, void* stream) {
  if (!d_enc_offsets || !d_sizes || batch == 0 || per < n_local) return fail(WBPC_ERR_INVALID_ARG, "bad arguments");
  if (per == 0) return 0;
  CUDA_TRY(launch_tile_sizes(reinterpret_cast<const u64*>(d_enc_offsets), (int)batch, (int)n_local, (int)per,
                             reinterpret_cast<u64*>(d_sizes), (cudaStream_t)stream));
  prof_mark("", (cudaStream_t)stream);
  return 0;
}

int wbpc_archive_index(const uint64_t* d_sizes_all, uint32_t n_tiles, uint32_t tiles_x, uint32_t tiles_y,
                       uint32_t first, uint32_t n_local, uint8_t* d_header, uint64_t* d_local_offsets,
                       uint64_t* d_base_total, void* stream) {
  if (!d_sizes_all || (u64)tiles_x * tiles_y != n_tiles || (u64)first + n_local > n_tiles)
    return fail(WBPC_ERR_INVALID_ARG, "archive index: tiles_x * tiles_y must equal n_tiles and the shard lie inside");
  CUDA_TRY(launch_archive_index(reinterpret_cast<const u64*>(d_sizes_all), (int)n_tiles, (int)tiles_x, (int)tiles_y,
                                (int)first, (int)n_local, d_header, reinterpret_cast<u64*>(d_local_offsets),
                                reinterpret_cast<u64*>(d_base_total), (cudaStream_t)stream));
  prof_mark("", (cudaStream_t)stream);
  return 0;
}

int wbpc_archive_gather(const uint8_t* d_store, uint64_t region_bytes, const uint64_t* d_enc_offsets, uint32_t batch,
                        uint32_t n_local, uint8_t* d_dst, const uint64_t* d_local_offsets, void* stream) {
  if (!d_store || !d_enc_offsets || !d_dst || !d_local_offsets || batch == 0)
    return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  CUDA_TRY(launch_gather_tiles(d_store, region_bytes, reinterpret_cast<const u64*>(d_enc_offsets), (int)batch,
                               (int)n_local, d_dst, reinterpret_cast<const u64*>(d_local_offsets),
                               (cudaStream_t)stream));
  prof_mark("", (cudaStream_t)stream);
  return 0;
}

int wbpc_archive_batch_offsets(const uint64_t* d_enc_offsets_k, uint32_t batch_tiles, uint64_t* d_local_offsets_k,
                               void* stream) {
  if (!d_enc_offsets_k || !d_local_offsets_k || batch_tiles == 0 || batch_tiles > 1023)
    return fail(WBPC_ERR_INVALID_ARG, "bad arguments");
  CUDA_TRY(launch_batch_offsets(reinterpret_cast<const u64*>(d_enc_offsets_k), (int)batch_tiles,
                                reinterpret_cast<u64*>(d_local_offsets_k), (cudaStream_t)stream));
  return 0;
}

int wbpc_query_status(const void* d_ws, void* stream, int32_t* status, uint64_t* aux) {
  if (!d_ws || !status) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  DevStatus hs;
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemcpyAsync(&hs, d_ws, sizeof hs, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (hs.key == ~0ull) {
    *status = 0;
    if (aux) *aux = hs.total;
    return 0;
  }
  *status = (int32_t)(hs.key & 0xFF);
  if (aux) *aux = *status == WBPC_ERR_OUT_CAPACITY ? hs.aux : ((hs.key >> 8) & 0xFFFFFFFFFFFull);
  return 0;
}

int wbpc_decode_tokens(const uint8_t* d_payload, int64_t start_bit, int64_t end_bit, const int32_t* d_left,
                       const int32_t* d_right, const int32_t* d_leaf_symbol, int32_t n_nodes, int32_t zr_symbol,
                       int32_t counter_width, const int64_t* d_seg_lengths, int32_t n_segments, uint8_t* d_out_symbols,
                       int64_t* d_out_seg_starts, int64_t* d_result, void* stream) {
  (void)n_nodes;
  if (!d_payload || !d_left || !d_right || !d_leaf_symbol || !d_result) return fail(WBPC_ERR_INVALID_ARG, "null pointer");
  u64 nbytes = (u64)((end_bit + 7) / 8);
  CUDA_TRY(launch_decode_tokens(d_payload, nbytes, start_bit, end_bit, d_left, d_right, d_leaf_symbol, zr_symbol,
                                counter_width, (const i64*)d_seg_lengths, n_segments, d_out_symbols,
                                (i64*)d_out_seg_starts, (i64*)d_result, (cudaStream_t)stream));
  return 0;
}

}  // extern "C"
