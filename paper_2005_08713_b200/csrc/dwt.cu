// dwt.cu — reversible colour transform + 5/3 integer lifting DWT, forward and inverse (sm_100a).
//
// Replaces (reference /root/reference/pkg/src/wbpc):
//   rct_forward / rct_inverse          transforms.py:79-104
//   _split_axis0 / _merge_axis0        transforms.py:107-162
//   _split_plane / _merge_plane        transforms.py:184-199
//   dwt2d_forward (recursion on LL)    transforms.py:202-216
//   decode_image level loop            container.py:324-335, _finish_image :301-306
//
// One CTA computes a TX x TY tile of every subband of one level (forward) or the matching
// 2TX x 2TY parent tile (inverse).  The input tile plus its 2-sample lifting halo is staged in
// shared memory; image edges use whole-sample symmetric extension, implemented by reflecting
// the load index (exactly the reference's mirroring for even/odd lengths and n == 1).  Rows
// are lifted first, then columns (forward); columns first, then rows (inverse), which pins the
// reference's H-then-V order.  All arithmetic is int32 with arithmetic shifts (floor), the
// static coefficient bound computed on the host guarantees no overflow.
//
// HBM traffic per level is one read of the input plane and one write of the four subbands;
// every tile writes its padded 128x128 block area so the block coder never bounds-checks.
#include "common.cuh"

namespace wb {

constexpr int TX = 32;            // subband tile width (one warp per row on store)
constexpr int TY = 16;            // subband tile height
constexpr int RW = 2 * TX + 3;    // staged input cols (2-left, 1-right halo + 1)
constexpr int RH = 2 * TY + 3;
constexpr int NT = 256;

struct FwdParams {
  Geom g;
  int level;               // producing level l (1..L)
  const void* src;         // level 1: image; level >1: coefficient base
  int src_dtype, src_layout;
  i64 src_img_stride;      // bytes between images (level 1)
  int32_t* coef;           // coefficient base (image-major: img_stride elements per image)
  unsigned* bmax;          // per (image, slot) max |c|
  DevStatus* st;
};

template <typename T>
static __device__ __forceinline__ int load_sample(const T* p) { return (int)*p; }

// Sample (channel ch, row y, col x) of image b from the raw pixel buffer.
static __device__ __forceinline__ int load_pixel(const FwdParams& P, int b, int ch, int y, int x) {
  const Geom& g = P.g;
  const char* base = (const char*)P.src + (i64)b * P.src_img_stride;
  i64 idx = P.src_layout == WBPC_LAYOUT_HWC ? ((i64)y * g.W + x) * g.C + ch : ((i64)ch * g.H + y) * g.W + x;
  switch (P.src_dtype) {
    case WBPC_DTYPE_U8: return ((const uint8_t*)base)[idx];
    case WBPC_DTYPE_U16: return ((const uint16_t*)base)[idx];
    case WBPC_DTYPE_I16: return ((const int16_t*)base)[idx];
    default: return ((const int32_t*)base)[idx];
  }
}

// Horizontal then vertical lifting of the staged tile X (RH x RW) -> 4 subband tiles; writes
// results to global and returns per-subband max |c| via smem reduce.
static __device__ void lift_fwd_tile(const FwdParams& P, int (*X)[RW], int (*Lx)[TX], int (*Hx)[TX + 1],
                              int (*VH)[TY + 1][TX], int32_t* chan_base, int n0x, int n0y,
                              unsigned* red, int is_top) {
  const Geom& g = P.g;
  const LevelGeom& lg = g.lv[P.level];
  const int tid = threadIdx.x;
  // horizontal highs: k in [0, TX] <-> n = n0x-1+k  (transforms.py:125)
  for (int i = tid; i < RH * (TX + 1); i += NT) {
    int r = i / (TX + 1), k = i - r * (TX + 1);
    Hx[r][k] = X[r][2 * k + 1] - ((X[r][2 * k] + X[r][2 * k + 2]) >> 1);
  }
  __syncthreads();
  // horizontal lows: k in [0, TX) <-> n = n0x+k  (transforms.py:133)
  for (int i = tid; i < RH * TX; i += NT) {
    int r = i / TX, k = i - r * TX;
    Lx[r][k] = X[r][2 * k + 2] + ((Hx[r][k] + Hx[r][k + 1] + 2) >> 2);
  }
  __syncthreads();
  // vertical highs of Lx (-> LH) and Hx (-> HH): k in [0, TY] <-> n = n0y-1+k
  for (int i = tid; i < 2 * (TY + 1) * TX; i += NT) {
    int a = i / ((TY + 1) * TX), rem = i - a * (TY + 1) * TX;
    int k = rem / TX, x = rem - k * TX;
    int v;
    if (a == 0) v = Lx[2 * k + 1][x] - ((Lx[2 * k][x] + Lx[2 * k + 2][x]) >> 1);
    else v = Hx[2 * k + 1][x + 1] - ((Hx[2 * k][x + 1] + Hx[2 * k + 2][x + 1]) >> 1);
    VH[a][k][x] = v;
  }
  __syncthreads();
  unsigned mhp = 0, mll = 0;
  // vertical lows + stores.  Each thread: 2 (arrays) x TY x TX / NT = 4 outputs per array pair.
  for (int i = tid; i < TY * TX; i += NT) {
    int k = i / TX, x = i - k * TX;
    int ll = Lx[2 * k + 2][x] + ((VH[0][k][x] + VH[0][k + 1][x] + 2) >> 2);
    int hl = Hx[2 * k + 2][x + 1] + ((VH[1][k][x] + VH[1][k + 1][x] + 2) >> 2);
    int lh = VH[0][k + 1][x];
    int hh = VH[1][k + 1][x];
    int gx = n0x + x, gy = n0y + k;
    // subband true dims (container.py:132-137): LL (cw,ch) LH (cw,fh) HL (fw,ch) HH (fw,fh)
    if (!(gx < lg.sw[0] && gy < lg.sh[0])) ll = 0;
    if (!(gx < lg.sw[1] && gy < lg.sh[1])) lh = 0;
    if (!(gx < lg.sw[2] && gy < lg.sh[2])) hl = 0;
    if (!(gx < lg.sw[3] && gy < lg.sh[3])) hh = 0;
    i64 o = (i64)gy * lg.pw + gx;
    chan_base[lg.off[0] + o] = ll;
    chan_base[lg.off[1] + o] = lh;
    chan_base[lg.off[2] + o] = hl;
    chan_base[lg.off[3] + o] = hh;
    mhp = max(mhp, max((unsigned)abs(lh), max((unsigned)abs(hl), (unsigned)abs(hh))));
    mll = max(mll, (unsigned)abs(ll));
  }
  // reduce max over the CTA
  for (int o = 16; o > 0; o >>= 1) {
    mhp = max(mhp, __shfl_xor_sync(0xffffffffu, mhp, o));
    mll = max(mll, __shfl_xor_sync(0xffffffffu, mll, o));
  }
  if ((tid & 31) == 0) { red[tid >> 5] = mhp; red[8 + (tid >> 5)] = mll; }
  __syncthreads();
  if (tid == 0) {
    unsigned a = 0, b = 0;
    for (int w = 0; w < NT / 32; ++w) { a = max(a, red[w]); b = max(b, red[8 + w]); }
    red[16] = a;
    red[17] = b;
  }
  __syncthreads();
  (void)is_top;
}

__global__ void __launch_bounds__(NT) k_dwt_fwd(FwdParams P) {
  __shared__ int X[3][RH][RW];
  __shared__ int Lx[RH][TX];
  __shared__ int Hx[RH][TX + 1];
  __shared__ int VH[2][TY + 1][TX];
  __shared__ unsigned red[20];
  const Geom& g = P.g;
  const int lev = P.level;
  const LevelGeom& lg = g.lv[lev];
  const LevelGeom& pg = g.lv[lev - 1];
  const int n0x = blockIdx.x * TX, n0y = blockIdx.y * TY;
  const int pw_true = pg.w, ph_true = pg.h;  // parent (input) dims
  const int tid = threadIdx.x;
  const bool first = lev == 1;
  const int nimg_ch = first ? 1 : g.C;
  const int b = blockIdx.z / nimg_ch;
  const int ch0 = first ? 0 : blockIdx.z % nimg_ch;
  const int ch1 = first ? g.C : ch0 + 1;
  int32_t* img_coef = P.coef + (i64)b * g.img_stride;
  const int x0 = 2 * n0x - 2, y0 = 2 * n0y - 2;
  const int by = n0y / WB_DIM, bx = n0x / WB_DIM;
  const int is_top = lev == g.L;

  if (first && g.rct) {
    // stage R,G,B, apply the RCT in place (transforms.py:86-88): Y=(R+2G+B)>>2, Cb=B-G, Cr=R-G
    const int lim = 1 << g.bd;
    bool bad = false;
    for (int i = tid; i < RH * RW; i += NT) {
      int r = i / RW, c = i - r * RW;
      int gy = reflect_pos(y0 + r, ph_true), gx = reflect_pos(x0 + c, pw_true);
      int R = load_pixel(P, b, 0, gy, gx), G = load_pixel(P, b, 1, gy, gx), B = load_pixel(P, b, 2, gy, gx);
      bad |= (unsigned)R >= (unsigned)lim || (unsigned)G >= (unsigned)lim || (unsigned)B >= (unsigned)lim;
      X[0][r][c] = (R + 2 * G + B) >> 2;
      X[1][r][c] = B - G;
      X[2][r][c] = R - G;
    }
    if (bad) record_error(P.st, WBPC_ERR_DOMAIN, 0, 0);  // validate_source, transforms.py:57-62
    __syncthreads();
    for (int ch = 0; ch < 3; ++ch) {
      int32_t* cb = img_coef + (i64)ch * g.chan_stride;
      lift_fwd_tile(P, X[ch], Lx, Hx, VH, cb, n0x, n0y, red, is_top);
      if (tid == 0) {
        unsigned* bm = P.bmax + (i64)b * g.slots_per_image + (i64)ch * g.slots_per_channel;
        atomicMax(&bm[lg.slot0 + by * lg.gw + bx], red[16]);
        if (is_top) atomicMax(&bm[by * lg.gw + bx], red[17]);
      }
      __syncthreads();
    }
    return;
  }
  for (int ch = ch0; ch < ch1; ++ch) {
    if (first) {
      const int lim = 1 << g.bd;
      bool bad = false;
      for (int i = tid; i < RH * RW; i += NT) {
        int r = i / RW, c = i - r * RW;
        int gy = reflect_pos(y0 + r, ph_true), gx = reflect_pos(x0 + c, pw_true);
        int v = load_pixel(P, b, ch, gy, gx);
        bad |= (unsigned)v >= (unsigned)lim;
        X[0][r][c] = v;
      }
      if (bad) record_error(P.st, WBPC_ERR_DOMAIN, 0, 0);
    } else {
      const int32_t* src = img_coef + (i64)ch * g.chan_stride + pg.off[0];
      for (int i = tid; i < RH * RW; i += NT) {
        int r = i / RW, c = i - r * RW;
        int gy = reflect_pos(y0 + r, ph_true), gx = reflect_pos(x0 + c, pw_true);
        X[0][r][c] = src[(i64)gy * pg.pw + gx];
      }
    }
    __syncthreads();
    int32_t* cb = img_coef + (i64)ch * g.chan_stride;
    lift_fwd_tile(P, X[0], Lx, Hx, VH, cb, n0x, n0y, red, is_top);
    if (tid == 0) {
      unsigned* bm = P.bmax + (i64)b * g.slots_per_image + (i64)ch * g.slots_per_channel;
      atomicMax(&bm[lg.slot0 + by * lg.gw + bx], red[16]);
      if (is_top) atomicMax(&bm[by * lg.gw + bx], red[17]);
    }
    __syncthreads();
  }
}

// L == 0: the LL grid is the (colour transformed) image itself, zero padded to 128 multiples.
__global__ void __launch_bounds__(NT) k_level0(FwdParams P) {
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
    for (int ch = 0; ch < g.C; ++ch) {
      v[ch] = load_pixel(P, b, ch, y, x);
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
  int32_t* img_coef = P.coef + (i64)b * g.img_stride;
  for (int ch = 0; ch < g.C; ++ch) {
    img_coef[(i64)ch * g.chan_stride + lg.off[0] + (i64)y * lg.pw + x] = v[ch];
    m[ch] = (unsigned)abs(v[ch]);
  }
  for (int ch = 0; ch < 4; ++ch)
    for (int o = 16; o > 0; o >>= 1) m[ch] = max(m[ch], __shfl_xor_sync(0xffffffffu, m[ch], o));
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

// ------------------------------------------------------------------------------- inverse
struct InvParams {
  Geom g;
  int level;           // merging level l (LL_l + details_l -> LL_{l-1})
  int32_t* coef;
  void* out;           // final output (when level == out_level + 1 && fused) else null
  int out_dtype, out_layout;
  i64 out_img_stride;  // bytes
  int out_channels;    // channels written (3 for RCT containers claiming 4)
};

static __device__ __forceinline__ void store_sample(void* base, int dtype, i64 idx, int v) {
  switch (dtype) {
    case WBPC_DTYPE_U8: ((uint8_t*)base)[idx] = (uint8_t)v; break;
    case WBPC_DTYPE_U16: ((uint16_t*)base)[idx] = (uint16_t)v; break;
    case WBPC_DTYPE_I16: ((int16_t*)base)[idx] = (int16_t)v; break;
    default: ((int32_t*)base)[idx] = v; break;
  }
}

// Loads subband value with reflected indices; `hy`/`hx` say whether the subband is high-pass
// along y/x.  ny/nx = signal lengths (parent dims).  Empty high band (n == 1) reads 0.
static __device__ __forceinline__ int load_sb(const int32_t* p, int pitch, int ky, int kx, int hy, int hx, int ny, int nx) {
  int py = 2 * ky + hy, px = 2 * kx + hx;
  if ((hy && ny == 1) || (hx && nx == 1)) return 0;
  py = reflect_pos(py, ny);
  px = reflect_pos(px, nx);
  return p[(i64)(py >> 1) * pitch + (px >> 1)];
}

// Inverse lifting of one channel's tile: S = 4 staged subbands (TY+2)x(TX+2) -> O (2TY x 2TX).
static __device__ void lift_inv_tile(int (*S)[TY + 2][TX + 2], int (*Lx)[TX + 2], int (*Hx)[TX + 2],
                              int (*XE)[TY + 1][TX + 2], int (*O)[2 * TX]) {
  const int tid = threadIdx.x;
  // vertical: xe[n] = low[n] - ((h[n-1] + h[n] + 2) >> 2), n = n0y + i, i in [0, TY]
  for (int i = tid; i < 2 * (TY + 1) * (TX + 2); i += NT) {
    int a = i / ((TY + 1) * (TX + 2)), rem = i - a * (TY + 1) * (TX + 2);
    int k = rem / (TX + 2), x = rem - k * (TX + 2);
    const int lo = a == 0 ? 0 : 2, hi = a == 0 ? 1 : 3;  // (LL,LH) or (HL,HH)
    XE[a][k][x] = S[lo][1 + k][x] - ((S[hi][k][x] + S[hi][1 + k][x] + 2) >> 2);
  }
  __syncthreads();
  for (int i = tid; i < 2 * TY * (TX + 2); i += NT) {
    int a = i / (TY * (TX + 2)), rem = i - a * TY * (TX + 2);
    int k = rem / (TX + 2), x = rem - k * (TX + 2);
    const int hi = a == 0 ? 1 : 3;
    int xe = XE[a][k][x];
    int xo = S[hi][1 + k][x] + ((xe + XE[a][k + 1][x]) >> 1);
    if (a == 0) { Lx[2 * k][x] = xe; Lx[2 * k + 1][x] = xo; }
    else { Hx[2 * k][x] = xe; Hx[2 * k + 1][x] = xo; }
  }
  __syncthreads();
  // horizontal per row y in [0, 2TY): xe at i in [0, TX], xo at i in [0, TX)
  for (int i = tid; i < 2 * TY * TX; i += NT) {
    int y = i / TX, k = i - y * TX;
    int xe0 = Lx[y][1 + k] - ((Hx[y][k] + Hx[y][1 + k] + 2) >> 2);
    int xe1 = Lx[y][2 + k] - ((Hx[y][1 + k] + Hx[y][2 + k] + 2) >> 2);
    int xo = Hx[y][1 + k] + ((xe0 + xe1) >> 1);
    O[y][2 * k] = xe0;
    O[y][2 * k + 1] = xo;
  }
  __syncthreads();
}

// Dynamic smem: S[4] + Lx + Hx + XE[2] + O[C]
constexpr int INV_S_BYTES = 4 * (TY + 2) * (TX + 2) * 4;
constexpr int INV_LX_BYTES = 2 * (2 * TY) * (TX + 2) * 4;  // Lx and Hx
constexpr int INV_XE_BYTES = 2 * (TY + 1) * (TX + 2) * 4;
constexpr int INV_O_BYTES = 2 * TY * 2 * TX * 4;

__global__ void __launch_bounds__(NT) k_dwt_inv(InvParams P) {
  extern __shared__ int smem[];
  int (*S)[TY + 2][TX + 2] = (int (*)[TY + 2][TX + 2])smem;
  int (*Lx)[TX + 2] = (int (*)[TX + 2])(smem + INV_S_BYTES / 4);
  int (*Hx)[TX + 2] = (int (*)[TX + 2])(smem + INV_S_BYTES / 4 + INV_LX_BYTES / 8);  // second half
  int (*XE)[TY + 1][TX + 2] = (int (*)[TY + 1][TX + 2])(smem + (INV_S_BYTES + INV_LX_BYTES) / 4);
  int* obase = smem + (INV_S_BYTES + INV_LX_BYTES + INV_XE_BYTES) / 4;
  const Geom& g = P.g;
  const int lev = P.level;
  const LevelGeom& lg = g.lv[lev];
  const LevelGeom& pg = g.lv[lev - 1];
  const int fused = P.out != nullptr;
  const int nch = fused ? g.C : 1;
  const int b = fused ? blockIdx.z : blockIdx.z / g.C;
  const int chs = fused ? 0 : blockIdx.z % g.C;
  const int n0x = blockIdx.x * TX, n0y = blockIdx.y * TY;
  const int tid = threadIdx.x;
  int32_t* img_coef = P.coef + (i64)b * g.img_stride;
  const int NY = pg.h, NX = pg.w;
  for (int cc = 0; cc < nch; ++cc) {
    const int ch = chs + cc;
    int32_t* cb = img_coef + (i64)ch * g.chan_stride;
    for (int i = tid; i < 4 * (TY + 2) * (TX + 2); i += NT) {
      int s = i / ((TY + 2) * (TX + 2)), rem = i - s * (TY + 2) * (TX + 2);
      int ky = rem / (TX + 2), kx = rem - ky * (TX + 2);
      // subband s: 0 LL (lo,lo) 1 LH (x lo, y hi) 2 HL (x hi, y lo) 3 HH
      int hy = (s == 1 || s == 3), hx = (s == 2 || s == 3);
      S[s][ky][kx] = load_sb(cb + lg.off[s], lg.pw, n0y - 1 + ky, n0x - 1 + kx, hy, hx, NY, NX);
    }
    __syncthreads();
    int (*O)[2 * TX] = (int (*)[2 * TX])(obase + (fused ? cc : 0) * (2 * TY * 2 * TX));
    lift_inv_tile(S, Lx, Hx, XE, O);
    if (!fused) {
      int32_t* dst = cb + pg.off[0];
      for (int i = tid; i < 2 * TY * 2 * TX; i += NT) {
        int y = i / (2 * TX), x = i - y * (2 * TX);
        int gy = 2 * n0y + y, gx = 2 * n0x + x;
        if (gy < pg.ph && gx < pg.pw) dst[(i64)gy * pg.pw + gx] = O[y][x];
      }
      __syncthreads();
    }
  }
  if (!fused) return;
  // final level: inverse RCT (transforms.py:101-103, no clamp) + format conversion
  const int OC = P.out_channels;
  char* ob = (char*)P.out + (i64)b * P.out_img_stride;
  for (int i = tid; i < 2 * TY * 2 * TX; i += NT) {
    int y = i / (2 * TX), x = i - y * (2 * TX);
    int gy = 2 * n0y + y, gx = 2 * n0x + x;
    if (gy >= NY || gx >= NX) continue;
    int v[4];
    for (int c = 0; c < g.C; ++c) v[c] = obase[c * (2 * TY * 2 * TX) + i];
    if (g.rct) {
      int Y = v[0], Cb = v[1], Cr = v[2];
      int G = Y - ((Cb + Cr) >> 2);
      v[0] = Cr + G;
      v[1] = G;
      v[2] = Cb + G;
    }
    for (int c = 0; c < OC; ++c) {
      i64 idx = P.out_layout == WBPC_LAYOUT_HWC ? ((i64)gy * NX + gx) * OC + c : ((i64)c * NY + gy) * NX + gx;
      store_sample(ob, P.out_dtype, idx, v[c]);
    }
  }
}

// Output from the LL planes at `level` (decode_image(level>0) or L == 0).
__global__ void k_finish(InvParams P) {
  const Geom& g = P.g;
  const LevelGeom& lg = g.lv[P.level];
  const int b = blockIdx.z;
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
  const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (x >= lg.w || y >= lg.h) return;
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
    i64 idx = P.out_layout == WBPC_LAYOUT_HWC ? ((i64)y * lg.w + x) * OC + c : ((i64)c * lg.h + y) * lg.w + x;
    store_sample(ob, P.out_dtype, idx, v[c]);
  }
}

// ------------------------------------------------------------------------------ launchers
cudaError_t launch_dwt_forward(const Geom& g, int batch, const void* src, int dtype, int layout, i64 img_stride,
                               int32_t* coef, unsigned* bmax, DevStatus* st, cudaStream_t s) {
  FwdParams P;
  P.g = g;
  P.src = src;
  P.src_dtype = dtype;
  P.src_layout = layout;
  P.src_img_stride = img_stride;
  P.coef = coef;
  P.bmax = bmax;
  P.st = st;
  if (g.L == 0) {
    P.level = 0;
    const LevelGeom& lg = g.lv[0];
    dim3 grid(lg.pw / 32, lg.ph / 8, batch);
    prof_mark("level0", s);
    k_level0<<<grid, NT, 0, s>>>(P);
    return cudaGetLastError();
  }
  for (int l = 1; l <= g.L; ++l) {
    P.level = l;
    const LevelGeom& lg = g.lv[l];
    dim3 grid(lg.pw / TX, lg.ph / TY, l == 1 ? batch : batch * g.C);
    prof_mark(l == 1 ? "dwt_fwd_l1" : "dwt_fwd", s);
    k_dwt_fwd<<<grid, NT, 0, s>>>(P);
  }
  return cudaGetLastError();
}

cudaError_t launch_dwt_inverse(const Geom& g, int batch, int out_level, int32_t* coef, void* out, int out_dtype,
                               int out_layout, i64 out_img_stride, int out_channels, cudaStream_t s) {
  InvParams P;
  P.g = g;
  P.coef = coef;
  P.out_dtype = out_dtype;
  P.out_layout = out_layout;
  P.out_img_stride = out_img_stride;
  P.out_channels = out_channels;
  static bool attr_set = false;
  const int smem_fused = INV_S_BYTES + INV_LX_BYTES + INV_XE_BYTES + 4 * INV_O_BYTES;
  if (!attr_set) {
    cudaFuncSetAttribute(k_dwt_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_fused);
    attr_set = true;
  }
  for (int l = g.L; l > out_level; --l) {
    P.level = l;
    const LevelGeom& lg = g.lv[l];
    const bool fuse = (l == out_level + 1) && out_level == 0;
    P.out = fuse ? out : nullptr;
    dim3 grid(lg.pw / TX, lg.ph / TY, fuse ? batch : batch * g.C);
    int smem = INV_S_BYTES + INV_LX_BYTES + INV_XE_BYTES + (fuse ? g.C : 1) * INV_O_BYTES;
    prof_mark(fuse ? "dwt_inv_l1" : "dwt_inv", s);
    k_dwt_inv<<<grid, NT, smem, s>>>(P);
  }
  if (out_level > 0 || g.L == 0) {
    P.level = out_level;
    P.out = out;
    const LevelGeom& lg = g.lv[out_level];
    dim3 grid((lg.w + 31) / 32, (lg.h + 7) / 8, batch);
    prof_mark("finish", s);
    k_finish<<<grid, 256, 0, s>>>(P);
  }
  return cudaGetLastError();
}

}  // namespace wb
