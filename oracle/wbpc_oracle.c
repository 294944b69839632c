/*
 * wbpc_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-file CPU restatement of the reference codec
 * (/root/reference/pkg/src/wbpc, Python/numpy + one numba kernel), used as the
 * parity checker for the B200 CUDA path and as the CPU baseline arm of bench.py.
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may load it; the
 * product package never links or imports it.
 *
 * Parity of this restatement is pinned against the reference itself: the
 * fixtures in tests/golden/ were produced by importing the unmodified reference
 * (tests/golden/make_golden.py) and tests/test_oracle_golden.py checks this file
 * byte for byte against them.
 *
 * Every function names the reference lines it restates.  Integer semantics
 * follow numpy int64: `>>` is an arithmetic (floor) shift, which gcc guarantees
 * for signed operands.
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdarg.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/wbpc_b200.h" /* status enum only (one value per errors.py class) */

typedef int64_t i64;
typedef uint64_t u64;

#define KIND_LL 0
#define KIND_HP3 1
#define MAX_CODE_BITS 32    /* entropy.py:29 */
#define MIN_CW 2            /* entropy.py:30 */
#define MAX_CW 16           /* entropy.py:31 */
#define MAX_LEVELS 30       /* transforms.py:21 */
#define MAX_DEPTH 63        /* bitplanes.py:28 */
#define DEPTH_BITS 6        /* blocks.py:39 */
#define CW_BITS 5           /* blocks.py:40 */
#define ZR_BITS 8           /* blocks.py:41 */
#define COUNT_BITS 16       /* blocks.py:42 */
#define HDR_SIZE 19         /* container.py:58  "<4sBIIBBBBH" */
#define IDX_SIZE 12         /* container.py:59  "<QI" */
#define BLOCK_DIM 128       /* container.py:54 */

static __thread char g_err[512];
static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}
const char* wbo_last_error(void) { return g_err; }
void wbo_free(void* p) { free(p); }

static int bitlen_u64(u64 v) { return v ? 64 - __builtin_clzll(v) : 0; }

/* ------------------------------------------------------------------ bit I/O */
/* BitWriter, bitio.py:15-50: MSB-first, big-endian fields, zero padded. */
typedef struct {
  uint8_t* buf;
  size_t cap; /* bytes */
  u64 nbits;
} BW;

static int bw_reserve(BW* w, u64 extra) {
  u64 need = (w->nbits + extra + 7) / 8 + 8;
  if (need <= w->cap) return 0;
  size_t nc = w->cap ? w->cap : 256;
  while (nc < need) nc *= 2;
  uint8_t* nb = (uint8_t*)realloc(w->buf, nc);
  if (!nb) return fail(WBPC_ERR_INVALID_ARG, "out of host memory");
  memset(nb + w->cap, 0, nc - w->cap);
  w->buf = nb;
  w->cap = nc;
  return 0;
}

/* BitWriter.write, bitio.py:26-35 (DomainError when the value does not fit). */
static int bw_write(BW* w, u64 value, int nbits) {
  if (nbits < 0) return fail(WBPC_ERR_DOMAIN, "negative field width");
  if (nbits < bitlen_u64(value))
    return fail(WBPC_ERR_DOMAIN, "value %llu does not fit in %d bits", (unsigned long long)value, nbits);
  if (nbits == 0) return 0;
  int rc = bw_reserve(w, (u64)nbits);
  if (rc) return rc;
  for (int i = nbits - 1; i >= 0; --i) {
    if ((value >> i) & 1) w->buf[w->nbits >> 3] |= (uint8_t)(0x80u >> (w->nbits & 7));
    w->nbits++;
  }
  return 0;
}

/* write_bit_array of a bit range copied from another MSB-first buffer (bitio.py:37-43). */
static int bw_copy_bits(BW* w, const uint8_t* src, u64 src_bit, u64 nbits) {
  int rc = bw_reserve(w, nbits);
  if (rc) return rc;
  for (u64 i = 0; i < nbits; ++i) {
    u64 sb = src_bit + i;
    if ((src[sb >> 3] >> (7 - (sb & 7))) & 1) w->buf[w->nbits >> 3] |= (uint8_t)(0x80u >> (w->nbits & 7));
    w->nbits++;
  }
  return 0;
}

static size_t bw_bytes(const BW* w) { return (size_t)((w->nbits + 7) / 8); } /* to_bytes, bitio.py:45-50 */

/* BitReader, bitio.py:53-100. */
typedef struct {
  const uint8_t* d;
  u64 nbits;
  u64 pos;
} BR;

static int br_read(BR* r, int nbits, u64* out) { /* bitio.py:80-93 */
  if (r->pos + (u64)nbits > r->nbits)
    return fail(WBPC_ERR_TRUNCATION, "need %d bits, %llu left", nbits, (unsigned long long)(r->nbits - r->pos));
  u64 v = 0;
  for (int i = 0; i < nbits; ++i) {
    u64 b = r->pos + (u64)i;
    v = (v << 1) | ((r->d[b >> 3] >> (7 - (b & 7))) & 1u);
  }
  r->pos += (u64)nbits;
  *out = v;
  return 0;
}

/* -------------------------------------------------------------- transforms */
/* rct_forward, transforms.py:79-89 */
static void rct_forward(const i64* r, const i64* g, const i64* b, i64* y, i64* cb, i64* cr, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    i64 R = r[i], G = g[i], B = b[i];
    y[i] = (R + 2 * G + B) >> 2;
    cb[i] = B - G;
    cr[i] = R - G;
  }
}

/* rct_inverse, transforms.py:92-104 */
static void rct_inverse(i64* y_r, i64* cb_g, i64* cr_b, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    i64 Y = y_r[i], Cb = cb_g[i], Cr = cr_b[i];
    i64 G = Y - ((Cb + Cr) >> 2);
    y_r[i] = Cr + G;
    cb_g[i] = G;
    cr_b[i] = Cb + G;
  }
}

/* _split_axis0 for one 1-D signal, transforms.py:107-134. */
static void split1d(const i64* x, int n, i64* low, i64* high) {
  if (n == 1) { low[0] = x[0]; return; }
  int m = n / 2;
  for (int i = 0; i < m; ++i) {
    i64 right = (2 * i + 2 < n) ? x[2 * i + 2] : x[2 * i]; /* :120-125 even-length mirror */
    high[i] = x[2 * i + 1] - ((x[2 * i] + right) >> 1);
  }
  int ne = (n + 1) / 2;
  for (int i = 0; i < ne; ++i) {
    i64 hl = high[i > 0 ? i - 1 : 0];     /* :126 h_left */
    i64 hr = high[i < m ? i : m - 1];     /* :127-132 h_right (odd mirror) */
    low[i] = x[2 * i] + ((hl + hr + 2) >> 2);
  }
}

/* _merge_axis0 for one 1-D signal, transforms.py:137-162 (lengths already validated). */
static void merge1d(const i64* low, int nl, const i64* high, int nh, i64* out) {
  if (nh == 0) { for (int i = 0; i < nl; ++i) out[i] = low[i]; return; }
  for (int i = 0; i < nl; ++i) {
    i64 hl = high[i > 0 ? i - 1 : 0];
    i64 hr = high[i < nh ? i : nh - 1];
    out[2 * i] = low[i] - ((hl + hr + 2) >> 2);
  }
  for (int i = 0; i < nh; ++i) {
    i64 xr = (i + 1 < nl) ? out[2 * i + 2] : out[2 * (nl - 1)];
    out[2 * i + 1] = high[i] + ((out[2 * i] + xr) >> 1);
  }
}

typedef struct {
  int w, h;       /* dims of the LL input at this level */
  i64 *lh, *hl, *hh;
} Detail;

typedef struct {
  int levels;
  i64* ll;
  int llw, llh;
  Detail det[MAX_LEVELS + 1]; /* det[k] = level k+1 */
} Pyramid;

/* _split_plane, transforms.py:184-191: rows first, then the columns of each half. */
static int split_plane(const i64* p, int w, int h, i64** ll, i64** lh, i64** hl, i64** hh) {
  int cw = (w + 1) / 2, fw = w / 2, ch = (h + 1) / 2, fh = h / 2;
  i64* lx = (i64*)malloc(sizeof(i64) * (size_t)h * cw + 8);
  i64* hx = (i64*)malloc(sizeof(i64) * (size_t)h * (fw ? fw : 1) + 8);
  int nmax = w > h ? w : h;
  i64* t0 = (i64*)malloc(sizeof(i64) * (size_t)nmax + 8);
  i64* t1 = (i64*)malloc(sizeof(i64) * (size_t)nmax + 8);
  i64* t2 = (i64*)malloc(sizeof(i64) * (size_t)nmax + 8);
  *ll = (i64*)malloc(sizeof(i64) * (size_t)ch * cw + 8);
  *lh = (i64*)malloc(sizeof(i64) * (size_t)fh * cw + 8);
  *hl = (i64*)malloc(sizeof(i64) * (size_t)ch * fw + 8);
  *hh = (i64*)malloc(sizeof(i64) * (size_t)fh * fw + 8);
  if (!lx || !hx || !t0 || !t1 || !t2 || !*ll || !*lh || !*hl || !*hh)
    return fail(WBPC_ERR_INVALID_ARG, "out of host memory");
  for (int y = 0; y < h; ++y) {
    split1d(p + (size_t)y * w, w, t1, t2);
    memcpy(lx + (size_t)y * cw, t1, sizeof(i64) * cw);
    if (fw) memcpy(hx + (size_t)y * fw, t2, sizeof(i64) * fw);
  }
  for (int x = 0; x < cw; ++x) {
    for (int y = 0; y < h; ++y) t0[y] = lx[(size_t)y * cw + x];
    split1d(t0, h, t1, t2);
    for (int y = 0; y < ch; ++y) (*ll)[(size_t)y * cw + x] = t1[y];
    for (int y = 0; y < fh; ++y) (*lh)[(size_t)y * cw + x] = t2[y];
  }
  for (int x = 0; x < fw; ++x) {
    for (int y = 0; y < h; ++y) t0[y] = hx[(size_t)y * fw + x];
    split1d(t0, h, t1, t2);
    for (int y = 0; y < ch; ++y) (*hl)[(size_t)y * fw + x] = t1[y];
    for (int y = 0; y < fh; ++y) (*hh)[(size_t)y * fw + x] = t2[y];
  }
  free(lx); free(hx); free(t0); free(t1); free(t2);
  return 0;
}

/* _merge_plane, transforms.py:194-199: columns of (ll,lh) and (hl,hh), then rows. */
static int merge_plane(const i64* ll, const i64* lh, const i64* hl, const i64* hh, int w, int h, i64* out) {
  int cw = (w + 1) / 2, fw = w / 2, ch = (h + 1) / 2, fh = h / 2;
  i64* lx = (i64*)malloc(sizeof(i64) * (size_t)h * cw + 8);
  i64* hx = (i64*)malloc(sizeof(i64) * (size_t)h * (fw ? fw : 1) + 8);
  int nmax = w > h ? w : h;
  i64* t0 = (i64*)calloc((size_t)nmax + 1, sizeof(i64));
  i64* t1 = (i64*)calloc((size_t)nmax + 1, sizeof(i64));
  i64* t2 = (i64*)calloc((size_t)nmax + 1, sizeof(i64));
  if (!lx || !hx || !t0 || !t1 || !t2) return fail(WBPC_ERR_INVALID_ARG, "out of host memory");
  for (int x = 0; x < cw; ++x) {
    for (int y = 0; y < ch; ++y) t0[y] = ll[(size_t)y * cw + x];
    for (int y = 0; y < fh; ++y) t1[y] = lh[(size_t)y * cw + x];
    merge1d(t0, ch, t1, fh, t2);
    for (int y = 0; y < h; ++y) lx[(size_t)y * cw + x] = t2[y];
  }
  for (int x = 0; x < fw; ++x) {
    for (int y = 0; y < ch; ++y) t0[y] = hl[(size_t)y * fw + x];
    for (int y = 0; y < fh; ++y) t1[y] = hh[(size_t)y * fw + x];
    merge1d(t0, ch, t1, fh, t2);
    for (int y = 0; y < h; ++y) hx[(size_t)y * fw + x] = t2[y];
  }
  for (int y = 0; y < h; ++y) merge1d(lx + (size_t)y * cw, cw, hx + (size_t)y * fw, fw, out + (size_t)y * w);
  free(lx); free(hx); free(t0); free(t1); free(t2);
  return 0;
}

static void pyramid_free(Pyramid* p) {
  free(p->ll);
  for (int k = 0; k < p->levels; ++k) { free(p->det[k].lh); free(p->det[k].hl); free(p->det[k].hh); }
  memset(p, 0, sizeof *p);
}

/* dwt2d_forward, transforms.py:202-216 */
static int dwt2d_forward(const i64* plane, int w, int h, int levels, Pyramid* out) {
  memset(out, 0, sizeof *out);
  if (levels < 0 || levels > MAX_LEVELS) return fail(WBPC_ERR_LEVEL_RANGE, "levels must be in [0, %d]", MAX_LEVELS);
  out->levels = levels;
  i64* ll = (i64*)malloc(sizeof(i64) * (size_t)w * h + 8);
  if (!ll) return fail(WBPC_ERR_INVALID_ARG, "out of host memory");
  memcpy(ll, plane, sizeof(i64) * (size_t)w * h);
  int cw = w, ch = h;
  for (int k = 0; k < levels; ++k) {
    i64 *nll, *lh, *hl, *hh;
    int rc = split_plane(ll, cw, ch, &nll, &lh, &hl, &hh);
    if (rc) return rc;
    free(ll);
    out->det[k].w = cw; out->det[k].h = ch;
    out->det[k].lh = lh; out->det[k].hl = hl; out->det[k].hh = hh;
    ll = nll;
    cw = (cw + 1) / 2; ch = (ch + 1) / 2;
  }
  out->ll = ll; out->llw = cw; out->llh = ch;
  return 0;
}

/* level_dims, transforms.py:227-232 */
static void level_dims(u64 w, u64 h, int level, u64* lw, u64* lh) {
  if (level >= 63) { *lw = w ? 1 : 0; *lh = h ? 1 : 0; return; }
  *lw = (w + (1ull << level) - 1) >> level;
  *lh = (h + (1ull << level) - 1) >> level;
}

/* default_levels, transforms.py:235-245 */
int wbo_default_levels(int w, int h) {
  if ((w > h ? w : h) > 512) return 5;
  int levels = 0;
  while (levels < MAX_LEVELS) {
    u64 lw, lh;
    level_dims((u64)w, (u64)h, levels + 1, &lw, &lh);
    if (lw < 16 || lh < 16) break;
    levels++;
  }
  return levels;
}

/* --------------------------------------------------------------- bit planes */
/* _area_order, bitplanes.py:148-170 (generic dims, including the height%4==2 tail). */
static void area_order(int w, int h, int* order) {
  int acols = w / 4, arows = h / 2, n = arows * acols;
  int per_band = 2 * acols, full = (arows / 2) * per_band;
  for (int k = 0; k < full; ++k) {
    int band = k / per_band, r = 2 * band + (k % 2), c = (k / 2) % acols;
    order[k] = r * acols + c;
  }
  for (int k = full; k < n; ++k) order[k] = (arows - 1) * acols + (k - full);
}

/* serialize_block, bitplanes.py:249-265 with _smr_planes :112-122 and _plane_symbols :224-229. */
static void serialize_block(const i64* const* grids, int nsub, int dim, int depth, const int* order, uint8_t* sym) {
  int acols = dim / 4, pp = dim * dim / 8;
  for (int b = 0; b < depth; ++b) {
    for (int s = 0; s < nsub; ++s) {
      const i64* g = grids[s];
      uint8_t* out = sym + (size_t)(b * nsub + s) * pp;
      for (int k = 0; k < pp; ++k) {
        int a = order[k], r = a / acols, c = a % acols;
        unsigned v = 0;
        for (int i = 0; i < 2; ++i)
          for (int j = 0; j < 4; ++j) {
            i64 x = g[(size_t)(2 * r + i) * dim + 4 * c + j];
            unsigned bit;
            if (b == 0) bit = x < 0;
            else { i64 m = x < 0 ? -x : x; bit = (unsigned)((m >> (depth - 1 - b)) & 1); }
            v |= bit << (4 * i + j); /* AREA_WEIGHTS, bitplanes.py:31 */
          }
        out[k] = (uint8_t)v;
      }
    }
  }
}

/* ----------------------------------------------------------------- entropy */
typedef struct {
  int n_nodes;
  int left[512], right[512], sym[512]; /* preorder flat arrays as build_huffman/read_tree */
  uint32_t code_val[256];
  int code_len[256]; /* -1 = symbol absent */
} Huff;

/* HuffmanCode._assign_codes, entropy.py:88-100 */
static int assign_codes(Huff* hc) {
  for (int i = 0; i < 256; ++i) { hc->code_len[i] = -1; hc->code_val[i] = 0; }
  int st_node[1100], st_len[1100];
  u64 st_code[1100];
  int sp = 0;
  st_node[sp] = 0; st_code[sp] = 0; st_len[sp] = 0; sp++;
  while (sp) {
    --sp;
    int node = st_node[sp], len = st_len[sp];
    u64 code = st_code[sp];
    if (hc->left[node] == -1) {
      int s = hc->sym[node];
      hc->code_val[s] = (uint32_t)code;
      hc->code_len[s] = len;
      continue;
    }
    if (len >= MAX_CODE_BITS) return fail(WBPC_ERR_CODE_LENGTH, "codeword longer than %d bits", MAX_CODE_BITS);
    st_node[sp] = hc->left[node]; st_code[sp] = code << 1; st_len[sp] = len + 1; sp++;
    st_node[sp] = hc->right[node]; st_code[sp] = (code << 1) | 1; st_len[sp] = len + 1; sp++;
  }
  return 0;
}

/* build_huffman, entropy.py:194-248: heapq on (frequency, min symbol); the first popped
 * tree becomes the left child.  Restated with an explicit binary min-heap; keys are
 * unique (distinct min symbols), so the pop sequence equals heapq's. */
typedef struct { i64 f; int m; int t; } HEnt;
static int hless(const HEnt* a, const HEnt* b) { return a->f < b->f || (a->f == b->f && a->m < b->m); }
static void hpush(HEnt* h, int* n, HEnt e) {
  int i = (*n)++;
  h[i] = e;
  while (i > 0) {
    int p = (i - 1) / 2;
    if (!hless(&h[i], &h[p])) break;
    HEnt t = h[i]; h[i] = h[p]; h[p] = t; i = p;
  }
}
static HEnt hpop(HEnt* h, int* n) {
  HEnt top = h[0];
  h[0] = h[--(*n)];
  int i = 0;
  for (;;) {
    int l = 2 * i + 1, r = l + 1, s = i;
    if (l < *n && hless(&h[l], &h[s])) s = l;
    if (r < *n && hless(&h[r], &h[s])) s = r;
    if (s == i) break;
    HEnt t = h[i]; h[i] = h[s]; h[s] = t; i = s;
  }
  return top;
}

int wbo_build_huffman(const i64* freq, Huff* hc) {
  /* tree nodes before flattening: t < 256 leaf symbol t, t >= 256 internal */
  int tl[512], tr[512];
  HEnt heap[300];
  int n = 0, nt = 256;
  for (int s = 0; s < 256; ++s)
    if (freq[s] > 0) { HEnt e = {freq[s], s, s}; hpush(heap, &n, e); }
  if (n == 0) return fail(WBPC_ERR_EMPTY_ALPHABET, "no symbol has a nonzero frequency");
  while (n > 1) {
    HEnt a = hpop(heap, &n), b = hpop(heap, &n);
    tl[nt] = a.t; tr[nt] = b.t;
    HEnt e = {a.f + b.f, a.m < b.m ? a.m : b.m, nt};
    nt++;
    hpush(heap, &n, e);
  }
  /* preorder flattening (entropy.py:225-247) */
  int stack[600], sp = 0, parent_slot[600];
  hc->n_nodes = 0;
  stack[sp] = heap[0].t; parent_slot[sp] = -1; sp++;
  while (sp) {
    --sp;
    int t = stack[sp], ps = parent_slot[sp];
    int idx = hc->n_nodes++;
    if (ps >= 0) { if (ps & 1) hc->right[ps >> 1] = idx; else hc->left[ps >> 1] = idx; }
    if (t < 256) { hc->left[idx] = hc->right[idx] = -1; hc->sym[idx] = t; }
    else {
      hc->left[idx] = hc->right[idx] = -1; hc->sym[idx] = -1;
      stack[sp] = tr[t]; parent_slot[sp] = idx * 2 + 1; sp++;
      stack[sp] = tl[t]; parent_slot[sp] = idx * 2; sp++;
    }
  }
  return assign_codes(hc);
}

/* write_tree, entropy.py:259-269 */
static int write_tree(const Huff* hc, BW* w) {
  int stack[600], sp = 0, rc;
  stack[sp++] = 0;
  while (sp) {
    int node = stack[--sp];
    if (hc->left[node] == -1) {
      if ((rc = bw_write(w, 1, 1)) || (rc = bw_write(w, (u64)hc->sym[node], 8))) return rc;
    } else {
      if ((rc = bw_write(w, 0, 1))) return rc;
      stack[sp++] = hc->right[node];
      stack[sp++] = hc->left[node];
    }
  }
  return 0;
}

/* read_tree, entropy.py:272-310 */
static int read_tree(BR* r, Huff* hc) {
  int pending[600], np = 0, first = 1, seen[256] = {0};
  hc->n_nodes = 0;
  while (first || np) {
    first = 0;
    u64 bit = 0, s = 0;
    if (br_read(r, 1, &bit)) return fail(WBPC_ERR_MALFORMED_TREE, "truncated tree encoding");
    int idx = hc->n_nodes;
    if (idx > 511) return fail(WBPC_ERR_MALFORMED_TREE, "tree larger than a byte alphabet allows");
    if (bit) {
      if (br_read(r, 8, &s)) return fail(WBPC_ERR_MALFORMED_TREE, "truncated tree encoding");
      if (seen[s]) return fail(WBPC_ERR_MALFORMED_TREE, "duplicate leaf symbol %d", (int)s);
      seen[s] = 1;
      hc->left[idx] = hc->right[idx] = -1; hc->sym[idx] = (int)s;
    } else {
      hc->left[idx] = hc->right[idx] = -2; hc->sym[idx] = -1;
    }
    hc->n_nodes++;
    if (idx > 0) {
      int parent = pending[np - 1];
      if (hc->left[parent] == -2) hc->left[parent] = idx;
      else { hc->right[parent] = idx; np--; }
    }
    if (!bit) pending[np++] = idx;
  }
  return assign_codes(hc); /* HuffmanCode(...) constructor, entropy.py:86 */
}

/* optimize_counter_width, entropy.py:171-191 */
int wbo_optimize_counter_width(const i64* runs, i64 n, int zr_code_bits, int max_width) {
  if (max_width < MIN_CW) return -fail(WBPC_ERR_DOMAIN, "max width must be >= %d", MIN_CW);
  if (n == 0) return MIN_CW;
  int best = MIN_CW;
  i64 best_cost = -1;
  for (int w = MIN_CW; w <= max_width; ++w) {
    i64 cap = ((i64)1 << w) - 1, cost = 0;
    for (i64 i = 0; i < n; ++i) cost += ((runs[i] + cap - 1) / cap) * (w + zr_code_bits);
    if (best_cost < 0 || cost < best_cost) { best_cost = cost; best = w; }
  }
  return best;
}

/* decode_tokens, _kernels.py:33-89 (argument for argument). Returns status, *end = bitpos. */
int wbo_decode_tokens(const uint8_t* payload, i64 start_bit, i64 end_bit, const int32_t* left,
                      const int32_t* right, const int32_t* leaf, int zr, int cw, const i64* seg_lengths,
                      int nseg, uint8_t* out, i64* seg_starts, i64* end) {
  i64 bitpos = start_bit, oi = 0;
  for (int s = 0; s < nseg; ++s) {
    seg_starts[s] = bitpos - start_bit;
    i64 remaining = seg_lengths[s];
    while (remaining > 0) {
      int node = 0;
      while (left[node] != -1) {
        if (bitpos >= end_bit) { *end = bitpos; return 1; }
        int bit = (payload[bitpos >> 3] >> (7 - (bitpos & 7))) & 1;
        bitpos++;
        node = bit ? right[node] : left[node];
      }
      int value = leaf[node];
      if (value == zr) {
        if (bitpos + cw > end_bit) { *end = bitpos; return 1; }
        i64 counter = 0;
        for (int i = 0; i < cw; ++i) {
          counter = (counter << 1) | ((payload[bitpos >> 3] >> (7 - (bitpos & 7))) & 1);
          bitpos++;
        }
        if (counter == 0) { out[oi++] = (uint8_t)value; remaining--; }
        else {
          if (counter > remaining) { *end = bitpos; return 2; }
          for (i64 i = 0; i < counter; ++i) out[oi++] = 0;
          remaining -= counter;
        }
      } else { out[oi++] = (uint8_t)value; remaining--; }
    }
  }
  *end = bitpos;
  return 0;
}

/* ------------------------------------------------------------------ blocks */
/* seek_entry_bits, blocks.py:45-50 */
static int seek_entry_bits(int w, int h, int depth, int kind) {
  int nsub = kind == KIND_LL ? 1 : 3;
  u64 total = (u64)depth * nsub * (u64)w * h / 8;
  return (bitlen_u64(total) - 1) + 5;
}

/* Zero runs >= 2 inside one segment (entropy._segment_runs, entropy.py:131-153). */
static i64 segment_runs(const uint8_t* sym, int nseg, int pp, i64* starts, i64* lens) {
  i64 nr = 0;
  for (int s = 0; s < nseg; ++s) {
    const uint8_t* seg = sym + (size_t)s * pp;
    int i = 0;
    while (i < pp) {
      if (seg[i] != 0) { i++; continue; }
      int j = i;
      while (j < pp && seg[j] == 0) j++;
      if (j - i >= 2) { starts[nr] = (i64)s * pp + i; lens[nr] = j - i; nr++; }
      i = j;
    }
  }
  return nr;
}

/* encode_block, blocks.py:84-120, with _plan_stream :53-81, tokenize entropy.py:324-378,
 * pack_tokens :385-421.  grids: nsub dim x dim int64 tiles; depth < 0 = minimal. */
int wbo_encode_block(int kind, const i64* const* grids, int dim, int depth, uint8_t** out, size_t* out_len) {
  int nsub = kind == KIND_LL ? 1 : 3;
  if (dim % 4 || dim % 2 || dim < 4) return fail(WBPC_ERR_SHAPE, "block dims must be positive multiples of (4, 2)");
  i64 peak = 0;
  for (int s = 0; s < nsub; ++s)
    for (size_t i = 0; i < (size_t)dim * dim; ++i) {
      i64 v = grids[s][i]; v = v < 0 ? -v : v;
      if (v > peak) peak = v;
    }
  if (depth < 0) depth = 1 + bitlen_u64((u64)peak); /* CoefficientBlock.build, bitplanes.py:77-79 */
  if (depth < 1 || depth > MAX_DEPTH) return fail(WBPC_ERR_DOMAIN, "depth must be 1..%d", MAX_DEPTH);
  if (depth - 1 < 63 && (u64)peak >= (1ull << (depth - 1)))
    return fail(WBPC_ERR_DEPTH_OVERFLOW, "coefficient magnitude %lld needs more than %d bits", (long long)peak, depth - 1);
  int pp = dim * dim / 8, nslots = nsub * depth;
  int* order = (int*)malloc(sizeof(int) * pp);
  uint8_t* sym = (uint8_t*)malloc((size_t)nslots * pp);
  uint8_t* kept = (uint8_t*)malloc((size_t)nslots * pp);
  i64* rstart = (i64*)malloc(sizeof(i64) * ((size_t)nslots * pp / 2 + 2));
  i64* rlen = (i64*)malloc(sizeof(i64) * ((size_t)nslots * pp / 2 + 2));
  i64* seek = (i64*)malloc(sizeof(i64) * (nslots + 1));
  int* stored = (int*)malloc(sizeof(int) * nslots);
  BW payload = {0}, w = {0};
  int rc = 0;
  if (!order || !sym || !kept || !rstart || !rlen || !seek || !stored) { rc = fail(WBPC_ERR_INVALID_ARG, "oom"); goto done; }
  area_order(dim, dim, order);
  serialize_block(grids, nsub, dim, depth, order, sym);
  int nstored = 0;
  for (int k = 0; k < nslots; ++k) { /* blocks.py:89-90 */
    stored[k] = 0;
    for (int i = 0; i < pp; ++i) if (sym[(size_t)k * pp + i]) { stored[k] = 1; break; }
    if (stored[k]) memcpy(kept + (size_t)nstored++ * pp, sym + (size_t)k * pp, pp);
  }
  int zr = 0, width = MIN_CW;
  Huff code;
  if (nstored) {
    size_t nk = (size_t)nstored * pp;
    i64 hist[256] = {0};
    for (size_t i = 0; i < nk; ++i) hist[kept[i]]++;
    zr = 0; /* select_zr_symbol, entropy.py:156-159: argmin, ties -> smallest */
    for (int s = 1; s < 256; ++s) if (hist[s] < hist[zr]) zr = s;
    i64 nr = segment_runs(kept, nstored, pp, rstart, rlen);
    if (nr > 0) { /* blocks.py:67-76 */
      i64 prov[256], zin = 0;
      memcpy(prov, hist, sizeof prov);
      for (i64 i = 0; i < nr; ++i) zin += rlen[i];
      prov[0] -= zin;
      prov[zr] += nr;
      if ((rc = wbo_build_huffman(prov, &code))) goto done;
      width = wbo_optimize_counter_width(rlen, nr, code.code_len[zr], MAX_CW);
    }
    i64 cap = ((i64)1 << width) - 1;
    /* token frequencies (entropy.py:381-382) of the tokenize() stream */
    i64 tf[256] = {0};
    {
      i64 ri = 0;
      for (int sg = 0; sg < nstored; ++sg) {
        for (int i = 0; i < pp;) {
          i64 pos = (i64)sg * pp + i;
          if (ri < nr && rstart[ri] == pos) { tf[zr] += (rlen[ri] + cap - 1) / cap; i += (int)rlen[ri]; ri++; }
          else { tf[kept[pos]]++; i++; }
        }
      }
    }
    if ((rc = wbo_build_huffman(tf, &code))) goto done; /* blocks.py:80 */
    /* pack_tokens: codeword then optional counter; per-segment first-token offsets */
    i64 ri = 0;
    for (int sg = 0; sg < nstored; ++sg) {
      seek[sg] = (i64)payload.nbits;
      for (int i = 0; i < pp;) {
        i64 pos = (i64)sg * pp + i;
        if (ri < nr && rstart[ri] == pos) {
          i64 L = rlen[ri], chunks = (L + cap - 1) / cap;
          for (i64 c = 0; c < chunks; ++c) {
            i64 v = (c == chunks - 1) ? L - cap * (chunks - 1) : cap; /* entropy.py:349-358 */
            if ((rc = bw_write(&payload, code.code_val[zr], code.code_len[zr])) || (rc = bw_write(&payload, (u64)v, width))) goto done;
          }
          i += (int)L; ri++;
        } else {
          int s = kept[pos];
          if ((rc = bw_write(&payload, code.code_val[s], code.code_len[s]))) goto done;
          if (s == zr && (rc = bw_write(&payload, 0, width))) goto done; /* literal escape, entropy.py:346 */
          i++;
        }
      }
    }
  }
  /* block writer, blocks.py:104-120 */
  if ((rc = bw_write(&w, (u64)depth, DEPTH_BITS)) || (rc = bw_write(&w, (u64)width, CW_BITS)) || (rc = bw_write(&w, (u64)zr, ZR_BITS))) goto done;
  for (int s = 0; s < nsub; ++s)
    for (int b = 0; b < depth; ++b)
      if ((rc = bw_write(&w, (u64)stored[b * nsub + s], 1))) goto done;
  if (nstored && (rc = write_tree(&code, &w))) goto done;
  if ((rc = bw_write(&w, (u64)nstored, COUNT_BITS))) goto done;
  {
    int t = seek_entry_bits(dim, dim, depth, kind);
    for (int sg = 0; sg < nstored; ++sg)
      if ((rc = bw_write(&w, (u64)seek[sg], t))) goto done;
  }
  if (payload.nbits && (rc = bw_copy_bits(&w, payload.buf, 0, payload.nbits))) goto done;
  if ((rc = bw_reserve(&w, 8))) goto done;
  *out_len = bw_bytes(&w);
  *out = w.buf;
  w.buf = NULL;
done:
  free(order); free(sym); free(kept); free(rstart); free(rlen); free(seek); free(stored);
  free(payload.buf); free(w.buf);
  return rc;
}

typedef struct {
  int depth, cw, zr, nsub, n_stored;
  uint8_t masks[3][64];
  int has_code;
  Huff code;
  i64 seek[3 * 64];
  u64 payload_start;
} BlockHeader;

/* parse_header, blocks.py:150-192 */
static int parse_header(const uint8_t* data, size_t len, int w, int h, int kind, BlockHeader* hd) {
  BR r = {data, (u64)len * 8, 0};
  u64 v = 0;
  int nsub = kind == KIND_LL ? 1 : 3;
  hd->nsub = nsub;
  if (br_read(&r, DEPTH_BITS, &v)) goto trunc;
  hd->depth = (int)v;
  if (hd->depth < 1) return fail(WBPC_ERR_BLOCK_PARSE, "plane depth must be >= 1");
  if (br_read(&r, CW_BITS, &v)) goto trunc;
  hd->cw = (int)v;
  if (br_read(&r, ZR_BITS, &v)) goto trunc;
  hd->zr = (int)v;
  int cnt = 0;
  for (int s = 0; s < nsub; ++s)
    for (int b = 0; b < hd->depth; ++b) {
      if (br_read(&r, 1, &v)) goto trunc;
      hd->masks[s][b] = (uint8_t)v;
      cnt += (int)v;
    }
  hd->n_stored = cnt;
  hd->has_code = 0;
  if (cnt) {
    int rc = read_tree(&r, &hd->code);
    if (rc) return rc;
    hd->has_code = 1;
  }
  if (br_read(&r, COUNT_BITS, &v)) goto trunc;
  if ((int)v != cnt) return fail(WBPC_ERR_CORRUPTION, "seek count %d != stored planes %d", (int)v, cnt);
  int t = seek_entry_bits(w, h, hd->depth, kind);
  for (int i = 0; i < cnt; ++i) {
    if (br_read(&r, t, &v)) goto trunc;
    hd->seek[i] = (i64)v;
  }
  for (int i = 1; i < cnt; ++i)
    if (hd->seek[i] < hd->seek[i - 1]) return fail(WBPC_ERR_CORRUPTION, "seek entries must be non-decreasing");
  hd->payload_start = r.pos;
  return 0;
trunc:
  return fail(WBPC_ERR_BLOCK_PARSE, "block header truncated");
}

/* decode_block, blocks.py:195-250 + deserialize_block, bitplanes.py:268-291.
 * keep < 0 means planes_to_keep=None.  grids: nsub outputs of dim*dim int64. */
int wbo_decode_block(const uint8_t* data, size_t len, int dim, int kind, int keep, i64* const* grids) {
  BlockHeader hd;
  int rc = parse_header(data, len, dim, dim, kind, &hd);
  if (rc) return rc;
  if (dim % 4 || dim % 2 || dim < 4) return fail(WBPC_ERR_SHAPE, "area grid needs dims that are multiples of (4, 2)");
  int depth = hd.depth, nsub = hd.nsub, pp = dim * dim / 8;
  int q = keep < 0 ? depth : (keep > depth ? depth : keep);
  /* stored slots in serialization order (BlockHeader.stored_slots, blocks.py:138-147) */
  int slot_of[3 * 64], ns = 0, decode_n = 0;
  for (int b = 0; b < depth; ++b)
    for (int s = 0; s < nsub; ++s)
      if (hd.masks[s][b]) { slot_of[ns++] = b * nsub + s; if (b < q) decode_n++; }
  uint8_t* symbols = (uint8_t*)calloc((size_t)depth * nsub * pp, 1);
  int* order = (int*)malloc(sizeof(int) * pp);
  if (!symbols || !order) { free(symbols); free(order); return fail(WBPC_ERR_INVALID_ARG, "oom"); }
  if (decode_n) {
    uint8_t* out = (uint8_t*)malloc((size_t)decode_n * pp);
    i64* seg_len = (i64*)malloc(sizeof(i64) * decode_n);
    i64* seg_start = (i64*)malloc(sizeof(i64) * decode_n);
    for (int i = 0; i < decode_n; ++i) seg_len[i] = pp;
    i64 end;
    int st = wbo_decode_tokens(data, (i64)hd.payload_start, (i64)len * 8, hd.code.left, hd.code.right, hd.code.sym,
                               hd.zr, hd.cw, seg_len, decode_n, out, seg_start, &end);
    if (st == 1) rc = fail(WBPC_ERR_TRUNCATION, "block payload truncated");
    else if (st == 2) rc = fail(WBPC_ERR_CORRUPTION, "zero-run counter overflows its plane");
    else {
      for (int i = 0; i < decode_n; ++i)
        if (seg_start[i] != hd.seek[i]) { rc = fail(WBPC_ERR_CORRUPTION, "seek entries disagree with decoded plane starts"); break; }
    }
    if (!rc)
      for (int i = 0; i < decode_n; ++i) memcpy(symbols + (size_t)slot_of[i] * pp, out + (size_t)i * pp, pp);
    free(out); free(seg_len); free(seg_start);
  }
  if (!rc) {
    area_order(dim, dim, order);
    int acols = dim / 4;
    for (int s = 0; s < nsub; ++s) {
      i64* g = grids[s];
      memset(g, 0, sizeof(i64) * (size_t)dim * dim);
      uint8_t* neg = (uint8_t*)calloc((size_t)dim * dim, 1);
      for (int b = 0; b < depth; ++b) {
        const uint8_t* seg = symbols + (size_t)(b * nsub + s) * pp;
        for (int k = 0; k < pp; ++k) {
          int sv = seg[k];
          if (!sv) continue;
          int a = order[k], r = a / acols, c = a % acols;
          for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 4; ++j)
              if ((sv >> (4 * i + j)) & 1) {
                size_t pos = (size_t)(2 * r + i) * dim + 4 * c + j;
                if (b == 0) neg[pos] = 1;
                else g[pos] |= (i64)1 << (depth - 1 - b); /* _planes_to_values, bitplanes.py:125-130 */
              }
        }
      }
      for (size_t i = 0; i < (size_t)dim * dim; ++i) if (neg[i]) g[i] = -g[i];
      free(neg);
    }
  }
  free(symbols); free(order);
  return rc;
}

/* truncate_block, blocks.py:264-304.  On return *out may alias data (unchanged block). */
int wbo_truncate_block(const uint8_t* data, size_t len, int dim, int kind, int n, uint8_t** out, size_t* out_len) {
  if (n < 0) return fail(WBPC_ERR_DOMAIN, "planes_dropped must be >= 0");
  *out = NULL;
  *out_len = len;
  if (n == 0) return 0;
  BlockHeader hd;
  int rc = parse_header(data, len, dim, dim, kind, &hd);
  if (rc) return rc;
  int q = hd.depth - n; if (q < 0) q = 0;
  int keep_n = 0, ns = 0;
  for (int b = 0; b < hd.depth; ++b)
    for (int s = 0; s < hd.nsub; ++s)
      if (hd.masks[s][b]) { ns++; if (b < q) keep_n++; }
  if (keep_n == ns) return 0;
  i64 cut = hd.seek[keep_n];
  if (hd.payload_start + (u64)cut > (u64)len * 8)
    return fail(WBPC_ERR_TRUNCATION, "need %lld bits", (long long)cut); /* read_bit_array, bitio.py:95-97 */
  BW w = {0};
  if ((rc = bw_write(&w, (u64)hd.depth, DEPTH_BITS)) || (rc = bw_write(&w, (u64)hd.cw, CW_BITS)) || (rc = bw_write(&w, (u64)hd.zr, ZR_BITS))) goto bad;
  for (int s = 0; s < hd.nsub; ++s)
    for (int b = 0; b < hd.depth; ++b)
      if ((rc = bw_write(&w, b < q ? hd.masks[s][b] : 0, 1))) goto bad;
  if (keep_n && hd.has_code && (rc = write_tree(&hd.code, &w))) goto bad;
  if ((rc = bw_write(&w, (u64)keep_n, COUNT_BITS))) goto bad;
  {
    int t = seek_entry_bits(dim, dim, hd.depth, kind);
    for (int i = 0; i < keep_n; ++i) if ((rc = bw_write(&w, (u64)hd.seek[i], t))) goto bad;
  }
  if (cut && (rc = bw_copy_bits(&w, data, hd.payload_start, (u64)cut))) goto bad;
  if ((rc = bw_reserve(&w, 8))) goto bad;
  *out_len = bw_bytes(&w);
  *out = w.buf;
  return 0;
bad:
  free(w.buf);
  return rc;
}

/* --------------------------------------------------------------- container */
typedef struct {
  u64 w, h;
  int c, bd, color, levels, dim;
} CHeader;

typedef struct { int kind, c, lev, r, col; } Slot;

/* iter_slots, container.py:115-129: per channel the LL grid at level L, then the
 * high-pass grids for levels L..1, each row major. */
static u64 slots_fill(const CHeader* hd, Slot* out) {
  u64 n = 0;
  int L = hd->levels;
  for (int c = 0; c < hd->c; ++c) {
    for (int pass = 0; pass <= L; ++pass) {
      int kind = pass == 0 ? KIND_LL : KIND_HP3;
      int l = pass == 0 ? L : L - pass + 1;
      u64 lw, lh;
      level_dims(hd->w, hd->h, l, &lw, &lh);
      u64 gw = (lw + hd->dim - 1) / hd->dim, gh = (lh + hd->dim - 1) / hd->dim;
      for (u64 r = 0; r < gh; ++r)
        for (u64 col = 0; col < gw; ++col) {
          if (out) { Slot s = {kind, c, l, (int)r, (int)col}; out[n] = s; }
          n++;
        }
    }
  }
  return n;
}

static void put_u16(uint8_t* p, unsigned v) { p[0] = v & 255; p[1] = (v >> 8) & 255; }
static void put_u32(uint8_t* p, u64 v) { for (int i = 0; i < 4; ++i) p[i] = (v >> (8 * i)) & 255; }
static void put_u64(uint8_t* p, u64 v) { for (int i = 0; i < 8; ++i) p[i] = (v >> (8 * i)) & 255; }
static u64 get_le(const uint8_t* p, int n) { u64 v = 0; for (int i = n - 1; i >= 0; --i) v = (v << 8) | p[i]; return v; }

/* ContainerHeader.pack, container.py:76-87 */
static void header_pack(const CHeader* h, uint8_t* p) {
  memcpy(p, "WBPC", 4);
  p[4] = 1;
  put_u32(p + 5, h->w);
  put_u32(p + 9, h->h);
  p[13] = (uint8_t)h->c; p[14] = (uint8_t)h->bd; p[15] = (uint8_t)h->color; p[16] = (uint8_t)h->levels;
  put_u16(p + 17, (unsigned)h->dim);
}

/* ContainerHeader.parse, container.py:89-108 */
static int header_parse(const uint8_t* d, size_t len, CHeader* h) {
  if (len < HDR_SIZE) return fail(WBPC_ERR_CONTAINER_PARSE, "container shorter than its header");
  if (memcmp(d, "WBPC", 4)) return fail(WBPC_ERR_CONTAINER_PARSE, "bad magic");
  if (d[4] != 1) return fail(WBPC_ERR_CONTAINER_PARSE, "unsupported version %d", d[4]);
  h->w = get_le(d + 5, 4); h->h = get_le(d + 9, 4);
  h->c = d[13]; h->bd = d[14]; h->color = d[15]; h->levels = d[16];
  h->dim = (int)get_le(d + 17, 2);
  if (h->w < 1 || h->h < 1 || h->c < 1 || h->c > 4 || h->dim < 8) return fail(WBPC_ERR_CONTAINER_PARSE, "invalid header geometry");
  return 0;
}

typedef struct {
  const CHeader* hd;
  const Slot* slots;
  u64 nslots;
  Pyramid* pyr; /* per channel */
  uint8_t** blobs;
  size_t* lens;
  atomic_ullong next;
  atomic_int err;
  atomic_ullong err_slot;
  char msg[512];
  pthread_mutex_t mu;
} EncJob;

static void record_err(atomic_int* err, atomic_ullong* err_slot, pthread_mutex_t* mu, char* msg, u64 slot, int rc) {
  pthread_mutex_lock(mu);
  if (atomic_load(err) == 0 || slot < atomic_load(err_slot)) {
    atomic_store(err, rc);
    atomic_store(err_slot, slot);
    snprintf(msg, 512, "%s", g_err);
  }
  pthread_mutex_unlock(mu);
}

/* _pad_tile + _encode_slot, container.py:140-164 */
static int encode_slot(const CHeader* hd, const Pyramid* pyr, const Slot* s, uint8_t** blob, size_t* len) {
  int dim = hd->dim;
  size_t tn = (size_t)dim * dim;
  i64* tiles = (i64*)calloc(3 * tn, sizeof(i64));
  const i64* g[3];
  int gw[3], gh[3], nsub;
  if (s->kind == KIND_LL) {
    nsub = 1; g[0] = pyr->ll; gw[0] = pyr->llw; gh[0] = pyr->llh;
  } else {
    const Detail* d = &pyr->det[s->lev - 1];
    int cw = (d->w + 1) / 2, fw = d->w / 2, ch = (d->h + 1) / 2, fh = d->h / 2;
    nsub = 3;
    g[0] = d->lh; gw[0] = cw; gh[0] = fh;
    g[1] = d->hl; gw[1] = fw; gh[1] = ch;
    g[2] = d->hh; gw[2] = fw; gh[2] = fh;
  }
  const i64* tp[3];
  for (int k = 0; k < nsub; ++k) {
    i64* t = tiles + k * tn;
    int y0 = s->r * dim, x0 = s->col * dim;
    for (int y = 0; y < dim && y0 + y < gh[k]; ++y)
      for (int x = 0; x < dim && x0 + x < gw[k]; ++x) t[(size_t)y * dim + x] = g[k][(size_t)(y0 + y) * gw[k] + x0 + x];
    tp[k] = t;
  }
  int rc = wbo_encode_block(s->kind, tp, dim, -1, blob, len);
  free(tiles);
  return rc;
}

static void* enc_worker(void* arg) {
  EncJob* j = (EncJob*)arg;
  for (;;) {
    u64 i = atomic_fetch_add(&j->next, 1);
    if (i >= j->nslots) break;
    const Slot* s = &j->slots[i];
    int rc = encode_slot(j->hd, &j->pyr[s->c], s, &j->blobs[i], &j->lens[i]);
    if (rc) record_err(&j->err, &j->err_slot, &j->mu, j->msg, i, rc);
  }
  return NULL;
}

static int run_pool(void* (*fn)(void*), void* job, int nthreads) {
  if (nthreads <= 1) { fn(job); return 0; }
  pthread_t th[256];
  if (nthreads > 256) nthreads = 256;
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, fn, job);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  return 0;
}

/* encode_image, container.py:167-206.  samples: C*H*W int64 (channel planar).
 * levels < 0 means None (default_levels). */
int wbo_encode_image(const i64* samples, int w, int h, int c, int bd, int levels, int use_rct, int nthreads,
                     uint8_t** out, size_t* out_len) {
  if (c < 1 || c > 4) return fail(WBPC_ERR_UNSUPPORTED_LAYOUT, "channels must be 1..4, got %d", c);
  if (bd < 1 || bd > 16) return fail(WBPC_ERR_DOMAIN, "bit depth must be 1..16, got %d", bd);
  if (w < 1 || h < 1) return fail(WBPC_ERR_DOMAIN, "image dimensions must be >= 1");
  size_t n = (size_t)w * h;
  for (size_t i = 0; i < n * c; ++i) /* validate_source, transforms.py:57-62 */
    if (samples[i] < 0 || samples[i] >= ((i64)1 << bd)) return fail(WBPC_ERR_DOMAIN, "samples out of range for bit depth %d", bd);
  if (levels < 0) levels = wbo_default_levels(w, h);
  if (use_rct && c != 3) return fail(WBPC_ERR_UNSUPPORTED_LAYOUT, "color transform needs exactly 3 channels");
  i64* planes = (i64*)malloc(sizeof(i64) * n * c);
  if (!planes) return fail(WBPC_ERR_INVALID_ARG, "oom");
  if (use_rct) rct_forward(samples, samples + n, samples + 2 * n, planes, planes + n, planes + 2 * n, n);
  else memcpy(planes, samples, sizeof(i64) * n * c);
  CHeader hd = {(u64)w, (u64)h, c, bd, use_rct ? 1 : 0, levels, BLOCK_DIM};
  Pyramid pyr[4];
  memset(pyr, 0, sizeof pyr);
  int rc = 0;
  for (int k = 0; k < c; ++k)
    if ((rc = dwt2d_forward(planes + k * n, w, h, levels, &pyr[k]))) { free(planes); for (int q = 0; q <= k; ++q) pyramid_free(&pyr[q]); return rc; }
  free(planes);
  u64 ns = slots_fill(&hd, NULL);
  Slot* slots = (Slot*)malloc(sizeof(Slot) * ns);
  slots_fill(&hd, slots);
  EncJob j;
  memset(&j, 0, sizeof j);
  j.hd = &hd; j.slots = slots; j.nslots = ns; j.pyr = pyr;
  j.blobs = (uint8_t**)calloc(ns, sizeof(uint8_t*));
  j.lens = (size_t*)calloc(ns, sizeof(size_t));
  atomic_init(&j.next, 0); atomic_init(&j.err, 0); atomic_init(&j.err_slot, 0);
  pthread_mutex_init(&j.mu, NULL);
  run_pool(enc_worker, &j, nthreads);
  rc = atomic_load(&j.err);
  if (rc) snprintf(g_err, sizeof g_err, "%s", j.msg);
  if (!rc) {
    size_t total = HDR_SIZE + IDX_SIZE * ns;
    for (u64 i = 0; i < ns; ++i) total += j.lens[i];
    uint8_t* buf = (uint8_t*)malloc(total ? total : 1);
    header_pack(&hd, buf);
    u64 off = HDR_SIZE + IDX_SIZE * ns;
    for (u64 i = 0; i < ns; ++i) {
      put_u64(buf + HDR_SIZE + IDX_SIZE * i, off);
      put_u32(buf + HDR_SIZE + IDX_SIZE * i + 8, j.lens[i]);
      memcpy(buf + off, j.blobs[i], j.lens[i]);
      off += j.lens[i];
    }
    *out = buf;
    *out_len = total;
  }
  for (u64 i = 0; i < ns; ++i) free(j.blobs[i]);
  free(j.blobs); free(j.lens); free(slots);
  pthread_mutex_destroy(&j.mu);
  for (int k = 0; k < c; ++k) pyramid_free(&pyr[k]);
  return rc;
}

/* ContainerReader, container.py:209-229: header + index validation. */
typedef struct {
  CHeader hd;
  u64 nslots;
  Slot* slots;
  u64* off;
  u64* len;
} Reader;

static void reader_free(Reader* r) { free(r->slots); free(r->off); free(r->len); memset(r, 0, sizeof *r); }

static int reader_open(const uint8_t* d, size_t len, Reader* r) {
  memset(r, 0, sizeof *r);
  int rc = header_parse(d, len, &r->hd);
  if (rc) return rc;
  r->nslots = slots_fill(&r->hd, NULL);
  u64 need = HDR_SIZE + IDX_SIZE * r->nslots;
  if ((u64)len < need) return fail(WBPC_ERR_CONTAINER_PARSE, "container shorter than its index");
  r->slots = (Slot*)malloc(sizeof(Slot) * (r->nslots + 1));
  r->off = (u64*)malloc(sizeof(u64) * (r->nslots + 1));
  r->len = (u64*)malloc(sizeof(u64) * (r->nslots + 1));
  slots_fill(&r->hd, r->slots);
  u64 prev_end = need;
  for (u64 i = 0; i < r->nslots; ++i) {
    u64 o = get_le(d + HDR_SIZE + IDX_SIZE * i, 8), l = get_le(d + HDR_SIZE + IDX_SIZE * i + 8, 4);
    if (o < prev_end || o + l > (u64)len) { reader_free(r); return fail(WBPC_ERR_CORRUPTION, "index entry outside file or overlapping"); }
    prev_end = o + l;
    r->off[i] = o; r->len[i] = l;
  }
  return 0;
}

/* per-slot planes dropped: global n, or per-level (drop_hp[lev-1], drop_ll) */
static int slot_drop(const Slot* s, int n, const int* drop_hp, int drop_ll) {
  if (!drop_hp) return n;
  return s->kind == KIND_LL ? drop_ll : drop_hp[s->lev - 1];
}

typedef struct {
  const uint8_t* data;
  const Reader* rd;
  int channel_planes_only; /* unused */
  int level;
  int n;
  const int* drop_hp;
  int drop_ll;
  /* per channel per level planes with true dims */
  i64** ll;        /* [c] LL at level L, dims llw x llh */
  i64** sub;       /* [(c*L + lev-1)*3 + k] */
  u64* llw; u64* llh;
  const u64* sel;  /* slot indices to decode */
  u64 nsel;
  atomic_ullong next;
  atomic_int err;
  atomic_ullong err_slot;
  char msg[512];
  pthread_mutex_t mu;
} DecJob;

/* decode_slot + _stitch tile placement, container.py:235-298 */
static int decode_one(DecJob* j, u64 si) {
  const Reader* rd = j->rd;
  const Slot* s = &rd->slots[si];
  int dim = rd->hd.dim;
  const uint8_t* blk = j->data + rd->off[si];
  size_t bl = (size_t)rd->len[si];
  int nd = slot_drop(s, j->n, j->drop_hp, j->drop_ll);
  int keep = -1, rc;
  if (nd != 0) {
    BlockHeader bh;
    if ((rc = parse_header(blk, bl, dim, dim, s->kind, &bh))) return rc;
    keep = bh.depth - nd; if (keep < 0) keep = 0;
  }
  size_t tn = (size_t)dim * dim;
  i64* tiles = (i64*)malloc(sizeof(i64) * 3 * tn);
  i64* gp[3] = {tiles, tiles + tn, tiles + 2 * tn};
  if ((rc = wbo_decode_block(blk, bl, dim, s->kind, keep, gp))) { free(tiles); return rc; }
  int L = rd->hd.levels;
  if (s->kind == KIND_LL) {
    i64* dst = j->ll[s->c];
    u64 W = j->llw[s->c], H = j->llh[s->c];
    for (int y = 0; y < dim; ++y) {
      u64 yy = (u64)s->r * dim + y;
      if (yy >= H) break;
      for (int x = 0; x < dim; ++x) {
        u64 xx = (u64)s->col * dim + x;
        if (xx >= W) break;
        dst[yy * W + xx] = gp[0][(size_t)y * dim + x];
      }
    }
  } else {
    u64 pw, ph;
    level_dims(rd->hd.w, rd->hd.h, s->lev - 1, &pw, &ph);
    u64 cw = (pw + 1) / 2, fw = pw / 2, ch = (ph + 1) / 2, fh = ph / 2;
    u64 dw[3] = {cw, fw, fw}, dh[3] = {fh, ch, fh}; /* _subband_dims, container.py:132-137 */
    for (int k = 0; k < 3; ++k) {
      i64* dst = j->sub[((size_t)s->c * L + s->lev - 1) * 3 + k];
      for (int y = 0; y < dim; ++y) {
        u64 yy = (u64)s->r * dim + y;
        if (yy >= dh[k]) break;
        for (int x = 0; x < dim; ++x) {
          u64 xx = (u64)s->col * dim + x;
          if (xx >= dw[k]) break;
          dst[yy * dw[k] + xx] = gp[k][(size_t)y * dim + x];
        }
      }
    }
  }
  free(tiles);
  return 0;
}

static void* dec_worker(void* arg) {
  DecJob* j = (DecJob*)arg;
  for (;;) {
    u64 i = atomic_fetch_add(&j->next, 1);
    if (i >= j->nsel) break;
    u64 si = j->sel[i];
    int rc = decode_one(j, si);
    if (rc) record_err(&j->err, &j->err_slot, &j->mu, j->msg, si, rc);
  }
  return NULL;
}

/* decode_image, container.py:309-335 (+ _finish_image :301-306).  Output: *out = C'*H'*W'
 * int64 planes of the level-`level` image; *oc = output channels (3 for an RCT container
 * claiming 4 channels, as the reference drops the 4th plane). drop_hp/drop_ll optional. */
/* decode_image (container.py:309-335) and, with `region` = {x, y, width, height}, decode_region
 * (container.py:338-390): only slots whose tile meets the per-level box of their level are
 * decoded (_stitch's tile ranges, container.py:261-280), then the window is cropped. */
static int decode_core(const uint8_t* data, size_t len, int level, int planes_dropped, const int* drop_hp,
                       int drop_ll, int nthreads, const int* region, i64** out, int* ow, int* oh, int* oc,
                       int* obd) {
  Reader rd;
  int rc = reader_open(data, len, &rd);
  if (rc) return rc;
  const CHeader* h = &rd.hd;
  if (level < 0 || level > h->levels) { reader_free(&rd); return fail(WBPC_ERR_LEVEL_RANGE, "level must be in [0, %d]", h->levels); }
  if (planes_dropped < 0) { reader_free(&rd); return fail(WBPC_ERR_DOMAIN, "planes_dropped must be >= 0"); }
  i64 box[65][4]; /* per level: r0, r1, c0, c1 (container.py:365-375) */
  if (region) {
    u64 lw, lh;
    level_dims(h->w, h->h, level, &lw, &lh);
    const i64 x = region[0], y = region[1], rw = region[2], rh = region[3];
    if (rw < 1 || rh < 1) { reader_free(&rd); return fail(WBPC_ERR_DOMAIN, "empty region"); }
    if (x < 0 || y < 0 || x + rw > (i64)lw || y + rh > (i64)lh) {
      reader_free(&rd);
      return fail(WBPC_ERR_DOMAIN, "region outside level dimensions");
    }
    box[level][0] = y; box[level][1] = y + rh; box[level][2] = x; box[level][3] = x + rw;
    for (int lev = level + 1; lev <= h->levels; ++lev) {
      u64 bw, bh;
      level_dims(h->w, h->h, lev, &bw, &bh);
      const i64* pb = box[lev - 1];
      i64 r0 = pb[0] / 2 - 4, c0 = pb[2] / 2 - 4;
      box[lev][0] = (r0 > 0 ? r0 : 0) & ~(i64)1;
      box[lev][2] = (c0 > 0 ? c0 : 0) & ~(i64)1;
      i64 r1 = (pb[1] + 1) / 2 + 4, c1 = (pb[3] + 1) / 2 + 4;
      box[lev][1] = r1 < (i64)bh ? r1 : (i64)bh;
      box[lev][3] = c1 < (i64)bw ? c1 : (i64)bw;
    }
  }
  if (h->dim % 4) { reader_free(&rd); return fail(WBPC_ERR_SHAPE, "area grid needs dims that are multiples of (4, 2)"); }
  int L = h->levels, C = h->c;
  DecJob j;
  memset(&j, 0, sizeof j);
  j.data = data; j.rd = &rd; j.level = level; j.n = planes_dropped; j.drop_hp = drop_hp; j.drop_ll = drop_ll;
  j.ll = (i64**)calloc(C, sizeof(i64*));
  j.sub = (i64**)calloc((size_t)C * (L ? L : 1) * 3, sizeof(i64*));
  j.llw = (u64*)calloc(C, sizeof(u64)); j.llh = (u64*)calloc(C, sizeof(u64));
  for (int c = 0; c < C; ++c) {
    level_dims(h->w, h->h, L, &j.llw[c], &j.llh[c]);
    j.ll[c] = (i64*)calloc(j.llw[c] * j.llh[c] + 1, sizeof(i64));
    for (int lev = level + 1; lev <= L; ++lev) {
      u64 pw, ph;
      level_dims(h->w, h->h, lev - 1, &pw, &ph);
      u64 cw = (pw + 1) / 2, fw = pw / 2, ch = (ph + 1) / 2, fh = ph / 2;
      u64 sz[3] = {cw * fh, fw * ch, fw * fh};
      for (int k = 0; k < 3; ++k) j.sub[((size_t)c * L + lev - 1) * 3 + k] = (i64*)calloc(sz[k] + 1, sizeof(i64));
    }
  }
  u64* sel = (u64*)malloc(sizeof(u64) * (rd.nslots + 1));
  u64 nsel = 0;
  for (u64 i = 0; i < rd.nslots; ++i) {
    const Slot* sl = &rd.slots[i];
    if (!(sl->kind == KIND_LL || sl->lev > level)) continue;
    if (region) {
      u64 gw, gh;
      level_dims(h->w, h->h, sl->lev, &gw, &gh);
      const i64* b = box[sl->lev];
      const i64 r1 = b[1] < (i64)gh ? b[1] : (i64)gh, c1 = b[3] < (i64)gw ? b[3] : (i64)gw;
      const i64 d = h->dim;
      if (sl->r < b[0] / d || sl->r >= (r1 + d - 1) / d || sl->col < b[2] / d || sl->col >= (c1 + d - 1) / d) continue;
    }
    sel[nsel++] = i;
  }
  j.sel = sel; j.nsel = nsel;
  atomic_init(&j.next, 0); atomic_init(&j.err, 0); atomic_init(&j.err_slot, 0);
  pthread_mutex_init(&j.mu, NULL);
  run_pool(dec_worker, &j, nthreads);
  rc = atomic_load(&j.err);
  if (rc) snprintf(g_err, sizeof g_err, "%s", j.msg);
  u64 FW = 0, FH = 0;
  level_dims(h->w, h->h, level, &FW, &FH);
  const u64 OX = region ? (u64)region[0] : 0, OY = region ? (u64)region[1] : 0;
  const u64 OW = region ? (u64)region[2] : FW, OH = region ? (u64)region[3] : FH;
  i64* res = NULL;
  if (!rc) {
    res = (i64*)malloc(sizeof(i64) * OW * OH * C + 8);
    for (int c = 0; c < C && !rc; ++c) {
      i64* ll = j.ll[c];
      u64 cw = j.llw[c], chh = j.llh[c];
      int owned = 0;
      for (int lev = L; lev > level; --lev) { /* container.py:328-333 */
        u64 pw, ph;
        level_dims(h->w, h->h, lev - 1, &pw, &ph);
        i64* nxt = (i64*)malloc(sizeof(i64) * pw * ph + 8);
        i64** sb = &j.sub[((size_t)c * L + lev - 1) * 3];
        if ((rc = merge_plane(ll, sb[0], sb[1], sb[2], (int)pw, (int)ph, nxt))) break;
        if (owned) free(ll);
        ll = nxt; owned = 1; cw = pw; chh = ph;
      }
      if (!rc)
        for (u64 y = 0; y < OH; ++y) memcpy(res + (size_t)c * OW * OH + y * OW, ll + (OY + y) * FW + OX, sizeof(i64) * OW);
      if (owned) free(ll);
      (void)cw; (void)chh;
    }
  }
  int outc = C;
  if (!rc && h->color == 1) { /* _finish_image, container.py:301-306 */
    if (C < 3) rc = fail(WBPC_ERR_INDEX, "list index out of range");
    else { rct_inverse(res, res + OW * OH, res + 2 * OW * OH, OW * OH); outc = 3; }
  }
  if (!rc && (h->bd < 1 || h->bd > 16)) rc = fail(WBPC_ERR_DOMAIN, "bit depth must be 1..16, got %d", h->bd);
  for (int c = 0; c < C; ++c) free(j.ll[c]);
  for (size_t k = 0; k < (size_t)C * (L ? L : 1) * 3; ++k) free(j.sub[k]);
  free(j.ll); free(j.sub); free(j.llw); free(j.llh); free(sel);
  pthread_mutex_destroy(&j.mu);
  reader_free(&rd);
  if (rc) { free(res); return rc; }
  *out = res; *ow = (int)OW; *oh = (int)OH; *oc = outc; *obd = h->bd;
  return 0;
}

int wbo_decode_image(const uint8_t* data, size_t len, int level, int planes_dropped, const int* drop_hp, int drop_ll,
                     int nthreads, i64** out, int* ow, int* oh, int* oc, int* obd) {
  return decode_core(data, len, level, planes_dropped, drop_hp, drop_ll, nthreads, NULL, out, ow, oh, oc, obd);
}

int wbo_decode_region(const uint8_t* data, size_t len, int x, int y, int width, int height, int level,
                      int planes_dropped, int nthreads, i64** out, int* ow, int* oh, int* oc, int* obd) {
  const int region[4] = {x, y, width, height};
  return decode_core(data, len, level, planes_dropped, NULL, 0, nthreads, region, out, ow, oh, oc, obd);
}

/* truncate_stream, container.py:393-417 (+ per-level drop vector extension). */
int wbo_truncate_stream(const uint8_t* data, size_t len, int planes_dropped, const int* drop_hp, int drop_ll,
                        uint8_t** out, size_t* out_len) {
  if (planes_dropped < 0) return fail(WBPC_ERR_DOMAIN, "planes_dropped must be >= 0");
  int any = planes_dropped != 0;
  if (drop_hp) { any = drop_ll != 0; for (int i = 0; i < 64; ++i) if (drop_hp[i]) any = 1; }
  if (!any) {
    uint8_t* b = (uint8_t*)malloc(len ? len : 1);
    memcpy(b, data, len);
    *out = b; *out_len = len;
    return 0;
  }
  Reader rd;
  int rc = reader_open(data, len, &rd);
  if (rc) return rc;
  uint8_t** blobs = (uint8_t**)calloc(rd.nslots + 1, sizeof(uint8_t*));
  size_t* lens = (size_t*)calloc(rd.nslots + 1, sizeof(size_t));
  size_t total = HDR_SIZE + IDX_SIZE * rd.nslots;
  for (u64 i = 0; i < rd.nslots && !rc; ++i) {
    int nd = slot_drop(&rd.slots[i], planes_dropped, drop_hp, drop_ll);
    rc = wbo_truncate_block(data + rd.off[i], (size_t)rd.len[i], rd.hd.dim, rd.slots[i].kind, nd, &blobs[i], &lens[i]);
    total += lens[i];
  }
  if (!rc) {
    uint8_t* buf = (uint8_t*)malloc(total);
    header_pack(&rd.hd, buf);
    u64 off = HDR_SIZE + IDX_SIZE * rd.nslots;
    for (u64 i = 0; i < rd.nslots; ++i) {
      put_u64(buf + HDR_SIZE + IDX_SIZE * i, off);
      put_u32(buf + HDR_SIZE + IDX_SIZE * i + 8, lens[i]);
      memcpy(buf + off, blobs[i] ? blobs[i] : data + rd.off[i], lens[i]);
      off += lens[i];
    }
    *out = buf; *out_len = total;
  }
  for (u64 i = 0; i < rd.nslots; ++i) free(blobs[i]);
  free(blobs); free(lens);
  reader_free(&rd);
  return rc;
}

/* ----------------------------------------------------------- test helpers */
/* dwt2d_forward with a packed output: details level 1..L as (lh, hl, hh), then LL. */
int wbo_dwt2d_forward_packed(const i64* plane, int w, int h, int levels, i64* out) {
  Pyramid p;
  int rc = dwt2d_forward(plane, w, h, levels, &p);
  if (rc) return rc;
  size_t o = 0;
  for (int k = 0; k < levels; ++k) {
    int cw = (p.det[k].w + 1) / 2, fw = p.det[k].w / 2, ch = (p.det[k].h + 1) / 2, fh = p.det[k].h / 2;
    memcpy(out + o, p.det[k].lh, sizeof(i64) * (size_t)cw * fh); o += (size_t)cw * fh;
    memcpy(out + o, p.det[k].hl, sizeof(i64) * (size_t)fw * ch); o += (size_t)fw * ch;
    memcpy(out + o, p.det[k].hh, sizeof(i64) * (size_t)fw * fh); o += (size_t)fw * fh;
  }
  memcpy(out + o, p.ll, sizeof(i64) * (size_t)p.llw * p.llh);
  pyramid_free(&p);
  return 0;
}

/* dwt2d_inverse of the packed layout above (transforms.py:219-224). */
int wbo_dwt2d_inverse_packed(const i64* packed, int w, int h, int levels, i64* out) {
  int dw[MAX_LEVELS + 2], dh[MAX_LEVELS + 2];
  size_t offs[MAX_LEVELS + 2];
  dw[0] = w; dh[0] = h;
  size_t o = 0;
  for (int k = 0; k < levels; ++k) {
    offs[k] = o;
    int cw = (dw[k] + 1) / 2, fw = dw[k] / 2, ch = (dh[k] + 1) / 2, fh = dh[k] / 2;
    o += (size_t)cw * fh + (size_t)fw * ch + (size_t)fw * fh;
    dw[k + 1] = cw; dh[k + 1] = ch;
  }
  i64* ll = (i64*)malloc(sizeof(i64) * (size_t)dw[levels] * dh[levels] + 8);
  memcpy(ll, packed + o, sizeof(i64) * (size_t)dw[levels] * dh[levels]);
  for (int k = levels - 1; k >= 0; --k) {
    int cw = (dw[k] + 1) / 2, fw = dw[k] / 2, ch = (dh[k] + 1) / 2, fh = dh[k] / 2;
    const i64* lh = packed + offs[k];
    const i64* hl = lh + (size_t)cw * fh;
    const i64* hh = hl + (size_t)fw * ch;
    i64* nxt = (i64*)malloc(sizeof(i64) * (size_t)dw[k] * dh[k] + 8);
    merge_plane(ll, lh, hl, hh, dw[k], dh[k], nxt);
    free(ll);
    ll = nxt;
  }
  memcpy(out, ll, sizeof(i64) * (size_t)w * h);
  free(ll);
  return 0;
}

/* build_huffman exposed flat: lengths/values per symbol, preorder tree arrays, tree bits. */
int wbo_huffman(const i64* freq, int32_t* code_len, uint32_t* code_val, int32_t* left, int32_t* right, int32_t* sym,
                int32_t* n_nodes, uint8_t* tree_bytes, int64_t* tree_bits) {
  Huff hc;
  int rc = wbo_build_huffman(freq, &hc);
  if (rc) return rc;
  for (int s = 0; s < 256; ++s) { code_len[s] = hc.code_len[s]; code_val[s] = hc.code_val[s]; }
  for (int i = 0; i < hc.n_nodes; ++i) { left[i] = hc.left[i]; right[i] = hc.right[i]; sym[i] = hc.sym[i]; }
  *n_nodes = hc.n_nodes;
  BW w = {0};
  if ((rc = write_tree(&hc, &w))) { free(w.buf); return rc; }
  memcpy(tree_bytes, w.buf, bw_bytes(&w));
  *tree_bits = (int64_t)w.nbits;
  free(w.buf);
  return 0;
}

/* serialize_block exposed: symbols of a block (depth < 0 = minimal); returns depth. */
int wbo_serialize_block(int kind, const i64* grids, int dim, int depth, uint8_t* sym, int* out_depth) {
  int nsub = kind == KIND_LL ? 1 : 3;
  const i64* g[3] = {grids, grids + (size_t)dim * dim, grids + 2 * (size_t)dim * dim};
  i64 peak = 0;
  for (int s = 0; s < nsub; ++s)
    for (size_t i = 0; i < (size_t)dim * dim; ++i) { i64 v = g[s][i] < 0 ? -g[s][i] : g[s][i]; if (v > peak) peak = v; }
  if (depth < 0) depth = 1 + bitlen_u64((u64)peak);
  int* order = (int*)malloc(sizeof(int) * dim * dim / 8);
  area_order(dim, dim, order);
  serialize_block(g, nsub, dim, depth, order, sym);
  free(order);
  *out_depth = depth;
  return 0;
}

int wbo_encode_block_flat(int kind, const i64* grids, int dim, uint8_t** out, size_t* out_len) {
  const i64* g[3] = {grids, grids + (size_t)dim * dim, grids + 2 * (size_t)dim * dim};
  return wbo_encode_block(kind, g, dim, -1, out, out_len);
}

int wbo_decode_block_flat(const uint8_t* data, size_t len, int dim, int kind, int keep, i64* grids) {
  i64* g[3] = {grids, grids + (size_t)dim * dim, grids + 2 * (size_t)dim * dim};
  return wbo_decode_block(data, len, dim, kind, keep, g);
}

u64 wbo_slot_count(int w, int h, int c, int levels) {
  CHeader hd = {(u64)w, (u64)h, c, 8, 0, levels, BLOCK_DIM};
  return slots_fill(&hd, NULL);
}
