/*
 * wbpc_b200.h — C ABI of the B200 (sm_100a) encode/decode hot path of the
 * wavelet bit-plane codec (arXiv 2005.08713; reference package `wbpc`).
 *
 * Every entry point takes plain pointers and sizes (device pointers where the
 * name says d_*), a cudaStream_t passed as void*, and returns a wbpc_status.
 * All device work is stream-ordered; the library allocates no persistent
 * device memory (the caller passes a workspace sized by the *_plan_size call).
 * Device-side errors (corrupt streams, out-of-range samples) are recorded in
 * the workspace and read back with wbpc_query_status().
 *
 * Reference interface each entry point replaces (paths under /root/reference):
 *   wbpc_parse_header      ContainerHeader.parse      pkg/src/wbpc/container.py:89-108
 *   wbpc_encode            encode_image               pkg/src/wbpc/container.py:167-206
 *   wbpc_decode            decode_image               pkg/src/wbpc/container.py:309-335
 *   wbpc_truncate          truncate_stream            pkg/src/wbpc/container.py:393-417
 *   wbpc_decode_tokens     _kernels.decode_tokens     pkg/src/wbpc/_kernels.py:33-89
 *   status codes           wbpc.errors classes        pkg/src/wbpc/errors.py:4-61
 */
#ifndef WBPC_B200_H
#define WBPC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One value per exception class of pkg/src/wbpc/errors.py (same order). */
typedef enum wbpc_status {
  WBPC_OK = 0,
  WBPC_ERR_UNSUPPORTED_LAYOUT = 1, /* UnsupportedLayoutError  errors.py:8  */
  WBPC_ERR_SHAPE = 2,              /* ShapeError              errors.py:12 */
  WBPC_ERR_DOMAIN = 3,             /* DomainError             errors.py:16 */
  WBPC_ERR_LEVEL_RANGE = 4,        /* LevelRangeError         errors.py:20 */
  WBPC_ERR_DEPTH_OVERFLOW = 5,     /* DepthOverflowError      errors.py:24 */
  WBPC_ERR_STREAM_INDEX = 6,       /* StreamIndexError        errors.py:28 */
  WBPC_ERR_EMPTY_ALPHABET = 7,     /* EmptyAlphabetError      errors.py:32 */
  WBPC_ERR_CODE_LENGTH = 8,        /* CodeLengthError         errors.py:36 */
  WBPC_ERR_MALFORMED_TREE = 9,     /* MalformedTreeError      errors.py:40 */
  WBPC_ERR_TRUNCATION = 10,        /* TruncationError         errors.py:44 */
  WBPC_ERR_MALFORMED_PAYLOAD = 11, /* MalformedPayloadError   errors.py:48 */
  WBPC_ERR_BLOCK_PARSE = 12,       /* BlockParseError         errors.py:52 */
  WBPC_ERR_CORRUPTION = 13,        /* CorruptionError         errors.py:56 */
  WBPC_ERR_CONTAINER_PARSE = 14,   /* ContainerParseError     errors.py:60 */
  WBPC_ERR_INDEX = 15,             /* builtin IndexError: RCT container with <3 channels (container.py:304) */
  /* library-level conditions (no reference counterpart) */
  WBPC_ERR_CUDA = 100,             /* a CUDA runtime call failed */
  WBPC_ERR_WORKSPACE = 101,        /* workspace smaller than *_plan_size reported */
  WBPC_ERR_OUT_CAPACITY = 102,     /* output buffer too small; the required size was still written */
  WBPC_ERR_INVALID_ARG = 103,      /* null pointer / unsupported dtype or layout */
  WBPC_ERR_UNSUPPORTED = 104       /* valid for the reference, outside this build (e.g. block_dim != 128) */
} wbpc_status;

/* Sample element types and layouts for pixel buffers. */
enum { WBPC_DTYPE_U8 = 0, WBPC_DTYPE_U16 = 1, WBPC_DTYPE_I16 = 2, WBPC_DTYPE_I32 = 3,
       /* decode output only: samples clipped to [0, 2^bit_depth - 1] and, for bit_depth > 8,
        * rescaled to 8 bits as (v*255 + maxval/2) / maxval -- the tile service's display
        * conversion (service.py:72-78) */
       WBPC_DTYPE_U8_DISPLAY = 4 };
enum { WBPC_LAYOUT_CHW = 0, WBPC_LAYOUT_HWC = 1 };

/* Parsed 19-byte container header (container.py:58,66-108). */
typedef struct wbpc_header {
  uint32_t width;
  uint32_t height;
  uint32_t channels;
  uint32_t bit_depth;
  uint32_t color_transform; /* 0 none, 1 reversible colour transform */
  uint32_t levels;
  uint32_t block_dim;       /* always 128 for containers this library writes */
} wbpc_header;

/* A batch of equally shaped images laid out back to back in device memory. */
typedef struct wbpc_image_desc {
  uint32_t width;
  uint32_t height;
  uint32_t channels;   /* 1..4 */
  uint32_t bit_depth;  /* 1..16 */
  int32_t dtype;       /* WBPC_DTYPE_U8 or WBPC_DTYPE_U16 (or I32 holding unsigned samples) */
  int32_t layout;      /* WBPC_LAYOUT_CHW (planar) or WBPC_LAYOUT_HWC (interleaved) */
  uint64_t image_stride_bytes; /* distance between consecutive images of the batch */
} wbpc_image_desc;

int wbpc_abi_version(void);
/* Human-readable message of the last failing call on this host thread. */
const char* wbpc_last_error(void);

/* Host-side header parse + validation (ContainerHeader.parse, container.py:89-108). */
int wbpc_parse_header(const uint8_t* host_data, size_t len, wbpc_header* out);
/* Number of block slots of a container with this header (iter_slots, container.py:115-129). */
int wbpc_slot_count(const wbpc_header* hdr, uint64_t* out_slots);

/* ---- encode: encode_image(image, levels, use_rct) for a batch of images ------------ */
int wbpc_encode_plan_size(const wbpc_image_desc* desc, uint32_t batch, int levels, int use_rct,
                          size_t* ws_bytes, size_t* out_cap_hint);
/* Bytes per stored wavelet coefficient the encoder uses for this configuration: 2 when the
 * static filter-norm bound keeps every coefficient inside int16 (8/9/10-bit images at the usual
 * level counts), else 4.  New (no reference counterpart): lets callers account the encode
 * kernels' algorithmic HBM bytes. */
int wbpc_encode_coef_bytes(const wbpc_image_desc* desc, int levels, int use_rct, int* out_bytes);
/* Containers are written back to back into d_out; d_out_offsets[0..batch] (device, u64)
 * receives the start of each container and the total length.  If the total exceeds
 * out_cap nothing past out_cap is written and wbpc_query_status reports
 * WBPC_ERR_OUT_CAPACITY with aux = required bytes. */
int wbpc_encode(const wbpc_image_desc* desc, const void* d_pixels, uint32_t batch, int levels,
                int use_rct, void* d_ws, size_t ws_bytes, uint8_t* d_out, size_t out_cap,
                uint64_t* d_out_offsets, void* stream);

/* ---- decode: decode_image(data, level, planes_dropped) ------------------------------ */
int wbpc_decode_plan_size(const wbpc_header* hdr, int level, size_t* ws_bytes);
/* drop_ll / drop_hp: optional per-level plane drops (host arrays; drop_hp[l-1] for detail
 * level l, drop_ll for the LL grid).  When both are NULL every block drops planes_dropped
 * planes, exactly as decode_image(planes_dropped=n).  Output samples are channel planar
 * (CHW) or interleaved (HWC) in out_dtype; values are NOT clamped (container.py:313-316). */
int wbpc_decode(const wbpc_header* hdr, const uint8_t* d_container, size_t container_len,
                int level, int planes_dropped, const int32_t* drop_hp, int32_t drop_ll,
                void* d_out, int out_dtype, int out_layout, void* d_ws, size_t ws_bytes,
                void* stream);

/* ---- truncate: truncate_stream(data, planes_dropped) --------------------------------- */
int wbpc_truncate_plan_size(const wbpc_header* hdr, size_t container_len, size_t* ws_bytes,
                            size_t* out_cap);
int wbpc_truncate(const wbpc_header* hdr, const uint8_t* d_container, size_t container_len,
                  int planes_dropped, const int32_t* drop_hp, int32_t drop_ll, void* d_ws,
                  size_t ws_bytes, uint8_t* d_out, size_t out_cap, uint64_t* d_out_len,
                  void* stream);

/* Synchronise `stream` and read the device status word of a workspace used by the
 * last encode/decode/truncate call: *status = wbpc_status, *aux = detail (slot index
 * of the first failing block, or required output bytes for WBPC_ERR_OUT_CAPACITY). */
int wbpc_query_status(const void* d_ws, void* stream, int32_t* status, uint64_t* aux);

/* Batched decode of `batch` equally shaped containers packed in d_data; d_img_offsets
 * (device, u64[batch+1]) delimits them (as written by wbpc_encode). */
int wbpc_decode_batch_plan_size(const wbpc_header* hdr, uint32_t batch, size_t* ws_bytes);
int wbpc_decode_batch(const wbpc_header* hdr, const uint8_t* d_data, size_t total_len,
                      const uint64_t* d_img_offsets, uint32_t batch, int level, int planes_dropped,
                      void* d_out, int out_dtype, int out_layout, void* d_ws, size_t ws_bytes,
                      void* stream);

/* plane_offsets (blocks.py:253-261): for one block (kind 0 = LL, 1 = HP3), the stored slots
 * (b*nsub + s, serialization order) and their payload bit offsets; *d_count = their number
 * (<= 96).  Errors as parse_header.  Workspace: wbpc_block_plan_size(kind, 1). */
int wbpc_plane_offsets(int kind, const uint8_t* d_block, size_t len, int32_t* d_slots, uint32_t* d_offsets,
                       int32_t* d_count, void* d_ws, size_t ws_bytes, void* stream);

/* Region decode: the (x, y, width, height) window of the level-`level` image, pixel identical
 * to cropping wbpc_decode's output.  Replaces wbpc.decode_region (container.py:338-390): only
 * blocks whose tile meets the per-level boxes (4-coefficient margin) are decoded, so errors
 * are raised only by those blocks.  d_out holds width*height*channels samples.  The workspace
 * is wbpc_decode_plan_size's. */
int wbpc_decode_region(const wbpc_header* hdr, const uint8_t* d_container, size_t len, int32_t x, int32_t y,
                       int32_t width, int32_t height, int level, int planes_dropped, void* d_out,
                       int out_dtype, int out_layout, void* d_ws, size_t ws_bytes, void* stream);

/* Per-block header summary for container_info (container.py:420-456): parses every block's
 * header (index order) and writes its depth and payload_start (header bits) to device arrays
 * of wbpc_slot_count() entries.  Errors as blockcodec.parse_header.  Workspace as decode. */
int wbpc_block_summary(const wbpc_header* hdr, const uint8_t* d_container, size_t len, int32_t* d_depth,
                       uint32_t* d_header_bits, void* d_ws, size_t ws_bytes, void* stream);

/* Sized copy for host-buffer pipelines: copies *d_nbytes bytes (a device-resident count, e.g.
 * the total of wbpc_encode's d_out_offsets) from src to dst, where either may be device memory
 * or pinned host memory (unified addressing).  Stream ordered, no host synchronisation. */
int wbpc_copy_sized(void* dst, const void* src, const uint64_t* d_nbytes, void* stream);

/* ---- whole-slide tile archive (BASELINE configs[3]) ----------
 * No reference counterpart: the reference encodes one image per container and has no
 * multi-container format (its index assembly loop is container.py:199-206; the archive layout is
 * paper_2005_08713_b200/archive.py: "WBPA" u8 1, u32 tiles_x, u32 tiles_y, (u64 off, u64 len)
 * per tile, then the tile containers).  A rank encodes its contiguous shard of tiles in batches
 * of `batch` tiles with wbpc_encode; batch k writes its containers into region k of a store
 * (k * region_bytes) and its offsets to d_enc_offsets[k * (batch + 1) ...].
 *   wbpc_archive_tile_sizes: this rank's per-tile container bytes into d_sizes[0..per) (zero
 *     padded past n_local) -- the payload of the all-gather across ranks (NCCL).
 *   wbpc_archive_index: from all tiles' sizes (row-major tile order), the archive header + index
 *     (d_header, 13 + 16 * n_tiles bytes, optional), this rank's tile offsets relative to its
 *     first tile (d_local_offsets, n_local + 1 entries) and d_base_total[0] = archive offset of
 *     the rank's first tile, d_base_total[1] = total archive bytes.
 *   wbpc_archive_gather: moves every tile of the rank from its batch region to
 *     d_dst + d_local_offsets[i] (the rank's contiguous range of the archive). */
int wbpc_archive_tile_sizes(const uint64_t* d_enc_offsets, uint32_t batch, uint32_t n_local, uint32_t per,
                            uint64_t* d_sizes, void* stream);
int wbpc_archive_index(const uint64_t* d_sizes_all, uint32_t n_tiles, uint32_t tiles_x, uint32_t tiles_y,
                       uint32_t first, uint32_t n_local, uint8_t* d_header, uint64_t* d_local_offsets,
                       uint64_t* d_base_total, void* stream);
int wbpc_archive_gather(const uint8_t* d_store, uint64_t region_bytes, const uint64_t* d_enc_offsets, uint32_t batch,
                        uint32_t n_local, uint8_t* d_dst, const uint64_t* d_local_offsets, void* stream);
/* Streaming assembly of a rank's archive range: after batch k is encoded, its tiles' rank-local
 * offsets follow from its own container offsets (d_enc_offsets_k, batch_tiles + 1 entries) and the
 * base d_local_offsets_k[0] written by batch k-1 (0 for the first batch); writes
 * d_local_offsets_k[1 .. batch_tiles].  Launches of consecutive batches must be ordered. */
int wbpc_archive_batch_offsets(const uint64_t* d_enc_offsets_k, uint32_t batch_tiles, uint64_t* d_local_offsets_k,
                               void* stream);

/* Per-kernel device timing with CUDA events recorded on the launching stream (bench/profiling
 * only; not thread safe).  collect() synchronises, aggregates by kernel name and resets. */
int wbpc_profile_enable(int on);
int wbpc_profile_collect(char* names, size_t names_len, double* ms, int* counts, int max_entries,
                         int* n_out);

/* ---- block API: encode_block / decode_block / truncate_block (blocks.py:84-304) --------------
 * n blocks of one kind (0 = LL, 1 = HP3), 128x128 each.  Coefficients (int32) are planar per
 * subband: LL [n][128][128], HP3 [3][n][128][128] (LH, HL, HH).  Blocks are packed back to back;
 * d_offsets[0..n] (device, u64) delimits them.  d_depth (optional, int32[n]) forces the plane
 * depth (CoefficientBlock.depth) instead of the minimal one; planes_to_keep < 0 means None. */
int wbpc_block_plan_size(int kind, uint32_t n, size_t* ws_bytes, size_t* out_cap_hint);
int wbpc_encode_blocks(int kind, uint32_t n, const int32_t* d_coeffs, const int32_t* d_depth, void* d_ws,
                       size_t ws_bytes, uint8_t* d_out, size_t out_cap, uint64_t* d_offsets, void* stream);
int wbpc_decode_blocks(int kind, uint32_t n, const uint8_t* d_data, size_t len, const uint64_t* d_offsets,
                       int planes_to_keep, int32_t* d_coeffs_out, void* d_ws, size_t ws_bytes, void* stream);
int wbpc_truncate_blocks(int kind, uint32_t n, const uint8_t* d_data, size_t len, const uint64_t* d_offsets,
                         int planes_dropped, void* d_ws, size_t ws_bytes, uint8_t* d_out, size_t out_cap,
                         uint64_t* d_out_offsets, void* stream);

/* ---- token decode, argument for argument the reference kernel ------------------------ */
/* _kernels.decode_tokens(payload, start_bit, end_bit, left, right, leaf_symbol, zr_symbol,
 * counter_width, seg_lengths, out_symbols, out_seg_starts) -> (status, end_bit).
 * All arrays are device pointers; d_result[0] = status (0 ok, 1 truncated, 2 overrun),
 * d_result[1] = end bit position. */
int wbpc_decode_tokens(const uint8_t* d_payload, int64_t start_bit, int64_t end_bit,
                       const int32_t* d_left, const int32_t* d_right,
                       const int32_t* d_leaf_symbol, int32_t n_nodes, int32_t zr_symbol,
                       int32_t counter_width, const int64_t* d_seg_lengths, int32_t n_segments,
                       uint8_t* d_out_symbols, int64_t* d_out_seg_starts, int64_t* d_result,
                       void* stream);

#ifdef __cplusplus
}
#endif
#endif /* WBPC_B200_H */
