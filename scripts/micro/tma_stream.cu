// Microbenchmark: row streaming through a cp.async.bulk ring (producer warp + TW consumer warps)
// with the consumers doing no math -- the data-supply ceiling of the level-1 forward DWT layout.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int TW = 4, NST = 16, ROWB = 16 + 384 * TW + 16;
__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(n)); }
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void bar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(b)) : "memory"); }
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(s_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s_u32(dst)), "l"(src), "r"(bytes), "r"(s_u32(b)) : "memory");
}
// mode 0: TMA ring, consumers only read; mode 1: + each consumer writes 12 u32 per row pair (int16 output volume)
__global__ void __launch_bounds__((TW + 1) * 32) k_ring(const uint8_t* img, int W, int H, int sr, uint32_t* out, int mode) {
  __shared__ __align__(128) uint8_t ring[NST][ROWB];
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N0 = blockIdx.x * TW * 64, m0 = blockIdx.y * sr, b = blockIdx.z;
  const long rowbytes = (long)W * 3;
  const long s0 = 6L * N0 - 16;
  const long c0 = s0 < 0 ? 0 : s0, c1 = s0 + ROWB < rowbytes ? s0 + ROWB : rowbytes;
  const uint32_t nb = (uint32_t)(c1 - c0);
  const uint8_t* base = img + (long)b * rowbytes * H;
  const int nrows = 2 * sr + 3;
  if (threadIdx.x == 0) { for (int i = 0; i < NST; ++i) { bar_init(&full[i], 1); bar_init(&empty[i], TW); } asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  if (warp == TW) {
    if (lane == 0)
      for (int r = 0; r < nrows; ++r) {
        const int sl = r % NST;
        if (r >= NST) bar_wait(&empty[sl], ((r / NST) - 1) & 1);
        int y = 2 * m0 - 2 + r; y = y < 0 ? -y : (y >= H ? 2 * H - 2 - y : y);
        bar_expect(&full[sl], nb);
        bulk_g2s(ring[sl] + (c0 - s0), base + (long)y * rowbytes + c0, nb, &full[sl]);
      }
    return;
  }
  uint32_t acc = 0;
  const long pw = W / 2;
  uint32_t* o = out + ((long)b * 12 * (H / 2) + m0) * (pw / 2) + (N0 + 64 * warp) / 2 + lane;
  for (int r = 0; r < nrows; ++r) {
    const int sl = r % NST;
    bar_wait(&full[sl], (r / NST) & 1);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(ring[sl] + 8 + 384 * warp + 12 * lane);
    acc += w[0] ^ w[1] ^ w[2] ^ w[3] ^ w[4] ^ w[5];
    __syncwarp();
    if (lane == 0) bar_arrive(&empty[sl]);
    const int work = mode & 0xFFFF;
    if (work >= 2) {  // fake lifting work: 6 independent chains, `mode` steps each
      uint32_t c[6];
#pragma unroll
      for (int i = 0; i < 6; ++i) c[i] = acc + i;
      for (int it = 0; it < work; ++it)
#pragma unroll
        for (int i = 0; i < 6; ++i) c[i] = c[i] * 3u + (c[(i + 1) % 6] >> 2);
      acc = c[0] ^ c[1] ^ c[2] ^ c[3] ^ c[4] ^ c[5];
    }
    if (!(mode & 0x10000) && mode >= 1 && r >= 3 && (r & 1)) {
      uint32_t* q = o + (long)((r - 3) / 2) * (pw / 2);
#pragma unroll
      for (int k = 0; k < 12; ++k) q[(long)k * (H / 2) * (pw / 2)] = acc + k;
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}
// plain LDG version: warp reads its 6 words per row directly from global
__global__ void __launch_bounds__(128) k_ldg(const uint8_t* img, int W, int H, int sr, uint32_t* out, int mode) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N0 = blockIdx.x * TW * 64, m0 = blockIdx.y * sr, b = blockIdx.z;
  const long rowbytes = (long)W * 3;
  const uint8_t* base = img + (long)b * rowbytes * H;
  const int nrows = 2 * sr + 3;
  long off = 6L * N0 + 384 * warp + 12 * lane - 8; if (off < 0) off = 0; if (off + 24 > rowbytes) off = rowbytes - 24;
  uint32_t acc = 0;
  const long pw = W / 2;
  uint32_t* o = out + ((long)b * 12 * (H / 2) + m0) * (pw / 2) + (N0 + 64 * warp) / 2 + lane;
  for (int r = 0; r < nrows; ++r) {
    int y = 2 * m0 - 2 + r; y = y < 0 ? -y : (y >= H ? 2 * H - 2 - y : y);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(base + (long)y * rowbytes + off);
    acc += __ldg(w) ^ __ldg(w + 1) ^ __ldg(w + 2) ^ __ldg(w + 3) ^ __ldg(w + 4) ^ __ldg(w + 5);
    if (mode == 1 && r >= 3 && (r & 1)) {
      uint32_t* q = o + (long)((r - 3) / 2) * (pw / 2);
#pragma unroll
      for (int k = 0; k < 12; ++k) q[(long)k * (H / 2) * (pw / 2)] = acc + k;
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}
int main(int argc, char** argv) {
  const int only = argc > 1 ? (int)strtol(argv[1], nullptr, 0) : -1;
  const int W = 2048, H = 2048, B = 8;
  uint8_t* img; uint32_t* out; uint8_t* flush;
  cudaMalloc(&img, (size_t)W * H * 3 * B); cudaMalloc(&out, (size_t)W * H * 3 * B * 2 + 64); cudaMalloc(&flush, 256 << 20);
  cudaMemset(img, 7, (size_t)W * H * 3 * B);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int sr : {16}) for (int kind = 0; kind < 1; ++kind) for (int mode : {0, 1, 10, 20, 40, 0x10000 + 10, 0x10000 + 20, 0x10000 + 40}) {
    if (only >= 0 && mode != only) continue;
    dim3 grid(W / 2 / (TW * 64), H / 2 / sr, B);
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
      cudaMemsetAsync(flush, it, 256 << 20);
      cudaEventRecord(e0);
      if (kind == 0) k_ring<<<grid, (TW + 1) * 32>>>(img, W, H, sr, out, mode);
      else k_ldg<<<grid, TW * 32>>>(img, W, H, sr, out, mode);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (it) best = ms < best ? ms : best;
    }
    printf("sr %d %s mode %x: %.1f us  (%s)\n", sr, kind ? "ldg " : "tma ", mode, best * 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
