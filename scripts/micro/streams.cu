// Microbenchmark: DRAM efficiency of strip-walking kernels as a function of the number of
// concurrent plane streams.  Each warp walks down a strip of R rows; per row it reads SEG bytes
// (coalesced) from each of NS source planes and writes SEG bytes to each of ND destination planes.
// Planes are (H x PITCH bytes).  Mode 1 interleaves the planes' rows (row r of plane k at
// (r * NP + k) * PITCH) instead of plane-major.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
template <int V>  // V = 4-byte words per lane per row
__global__ void __launch_bounds__(256) k_walk(const uint32_t* src, uint32_t* dst, int ns, int nd, int H, int pitchw,
                                               int R, int inter) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sxn = pitchw / (32 * V);
  const int strip = blockIdx.x * 8 + warp;
  const int sx = strip % sxn, sy = strip / sxn;
  if (sy * R >= H) return;
  const long plane = (long)H * pitchw;
  uint32_t acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = 0;
  for (int r = sy * R; r < sy * R + R && r < H; ++r) {
    for (int k = 0; k < ns; ++k) {
      const long off = inter ? ((long)r * ns + k) * pitchw : k * plane + (long)r * pitchw;
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] += __ldg(src + off + sx * 32 * V + v * 32 + lane);
    }
    for (int k = 0; k < nd; ++k) {
      const long off = inter ? ((long)r * nd + k) * pitchw : k * plane + (long)r * pitchw;
#pragma unroll
      for (int v = 0; v < V; ++v) dst[off + sx * 32 * V + v * 32 + lane] = acc[v] + k;
    }
  }
}
int main() {
  const int H = 8192, pitchw = 2048;  // 8 KB rows, 64 MB planes
  const int NP = 16;
  uint32_t *src, *dst;
  cudaMalloc(&src, (size_t)NP * H * pitchw * 4);
  cudaMalloc(&dst, (size_t)NP * H * pitchw * 4);
  cudaMemset(src, 1, (size_t)NP * H * pitchw * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int cfgs[][2] = {{1, 1}, {2, 2}, {4, 4}, {8, 8}, {12, 1}, {12, 3}, {1, 12}, {3, 12}, {16, 16}, {6, 6}};
  for (int inter = 0; inter < 2; ++inter)
    for (int V = 1; V <= 4; V *= 2)
      for (int R : {16, 64})
        for (auto& c : cfgs) {
          const int ns = c[0], nd = c[1];
          const int strips = (pitchw / (32 * V)) * ((H + R - 1) / R);
          float best = 1e9;
          for (int it = 0; it < 4; ++it) {
            cudaEventRecord(e0);
            if (V == 1) k_walk<1><<<(strips + 7) / 8, 256>>>(src, dst, ns, nd, H, pitchw, R, inter);
            else if (V == 2) k_walk<2><<<(strips + 7) / 8, 256>>>(src, dst, ns, nd, H, pitchw, R, inter);
            else k_walk<4><<<(strips + 7) / 8, 256>>>(src, dst, ns, nd, H, pitchw, R, inter);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
          }
          const double bytes = (double)(ns + nd) * H * pitchw * 4;
          printf("inter=%d V=%d R=%2d ns=%2d nd=%2d  %.3f ms  %.0f GB/s\n", inter, V, R, ns, nd, best, bytes / best / 1e6);
        }
  return 0;
}
