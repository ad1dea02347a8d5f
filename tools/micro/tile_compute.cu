// Microbenchmark: cycles of the sweep's per-tile arithmetic (one CTA, tile resident
// in shared memory, clock64 around N repetitions).  Includes sweep.cu for its
// tile functions.  ./tile_compute
#include "../../paper_2311_18783_b200/csrc/sweep.cu"
#include <cstdio>

namespace mdd {
namespace dev {
__global__ void k_tilebench(int which, int nr, int c0, int C, int reps, long long* cyc, double* out) {
  extern __shared__ __align__(128) double smx[];
  double* T = smx;
  double* v = smx + kTileMax;
  double* red = v + kVecMax + 2;
  double* vec2 = red + kSweepThreads;
  for (int i = threadIdx.x; i < kTileMax; i += blockDim.x) T[i] = 1.0 + 1e-3 * i;
  for (int i = threadIdx.x; i < kVecMax; i += blockDim.x) { v[i] = 0.5 + 1e-4 * i; vec2[i] = 0.0; }
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (which == 0) tile_matvec_packed(T, nr, c0, C, v, red, [&](int i, double y) { vec2[i] += y; });
    else if (which == 1) tile_matvec_t_packed(T, nr, c0, C, v, red, [&](int j, double y) { vec2[j] += y; });
    else if (which == 2) tile_matvec(T, nr, C, v, red, [&](int i, double y) { vec2[i] += y; });
    else tile_matvec_t(T, nr, C, v, red, [&](int j, double y) { vec2[j] += y; });
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = (t1 - t0) / reps;
  if (threadIdx.x < 4) out[threadIdx.x] = vec2[threadIdx.x];
}
}  // namespace dev
}  // namespace mdd

int main() {
  long long* cyc;
  double* out;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&out, 64);
  const int smem = (mdd::dev::kTileMax + 2 * mdd::dev::kVecMax + 2 + mdd::dev::kSweepThreads) * 8;
  cudaFuncSetAttribute(mdd::dev::k_tilebench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  struct Case { int which, nr, c0, C; const char* name; } cases[] = {
      {0, 125, 0, 30, "fwd packed nr=125 C=30"}, {0, 200, 0, 18, "fwd packed nr=200 C=18"},
      {0, 80, 0, 48, "fwd packed nr=80 C=48"}, {1, 125, 0, 30, "bwd packed nr=125 C=30"},
      {1, 200, 0, 18, "bwd packed nr=200 C=18"}, {2, 52, 0, 64, "fwd 2-D 52x64"},
      {3, 52, 0, 64, "bwd 2-D 52x64"}, {2, 16, 0, 200, "fwd strip 16x200"}, {3, 300, 0, 11, "bwd strip 300x11"}};
  for (auto& c : cases) {
    mdd::dev::k_tilebench<<<1, mdd::dev::kSweepThreads, smem>>>(c.which, c.nr, c.c0, c.C, 200, cyc, out);
    long long h = 0;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-26s %6lld cycles per tile (incl. one __syncthreads)  %s\n", c.name, h,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
