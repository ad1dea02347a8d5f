// Variant tile arithmetic vs the sweep's current one (cycles per tile).
#include "../../paper_2311_18783_b200/csrc/sweep.cu"
#include <cstdio>

namespace mdd {
namespace dev {
// division-free slice mapping: power-of-two row groups and slice counts
template <class Fin>
__device__ __forceinline__ void tile_matvec_v2(const double* T, int R, int C, const double* v, double* red, Fin fin) {
  const int tid = threadIdx.x;
  if (R > kSweepThreads / 2) {
    for (int i = tid; i < R; i += kSweepThreads) {
      double s0 = 0.0, s1 = 0.0;
      int j = 0;
      for (; j + 2 <= C; j += 2) {
        s0 += T[j * R + i] * v[j];
        s1 += T[(j + 1) * R + i] * v[j + 1];
      }
      if (j < C) s0 += T[j * R + i] * v[j];
      fin(i, s0 + s1);
    }
    return;
  }
  const int lg = R <= 4 ? 2 : R <= 8 ? 3 : R <= 16 ? 4 : R <= 32 ? 5 : R <= 64 ? 6 : 7;
  const int lgs = 8 - lg;  // log2 of the slice count (kSweepThreads = 256)
  const int i = tid & ((1 << lg) - 1), sl = tid >> lg;
  // slice sl covers columns [sl*C >> lgs, (sl+1)*C >> lgs) (possibly empty)
  if (i < R) {
    const int ja = (sl * C) >> lgs, jb = ((sl + 1) * C) >> lgs;
    double s0 = 0.0, s1 = 0.0;
    int j = ja;
    for (; j + 2 <= jb; j += 2) {
      s0 += T[j * R + i] * v[j];
      s1 += T[(j + 1) * R + i] * v[j + 1];
    }
    if (j < jb) s0 += T[j * R + i] * v[j];
    red[tid] = s0 + s1;  // = red[sl * Rp + i]
  }
  __syncthreads();
  if (tid < R) {
    double s = 0.0;
    for (int q = 0; q < (1 << lgs); ++q) s += red[(q << lg) + tid];
    fin(tid, s);
  }
}
template <class Fin>
__device__ __forceinline__ void tile_matvec_packed_v2(const double* T, int nr, int c0, int C, const double* v,
                                                      double* red, Fin fin) {
  const int tid = threadIdx.x;
  const int R = nr - c0;
  const int lg = R <= 32 ? 5 : R <= 64 ? 6 : R <= 128 ? 7 : 8;
  const int Rp = 1 << lg;
  const int nsl = R > 256 ? 1 : min(kSweepThreads >> lg, C);
  if (R > 256) {
    for (int ip = tid; ip < R; ip += kSweepThreads) {
      const int jb = min(C, ip + 1);
      double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
      int jj = 0;
      for (; jj + 4 <= jb; jj += 4) {
        const int a0 = jj * R - (jj * (jj - 1)) / 2 + ip - jj;
        const int a1 = a0 + R - jj - 1, a2 = a1 + R - jj - 2, a3 = a2 + R - jj - 3;
        s0 += T[a0] * v[jj]; s1 += T[a1] * v[jj + 1]; s2 += T[a2] * v[jj + 2]; s3 += T[a3] * v[jj + 3];
      }
      for (; jj < jb; ++jj) s0 += T[jj * R - (jj * (jj - 1)) / 2 + ip - jj] * v[jj];
      fin(c0 + ip, (s0 + s1) + (s2 + s3));
    }
    return;
  }
  const int ip = tid & (Rp - 1), sl = tid >> lg;
  if (sl < nsl && ip < R) {
    const int ja = (sl * C) / nsl, jb = min(((sl + 1) * C) / nsl, ip + 1);
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    int jj = ja;
    for (; jj + 4 <= jb; jj += 4) {
      const int a0 = jj * R - (jj * (jj - 1)) / 2 + ip - jj;
      const int a1 = a0 + R - jj - 1, a2 = a1 + R - jj - 2, a3 = a2 + R - jj - 3;
      s0 += T[a0] * v[jj]; s1 += T[a1] * v[jj + 1]; s2 += T[a2] * v[jj + 2]; s3 += T[a3] * v[jj + 3];
    }
    for (; jj < jb; ++jj) s0 += T[jj * R - (jj * (jj - 1)) / 2 + ip - jj] * v[jj];
    if (nsl == 1) { fin(c0 + ip, (s0 + s1) + (s2 + s3)); return; }
    red[sl * Rp + ip] = (s0 + s1) + (s2 + s3);
  }
  if (nsl == 1) return;
  __syncthreads();
  for (int q2 = tid; q2 < R; q2 += kSweepThreads) {
    double s = 0.0;
    for (int q = 0; q < nsl; ++q) s += red[q * Rp + q2];
    fin(c0 + q2, s);
  }
}

__global__ void k_tilebench(int which, int nr, int C, int reps, long long* cyc, double* out) {
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
    if (which == 0) tile_matvec_packed(T, nr, 0, C, v, red, [&](int i, double y) { vec2[i] += y; });
    else if (which == 1) tile_matvec_packed_v2(T, nr, 0, C, v, red, [&](int i, double y) { vec2[i] += y; });
    else if (which == 2) tile_matvec(T, nr, C, v, red, [&](int i, double y) { vec2[i] += y; });
    else tile_matvec_v2(T, nr, C, v, red, [&](int i, double y) { vec2[i] += y; });
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
  struct Case { int which, nr, C; const char* name; } cases[] = {
      {2, 52, 8, "2-D new 52x8"}, {2, 52, 64, "2-D new 52x64"}, {2, 16, 200, "strip new 16x200"},
      {2, 6, 500, "strip new 6x500"}, {2, 100, 33, "strip new 100x33"}, {0, 125, 30, "packed new 125x30"},
      {0, 80, 48, "packed new 80x48"}, {0, 12, 10, "packed new 12x10"}, {0, 200, 18, "packed new 200x18"}};
  for (auto& c : cases) {
    mdd::dev::k_tilebench<<<1, mdd::dev::kSweepThreads, smem>>>(c.which, c.nr, c.C, 200, cyc, out);
    long long h = 0;
    double o[4];
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(o, out, 32, cudaMemcpyDeviceToHost);
    printf("%-26s %6lld cycles  out0 %.10e %s\n", c.name, h, o[0], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
