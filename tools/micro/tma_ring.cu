// Microbenchmark: aggregate HBM read bandwidth of per-CTA TMA bulk-copy rings
// (cp.async.bulk + mbarrier), the streaming pattern of k_sweep's tile phases.
// ./tma_ring <tile_bytes> <stages> <ctas_per_sm> <tiles_per_cta>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b)));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(par)
      : "memory");
}
__global__ void ring(const double* __restrict__ src, size_t nwords, int tile_bytes, int stages, int tiles,
                     double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar[16];  // stages <= 16
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int q = 0; q < stages; ++q) mbar_init(&mbar[q]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t tw = tile_bytes / 8;
  const size_t ntile_total = nwords / tw;
  auto issue = [&](int k) {
    const int s = k % stages;
    const size_t t = ((size_t)blockIdx.x * tiles + k) * 2654435761ull % ntile_total;  // scattered
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar[s])),
                 "r"((uint32_t)tile_bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(sm + (size_t)s * tile_bytes)),
        "l"(src + t * tw), "r"((uint32_t)tile_bytes), "r"(smem_u32(&mbar[s]))
        : "memory");
  };
  if (tid == 0)
    for (int k = 0; k < stages && k < tiles; ++k) issue(k);
  double acc = 0.0;
  uint32_t par = 0;
  for (int k = 0; k < tiles; ++k) {
    const int s = k % stages;
    mbar_wait(&mbar[s], (par >> s) & 1u);
    par ^= 1u << s;
    const double* T = reinterpret_cast<const double*>(sm + (size_t)s * tile_bytes);
    for (int i = tid; i < tile_bytes / 8; i += blockDim.x) acc += T[i];
    __syncthreads();
    if (tid == 0 && k + stages < tiles) issue(k + stages);
  }
  if (acc == 12345.678) out[0] = acc;
}
int main(int argc, char** argv) {
  int tile = atoi(argv[1]), stages = atoi(argv[2]), per_sm = atoi(argv[3]), tiles = atoi(argv[4]);
  size_t nwords = (size_t)2 << 30 >> 3;  // 2 GB
  double* src;
  double* out;
  cudaMalloc(&src, nwords * 8);
  cudaMemset(src, 0, nwords * 8);
  cudaMalloc(&out, 8);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  size_t smem = (size_t)tile * stages;
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ring, 256, smem);
  int grid = nsm * (per_sm < occ ? per_sm : occ);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    ring<<<grid, 256, smem>>>(src, nwords, tile, stages, tiles, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double bytes = (double)grid * tiles * tile;
  printf("tile %6d stages %d ctas/SM %d (occ %d) grid %4d tiles/cta %4d: %.1f us  %.0f GB/s  err=%s\n", tile, stages,
         per_sm, occ, grid, tiles, ms * 1e3, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
