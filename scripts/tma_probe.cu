// tma_probe.cu — experiment (not part of libbps): TMA streaming throughput for the access
// pattern of the transposed layout.  X is n vectors × d bf16 elements (row pitch d·2 bytes);
// CTA (tile, range) streams boxes of BOXK elements × BOXR vectors along its d-range through a
// 4-deep smem ring; a consumer thread releases each stage as soon as it lands.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_probe scripts/tma_probe.cu -lcuda
//   ./tma_probe d n boxr boxk swizzle(0/1) [ctas] [ring depth]
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "../paper_2602_06071_b200/csrc/bps_ptx.cuh"

using namespace bps;

constexpr int NSTMAX = 64;  // ring depth: argv[7] (default 4)

__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, uint64_t* bar, int32_t c0, int32_t c1, int32_t c2,
                                            uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(
          ptx::smem_u32(dst)),
      "l"(tmap), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
      : "memory");
}

__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap tm, int d, int n, int boxr, int boxk,
                                               int ntiles, int R, int stage_bytes, int NST) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[NSTMAX], empty[NSTMAX];
  const bool rowmajor = ntiles == 0;  // rows of d elements (d ≤ boxk), CTAs stream row boxes
  const int tile = rowmajor ? 0 : blockIdx.x % ntiles, rr = rowmajor ? blockIdx.x : blockIdx.x / ntiles;
  const int64_t nk = rowmajor ? (int64_t)n / boxr : d / (boxk < 0 ? -boxk : boxk);
  const int64_t k0 = nk * rr / R, k1 = nk * (rr + 1) / R;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) ptx::mbar_init(&full[i], 1), ptx::mbar_init(&empty[i], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t pol = ptx::policy_evict_first();
    int s = 0;
    uint32_t ph = 0;
    for (int64_t k = k0; k < k1; ++k) {
      ptx::mbar_wait(&empty[s], ph ^ 1);
      ptx::mbar_arrive_expect_tx(&full[s], stage_bytes);
      if (rowmajor)
        ptx::tma_load_2d(smem + s * stage_bytes, &tm, &full[s], 0, (int32_t)(k * boxr), pol);
      else if (boxk < 0)  // 3D core-matrix box: (8 elements, boxr vectors, -boxk/8 chunks)
        tma_load_3d(smem + s * stage_bytes, &tm, &full[s], 0, tile * boxr, (int32_t)(k * (-boxk / 8)), pol);
      else
        ptx::tma_load_2d(smem + s * stage_bytes, &tm, &full[s], (int32_t)(k * boxk), tile * boxr, pol);
      if (++s == NST) s = 0, ph ^= 1;
    }
  } else if (threadIdx.x == 32) {
    int s = 0;
    uint32_t ph = 0;
    for (int64_t k = k0; k < k1; ++k) {
      ptx::mbar_wait(&full[s], ph);
      ptx::mbar_arrive(&empty[s]);
      if (++s == NST) s = 0, ph ^= 1;
    }
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int64_t d = atoll(argv[1]), n = atoll(argv[2]);
  const int boxr = atoi(argv[3]), boxk = atoi(argv[4]), swz = atoi(argv[5]);
  int ctas = argc > 6 ? atoi(argv[6]) : 148;
  const int NST = argc > 7 ? atoi(argv[7]) : 4;
  void* X;
  if (cudaMalloc(&X, d * n * 2) != cudaSuccess) return 1;
  cudaMemset(X, 0, d * n * 2);
  EncFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)n, 1}, strides[2] = {(cuuint64_t)d * 2, 0};
  cuuint32_t box[3] = {(cuuint32_t)boxk, (cuuint32_t)boxr, 1}, es[3] = {1, 1, 1};
  int rank = 2;
  if (boxk < 0) {  // (8 elems, n vectors, d/8 chunks): strides ldx, 16 B
    rank = 3;
    dims[0] = 8; dims[1] = n; dims[2] = d / 8;
    strides[0] = (cuuint64_t)d * 2; strides[1] = 16;
    box[0] = 8; box[1] = boxr; box[2] = -boxk / 8;
  }
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    return 1;
  }
  int ntiles = (int)(n / boxr);
  int R = ctas / ntiles > 0 ? ctas / ntiles : 1;
  if (d <= boxk) ntiles = 0, R = ctas;  // row-major mode
  const int grid = ntiles ? ntiles * R : R;
  const int sb = boxr * (boxk < 0 ? -boxk : boxk) * 2;
  const int smem = NST * sb + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // the whole matrix is streamed once per launch only if ntiles*R covers it: tiles beyond grid are skipped
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) probe<<<grid, 64, smem>>>(tm, (int)d, (int)n, boxr, boxk, ntiles, R, sb, NST);
  cudaEventRecord(e0);
  const int it = 5;
  for (int w = 0; w < it; ++w) probe<<<grid, 64, smem>>>(tm, (int)d, (int)n, boxr, boxk, ntiles, R, sb, NST);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)d * n * 2;
  printf("nst=%d d=%lld n=%lld boxr=%d boxk=%d swz=%d grid=%d (tiles %d x ranges %d): %.3f ms  %.0f GB/s  err=%s\n",
         NST, (long long)d, (long long)n, boxr, boxk, swz, grid, ntiles, R, ms / it, bytes / (ms / it * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
