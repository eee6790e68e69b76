// TMA tile::gather4 probe: which tensor-map box height it needs and how it lays
// out 4 gathered 128-byte rows under the 128-byte swizzle (sm_100a).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void k(const __grid_constant__ CUtensorMap m, int col, int r0, int r1, int r2, int r3,
                  uint16_t* out) {
  __shared__ __align__(1024) uint16_t buf[8 * 64];
  __shared__ __align__(8) uint64_t bar;
  // destination rows 4..7 of a 1024-byte swizzle atom: is the XOR taken from the
  // shared-memory address (4..7) or from the row inside the gather (0..3)?
  for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) buf[i] = 0x7777;
  __syncthreads();
  uint32_t d = (uint32_t)__cvta_generic_to_shared(buf + 4 * 64), b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(512) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d),
        "l"(&m), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b)
        : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(b)
        : "memory");
    for (int i = 0; i < 256; ++i) out[i] = buf[4 * 64 + i];
  }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                        const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                        CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                        CUtensorMapFloatOOBfill);

int main() {
  const int R = 1000, Ccols = 128;
  uint16_t* h = (uint16_t*)malloc(R * Ccols * 2);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < Ccols; ++c) h[r * Ccols + c] = (uint16_t)(r * 256 + c);  // row/col tag
  uint16_t *dsrc, *dout;
  cudaMalloc(&dsrc, R * Ccols * 2);
  cudaMalloc(&dout, 512);
  cudaMemcpy(dsrc, h, R * Ccols * 2, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Enc enc = (Enc)p;
  for (int bh = 1; bh <= 1; bh *= 4) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)Ccols, (cuuint64_t)R};
    cuuint64_t str[1] = {(cuuint64_t)Ccols * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)bh};
    cuuint32_t es[2] = {1, 1};
    CUresult e = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dsrc, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("box height %d: encode %d\n", bh, (int)e);
    if (e) continue;
    cudaMemset(dout, 0xff, 512);
    k<<<1, 32>>>(m, 64, 5, 900, 1 << 20, 3, dout);  // the third row is out of bounds
    cudaError_t ce = cudaDeviceSynchronize();
    printf("  launch %s\n", cudaGetErrorString(ce));
    if (ce) return 1;
    uint16_t o[256];
    cudaMemcpy(o, dout, 512, cudaMemcpyDeviceToHost);
    for (int row = 0; row < 4; ++row) {
      printf("  smem row %d:", row);
      for (int ch = 0; ch < 8; ++ch) {
        const uint16_t v = o[row * 64 + ch * 8];
        printf(" [%04x r%d c%d]", v, v >> 8, v & 255);
      }
      printf("\n");
    }
  }
  return 0;
}
