// Dev probe: a 3D TMA tile load with an mbarrier, variants of the PTX form.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int V>
__global__ void k(const __grid_constant__ CUtensorMap map, const CUtensorMap *gmap, float *out, int cx, int cy, int cz, int bytes) {
  __shared__ __align__(128) float buf[36 * 18];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bytes) : "memory");
    const CUtensorMap *m = V == 2 ? gmap : &map;
    if (V == 0)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                   ::"r"(su(buf)), "l"((uint64_t)m), "r"(su(&bar)), "r"(cx), "r"(cy), "r"(cz) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                   ::"r"(su(buf)), "l"((uint64_t)m), "r"(su(&bar)), "r"(cx), "r"(cy), "r"(cz) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(su(&bar)) : "memory");
  for (int i = threadIdx.x; i < 36 * 18; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int nx = 16, ny = 16, nz = 16;
  float *g, *out;
  cudaMalloc(&g, nx * ny * nz * 4);
  cudaMalloc(&out, 36 * 18 * 4);
  float h[nx * ny * nz];
  for (int i = 0; i < nx * ny * nz; ++i) h[i] = (float)i;
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  printf("entry %p q %d\n", fn, (int)q);
  CUtensorMap map;
  const cuuint64_t dim[3] = {nx, ny, nz}, str[2] = {nx * 4, nx * ny * 4};
  const int BX = BOXX, BY = BOXY;
  const cuuint32_t box[3] = {BX, BY, 1}, es[3] = {1, 1, 1};
  CUresult r = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, g, dim, str, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  CUtensorMap *gm;
  cudaMalloc(&gm, sizeof(map));
  cudaMemcpy(gm, &map, sizeof(map), cudaMemcpyHostToDevice);
  float o[36 * 18];
  k<0><<<1, 128>>>(map, gm, out, CX, CY, 1, BX * BY * 4);
  printf("box %d x %d at (%d,%d): %s\n", BX, BY, CX, CY, cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
  printf("  o[0..3] %g %g %g %g  o[37] %g\n", o[0], o[1], o[2], o[3], o[37]);
  return 0;
}
