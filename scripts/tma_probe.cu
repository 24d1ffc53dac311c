// Isolates the 2-D TMA halo load used by the config-5 tile body.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cstdlib>

struct Big { int64_t pad[64]; alignas(64) CUtensorMap map[2]; int x; };

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap m0, const __grid_constant__ Big big, uint32_t* out, int cx, int cy,
                  int bytes) {
  extern __shared__ __align__(128) uint8_t dyn[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t off = ((su(dyn) + 127u) & ~127u) - su(dyn);
  uint32_t* box = (uint32_t*)(dyn + off);
  const CUtensorMap* map = MODE == 0 ? &m0 : &big.map[1];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su(box)), "l"(map), "r"(cx), "r"(cy), "r"(su(&bar)) : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(su(&bar)) : "memory");
  for (int i = threadIdx.x; i < 68 * 66; i += blockDim.x) out[i] = box[i];
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int bw = argc > 2 ? atoi(argv[2]) : 68, bh = argc > 3 ? atoi(argv[3]) : 66;
  const int cx = argc > 4 ? atoi(argv[4]) : -2, cy = argc > 5 ? atoi(argv[5]) : -1;
  const int prom = argc > 6 ? atoi(argv[6]) : 3;
  const int nx = 256, ny = 256;
  uint32_t *g, *out;
  cudaMalloc(&g, nx * ny * 4);
  cudaMalloc(&out, 68 * 66 * 4);
  uint32_t* h = (uint32_t*)malloc(nx * ny * 4);
  for (int i = 0; i < nx * ny; ++i) h[i] = i + 1;
  cudaMemcpy(g, h, nx * ny * 4, cudaMemcpyHostToDevice);
  typedef CUresult (*enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fp;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  CUtensorMap m;
  const cuuint64_t dims[2] = {nx, ny}, str[1] = {nx * 4};
  const cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh}, es[2] = {1, 1};
  CUresult r = ((enc)fp)(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d\n", (int)r);
  Big b;
  memset(&b, 0, sizeof b);
  b.map[0] = m;
  b.map[1] = m;
  const int dyn = bw * bh * 4 + 128;
  auto fn = mode == 0 ? k<0> : k<1>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
  if (mode == 2) {
    int bytes = bw * bh * 4;
    int xx = cx, yy = cy;
    void* args[] = {&m, &b, &out, &xx, &yy, &bytes};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k<1>, dim3(1), dim3(128), args, dyn, 0);
    printf("coop launch: %s\n", cudaGetErrorString(e));
  } else {
    fn<<<1, 128, dyn>>>(m, b, out, cx, cy, bw * bh * 4);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("mode %d box %dx%d at (%d,%d) prom %d: %s\n", mode, bw, bh, cx, cy, prom, cudaGetErrorString(e));
  uint32_t ho[68 * 66];
  cudaMemcpy(ho, out, sizeof ho, cudaMemcpyDeviceToHost);
  // box row 0 is y=-1 (zeros), row 1 col 2 is (0,0) = 1
  printf("box[0]=%u box[1*68+2]=%u box[1*68+1]=%u box[2*68+2]=%u\n", ho[0], ho[68 + 2], ho[68 + 1], ho[2 * 68 + 2]);
  return 0;
}
