// standalone TMA probe (development aid): fp64 box loads of various ranks / boxes
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap M, double* out, int rank, int c0, int c1, unsigned bytes) {
  extern __shared__ __align__(1024) double sm[];
  __shared__ __align__(8) unsigned long long bar;
  unsigned sb = (unsigned)__cvta_generic_to_shared(&bar), sd = (unsigned)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(bytes));
    if (rank == 2)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(sd), "l"(&M), "r"(c0), "r"(c1), "r"(sb) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(sd), "l"(&M), "r"(c0), "r"(c1), "r"(0), "r"(sb) : "memory");
  }
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(sb));
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = sm[i];
}
int main(int argc, char** argv) {
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  PFN enc = (PFN)p;
  std::vector<double> h(100000);
  for (size_t i = 0; i < h.size(); ++i) h[i] = i;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8); cudaMalloc(&o, 256 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  struct Case { const char* name; int rank; cuuint64_t dims[3]; cuuint64_t str[2]; cuuint32_t box[3]; int c0, c1; };
  Case cs[] = {
      {"2d 17x17 box128x1 pp24", 2, {17, 17}, {24 * 8}, {128, 1}, -3, 4},
      {"2d 17x17 box16x1 pp24", 2, {17, 17}, {24 * 8}, {16, 1}, 0, 4},
      {"2d 17x17 box16x2 pp24", 2, {17, 17}, {24 * 8}, {16, 2}, 0, 4},
      {"2d 200x17 box128x1 pp256", 2, {200, 17}, {256 * 8}, {128, 1}, 0, 4},
      {"2d 17x17 box16x1 pp32", 2, {17, 17}, {32 * 8}, {16, 1}, 0, 4},
      {"3d 17x17x1 box128x1x1 pp24", 3, {17, 17, 1}, {24 * 8, 24 * 17 * 8}, {128, 1, 1}, -3, 4},
      {"3d 33x33x2 box256x2x2 pu40", 3, {33, 33, 2}, {40 * 8, 1344 * 8}, {256, 2, 2}, -6, 3},
      {"2d 17x17 box32 pp24", 2, {17, 17}, {24 * 8}, {32, 1}, 0, 4},
      {"2d 17x17 box64 pp24", 2, {17, 17}, {24 * 8}, {64, 1}, 0, 4},
      {"2d 33x33 box128 pp40", 2, {33, 33}, {40 * 8}, {128, 1}, 0, 4},
      {"2d 33x33 box256 pp40", 2, {33, 33}, {40 * 8}, {256, 1}, 0, 4},
      {"2d 17x17 box128 pp32", 2, {17, 17}, {32 * 8}, {128, 1}, 0, 4},
      {"2d 65x65 box128 pp72", 2, {65, 65}, {72 * 8}, {128, 1}, 0, 4},
      {"2d 129x129 box128 pp136", 2, {129, 129}, {136 * 8}, {128, 1}, 0, 4},
      {"2d 17x17 box128 pp24 c0=0", 2, {17, 17}, {24 * 8}, {128, 1}, 0, 4},
      {"2d 33x33 box256x2 pp40", 2, {33, 33}, {40 * 8}, {256, 2}, 0, 4},
  };
  int sel = argc > 1 ? atoi(argv[1]) : 0;
  Case& c = cs[sel];
  CUtensorMap M;
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&M, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, c.rank, d + 2688, c.dims, c.str, c.box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned bytes = c.box[0] * c.box[1] * (c.rank == 3 ? c.box[2] : 1) * 8;
  k<<<1, 128, 40000>>>(M, o, c.rank, c.c0, c.c1, bytes);
  cudaError_t e = cudaDeviceSynchronize();
  double rr[256]; cudaMemcpy(rr, o, 2048, cudaMemcpyDeviceToHost);
  printf("%-32s encode %d: %s  [%g %g %g %g]\n", c.name, r, cudaGetErrorString(e), rr[0], rr[1], rr[3], rr[4]);
}
