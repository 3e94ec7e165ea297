// TMA box loads from a partially mapped virtual-memory range (development aid):
// reserve 32 MB, map [8 MB, 16 MB), encode a 2D fp64 tensor over the whole range
// (rows of 8 KB), load a box whose rows lie inside the mapped part.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap M, double* out, int c0, int c1, int three) {
  extern __shared__ __align__(1024) double sm[];
  __shared__ __align__(8) unsigned long long bar;
  unsigned sb = (unsigned)__cvta_generic_to_shared(&bar), sd = (unsigned)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(128 * 2 * 8 * (three ? 2 : 1)));
    if (three)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(sd), "l"(&M), "r"(c0), "r"(c1), "r"(0), "r"(sb) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(sd), "l"(&M), "r"(c0), "r"(c1), "r"(sb) : "memory");
  }
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(sb));
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = sm[i];
}
#define G(n) get(#n)
void* get(const char* n) {
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint(n, &p, cudaEnableDefault, &q);
  return p;
}
int main(int argc, char** argv) {
  cudaFree(0);
  auto reserve = (CUresult(*)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long))G(cuMemAddressReserve);
  auto create = (CUresult(*)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long))G(cuMemCreate);
  auto map = (CUresult(*)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long))G(cuMemMap);
  auto access = (CUresult(*)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t))G(cuMemSetAccess);
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  const size_t MB = 1 << 20;
  CUdeviceptr base;
  printf("reserve %d\n", reserve(&base, 32 * MB, 2 * MB, 0, 0));
  CUmemGenericAllocationHandle h;
  printf("create %d\n", create(&h, 8 * MB, &prop, 0));
  printf("map %d\n", map(base + 8 * MB, 8 * MB, 0, h, 0));
  CUmemAccessDesc acc{};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  printf("access %d\n", access(base + 8 * MB, 8 * MB, &acc, 1));
  cudaMemset((void*)(base + 8 * MB), 0, 8 * MB);
  PFN enc = (PFN)G(cuTensorMapEncodeTiled);
  CUtensorMap M;
  cuuint64_t dims[2] = {1024, 4096}, str[1] = {8192};
  cuuint32_t box[2] = {128, 2}, es[2] = {1, 1};
  CUresult r = enc(&M, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  double* o;
  cudaMalloc(&o, 2048);
  int row = argc > 1 ? atoi(argv[1]) : 1500;  // rows 1024..2047 are mapped
  if (argc > 2) {  // rank 0 of P=2 at N=512: 3D {1025, 1025, 2}, mapped [0,6) [8,14) [16,20) MB of 20 MB
    CUdeviceptr b2;
    const char* hint = getenv("HINT");
    printf("reserve2 %d\n", reserve(&b2, 20 * MB, 2 * MB, hint ? (CUdeviceptr)strtoull(hint, 0, 16) : 0, 0));
    printf("base2 %p\n", (void*)b2);
    const size_t ranges[3][2] = {{0, 6}, {8, 14}, {16, 20}};
    for (auto& r : ranges) {
      CUmemGenericAllocationHandle hh;
      create(&hh, (r[1] - r[0]) * MB, &prop, 0);
      map(b2 + r[0] * MB, (r[1] - r[0]) * MB, 0, hh, 0);
      access(b2 + r[0] * MB, (r[1] - r[0]) * MB, &acc, 1);
      cudaMemset((void*)(b2 + r[0] * MB), 0, (r[1] - r[0]) * MB);
    }
    cuuint64_t d3[3] = {1025, 1025, 2}, s3[2] = {1032 * 8, 1057800ull * 8};
    cuuint32_t bx3[3] = {128, 2, 2}, e3[3] = {1, 1, 1};
    CUtensorMap M3;
    CUresult r3 = enc(&M3, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)b2, d3, s3, bx3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int col = atoi(argv[2]);
    k<<<1, 128, 8192>>>(M3, o, col, row, 1);
    printf("3d encode %d col %d row %d: %s\n", r3, col, row, cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
  }
  k<<<1, 128, 8192>>>(M, o, 0, row, 0);
  printf("encode %d row %d: %s\n", r, row, cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
