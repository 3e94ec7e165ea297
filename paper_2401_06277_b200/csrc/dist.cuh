// dist.cuh -- multi-GPU plumbing of libsvk (not in the paper).
//
// Row slabs: on the distributed levels (node rows per rank >= agglom_rows) rank
// r owns node rows [r0, r1) and lattice rows [2 r0, min(2 r1, 2N+1)); slabs are
// nested across levels (r0 doubles from one level to the next finer one).  The
// coarser levels are replicated: every rank runs them redundantly after an
// all-gather of the restricted residual.  Vectors keep the full-size pitched
// layout on every rank; only the owned rows (plus a halo of kHalo = 4 node rows per
// side, refreshed by `exchange`) are meaningful.
//
// Transports:
//  * NcclTransport -- NCCL (loaded with dlopen, so libsvk has no link-time NCCL
//    dependency): grouped ncclSend/ncclRecv with the two neighbours for halos,
//    ncclAllReduce (fp64 sum) for dot products and the all-gather.
//  * EmulTransport -- p logical ranks of one process on one GPU (one host
//    thread per rank): the same operations through a shared group object,
//    device-to-device copies and a host barrier.  Test mode only.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace svk {

// node-row slab of `rank` on a level with N elements, given the coarsest
// distributed level's N (Nla): rows scale by N / Nla so slabs nest.
inline void slab_rows(int N, int Nla, int nranks, int rank, int* r0, int* r1) {
  const int64_t s = N / Nla;
  *r0 = (int)(((int64_t)rank * Nla / nranks) * s);
  *r1 = rank == nranks - 1 ? N + 1 : (int)(((int64_t)(rank + 1) * Nla / nranks) * s);
}

// ----------------------------------------------------------------- slab-local memory
// Virtual-memory-managed vectors: the whole pitched vector is reserved as
// address space and device memory is created and mapped only for given byte
// ranges (rounded to the allocation granularity).  Every other granule of the
// reservation maps ONE shared scratch granule: with the gaps left unmapped,
// TMA tensor loads of these vectors raised illegal-address faults on B200 even
// with every requested row inside the mapped ranges (clamped coordinates,
// compute-sanitizer), while a standalone partially-mapped TMA probe
// (tools/tma_vmm_test.cu) did not; the scratch granule removes the fault at the
// cost of one granule per vector.  No result reads those rows: the
// distributed parity tests poison every row beyond the halo with NaN.
// Driver entry points are fetched with cudaGetDriverEntryPoint (no link-time
// libcuda dependency).
struct SlabMem {
  uintptr_t base = 0;
  size_t reserved = 0;
  std::vector<std::pair<int64_t, int64_t>> maps;  // (offset, bytes) of each mapped range
  std::vector<unsigned long long> handles;        // CUmemGenericAllocationHandle per range
  int64_t mapped = 0;
  // every other granule of the reservation maps one shared scratch granule
  // (never read for results: rows outside the slab + halo are not used)
  unsigned long long scratch = 0;
  std::vector<int64_t> scratch_maps;  // offsets of the granules mapped to `scratch`
  int64_t gran = 0;
};
struct VmmApi {
  CUresult (*AddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*AddressFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*Create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*Release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*Map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*Unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*SetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*Granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  bool ok() const { return AddressReserve && AddressFree && Create && Release && Map && Unmap && SetAccess && Granularity; }
};
inline VmmApi& vmm_api() {
  static VmmApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* n) -> void* {
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(n, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        return nullptr;
      return p;
    };
    a.AddressReserve = (decltype(a.AddressReserve))get("cuMemAddressReserve");
    a.AddressFree = (decltype(a.AddressFree))get("cuMemAddressFree");
    a.Create = (decltype(a.Create))get("cuMemCreate");
    a.Release = (decltype(a.Release))get("cuMemRelease");
    a.Map = (decltype(a.Map))get("cuMemMap");
    a.Unmap = (decltype(a.Unmap))get("cuMemUnmap");
    a.SetAccess = (decltype(a.SetAccess))get("cuMemSetAccess");
    a.Granularity = (decltype(a.Granularity))get("cuMemGetAllocationGranularity");
  });
  return a;
}
inline void slab_free(SlabMem& m) {
  VmmApi& a = vmm_api();
  for (int64_t off : m.scratch_maps) a.Unmap((CUdeviceptr)(m.base + off), (size_t)m.gran);
  if (m.scratch) a.Release((CUmemGenericAllocationHandle)m.scratch);
  for (size_t k = 0; k < m.maps.size(); ++k) {
    if (k < m.handles.size()) {
      a.Unmap((CUdeviceptr)(m.base + m.maps[k].first), (size_t)m.maps[k].second);
      a.Release((CUmemGenericAllocationHandle)m.handles[k]);
    }
  }
  if (m.base) a.AddressFree((CUdeviceptr)m.base, m.reserved);
  m = SlabMem{};
}
// reserve `bytes` of address space on `device` and map the byte ranges `want`
inline int slab_alloc(int device, int64_t bytes, std::vector<std::pair<int64_t, int64_t>> want, SlabMem* out,
                      std::string& err) {
  VmmApi& a = vmm_api();
  if (!a.ok()) {
    err = "CUDA virtual memory management entry points unavailable";
    return -1;
  }
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  size_t gran = 0;
  if (a.Granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || gran == 0) {
    err = "cuMemGetAllocationGranularity failed";
    return -1;
  }
  const int64_t G = (int64_t)gran;
  SlabMem m;
  m.reserved = (size_t)((bytes + G - 1) / G * G);
  CUdeviceptr base = 0;
  if (a.AddressReserve(&base, m.reserved, (size_t)G, 0, 0) != CUDA_SUCCESS) {
    err = "cuMemAddressReserve failed";
    return -1;
  }
  m.base = (uintptr_t)base;
  // round to the granularity, sort, merge
  for (auto& r : want) {
    const int64_t lo = r.first / G * G, hi = std::min<int64_t>((r.second + G - 1) / G * G, (int64_t)m.reserved);
    r = {lo, hi};
  }
  std::sort(want.begin(), want.end());
  std::vector<std::pair<int64_t, int64_t>> merged;
  for (const auto& r : want) {
    if (r.second <= r.first) continue;
    if (!merged.empty() && r.first <= merged.back().second) merged.back().second = std::max(merged.back().second, r.second);
    else merged.push_back(r);
  }
  CUmemAccessDesc acc{};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  for (const auto& r : merged) {
    const size_t sz = (size_t)(r.second - r.first);
    CUmemGenericAllocationHandle h;
    if (a.Create(&h, sz, &prop, 0) != CUDA_SUCCESS) {
      err = "cuMemCreate failed (device memory exhausted?)";
      slab_free(m);
      return -1;
    }
    if (a.Map((CUdeviceptr)(m.base + r.first), sz, 0, h, 0) != CUDA_SUCCESS) {
      a.Release(h);
      err = "cuMemMap failed";
      slab_free(m);
      return -1;
    }
    m.maps.push_back({r.first, (int64_t)sz});
    m.handles.push_back((unsigned long long)h);
    m.mapped += (int64_t)sz;
    if (a.SetAccess((CUdeviceptr)(m.base + r.first), sz, &acc, 1) != CUDA_SUCCESS) {
      err = "cuMemSetAccess failed";
      slab_free(m);
      return -1;
    }
  }
  // the gaps: one shared scratch granule mapped at each
  m.gran = G;
  CUmemGenericAllocationHandle sh;
  if (a.Create(&sh, (size_t)G, &prop, 0) != CUDA_SUCCESS) {
    err = "cuMemCreate (scratch granule) failed";
    slab_free(m);
    return -1;
  }
  m.scratch = (unsigned long long)sh;
  m.mapped += G;
  size_t k = 0;
  for (int64_t off = 0; off < (int64_t)m.reserved; off += G) {
    while (k < merged.size() && merged[k].second <= off) ++k;
    if (k < merged.size() && merged[k].first <= off) continue;  // a real range
    if (a.Map((CUdeviceptr)(m.base + off), (size_t)G, 0, sh, 0) != CUDA_SUCCESS ||
        a.SetAccess((CUdeviceptr)(m.base + off), (size_t)G, &acc, 1) != CUDA_SUCCESS) {
      err = "cuMemMap (scratch granule) failed";
      slab_free(m);
      return -1;
    }
    m.scratch_maps.push_back(off);
  }
  *out = m;
  return 0;
}

// A contiguous block of doubles to send / receive.
struct Block {
  double* ptr;
  int64_t count;
};

class Transport {
 public:
  virtual ~Transport() {}
  // send lo_send to rank-1 and hi_send to rank+1; receive lo_recv from rank-1 and
  // hi_recv from rank+1 (blocks of a side are absent at the domain edges)
  virtual int exchange(const std::vector<Block>& lo_send, const std::vector<Block>& lo_recv,
                       const std::vector<Block>& hi_send, const std::vector<Block>& hi_recv, cudaStream_t s,
                       std::string& err) = 0;
  virtual int allreduce_sum(double* buf, int64_t count, cudaStream_t s, std::string& err) = 0;
  // recv[r * count .. (r+1) * count) = rank r's send[0 .. count) for every rank r
  // (send may alias recv + rank * count)
  virtual int allgather(const double* send, double* recv, int64_t count, cudaStream_t s, std::string& err) = 0;
  // whether its operations may be captured into a CUDA graph (stream-ordered, no host sync)
  virtual bool capturable() const = 0;
  // an asynchronous communication error since the last call (NCCL: ncclCommGetAsyncError), 0 if none
  virtual int async_error(std::string& err) { (void)err; return 0; }
};

// ----------------------------------------------------------------- NCCL
typedef int ncclResult_t_;
typedef void* ncclComm_t_;
struct NcclId {
  char internal[128];
};
struct NcclApi {
  void* h = nullptr;
  ncclResult_t_ (*GetUniqueId)(NcclId*) = nullptr;
  ncclResult_t_ (*CommInitRank)(ncclComm_t_*, int, NcclId, int) = nullptr;
  ncclResult_t_ (*CommDestroy)(ncclComm_t_) = nullptr;
  ncclResult_t_ (*Send)(const void*, size_t, int, int, ncclComm_t_, cudaStream_t) = nullptr;
  ncclResult_t_ (*Recv)(void*, size_t, int, int, ncclComm_t_, cudaStream_t) = nullptr;
  ncclResult_t_ (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t_, cudaStream_t) = nullptr;
  ncclResult_t_ (*AllGather)(const void*, void*, size_t, int, ncclComm_t_, cudaStream_t) = nullptr;
  ncclResult_t_ (*GroupStart)() = nullptr;
  ncclResult_t_ (*GroupEnd)() = nullptr;
  ncclResult_t_ (*CommGetAsyncError)(ncclComm_t_, ncclResult_t_*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t_) = nullptr;
  bool ok() const {
    return h && GetUniqueId && CommInitRank && Send && Recv && AllReduce && AllGather && GroupStart && GroupEnd;
  }
};
inline NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(api.h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(api.h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(api.h, "ncclCommDestroy");
    api.Send = (decltype(api.Send))dlsym(api.h, "ncclSend");
    api.Recv = (decltype(api.Recv))dlsym(api.h, "ncclRecv");
    api.AllReduce = (decltype(api.AllReduce))dlsym(api.h, "ncclAllReduce");
    api.AllGather = (decltype(api.AllGather))dlsym(api.h, "ncclAllGather");
    api.GroupStart = (decltype(api.GroupStart))dlsym(api.h, "ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))dlsym(api.h, "ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(api.h, "ncclGetErrorString");
    api.CommGetAsyncError = (decltype(api.CommGetAsyncError))dlsym(api.h, "ncclCommGetAsyncError");
  });
  return api;
}
constexpr int kNcclDouble = 8, kNcclSum = 0;  // ncclFloat64, ncclSum

class NcclTransport : public Transport {
 public:
  NcclTransport(int rank, int nranks) : rank_(rank), nranks_(nranks) {}
  ~NcclTransport() override {
    if (comm_ && nccl_api().CommDestroy) nccl_api().CommDestroy(comm_);
  }
  int init(const uint8_t id[128], std::string& err) {
    NcclApi& a = nccl_api();
    if (!a.ok()) {
      err = "NCCL (libnccl.so.2) could not be loaded";
      return -1;
    }
    NcclId nid;
    std::memcpy(nid.internal, id, 128);
    const int r = a.CommInitRank(&comm_, nranks_, nid, rank_);
    if (r != 0) {
      err = std::string("ncclCommInitRank: ") + (a.GetErrorString ? a.GetErrorString(r) : "error");
      return -1;
    }
    return 0;
  }
  int exchange(const std::vector<Block>& lo_send, const std::vector<Block>& lo_recv, const std::vector<Block>& hi_send,
               const std::vector<Block>& hi_recv, cudaStream_t s, std::string& err) override {
    NcclApi& a = nccl_api();
    int r = a.GroupStart();
    for (const Block& b : lo_send)
      if (!r && b.count) r = a.Send(b.ptr, b.count, kNcclDouble, rank_ - 1, comm_, s);
    for (const Block& b : lo_recv)
      if (!r && b.count) r = a.Recv(b.ptr, b.count, kNcclDouble, rank_ - 1, comm_, s);
    for (const Block& b : hi_send)
      if (!r && b.count) r = a.Send(b.ptr, b.count, kNcclDouble, rank_ + 1, comm_, s);
    for (const Block& b : hi_recv)
      if (!r && b.count) r = a.Recv(b.ptr, b.count, kNcclDouble, rank_ + 1, comm_, s);
    const int r2 = a.GroupEnd();
    if (r || r2) {
      err = "NCCL halo exchange failed";
      return -1;
    }
    return 0;
  }
  int allreduce_sum(double* buf, int64_t count, cudaStream_t s, std::string& err) override {
    if (nccl_api().AllReduce(buf, buf, (size_t)count, kNcclDouble, kNcclSum, comm_, s) != 0) {
      err = "ncclAllReduce failed";
      return -1;
    }
    return 0;
  }
  bool capturable() const override { return true; }  // NCCL operations are stream-capturable
  int async_error(std::string& err) override {
    NcclApi& a = nccl_api();
    if (!a.CommGetAsyncError || !comm_) return 0;
    ncclResult_t_ r = 0;
    if (a.CommGetAsyncError(comm_, &r) != 0 || r != 0) {
      err = std::string("NCCL asynchronous error: ") + (a.GetErrorString ? a.GetErrorString(r) : "error");
      return -1;
    }
    return 0;
  }
  int allgather(const double* send, double* recv, int64_t count, cudaStream_t s, std::string& err) override {
    if (nccl_api().AllGather(send, recv, (size_t)count, kNcclDouble, comm_, s) != 0) {
      err = "ncclAllGather failed";
      return -1;
    }
    return 0;
  }

 private:
  int rank_, nranks_;
  ncclComm_t_ comm_ = nullptr;
};

// ----------------------------------------------------------------- emulation
// p logical ranks in one process (one host thread each) on one device.
struct EmulGroup {
  int nranks;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  // per-rank slots for the current collective
  std::vector<std::vector<Block>> lo_send, hi_send;
  std::vector<std::vector<double>> red;
  std::vector<const double*> gsend;
  explicit EmulGroup(int n) : nranks(n), lo_send(n), hi_send(n), red(n), gsend(n, nullptr) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t gen = generation;
    if (++arrived == nranks) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};
inline std::mutex& emul_registry_mu() {
  static std::mutex m;
  return m;
}
inline std::map<int, std::weak_ptr<EmulGroup>>& emul_registry() {
  static std::map<int, std::weak_ptr<EmulGroup>> r;
  return r;
}

class EmulTransport : public Transport {
 public:
  EmulTransport(int rank, int nranks, int key) : rank_(rank) {
    std::lock_guard<std::mutex> lk(emul_registry_mu());
    auto& w = emul_registry()[key];
    group_ = w.lock();
    if (!group_) {
      group_ = std::make_shared<EmulGroup>(nranks);
      w = group_;
    }
  }
  int exchange(const std::vector<Block>& lo_send, const std::vector<Block>& lo_recv, const std::vector<Block>& hi_send,
               const std::vector<Block>& hi_recv, cudaStream_t s, std::string& err) override {
    if (const cudaError_t e = cudaStreamSynchronize(s); e != cudaSuccess) {
      err = std::string("emulated exchange: stream sync failed: ") + cudaGetErrorString(e);
      return -1;
    }
    EmulGroup& G = *group_;
    G.lo_send[rank_] = lo_send;
    G.hi_send[rank_] = hi_send;
    G.barrier();
    // my lo_recv = (rank-1)'s hi_send; my hi_recv = (rank+1)'s lo_send
    cudaError_t e = cudaSuccess;
    for (size_t k = 0; k < lo_recv.size(); ++k) {
      const cudaError_t ek = cudaMemcpy(lo_recv[k].ptr, G.hi_send[rank_ - 1][k].ptr, lo_recv[k].count * sizeof(double),
                                        cudaMemcpyDeviceToDevice);
      if (e == cudaSuccess) e = ek;
    }
    for (size_t k = 0; k < hi_recv.size(); ++k) {
      const cudaError_t ek = cudaMemcpy(hi_recv[k].ptr, G.lo_send[rank_ + 1][k].ptr, hi_recv[k].count * sizeof(double),
                                        cudaMemcpyDeviceToDevice);
      if (e == cudaSuccess) e = ek;
    }
    G.barrier();  // every rank reaches it, also on error (no rank may be left waiting)
    if (e != cudaSuccess) {
      err = std::string("emulated exchange: copy failed: ") + cudaGetErrorString(e);
      return -1;
    }
    return 0;
  }
  int allreduce_sum(double* buf, int64_t count, cudaStream_t s, std::string& err) override {
    EmulGroup& G = *group_;
    G.red[rank_].resize(count);
    if (cudaMemcpyAsync(G.red[rank_].data(), buf, count * sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
      err = "emulated allreduce: copy failed";
      return -1;
    }
    G.barrier();
    std::vector<double> sum(count, 0.0);
    for (int r = 0; r < G.nranks; ++r)  // fixed rank order: deterministic
      for (int64_t i = 0; i < count; ++i) sum[i] += G.red[r][i];
    G.barrier();
    if (const cudaError_t e = cudaMemcpy(buf, sum.data(), count * sizeof(double), cudaMemcpyHostToDevice);
        e != cudaSuccess) {
      err = std::string("emulated allreduce: copy back failed: ") + cudaGetErrorString(e);
      return -1;
    }
    return 0;
  }
  bool capturable() const override { return false; }  // host barriers
  int allgather(const double* send, double* recv, int64_t count, cudaStream_t s, std::string& err) override {
    if (const cudaError_t e = cudaStreamSynchronize(s); e != cudaSuccess) {
      err = std::string("emulated allgather: stream sync failed: ") + cudaGetErrorString(e);
      return -1;
    }
    EmulGroup& G = *group_;
    std::vector<double> mine((size_t)count);  // a copy, so that send may alias recv
    cudaError_t e = cudaMemcpy(mine.data(), send, count * sizeof(double), cudaMemcpyDeviceToHost);
    G.red[rank_] = mine;
    G.barrier();
    for (int r = 0; r < G.nranks; ++r) {
      const cudaError_t er = cudaMemcpy(recv + (int64_t)r * count, G.red[r].data(), count * sizeof(double),
                                        cudaMemcpyHostToDevice);
      if (e == cudaSuccess) e = er;
    }
    G.barrier();
    if (e != cudaSuccess) {
      err = std::string("emulated allgather: copy failed: ") + cudaGetErrorString(e);
      return -1;
    }
    return 0;
  }

 private:
  int rank_;
  std::shared_ptr<EmulGroup> group_;
};

}  // namespace svk
