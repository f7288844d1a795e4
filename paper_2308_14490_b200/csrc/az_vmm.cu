// Growable device buffers on the CUDA virtual-memory API: one virtual range is reserved for the
// largest size a buffer can reach (the sketch S of az_factorize at max_blocks probe blocks, up to
// ~160 GB on the c5 configuration), and physical HBM is mapped behind it only as probe blocks are
// added; the unused tail is unmapped and returned once the block count is final.  The pointer stays
// valid (and the layout, ld = rows, unchanged) throughout, so kernels see one contiguous matrix.
//
// The driver entry points are fetched through cudaGetDriverEntryPoint, so libaz links only the
// runtime.
#include <cuda.h>

#include <vector>

#include "az_internal.h"

namespace {
using PFN_create = CUresult (*)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
using PFN_release = CUresult (*)(CUmemGenericAllocationHandle);
using PFN_reserve = CUresult (*)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
using PFN_free = CUresult (*)(CUdeviceptr, size_t);
using PFN_map = CUresult (*)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
using PFN_unmap = CUresult (*)(CUdeviceptr, size_t);
using PFN_access = CUresult (*)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
using PFN_gran = CUresult (*)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);

struct Drv {
  PFN_create create = nullptr;
  PFN_release release = nullptr;
  PFN_reserve reserve = nullptr;
  PFN_free vfree = nullptr;
  PFN_map map = nullptr;
  PFN_unmap unmap = nullptr;
  PFN_access access = nullptr;
  PFN_gran gran = nullptr;
  bool ok = false;
};

template <typename F>
bool entry(const char* name, F* fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
      !p) {
    cudaGetLastError();
    return false;
  }
  *fn = (F)p;
  return true;
}

const Drv& drv() {
  static Drv d = [] {
    Drv x;
    x.ok = entry("cuMemCreate", &x.create) && entry("cuMemRelease", &x.release) &&
           entry("cuMemAddressReserve", &x.reserve) && entry("cuMemAddressFree", &x.vfree) &&
           entry("cuMemMap", &x.map) && entry("cuMemUnmap", &x.unmap) && entry("cuMemSetAccess", &x.access) &&
           entry("cuMemGetAllocationGranularity", &x.gran);
    return x;
  }();
  return d;
}
}  // namespace

struct az_vbuf_s {
  CUdeviceptr base = 0;
  size_t reserved = 0, mapped = 0, gran = 0;
  int dev = 0;
  std::vector<CUmemGenericAllocationHandle> chunks;   // one handle per mapped chunk
  std::vector<size_t> sizes;
};

static CUmemAllocationProp vprop(int dev) {
  CUmemAllocationProp pr = {};
  pr.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  pr.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  pr.location.id = dev;
  return pr;
}

az_vbuf_s* az_vbuf_reserve(size_t max_bytes) {
  const Drv& d = drv();
  if (!d.ok || max_bytes == 0) return nullptr;
  az_vbuf_s* v = new az_vbuf_s();
  cudaGetDevice(&v->dev);
  CUmemAllocationProp pr = vprop(v->dev);
  if (d.gran(&v->gran, &pr, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || v->gran == 0) {
    delete v;
    return nullptr;
  }
  v->reserved = (max_bytes + v->gran - 1) / v->gran * v->gran;
  if (d.reserve(&v->base, v->reserved, 0, 0, 0) != CUDA_SUCCESS) {
    delete v;
    return nullptr;
  }
  return v;
}

void* az_vbuf_ptr(az_vbuf_s* v) { return v ? (void*)v->base : nullptr; }

// map physical memory so that [0, bytes) is backed; false (nothing changed) when HBM is short
bool az_vbuf_ensure(az_vbuf_s* v, size_t bytes) {
  const Drv& d = drv();
  if (!v || bytes > v->reserved) return false;
  if (bytes <= v->mapped) return true;
  const size_t want = (bytes + v->gran - 1) / v->gran * v->gran;
  const size_t add = want - v->mapped;
  CUmemAllocationProp pr = vprop(v->dev);
  CUmemGenericAllocationHandle h;
  if (d.create(&h, add, &pr, 0) != CUDA_SUCCESS) return false;
  if (d.map(v->base + v->mapped, add, 0, h, 0) != CUDA_SUCCESS) {
    d.release(h);
    return false;
  }
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = v->dev;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (d.access(v->base + v->mapped, add, &ad, 1) != CUDA_SUCCESS) {
    d.unmap(v->base + v->mapped, add);
    d.release(h);
    return false;
  }
  v->chunks.push_back(h);
  v->sizes.push_back(add);
  v->mapped = want;
  return true;
}

// unmap and release whole chunks lying entirely beyond `bytes` (callers synchronise first)
void az_vbuf_trim(az_vbuf_s* v, size_t bytes) {
  const Drv& d = drv();
  if (!v) return;
  while (!v->chunks.empty() && v->mapped - v->sizes.back() >= bytes) {
    const size_t sz = v->sizes.back();
    d.unmap(v->base + v->mapped - sz, sz);
    d.release(v->chunks.back());
    v->chunks.pop_back();
    v->sizes.pop_back();
    v->mapped -= sz;
  }
}

size_t az_vbuf_mapped(az_vbuf_s* v) { return v ? v->mapped : 0; }

void az_vbuf_free(az_vbuf_s* v) {
  if (!v) return;
  const Drv& d = drv();
  az_vbuf_trim(v, 0);
  if (v->base) d.vfree(v->base, v->reserved);
  delete v;
}
