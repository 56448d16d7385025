// Experiment: a torch pluggable allocator that backs large buffers with ONE
// physical allocation mapped at a 512 MB-aligned virtual address (CUDA virtual
// memory management API), so the driver is free to map it with pages larger
// than 2 MB.  Stage 3 visits 1024 rows 8.4 MB apart per tile: with 2 MB pages
// every row visit is a different page (4096 pages per slab).
//
//   nvcc -shared -Xcompiler -fPIC -o tools/micro/libhugealloc.so tools/micro/hugealloc.cu -ldl
//   torch.cuda.memory.CUDAPluggableAllocator(path, "huge_malloc", "huge_free")
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sys/types.h>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>

namespace {
struct Drv {
  CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
  CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  CUresult (*access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  CUresult (*release)(CUmemGenericAllocationHandle);
  CUresult (*unmap)(CUdeviceptr, size_t);
  CUresult (*addrfree)(CUdeviceptr, size_t);
  CUresult (*gran)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
  bool ok = false;
} drv;
std::mutex mu;
std::map<void*, size_t> big;  // VMM-backed pointers -> mapped size

bool load() {
  if (drv.ok) return true;
  void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
#define SYM(f, n) *(void**)(&drv.f) = dlsym(h, n); if (!drv.f) return false;
  SYM(create, "cuMemCreate") SYM(reserve, "cuMemAddressReserve") SYM(map, "cuMemMap") SYM(access, "cuMemSetAccess")
  SYM(release, "cuMemRelease") SYM(unmap, "cuMemUnmap") SYM(addrfree, "cuMemAddressFree")
  SYM(gran, "cuMemGetAllocationGranularity")
#undef SYM
  drv.ok = true;
  return true;
}
}  // namespace

extern "C" void* huge_malloc(ssize_t size, int device, cudaStream_t) {
  static const size_t min_big = (size_t)(getenv("HUGE_MIN_MB") ? atol(getenv("HUGE_MIN_MB")) : 256) << 20;
  static const size_t align = (size_t)(getenv("HUGE_ALIGN_MB") ? atol(getenv("HUGE_ALIGN_MB")) : 512) << 20;
  static const bool verbose = getenv("HUGE_VERBOSE") != nullptr;
  cudaSetDevice(device);
  cudaFree(0);
  if ((size_t)size < min_big || !load()) {
    void* p = nullptr;
    return cudaMalloc(&p, size) == cudaSuccess ? p : nullptr;
  }
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  size_t gmin = 0, grec = 0;
  drv.gran(&gmin, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
  drv.gran(&grec, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  const size_t sz = ((size_t)size + align - 1) / align * align;
  CUmemGenericAllocationHandle h;
  CUdeviceptr va = 0;
  CUresult r = drv.create(&h, sz, &prop, 0);
  if (r != CUDA_SUCCESS) { fprintf(stderr, "hugealloc: cuMemCreate(%zu) -> %d\n", sz, (int)r); return nullptr; }
  r = drv.reserve(&va, sz, align, 0, 0);
  if (r != CUDA_SUCCESS) { fprintf(stderr, "hugealloc: reserve -> %d\n", (int)r); drv.release(h); return nullptr; }
  r = drv.map(va, sz, 0, h, 0);
  if (r != CUDA_SUCCESS) { fprintf(stderr, "hugealloc: map -> %d\n", (int)r); drv.addrfree(va, sz); drv.release(h); return nullptr; }
  CUmemAccessDesc acc = {};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  r = drv.access(va, sz, &acc, 1);
  drv.release(h);  // the mapping keeps the memory alive
  if (r != CUDA_SUCCESS) { fprintf(stderr, "hugealloc: access -> %d\n", (int)r); drv.unmap(va, sz); drv.addrfree(va, sz); return nullptr; }
  if (verbose)
    fprintf(stderr, "hugealloc: %zu MB at %p (mapped %zu MB, align %zu MB; granularity min %zu KB, recommended %zu KB)\n",
            (size_t)size >> 20, (void*)va, sz >> 20, align >> 20, gmin >> 10, grec >> 10);
  std::lock_guard<std::mutex> g(mu);
  big[(void*)va] = sz;
  return (void*)va;
}

extern "C" void huge_free(void* ptr, ssize_t, int device, cudaStream_t) {
  cudaSetDevice(device);
  size_t sz = 0;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = big.find(ptr);
    if (it != big.end()) { sz = it->second; big.erase(it); }
  }
  if (!sz) { cudaFree(ptr); return; }
  cudaDeviceSynchronize();
  drv.unmap((CUdeviceptr)ptr, sz);
  drv.addrfree((CUdeviceptr)ptr, sz);
}
