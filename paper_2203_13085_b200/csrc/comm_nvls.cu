// NVLink SHARP (tolerance mode): the mean all-reduce reduced inside the NVSwitch.
//
// The communicator's two snapshot slots and its mean buffer move into one cuMem
// allocation per rank, bound to a multicast object that spans every rank's GPU.  A
// rank reduces its chunk of partition_chunks(n, P) with multimem.ld_reduce on the
// multicast address of the current slot (the switch fetches the P copies and adds
// them), scales by 1/P and multicasts the mean into every rank's mean buffer with
// multimem.st.  Per link direction a rank moves (P+1)/P*B instead of the P2P
// kernels' 2(P-1)/P*B; the SMs issue B/P loads and B/P stores.  The switch's
// summation order is not the reference ring's, so the result matches
// execute_allreduce (collective.py:154-203) only to rounding (the north star's 1e-6
// relative) — but every rank receives the same bits, because one switch result is
// multicast to all.  The bit-exact algorithms stay the default.
//
// Setup (lasgd_comm_nvls_*): rank 0 creates the multicast object and exports it as a
// POSIX file descriptor, which the host layer passes to the other ranks (SCM_RIGHTS
// over a UNIX socket); every rank imports it, adds its device, and — once all have —
// binds its own physical allocation and maps both the unicast and the multicast
// view.  Driver entry points come from cudaGetDriverEntryPoint (no libcuda link).
#include <cuda.h>
#include <string.h>
#include <unistd.h>

#include "comm_nvls.h"

namespace lasgd {

// ------------------------------------------------------------------ driver entry points
namespace {
struct Drv {
  bool ok = false;
  CUresult (*MulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                               unsigned long long) = nullptr;
  CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*MulticastGetGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*MemRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*MemAddressFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*MemUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*MemExportToShareableHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                         unsigned long long) = nullptr;
  CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
  CUresult (*DeviceGet)(CUdevice*, int) = nullptr;
  CUresult (*DeviceGetAttribute)(int*, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*GetErrorString)(CUresult, const char**) = nullptr;
};

template <typename F>
bool sym(const char* name, F& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess || !p)
    return false;
  fn = reinterpret_cast<F>(p);
  return true;
}

const Drv& drv() {
  static Drv d;
  static bool init = false;
  if (!init) {
    init = true;
    d.ok = sym("cuMulticastCreate", d.MulticastCreate) && sym("cuMulticastAddDevice", d.MulticastAddDevice) &&
           sym("cuMulticastBindMem", d.MulticastBindMem) && sym("cuMulticastUnbind", d.MulticastUnbind) &&
           sym("cuMulticastGetGranularity", d.MulticastGetGranularity) && sym("cuMemCreate", d.MemCreate) &&
           sym("cuMemRelease", d.MemRelease) && sym("cuMemAddressReserve", d.MemAddressReserve) &&
           sym("cuMemAddressFree", d.MemAddressFree) && sym("cuMemMap", d.MemMap) && sym("cuMemUnmap", d.MemUnmap) &&
           sym("cuMemSetAccess", d.MemSetAccess) && sym("cuMemExportToShareableHandle", d.MemExportToShareableHandle) &&
           sym("cuMemImportFromShareableHandle", d.MemImportFromShareableHandle) && sym("cuDeviceGet", d.DeviceGet) &&
           sym("cuDeviceGetAttribute", d.DeviceGetAttribute) && sym("cuGetErrorString", d.GetErrorString);
  }
  return d;
}

int cu_fail(CUresult r, const char* what) {
  const char* s = nullptr;
  if (drv().GetErrorString) drv().GetErrorString(r, &s);
  return fail(LASGD_ERR_CUDA, "%s: %s (%d)", what, s ? s : "?", (int)r);
}
#define CU_TRY(expr)                                  \
  do {                                                \
    CUresult _r = (expr);                             \
    if (_r != CUDA_SUCCESS) return cu_fail(_r, #expr); \
  } while (0)
}  // namespace

struct NvlsState {
  int device = 0, world = 1;
  size_t bytes = 0;  // mapped size (multiple of the multicast granularity)
  size_t gran = 0;
  CUmemGenericAllocationHandle mc = 0, mem = 0;
  bool have_mc = false, have_mem = false, bound = false, added = false;
  CUdeviceptr uc = 0, mcva = 0;
};

int nvls_supported(int device) {
  const Drv& d = drv();
  if (!d.ok) return 0;
  CUdevice dev;
  if (d.DeviceGet(&dev, device) != CUDA_SUCCESS) return 0;
  int mc = 0, fd = 0;
  d.DeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  d.DeviceGetAttribute(&fd, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev);
  return mc && fd ? 1 : 0;
}

static CUmulticastObjectProp mc_prop(int world, size_t bytes) {
  CUmulticastObjectProp p;
  memset(&p, 0, sizeof(p));
  p.numDevices = (unsigned)world;
  p.size = bytes;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return p;
}

int nvls_create(NvlsState** out, int device, int world, size_t payload_bytes, int* fd_out) {
  const Drv& d = drv();
  if (!d.ok) return fail(LASGD_ERR_UNSUPPORTED, "driver has no multicast entry points");
  NvlsState* s = new NvlsState();
  s->device = device;
  s->world = world;
  CUmulticastObjectProp p = mc_prop(world, payload_bytes);
  CUresult r = d.MulticastGetGranularity(&s->gran, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED);
  if (r != CUDA_SUCCESS) {
    delete s;
    return cu_fail(r, "cuMulticastGetGranularity");
  }
  s->bytes = (payload_bytes + s->gran - 1) / s->gran * s->gran;
  p.size = s->bytes;
  if (fd_out) {  // the creating rank
    r = d.MulticastCreate(&s->mc, &p);
    if (r != CUDA_SUCCESS) {
      delete s;
      return cu_fail(r, "cuMulticastCreate");
    }
    s->have_mc = true;
    int fd = -1;
    r = d.MemExportToShareableHandle(&fd, s->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    if (r != CUDA_SUCCESS) {
      nvls_destroy(s);
      return cu_fail(r, "cuMemExportToShareableHandle(multicast)");
    }
    *fd_out = fd;
  }
  *out = s;
  return LASGD_OK;
}

int nvls_import(NvlsState* s, int fd) {
  if (s->have_mc) {
    close(fd);
    return fail(LASGD_ERR_STATE, "multicast object already present");
  }
  const CUresult r =
      drv().MemImportFromShareableHandle(&s->mc, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  close(fd);  // the import holds its own reference
  if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemImportFromShareableHandle(multicast)");
  s->have_mc = true;
  return LASGD_OK;
}

int nvls_add_device(NvlsState* s) {
  if (!s->have_mc) return fail(LASGD_ERR_STATE, "no multicast object");
  CUdevice dev;
  CU_TRY(drv().DeviceGet(&dev, s->device));
  CU_TRY(drv().MulticastAddDevice(s->mc, dev));
  s->added = true;
  return LASGD_OK;
}

int nvls_bind(NvlsState* s, void** uc, void** mc) {
  const Drv& d = drv();
  if (!s->added) return fail(LASGD_ERR_STATE, "add the device to the multicast object first");
  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = s->device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;  // the multicast object's handle type
  CU_TRY(d.MemCreate(&s->mem, s->bytes, &ap, 0));
  s->have_mem = true;
  CU_TRY(d.MulticastBindMem(s->mc, 0, s->mem, 0, s->bytes, 0));
  s->bound = true;
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = s->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU_TRY(d.MemAddressReserve(&s->uc, s->bytes, s->gran, 0, 0));
  CU_TRY(d.MemMap(s->uc, s->bytes, 0, s->mem, 0));
  CU_TRY(d.MemSetAccess(s->uc, s->bytes, &acc, 1));
  CU_TRY(d.MemAddressReserve(&s->mcva, s->bytes, s->gran, 0, 0));
  CU_TRY(d.MemMap(s->mcva, s->bytes, 0, s->mc, 0));
  CU_TRY(d.MemSetAccess(s->mcva, s->bytes, &acc, 1));
  LASGD_CUDA_TRY(cudaMemset(reinterpret_cast<void*>(s->uc), 0, s->bytes));
  *uc = reinterpret_cast<void*>(s->uc);
  *mc = reinterpret_cast<void*>(s->mcva);
  return LASGD_OK;
}

void nvls_destroy(NvlsState* s) {
  if (!s) return;
  const Drv& d = drv();
  if (d.ok) {
    if (s->mcva) {
      d.MemUnmap(s->mcva, s->bytes);
      d.MemAddressFree(s->mcva, s->bytes);
    }
    if (s->uc) {
      d.MemUnmap(s->uc, s->bytes);
      d.MemAddressFree(s->uc, s->bytes);
    }
    if (s->bound) {
      CUdevice dev;
      if (d.DeviceGet(&dev, s->device) == CUDA_SUCCESS) d.MulticastUnbind(s->mc, dev, 0, s->bytes);
    }
    if (s->have_mem) d.MemRelease(s->mem);
    if (s->have_mc) d.MemRelease(s->mc);
  }
  delete s;
}

// ------------------------------------------------------------------ the in-switch mean
__device__ __forceinline__ float4 mm_ld_reduce_v4(const float* p) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ float mm_ld_reduce(const float* p) {
  float v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mm_st_v4(float* p, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mm_st(float* p, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

template <int P>
__device__ __forceinline__ float nvls_scale(float s) {
  return mean_div<float, P>(s);
}

// CTA b of every rank reduces slice b of its own chunk.  Entry: the per-CTA barrier (every
// rank's snapshot slot final; every peer done reading our mean buffer of the previous
// launch).  Exit: every CTA fences its multicast stores and counts itself out; the last
// CTA signals every peer and waits for all of them, so the launch completes only when the
// whole mean has landed in this rank's buffer (the next pull is stream-ordered after it).
template <int P>
__global__ void __launch_bounds__(256, 2) k_nvls_mean(CommArgs a, const float* mc_src, float* mc_dst) {
  pdl_entry();
  const int rank = a.rank, b = blockIdx.x;
  trace_mark(a, b, 0);
  bool ok = cta_barrier<P>(a, 0, b, rank);
  trace_mark(a, b, 1);
  unsigned bad = 0;
  if (ok) {
    const size_t n = a.n;
    size_t cs, ce, cp0, cp1;
    chunk_packs<float, P>(n, rank, cs, ce, cp0, cp1);
    size_t p0, p1;
    split(cp1 - cp0, a.nblocks, b, p0, p1);
    constexpr int U = 4;
    for (size_t p = cp0 + p0 + threadIdx.x; p < cp0 + p1; p += (size_t)U * blockDim.x) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t pu = p + (size_t)u * blockDim.x;
        if (pu < cp0 + p1) v[u] = mm_ld_reduce_v4(mc_src + 4 * pu);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t pu = p + (size_t)u * blockDim.x;
        if (pu < cp0 + p1) {
          float4 m = make_float4(nvls_scale<P>(v[u].x), nvls_scale<P>(v[u].y), nvls_scale<P>(v[u].z),
                                 nvls_scale<P>(v[u].w));
          bad += !finite(m.x) + !finite(m.y) + !finite(m.z) + !finite(m.w);
          mm_st_v4(mc_dst + 4 * pu, m);
        }
      }
    }
    if (b == 0) {  // unaligned head / tail of the chunk
      const size_t he = cp0 * 4 < ce ? cp0 * 4 : ce;
      const size_t ts = cp1 * 4 > he ? cp1 * 4 : he;
      for (size_t j = cs + threadIdx.x; j < he; j += blockDim.x) {
        const float m = nvls_scale<P>(mm_ld_reduce(mc_src + j));
        bad += !finite(m);
        mm_st(mc_dst + j, m);
      }
      for (size_t j = ts + threadIdx.x; j < ce; j += blockDim.x) {
        const float m = nvls_scale<P>(mm_ld_reduce(mc_src + j));
        bad += !finite(m);
        mm_st(mc_dst + j, m);
      }
    }
  }
  report_nonfinite(a.nonfinite, bad);
  // the multicast stores went through another virtual alias of the same memory
  asm volatile("fence.proxy.alias;" ::: "memory");
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    unsigned* ctr = cend(a);
    const unsigned prev = atomicAdd(ctr, 1u);
    s_last = prev == (unsigned)a.nblocks - 1u;
    if (s_last) *ctr = 0u;
  }
  __syncthreads();
  if (s_last && ok) {
    const size_t slot = (size_t)2 * kMaxB * kMaxR + (size_t)1 * kMaxR;
    if (threadIdx.x < P) {
      __threadfence_system();
      st_release_sys(a.pad[threadIdx.x] + slot + rank, cepoch(a));
    }
    rank_wait<P>(a, 1, cepoch(a), b, rank);
  }
  trace_mark(a, b, 3);
  publish_done(a);
}

int launch_nvls_mean(int P, const CommArgs& a, const void* mc_src, void* mc_dst, int nblocks, cudaStream_t s) {
  const float* src = reinterpret_cast<const float*>(mc_src);
  float* dst = reinterpret_cast<float*>(mc_dst);
  switch (P) {
#define LASGD_NCASE(PP) \
  case PP: return launch_kernel(false, k_nvls_mean<PP>, dim3(nblocks), 256, s, a, src, dst);
    LASGD_NCASE(2)
    LASGD_NCASE(3)
    LASGD_NCASE(4)
    LASGD_NCASE(5)
    LASGD_NCASE(6)
    LASGD_NCASE(7)
    LASGD_NCASE(8)
#undef LASGD_NCASE
    default: return fail(LASGD_ERR_UNSUPPORTED, "NVLS mean needs 2 <= P <= %d, got %d", kMaxR, P);
  }
}

}  // namespace lasgd
