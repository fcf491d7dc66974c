// NVLink SHARP (NVLS) multicast memory for the multi-GPU SPB step.
//
// A multicast buffer is one physical allocation per GPU, all bound to one
// CUDA multicast object: each rank sees its own copy through a unicast VA and
// every copy at once through a multicast VA. On that VA
//   multimem.ld_reduce.add  returns the element-wise sum over all ranks'
//                           copies, reduced inside the NVSwitch, and
//   multimem.st             writes to every rank's copy in one store,
// which is what the fused "reduce my gradient shard -> optimizer -> broadcast
// my weight shard" kernel (fused_reduce_update_kernel) is built on.
//
// Setup is collective over the ranks of one node: rank 0 creates the
// multicast object and hands its POSIX file descriptor to the other rank
// processes over an abstract Unix socket (SCM_RIGHTS); everyone adds its
// device, binds its own physical memory and maps both VAs. Barriers between
// the steps are passed in by the caller (the engine uses its NCCL comm).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <chrono>
#include <cstring>
#include <functional>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>

#include "launch.hpp"
#include "nvls.hpp"

namespace spb {
namespace {

struct Drv {
  PFN_cuMulticastCreate_v12010 MulticastCreate;
  PFN_cuMulticastAddDevice_v12010 MulticastAddDevice;
  PFN_cuMulticastBindMem_v12010 MulticastBindMem;
  PFN_cuMulticastUnbind_v12010 MulticastUnbind;
  PFN_cuMulticastGetGranularity_v12010 MulticastGetGranularity;
  PFN_cuMemCreate_v10020 MemCreate;
  PFN_cuMemRelease_v10020 MemRelease;
  PFN_cuMemMap_v10020 MemMap;
  PFN_cuMemUnmap_v10020 MemUnmap;
  PFN_cuMemAddressReserve_v10020 MemAddressReserve;
  PFN_cuMemAddressFree_v10020 MemAddressFree;
  PFN_cuMemSetAccess_v10020 MemSetAccess;
  PFN_cuMemExportToShareableHandle_v10020 MemExportToShareableHandle;
  PFN_cuMemImportFromShareableHandle_v10020 MemImportFromShareableHandle;
  PFN_cuMemGetAllocationGranularity_v10020 MemGetAllocationGranularity;
  PFN_cuDeviceGet_v2000 DeviceGet;
  PFN_cuDeviceGetAttribute_v2000 DeviceGetAttribute;
};

const Drv& drv() {
  static Drv d{};
  static std::string fail;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [&](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess || !*fn)
        if (fail.empty()) fail = std::string("nvls: driver entry point missing: ") + name;
    };
    get("cuMulticastCreate", reinterpret_cast<void**>(&d.MulticastCreate));
    get("cuMulticastAddDevice", reinterpret_cast<void**>(&d.MulticastAddDevice));
    get("cuMulticastBindMem", reinterpret_cast<void**>(&d.MulticastBindMem));
    get("cuMulticastUnbind", reinterpret_cast<void**>(&d.MulticastUnbind));
    get("cuMulticastGetGranularity", reinterpret_cast<void**>(&d.MulticastGetGranularity));
    get("cuMemCreate", reinterpret_cast<void**>(&d.MemCreate));
    get("cuMemRelease", reinterpret_cast<void**>(&d.MemRelease));
    get("cuMemMap", reinterpret_cast<void**>(&d.MemMap));
    get("cuMemUnmap", reinterpret_cast<void**>(&d.MemUnmap));
    get("cuMemAddressReserve", reinterpret_cast<void**>(&d.MemAddressReserve));
    get("cuMemAddressFree", reinterpret_cast<void**>(&d.MemAddressFree));
    get("cuMemSetAccess", reinterpret_cast<void**>(&d.MemSetAccess));
    get("cuMemExportToShareableHandle", reinterpret_cast<void**>(&d.MemExportToShareableHandle));
    get("cuMemImportFromShareableHandle", reinterpret_cast<void**>(&d.MemImportFromShareableHandle));
    get("cuMemGetAllocationGranularity", reinterpret_cast<void**>(&d.MemGetAllocationGranularity));
    get("cuDeviceGet", reinterpret_cast<void**>(&d.DeviceGet));
    get("cuDeviceGetAttribute", reinterpret_cast<void**>(&d.DeviceGetAttribute));
  });
  if (!fail.empty()) throw std::runtime_error(fail);
  return d;
}

void cu_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw std::runtime_error(std::string("nvls: ") + what + " failed (" + std::to_string(r) + ")");
}

// ---- FD passing over an abstract Unix socket ------------------------------
sockaddr_un sock_addr(const std::string& name, socklen_t* len) {
  sockaddr_un a{};
  a.sun_family = AF_UNIX;
  a.sun_path[0] = '\0';  // abstract namespace: nothing on the filesystem
  const size_t n = std::min(name.size(), sizeof(a.sun_path) - 2);
  std::memcpy(a.sun_path + 1, name.data(), n);
  *len = static_cast<socklen_t>(offsetof(sockaddr_un, sun_path) + 1 + n);
  return a;
}

void send_fd(int sock, int fd) {
  char byte = 1;
  iovec iov{&byte, 1};
  char ctrl[CMSG_SPACE(sizeof(int))] = {};
  msghdr m{};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = ctrl;
  m.msg_controllen = sizeof ctrl;
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  c->cmsg_level = SOL_SOCKET;
  c->cmsg_type = SCM_RIGHTS;
  c->cmsg_len = CMSG_LEN(sizeof(int));
  std::memcpy(CMSG_DATA(c), &fd, sizeof(int));
  if (sendmsg(sock, &m, 0) != 1) throw std::runtime_error("nvls: sendmsg failed");
}

int recv_fd(int sock) {
  char byte = 0;
  iovec iov{&byte, 1};
  char ctrl[CMSG_SPACE(sizeof(int))] = {};
  msghdr m{};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = ctrl;
  m.msg_controllen = sizeof ctrl;
  if (recvmsg(sock, &m, 0) != 1) throw std::runtime_error("nvls: recvmsg failed");
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  if (!c || c->cmsg_type != SCM_RIGHTS) throw std::runtime_error("nvls: no fd received");
  int fd;
  std::memcpy(&fd, CMSG_DATA(c), sizeof(int));
  return fd;
}

// Rank 0 serves `fd` to nranks-1 peers; others receive it.
int share_fd(const std::string& name, int rank, int nranks, int fd) {
  socklen_t len;
  sockaddr_un a = sock_addr(name, &len);
  if (rank == 0) {
    int s = socket(AF_UNIX, SOCK_STREAM, 0);
    if (s < 0 || bind(s, reinterpret_cast<sockaddr*>(&a), len) != 0 || listen(s, nranks) != 0) {
      if (s >= 0) close(s);
      throw std::runtime_error("nvls: cannot listen on " + name);
    }
    for (int i = 1; i < nranks; ++i) {
      int c = accept(s, nullptr, nullptr);
      if (c < 0) {
        close(s);
        throw std::runtime_error("nvls: accept failed");
      }
      send_fd(c, fd);
      close(c);
    }
    close(s);
    return fd;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    int s = socket(AF_UNIX, SOCK_STREAM, 0);
    if (s >= 0 && connect(s, reinterpret_cast<sockaddr*>(&a), len) == 0) {
      int got = recv_fd(s);
      close(s);
      return got;
    }
    if (s >= 0) close(s);
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60))
      throw std::runtime_error("nvls: timed out connecting to " + name);
    std::this_thread::sleep_for(std::chrono::milliseconds(2));
  }
}

}  // namespace

bool nvls_supported(int device) {
  try {
    const Drv& d = drv();
    CUdevice cudev;
    int v = 0;
    if (d.DeviceGet(&cudev, device) != CUDA_SUCCESS) return false;
    if (d.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cudev) != CUDA_SUCCESS) return false;
    return v != 0;
  } catch (const std::exception&) {
    return false;
  }
}

McBuffer nvls_alloc(size_t bytes, int device, int rank, int nranks, const std::string& name,
                    const std::function<void()>& barrier) {
  const Drv& d = drv();
  CUdevice cudev;
  cu_check(d.DeviceGet(&cudev, device), "cuDeviceGet");
  CUmulticastObjectProp mp{};
  mp.numDevices = static_cast<unsigned>(nranks);
  mp.size = bytes;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g_mc = 0, g_mem = 0;
  cu_check(d.MulticastGetGranularity(&g_mc, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = device;
  // The physical memory must carry the multicast object's handle type
  // (cuMulticastBindMem rejects it otherwise).
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  ap.allocFlags.gpuDirectRDMACapable = 1;
  cu_check(d.MemGetAllocationGranularity(&g_mem, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED),
           "cuMemGetAllocationGranularity");
  const size_t gran = std::max(g_mc, g_mem);
  McBuffer b;
  b.size = (bytes + gran - 1) / gran * gran;
  mp.size = b.size;
  int fd = -1;
  if (rank == 0) {
    cu_check(d.MulticastCreate(&b.mc, &mp), "cuMulticastCreate");
    cu_check(d.MemExportToShareableHandle(&fd, b.mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
             "cuMemExportToShareableHandle");
  }
  fd = share_fd(name, rank, nranks, fd);
  if (rank != 0) {
    cu_check(d.MemImportFromShareableHandle(&b.mc, reinterpret_cast<void*>(static_cast<intptr_t>(fd)),
                                            CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
             "cuMemImportFromShareableHandle");
  }
  close(fd);
  cu_check(d.MulticastAddDevice(b.mc, cudev), "cuMulticastAddDevice");
  barrier();  // every device joined before anyone binds
  cu_check(d.MemCreate(&b.mem, b.size, &ap, 0), "cuMemCreate");
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  cu_check(d.MemAddressReserve(&b.mcva, b.size, gran, 0, 0), "cuMemAddressReserve");
  cu_check(d.MemMap(b.mcva, b.size, 0, b.mc, 0), "cuMemMap(mc)");
  cu_check(d.MemSetAccess(b.mcva, b.size, &acc, 1), "cuMemSetAccess(mc)");
  cu_check(d.MulticastBindMem(b.mc, 0, b.mem, 0, b.size, 0), "cuMulticastBindMem");
  cu_check(d.MemAddressReserve(&b.uc, b.size, gran, 0, 0), "cuMemAddressReserve");
  cu_check(d.MemMap(b.uc, b.size, 0, b.mem, 0), "cuMemMap(uc)");
  cu_check(d.MemSetAccess(b.uc, b.size, &acc, 1), "cuMemSetAccess(uc)");
  barrier();
  b.device = cudev;
  SPB_CUDA(cudaMemset(reinterpret_cast<void*>(b.uc), 0, b.size));
  SPB_CUDA(cudaDeviceSynchronize());  // the zeroing (legacy stream) before any use on other streams
  barrier();
  return b;
}

void nvls_free(McBuffer& b) {
  if (!b.mc) return;
  const Drv& d = drv();
  if (b.mcva) d.MemUnmap(b.mcva, b.size), d.MemAddressFree(b.mcva, b.size);
  if (b.uc) d.MemUnmap(b.uc, b.size), d.MemAddressFree(b.uc, b.size);
  d.MulticastUnbind(b.mc, b.device, 0, b.size);
  if (b.mem) d.MemRelease(b.mem);
  d.MemRelease(b.mc);
  b = McBuffer{};
}

// ---- device side ----------------------------------------------------------

namespace {

__device__ __forceinline__ void spin_until_ge(const int* flag, int target) {
  int v = 0;
  uint64_t t0 = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v >= target) return;
    if ((spin & 0x3FFu) == 0x3FFu) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      else if (t - t0 > 30000000000ull) __trap();  // a missing rank must fail, not hang the GPU
    }
  }
}

// Cross-rank barrier on slot `slot`: every rank adds 1 to the slot in every
// rank's copy, then waits until its own copy reaches nranks * (epoch + 1).
__global__ void nvls_barrier_kernel(int* flags_mc, const int* flags_uc, int slot, int nranks, const int* epoch) {
  __threadfence_system();
  asm volatile("multimem.red.release.sys.global.add.s32 [%0], 1;" ::"l"(flags_mc + slot) : "memory");
  spin_until_ge(flags_uc + slot, nranks * (*epoch + 1));
}

__global__ void nvls_epoch_kernel(int* epoch) { *epoch += 1; }

// Fused aggregate + optimizer + broadcast for one shard of one layer:
//   g   = sum over ranks of grad (multimem.ld_reduce in the switch)
//   w   = hi + lo (this rank's copy; all copies are identical)
//   g' = g + wd*w; buf = mu*buf + g'; w -= lr*buf   (buf local to the owner)
//   hi, lo = split(w) -> multimem.st to every rank's copy
// U independent 16-byte switch reductions in flight per thread: the
// round trip through the switch is long, so bandwidth needs many of them.
template <int U>
__global__ void __launch_bounds__(256) fused_reduce_update_kernel(const float* __restrict__ grad_mc,
                                                                  const float* __restrict__ hi_uc,
                                                                  const float* __restrict__ lo_uc, float* hi_mc,
                                                                  float* lo_mc, float* __restrict__ mom, long n4,
                                                                  float lr, float mu, float wd) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i0 = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n4; i0 += stride * U) {
    float g[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long i = i0 + u * stride;
      if (i < n4)
        asm volatile("multimem.ld_reduce.weak.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(g[u][0]), "=f"(g[u][1]), "=f"(g[u][2]), "=f"(g[u][3])
                     : "l"(grad_mc + 4 * i)
                     : "memory");
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long i = i0 + u * stride;
      if (i >= n4) break;
      const float4 h = reinterpret_cast<const float4*>(hi_uc)[i];
      const float4 l = reinterpret_cast<const float4*>(lo_uc)[i];
      float w[4] = {h.x + l.x, h.y + l.y, h.z + l.z, h.w + l.w};
      float b[4] = {0.f, 0.f, 0.f, 0.f};
      if (mom) {
        const float4 m = reinterpret_cast<const float4*>(mom)[i];
        b[0] = m.x, b[1] = m.y, b[2] = m.z, b[3] = m.w;
      }
      float nh[4], nl[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float gg = fmaf(wd, w[j], g[u][j]);
        if (mom) {
          b[j] = fmaf(mu, b[j], gg);
          gg = b[j];
        }
        const float wn = w[j] - lr * gg;
        uint32_t r;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(wn));
        nh[j] = __uint_as_float(r);
        nl[j] = wn - nh[j];
      }
      asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(hi_mc + 4 * i), "f"(nh[0]),
                   "f"(nh[1]), "f"(nh[2]), "f"(nh[3])
                   : "memory");
      asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(lo_mc + 4 * i), "f"(nl[0]),
                   "f"(nl[1]), "f"(nl[2]), "f"(nl[3])
                   : "memory");
      if (mom) reinterpret_cast<float4*>(mom)[i] = make_float4(b[0], b[1], b[2], b[3]);
    }
  }
  __threadfence_system();
}

// Microbenchmark pieces: switch reduce only / multicast store only.
template <int U>
__global__ void __launch_bounds__(256) ldreduce_only_kernel(const float* grad_mc, float* out, long n4) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i0 = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n4; i0 += stride * U) {
    float g[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long i = i0 + u * stride;
      if (i < n4)
        asm volatile("multimem.ld_reduce.weak.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(g[u][0]), "=f"(g[u][1]), "=f"(g[u][2]), "=f"(g[u][3])
                     : "l"(grad_mc + 4 * i)
                     : "memory");
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long i = i0 + u * stride;
      if (i < n4) reinterpret_cast<float4*>(out)[i] = make_float4(g[u][0], g[u][1], g[u][2], g[u][3]);
    }
  }
}

__global__ void __launch_bounds__(256) mcstore_only_kernel(const float* in, float* out_mc, long n4) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = reinterpret_cast<const float4*>(in)[i];
    asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(out_mc + 4 * i), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
  }
  __threadfence_system();
}

int g_fused_unroll = 4, g_fused_blocks_per_sm = 4;

// Self-test: out[i] = sum over ranks of (rank + 1) * (i + 1) via ld_reduce,
// then multimem.st of the sum into every copy of `bcast`.
__global__ void selftest_kernel(const float* in_mc, float* bcast_mc, long n) {
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += static_cast<long>(gridDim.x) *
                                                                                          blockDim.x) {
    float v;
    asm volatile("multimem.ld_reduce.weak.global.add.f32 %0, [%1];" : "=f"(v) : "l"(in_mc + i) : "memory");
    asm volatile("multimem.st.weak.global.f32 [%0], %1;" ::"l"(bcast_mc + i), "f"(v) : "memory");
  }
  __threadfence_system();
}

__global__ void fill_kernel(float* p, long n, float scale) {
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += static_cast<long>(gridDim.x) *
                                                                                          blockDim.x)
    p[i] = scale * static_cast<float>(i % 1024 + 1);
}

}  // namespace

void launch_nvls_barrier(int* flags_mc, const int* flags_uc, int slot, int nranks, const int* epoch, cudaStream_t s) {
  nvls_barrier_kernel<<<1, 1, 0, s>>>(flags_mc, flags_uc, slot, nranks, epoch);
  SPB_CUDA(cudaGetLastError());
}

void launch_nvls_epoch(int* epoch, cudaStream_t s) {
  nvls_epoch_kernel<<<1, 1, 0, s>>>(epoch);
  SPB_CUDA(cudaGetLastError());
}

void launch_fused_reduce_update(const float* grad_mc, const float* hi_uc, const float* lo_uc, float* hi_mc, float* lo_mc,
                                float* mom, long n, float lr, float mu, float wd, cudaStream_t s) {
  if (n <= 0) return;
  if (n % 4) throw std::invalid_argument("nvls: shard must be a multiple of 4 floats");
  const long n4 = n / 4;
  const int U = g_fused_unroll;
  const int grid = static_cast<int>(std::max<long>(1, std::min<long>((n4 + 256L * U - 1) / (256L * U),
                                                                     148L * g_fused_blocks_per_sm)));
  switch (U) {
    case 1: fused_reduce_update_kernel<1><<<grid, 256, 0, s>>>(grad_mc, hi_uc, lo_uc, hi_mc, lo_mc, mom, n4, lr, mu, wd); break;
    case 2: fused_reduce_update_kernel<2><<<grid, 256, 0, s>>>(grad_mc, hi_uc, lo_uc, hi_mc, lo_mc, mom, n4, lr, mu, wd); break;
    case 8: fused_reduce_update_kernel<8><<<grid, 256, 0, s>>>(grad_mc, hi_uc, lo_uc, hi_mc, lo_mc, mom, n4, lr, mu, wd); break;
    default: fused_reduce_update_kernel<4><<<grid, 256, 0, s>>>(grad_mc, hi_uc, lo_uc, hi_mc, lo_mc, mom, n4, lr, mu, wd);
  }
  SPB_CUDA(cudaGetLastError());
}

void nvls_set_launch(int unroll, int blocks_per_sm) {
  if (unroll > 0) g_fused_unroll = unroll;
  if (blocks_per_sm > 0) g_fused_blocks_per_sm = blocks_per_sm;
}

// Standalone timings (rank 0 prints): switch reduce only, multicast store
// only, and the fused kernel over (unroll, blocks/SM) on this rank's shard of
// an n-float layer, all ranks running concurrently.
void nvls_bench(int device, int rank, int nranks, const std::string& name, const std::function<void()>& barrier, long n,
                int reps) {
  n = (n + 4L * nranks - 1) / (4L * nranks) * (4L * nranks);
  McBuffer g = nvls_alloc(n * 4, device, rank, nranks, name + "-g", barrier);
  McBuffer h = nvls_alloc(n * 4, device, rank, nranks, name + "-h", barrier);
  McBuffer l = nvls_alloc(n * 4, device, rank, nranks, name + "-l", barrier);
  float* mom = nullptr;
  float* loc = nullptr;
  SPB_CUDA(cudaMalloc(&mom, n * 4));
  SPB_CUDA(cudaMalloc(&loc, n * 4));
  SPB_CUDA(cudaMemset(mom, 0, n * 4));
  SPB_CUDA(cudaMemset(loc, 0, n * 4));
  cudaStream_t st;
  SPB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  SPB_CUDA(cudaEventCreate(&e0));
  SPB_CUDA(cudaEventCreate(&e1));
  const long shard = n / nranks, a = shard * rank;
  const long n4 = shard / 4;
  auto mc = [&](const McBuffer& b) { return reinterpret_cast<float*>(b.mcva) + a; };
  auto uc = [&](const McBuffer& b) { return reinterpret_cast<float*>(b.uc) + a; };
  auto timeit = [&](const char* what, const std::function<void()>& body, double bytes) {
    body();
    SPB_CUDA(cudaStreamSynchronize(st));
    barrier();
    SPB_CUDA(cudaEventRecord(e0, st));
    for (int r = 0; r < reps; ++r) body();
    SPB_CUDA(cudaEventRecord(e1, st));
    SPB_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    SPB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    barrier();
    const double us = 1e3 * ms / reps;
    if (rank == 0)
      std::printf("nvls_bench N=%d n=%ld %-28s %9.1f us  %8.1f GB/s (shard bytes/us)\n", nranks, n, what, us,
                  bytes / (us * 1e3));
    std::fflush(stdout);
  };
  const double sb = static_cast<double>(shard) * 4.0;
  for (int bps : {1, 2, 4, 8}) {
    const int grid1 = static_cast<int>(std::min<long>((n4 + 1023) / 1024, 148L * bps));
    char tag[64];
    std::snprintf(tag, sizeof tag, "ldreduce U4 b%d", bps);
    timeit(tag, [&] { ldreduce_only_kernel<4><<<grid1, 256, 0, st>>>(mc(g), loc, n4); }, sb);
    std::snprintf(tag, sizeof tag, "mcstore b%d", bps);
    const int grid2 = static_cast<int>(std::min<long>((n4 + 255) / 256, 148L * bps));
    timeit(tag, [&] { mcstore_only_kernel<<<grid2, 256, 0, st>>>(loc, mc(h), n4); }, sb);
  }
  for (int U : {1, 2, 4, 8})
    for (int bps : {1, 2, 4, 8}) {
      nvls_set_launch(U, bps);
      char tag[64];
      std::snprintf(tag, sizeof tag, "fused U%d b%d", U, bps);
      timeit(tag, [&] { launch_fused_reduce_update(mc(g), uc(h), uc(l), mc(h), mc(l), mom + a, shard, 1e-3f, 0.9f, 0.f, st); },
             sb);
    }
  nvls_set_launch(4, 4);
  SPB_CUDA(cudaStreamDestroy(st));
  cudaEventDestroy(e0), cudaEventDestroy(e1);
  cudaFree(mom), cudaFree(loc);
  barrier();
  nvls_free(g), nvls_free(h), nvls_free(l);
}

// Returns the number of mismatching elements (0 = multicast reduce + store work).
long nvls_selftest(int device, int rank, int nranks, const std::string& name, const std::function<void()>& barrier) {
  const long n = 1 << 20;
  McBuffer in = nvls_alloc(n * 4, device, rank, nranks, name + "-a", barrier);
  McBuffer out = nvls_alloc(n * 4, device, rank, nranks, name + "-b", barrier);
  fill_kernel<<<256, 256>>>(reinterpret_cast<float*>(in.uc), n, static_cast<float>(rank + 1));
  SPB_CUDA(cudaDeviceSynchronize());
  barrier();
  // Each rank reduces and broadcasts its own quarter (disjoint slices).
  const long part = n / nranks;
  selftest_kernel<<<256, 256>>>(reinterpret_cast<const float*>(in.mcva) + rank * part,
                                reinterpret_cast<float*>(out.mcva) + rank * part, part);
  SPB_CUDA(cudaDeviceSynchronize());
  barrier();
  std::vector<float> h(n);
  SPB_CUDA(cudaMemcpy(h.data(), reinterpret_cast<void*>(out.uc), n * 4, cudaMemcpyDeviceToHost));
  const float tri = static_cast<float>(nranks * (nranks + 1) / 2);
  long bad = 0;
  for (long i = 0; i < part * nranks; ++i)
    if (h[i] != tri * static_cast<float>(i % 1024 + 1)) ++bad;
  barrier();
  nvls_free(in);
  nvls_free(out);
  return bad;
}

}  // namespace spb
