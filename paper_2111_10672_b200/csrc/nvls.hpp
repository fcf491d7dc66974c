// NVLS multicast buffers and the fused reduce->update->broadcast kernel
// (nvls.cu). Internal to the engine.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <functional>
#include <string>
#include <vector>

namespace spb {

struct McBuffer {
  size_t size = 0;
  CUmemGenericAllocationHandle mc = 0, mem = 0;
  CUdeviceptr uc = 0, mcva = 0;  // this rank's copy / all copies
  CUdevice device = 0;
};

bool nvls_supported(int device);
// Collective over the ranks of one node (all call it in the same order with
// the same name). `barrier` must synchronise all ranks (host side).
McBuffer nvls_alloc(size_t bytes, int device, int rank, int nranks, const std::string& name,
                    const std::function<void()>& barrier);
void nvls_free(McBuffer& b);

void launch_nvls_barrier(int* flags_mc, const int* flags_uc, int slot, int nranks, const int* epoch, cudaStream_t s);
void launch_nvls_epoch(int* epoch, cudaStream_t s);
// n floats of one rank's shard: reduce the gradient over ranks (in the
// switch), apply the optimizer, broadcast hi / lo to every rank.
void launch_fused_reduce_update(const float* grad_mc, const float* hi_uc, const float* lo_uc, float* hi_mc, float* lo_mc,
                                float* mom, long n, float lr, float mu, float wd, cudaStream_t s);
void nvls_set_launch(int unroll, int blocks_per_sm);
void nvls_bench(int device, int rank, int nranks, const std::string& name, const std::function<void()>& barrier, long n,
                int reps);
long nvls_selftest(int device, int rank, int nranks, const std::string& name, const std::function<void()>& barrier);

}  // namespace spb
