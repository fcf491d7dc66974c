// Peer-to-peer per-layer aggregation kernels (p2p.cu). Internal to the engine.
#pragma once
#include <cuda_runtime.h>

namespace spb {

constexpr int kMaxPeers = 8;

template <class T>
struct PeerPtrs {
  T* p[kMaxPeers];
};

// Epoch-stamped flags: flags[slot * nranks + src].
void launch_p2p_signal(const PeerPtrs<int>& flags, int slot, int nranks, int rank, const int* epoch, cudaStream_t s);
void launch_p2p_wait(const int* flags, int slot, int nranks, unsigned mask, const int* epoch, cudaStream_t s);
void launch_p2p_epoch(int* epoch, cudaStream_t s);
// Sum of nsrc gradient shards -> optimizer -> hi, lo, mom, w32 (n floats).
void launch_p2p_update(const PeerPtrs<const float>& src, int nsrc, float* hi, float* lo, float* mom, float* w32, long n,
                       float lr, float mu, float wd, cudaStream_t s);
// (hi, lo) = split(w32) on [0, n) except [hole0, hole1).
void launch_p2p_split(const float* w32, float* hi, float* lo, long n, long hole0, long hole1, cudaStream_t s);

}  // namespace spb
