// Peer-to-peer per-layer aggregation kernels (p2p.cu). Internal to the engine.
#pragma once
#include <cuda_runtime.h>

namespace spb {

constexpr int kMaxPeers = 8;

template <class T>
struct PeerPtrs {
  T* p[kMaxPeers];
};

// Epoch-stamped flags: flags[slot * nranks + src]; step `sub` of a graph
// signals / waits for epoch + sub + 1; the epoch then advances by `add`.
void launch_p2p_signal(const PeerPtrs<int>& flags, int slot, int nranks, int rank, const int* epoch, int sub,
                       cudaStream_t s);
void launch_p2p_wait(const int* flags, int slot, int nranks, unsigned mask, const int* epoch, int sub, cudaStream_t s);
void launch_p2p_epoch(int* epoch, int add, cudaStream_t s);
// Sum of nsrc gradient shards -> optimizer -> hi, lo, mom, w32 (n floats).
void launch_p2p_update(const PeerPtrs<const float>& src, int nsrc, float* hi, float* lo, float* mom, float* w32, long n,
                       float lr, float mu, float wd, cudaStream_t s);
// (hi, lo) = split(w32) on [0, n) except [hole0, hole1).
void launch_p2p_split(const float* w32, float* hi, float* lo, long n, long hole0, long hole1, cudaStream_t s);

// dst += src (n floats, n % 4 == 0): a reduce round of the rh mode.
void launch_rh_add(float* dst, const float* src, long n, cudaStream_t s);
// "push" mode (push.cu): see the file comment for the protocol.
void launch_push_signal(const PeerPtrs<int>& flags, int slot, int nranks, int rank, const int* epoch, int sub,
                        const float* gw, long ldw, const float* gb, int rpo, int n_rows, const PeerPtrs<float>& wdst,
                        const PeerPtrs<float>& bdst, cudaStream_t s);
void launch_push_update(const PeerPtrs<const float>& src, int nsrc, float* hi, float* lo, float* mom,
                        const PeerPtrs<float>& dst, int ndst, long n, float lr, float mu, float wd, cudaStream_t s);
void launch_push_split(const float* w32, float* hi, float* lo, long n, long hole0, long hole1, cudaStream_t s);

}  // namespace spb
