// SPB bookkeeping on the host: integer-exact restatements of the reference's
// suffix rule, chunk layout and contributor sets, the counter-based Rng, and
// the multi-GPU worker placement. Everything here is pure integer work.
#pragma once
#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace spb {

// The reference's error taxonomy (include/jigsaw/errors.hpp:9-25), mapped to
// spb_status codes at the C ABI.
struct ArgumentError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct ProtocolError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Counter-based splittable generator, bit-identical to include/jigsaw/rng.hpp.
class Rng {
 public:
  explicit Rng(uint64_t key) : key_(key) {}
  Rng split(uint64_t tag) const { return Rng(mix(key_, tag)); }  // rng.hpp:18
  uint64_t next_u64() { return mix(key_, ++counter_); }           // rng.hpp:20
  uint64_t next_below(uint64_t n) {                               // rng.hpp:26-29
    return static_cast<uint64_t>((static_cast<unsigned __int128>(next_u64()) * n) >> 64);
  }
  static uint64_t mix(uint64_t a, uint64_t b) {  // rng.hpp:47-53
    uint64_t z = a ^ (b + 0x9E3779B97F4A7C15ULL + (a << 6) + (a >> 2));
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }

 private:
  uint64_t key_;
  uint64_t counter_ = 0;
};

// suffix_layers spb.cpp:16-21: ceil(j*L/k) in 64-bit integers.
inline int suffix_layers(int j, int k, int L) {
  if (k < 1 || L < 1) throw ArgumentError("suffix_layers: k and L must be >= 1");
  if (j < 1 || j > k) throw ArgumentError("suffix_layers: worker index out of range");
  return static_cast<int>((static_cast<long long>(j) * L + k - 1) / k);
}

// chunk_coverage spb.cpp:23-29: chunk m is computed by workers {k-m+1..k}.
inline std::vector<int> chunk_coverage(int m, int k) {
  if (k < 1) throw ArgumentError("chunk_coverage: k must be >= 1");
  if (m < 1 || m > k) throw ArgumentError("chunk_coverage: chunk index out of range");
  std::vector<int> w(m);
  std::iota(w.begin(), w.end(), k - m + 1);
  return w;
}

// chunk_layout spb.cpp:31-41: chunk m spans [L - s(k-m+1) + 1, L - s(k-m)],
// the last chunk ending at L; empty chunks have first > last.
inline std::vector<std::pair<int, int>> chunk_layout(int k, int L) {
  if (k < 1 || L < 1) throw ArgumentError("chunk_layout: k and L must be >= 1");
  std::vector<std::pair<int, int>> spans(k);
  for (int m = 1; m <= k; ++m) {
    const int first = L - suffix_layers(k - m + 1, k, L) + 1;
    const int last = (m == k) ? L : L - suffix_layers(k - m, k, L);
    spans[m - 1] = {first, last};
  }
  return spans;
}

// layer_chunks spb.cpp:43-49: chunk (= contributor count) of each layer.
inline std::vector<int> layer_chunks(int k, int L) {
  auto spans = chunk_layout(k, L);
  std::vector<int> chunk_of(L, 0);
  for (int m = 1; m <= k; ++m)
    for (int l = spans[m - 1].first; l <= spans[m - 1].second; ++l) chunk_of[l - 1] = m;
  return chunk_of;
}

// First covered layer of worker j (1-based): L - ceil(jL/k) + 1.
inline int worker_stop(int j, int k, int L) { return L - suffix_layers(j, k, L) + 1; }

// Workers (1-based, ascending) hosted by `rank` of `nranks`. Worker j's
// backward costs ~ s_j layers, so pairs (j, k+1-j) carry equal work; pairs are
// dealt out snake-wise. Falls back to a count-balanced greedy (largest
// suffix first to the least-loaded rank) when the pairing does not divide.
// Contiguous placement instead deals out consecutive workers (rank r gets
// workers r*k/N+1 .. (r+1)*k/N): backward work is then unbalanced, but the
// ranks hosting only low workers contribute to few layers, so the exchange
// moves fewer gradient bytes -- the saving SPB promises on the network. It is
// the default from 4 ranks on (measured, cfg3 at 4 B200s: push 232.3 k vs
// 224.7 k samples/s, rh 208.0 k vs 199.2 k; at 2 ranks it loses: p2p 210.4 k
// vs 227.5 k); SPB_PLACEMENT=balanced | contiguous overrides.
inline bool contiguous_placement(int nranks) {
  static const int forced = [] {
    const char* p = std::getenv("SPB_PLACEMENT");
    if (!p) return -1;
    return std::string(p) == "contiguous" ? 1 : (std::string(p) == "balanced" ? 0 : -1);
  }();
  return forced >= 0 ? forced == 1 : nranks >= 4;
}

inline std::vector<int> rank_workers(int k, int L, int rank, int nranks) {
  if (k < 1 || nranks < 1 || rank < 0 || rank >= nranks) throw ArgumentError("rank_workers: bad arguments");
  if (nranks > k) throw ArgumentError("rank_workers: more ranks than workers");
  std::vector<std::vector<int>> owned(nranks);
  if (nranks == k) {
    for (int r = 0; r < nranks; ++r) owned[r] = {r + 1};
  } else if (contiguous_placement(nranks)) {
    for (int r = 0; r < nranks; ++r)
      for (int j = static_cast<int>(static_cast<long long>(r) * k / nranks) + 1;
           j <= static_cast<int>(static_cast<long long>(r + 1) * k / nranks); ++j)
        owned[r].push_back(j);
  } else if (k % (2 * nranks) == 0) {
    const int pairs = k / 2;
    for (int p = 0; p < pairs; ++p) {
      const int round = p / nranks, pos = p % nranks;
      const int r = (round % 2 == 0) ? pos : nranks - 1 - pos;
      owned[r].push_back(p + 1);
      owned[r].push_back(k - p);
    }
  } else {
    const int base = k / nranks, extra = k % nranks;
    std::vector<long long> load(nranks, 0);
    std::vector<int> order(k);
    std::iota(order.begin(), order.end(), 1);
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return suffix_layers(a, k, L) > suffix_layers(b, k, L); });
    for (int j : order) {
      int best = -1;
      for (int r = 0; r < nranks; ++r) {
        const int cap = base + (r < extra ? 1 : 0);
        if (static_cast<int>(owned[r].size()) >= cap) continue;
        if (best < 0 || load[r] < load[best]) best = r;
      }
      owned[best].push_back(j);
      load[best] += suffix_layers(j, k, L) + L;
    }
  }
  auto w = owned[rank];
  std::sort(w.begin(), w.end());
  return w;
}

// Per-layer gradient buckets for the multi-GPU step (issued as soon as the
// backward pass has produced that layer, so the collectives overlap the rest
// of the backward). Layer l's contributor RANKS are the ranks hosting a
// worker j with stop_j <= l (every rank when `full`). A bucket with a single
// contributing rank is BROADCAST from it (the others have nothing to add);
// any other bucket is ALL-REDUCED over all ranks, non-contributors adding
// zeros. For ring collectives this is the per-rank-byte-optimal choice: a
// sub-group all-reduce followed by a broadcast costs 2(s-1)/s + 1 > 2(N-1)/N
// bucket sizes whenever s >= 2.
struct Bucket {
  int l_lo, l_hi;          // 1-based layer range [l_lo, l_hi]
  std::vector<int> ranks;  // contributing ranks, ascending
  int kind;                // 0 = all-reduce, 1 = broadcast from root
  int root;
};

inline std::vector<Bucket> bucket_plan(int k, int L, int nranks, bool full) {
  std::vector<std::vector<int>> owned(nranks);
  for (int r = 0; r < nranks; ++r) owned[r] = rank_workers(k, L, r, nranks);
  std::vector<std::vector<int>> per_layer(L + 1);
  for (int l = 1; l <= L; ++l)
    for (int r = 0; r < nranks; ++r)
      for (int j : owned[r])
        if (full || worker_stop(j, k, L) <= l) {
          per_layer[l].push_back(r);
          break;
        }
  std::vector<Bucket> out;
  for (int l = L; l >= 1; --l) {
    Bucket b{l, l, per_layer[l], 0, 0};
    if (b.ranks.size() == 1) b.kind = 1, b.root = b.ranks[0];
    out.push_back(b);
  }
  return out;  // top (layer L) bucket first: the order backward produces them
}

}  // namespace spb
