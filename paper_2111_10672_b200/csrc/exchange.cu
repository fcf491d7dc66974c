// Multi-GPU aggregation of one layer, enqueued from the backward as soon as
// the layer's local wgrad is done (Engine::enqueue_step's on_grad hook):
//   p2p  -- sharded owner pulls with the copy engines + owner update + weight pulls;
//   rh   -- the same buffers on Rabenseifner's recursive-halving schedule;
//   push -- gradient rows stored to their owners by the wgrad epilogue (push.cu);
//   sub  -- NCCL over the layer's contributor sub-communicator.
// DESIGN.md "Multi-GPU" has the measurements behind the defaults.
#include "engine.hpp"

namespace spb {

int Engine::enqueue_p2p_layer(int l, bool full, cudaStream_t gs, cudaStream_t s) {
  const Bucket* bk = nullptr;
  for (auto& b : buckets[full])
    if (b.l_lo <= l && l <= b.l_hi) bk = &b;
  if (!bk) throw ConfigError("comm: no bucket for layer");
  unsigned contrib = 0;
  for (int r : bk->ranks) contrib |= 1u << r;
  const long off = w_off[l], cnt = b_off[l] + round_up(w[l], 32) - w_off[l], n4 = cnt / 4;
  auto lo_of = [&](int r) { return n4 * r / nranks * 4; };
  const long a = lo_of(rank), b = lo_of(rank + 1), sh = b - a;
  // Layer events: 0 dgrad_l issued (s), 1 shard updated (s3), 8+p gradient
  // pull from p done, 16+p weight pull from p done.
  auto evl = [&](int k) { return ev(kEvP2pLayer + 32 * l + k); };
  int n = 0;
  // 1. gradient of l final here -> G[l] to every rank.
  launch_p2p_signal(peer_flags, 2 * l, nranks, rank, epoch_dev, chain_sub, gs);
  SPB_CUDA(cudaEventRecord(evl(0), s));  // dgrad_l issued on s before this point
  ++n;
  // 2. copy engines, one stream per peer: wait for the peer's G[l] (every
  // peer's, contributor or not: that also orders this step's writes after
  // every peer finished the previous step), then pull its gradient of this
  // shard if it contributes.
  float* st_buf = stage + static_cast<long>(l % 2) * (nranks - 1) * stage_shard;
  PeerPtrs<const float> src{};
  int nsrc = 0, slot = 0;
  for (int r = 0; r < nranks; ++r) {
    if (r == rank) {
      if (contrib >> r & 1u) src.p[nsrc++] = grad + off + a;
      continue;
    }
    cudaStream_t cs = gpull[r];
    // Staging buffer l % 2 was last read by the shard update of layer l + 2,
    // or (top layers, chained step) of layer 1 / 2 of the previous step.
    if (l + 2 <= L)
      SPB_CUDA(cudaStreamWaitEvent(cs, ev(kEvP2pLayer + 32 * (l + 2) + 1), 0));
    else if (chain_sub > 0 && l + 2 - L >= 1 && l + 2 - L <= 2)
      SPB_CUDA(cudaStreamWaitEvent(cs, ev(kEvP2pLayer + 32 * ((l % 2) == 1 ? 1 : 2) + 1), 0));
    tbeg(cs);
    launch_p2p_wait(flags, 2 * l, nranks, 1u << r, epoch_dev, chain_sub, cs);
    tend(kTraceWait, cs);
    ++n;
    if (contrib >> r & 1u) {
      float* dst = st_buf + static_cast<long>(slot++) * stage_shard;
      pbeg(cs);
      if (sh > 0) SPB_CUDA(cudaMemcpyAsync(dst, peer_grad[r] + off + a, sh * 4, cudaMemcpyDeviceToDevice, cs));
      pend(kClsComm, static_cast<double>(sh) * 4.0, cs);
      src.p[nsrc++] = dst;
    }
    SPB_CUDA(cudaEventRecord(evl(8 + r), cs));
  }
  // 3. shard update (SMs) -> U[l].
  for (int r = 0; r < nranks; ++r)
    if (r != rank) SPB_CUDA(cudaStreamWaitEvent(s3, evl(8 + r), 0));
  SPB_CUDA(cudaStreamWaitEvent(s3, evl(0), 0));
  if (contrib >> rank & 1u) {
    SPB_CUDA(cudaEventRecord(ev(kEvBucket + l), gs));
    SPB_CUDA(cudaStreamWaitEvent(s3, ev(kEvBucket + l), 0));
  }
  pbeg(s3);
  launch_p2p_update(src, nsrc, p_hi + off + a, p_lo + off + a, mom ? mom + off + a : nullptr, w32 + off + a, sh, lr, mu,
                    wd, s3);
  pend(kClsUpdate, static_cast<double>(sh) * 4.0 * (nsrc + (mom ? 7 : 5)), s3);
  launch_p2p_signal(peer_flags, 2 * l + 1, nranks, rank, epoch_dev, chain_sub, s3);
  SPB_CUDA(cudaEventRecord(evl(1), s3));
  n += 2;
  // 4. copy engines, one stream per peer: pull its updated fp32 shard.
  for (int r = 0; r < nranks; ++r) {
    if (r == rank) continue;
    cudaStream_t cs = wpull[r];
    tbeg(cs);
    launch_p2p_wait(flags, 2 * l + 1, nranks, 1u << r, epoch_dev, chain_sub, cs);
    tend(kTraceWait, cs);
    ++n;
    const long ra = lo_of(r), rb = lo_of(r + 1);
    pbeg(cs);
    if (rb > ra)
      SPB_CUDA(cudaMemcpyAsync(w32 + off + ra, peer_w32[r] + off + ra, (rb - ra) * 4, cudaMemcpyDeviceToDevice, cs));
    pend(kClsComm, static_cast<double>(rb - ra) * 4.0, cs);
    SPB_CUDA(cudaEventRecord(evl(16 + r), cs));
    SPB_CUDA(cudaStreamWaitEvent(s4, evl(16 + r), 0));
  }
  // 5. split the pulled shards into (hi, lo) (after dgrad_l).
  SPB_CUDA(cudaStreamWaitEvent(s4, evl(0), 0));
  pbeg(s4);
  launch_p2p_split(w32 + off, p_hi + off, p_lo + off, cnt, a, b, s4);
  pend(kClsUpdate, static_cast<double>(cnt - sh) * 12.0, s4);
  ++n;
  // W_l final here: the peers' shards split (s4) and this rank's own (s3).
  SPB_CUDA(cudaStreamWaitEvent(s4, evl(1), 0));
  SPB_CUDA(cudaEventRecord(ev(ev_ready(l)), s4));
  fwd_wait[l] = ev_ready(l);
  return n;
}

int Engine::enqueue_rh_layer(int l, bool full, cudaStream_t gs, cudaStream_t s) {
  const Bucket* bk = nullptr;
  for (auto& b : buckets[full])
    if (b.l_lo <= l && l <= b.l_hi) bk = &b;
  if (!bk) throw ConfigError("comm: no bucket for layer");
  unsigned contrib = 0;
  for (int r : bk->ranks) contrib |= 1u << r;
  const int d = flag_slots / 2;
  const long off = w_off[l], cnt = b_off[l] + round_up(w[l], 32) - w_off[l], n4 = cnt / 4;
  auto lo_of = [&](int sidx) { return n4 * sidx / nranks * 4; };
  auto evl = [&](int k) { return ev(kEvP2pLayer + 32 * l + k); };
  auto slot = [&](int j) { return flag_slots * l + j; };
  // Ranks whose contributions a partial held by rank q before reduce round
  // k covers: those agreeing with q on bits 0..b (b = d-1-k).
  auto covers = [&](int q, int b) {
    unsigned m = 0;
    const int low = (1 << (b + 1)) - 1;
    for (int x = 0; x < nranks; ++x)
      if ((x & low) == (q & low)) m |= 1u << x;
    return m;
  };
  int n = 0;
  SPB_CUDA(cudaEventRecord(evl(0), s));  // dgrad_l (last reader of W_l) issued on s
  launch_p2p_signal(peer_flags, slot(0), nranks, rank, epoch_dev, chain_sub, gs);
  ++n;
  SPB_CUDA(cudaEventRecord(ev(kEvBucket + l), gs));
  SPB_CUDA(cudaStreamWaitEvent(s3, ev(kEvBucket + l), 0));
  SPB_CUDA(cudaStreamWaitEvent(s3, evl(0), 0));
  float* st_buf = stage + static_cast<long>(l % 2) * (nranks - 1) * stage_shard;
  long st_off = 0;
  bool own = contrib >> rank & 1u;  // does this rank's buffer hold a valid partial?
  PeerPtrs<const float> fin{};
  int nfin = 0;
  for (int k = 0; k < d; ++k) {
    const int b = d - 1 - k, p = rank ^ (1 << b);
    const int base = (rank >> (b + 1)) << (b + 1), s0 = base + (((rank >> b) & 1) << b), s1 = s0 + (1 << b);
    const long a0 = lo_of(s0), a1 = lo_of(s1), len = a1 - a0;
    const bool theirs = (covers(p, b) & contrib) != 0;
    cudaStream_t cs = gpull[p];
    // Staging reuse: the buffer of layer l % 2 was last read by layer l + 2's
    // update, or (top layers, chained step) by layer 1 / 2's update of the
    // previous step -- the same explicit wait as the p2p mode, instead of
    // relying on the transitive cross-rank flag ordering alone.
    if (k == 0 && l + 2 <= L)
      SPB_CUDA(cudaStreamWaitEvent(cs, ev(kEvP2pLayer + 32 * (l + 2) + 1), 0));
    else if (k == 0 && chain_sub > 0 && l + 2 - L >= 1 && l + 2 - L <= 2)
      SPB_CUDA(cudaStreamWaitEvent(cs, ev(kEvP2pLayer + 32 * ((l % 2) == 1 ? 1 : 2) + 1), 0));
    if (k > 0) SPB_CUDA(cudaStreamWaitEvent(cs, evl(3 + k - 1 + 8), 0));  // my previous round's sum done
    tbeg(cs);
    launch_p2p_wait(flags, k == 0 ? slot(0) : slot(k), nranks, 1u << p, epoch_dev, chain_sub, cs);
    tend(kTraceWait, cs);
    ++n;
    float* dst = nullptr;
    if (theirs) {
      dst = own ? st_buf + st_off : grad + off + a0;
      if (!own && k == 0) SPB_CUDA(cudaStreamWaitEvent(cs, ev(kEvBucket + l), 0));  // (own grad unused; order anyway)
      pbeg(cs);
      if (len > 0) SPB_CUDA(cudaMemcpyAsync(dst, peer_grad[p] + off + a0, len * 4, cudaMemcpyDeviceToDevice, cs));
      pend(kClsComm, static_cast<double>(len) * 4.0, cs);
    }
    SPB_CUDA(cudaEventRecord(evl(3 + k), cs));
    SPB_CUDA(cudaStreamWaitEvent(s3, evl(3 + k), 0));
    if (k < d - 1) {
      if (theirs && own) {
        pbeg(s3);
        launch_rh_add(grad + off + a0, st_buf + st_off, len, s3);
        pend(kClsUpdate, static_cast<double>(len) * 12.0, s3);
        ++n;
      }
      own = own || theirs;
      launch_p2p_signal(peer_flags, slot(1 + k), nranks, rank, epoch_dev, chain_sub, s3);
      ++n;
      SPB_CUDA(cudaEventRecord(evl(3 + k + 8), s3));
    } else {
      if (own) fin.p[nfin++] = grad + off + a0;
      if (theirs && own) fin.p[nfin++] = st_buf + st_off;
      if (theirs && !own) fin.p[nfin++] = grad + off + a0;
    }
    if (theirs && own) st_off += len;
  }
  // Update of shard `rank` (the last round's range) -> hi, lo, mom, w32.
  const long a = lo_of(rank), sh = lo_of(rank + 1) - a;
  pbeg(s3);
  launch_p2p_update(fin, nfin, p_hi + off + a, p_lo + off + a, mom ? mom + off + a : nullptr, w32 + off + a, sh, lr, mu,
                    wd, s3);
  pend(kClsUpdate, static_cast<double>(sh) * 4.0 * (nfin + (mom ? 7 : 5)), s3);
  launch_p2p_signal(peer_flags, slot(d), nranks, rank, epoch_dev, chain_sub, s3);
  SPB_CUDA(cudaEventRecord(evl(1), s3));
  n += 2;
  // All-gather rounds: pull the partner's final weight block of 2^b shards.
  cudaStream_t prev = s3;
  for (int b = 0; b < d; ++b) {
    const int p = rank ^ (1 << b);
    const int pb = (p >> b) << b;
    const long a0 = lo_of(pb), a1 = lo_of(pb + (1 << b));
    cudaStream_t cs = wpull[p];
    SPB_CUDA(cudaEventRecord(evl(24 + b), prev));
    SPB_CUDA(cudaStreamWaitEvent(cs, evl(24 + b), 0));  // my block of 2^b shards final
    tbeg(cs);
    launch_p2p_wait(flags, slot(d + b), nranks, 1u << p, epoch_dev, chain_sub, cs);
    tend(kTraceWait, cs);
    pbeg(cs);
    if (a1 > a0) SPB_CUDA(cudaMemcpyAsync(w32 + off + a0, peer_w32[p] + off + a0, (a1 - a0) * 4,
                                          cudaMemcpyDeviceToDevice, cs));
    pend(kClsComm, static_cast<double>(a1 - a0) * 4.0, cs);
    n += 1;
    if (b + 1 < d) {
      launch_p2p_signal(peer_flags, slot(d + b + 1), nranks, rank, epoch_dev, chain_sub, cs);
      ++n;
    }
    prev = cs;
  }
  // Split every shard but this rank's own into (hi, lo), after dgrad_l.
  SPB_CUDA(cudaEventRecord(evl(16), prev));
  SPB_CUDA(cudaStreamWaitEvent(s4, evl(16), 0));
  SPB_CUDA(cudaStreamWaitEvent(s4, evl(0), 0));
  pbeg(s4);
  launch_p2p_split(w32 + off, p_hi + off, p_lo + off, cnt, a, a + sh, s4);
  pend(kClsUpdate, static_cast<double>(cnt - sh) * 12.0, s4);
  ++n;
  SPB_CUDA(cudaStreamWaitEvent(s4, evl(1), 0));
  SPB_CUDA(cudaEventRecord(ev(ev_ready(l)), s4));
  fwd_wait[l] = ev_ready(l);
  return n;
}

int Engine::enqueue_sub_layer(int l, bool full, cudaStream_t gs, cudaStream_t s) {
  const Bucket* bk = nullptr;
  for (auto& b : buckets[full])
    if (b.l_lo <= l && l <= b.l_hi) bk = &b;
  if (!bk) throw ConfigError("comm: no bucket for layer");
  const std::vector<int>& C = bk->ranks;
  const int nc = static_cast<int>(C.size());
  const int me = static_cast<int>(std::find(C.begin(), C.end(), rank) - C.begin());  // nc: not a member
  const long off = w_off[l], cnt = b_off[l] + round_up(w[l], 32) - w_off[l];
  const long sh = layer_shard(cnt, nc);
  auto lo_of = [&](int i) { return std::min(cnt, sh * i); };
  auto evl = [&](int k) { return ev(kEvP2pLayer + 32 * l + k); };
  SPB_CUDA(cudaEventRecord(ev(kEvBucket + l), gs));
  SPB_CUDA(cudaStreamWaitEvent(cst, ev(kEvBucket + l), 0));
  SPB_CUDA(cudaEventRecord(evl(0), s));  // dgrad_l issued on s before this point
  int n = 0;
  long a = 0, b = 0;  // the range this rank updates itself
  pbeg(cst);
  if (me < nc) {
    a = lo_of(me), b = lo_of(me + 1);
    const float* g = grad + off + a;
    if (nc > 1) {  // reduce-scatter among the contributors (reads up to nc*sh: grad has tail slack)
      auto it = subcomms.find(C);
      if (it == subcomms.end() || !it->second) throw ConfigError("comm: missing contributor communicator");
      nccl_check(nccl().ReduceScatter(grad + off, stage, sh, ncclFloat32, ncclSum, it->second, cst));
      g = stage;
    }
    SPB_CUDA(cudaStreamWaitEvent(cst, evl(0), 0));
    if (b > a) {
      PeerPtrs<const float> src{};
      src.p[0] = g;
      launch_p2p_update(src, 1, p_hi + off + a, p_lo + off + a, mom ? mom + off + a : nullptr, w32 + off + a, b - a,
                        lr, mu, wd, cst);
      ++n;
    }
  } else {
    SPB_CUDA(cudaStreamWaitEvent(cst, evl(0), 0));
  }
  nccl_check(nccl().GroupStart());
  for (int i = 0; i < nc; ++i) {
    const long ia = lo_of(i), ib = lo_of(i + 1);
    if (ib > ia) nccl_check(nccl().Broadcast(w32 + off + ia, w32 + off + ia, ib - ia, ncclFloat32, C[i], comm, cst));
  }
  nccl_check(nccl().GroupEnd());
  // Bytes this rank moves: its reduce-scatter share (contributors) plus the
  // weight shards it receives.
  pend(kClsComm, 4.0 * ((me < nc && nc > 1 ? static_cast<double>(sh) * (nc - 1) : 0.0) + (cnt - (b - a))), cst);
  pbeg(cst);
  launch_p2p_split(w32 + off, p_hi + off, p_lo + off, cnt, a, b, cst);
  pend(kClsUpdate, static_cast<double>(cnt - (b - a)) * 12.0, cst);
  return n + 1;
}

void Engine::setup_sub() {
  w32 = alloc<float>(nflat);
  long maxcnt = 0;
  for (int l = 1; l <= L; ++l) maxcnt = std::max(maxcnt, b_off[l] + round_up(w[l], 32) - w_off[l]);
  stage_shard = layer_shard(maxcnt, 2);
  stage = alloc<float>(stage_shard);
  // One communicator per distinct contributor set, split collectively in
  // the same (sorted) order on every rank.
  std::vector<std::vector<int>> sets;
  for (int f = 0; f < 2; ++f)
    for (const Bucket& b : buckets[f])
      if (b.ranks.size() > 1 && std::find(sets.begin(), sets.end(), b.ranks) == sets.end()) sets.push_back(b.ranks);
  std::sort(sets.begin(), sets.end());
  for (const auto& set : sets) {
    const bool member = std::find(set.begin(), set.end(), rank) != set.end();
    ncclComm_t c = nullptr;
    nccl_check(nccl().CommSplit(comm, member ? 0 : NCCL_SPLIT_NOCOLOR, rank, &c, nullptr));
    subcomms[set] = member ? c : nullptr;
  }
  comm_mode = 3;
  invalidate_graphs();
}

void Engine::setup_p2p(int slots_per_layer) {
  if (nranks > kMaxPeers) throw ConfigError("comm: p2p mode supports at most 8 ranks");
  if (!bar_dev) bar_dev = alloc<float>(1);
  w32 = alloc<float>(nflat);
  flag_slots = slots_per_layer;
  flags = alloc<int>(static_cast<long>(slots_per_layer) * (L + 1) * nranks);
  epoch_dev = alloc<int>(1);
  long maxcnt = 0;
  for (int l = 1; l <= L; ++l) maxcnt = std::max(maxcnt, b_off[l] + round_up(w[l], 32) - w_off[l]);
  stage_shard = round_up((maxcnt / 4 + nranks - 1) / nranks * 4, 32);
  stage = alloc<float>(2L * std::max(1, nranks - 1) * stage_shard);
  cudaIpcMemHandle_t mine[3];
  SPB_CUDA(cudaIpcGetMemHandle(&mine[0], grad));
  SPB_CUDA(cudaIpcGetMemHandle(&mine[1], w32));
  SPB_CUDA(cudaIpcGetMemHandle(&mine[2], flags));
  const size_t hb = sizeof mine;
  char* dbuf = nullptr;
  SPB_CUDA(cudaMalloc(&dbuf, hb * (nranks + 1)));
  SPB_CUDA(cudaMemcpy(dbuf, mine, hb, cudaMemcpyHostToDevice));
  nccl_check(nccl().AllGather(dbuf, dbuf + hb, hb, ncclUint8, comm, cst));
  SPB_CUDA(cudaStreamSynchronize(cst));
  std::vector<cudaIpcMemHandle_t> all(3 * nranks);
  SPB_CUDA(cudaMemcpy(all.data(), dbuf + hb, hb * nranks, cudaMemcpyDeviceToHost));
  cudaFree(dbuf);
  peer_grad.assign(nranks, nullptr);
  peer_w32.assign(nranks, nullptr);
  for (int p = 0; p < nranks; ++p) {
    if (p == rank) {
      peer_grad[p] = grad, peer_w32[p] = w32, peer_flags.p[p] = flags;
      continue;
    }
    void* q = nullptr;
    SPB_CUDA(cudaIpcOpenMemHandle(&q, all[3 * p + 0], cudaIpcMemLazyEnablePeerAccess));
    peer_grad[p] = static_cast<float*>(q);
    SPB_CUDA(cudaIpcOpenMemHandle(&q, all[3 * p + 1], cudaIpcMemLazyEnablePeerAccess));
    peer_w32[p] = static_cast<float*>(q);
    SPB_CUDA(cudaIpcOpenMemHandle(&q, all[3 * p + 2], cudaIpcMemLazyEnablePeerAccess));
    peer_flags.p[p] = static_cast<int*>(q);
  }
  SPB_CUDA(cudaStreamCreateWithFlags(&s4, cudaStreamNonBlocking));
  gpull.assign(nranks, nullptr);
  wpull.assign(nranks, nullptr);
  for (int p = 0; p < nranks; ++p) {
    if (p == rank) continue;
    SPB_CUDA(cudaStreamCreateWithFlags(&gpull[p], cudaStreamNonBlocking));
    SPB_CUDA(cudaStreamCreateWithFlags(&wpull[p], cudaStreamNonBlocking));
  }
  comm_mode = 2;
  invalidate_graphs();
  host_barrier();
}

void Engine::setup_push() {
  if (nranks > kMaxPeers) throw ConfigError("comm: push mode supports at most 8 ranks");
  if (conv_model) throw ConfigError("comm: push mode is MLP-only");
  if (!bar_dev) bar_dev = alloc<float>(1);
  w32 = alloc<float>(nflat);
  flags = alloc<int>(2L * (L + 1) * nranks);
  epoch_dev = alloc<int>(1);
  prpo.assign(L + 1, 0);
  pstage_off.assign(L + 1, 0);
  pslot.assign(L + 1, 0);
  long tot = 0;
  for (int l = 1; l <= L; ++l) {
    prpo[l] = (w[l] + nranks - 1) / nranks;
    pslot[l] = round_up(static_cast<long>(prpo[l]) * ld[l - 1] + prpo[l], 32);
    pstage_off[l] = tot;
    tot += pslot[l] * nranks;
  }
  pstage = alloc<float>(tot);
  cudaIpcMemHandle_t mine[3];
  SPB_CUDA(cudaIpcGetMemHandle(&mine[0], pstage));
  SPB_CUDA(cudaIpcGetMemHandle(&mine[1], w32));
  SPB_CUDA(cudaIpcGetMemHandle(&mine[2], flags));
  const size_t hb = sizeof mine;
  char* dbuf = nullptr;
  SPB_CUDA(cudaMalloc(&dbuf, hb * (nranks + 1)));
  SPB_CUDA(cudaMemcpy(dbuf, mine, hb, cudaMemcpyHostToDevice));
  nccl_check(nccl().AllGather(dbuf, dbuf + hb, hb, ncclUint8, comm, cst));
  SPB_CUDA(cudaStreamSynchronize(cst));
  std::vector<cudaIpcMemHandle_t> all(3 * nranks);
  SPB_CUDA(cudaMemcpy(all.data(), dbuf + hb, hb * nranks, cudaMemcpyDeviceToHost));
  cudaFree(dbuf);
  peer_grad.assign(nranks, nullptr);
  peer_pstage.assign(nranks, nullptr);
  peer_w32.assign(nranks, nullptr);
  for (int p = 0; p < nranks; ++p) {
    if (p == rank) {
      peer_pstage[p] = pstage, peer_w32[p] = w32, peer_flags.p[p] = flags;
      continue;
    }
    void* q = nullptr;
    SPB_CUDA(cudaIpcOpenMemHandle(&q, all[3 * p + 0], cudaIpcMemLazyEnablePeerAccess));
    peer_pstage[p] = static_cast<float*>(q);
    SPB_CUDA(cudaIpcOpenMemHandle(&q, all[3 * p + 1], cudaIpcMemLazyEnablePeerAccess));
    peer_w32[p] = static_cast<float*>(q);
    SPB_CUDA(cudaIpcOpenMemHandle(&q, all[3 * p + 2], cudaIpcMemLazyEnablePeerAccess));
    peer_flags.p[p] = static_cast<int*>(q);
  }
  SPB_CUDA(cudaStreamCreateWithFlags(&s4, cudaStreamNonBlocking));
  wpull.assign(nranks, nullptr);
  for (int p = 0; p < nranks; ++p)
    if (p != rank) SPB_CUDA(cudaStreamCreateWithFlags(&wpull[p], cudaStreamNonBlocking));
  comm_mode = 4;
  invalidate_graphs();
  host_barrier();
}

void Engine::push_route(int l, GemmEpilogue& ep) const {
  ep.route_rows = prpo[l];
  for (int o = 0; o < nranks; ++o)
    ep.route[o] = o == rank ? grad + w_off[l] + static_cast<long>(o) * prpo[l] * ld[l - 1]
                            : peer_pstage[o] + pstage_off[l] + static_cast<long>(rank) * pslot[l];
}

int Engine::enqueue_push_layer(int l, bool full, cudaStream_t gs, cudaStream_t s) {
  const Bucket* bk = nullptr;
  for (auto& b : buckets[full])
    if (b.l_lo <= l && l <= b.l_hi) bk = &b;
  if (!bk) throw ConfigError("comm: no bucket for layer");
  unsigned contrib = 0;
  for (int r : bk->ranks) contrib |= 1u << r;
  const bool mine = contrib >> rank & 1u;
  const unsigned peers = ((1u << nranks) - 1u) & ~(1u << rank);
  const long ldw = ld[l - 1];
  const int rpo = prpo[l];
  const int r0 = std::min(w[l], rank * rpo), r1 = std::min(w[l], (rank + 1) * rpo);
  auto evl = [&](int k) { return ev(kEvP2pLayer + 32 * l + k); };
  // Layer L's weight gradient comes from a column reduction, not the routed
  // wgrad GEMM: its rows travel with the signal.
  const bool rows_in_signal = l == L || conv_model;
  PeerPtrs<float> wdst{}, bdst{};
  for (int o = 0; o < nranks; ++o) {
    if (o == rank) continue;
    wdst.p[o] = peer_pstage[o] + pstage_off[l] + static_cast<long>(rank) * pslot[l];
    bdst.p[o] = wdst.p[o] + static_cast<long>(rpo) * ldw;
  }
  // 1. bias rows (+ head weight rows) to their owners, fence, G[l].
  pbeg(gs);
  launch_push_signal(peer_flags, 2 * l, nranks, rank, epoch_dev, chain_sub,
                     mine && rows_in_signal ? grad + w_off[l] : nullptr, ldw, mine ? grad + b_off[l] : nullptr, rpo,
                     w[l], wdst, bdst, gs);
  // Bytes this rank sends to the owners (the wgrad epilogue's routed rows
  // and the bias rows): its share of the exchange, like a pull elsewhere.
  pend(kClsComm, mine ? static_cast<double>(w[l] - (r1 - r0)) * (ldw + 1) * 4.0 : 0.0, gs);
  SPB_CUDA(cudaEventRecord(evl(0), s));  // dgrad_l issued on s before this point
  SPB_CUDA(cudaEventRecord(ev(kEvBucket + l), gs));
  // 2. owner update on s3: every rank's G[l], own gradient final, dgrad_l
  // done (the update rewrites W_l rows in place).
  SPB_CUDA(cudaStreamWaitEvent(s3, ev(kEvBucket + l), 0));
  SPB_CUDA(cudaStreamWaitEvent(s3, evl(0), 0));
  tbeg(s3);
  launch_p2p_wait(flags, 2 * l, nranks, peers, epoch_dev, chain_sub, s3);
  tend(kTraceWait, s3);
  const long nw = static_cast<long>(r1 - r0) * ldw, nb = r1 - r0;
  PeerPtrs<const float> sw{}, sb{};
  PeerPtrs<float> dw{}, db{};
  int nsrc = 0, ndst = 0;
  for (int r = 0; r < nranks; ++r) {
    if (!(contrib >> r & 1u)) continue;
    if (r == rank) {
      sw.p[nsrc] = grad + w_off[l] + static_cast<long>(r0) * ldw;
      sb.p[nsrc] = grad + b_off[l] + r0;
    } else {
      sw.p[nsrc] = pstage + pstage_off[l] + static_cast<long>(r) * pslot[l];
      sb.p[nsrc] = sw.p[nsrc] + static_cast<long>(rpo) * ldw;
    }
    ++nsrc;
  }
  // The owner's new fp32 rows go to its own w32; the peers pull them (copy
  // engines), as in the p2p mode.
  dw.p[ndst] = w32 + w_off[l] + static_cast<long>(r0) * ldw;
  db.p[ndst] = w32 + b_off[l] + r0;
  ++ndst;
  pbeg(s3);
  launch_push_update(sw, nsrc, p_hi + w_off[l] + r0 * ldw, p_lo + w_off[l] + r0 * ldw,
                     mom ? mom + w_off[l] + r0 * ldw : nullptr, dw, ndst, nw, lr, mu, wd, s3);
  launch_push_update(sb, nsrc, p_hi + b_off[l] + r0, p_lo + b_off[l] + r0, mom ? mom + b_off[l] + r0 : nullptr, db,
                     ndst, nb, lr, mu, wd, s3);
  pend(kClsUpdate, static_cast<double>(nw + nb) * 4.0 * (nsrc + (mom ? 6 : 5)), s3);
  launch_p2p_signal(peer_flags, 2 * l + 1, nranks, rank, epoch_dev, chain_sub, s3);
  SPB_CUDA(cudaEventRecord(evl(1), s3));
  // 3. every other owner's rows: wait for its U[l], pull (copy engines);
  // then split after dgrad_l.
  for (int o = 0; o < nranks; ++o) {
    if (o == rank) continue;
    const int q0 = std::min(w[l], o * rpo), q1 = std::min(w[l], (o + 1) * rpo);
    cudaStream_t cs = wpull[o];
    tbeg(cs);
    launch_p2p_wait(flags, 2 * l + 1, nranks, 1u << o, epoch_dev, chain_sub, cs);
    tend(kTraceWait, cs);
    if (q1 > q0) {
      pbeg(cs);
      SPB_CUDA(cudaMemcpyAsync(w32 + w_off[l] + static_cast<long>(q0) * ldw, peer_w32[o] + w_off[l] + q0 * ldw,
                               static_cast<size_t>(q1 - q0) * ldw * 4, cudaMemcpyDeviceToDevice, cs));
      SPB_CUDA(cudaMemcpyAsync(w32 + b_off[l] + q0, peer_w32[o] + b_off[l] + q0, static_cast<size_t>(q1 - q0) * 4,
                               cudaMemcpyDeviceToDevice, cs));
      pend(kClsComm, static_cast<double>(q1 - q0) * (ldw + 1) * 4.0, cs);
    }
    SPB_CUDA(cudaEventRecord(evl(16 + o), cs));
    SPB_CUDA(cudaStreamWaitEvent(s4, evl(16 + o), 0));
  }
  SPB_CUDA(cudaStreamWaitEvent(s4, evl(0), 0));
  pbeg(s4);
  launch_push_split(w32 + w_off[l], p_hi + w_off[l], p_lo + w_off[l], static_cast<long>(w[l]) * ldw, r0 * ldw,
                    r1 * ldw, s4);
  launch_push_split(w32 + b_off[l], p_hi + b_off[l], p_lo + b_off[l], w[l], r0, r1, s4);
  pend(kClsUpdate, static_cast<double>(w[l] - (r1 - r0)) * (ldw + 1) * 12.0, s4);
  SPB_CUDA(cudaStreamWaitEvent(s4, evl(1), 0));
  SPB_CUDA(cudaEventRecord(ev(ev_ready(l)), s4));
  fwd_wait[l] = ev_ready(l);
  return 6;
}

void Engine::host_barrier() {
  nccl_check(nccl().AllReduce(bar_dev, bar_dev, 1, ncclFloat32, ncclSum, comm, cst));
  SPB_CUDA(cudaStreamSynchronize(cst));
}

}  // namespace spb
