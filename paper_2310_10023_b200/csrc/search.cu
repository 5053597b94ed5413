// search.cu — K5/K6 (branching + best-first frontier) and the search driver.
//
// Replaces search() (search.hpp:72-186).  The reference's loop is replayed
// EXACTLY on the device as flush epochs:
//   * the queue is a sorted array; keys encode EntryCompare (search.hpp:47-59):
//       BFS  (score desc, level desc, seq asc)
//       DFS  (level asc, score desc, seq desc)
//   * between flushes nothing is pushed, so an epoch pops a queue PREFIX.
//     With B_i = max(B_0, max leaf score before i), entry i is pruned when
//     score_i < B_i, a surviving leaf sets the incumbent, a surviving inner
//     node adds c_i = 8 * prod(in-range rotational children) to `pending`,
//     and the flush happens at the first i with sum(c) > b (or on drain);
//   * the flush scores pending (score.cu), keeps score >= B, assigns seq in
//     pending order, sorts the survivors by key and merges them into the
//     remaining queue.
// Kernels per epoch: frontier (1 CTA scan) -> branch -> score -> survivors
// (1 CTA compaction) -> rank-sort -> merge -> finalize.  Every kernel reads
// its sizes from the device-resident EpochState, so epochs are enqueued back
// to back with no host round-trip; the host reads the 100-byte state every
// few epochs (or every epoch when an incumbent exchange is configured).
#include <nvtx3/nvToolsExt.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <exception>
#include <mutex>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <vector>

#include "bbs_comm.h"
#include "bbs_map_impl.h"
#include "device_common.cuh"
#include "kernels.h"
#include "score_common.cuh"

namespace bbs {

thread_local unsigned g_grid_share = 1;
thread_local bool g_blocking_sync = false;

namespace {

constexpr unsigned long long kSMax = (1ull << 20) - 1;
constexpr unsigned long long kSeqMax = (1ull << 40) - 1;

struct EpochState {
  int32_t best;          // incumbent B (search.hpp:99)
  int32_t matched;
  bbs_node best_node;
  uint32_t q_len;        // queue length (in buffer `cur`)
  uint32_t cur;
  unsigned long long seq;  // next insertion sequence number (search.hpp:107)
  unsigned long long nodes_generated, nodes_pruned, batches_flushed, epochs;
  unsigned long long trace_len;
  int32_t last_best_epoch;  // frontier pass that set the incumbent last
  int32_t active;
  uint32_t n_cons, n_children, n_expand, n_surv;
  int32_t flush_best;
  uint32_t pass;           // frontier passes executed while active
  uint32_t q_peak;
  uint32_t n_keep;         // queue remainder kept after the incumbent trim
  uint32_t surv_ticket;    // survivors tile tickets (reset by the frontier)
  uint32_t merge_done;     // merge CTAs finished (the last one finalizes the epoch)
  uint32_t fuse_claim, fuse_done, fuse_a;  // fused merge prologue: tasks claimed / finished / tile sorts finished
  uint32_t tile_rank_min;  // survivors from which the fused sort ranks against sorted tiles
  uint32_t merge_all;      // A/B: every merge CTA ranks the survivors (BBS_MERGE_IDLE=0)
  uint32_t cache_raw;      // levels whose histogram builds gave up (flush cache, per frontier pass)
  uint32_t n_own;          // batch-split exact mode: children of this rank's runs
  int32_t any_active;      // sharded (device exchange): any rank still active
  uint32_t spec_n;         // speculative round: epochs the frontier formed
  uint32_t spec_acc;       // ... of which the validation accepted (a prefix)
  uint32_t spec_k;         // epochs the next round may form (adaptive, 1..spec_kmax)
  uint32_t spec_kmax;
  uint32_t spec_mode;       // device-switched rounds (spec_auto): 1 = this epoch is a speculative round
  uint32_t spec_votes;      // consecutive plain epochs whose next epoch a round would have kept
  unsigned long long look_key;  // plain epoch (voting): key of the entry the next epoch would pop last (~0 unknown)
  unsigned long long level_evals[kMaxLevels];  // flush evaluations per level
  // kept ranges of the remainder: one per key segment (BFS: 1, DFS: level)
  uint32_t seg_lo[kMaxLevels], seg_len[kMaxLevels], seg_pre[kMaxLevels + 1];
};

// The queue is a sorted array of 64-bit keys (double-buffered); a key embeds
// its entry's insertion seq, and the entry's node lives at pool[seq] (an
// append-only pool written once per push), so re-ordering moves 8 B keys.
struct Queue {
  unsigned long long* key[2];
  bbs_node* pool;
  // select, not index: a runtime index into a by-value kernel parameter
  // array makes the compiler copy the struct to local memory
  __device__ __forceinline__ unsigned long long* keys(uint32_t b) const { return b ? key[1] : key[0]; }
};

__device__ __forceinline__ unsigned long long queue_key(int strategy, int32_t score, int32_t level,
                                                        unsigned long long seq) {
  const unsigned long long s = kSMax - static_cast<unsigned long long>(score);
  if (strategy == BBS_STRATEGY_BFS)
    return (s << 44) | (static_cast<unsigned long long>(15 - level) << 40) | seq;
  return (static_cast<unsigned long long>(level) << 60) | (s << 40) | (kSeqMax - seq);
}

__device__ __forceinline__ uint32_t key_seq(int strategy, unsigned long long key) {
  const unsigned long long low = key & kSeqMax;
  return static_cast<uint32_t>(strategy == BBS_STRATEGY_BFS ? low : kSeqMax - low);
}

// Per-axis in-range rotational children of branch(), nodes.hpp:99-111.
__device__ __forceinline__ void child_counts(const GridView& G, const bbs_node& n, int32_t a[3],
                                             int32_t c[3]) {
  const int l = n.level, cl = n.level - 1;
  const int32_t idx[3] = {n.iroll, n.ipitch, n.iyaw};
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    a[ax] = G.div[l * 3 + ax];
    const long long room = static_cast<long long>(G.max_index[cl * 3 + ax]) -
                           static_cast<long long>(a[ax]) * idx[ax] + 1;
    c[ax] = static_cast<int32_t>(room < 0 ? 0 : (room > a[ax] ? a[ax] : room));
  }
}

__device__ __forceinline__ uint32_t n_children_of(const GridView& G, const bbs_node& n) {
  int32_t a[3], c[3];
  child_counts(G, n, a, c);
  return 8u * static_cast<uint32_t>(c[0]) * static_cast<uint32_t>(c[1]) * static_cast<uint32_t>(c[2]);
}

constexpr int kFT = 256;
constexpr int kFIPT = 4;
constexpr int kFChunk = kFT * kFIPT;

// E1: which queue prefix this epoch pops, pruning, leaf updates, children.
__device__ __forceinline__ void frontier_kernel_body(EpochState* st,
                                                     Queue q,
                                                     const GridView& G,
                                                     unsigned long long b,
                                                     uint32_t* __restrict__ exp_parent,
                                                     uint32_t* __restrict__ exp_off,
                                                     int32_t* __restrict__ trace,
                                                     unsigned long long trace_cap,
                                                     int strategy,
                                                     uint32_t* __restrict__ cache_ctl,
                                                     int active_pre = -1,
                                                     bool look = false) {
  pdl_wait();

  using ScanI = cub::BlockScan<int, kFT>;
  using ScanU = cub::BlockScan<unsigned long long, kFT>;
  using RedI = cub::BlockReduce<int, kFT>;
  __shared__ union {
    typename ScanI::TempStorage si;
    typename ScanU::TempStorage su;
    typename RedI::TempStorage ri;
    typename cub::BlockReduce<unsigned long long, kFT>::TempStorage ru;
  } tmp;
  __shared__ int s_cut, s_lastlu;
  __shared__ unsigned long long s_sum_at_cut, s_look;
  __shared__ int s_active;

  const int tid = threadIdx.x;
  if (tid == 0) s_look = ~0ull;  // unknown unless the cut and the next one fall in one chunk
  if (tid == 0) s_active = active_pre >= 0 ? active_pre : st->active;
  __syncthreads();
  if (!s_active) {
    if (tid == 0) st->n_children = 0;
    return;
  }
  const uint32_t qlen = st->q_len;
  const unsigned long long* __restrict__ qk = q.keys(st->cur);
  const bbs_node* __restrict__ pool = q.pool;
  int carry_best = st->best;
  unsigned long long carry_sum = 0, carry_trace = st->trace_len;
  uint32_t carry_exp = 0;
  uint32_t consumed = qlen;
  unsigned long long pruned = 0;
  int best_i = -1;

  for (uint32_t base = 0; base < qlen; base += kFChunk) {
    bbs_node nd[kFIPT];
    bool valid[kFIPT];
    int lm = INT_MIN;
#pragma unroll
    for (int k = 0; k < kFIPT; ++k) {
      const uint32_t i = base + tid * kFIPT + k;
      valid[k] = i < qlen;
      if (valid[k]) {
        nd[k] = pool[key_seq(strategy, qk[i])];
        if (nd[k].level == 0) lm = max(lm, nd[k].score);
      }
    }
    int excl;
    ScanI(tmp.si).ExclusiveScan(lm, excl, INT_MIN, cub::Max());
    __syncthreads();
    int B = max(carry_best, excl);
    uint32_t c[kFIPT];
    bool pr[kFIPT], lu[kFIPT];
    unsigned long long csum = 0;
#pragma unroll
    for (int k = 0; k < kFIPT; ++k) {
      c[k] = 0;
      pr[k] = lu[k] = false;
      if (!valid[k]) continue;
      const int s = nd[k].score;
      pr[k] = s < B;  // search.hpp:150-153
      const bool leaf = nd[k].level == 0;
      lu[k] = !pr[k] && leaf;  // search.hpp:154-160
      if (lu[k]) B = s;
      if (!pr[k] && !leaf) c[k] = n_children_of(G, nd[k]);
      csum += c[k];
    }
    unsigned long long sexcl, stotal;
    ScanU(tmp.su).ExclusiveSum(csum, sexcl, stotal);
    __syncthreads();
    unsigned long long S = carry_sum + sexcl;
    unsigned long long sbefore[kFIPT];
    int mycut = INT_MAX;
#pragma unroll
    for (int k = 0; k < kFIPT; ++k) {
      sbefore[k] = S;
      S += c[k];
      if (valid[k] && c[k] && S > b && mycut == INT_MAX) mycut = static_cast<int>(base + tid * kFIPT + k);
    }
    const int cut = RedI(tmp.ri).Reduce(mycut, cub::Min());
    if (tid == 0) s_cut = cut;
    __syncthreads();
    const int chunk_cut = s_cut;
    if (chunk_cut != INT_MAX && static_cast<int>(base + tid * kFIPT) <= chunk_cut &&
        chunk_cut < static_cast<int>(base + tid * kFIPT + kFIPT)) {
      s_sum_at_cut = sbefore[chunk_cut - (base + tid * kFIPT)] + c[chunk_cut - (base + tid * kFIPT)];
    }
    const long long limit = chunk_cut != INT_MAX ? chunk_cut : static_cast<long long>(base) + kFChunk - 1;
    int ne = 0, nt = 0, lastlu = -1;
#pragma unroll
    for (int k = 0; k < kFIPT; ++k) {
      const long long i = base + tid * kFIPT + k;
      if (!valid[k] || i > limit) continue;
      if (c[k]) ++ne;
      if (lu[k]) {
        ++nt;
        lastlu = static_cast<int>(i);
      }
      if (pr[k]) ++pruned;
    }
    int epos, etot;
    ScanI(tmp.si).ExclusiveSum(ne, epos, etot);
    __syncthreads();
    int tpos, ttot;
    ScanI(tmp.si).ExclusiveSum(nt, tpos, ttot);
    __syncthreads();
    if (look && chunk_cut != INT_MAX) {
      // lookahead for the round vote (merge kernel): the entry the NEXT
      // epoch would pop last if it were formed from this chunk now
      const unsigned long long lim2 = s_sum_at_cut + b;
      int mycut2 = INT_MAX;
#pragma unroll
      for (int k = 0; k < kFIPT; ++k) {
        const int i = static_cast<int>(base + tid * kFIPT + k);
        if (valid[k] && i > chunk_cut && c[k] && sbefore[k] + c[k] > lim2 && mycut2 == INT_MAX) mycut2 = i;
      }
      const int cut2 = RedI(tmp.ri).Reduce(mycut2, cub::Min());
      if (tid == 0) s_look = cut2 == INT_MAX ? ~0ull : qk[cut2];
      __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < kFIPT; ++k) {
      const long long i = base + tid * kFIPT + k;
      if (!valid[k] || i > limit) continue;
      if (c[k]) {
        exp_parent[carry_exp + epos] = key_seq(strategy, qk[i]);  // the parent's pool slot
        exp_off[carry_exp + epos] = static_cast<uint32_t>(sbefore[k]);
        ++epos;
      }
      if (lu[k]) {
        const unsigned long long t = carry_trace + tpos;
        if (t < trace_cap) trace[t] = nd[k].score;
        ++tpos;
      }
    }
    const int chunk_last = RedI(tmp.ri).Reduce(lastlu, cub::Max());
    if (tid == 0) s_lastlu = chunk_last;
    __syncthreads();
    if (s_lastlu >= 0) {
      best_i = s_lastlu;
      carry_best = pool[key_seq(strategy, qk[best_i])].score;  // leaf updates are non-decreasing
    }
    carry_exp += static_cast<uint32_t>(etot);
    carry_trace += static_cast<unsigned long long>(ttot);
    if (chunk_cut != INT_MAX) {
      carry_sum = s_sum_at_cut;
      consumed = static_cast<uint32_t>(chunk_cut) + 1;
      break;
    }
    carry_sum += stotal;
    if (strategy == BBS_STRATEGY_BFS) {
      // BFS pops in non-increasing score order and B never decreases, so
      // everything after the first pruned entry is pruned too (no children,
      // no leaf updates): the queue drains here without walking the rest.
      bool has_pr = false;
#pragma unroll
      for (int k = 0; k < kFIPT; ++k) has_pr |= valid[k] && pr[k];
      if (__syncthreads_or(has_pr)) {
        const uint32_t end = base + kFChunk;
        if (tid == 0 && qlen > end) pruned += qlen - end;
        break;
      }
    }
    __syncthreads();
  }
  __syncthreads();
  const unsigned long long pruned_all = cub::BlockReduce<unsigned long long, kFT>(tmp.ru).Sum(pruned);
  if (tid == 0 && cache_ctl) {
    cache_ctl[2] = 0;  // builds claimed this flush
    cache_ctl[3] = 0;  // runs listed for the cube kernel
    cache_ctl[kCtlDirect] = 0;
    cache_ctl[kCtlDirectItem] = 0;
    uint32_t raw = 0;
    for (int l = 0; l < kMaxLevels; ++l) raw |= cache_ctl[4 + l] ? 1u << l : 0u;
    st->cache_raw = raw;  // lets the host stop launching empty build kernels
  }
  if (tid == 0) {
    if (look) st->look_key = s_look;
    st->surv_ticket = 0;
    st->nodes_pruned += pruned_all;
    st->best = carry_best;
    st->flush_best = carry_best;
    st->trace_len = carry_trace;
    st->n_cons = consumed;
    st->n_expand = carry_exp;
    st->n_children = static_cast<uint32_t>(carry_sum);
    if (best_i >= 0) {
      st->best_node = pool[key_seq(strategy, qk[best_i])];
      st->matched = 1;
      st->last_best_epoch = static_cast<int32_t>(st->pass);
    }
    st->pass += 1;
    if (carry_sum == 0) {
      // queue drained with nothing pending: the loop ends (search.hpp:145)
      st->active = 0;
      st->q_len = 0;
    } else {
      st->nodes_generated += carry_sum;
      st->batches_flushed += 1;
      st->epochs += 1;
    }
  }
}

__global__ void __launch_bounds__(kFT) frontier_kernel(EpochState* st, Queue q, GridView G,
                                                       unsigned long long b,
                                                       uint32_t* __restrict__ exp_parent,
                                                       uint32_t* __restrict__ exp_off,
                                                       int32_t* __restrict__ trace,
                                                       unsigned long long trace_cap,
                                                       int strategy, uint32_t* __restrict__ cache_ctl) {
  frontier_kernel_body(st, q, G, b, exp_parent, exp_off, trace, trace_cap, strategy, cache_ctl);
}

// ---- speculative rounds (BFS) ----------------------------------------------
// Between two flushes nothing is pushed, and in BFS a flush's survivors only
// change later pops when their key precedes an entry those pops take.  A
// round therefore forms up to k consecutive epochs from the current queue as
// if no flush had survivors (frontier_spec_kernel; the incumbent B is carried
// through leaf pops exactly as in the sequential loop, so every prune is
// exact), branches and scores ALL their children with one launch of each
// kernel, and validates (survivors_spec_kernel): epoch j is kept only when no
// survivor of the kept epochs < j has a key below the last entry epoch j
// popped (a drain epoch: when those epochs had no survivors at all).  The
// kept epochs are a prefix; their Stats, trace and survivors are committed
// exactly as the sequential schedule makes them (search.hpp:132-169), the
// rest is discarded and re-formed by the next round from the true queue.
constexpr uint64_t kTraceStage = 256;  // incumbent-trace entries staged with every host check
constexpr int kSpecMax = 16;
struct SpecRec {
  unsigned long long lastkey;    // key of the epoch's last pop (its cut entry)
  unsigned long long pruned;     // pops pruned, cumulative over the round
  unsigned long long trace_end;  // trace length after the epoch
  unsigned long long minkey;     // smallest survivor key, seq taken as newest (survivors_spec_kernel; ~0 none)
  uint32_t child_end;            // children of epochs <= this one (pending offset end)
  uint32_t cons_end;             // queue entries consumed through this epoch
  uint32_t exp_end;              // expanding parents through this epoch
  uint32_t n_surv;               // survivors of the epoch (survivors_spec_kernel)
  int32_t B;                     // incumbent after the epoch's pops: its flush threshold
  int32_t best_i;                // queue index of the round's last leaf update through this epoch (-1)
  int32_t drained;               // 1: the queue ran out (drain flush, search.hpp:146-148)
  int32_t pad;
  uint32_t lv[kMaxLevels];       // the epoch's children per level (survivors_spec_kernel)
};

// per-pop counts packed for one block scan: pruned | leaf updates | expanding
__device__ __forceinline__ unsigned long long pack3(uint32_t pr, uint32_t lu, uint32_t ex) {
  return (static_cast<unsigned long long>(pr) << 42) | (static_cast<unsigned long long>(lu) << 21) | ex;
}

__device__ __forceinline__ void frontier_spec_kernel_body(EpochState* st,
                                                          Queue q,
                                                          const GridView& G,
                                                          unsigned long long b,
                                                          int k_max,
                                                          uint32_t* __restrict__ exp_parent,
                                                          uint32_t* __restrict__ exp_off,
                                                          int32_t* __restrict__ trace,
                                                          unsigned long long trace_cap,
                                                          uint32_t* __restrict__ cache_ctl,
                                                          SpecRec* __restrict__ rec,
                                                          int active_pre = -1) {
  pdl_wait();

  using ScanI = cub::BlockScan<int, kFT>;
  using ScanU = cub::BlockScan<unsigned long long, kFT>;
  using RedI = cub::BlockReduce<int, kFT>;
  __shared__ union {
    typename ScanI::TempStorage si;
    typename ScanU::TempStorage su;
    typename RedI::TempStorage ri;
  } tmp;
  __shared__ int s_i;
  __shared__ int s_active;
  __shared__ struct {
    unsigned long long S[kFChunk];  // inclusive children sums (round-global); ~0 past the queue
    unsigned long long C[kFChunk];  // inclusive packed counts (chunk)
    unsigned long long K[kFChunk];  // the chunk's queue keys (an epoch record's last key)
    int L[kFChunk];                 // last leaf update through the pop
    int Bk[kFChunk];                // incumbent after the pop
    int ep, limit;
    unsigned long long cut_base;
  } sh;

  const int tid = threadIdx.x;
  if (tid == 0) s_active = active_pre >= 0 ? active_pre : st->active;
  __syncthreads();
  if (!s_active) {
    if (tid == 0) {
      st->n_children = 0;
      st->spec_n = 0;
    }
    return;
  }
  const uint32_t qlen = st->q_len;
  const unsigned long long* __restrict__ qk = q.keys(st->cur);
  const bbs_node* __restrict__ pool = q.pool;
  k_max = max(1, min(k_max, static_cast<int>(st->spec_k)));  // adaptive depth of this round
  int carry_best = st->best;
  unsigned long long carry_sum = 0, carry_trace = st->trace_len, carry_pruned = 0;
  unsigned long long cut_base = 0;  // children of the epochs formed so far
  uint32_t carry_exp = 0;
  int carry_lu = -1;                // queue index of the round's last leaf update
  int ep = 0;

  // the next chunk's entries are loaded while this one is processed (a
  // round scans several chunks one after another: C3 ~6)
  bbs_node nd_next[kFIPT];
  unsigned long long key_next[kFIPT];
#pragma unroll
  for (int k = 0; k < kFIPT; ++k) {
    const uint32_t i = tid * kFIPT + k;
    key_next[k] = i < qlen ? qk[i] : ~0ull;
    if (i < qlen) nd_next[k] = pool[key_seq(BBS_STRATEGY_BFS, key_next[k])];
  }
  for (uint32_t base = 0; base < qlen && ep < k_max; base += kFChunk) {
    bbs_node nd[kFIPT];
    unsigned long long key[kFIPT];
    bool valid[kFIPT];
    int lm = INT_MIN;
#pragma unroll
    for (int k = 0; k < kFIPT; ++k) {
      const uint32_t i = base + tid * kFIPT + k;
      valid[k] = i < qlen;
      nd[k] = nd_next[k];
      key[k] = key_next[k];
      if (valid[k] && nd[k].level == 0) lm = max(lm, nd[k].score);
    }
#pragma unroll
    for (int k = 0; k < kFIPT; ++k) {
      const uint32_t i = base + kFChunk + tid * kFIPT + k;
      key_next[k] = i < qlen ? qk[i] : ~0ull;
      if (i < qlen) nd_next[k] = pool[key_seq(BBS_STRATEGY_BFS, key_next[k])];
    }
    int excl;
    ScanI(tmp.si).ExclusiveScan(lm, excl, INT_MIN, cub::Max());
    __syncthreads();
    int B = max(carry_best, excl);
    uint32_t c[kFIPT];
    bool pr[kFIPT], lu[kFIPT];
    int Bk[kFIPT];
    unsigned long long csum = 0, cnt = 0;
    int mylu = -1;
#pragma unroll
    for (int k = 0; k < kFIPT; ++k) {
      c[k] = 0;
      pr[k] = lu[k] = false;
      if (valid[k]) {
        const int sc = nd[k].score;
        pr[k] = sc < B;  // search.hpp:150-153
        const bool leaf = nd[k].level == 0;
        lu[k] = !pr[k] && leaf;  // search.hpp:154-160
        if (lu[k]) {
          B = sc;
          mylu = static_cast<int>(base + tid * kFIPT + k);
        }
        if (!pr[k] && !leaf) c[k] = n_children_of(G, nd[k]);
      }
      Bk[k] = B;  // the incumbent after this pop
      csum += c[k];
      cnt += pack3(pr[k] ? 1u : 0u, lu[k] ? 1u : 0u, c[k] ? 1u : 0u);
    }
    unsigned long long sexcl, stotal;
    ScanU(tmp.su).ExclusiveSum(csum, sexcl, stotal);
    __syncthreads();
    unsigned long long cexcl, ctotal;
    ScanU(tmp.su).ExclusiveSum(cnt, cexcl, ctotal);
    __syncthreads();
    int luexcl;
    ScanI(tmp.si).ExclusiveScan(mylu, luexcl, -1, cub::Max());
    __syncthreads();
    // inclusive per pop: children sum (round-global), packed counts, last leaf update
    unsigned long long Sin[kFIPT], Cin[kFIPT];
    int Lin[kFIPT];
    {
      unsigned long long S = carry_sum + sexcl, Cc = cexcl;
      int Lc = max(carry_lu, luexcl);
#pragma unroll
      for (int k = 0; k < kFIPT; ++k) {
        S += c[k];
        Cc += pack3(pr[k] ? 1u : 0u, lu[k] ? 1u : 0u, c[k] ? 1u : 0u);
        if (lu[k]) Lc = static_cast<int>(base + tid * kFIPT + k);
        Sin[k] = S;
        Cin[k] = Cc;
        Lin[k] = Lc;
      }
    }
    // successive cuts in this chunk: the first pop whose inclusive children
    // sum exceeds the previous cut's by more than b (search.hpp:166).  The
    // sums are non-decreasing, so warp 0 finds each cut with a 32-ary search
    // over the chunk's sums in shared memory (the first index past a sum is
    // a pop with children) and writes the epoch records.
#pragma unroll
    for (int k = 0; k < kFIPT; ++k) {
      const int li = tid * kFIPT + k;
      sh.S[li] = valid[k] ? Sin[k] : ~0ull;
      sh.C[li] = Cin[k];
      sh.K[li] = key[k];
      sh.L[li] = Lin[k];
      sh.Bk[li] = Bk[k];
    }
    __syncthreads();
    if (tid < 32) {
      const uint32_t lane = tid;
      const uint32_t nv = min(static_cast<uint32_t>(kFChunk), qlen - base);
      uint32_t lo = 0;
      int e = ep;
      unsigned long long cb = cut_base;
      int lim = kFChunk - 1;
      while (e < k_max && lo < nv) {
        // first li in [lo, nv) with S[li] > cb + b
        const unsigned long long x = cb + b;
        uint32_t l = lo, h = nv;
        while (l < h) {
          const uint32_t step = (h - l + 31u) >> 5;
          const uint32_t pos = l + (lane + 1u) * step - 1u;
          const bool le = pos < h && sh.S[pos] <= x;
          const uint32_t c = static_cast<uint32_t>(__popc(__ballot_sync(0xffffffffu, le)));
          const uint32_t nh = l + (c + 1u) * step - 1u;
          l += c * step;
          if (nh < h) h = nh;
        }
        if (l >= nv) break;
        if (lane == 0) {
          const unsigned long long Cc = sh.C[l];
          SpecRec r;
          r.lastkey = sh.K[l];
          r.pruned = carry_pruned + (Cc >> 42);
          r.trace_end = carry_trace + ((Cc >> 21) & 0x1FFFFFull);
          r.minkey = ~0ull;
          r.child_end = static_cast<uint32_t>(sh.S[l]);
          r.cons_end = base + l + 1u;
          r.exp_end = carry_exp + static_cast<uint32_t>(Cc & 0x1FFFFFull);
          r.n_surv = 0;
          r.B = sh.Bk[l];
          r.best_i = sh.L[l];
          r.drained = 0;
          r.pad = 0;
          for (int lv = 0; lv < kMaxLevels; ++lv) r.lv[lv] = 0;
          rec[e] = r;
        }
        cb = sh.S[l];
        lo = l + 1;
        ++e;
        if (e == k_max) lim = static_cast<int>(l);
      }
      if (lane == 0) {
        sh.ep = e;
        sh.cut_base = cb;
        sh.limit = lim;
      }
    }
    __syncthreads();
    ep = sh.ep;
    cut_base = sh.cut_base;
    const long long limit = static_cast<long long>(base) + sh.limit;  // pops this round emits
    __syncthreads();
    // expanding parents (branch inputs) and leaf updates (trace) of the pops
    // up to `limit`, at their round-global positions
#pragma unroll
    for (int k = 0; k < kFIPT; ++k) {
      const long long i = base + tid * kFIPT + k;
      if (!valid[k] || i > limit) continue;
      if (c[k]) {
        const uint32_t e = carry_exp + static_cast<uint32_t>(Cin[k] & 0x1FFFFFull) - 1u;
        exp_parent[e] = key_seq(BBS_STRATEGY_BFS, key[k]);  // the parent's pool slot
        exp_off[e] = static_cast<uint32_t>(Sin[k] - c[k]);
      }
      if (lu[k]) {
        const unsigned long long t = carry_trace + ((Cin[k] >> 21) & 0x1FFFFFull) - 1u;
        if (t < trace_cap) trace[t] = nd[k].score;
      }
    }
    if (ep == k_max) break;
    // the whole chunk belongs to the round: carry it
    carry_sum += stotal;
    carry_pruned += ctotal >> 42;
    carry_trace += (ctotal >> 21) & 0x1FFFFFull;
    carry_exp += static_cast<uint32_t>(ctotal & 0x1FFFFFull);
    {
      const int lmax = RedI(tmp.ri).Reduce(Lin[kFIPT - 1], cub::Max());
      if (tid == 0) s_i = lmax;
      __syncthreads();
      carry_lu = s_i;
      __syncthreads();
    }
    // the incumbent after the chunk: the last pop's B (non-decreasing)
    if (tid == kFT - 1) s_i = Bk[kFIPT - 1];
    __syncthreads();
    carry_best = s_i;
    __syncthreads();
    // BFS: the first pruned pop ends the queue (scores non-increasing, B never
    // decreases): all later pops are pruned, with no children
    bool has_pr = false;
#pragma unroll
    for (int k = 0; k < kFIPT; ++k) has_pr |= valid[k] && pr[k];
    if (__syncthreads_or(has_pr)) {
      const uint32_t end = base + kFChunk;
      if (qlen > end) carry_pruned += qlen - end;
      break;
    }
  }
  if (tid != 0) return;
  if (ep < k_max) {
    // the queue ran out (or only pruned pops remain) with the open epoch
    if (carry_sum > cut_base) {
      // its children are flushed on the drain (search.hpp:146-148)
      SpecRec r;
      r.lastkey = ~0ull;
      r.pruned = carry_pruned;
      r.trace_end = carry_trace;
      r.minkey = ~0ull;
      r.child_end = static_cast<uint32_t>(carry_sum);
      r.cons_end = qlen;
      r.exp_end = carry_exp;
      r.n_surv = 0;
      r.B = carry_best;
      r.best_i = carry_lu;
      r.drained = 1;
      r.pad = 0;
      for (int l = 0; l < kMaxLevels; ++l) r.lv[l] = 0;
      rec[ep] = r;
      ++ep;
    } else if (ep == 0) {
      // queue drained with nothing pending: the loop ends (search.hpp:145);
      // commit the last pops (prunes, leaf updates) here
      st->nodes_pruned += carry_pruned;
      st->best = carry_best;
      st->flush_best = carry_best;
      st->trace_len = carry_trace;
      if (carry_lu >= 0) {
        st->best_node = pool[key_seq(BBS_STRATEGY_BFS, qk[carry_lu])];
        st->matched = 1;
        st->last_best_epoch = static_cast<int32_t>(st->pass);
      }
      st->pass += 1;
      st->active = 0;
      st->q_len = 0;
      st->n_children = 0;
      st->spec_n = 0;
      return;
    }
    // else: the trailing pops (no children) are left to the next round
  }
  if (cache_ctl) {
    cache_ctl[2] = 0;  // builds claimed this flush
    cache_ctl[3] = 0;  // runs listed for the cube kernel
    cache_ctl[kCtlDirect] = 0;
    cache_ctl[kCtlDirectItem] = 0;
    uint32_t raw = 0;
    for (int l = 0; l < kMaxLevels; ++l) raw |= cache_ctl[4 + l] ? 1u << l : 0u;
    st->cache_raw = raw;
  }
  st->surv_ticket = 0;
  st->spec_n = static_cast<uint32_t>(ep);
  st->n_children = rec[ep - 1].child_end;  // every formed epoch's children are scored
  st->n_expand = rec[ep - 1].exp_end;
}

__global__ void __launch_bounds__(kFT) frontier_spec_kernel(EpochState* st, Queue q, GridView G,
                                                            unsigned long long b, int k_max,
                                                            uint32_t* __restrict__ exp_parent,
                                                            uint32_t* __restrict__ exp_off,
                                                            int32_t* __restrict__ trace,
                                                            unsigned long long trace_cap,
                                                            uint32_t* __restrict__ cache_ctl,
                                                            SpecRec* __restrict__ rec) {
  frontier_spec_kernel_body(st, q, G, b, k_max, exp_parent, exp_off, trace, trace_cap, cache_ctl, rec);
}

// E2: branch() (nodes.hpp:91-121) for every expanding parent, children in
// pop order, each parent's children in (jr, jp, jw, jx, jy, jz) order.
// Batch-split exact mode: the flush's runs of 8 children are
// dealt round-robin over the ranks; this rank scores its runs from a compact
// copy (pending_own) and the scores are scattered back and max-all-reduced.
struct RunSplit {
  bbs_node* pending_own;
  int32_t* pscores_own;
  uint32_t rank, world;  // world == 0: no split
};

__device__ __forceinline__ uint32_t own_children(uint32_t n, uint32_t rank, uint32_t world) {
  const uint32_t runs = n >> 3;
  return runs > rank ? ((runs - rank + world - 1) / world) * 8u : 0u;
}

__device__ __forceinline__ void branch_kernel_body(EpochState* st,
                                                   Queue q,
                                                   const GridView& G,
                                                   const uint32_t* __restrict__ exp_parent,
                                                   const uint32_t* __restrict__ exp_off,
                                                   bbs_node* __restrict__ pending,
                                                   int32_t* __restrict__ pscores,
                                                   const RotCache& cache,
                                                   RunSplit split) {
  pdl_wait();

  const uint32_t n = st->n_children;
  // read with the state above (one round trip), not per run
  const bool direct_on = cache.direct_flag && (!cache.direct_gate || *cache.direct_gate);
  if (split.world && blockIdx.x == 0 && threadIdx.x == 0) st->n_own = own_children(n, split.rank, split.world);
  if (n == 0) return;
  const uint32_t ne = st->n_expand;
  const bbs_node* __restrict__ pool = q.pool;
  const uint32_t lane = threadIdx.x & 31u;
  // warps take 32 consecutive children: lane 0 binary-searches the first
  // one's parent, the lanes step forward from it (a parent has >= 8
  // children, so a warp spans at most 5 parents)
  for (uint32_t w0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); w0 < n; w0 += gridDim.x * blockDim.x) {
    uint32_t m0 = 0;
    if (lane == 0) {
      uint32_t lo = 0, hi = ne - 1;  // largest m with exp_off[m] <= w0
      while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (exp_off[mid] <= w0)
          lo = mid;
        else
          hi = mid - 1;
      }
      m0 = lo;
    }
    m0 = __shfl_sync(0xffffffffu, m0, 0);
    const uint32_t i = w0 + lane;
    if (i >= n) continue;
    uint32_t lo = m0;
    while (lo + 1 < ne && exp_off[lo + 1] <= i) ++lo;
    const bbs_node p = pool[exp_parent[lo]];
    const uint32_t local = i - exp_off[lo];
    int32_t a[3], c[3];
    child_counts(G, p, a, c);
    const uint32_t kk = local >> 3, t = local & 7u;
    const int32_t jw = static_cast<int32_t>(kk % c[2]);
    const int32_t jp = static_cast<int32_t>((kk / c[2]) % c[1]);
    const int32_t jr = static_cast<int32_t>(kk / (c[2] * c[1]));
    bbs_node ch;
    ch.ix = 2 * p.ix + static_cast<int32_t>(t >> 2);
    ch.iy = 2 * p.iy + static_cast<int32_t>((t >> 1) & 1u);
    ch.iz = 2 * p.iz + static_cast<int32_t>(t & 1u);
    ch.iroll = a[0] * p.iroll + jr;
    ch.ipitch = a[1] * p.ipitch + jp;
    ch.iyaw = a[2] * p.iyaw + jw;
    ch.level = p.level - 1;
    ch.score = -1;
    pending[i] = ch;
    bool own = true;
    if (split.world) {
      const uint32_t run = i >> 3;
      own = run % split.world == split.rank;
      pscores[i] = -1;  // other ranks' runs: filled by the max-all-reduce
      if (own) {
        const uint32_t j = (run / split.world) * 8u + t;
        split.pending_own[j] = ch;
        split.pscores_own[j] = 0;
      }
    } else {
      pscores[i] = 0;  // the flush kernels accumulate into it
    }
    // first child of a run (8 translation siblings): claim its rotation's
    // histogram slot (epoch_cache.cu), or list the run as direct when it can
    // have no histogram this flush
    if (cache.enabled && t == 0 && own) {
      const int4 ra = make_int4(ch.ix, ch.iy, ch.iz, ch.iroll), rb = make_int4(ch.ipitch, ch.iyaw, ch.level, ch.score);
      if (direct_on) {
        // the run's index in the array the score kernels read (exact mode:
        // this rank's compact copy)
        const uint32_t r = split.world ? (i >> 3) / split.world : (i >> 3);
        const bool direct = run_is_direct(cache, G, ra, rb);
        cache.direct_flag[r] = direct ? 1 : 0;
        if (direct) cache.direct_runs[atomicAdd(&cache.ctl[kCtlDirect], 1u)] = r;
        if (!direct) cache_claim_run(cache, G, ra, rb);
      } else {
        cache_claim_run(cache, G, ra, rb);
      }
    }
  }
}

__global__ void branch_kernel(EpochState* st, Queue q, GridView G,
                              const uint32_t* __restrict__ exp_parent,
                              const uint32_t* __restrict__ exp_off, bbs_node* __restrict__ pending,
                              int32_t* __restrict__ pscores, RotCache cache, RunSplit split) {
  branch_kernel_body(st, q, G, exp_parent, exp_off, pending, pscores, cache, split);
}

constexpr int kST = 256;   // survivors: threads per tile
constexpr int kSIPT = 8;  // items per thread (2048 per tile)
constexpr int kSTile = kST * kSIPT;

__device__ __forceinline__ uint32_t lower_bound_u64(const unsigned long long* a, uint32_t n,
                                                    unsigned long long v) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// First index i in [0, n) with a[i] >= v (n if none), searched by the whole
// warp (uniform arguments): each round the 32 lanes probe 32 evenly spaced
// positions, so a queue of ~500k keys takes 4 dependent rounds instead of 19.
__device__ __forceinline__ uint32_t warp_lower_bound_u64(const unsigned long long* __restrict__ a, uint32_t n,
                                                         unsigned long long v) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t lo = 0, hi = n;  // a[i] < v for i < lo, a[i] >= v for i >= hi
  while (lo < hi) {
    const uint32_t step = (hi - lo + 31u) >> 5;
    const uint32_t pos = lo + (lane + 1u) * step - 1u;
    const bool less = pos < hi && a[pos] < v;
    const uint32_t c = static_cast<uint32_t>(__popc(__ballot_sync(0xffffffffu, less)));
    const uint32_t nhi = lo + (c + 1u) * step - 1u;
    lo += c * step;
    if (nhi < hi) hi = nhi;
  }
  return lo;
}

// Incumbent trim (one warp).  B never decreases, so a queued entry with
// score < B is pruned whenever it is popped (search.hpp:150-153) and never
// branches or updates the incumbent: dropping it now and counting it as
// pruned leaves Stats, trace and every later pop unchanged.  Within a key
// segment (BFS: the whole key space; DFS: one level) entries are ordered by
// descending score, so the dropped entries form a suffix of each segment.
__device__ void trim_remainder(EpochState* st, const Queue& q, int strategy, int32_t B) {
  const int lane = threadIdx.x & 31;
  const uint32_t n_cons = st->n_cons;
  const uint32_t n_rem = st->q_len - n_cons;
  const unsigned long long* qk = q.keys(st->cur) + n_cons;
  const int nseg = strategy == BBS_STRATEGY_BFS ? 1 : kMaxLevels;
  uint32_t lo = 0, hi = 0;
  if (strategy == BBS_STRATEGY_BFS) {
    // one segment: the whole warp searches it (log32 rounds of L2 latency)
    const unsigned long long sb = kSMax - static_cast<unsigned long long>(B < 0 ? 0 : B) + 1;
    const uint32_t h = B > 0 ? warp_lower_bound_u64(qk, n_rem, sb << 44) : n_rem;
    hi = lane == 0 ? h : 0;
  } else if (lane < nseg) {
    unsigned long long seg_base = 0, seg_end_key = ~0ull, cut_key;
    const unsigned long long sb = kSMax - static_cast<unsigned long long>(B < 0 ? 0 : B) + 1;
    if (strategy == BBS_STRATEGY_BFS) {
      cut_key = sb << 44;  // keys below: score >= B
      lo = 0;
      hi = n_rem;
    } else {
      seg_base = static_cast<unsigned long long>(lane) << 60;
      seg_end_key = lane + 1 < kMaxLevels ? static_cast<unsigned long long>(lane + 1) << 60 : ~0ull;
      cut_key = seg_base | (sb << 40);
      lo = lower_bound_u64(qk, n_rem, seg_base);
      hi = lane + 1 < kMaxLevels ? lower_bound_u64(qk, n_rem, seg_end_key) : n_rem;
    }
    if (B > 0) hi = lo + lower_bound_u64(qk + lo, hi - lo, cut_key);
  }
  const uint32_t len = hi - lo;
  uint32_t pre = len;  // inclusive scan over lanes
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, pre, d);
    if (lane >= d) pre += v;
  }
  const uint32_t kept = __shfl_sync(0xffffffffu, pre, 31);
  if (lane < kMaxLevels) {
    st->seg_lo[lane] = lo;
    st->seg_len[lane] = len;
    st->seg_pre[lane] = pre - len;
  }
  if (lane == 0) {
    st->seg_pre[kMaxLevels] = kept;
    st->n_keep = kept;
    atomicAdd(&st->nodes_pruned, static_cast<unsigned long long>(n_rem - kept));
  }
}

// Decoupled look-back by one whole warp (ordered compaction across tiles):
// tile `tile` publishes its aggregate `tot`, then the 32 lanes read 32
// predecessor words at a time, stop at the nearest inclusive prefix and sum
// the aggregates after it; returns the exclusive prefix of `tile` and
// publishes the inclusive one.  Words: tag | status << 32 | value (status 1
// aggregate, 2 inclusive); tile 0 is inclusive at once, so the walk ends.
__device__ uint32_t warp_lookback(unsigned long long* tiles, uint32_t tile, uint32_t tot,
                                  unsigned long long tag) {
  const uint32_t lane = threadIdx.x & 31u;
  constexpr unsigned long long kTagMask = ~((1ull << 34) - 1);
  if (tile == 0) {
    if (lane == 0) atomicExch(&tiles[0], tag | (2ull << 32) | tot);
    return 0;
  }
  if (lane == 0) atomicExch(&tiles[tile], tag | (1ull << 32) | tot);
  uint32_t excl = 0;
  int64_t t = static_cast<int64_t>(tile) - 1;  // the window is tiles t, t-1, ..., t-31
  for (;;) {
    const int64_t j = t - static_cast<int64_t>(lane);
    unsigned long long w = 0;
    bool pub = true;
    if (j >= 0) {
      w = atomicAdd(&tiles[j], 0ull);
      pub = (w & kTagMask) == tag;
    }
    const unsigned incl = __ballot_sync(0xffffffffu, j >= 0 && pub && ((w >> 32) & 3u) == 2u);
    const unsigned unpub = __ballot_sync(0xffffffffu, j >= 0 && !pub);
    const int stop = incl ? __ffs(incl) - 1 : 31;  // lanes 0..stop are needed
    const unsigned need = stop == 31 ? 0xffffffffu : ((2u << stop) - 1u);
    if (unpub & need) continue;  // a needed predecessor has not published yet
    uint32_t v = (j >= 0 && static_cast<int>(lane) <= stop) ? static_cast<uint32_t>(w) : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (incl) break;
    t -= 32;
  }
  if (lane == 0) atomicExch(&tiles[tile], tag | (2ull << 32) | (excl + tot));
  return excl;
}

// E4a: flush pruning (search.hpp:134-140): keep score >= B in pending order
// and give them consecutive seq numbers.  Single-pass ordered compaction:
// tiles take tickets in order and chain their prefix through `tiles`
// (decoupled look-back; words tagged with the epoch so nothing is cleared).
// Block 0's first warp also trims the queue remainder.
__device__ __forceinline__ void survivors_kernel_body(EpochState* st,
                                                      Queue q,
                                                      int strategy,
                                                      const bbs_node* __restrict__ pending,
                                                      const int32_t* __restrict__ scores,
                                                      unsigned long long* __restrict__ s_key,
                                                      unsigned long long* __restrict__ tiles) {
  pdl_wait();

  using Load = cub::BlockLoad<int32_t, kST, kSIPT, cub::BLOCK_LOAD_WARP_TRANSPOSE>;
  using ScanI = cub::BlockScan<int, kST>;
  __shared__ union {
    typename Load::TempStorage load;
    typename ScanI::TempStorage scan;
  } tmp;
  __shared__ uint32_t s_tile, s_excl;
  __shared__ uint32_t s_lv[kMaxLevels];  // evaluations per level, this CTA
  if (threadIdx.x < kMaxLevels) s_lv[threadIdx.x] = 0;
  const uint32_t n = st->n_children;
  if (n == 0) return;
  const int32_t B = st->flush_best;
  const unsigned long long seq0 = st->seq;
  const unsigned long long tag = static_cast<unsigned long long>(st->pass & 0x3FFFFFFFu) << 34;
  if (blockIdx.x == 0 && threadIdx.x < 32) trim_remainder(st, q, strategy, B);
  const uint32_t n_tiles = (n + kSTile - 1) / kSTile;
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&st->surv_ticket, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= n_tiles) {
      if (threadIdx.x < kMaxLevels && s_lv[threadIdx.x])
        atomicAdd(&st->level_evals[threadIdx.x], static_cast<unsigned long long>(s_lv[threadIdx.x]));
      break;
    }
    const uint32_t base = tile * kSTile;
    const uint32_t valid = min(static_cast<uint32_t>(kSTile), n - base);
    int32_t sc[kSIPT];
    Load(tmp.load).Load(scores + base, sc, static_cast<int>(valid), INT_MIN);
    __syncthreads();
    // runs of 8 share a level; a thread holds kSIPT / 8 whole runs
    static_assert(kSIPT % 8 == 0, "tile rows must hold whole runs");
#pragma unroll
    for (int rr = 0; rr < kSIPT / 8; ++rr) {
      const uint32_t li = threadIdx.x * kSIPT + rr * 8;
      const int lvl = li < valid ? pending[base + li].level & (kMaxLevels - 1) : -1;
      const unsigned same = __match_any_sync(0xffffffffu, lvl);
      if (lvl >= 0 && (__ffs(same) - 1) == (threadIdx.x & 31)) atomicAdd(&s_lv[lvl], 8u * __popc(same));
    }
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < kSIPT; ++k) {
      if (threadIdx.x * kSIPT + k >= valid) sc[k] = INT_MIN;
      cnt += sc[k] >= B ? 1 : 0;
    }
    int pos, tot;
    ScanI(tmp.scan).ExclusiveSum(cnt, pos, tot);
    if (threadIdx.x < 32) {
      const uint32_t excl = warp_lookback(tiles, tile, static_cast<uint32_t>(tot), tag);
      if (threadIdx.x == 0) s_excl = excl;
      if (threadIdx.x == 0 && tile == n_tiles - 1) {
        const uint32_t kept = excl + static_cast<uint32_t>(tot);
        st->n_surv = kept;
        st->seq = seq0 + kept;
        atomicAdd(&st->nodes_pruned, static_cast<unsigned long long>(n - kept));
      }
    }
    __syncthreads();
    uint32_t o = s_excl + static_cast<uint32_t>(pos);
#pragma unroll
    for (int k = 0; k < kSIPT; ++k) {
      if (sc[k] < B || threadIdx.x * kSIPT + k >= valid) continue;
      const uint32_t i = base + threadIdx.x * kSIPT + k;
      bbs_node nd = pending[i];
      nd.score = sc[k];
      q.pool[seq0 + o] = nd;  // push: the node's permanent slot
      s_key[o] = queue_key(strategy, nd.score, nd.level, seq0 + o);
      ++o;
    }
  }
}

__global__ void __launch_bounds__(kST) survivors_kernel(EpochState* st, Queue q, int strategy,
                                                        const bbs_node* __restrict__ pending,
                                                        const int32_t* __restrict__ scores,
                                                        unsigned long long* __restrict__ s_key,
                                                        unsigned long long* __restrict__ tiles) {
  survivors_kernel_body(st, q, strategy, pending, scores, s_key, tiles);
}


// E4a, speculative round: survivors of EVERY formed epoch (each against its
// own B) compacted in pending order -- the kept epochs' survivors are a
// prefix of them -- while each tile adds its per-epoch survivor count, its
// smallest survivor key and its per-(epoch, level) evaluations to the round
// records BEFORE publishing its look-back aggregate; the last tile then
// holds every tile's contribution, validates the round (epoch j kept while
// no kept survivor precedes its last pop; a drain epoch only without
// earlier survivors) and commits the kept epochs into EpochState exactly as
// the sequential loop would have (search.hpp:132-169).  The queue trim runs
// in the next kernel (it needs the committed B and consumed count).
__device__ __forceinline__ void survivors_spec_kernel_body(EpochState* st,
                                                           Queue q,
                                                           const bbs_node* __restrict__ pending,
                                                           const int32_t* __restrict__ scores,
                                                           unsigned long long* __restrict__ s_key,
                                                           unsigned long long* __restrict__ tiles,
                                                           SpecRec* __restrict__ rec) {
  pdl_wait();

  using Load = cub::BlockLoad<int32_t, kST, kSIPT, cub::BLOCK_LOAD_WARP_TRANSPOSE>;
  using ScanI = cub::BlockScan<int, kST>;
  __shared__ union {
    typename Load::TempStorage load;
    typename ScanI::TempStorage scan;
  } tmp;
  __shared__ uint32_t s_tile, s_excl;
  __shared__ uint32_t s_end[kSpecMax];
  __shared__ int32_t s_B[kSpecMax];
  __shared__ unsigned long long s_min[kSpecMax];
  __shared__ uint32_t s_cnt[kSpecMax];
  __shared__ uint32_t s_lv[kSpecMax * kMaxLevels];
  const uint32_t ne = st->spec_n;
  if (ne == 0) return;  // nothing formed: the search ended in the frontier
  if (threadIdx.x < ne) {
    s_end[threadIdx.x] = rec[threadIdx.x].child_end;
    s_B[threadIdx.x] = rec[threadIdx.x].B;
  }
  const uint32_t n = st->n_children;  // every formed epoch's children
  const unsigned long long seq0 = st->seq;
  // look-back tag of this round: never 0 (the zeroed tile words), and the
  // round's pass is only incremented by the commit below
  const unsigned long long tag = static_cast<unsigned long long>(st->pass % 0x3FFFFFFFu + 1u) << 34;
  const uint32_t n_tiles = (n + kSTile - 1) / kSTile;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_tile = atomicAdd(&st->surv_ticket, 1u);
    if (threadIdx.x < kSpecMax) {
      s_min[threadIdx.x] = ~0ull;
      s_cnt[threadIdx.x] = 0;
    }
    for (int t = threadIdx.x; t < kSpecMax * kMaxLevels; t += kST) s_lv[t] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= n_tiles) break;
    const uint32_t base = tile * kSTile;
    const uint32_t valid = min(static_cast<uint32_t>(kSTile), n - base);
    int32_t sc[kSIPT];
    Load(tmp.load).Load(scores + base, sc, static_cast<int>(valid), INT_MIN);
    __syncthreads();
    // each thread's kSIPT items lie in at most a few epochs (boundaries are
    // multiples of 8, the runs of one parent's translation cube)
    uint32_t ek[kSIPT];
    int cnt = 0;
    {
      uint32_t e = 0;
#pragma unroll
      for (int k = 0; k < kSIPT; ++k) {
        const uint32_t i = base + threadIdx.x * kSIPT + k;
        if (threadIdx.x * kSIPT + k >= valid) sc[k] = INT_MIN;
        while (e + 1 < ne && s_end[e] <= i) ++e;
        ek[k] = e;
        cnt += sc[k] >= s_B[e] ? 1 : 0;
      }
    }
    static_assert(kSIPT % 8 == 0, "tile rows must hold whole runs");
#pragma unroll
    for (int rr = 0; rr < kSIPT / 8; ++rr) {
      const uint32_t li = threadIdx.x * kSIPT + rr * 8;
      const int lvl = li < valid ? static_cast<int>(ek[rr * 8] * kMaxLevels) + (pending[base + li].level & (kMaxLevels - 1)) : -1;
      const unsigned same = __match_any_sync(0xffffffffu, lvl);
      if (lvl >= 0 && (__ffs(same) - 1) == (threadIdx.x & 31)) atomicAdd(&s_lv[lvl], 8u * __popc(same));
    }
#pragma unroll
    for (int k = 0; k < kSIPT; ++k) {
      if (threadIdx.x * kSIPT + k >= valid || sc[k] < s_B[ek[k]]) continue;
      const uint32_t i = base + threadIdx.x * kSIPT + k;
      // a survivor's seq is newer than every queued entry's
      atomicMin(&s_min[ek[k]], queue_key(BBS_STRATEGY_BFS, sc[k], pending[i].level, kSeqMax));
      atomicAdd(&s_cnt[ek[k]], 1u);
    }
    __syncthreads();
    // this tile's contributions to the round records, then its aggregate
    {
      bool wrote = false;
      if (threadIdx.x < ne && s_cnt[threadIdx.x]) {
        atomicMin(&rec[threadIdx.x].minkey, s_min[threadIdx.x]);
        atomicAdd(&rec[threadIdx.x].n_surv, s_cnt[threadIdx.x]);
        wrote = true;
      }
      for (int t = threadIdx.x; t < static_cast<int>(ne) * kMaxLevels; t += kST)
        if (s_lv[t]) {
          atomicAdd(&rec[t / kMaxLevels].lv[t % kMaxLevels], s_lv[t]);
          wrote = true;
        }
      if (wrote) __threadfence();  // before this tile's aggregate is published
    }
    __syncthreads();
    int pos, tot;
    ScanI(tmp.scan).ExclusiveSum(cnt, pos, tot);
    if (threadIdx.x < 32) {
      const uint32_t excl = warp_lookback(tiles, tile, static_cast<uint32_t>(tot), tag);
      if (threadIdx.x == 0) s_excl = excl;
      if (tile == n_tiles - 1) {
        // every tile published after adding to the records: validate and
        // commit, warp-parallel (lane e reads epoch e's record)
        __threadfence();
        const uint32_t lane = threadIdx.x;
        const bool has = lane < ne;
        const uint32_t ns = has ? __ldcg(&rec[lane].n_surv) : 0u;
        const unsigned long long mk = has ? __ldcg(&rec[lane].minkey) : ~0ull;
        const unsigned long long lk = has ? __ldcg(&rec[lane].lastkey) : 0ull;
        const int dr = has ? __ldcg(&rec[lane].drained) : 0;
        // epoch j > 0 is overtaken when a survivor of an earlier epoch
        // precedes its last pop (drain epoch: any earlier survivor)
        unsigned long long pm = mk;  // inclusive prefix min of the survivor keys
        uint32_t ps = ns;            // inclusive prefix sum of the survivor counts
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const unsigned long long om = __shfl_up_sync(0xffffffffu, pm, d);
          const uint32_t os = __shfl_up_sync(0xffffffffu, ps, d);
          if (static_cast<int>(lane) >= d) {
            pm = min(pm, om);
            ps += os;
          }
        }
        const unsigned long long pm_before = __shfl_up_sync(0xffffffffu, pm, 1);
        const uint32_t ps_before = __shfl_up_sync(0xffffffffu, ps, 1);
        const bool bad = has && lane > 0 && (dr ? ps_before != 0 : !(pm_before > lk));
        const unsigned badm = __ballot_sync(0xffffffffu, bad);
        const uint32_t A = badm ? static_cast<uint32_t>(__ffs(badm) - 1) : ne;
        const uint32_t S_acc = __shfl_sync(0xffffffffu, ps, A - 1);
        // per-level evaluations of the kept epochs: lane l sums level l
        if (lane < kMaxLevels) {
          unsigned long long v = 0;
          for (uint32_t e = 0; e < A; ++e) v += __ldcg(&rec[e].lv[lane]);
          if (v) st->level_evals[lane] += v;
        }
        if (lane == 0) {
          const SpecRec& r = rec[A - 1];
          const uint32_t child_acc = r.child_end;
          st->spec_acc = A;
          st->n_surv = S_acc;
          st->seq = seq0 + S_acc;
          st->n_children = child_acc;
          st->n_cons = r.cons_end;
          st->n_expand = r.exp_end;
          st->nodes_pruned += r.pruned + (child_acc - S_acc);
          st->best = r.B;
          st->flush_best = r.B;
          st->trace_len = r.trace_end;
          if (r.best_i >= 0) {
            st->best_node = q.pool[key_seq(BBS_STRATEGY_BFS, q.keys(st->cur)[r.best_i])];
            st->matched = 1;
            st->last_best_epoch = static_cast<int32_t>(st->pass);
          }
          st->pass += 1;
          st->nodes_generated += child_acc;
          st->batches_flushed += A;
          st->epochs += A;
          // depth of the next round: double after a fully kept round, else
          // one more than this round kept (a discarded epoch costs its
          // scoring; a kept one saves a whole kernel chain)
          st->spec_k = A == ne ? min(2u * st->spec_k, st->spec_kmax) : min(A + 1u, st->spec_kmax);
        }
      }
    }
    __syncthreads();
    uint32_t o = s_excl + static_cast<uint32_t>(pos);
#pragma unroll
    for (int k = 0; k < kSIPT; ++k) {
      if (sc[k] < s_B[ek[k]] || threadIdx.x * kSIPT + k >= valid) continue;
      const uint32_t i = base + threadIdx.x * kSIPT + k;
      bbs_node c = pending[i];
      c.score = sc[k];
      q.pool[seq0 + o] = c;  // push: the node's permanent slot (kept prefix only survives)
      s_key[o] = queue_key(BBS_STRATEGY_BFS, c.score, c.level, seq0 + o);
      ++o;
    }
  }
}

__global__ void __launch_bounds__(kST) survivors_spec_kernel(EpochState* st, Queue q,
                                                             const bbs_node* __restrict__ pending,
                                                             const int32_t* __restrict__ scores,
                                                             unsigned long long* __restrict__ s_key,
                                                             unsigned long long* __restrict__ tiles,
                                                             SpecRec* __restrict__ rec) {
  survivors_spec_kernel_body(st, q, pending, scores, s_key, tiles, rec);
}

// E4b: order the survivors by key.  Keys are unique (they embed seq), so a
// survivor's rank = #keys below it; ranks are computed against smem tiles.
// Up to kMergeSortSmall survivors (C2: 14-107 per flush) are left to the
// merge kernel, whose CTAs each rank them in shared memory.
constexpr int kRT = 256;
constexpr uint32_t kMergeSortSmall = 256;
__device__ __forceinline__ void rank_sort_kernel_body(EpochState* st,
                                                      const unsigned long long* __restrict__ key,
                                                      unsigned long long* __restrict__ out_key,
                                                      Queue q,
                                                      int trim_strategy) {
  pdl_wait();

  __shared__ unsigned long long tile[kRT];
  // speculative rounds: the incumbent trim of the queue remainder runs here,
  // after survivors_spec_kernel committed the round (trim_strategy >= 0)
  if (trim_strategy >= 0 && blockIdx.x == 0 && threadIdx.x < 32 && st->n_children)
    trim_remainder(st, q, trim_strategy, st->flush_best);
  const uint32_t n = st->n_children ? st->n_surv : 0;
  if (n <= kMergeSortSmall) return;  // the merge kernel sorts these itself (none: nothing to do)
  for (uint32_t base = blockIdx.x * kRT; base < n; base += gridDim.x * kRT) {
    const uint32_t j = base + threadIdx.x;
    const unsigned long long kj = j < n ? key[j] : ~0ull;
    uint32_t rank = 0;
    for (uint32_t t0 = 0; t0 < n; t0 += kRT) {
      __syncthreads();
      tile[threadIdx.x] = (t0 + threadIdx.x < n) ? key[t0 + threadIdx.x] : ~0ull;
      __syncthreads();
      const uint32_t lim = min(static_cast<uint32_t>(kRT), n - t0);
#pragma unroll 8
      for (uint32_t i = 0; i < lim; ++i) rank += tile[i] < kj ? 1u : 0u;
    }
    if (j < n) out_key[rank] = kj;
  }
}

__global__ void __launch_bounds__(kRT) rank_sort_kernel(EpochState* st,
                                                        const unsigned long long* __restrict__ key,
                                                        unsigned long long* __restrict__ out_key,
                                                        Queue q, int trim_strategy) {
  rank_sort_kernel_body(st, key, out_key, q, trim_strategy);
}

// E4b': large flushes (batch_size above kRankSortMax): the unused tail of
// the survivor keys is set to the largest key and the whole buffer goes
// through a CUB radix sort (O(n) instead of rank_sort's O(n^2)).
constexpr uint64_t kRankSortMax = 16384;
__global__ void pad_keys_kernel(EpochState* st, unsigned long long* __restrict__ key, uint64_t cap, Queue q,
                                int trim_strategy) {
  pdl_wait();
  if (trim_strategy >= 0 && blockIdx.x == 0 && threadIdx.x < 32 && st->n_children)
    trim_remainder(st, q, trim_strategy, st->flush_best);
  const uint64_t n = st->n_children ? st->n_surv : 0;
  for (uint64_t i = n + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < cap; i += uint64_t(gridDim.x) * blockDim.x)
    key[i] = ~0ull;
}

// E6: merge the sorted survivors into the trimmed queue remainder (push,
// search.hpp:139).  The remainder A is read through the kept segment ranges
// (one per key segment); the survivors B are sorted; keys are unique.  Keys
// only (nodes stay in the pool).  Merge path: each CTA owns kMTile outputs,
// two warps find the tile's diagonal splits with 32-ary searches, the tile's
// A and B ranges are staged in shared memory and each thread merges 8
// outputs from its own in-tile split.
constexpr uint32_t kMT = 256, kMItems = 8, kMTile = kMT * kMItems;

struct RemView {
  const unsigned long long* qk;
  const uint32_t* lo;   // smem: segment start in qk
  const uint32_t* pre;  // smem: segment start in the kept order (kMaxLevels + 1)
  bool bfs;
  __device__ __forceinline__ unsigned long long operator[](uint32_t i) const {
    int sg = 0;
    if (!bfs)
      while (pre[sg + 1] <= i) ++sg;
    return qk[lo[sg] + (i - pre[sg])];
  }
};

// #A elements among the first d merged outputs (warp-uniform arguments).
__device__ __forceinline__ uint32_t warp_merge_split(const RemView& A, uint32_t na,
                                                     const unsigned long long* __restrict__ B, uint32_t nb,
                                                     uint32_t d) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t lo = d > nb ? d - nb : 0u, hi = min(d, na);  // P(a) = A[a] < B[d-1-a], true below the answer
  while (lo < hi) {
    const uint32_t step = (hi - lo + 31u) >> 5;
    const uint32_t a = lo + (lane + 1u) * step - 1u;
    const bool p = a < hi && A[a] < B[d - 1u - a];
    const uint32_t c = static_cast<uint32_t>(__popc(__ballot_sync(0xffffffffu, p)));
    const uint32_t nhi = lo + (c + 1u) * step - 1u;
    lo += c * step;
    if (nhi < hi) hi = nhi;
  }
  return lo;
}

// fused: this kernel also does the rank-sort kernel's work first (the
// incumbent trim of a round, trim >= 0 or -2 = by st->spec_mode; the rank
// sort of more than kMergeSortSmall survivors into sorted_key), one launch
// less per flush.  That work is split into tasks (trim, then one per tile of
// kMT keys; above st->tile_rank_min survivors two per tile: the tiles sorted
// in place in unsorted_key, then ranked against each other) that CTAs claim
// with an atomic counter; a CTA waits only for tasks already claimed by
// running CTAs, so the wait cannot starve whatever share of the grid is
// resident (other searches on other streams included).
__device__ __forceinline__ void merge_kernel_body(EpochState* st,
                                                  Queue q,
                                                  int strategy,
                                                  const unsigned long long* sorted_key,
                                                  const unsigned long long* unsorted_key,
                                                  int vote = 0, bool fused = false, int trim = -1) {
  pdl_wait();

  __shared__ uint32_t s_lo[kMaxLevels], s_pre[kMaxLevels + 1];
  __shared__ uint32_t s_split[2];
  __shared__ unsigned long long s_ab[kMTile];
  if (st->n_children == 0) return;
  if (fused) {
    if (trim == -2) trim = st->spec_mode ? strategy : -1;
    const uint32_t n = st->n_surv;
    const uint32_t n_trim = trim >= 0 ? 1u : 0u;
    const uint32_t n_tiles = (n + kMT - 1u) / kMT;
    // many survivors (a deep round): sort every tile in place first, then
    // rank each key by binary searches in the other sorted tiles, n^2/32
    // shared-memory reads instead of n^2 compares
    const bool tiled = n > st->tile_rank_min;
    const uint32_t tasks = n_trim + (n > kMergeSortSmall ? (tiled ? 2u : 1u) * n_tiles : 0u);
    if (tasks) {
      __shared__ uint32_t s_task;
      unsigned long long* out = const_cast<unsigned long long*>(sorted_key);
      for (;;) {
        if (threadIdx.x == 0) {  // no atomic once every task is out (most of the grid)
          const uint32_t c = *reinterpret_cast<volatile uint32_t*>(&st->fuse_claim);
          s_task = c >= tasks ? c : atomicAdd(&st->fuse_claim, 1u);
        }
        __syncthreads();
        const uint32_t t = s_task;
        __syncthreads();
        if (t >= tasks) break;
        bool phase_a = false;
        if (t < n_trim) {
          if (threadIdx.x < 32) trim_remainder(st, q, trim, st->flush_best);
        } else if (tiled) {
          unsigned long long* keys = const_cast<unsigned long long*>(unsorted_key);
          const uint32_t u = t - n_trim;
          if (u < n_tiles) {  // phase A: tile u sorted in place (its keys are touched by this task only)
            phase_a = true;
            const uint32_t j = u * kMT + threadIdx.x;
            const unsigned long long kj = j < n ? __ldcg(keys + j) : ~0ull;
            s_ab[threadIdx.x] = kj;
            __syncthreads();
            uint32_t rank = 0;
#pragma unroll 8
            for (uint32_t i = 0; i < kMT; ++i) rank += s_ab[i] < kj ? 1u : 0u;
            if (j < n) keys[u * kMT + rank] = kj;
          } else {  // phase B: tile u - n_tiles against every other sorted tile
            const uint32_t tt = u - n_tiles;
            if (threadIdx.x == 0)  // every tile sort was claimed before this task: running CTAs
              while (*reinterpret_cast<volatile uint32_t*>(&st->fuse_a) < n_tiles) __nanosleep(32);
            __syncthreads();
            const uint32_t j = tt * kMT + threadIdx.x;
            const unsigned long long kj = j < n ? __ldcg(keys + j) : ~0ull;
            uint32_t rank = threadIdx.x;  // within its own sorted tile
            for (uint32_t v0 = 0; v0 < n_tiles; v0 += kMItems) {
              __syncthreads();
              for (uint32_t i = threadIdx.x; i < kMTile; i += kMT) {
                const uint32_t g = v0 * kMT + i;
                s_ab[i] = g < n ? __ldcg(keys + g) : ~0ull;
              }
              __syncthreads();
              const uint32_t nv = min(static_cast<uint32_t>(kMItems), n_tiles - v0);
              for (uint32_t w = 0; w < nv; ++w) {
                if (v0 + w == tt) continue;
                const unsigned long long* a = s_ab + w * kMT;
                uint32_t lo = 0, hi = min(static_cast<uint32_t>(kMT), n - (v0 + w) * kMT);
                while (lo < hi) {
                  const uint32_t mid = (lo + hi) >> 1;
                  if (a[mid] < kj)
                    lo = mid + 1u;
                  else
                    hi = mid;
                }
                rank += lo;
              }
            }
            if (j < n) out[rank] = kj;
          }
        } else {  // rank sort of one tile (rank_sort_kernel_body), smem tiles in s_ab
          const uint32_t j = (t - n_trim) * kMT + threadIdx.x;
          const unsigned long long kj = j < n ? __ldg(unsorted_key + j) : ~0ull;
          uint32_t rank = 0;
          for (uint32_t t0 = 0; t0 < n; t0 += kMT) {
            __syncthreads();
            s_ab[threadIdx.x] = (t0 + threadIdx.x < n) ? __ldg(unsorted_key + t0 + threadIdx.x) : ~0ull;
            __syncthreads();
            const uint32_t lim = min(static_cast<uint32_t>(kMT), n - t0);
#pragma unroll 8
            for (uint32_t i = 0; i < lim; ++i) rank += s_ab[i] < kj ? 1u : 0u;
          }
          if (j < n) out[rank] = kj;
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
          if (phase_a) atomicAdd(&st->fuse_a, 1u);
          atomicAdd(&st->fuse_done, 1u);
        }
      }
      if (threadIdx.x == 0)
        while (*reinterpret_cast<volatile uint32_t*>(&st->fuse_done) < tasks) __nanosleep(32);
      __threadfence();
      __syncthreads();
    }
  }
  // L2 reads: the trim may have written these in this launch
  if (threadIdx.x < kMaxLevels) {
    s_lo[threadIdx.x] = __ldcg(st->seg_lo + threadIdx.x);
    s_pre[threadIdx.x] = __ldcg(st->seg_pre + threadIdx.x);
  }
  if (threadIdx.x == 0) s_pre[kMaxLevels] = __ldcg(st->seg_pre + kMaxLevels);
  __syncthreads();
  const uint32_t cur = st->cur;
  const uint32_t n_keep = __ldcg(&st->n_keep);
  const uint32_t n_s = st->n_surv;
  // the grid is sized for the queue's capacity (the root count on the first
  // flushes: C2 1184 CTAs for ~20 output tiles): CTAs without an output
  // tile skip the survivor ranking and the merge (they still count towards
  // merge_done, so the finalising CTA is the last CTA of the grid -- every
  // CTA is then past the claimed-task prologue)
  const bool idle = !st->merge_all && static_cast<uint64_t>(blockIdx.x) * kMTile >= static_cast<uint64_t>(n_keep) + n_s;
  // few survivors: every CTA ranks them in shared memory (no sort kernel)
  __shared__ unsigned long long s_b[kMergeSortSmall];
  const unsigned long long* skey = sorted_key;
  if (n_s <= kMergeSortSmall && !idle) {
    static_assert(kMergeSortSmall == kMT, "one survivor per thread");
    const unsigned long long kj = threadIdx.x < n_s ? __ldcg(unsorted_key + threadIdx.x) : ~0ull;
    s_ab[threadIdx.x] = kj;
    __syncthreads();
    uint32_t rank = 0;
    for (uint32_t i = 0; i < n_s; ++i) rank += s_ab[i] < kj ? 1u : 0u;
    if (threadIdx.x < n_s) s_b[rank] = kj;
    __syncthreads();
    skey = s_b;
  }
  const RemView A{q.keys(cur) + st->n_cons, s_lo, s_pre, strategy == BBS_STRATEGY_BFS};
  unsigned long long* __restrict__ ok = q.keys(cur ^ 1u);
  // the vote's two keys, loaded before the merge work (inputs, unchanged by it)
  unsigned long long vote_s = 0, vote_a = 0;
  if (vote && threadIdx.x < 32 && !st->spec_mode && n_s) {
    if (idle && n_s <= kMergeSortSmall) {  // not ranked here: the smallest survivor key
      unsigned long long m = ~0ull;
      for (uint32_t i = threadIdx.x; i < n_s; i += 32) m = min(m, __ldcg(unsorted_key + i));
#pragma unroll
      for (int d = 16; d; d >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, d));
      vote_s = m;
    } else {
      vote_s = skey[0];  // sorted (rank sort / the prologue), or ranked in shared memory above
    }
    vote_a = st->look_key;
  }
  const uint32_t total = n_keep + n_s;
  const uint32_t warp = threadIdx.x >> 5;
  for (uint32_t d0 = idle ? total : blockIdx.x * kMTile; d0 < total; d0 += gridDim.x * kMTile) {
    const uint32_t d1 = min(total, d0 + kMTile);
    if (warp < 2) {
      const uint32_t sp = warp_merge_split(A, n_keep, skey, n_s, warp ? d1 : d0);
      if ((threadIdx.x & 31u) == 0) s_split[warp] = sp;
    }
    __syncthreads();
    const uint32_t a0 = s_split[0], a1 = s_split[1];
    const uint32_t na = a1 - a0, nb = (d1 - d0) - na, b0 = d0 - a0;
    for (uint32_t i = threadIdx.x; i < na + nb; i += kMT)
      s_ab[i] = i < na ? A[a0 + i] : skey[b0 + (i - na)];
    __syncthreads();
    const unsigned long long* sa = s_ab;
    const unsigned long long* sb = s_ab + na;
    const uint32_t dt = threadIdx.x * kMItems;
    if (dt < na + nb) {
      uint32_t lo = dt > nb ? dt - nb : 0u, hi = min(dt, na);
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (sa[mid] < sb[dt - 1u - mid])
          lo = mid + 1u;
        else
          hi = mid;
      }
      uint32_t i = lo, j = dt - lo;
      const uint32_t end = min(dt + kMItems, na + nb);
      for (uint32_t o = dt; o < end; ++o) {
        const bool take_a = j >= nb || (i < na && sa[i] < sb[j]);
        ok[d0 + o] = take_a ? sa[i++] : sb[j++];
      }
    }
    __syncthreads();
  }
  // E7 (last CTA): swap queue buffers; the loop ends when queue and pending
  // are empty
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&st->merge_done, 1u) == gridDim.x - 1) {
      __threadfence();
      const uint32_t len = n_keep + n_s;
      st->q_len = len;
      st->cur ^= 1u;
      st->q_peak = max(st->q_peak, len);
      if (len == 0) st->active = 0;
      st->merge_done = 0;
      st->fuse_claim = 0;  // every CTA is past the prologue
      st->fuse_done = 0;
      st->fuse_a = 0;
      if (vote && !st->spec_mode) {
        // would a speculative round have kept the next epoch?  It is formed
        // from the remainder alone; the survivors displace it when the
        // smallest survivor key precedes the entry it would pop last (the
        // frontier's lookahead, ~0 when unknown: no vote)
        bool keep = n_s == 0;
        if (n_s) keep = vote_a != ~0ull && vote_s > vote_a;
        st->spec_votes = keep ? st->spec_votes + 1u : 0u;
        if (st->spec_votes >= static_cast<uint32_t>(vote & 0xFF)) {
          st->spec_mode = 1u;
          // first round depth (A/B: vote >> 8)
          if (vote >> 8) st->spec_k = min(static_cast<uint32_t>(vote >> 8), st->spec_kmax);
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kMT) merge_kernel(EpochState* st, Queue q, int strategy,
                                                    const unsigned long long* skey,
                                                    const unsigned long long* ukey, int fused_trim) {
  // fused_trim: -3 = not fused (a rank-sort kernel ran), else the trim strategy (-1 none)
  merge_kernel_body(st, q, strategy, skey, ukey, 0, fused_trim != -3, fused_trim);
}

// ---- device-switched speculative rounds (BFS, single searches) -------------
// Every epoch of a batch runs these kernels; each takes the plain or the
// speculative body by st->spec_mode.  Plain epochs vote: the merge kernel's
// finalising CTA turns speculation on once two consecutive epochs show that
// a round would have kept their successor.  A search whose survivors keep
// overtaking the next prefix (C2: 7 flushes) never switches; long searches
// switch after their first epochs instead of after a whole host check.
__global__ void __launch_bounds__(kFT) frontier_auto_kernel(EpochState* st, Queue q, GridView G,
                                                            unsigned long long b, int k_max,
                                                            uint32_t* __restrict__ exp_parent,
                                                            uint32_t* __restrict__ exp_off,
                                                            int32_t* __restrict__ trace,
                                                            unsigned long long trace_cap, int strategy,
                                                            uint32_t* __restrict__ cache_ctl,
                                                            SpecRec* __restrict__ rec) {
  pdl_wait();
  // the mode and the activity flag in one round trip
  __shared__ uint32_t s_mode;
  __shared__ int s_act;
  if (threadIdx.x == 0) {
    const uint32_t mode = st->spec_mode;
    const int act = st->active;
    s_mode = mode;
    s_act = act ? 1 : 0;
  }
  __syncthreads();
  if (s_mode)
    frontier_spec_kernel_body(st, q, G, b, k_max, exp_parent, exp_off, trace, trace_cap, cache_ctl, rec, s_act);
  else
    frontier_kernel_body(st, q, G, b, exp_parent, exp_off, trace, trace_cap, strategy, cache_ctl, s_act, true);
}

__global__ void __launch_bounds__(kST) survivors_auto_kernel(EpochState* st, Queue q, int strategy,
                                                             const bbs_node* __restrict__ pending,
                                                             const int32_t* __restrict__ scores,
                                                             unsigned long long* __restrict__ s_key,
                                                             unsigned long long* __restrict__ tiles,
                                                             SpecRec* __restrict__ rec) {
  pdl_wait();
  if (st->spec_mode)
    survivors_spec_kernel_body(st, q, pending, scores, s_key, tiles, rec);
  else
    survivors_kernel_body(st, q, strategy, pending, scores, s_key, tiles);
}

__global__ void __launch_bounds__(kRT) rank_sort_auto_kernel(EpochState* st,
                                                             const unsigned long long* __restrict__ key,
                                                             unsigned long long* __restrict__ out_key, Queue q,
                                                             int strategy) {
  pdl_wait();
  rank_sort_kernel_body(st, key, out_key, q, st->spec_mode ? strategy : -1);
}

__global__ void __launch_bounds__(kMT) merge_auto_kernel(EpochState* st, Queue q, int strategy,
                                                         const unsigned long long* skey,
                                                         const unsigned long long* ukey, int votes,
                                                         int fused) {
  merge_kernel_body(st, q, strategy, skey, ukey, votes, fused != 0, -2);
}



// ---- co-batched flushes (bbs_search_scans) --------------------------------
// One launch per epoch kernel for a group of searches: blockIdx.y = slot,
// each slot's pointers and views in a device array.  The kernel bodies are
// the single-search ones; a slot whose search has ended (or that holds no
// search: a dummy state with active = 0) falls through them as a no-op.
struct SlotArgs {
  ScoreSlot sc;  // first: the score kernels read this prefix
  EpochState* st;
  Queue q;
  uint32_t* exp_parent;
  uint32_t* exp_off;
  int32_t* trace;
  unsigned long long trace_cap;
  bbs_node* pending;
  int32_t* pscores;
  unsigned long long* s_key;
  unsigned long long* s_key2;
  unsigned long long* surv_tiles;
  SpecRec* rec;
  int k_max;
  int spec;  // this round is speculative (BFS, from the search's second host check on)
};

__global__ void __launch_bounds__(kFT) frontier_group(const SlotArgs* __restrict__ ga, unsigned long long b,
                                                      int strategy) {
  const SlotArgs& a = ga[blockIdx.y];
  uint32_t* ctl = a.sc.cache.enabled ? a.sc.cache.ctl : nullptr;
  if (a.spec)
    frontier_spec_kernel_body(a.st, a.q, a.sc.G, b, a.k_max, a.exp_parent, a.exp_off, a.trace, a.trace_cap, ctl,
                              a.rec);
  else
    frontier_kernel_body(a.st, a.q, a.sc.G, b, a.exp_parent, a.exp_off, a.trace, a.trace_cap, strategy, ctl);
}

__global__ void branch_group(const SlotArgs* __restrict__ ga) {
  const SlotArgs& a = ga[blockIdx.y];
  branch_kernel_body(a.st, a.q, a.sc.G, a.exp_parent, a.exp_off, a.pending, a.pscores, a.sc.cache, RunSplit{});
}

__global__ void __launch_bounds__(kST) survivors_group(const SlotArgs* __restrict__ ga, int strategy) {
  const SlotArgs& a = ga[blockIdx.y];
  if (a.spec)
    survivors_spec_kernel_body(a.st, a.q, a.pending, a.pscores, a.s_key, a.surv_tiles, a.rec);
  else
    survivors_kernel_body(a.st, a.q, strategy, a.pending, a.pscores, a.s_key, a.surv_tiles);
}

__global__ void __launch_bounds__(kRT) rank_sort_group(const SlotArgs* __restrict__ ga, int strategy) {
  const SlotArgs& a = ga[blockIdx.y];
  rank_sort_kernel_body(a.st, a.s_key, a.s_key2, a.q, a.spec ? strategy : -1);
}

__global__ void __launch_bounds__(kMT) merge_group(const SlotArgs* __restrict__ ga, int strategy) {
  const SlotArgs& a = ga[blockIdx.y];
  merge_kernel_body(a.st, a.q, strategy, a.s_key2, a.s_key);
}

// Exact mode: this rank's run scores back to their pending positions.
__global__ void scatter_own_kernel(const EpochState* st, RunSplit split, int32_t* __restrict__ pscores) {
  pdl_wait();
  const uint32_t n = st->n_own;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    pscores[((j >> 3) * split.world + split.rank) * 8u + (j & 7u)] = split.pscores_own[j];
}

// Roots mode, device exchange: {incumbent, active} out, max-reduced back in.
__global__ void xchg_pack_kernel(const EpochState* st, int32_t* x) {
  x[0] = st->best;
  x[1] = st->active;
}
__global__ void xchg_unpack_kernel(EpochState* st, const int32_t* x) {
  if (x[0] > st->best) st->best = x[0];
  st->any_active = x[1];
}

// Root survivors -> queue entries (seq = rank in initial_nodes order).  All
// roots share one level, so the queue order is (score desc, seq asc) for BFS
// and (score desc, seq desc) for DFS: a STABLE sort on the short key
// smax - score, fed in seq order (BFS) or reversed (DFS), yields it.
__global__ void roots_to_queue_kernel(const unsigned long long* __restrict__ ref_idx, uint32_t n,
                                      const int32_t* __restrict__ scores, BoxParams bp,
                                      int strategy, int32_t smax, uint32_t* __restrict__ skey,
                                      uint32_t* __restrict__ perm, bbs_node* __restrict__ node) {
  const unsigned long long nrot = static_cast<unsigned long long>(bp.nr) * bp.np * bp.nw;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long r = ref_idx[i];
    const unsigned long long rot = r % nrot, t = r / nrot;
    bbs_node nd;
    nd.iyaw = static_cast<int32_t>(rot % bp.nw);
    nd.ipitch = static_cast<int32_t>((rot / bp.nw) % bp.np);
    nd.iroll = static_cast<int32_t>(rot / (static_cast<unsigned long long>(bp.nw) * bp.np));
    nd.iz = bp.z0 + static_cast<int32_t>(t % bp.nz);
    nd.iy = bp.y0 + static_cast<int32_t>((t / bp.nz) % bp.ny);
    nd.ix = bp.x0 + static_cast<int32_t>(t / (static_cast<unsigned long long>(bp.nz) * bp.ny));
    nd.level = bp.level;
    nd.score = scores[r];
    node[i] = nd;
    const uint32_t j = strategy == BBS_STRATEGY_BFS ? i : n - 1 - i;
    skey[j] = static_cast<uint32_t>(smax - nd.score);
    perm[j] = i;
  }
}

__global__ void queue_keys_kernel(const uint32_t* __restrict__ perm, const bbs_node* __restrict__ pool,
                                  int strategy, unsigned long long* __restrict__ key, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t seq = perm[i];
    const bbs_node nd = pool[seq];
    key[i] = queue_key(strategy, nd.score, nd.level, seq);
  }
}

// Root survivors -> sorted queue without a host round trip (the push of the
// root batch, search.hpp:120-124).  The same order as roots_to_queue + the
// stable radix sort above, with every size kept on the device:
//  1. root_select_kernel: ordered compaction of the roots with score >=
//     threshold (decoupled look-back over tiles taken by ticket); survivor o
//     (seq o) goes to pool[o], its short key smax - score to bkey[o]; the
//     digit histograms of the <= 2 radix passes are counted on the way and
//     the last tile sets the queue length.
//  2. root_pass_kernel, one launch per 8-bit digit: stable LSD pass (match-
//     based block rank in warp-striped order + per-digit look-back across
//     tiles); the last pass writes the 64-bit queue keys directly.  DFS feeds
//     the survivors in reverse so ties order by seq descending.
constexpr int kRST = 256, kRSIPT = 16, kRSTile = kRST * kRSIPT;
constexpr int kRPT = 256, kRPIPT = 8, kRPTile = kRPT * kRPIPT;
constexpr int kRCtlHist = 4;  // ctl: [0] select ticket, [1 + p] pass tickets, [4 + 256 p + d] digit counts

struct RootInit {
  uint32_t* ctl;
  unsigned long long* sel_tiles;   // one look-back word per selection tile
  unsigned long long* pass_tiles;  // 256 look-back words per pass tile, per pass
  uint32_t pass_tiles_cap;
  unsigned long long tag;          // per-search tag (bits 34+): nothing to clear between searches
  uint32_t* bkey;                  // smax - score, seq order
  uint32_t* k1;                    // after pass 0 (two-pass sorts)
  uint32_t* v1;
};

__device__ __forceinline__ unsigned long long lookback_excl(unsigned long long* words, uint32_t tile,
                                                            uint32_t stride, unsigned long long tag,
                                                            uint32_t count) {
  // words[t * stride]: tag | flag << 32 | value (flag 1 aggregate, 2 inclusive)
  if (tile == 0) {
    atomicExch(&words[0], tag | (2ull << 32) | count);
    return 0;
  }
  atomicExch(&words[static_cast<size_t>(tile) * stride], tag | (1ull << 32) | count);
  // 8 predecessors per round trip (independent loads), nearest first; tile 0
  // is always inclusive, so the walk stops at or above it
  uint32_t excl = 0;
  constexpr int kB = 8;
  for (int64_t t = static_cast<int64_t>(tile) - 1;; t -= kB) {
    const volatile unsigned long long* p = words;
    unsigned long long w[kB];
#pragma unroll
    for (int j = 0; j < kB; ++j) w[j] = t - j >= 0 ? p[static_cast<size_t>(t - j) * stride] : 0ull;
    bool done = false;
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      if (done || t - j < 0) continue;
      while ((w[j] & ~((1ull << 34) - 1)) != tag) w[j] = p[static_cast<size_t>(t - j) * stride];  // not published yet
      excl += static_cast<uint32_t>(w[j]);
      done = ((w[j] >> 32) & 3u) == 2u;
    }
    if (done) break;
  }
  atomicExch(&words[static_cast<size_t>(tile) * stride], tag | (2ull << 32) | (excl + count));
  return excl;
}

// One contiguous chunk of tiles per CTA (grid = chunks): the chunk's
// survivors are counted first, one warp look-back over the chunks gives its
// output offset, then the chunk's tiles are scanned again (L1/L2 hits) and
// the survivors scattered in order.  A look-back per 4096-root tile (969
// tiles on C2, 1.3 waves of CTAs) chained ~20 round trips: 27 us.
__global__ void __launch_bounds__(kRST) root_select_kernel(EpochState* st, const int32_t* __restrict__ scores,
                                                           uint32_t n, unsigned long long n_scored,
                                                           int32_t threshold, int32_t smax, BoxParams bp,
                                                           bbs_node* __restrict__ pool, RootInit ri, EpochState h0) {
  pdl_wait();

  using Load = cub::BlockLoad<int32_t, kRST, kRSIPT, cub::BLOCK_LOAD_WARP_TRANSPOSE>;
  using ScanI = cub::BlockScan<int, kRST>;
  using RedI = cub::BlockReduce<int, kRST>;
  __shared__ union {
    typename Load::TempStorage load;
    typename ScanI::TempStorage scan;
    typename RedI::TempStorage red;
  } tmp;
  __shared__ uint32_t s_tile, s_excl;
  __shared__ uint32_t s_h[2 * 256];
  for (int i = threadIdx.x; i < 2 * 256; i += kRST) s_h[i] = 0;
  const uint32_t n_tiles = (n + kRSTile - 1) / kRSTile;
  const unsigned long long nrot = static_cast<unsigned long long>(bp.nr) * bp.np * bp.nw;
  // tickets in launch order: a chunk's predecessors belong to running CTAs
  if (threadIdx.x == 0) s_tile = atomicAdd(&ri.ctl[0], 1u);
  __syncthreads();
  const uint32_t chunk = s_tile, n_chunks = gridDim.x;
  const uint32_t t_lo = static_cast<uint32_t>(static_cast<unsigned long long>(chunk) * n_tiles / n_chunks);
  const uint32_t t_hi = static_cast<uint32_t>(static_cast<unsigned long long>(chunk + 1) * n_tiles / n_chunks);
  const uint32_t lo = t_lo * kRSTile, hi = min(n, t_hi * kRSTile);
  // pass 1: the chunk's survivor count (order does not matter here)
  int cnt = 0;
  for (uint32_t i = lo + threadIdx.x; i < hi; i += kRST * 4) {
    int32_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = i + k * kRST < hi ? scores[i + k * kRST] : INT_MIN;
#pragma unroll
    for (int k = 0; k < 4; ++k) cnt += v[k] >= threshold ? 1 : 0;
  }
  const int tot = RedI(tmp.red).Sum(cnt);
  if (threadIdx.x < 32) {
    const uint32_t excl =
        warp_lookback(ri.sel_tiles, chunk, static_cast<uint32_t>(__shfl_sync(0xffffffffu, tot, 0)), ri.tag);
    if (threadIdx.x == 0) s_excl = excl;
    if (threadIdx.x == 0 && chunk == n_chunks - 1) {
      // the loop's initial state (no host copy on this path)
      const uint32_t kept = excl + static_cast<uint32_t>(tot);
      h0.q_len = kept;
      h0.seq = kept;
      h0.q_peak = kept;
      h0.nodes_pruned = n_scored - kept;
      h0.active = kept > 0 ? 1 : 0;
      h0.any_active = h0.active;
      *st = h0;
    }
  }
  __syncthreads();
  uint32_t run = s_excl;
  // pass 2: tiles in order, survivors scattered in initial_nodes order
  for (uint32_t tile = t_lo; tile < t_hi; ++tile) {
    const uint32_t base = tile * kRSTile;
    const uint32_t valid = min(static_cast<uint32_t>(kRSTile), n - base);
    int32_t sc[kRSIPT];
    __syncthreads();
    Load(tmp.load).Load(scores + base, sc, static_cast<int>(valid), INT_MIN);
    __syncthreads();
    int c = 0;
#pragma unroll
    for (int k = 0; k < kRSIPT; ++k) c += sc[k] >= threshold ? 1 : 0;
    int pos, ttot;
    ScanI(tmp.scan).ExclusiveSum(c, pos, ttot);
    uint32_t o = run + static_cast<uint32_t>(pos);
    run += static_cast<uint32_t>(ttot);
    if (c == 0) continue;
#pragma unroll
    for (int k = 0; k < kRSIPT; ++k) {
      if (sc[k] < threshold) continue;
      const unsigned long long r = base + threadIdx.x * kRSIPT + k;
      const unsigned long long rot = r % nrot, t = r / nrot;
      bbs_node nd;
      nd.iyaw = static_cast<int32_t>(rot % bp.nw);
      nd.ipitch = static_cast<int32_t>((rot / bp.nw) % bp.np);
      nd.iroll = static_cast<int32_t>(rot / (static_cast<unsigned long long>(bp.nw) * bp.np));
      nd.iz = bp.z0 + static_cast<int32_t>(t % bp.nz);
      nd.iy = bp.y0 + static_cast<int32_t>((t / bp.nz) % bp.ny);
      nd.ix = bp.x0 + static_cast<int32_t>(t / (static_cast<unsigned long long>(bp.nz) * bp.ny));
      nd.level = bp.level;
      nd.score = sc[k];
      pool[o] = nd;
      const uint32_t b = static_cast<uint32_t>(smax - sc[k]);
      ri.bkey[o] = b;
      atomicAdd(&s_h[b & 255u], 1u);
      atomicAdd(&s_h[256 + ((b >> 8) & 255u)], 1u);
      ++o;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * 256; i += kRST)
    if (s_h[i]) atomicAdd(&ri.ctl[kRCtlHist + i], s_h[i]);
}

struct RootDigit {
  uint32_t shift;
  __device__ __forceinline__ uint32_t Digit(uint32_t key) const { return (key >> shift) & 255u; }
};

template <bool kFinal>
__global__ void __launch_bounds__(kRPT) root_pass_kernel(const EpochState* st, RootInit ri, uint32_t pass,
                                                         int strategy, int32_t smax, int32_t level,
                                                         const uint32_t* __restrict__ kin,
                                                         const uint32_t* __restrict__ vin,
                                                         uint32_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                         unsigned long long* __restrict__ qkey) {
  pdl_wait();

  using Rank = cub::BlockRadixRankMatch<kRPT, 8, false>;
  using ScanU = cub::BlockScan<uint32_t, kRPT>;
  __shared__ union {
    typename Rank::TempStorage rank;
    typename ScanU::TempStorage scan;
  } tmp;
  __shared__ uint32_t s_tile, s_pre[256], s_base[256];
  const uint32_t n = st->q_len;
  const uint32_t n_tiles = (n + kRPTile - 1) / kRPTile;
  unsigned long long* words = ri.pass_tiles + static_cast<size_t>(pass) * ri.pass_tiles_cap * 256;
  // the pass's global digit offsets
  uint32_t gpre;
  ScanU(tmp.scan).ExclusiveSum(ri.ctl[kRCtlHist + 256 * pass + threadIdx.x], gpre);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const RootDigit dig{8u * pass};
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&ri.ctl[1 + pass], 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= n_tiles) break;
    const uint32_t base = tile * kRPTile;
    const uint32_t valid = min(static_cast<uint32_t>(kRPTile), n - base);
    // warp-striped: the match-based rank is stable in this order
    uint32_t key[kRPIPT], val[kRPIPT];
#pragma unroll
    for (int k = 0; k < kRPIPT; ++k) {
      const uint32_t j = warp * (32 * kRPIPT) + k * 32 + lane;
      key[k] = 0xFFFFFFFFu;  // digit 255, after every real key of the tile
      val[k] = 0;
      if (j < valid) {
        if (pass == 0) {
          const uint32_t src = strategy == BBS_STRATEGY_BFS ? base + j : n - 1 - (base + j);
          key[k] = kin[src];
          val[k] = src;
        } else {
          key[k] = kin[base + j];
          val[k] = vin[base + j];
        }
      }
    }
    int ranks[kRPIPT];
    int pre[1];
    Rank(tmp.rank).RankKeys(key, ranks, dig, pre);
    s_pre[threadIdx.x] = static_cast<uint32_t>(pre[0]);
    __syncthreads();
    uint32_t cnt = (threadIdx.x < 255 ? s_pre[threadIdx.x + 1] : static_cast<uint32_t>(kRPTile)) - s_pre[threadIdx.x];
    if (threadIdx.x == 255) cnt -= kRPTile - valid;  // the padding
    const uint32_t excl = lookback_excl(words + threadIdx.x, tile, 256, ri.tag, cnt);
    s_base[threadIdx.x] = gpre + excl - s_pre[threadIdx.x];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kRPIPT; ++k) {
      const uint32_t j = warp * (32 * kRPIPT) + k * 32 + lane;
      if (j >= valid) continue;
      const uint32_t p = s_base[dig.Digit(key[k])] + static_cast<uint32_t>(ranks[k]);
      if (kFinal) {
        qkey[p] = queue_key(strategy, smax - static_cast<int32_t>(key[k]), level, val[k]);
      } else {
        kout[p] = key[k];
        vout[p] = val[k];
      }
    }
    __syncthreads();
  }
}

__global__ void soa_kernel(const double* __restrict__ aos, uint64_t k, double* __restrict__ soa) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < k;
       i += uint64_t(gridDim.x) * blockDim.x) {
    soa[i] = aos[3 * i];
    soa[k + i] = aos[3 * i + 1];
    soa[2 * k + i] = aos[3 * i + 2];
  }
}
// Survivors of the root batch (score >= threshold), counted.
__global__ void count_survivors_kernel(const int32_t* __restrict__ scores, uint64_t n, int32_t threshold,
                                       unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    c += scores[i] >= threshold ? 1u : 0u;
  c = cub::BlockReduce<unsigned long long, 256>().Sum(c);
  if (threadIdx.x == 0 && c) atomicAdd(out, c);
}

// Root ownership predicate over initial_nodes() order: the root scores buffer
// is pre-filled with -1, so only owned roots can reach the threshold (>= 0).
struct RootSurvives {
  const int32_t* scores;
  int32_t threshold;
  __host__ __device__ bool operator()(const unsigned long long& r) const {
    return scores[r] >= threshold;
  }
};

unsigned grid1(uint64_t n, int threads = 256) {
  return static_cast<unsigned>(std::min<uint64_t>(std::max<uint64_t>((n + threads - 1) / threads, 1), share_cap(148ull * 16)));
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  BBS_CUDA(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

// trans_index_range, nodes.hpp:53-56 (x86 conversion semantics).
void trans_index_range(double lo, double hi, double cell, int32_t* mn, int32_t* mx) {
  const double f = std::floor(lo / cell), c = std::ceil(hi / cell);
  *mn = (f >= -2147483648.0 && f < 2147483648.0) ? static_cast<int32_t>(f) : INT32_MIN;
  *mx = (c >= -2147483648.0 && c < 2147483648.0) ? static_cast<int32_t>(c) : INT32_MIN;
}

template <typename T>
T* dalloc(size_t n, cudaStream_t s) {
  T* p = nullptr;
  BBS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(n, 1) * sizeof(T), s));
  return p;
}

// Device buffer that only ever grows; reused across searches.
template <typename T>
struct Buf {
  T* p = nullptr;
  size_t cap = 0;
  T* get(size_t n, cudaStream_t s, bool keep = false, size_t keep_n = 0) {
    if (n <= cap) return p;
    const size_t c = std::max<size_t>(n, cap + cap / 2);
    T* np = dalloc<T>(c, s);
    if (keep && p && keep_n) BBS_CUDA(cudaMemcpyAsync(np, p, keep_n * sizeof(T), cudaMemcpyDeviceToDevice, s));
    if (p) BBS_CUDA(cudaFreeAsync(p, s));
    p = np;
    cap = c;
    return p;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

}  // namespace

// Persistent device workspace of one search (K5/K6 buffers, root scratch,
// pinned status mirror, event pool).  Acquired from the map's pool per call,
// so steady-state searches allocate nothing.
struct Workspace {
  Buf<double2> lut;
  Buf<int32_t> root_scores;
  Buf<unsigned long long> probes, surv_idx, qk0, qk1, s_key, s_key2, surv_tiles;
  Buf<int> nsel;
  Buf<unsigned char> temp, sort_temp, spec;
  Buf<bbs_node> pool, pending, pending_own;
  Buf<uint32_t> perm0, perm1, sk0, sk1, exp_parent, exp_off;
  Buf<int32_t> pscores, trace, hist_n, pscores_own, xchg;
  Buf<int4> hist_ent, cache_info, cache_pool, cache_builds, cache_pre;
  Buf<uint32_t> cache_u32, cache_amb, cache_fb, stage_win, cache_direct;
  Buf<unsigned char> cache_dflag;
  Buf<int32_t> cache_builds_w, cache_pre_w;
  Buf<uint32_t> hist_amb, rinit_ctl;
  Buf<unsigned long long> rinit_tiles;
  unsigned long long rinit_tag = 0;
  GridView lut_view;  // the rotation LUT in `lut`, built for lut_key
  double lut_key[7] = {};
  bool lut_valid = false;
  Buf<EpochState> st;
  EpochState* h_st = nullptr;
  cudaStream_t side = nullptr;            // prebuild stream (forked per search)
  cudaGraphExec_t graph_exec = nullptr;   // epoch-batch graph, updated in place per search
  cudaEvent_t block_ev = nullptr;         // blocking-sync event (host checks of concurrent searches)
  unsigned long long* h_small = nullptr;  // pinned: probes, n_root_surv, then kTraceStage trace entries
  std::vector<cudaEvent_t> ev;
  size_t ev_used = 0;
  cudaEvent_t next_event() {
    if (ev_used == ev.size()) {
      cudaEvent_t e;
      BBS_CUDA(cudaEventCreate(&e));
      ev.push_back(e);
    }
    return ev[ev_used++];
  }
  void release_all() {
    for (auto* b : {&root_scores, &pscores, &trace, &hist_n, &pscores_own, &xchg}) b->release();
    for (auto* b : {&probes, &surv_idx, &qk0, &qk1, &s_key, &s_key2, &surv_tiles}) b->release();
    for (auto* b : {&pool, &pending, &pending_own}) b->release();
    for (auto* b : {&perm0, &perm1, &sk0, &sk1, &exp_parent, &exp_off, &hist_amb, &rinit_ctl}) b->release();
    rinit_tiles.release();
    lut.release();
    lut_valid = false;
    nsel.release();
    temp.release();
    sort_temp.release();
    spec.release();
    hist_ent.release();
    cache_info.release();
    cache_pool.release();
    cache_builds.release();
    cache_u32.release();
    cache_amb.release();
    cache_fb.release();
    cache_direct.release();
    cache_dflag.release();
    stage_win.release();
    cache_builds_w.release();
    cache_pre.release();
    cache_pre_w.release();
    st.release();
    if (h_st) cudaFreeHost(h_st);
    if (h_small) cudaFreeHost(h_small);
    for (auto e : ev) cudaEventDestroy(e);
    if (side) cudaStreamDestroy(side);
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    if (block_ev) cudaEventDestroy(block_ev);
  }
};

void free_workspace(Workspace* w) {
  if (!w) return;
  w->release_all();
  delete w;
}

namespace {

// RAII lease of a workspace from the map's pool.
struct Lease {
  bbs_map* m;
  Workspace* w;
  explicit Lease(bbs_map* map) : m(map), w(nullptr) {
    std::lock_guard<std::mutex> lk(m->ws_mu);
    if (!m->ws_pool.empty()) {
      w = m->ws_pool.back();
      m->ws_pool.pop_back();
    }
    if (!w) {
      w = new Workspace();
      BBS_CUDA(cudaMallocHost(reinterpret_cast<void**>(&w->h_st), sizeof(EpochState)));
      // pinned: 4 counters + the staged head of the incumbent trace
      BBS_CUDA(cudaMallocHost(reinterpret_cast<void**>(&w->h_small),
                              4 * sizeof(unsigned long long) + kTraceStage * sizeof(int32_t)));
    }
    w->ev_used = 0;
  }
  ~Lease() {
    std::lock_guard<std::mutex> lk(m->ws_mu);
    m->ws_pool.push_back(w);
  }
};

}  // namespace

void set_pool_retention(int device) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

bbs_scan* upload_scan(bbs_map* m, const double* xyz, uint64_t k, bool sync) {
  DeviceGuard g(m->device);
  std::unique_ptr<bbs_scan> sc(new bbs_scan());  // released to the caller on success
  sc->map = m;
  sc->k = k;
  // the copy and the SoA transform go first: they run while the host scans
  // the points below
  cudaStream_t s = m->stream;
  sc->soa = dalloc<double>(3 * std::max<uint64_t>(k, 1), s);
  if (k) {
    StreamAllocs al(s);
    double* aos = al.get<double>(3 * k);
    BBS_CUDA(cudaMemcpyAsync(aos, xyz, 3 * k * sizeof(double), cudaMemcpyHostToDevice, s));
    soa_kernel<<<grid1(k), 256, 0, s>>>(aos, k, sc->soa);
    BBS_CUDA(cudaGetLastError());
  }
  // one pass: max_range (point_cloud.hpp:58-63) as sqrt of the largest
  // x*x + y*y + z*z (sqrt is correctly rounded and monotonic, so this is the
  // max of the per-point ranges bit for bit), the z range and max |x| + |y|
  double r2 = 0.0;
  for (uint64_t i = 0; i < k; ++i) {
    const double x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
    r2 = std::max(r2, x * x + y * y + z * z);
    sc->z_min = i ? std::min(sc->z_min, z) : z;
    sc->z_max = i ? std::max(sc->z_max, z) : z;
    sc->l1xy_max = std::max(sc->l1xy_max, std::fabs(x) + std::fabs(y));
  }
  sc->d_max = std::sqrt(r2);
  if (sync) BBS_CUDA(cudaStreamSynchronize(s));  // callers on other streams see a complete scan
  return sc.release();
}

// ---- co-batched flushes: the group of searches ----------------------------
// bbs_search_scans runs T searches on T host threads; each one's root batch
// and queue build run on its own stream, then it joins the group and every
// host check (E epochs) becomes a rendezvous: the last member to arrive
// uploads the slots' arguments, launches ONE graph of E epochs whose kernels
// cover every slot (blockIdx.y), and reads every member's EpochState back.
// Members leave when their search ends; a thread's next search joins a free
// slot (continuous batching).  The epoch kernels are the single-search
// bodies, so every result equals the search's own (tests/test_search_gpu.py).
struct SearchGroup {
  int device = 0;
  uint32_t n_slots = 0;
  int strategy = 0;
  unsigned long long b = 0;
  int E = 8;
  MapView map{};
  std::mutex mu;
  std::condition_variable cv;
  uint32_t members = 0, arrived = 0;
  uint64_t gen = 0;
  std::vector<uint32_t> free_slots;
  std::vector<char> present;
  std::vector<cudaEvent_t> arrive_ev;
  std::vector<std::pair<const EpochState*, EpochState*>> readback;
  SlotArgs* h_args = nullptr;   // the members' current arguments
  SlotArgs* h_stage = nullptr;  // pinned copy the step's upload reads (members may rewrite h_args
                                // before the upload executes on the device)
  SlotArgs* d_args = nullptr;
  SlotArgs dummy{};
  EpochState* d_dummy = nullptr;
  cudaStream_t gs = nullptr;
  cudaEvent_t done = nullptr;
  cudaGraphExec_t gexec = nullptr;
  std::exception_ptr err;
  uint64_t steps = 0;

  int debug = 0;  // BBS_DEBUG_GROUP=1: no graph, a checked sync after every kernel; 2: after every step
  void check(const char* what) {
    if (debug != 1) return;
    const cudaError_t e = cudaStreamSynchronize(gs);
    if (e != cudaSuccess) {
      std::fprintf(stderr, "[group] step %llu: %s failed: %s\n", static_cast<unsigned long long>(steps), what,
                   cudaGetErrorString(e));
      for (uint32_t i = 0; i < n_slots; ++i)
        std::fprintf(stderr, "[group]  slot %u: st %p present %d k_max %d cache %d stg %d\n", i,
                     static_cast<void*>(h_args[i].st), present[i], h_args[i].k_max, h_args[i].sc.cache.enabled,
                     h_args[i].sc.cache.stg_level);
      throw Error(BBS_ERR_CUDA, "search group: kernel failed");
    }
  }
  void enqueue_epoch() {
    const uint32_t n = n_slots;
    launch_pdl(frontier_group, dim3(1, n), kFT, 0, gs, static_cast<const SlotArgs*>(d_args), b, strategy);
    BBS_CUDA(cudaGetLastError());
    check("frontier");
    launch_pdl(branch_group, dim3(per_slot(148 * 16, n), n), 256, 0, gs, static_cast<const SlotArgs*>(d_args));
    BBS_CUDA(cudaGetLastError());
    check("branch");
    launch_epoch_score_group(map, reinterpret_cast<const ScoreSlot*>(d_args), sizeof(SlotArgs), n, gs);
    check("score kernels");
    launch_pdl(survivors_group, dim3(per_slot(148 * 4, n), n), kST, 0, gs, static_cast<const SlotArgs*>(d_args),
               strategy);
    BBS_CUDA(cudaGetLastError());
    check("survivors");
    launch_pdl(rank_sort_group, dim3(per_slot(148 * 16, n), n), kRT, 0, gs, static_cast<const SlotArgs*>(d_args),
               strategy);
    BBS_CUDA(cudaGetLastError());
    check("rank_sort");
    launch_pdl(merge_group, dim3(per_slot(148 * 8, n), n), kMT, 0, gs, static_cast<const SlotArgs*>(d_args), strategy);
    BBS_CUDA(cudaGetLastError());
    check("merge");
  }

  // the last arrival (lock held): one graph of E epochs over every slot
  void coordinate() {
    try {
      for (uint32_t i = 0; i < n_slots; ++i)
        if (present[i]) {
          if (debug == 3) BBS_CUDA(cudaEventSynchronize(arrive_ev[i]));
          BBS_CUDA(cudaStreamWaitEvent(gs, arrive_ev[i], 0));
        }
      // h_stage is free again: the previous upload ran before the previous
      // step's `done`, which every member still in the group has waited for
      std::memcpy(h_stage, h_args, n_slots * sizeof(SlotArgs));
      BBS_CUDA(cudaMemcpyAsync(d_args, h_stage, n_slots * sizeof(SlotArgs), cudaMemcpyHostToDevice, gs));
      if (debug == 1) {
        for (int e = 0; e < E; ++e) enqueue_epoch();
      } else if (!gexec) {
        cudaGraph_t graph;
        BBS_CUDA(cudaStreamBeginCapture(gs, cudaStreamCaptureModeRelaxed));
        for (int e = 0; e < E; ++e) enqueue_epoch();
        BBS_CUDA(cudaStreamEndCapture(gs, &graph));
        const cudaError_t r = cudaGraphInstantiate(&gexec, graph, 0);
        cudaGraphDestroy(graph);
        BBS_CUDA(r);
      }
      if (debug != 1) BBS_CUDA(cudaGraphLaunch(gexec, gs));
      if (debug == 2) {
        debug = 1;
        check("graph");
        debug = 2;
      }
      for (uint32_t i = 0; i < n_slots; ++i)
        if (present[i])
          BBS_CUDA(cudaMemcpyAsync(readback[i].second, readback[i].first, sizeof(EpochState), cudaMemcpyDeviceToHost,
                                   gs));
      BBS_CUDA(cudaEventRecord(done, gs));
      ++steps;
    } catch (...) {
      err = std::current_exception();
    }
    arrived = 0;
    std::fill(present.begin(), present.end(), 0);
    ++gen;
    cv.notify_all();
  }

  uint32_t join() {
    std::unique_lock<std::mutex> lk(mu);
    if (err) std::rethrow_exception(err);
    if (free_slots.empty()) throw Error(BBS_ERR_GENERIC, "search group: no free slot");
    const uint32_t slot = free_slots.back();
    free_slots.pop_back();
    ++members;
    return slot;
  }

  void leave(uint32_t slot) {
    std::unique_lock<std::mutex> lk(mu);
    h_args[slot] = dummy;
    free_slots.push_back(slot);
    --members;
    if (arrived > 0 && arrived == members) coordinate();
  }

  // E epochs of this member's search (with every other member's); on return
  // *h_dst holds its state after them
  void step(uint32_t slot, const SlotArgs& a, cudaStream_t member_stream, const EpochState* d_src, EpochState* h_dst) {
    BBS_CUDA(cudaEventRecord(arrive_ev[slot], member_stream));
    std::unique_lock<std::mutex> lk(mu);
    if (err) std::rethrow_exception(err);
    h_args[slot] = a;
    readback[slot] = {d_src, h_dst};
    present[slot] = 1;
    const uint64_t my = gen;
    if (++arrived == members)
      coordinate();
    else
      cv.wait(lk, [&] { return gen != my; });
    if (err) std::rethrow_exception(err);
    lk.unlock();
    BBS_CUDA(cudaEventSynchronize(done));  // no later step can start before this member arrives again
  }

  void release() {
    if (gexec) cudaGraphExecDestroy(gexec);
    for (auto e : arrive_ev) cudaEventDestroy(e);
    if (done) cudaEventDestroy(done);
    if (gs) cudaStreamDestroy(gs);
    if (h_args) cudaFreeHost(h_args);
    if (h_stage) cudaFreeHost(h_stage);
    if (d_args) cudaFree(d_args);
    if (d_dummy) cudaFree(d_dummy);
  }
};

thread_local SearchGroup* g_group = nullptr;

SearchGroup* group_create(bbs_map* m, const bbs_search_config& cfg, uint32_t n_slots) {
  DeviceGuard dg(m->device);
  std::unique_ptr<SearchGroup> g(new SearchGroup());
  struct Rel {
    SearchGroup* g;
    ~Rel() {
      if (g) g->release();
    }
  } rel{g.get()};
  g->device = m->device;
  g->n_slots = n_slots;
  g->strategy = cfg.strategy;
  g->b = cfg.batch_size;
  g->map = m->view;
  if (const char* v = std::getenv("BBS_DEBUG_GROUP")) g->debug = std::atoi(v);
  if (const char* v = std::getenv("BBS_GROUP_E")) g->E = std::max(1, std::atoi(v));
  g->present.assign(n_slots, 0);
  g->readback.assign(n_slots, {nullptr, nullptr});
  for (uint32_t i = 0; i < n_slots; ++i) g->free_slots.push_back(n_slots - 1 - i);
  BBS_CUDA(cudaStreamCreateWithFlags(&g->gs, cudaStreamNonBlocking));
  BBS_CUDA(cudaEventCreateWithFlags(&g->done, cudaEventDisableTiming));
  g->arrive_ev.resize(n_slots);
  for (auto& e : g->arrive_ev) BBS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  BBS_CUDA(cudaMallocHost(reinterpret_cast<void**>(&g->h_args), n_slots * sizeof(SlotArgs)));
  BBS_CUDA(cudaMallocHost(reinterpret_cast<void**>(&g->h_stage), n_slots * sizeof(SlotArgs)));
  BBS_CUDA(cudaMalloc(reinterpret_cast<void**>(&g->d_args), n_slots * sizeof(SlotArgs)));
  // a slot without a search: an ended state, no cache, no children
  BBS_CUDA(cudaMalloc(reinterpret_cast<void**>(&g->d_dummy), sizeof(EpochState)));
  BBS_CUDA(cudaMemset(g->d_dummy, 0, sizeof(EpochState)));
  g->dummy.st = g->d_dummy;
  g->dummy.sc.d_n = reinterpret_cast<const uint32_t*>(reinterpret_cast<char*>(g->d_dummy) +
                                                      offsetof(EpochState, n_children));
  g->dummy.sc.n_ptiles = 1;
  g->dummy.sc.cache.enabled = 0;
  g->dummy.sc.cache.stg_level = -1;
  g->dummy.k_max = 1;
  for (uint32_t i = 0; i < n_slots; ++i) g->h_args[i] = g->dummy;
  rel.g = nullptr;
  return g.release();
}

void group_destroy(SearchGroup* g) {
  if (!g) return;
  {
    DeviceGuard dg(g->device);
    if (g->gs) cudaStreamSynchronize(g->gs);
    g->release();
  }
  delete g;
}

// search(), search.hpp:72-186, on the device.  `shard` may be null;
// `stream` null = the map's stream (concurrent searches use their own).
// NVTX range for profilers (nsys / ncu --nvtx); free when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

void run_search(bbs_map* m, bbs_scan* scan, const bbs_search_config& cfg, const bbs_shard* shard,
                bbs_search_result* out, cudaStream_t stream, bbs_search_dump* dump) {
  NvtxRange nv_search("bbs::search");  // search.hpp:72-186
  // validation, search.hpp:79-89, same order and messages
  if (scan->k == 0) throw Error(BBS_ERR_DEGENERATE_SCAN, "search: empty scan");
  if (m->r != cfg.min_resolution) throw Error(BBS_ERR_CONFIG, "search: config r does not match the map");
  if (cfg.max_level < 1 || cfg.max_level > m->max_level)
    throw Error(BBS_ERR_CONFIG, "search: max_level must be in [1, map max level]");
  if (cfg.batch_size < 1) throw Error(BBS_ERR_CONFIG, "search: batch_size must be >= 1");
  if (!(cfg.score_threshold_fraction > 0.0 && cfg.score_threshold_fraction <= 1.0))
    throw Error(BBS_ERR_CONFIG, "search: score_threshold_fraction must be in (0, 1]");
  const double d_max = cfg.has_d_max ? cfg.d_max : scan->d_max;
  if (!(d_max > 0.0)) throw Error(BBS_ERR_DEGENERATE_SCAN, "search: maximum scan range is zero");
  const HostGrid grid = make_grid(cfg, d_max);
  const bbs_aabb tr = cfg.has_translation_range ? cfg.translation_range : m->bbox;
  if (scan->k > static_cast<uint64_t>(kMaxScorePoints))
    throw Error(BBS_ERR_TOO_LARGE, "search: scans above 1048575 points are not supported");
  if (cfg.batch_size > (1ull << 28))
    throw Error(BBS_ERR_TOO_LARGE, "search: batch_size above 2^28 is not supported");
  const int rank = shard ? shard->rank : 0;
  const int world = shard ? std::max(1, shard->world_size) : 1;
  if (rank < 0 || rank >= world) throw Error(BBS_ERR_CONFIG, "search: shard rank out of range");
  // exchanges: on the device through NCCL when a communicator is
  // given, else through the caller's host all-reduce
  const bool exact = shard && shard->mode == BBS_SHARD_EXACT;
  Comm* comm = shard ? reinterpret_cast<Comm*>(shard->comm) : nullptr;
  const bool host_x = shard && !comm && shard->allreduce_max;
  if (exact && world > 1 && !comm && !host_x)
    throw Error(BBS_ERR_CONFIG, "search: the exact shard mode needs an all-reduce");
  const bool roots_dev_x = comm && !exact;    // incumbent exchange every epoch, on the device
  const bool roots_host_x = host_x && !exact; // ... on the host

  DeviceGuard dg(m->device);
  Lease lease(m);
  Workspace& W = *lease.w;
  cudaStream_t s = stream ? stream : m->stream;
  const uint64_t K = scan->k;
  const int32_t threshold =
      static_cast<int32_t>(std::floor(cfg.score_threshold_fraction * static_cast<double>(K)));
  const int L = cfg.max_level;
  uint64_t h2d = 0, d2h = 0;

  // in-place element-wise MAX of n int32 over the ranks (same call count on
  // every rank: the sizes below are identical across ranks)
  std::vector<int32_t> xh;
  std::vector<int64_t> xw;
  auto xmax = [&](int32_t* d, size_t n) {
    if (n == 0) return;
    if (comm) {
      comm_allreduce_max_i32(comm, d, n, s);
      return;
    }
    if (!host_x) return;
    xh.resize(n);
    BBS_CUDA(cudaMemcpyAsync(xh.data(), d, n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    BBS_CUDA(cudaStreamSynchronize(s));
    d2h += n * sizeof(int32_t);
    constexpr size_t kChunk = size_t(1) << 24;
    for (size_t o = 0; o < n; o += kChunk) {
      const size_t c = std::min(kChunk, n - o);
      xw.assign(xh.begin() + o, xh.begin() + o + c);
      if (shard->allreduce_max(xw.data(), static_cast<int32_t>(c), shard->user) != 0)
        throw Error(BBS_ERR_GENERIC, "search: score all-reduce failed");
      for (size_t i = 0; i < c; ++i) xh[o + i] = static_cast<int32_t>(xw[i]);
    }
    BBS_CUDA(cudaMemcpyAsync(d, xh.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    BBS_CUDA(cudaStreamSynchronize(s));
    h2d += n * sizeof(int32_t);
  };

  // root set, initial_nodes (nodes.hpp:60-85)
  const double cell = std::ldexp(cfg.min_resolution, L);
  int32_t x0, x1, y0, y1, z0, z1;
  trans_index_range(tr.min.x, tr.max.x, cell, &x0, &x1);
  trans_index_range(tr.min.y, tr.max.y, cell, &y0, &y1);
  trans_index_range(tr.min.z, tr.max.z, cell, &z0, &z1);
  int64_t nx = static_cast<int64_t>(x1) - x0 + 1, ny = static_cast<int64_t>(y1) - y0 + 1,
          nz = static_cast<int64_t>(z1) - z0 + 1;
  const int64_t nr = grid.axis(0, L).index_count(), np = grid.axis(1, L).index_count(),
                nw = grid.axis(2, L).index_count();
  int64_t total = nx * ny * nz * nr * np * nw;
  if (total <= 0) throw Error(BBS_ERR_EMPTY_SEARCH_SPACE, "initial node set is empty");
  if (nx <= 0 || ny <= 0 || nz <= 0) {
    // two negative extents: the reference's product is positive but its
    // loops produce no node (nodes.hpp:77-79)
    nx = ny = nz = 0;
    total = 0;
  }
  if (nx * ny * nz >= (1ll << 32) || nr * np * nw >= (1ll << 32) || total >= (1ll << 40))
    throw Error(BBS_ERR_TOO_LARGE, "search: root set too large");

  GridView gv;
  // BBS_DEBUG_HOST: host-side timestamps of one search (stderr)
  const bool dbg_host = std::getenv("BBS_DEBUG_HOST") != nullptr;
  const auto th0 = std::chrono::steady_clock::now();
  std::vector<std::pair<const char*, double>> th;
  auto tmark = [&](const char* what) {
    if (dbg_host)
      th.emplace_back(what, std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - th0).count());
  };
  // the rotation LUT depends on make_grid's inputs only: a workspace keeps
  // the last one on the device (sequential searches with one config skip the
  // host libm pass and the copy)
  const double lut_key[7] = {cfg.min_resolution, static_cast<double>(cfg.max_level), cfg.roll_pitch_half_range,
                             cfg.yaw_min, cfg.yaw_max, static_cast<double>(cfg.branch_mode), d_max};
  if (W.lut_valid && std::memcmp(W.lut_key, lut_key, sizeof(lut_key)) == 0) {
    gv = W.lut_view;
  } else {
    W.lut_valid = false;
    const std::vector<double> lut = build_lut(grid, &gv);
    double2* d_lut = W.lut.get(lut.size() / 2, s);
    BBS_CUDA(cudaMemcpyAsync(d_lut, lut.data(), lut.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    h2d += lut.size() * sizeof(double);
    gv.lut = d_lut;
    std::memcpy(W.lut_key, lut_key, sizeof(lut_key));
    W.lut_view = gv;
    W.lut_valid = true;
  }
  tmark("lut");
  const ScanView sv{scan->soa, scan->soa + K, scan->soa + 2 * K, static_cast<uint32_t>(K)};
  const uint64_t maxc = max_children(grid);
  const int strategy = cfg.strategy;
  const uint64_t pend_epoch = cfg.batch_size + maxc;  // children of one flush, at most
  // speculative rounds (BFS, unsharded, no dump): up to spec_k epochs per
  // round (frontier_spec_kernel); BBS_SPEC=n overrides (1 = one epoch per round)
  const int spec_k = [&] {
    if (dump || shard || strategy != BBS_STRATEGY_BFS) return 1;
    const char* v = std::getenv("BBS_SPEC");
    int k = v ? std::atoi(v) : 16;
    k = std::max(1, std::min(k, kSpecMax));
    while (k > 1 && pend_epoch * static_cast<uint64_t>(k) > (1ull << 21)) --k;
    return k;
  }();
  const uint64_t pend_cap = pend_epoch * static_cast<uint64_t>(spec_k);  // children of one round
  uint64_t launches = 0;

  cudaEvent_t ev_start = W.next_event(), ev_roots0 = W.next_event(), ev_roots1 = W.next_event(),
              ev_loop = W.next_event(), ev_sel = W.next_event(), ev_q0 = W.next_event();
  BBS_CUDA(cudaEventRecord(ev_start, s));

  // ---- root batch (search.hpp:111-124) ----
  BoxParams bp{};
  bp.level = L;
  bp.x0 = x0;
  bp.y0 = y0;
  bp.z0 = z0;
  bp.nx = static_cast<uint32_t>(nx);
  bp.ny = static_cast<uint32_t>(ny);
  bp.nz = static_cast<uint32_t>(nz);
  bp.nr = static_cast<uint32_t>(nr);
  bp.np = static_cast<uint32_t>(np);
  bp.nw = static_cast<uint32_t>(nw);
  bp.threshold = threshold;
  bp.rank = static_cast<uint32_t>(rank);
  bp.world = static_cast<uint32_t>(world);
  bp.fpad = static_cast<int32_t>(std::min(std::ceil(scan->d_max / m->view.level[L].cell) + 2.0, 1e6));
  const uint32_t nrot = bp.nr * bp.np * bp.nw;
  uint64_t n_own = 0;  // roots owned by this rank
  {
    uint32_t P = 1, x0r = 0;
    for (uint32_t rot = 0; rot < nrot; ++rot)
      if (owned_slabs(bp, nrot, rot, &P, &x0r) && x0r < bp.nx)
        n_own += static_cast<uint64_t>((bp.nx - x0r + P - 1) / P) * bp.ny * bp.nz;
    BoxParams b0 = bp;
    owned_slabs(b0, nrot, 0, &P, &x0r);
    const uint64_t own_max = static_cast<uint64_t>((bp.nx + P - 1) / P) * bp.ny * bp.nz;
    bp.n_tchunks = static_cast<uint32_t>((own_max + kBoxTransPerCta - 1) / kBoxTransPerCta);
    const double tmax = std::max({std::fabs(static_cast<double>(x0)), std::fabs(static_cast<double>(x1)),
                                  std::fabs(static_cast<double>(y0)), std::fabs(static_cast<double>(y1)),
                                  std::fabs(static_cast<double>(z0)), std::fabs(static_cast<double>(z1))});
    bp.tmax = tmax + 2.0;
  }
  // dense histogram box of a rotated scan at a level's cell (root batch and
  // the flush cache): |fx|, |fy| <= d_max / cell + 2; the rotated z of a
  // point moves by at most sin(t)(|x| + |y|) + (1 - cos^2 t)|z| for
  // roll/pitch within t (the third row of Rz Ry Rx is yaw-free).  A point
  // outside the box makes that histogram fall back (never wrong).  eps bounds
  // fast_floor's per-point eps for every in-box offset.
  auto dense_box = [&](double cell, double tmax_l, int32_t* dr, int32_t* dzlo, int32_t* dnz, double* eps,
                       double* eps1) {
    *dr = 0;
    const double t = std::fabs(cfg.roll_pitch_half_range) + 1e-6;
    const double zabs = std::max(std::fabs(scan->z_min), std::fabs(scan->z_max));
    const double dz = std::sin(t) * scan->l1xy_max + (1.0 - std::cos(t) * std::cos(t)) * zabs + 1e-6 * (1.0 + d_max);
    const double r = std::floor(scan->d_max / cell) + 2.0;
    const double zlo = std::floor((scan->z_min - dz) / cell) - 1.0;
    const double zhi = std::floor((scan->z_max + dz) / cell) + 1.0;
    const double cells = (2.0 * r + 1.0) * (2.0 * r + 1.0) * (zhi - zlo + 1.0);
    if (cells <= static_cast<double>(kCacheDenseCells) && K < 65536 && t < 0.5 &&
        std::getenv("BBS_DENSE_HIST") == nullptr) {
      *dr = static_cast<int32_t>(r);
      *dzlo = static_cast<int32_t>(zlo);
      *dnz = static_cast<int32_t>(zhi - zlo + 1.0);
      const double W = std::max({r, std::fabs(zlo), std::fabs(zhi + 1.0)}) + 1.0;
      *eps = (W + tmax_l) * 0x1p-48;
      *eps1 = 1.0 - *eps;
    }
  };
  tmark("box");
  dense_box(m->view.level[L].cell, bp.tmax, &bp.dn_r, &bp.dn_zlo, &bp.dn_nz, &bp.dn_eps, &bp.dn_eps1);
  // parity dump: no survivor-bound early exit in the root column kernel
  if (dump && dump->exact_roots) bp.threshold = INT32_MIN;
  int32_t* root_scores = W.root_scores.get(static_cast<size_t>(std::max<int64_t>(total, 1)), s);
  // [0] root probes, [1] survivor count, [2] column words read by the root kernel
  unsigned long long* d_probes = W.probes.get(4, s);
  int* d_nsel = W.nsel.get(1, s);
  RootHist hist{};
  hist.entries = W.hist_ent.get(static_cast<size_t>(kRotBatch) * kHistCap, s);
  hist.amb = W.hist_amb.get(static_cast<size_t>(kRotBatch) * kAmbCap, s);
  int32_t* hn = W.hist_n.get(4 * kRotBatch + 1, s);
  hist.n_ent = hn;
  hist.n_amb = hn + kRotBatch;
  hist.overflow = hn + 2 * kRotBatch;  // kRotBatch flags + 1 overflow counter
  hist.total = hn + 3 * kRotBatch + 1;
  // unowned roots must read -1 (below any threshold); a single rank scores
  // and writes every root
  if (world > 1) BBS_CUDA(cudaMemsetAsync(root_scores, 0xFF, static_cast<size_t>(std::max<int64_t>(total, 1)) * 4, s));
  BBS_CUDA(cudaMemsetAsync(d_probes, 0, 3 * sizeof(unsigned long long), s));
  // root survivors -> queue on the device (root_select + root_pass kernels)
  // when the short key (smax - score) takes <= 2 digit passes and the roots
  // fit 32-bit positions; else CUB select + sort after a host sync
  const int32_t smax = static_cast<int32_t>(std::min<size_t>(K, 0x7FFFFFFF));
  const uint32_t span = static_cast<uint32_t>(smax - std::max<int32_t>(0, std::min(threshold, smax)));
  int end_bit = 1;
  while (end_bit < 32 && (span >> end_bit) != 0) ++end_bit;
  const char* init_env = std::getenv("BBS_ROOT_INIT");  // "host" / "device": A/B override
  const bool dev_init_ok = total > 0 && static_cast<uint64_t>(total) <= (64ull << 20) && end_bit <= 16 &&
                           !(init_env && std::strcmp(init_env, "host") == 0);
  RootInit rinit{};
  if (dev_init_ok) {
    const uint64_t n = static_cast<uint64_t>(total);
    const uint64_t sel_tiles = (n + kRSTile - 1) / kRSTile, pass_tiles = (n + kRPTile - 1) / kRPTile;
    const size_t words = sel_tiles + 2 * 256 * pass_tiles;
    const size_t had = W.rinit_tiles.cap;
    unsigned long long* tw = W.rinit_tiles.get(words, s);
    if (W.rinit_tiles.cap != had)  // fresh words: no tag matches zero
      BBS_CUDA(cudaMemsetAsync(tw, 0, W.rinit_tiles.cap * sizeof(unsigned long long), s));
    rinit.sel_tiles = tw;
    rinit.pass_tiles = tw + sel_tiles;
    rinit.pass_tiles_cap = static_cast<uint32_t>(pass_tiles);
    W.rinit_tag = (W.rinit_tag % ((1ull << 30) - 1)) + 1;
    rinit.tag = W.rinit_tag << 34;
    rinit.ctl = W.rinit_ctl.get(kRCtlHist + 512, s);
    BBS_CUDA(cudaMemsetAsync(rinit.ctl, 0, (kRCtlHist + 512) * sizeof(uint32_t), s));
  }
  tmark("root setup");
  cudaEvent_t ev_col0 = W.next_event(), ev_col1 = W.next_event();
  bool col_timed = false;
  BBS_CUDA(cudaEventRecord(ev_roots0, s));
  BBS_CUDA(cudaEventRecord(ev_col0, s));  // re-recorded around the column kernels when they run
  BBS_CUDA(cudaEventRecord(ev_col1, s));
  if (total > 0) {
    NvtxRange nv_roots("bbs::root batch");  // search.hpp:111-124
    col_timed = true;
    launch_score_roots(m->view, gv, sv, bp, hist, root_scores, d_probes, s, ev_col0, ev_col1);
    launches += 3 * ((nrot + kRotBatch - 1) / kRotBatch);
  }
  BBS_CUDA(cudaEventRecord(ev_roots1, s));
  tmark("roots enqueued");
  if (dump) {
    dump->root_count = static_cast<uint64_t>(std::max<int64_t>(total, 0));
    const uint64_t nr_out = std::min(dump->root_count, dump->root_scores ? dump->root_capacity : 0);
    if (nr_out) {
      BBS_CUDA(cudaMemcpyAsync(dump->root_scores, root_scores, nr_out * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      BBS_CUDA(cudaStreamSynchronize(s));
    }
    dump->flush_count = 0;
    dump->epoch_count = 0;
    if (dump->epoch_offsets) dump->epoch_offsets[0] = 0;
  }
  uint64_t dump_epoch = 0;  // flushes seen so far (dump mode)
  cudaEvent_t ev_fork = W.next_event(), ev_prebuilt = W.next_event();
  bool prebuild_pending = false;
  // per-search (level, rotation) histogram cache for the flushes (epoch_cache.cu)
  const bool cache_on = [] {
    const char* v = std::getenv("BBS_ROT_CACHE");  // "0" disables (A/B timing, tests)
    return !(v && v[0] == '0');
  }();
  RotCache cache{};
  cache.stg_level = -1;
  cache.pre_level = -1;
  // a histogram build costs about one direct run, so small scans do not
  // amortize it; measured crossover (C1 room / C2 campus maps, device ms
  // with / without the cache): K 1000 2.17 / 1.66, 1500 2.43 / 1.98, 2000
  // 1.61 / 2.04, 3000 2.47 / 4.04, 5000 2.62 / 5.53; C2 K 1000 1.60 / 1.19,
  // K 3000 0.78 / 0.91
  const uint64_t cache_min_k = [] {
    const char* v = std::getenv("BBS_CACHE_MIN_K");  // A/B timing
    return v ? static_cast<uint64_t>(std::atoll(v)) : uint64_t(2000);
  }();
  if (cache_on && K >= cache_min_k) {
    uint64_t slots = 0;
    const double M = std::max({std::fabs(static_cast<double>(x0)), std::fabs(static_cast<double>(x1)),
                               std::fabs(static_cast<double>(y0)), std::fabs(static_cast<double>(y1)),
                               std::fabs(static_cast<double>(z0)), std::fabs(static_cast<double>(z1))});
    for (int l = 0; l < kMaxLevels; ++l) {
      cache.base[l] = 0xFFFFFFFFu;
      cache.tmax[l] = 0.0;
    }
    for (int l = 0; l < L; ++l) {
      const uint64_t n_rot = static_cast<uint64_t>(grid.axis(0, l).index_count()) *
                             grid.axis(1, l).index_count() * grid.axis(2, l).index_count();
      // nodes at level l have |index| <= (M + 1) * 2^(L - l) (children 2c + j)
      cache.tmax[l] = (M + 1.0) * std::ldexp(1.0, L - l) + 2.0;
      if (n_rot <= (1ull << 20) && slots + n_rot <= (1ull << 23) && cache.tmax[l] < 0x1p28) {
        cache.base[l] = static_cast<uint32_t>(slots);
        slots += n_rot;
        dense_box(m->view.level[l].cell, cache.tmax[l], &cache.dn_r[l], &cache.dn_zlo[l], &cache.dn_nz[l],
                  &cache.dn_eps[l], &cache.dn_eps1[l]);
      }
    }
    cache.stg_level = -1;
    {
      // stage level L-1 (it carries almost all cached flush work): needs a
      // dense box, a single z word per column with 8 bits of headroom, and a
      // padded window that fits shared memory
      const int l = L - 1;
      const LevelView& LV = m->view.level[l];
      if (l >= 0 && cache.base[l] != 0xFFFFFFFFu && cache.dn_r[l] > 0 && LV.layout == BBS_LAYOUT_BITMAP &&
          LV.nwz == 1 && LV.dim[2] <= 24 && cache.dn_zlo[l] >= -128 && cache.dn_zlo[l] + cache.dn_nz[l] <= 128 &&
          std::getenv("BBS_STAGE_PROBE") == nullptr) {
        // child translations at level L-1 span [2 x0, 2 x1 + 1] (+1 for the cube)
        const int64_t R = cache.dn_r[l];
        const int64_t x_lo = 2ll * x0 - LV.box_min[0] - R, x_hi = 2ll * x1 + 2 - LV.box_min[0] + R + 1;
        const int64_t y_lo = 2ll * y0 - LV.box_min[1] - R, y_hi = 2ll * y1 + 2 - LV.box_min[1] + R + 1;
        const int64_t words = (x_hi - x_lo) * (y_hi - y_lo);
        if (words > 0 && words * 4 <= kStageWindowMax) {
          cache.stg_level = l;
          cache.stg_sx0 = static_cast<int32_t>(x_lo);
          cache.stg_sy0 = static_cast<int32_t>(y_lo);
          cache.stg_pitch = static_cast<uint32_t>(x_hi - x_lo);
          cache.stg_rows = static_cast<uint32_t>(y_hi - y_lo);
        }
      }
    }
    if (slots > 0) {
      cache.enabled = 1;
      cache.pool_cap = 16ull << 20;  // entries (16 B each): C3's level-5 histograms use ~1/8 of it
      cache.amb_cap = 8ull << 20;
      cache.info = W.cache_info.get(slots, s);
      cache.amb_off = W.cache_u32.get(slots + kCacheCtl, s);
      cache.ctl = cache.amb_off + slots;
      cache.pool = W.cache_pool.get(cache.pool_cap, s);
      cache.amb_pool = W.cache_amb.get(cache.amb_cap, s);
      // level L-1 is prebuilt in one launch when its rotation count is modest
      const int pl = L - 1;
      const uint64_t pre_rot = (pl >= 0 && cache.base[pl] != 0xFFFFFFFFu)
                                   ? static_cast<uint64_t>(grid.axis(0, pl).index_count()) *
                                         grid.axis(1, pl).index_count() * grid.axis(2, pl).index_count()
                                   : 0;
      const bool prebuild = pre_rot > 0 && pre_rot <= 16384 && [] {
        const char* v = std::getenv("BBS_PREBUILD");  // "0" disables (A/B timing)
        return !(v && v[0] == '0');
      }();
      const uint64_t mr = (pend_cap + 7) / 8;
      cache.builds = W.cache_builds.get(mr, s);
      cache.builds_w = W.cache_builds_w.get(mr, s);
      cache.fb_runs = W.cache_fb.get(mr, s);
      // runs that can have no histogram are scored in the probe kernel's
      // direct phase (BBS_DIRECT_RUNS=0: by the cube kernel after the probe)
      if ([] {
            const char* v = std::getenv("BBS_DIRECT_RUNS");
            return !(v && v[0] == '0');
          }()) {
        cache.direct_runs = W.cache_direct.get(mr, s);
        cache.direct_flag = W.cache_dflag.get(mr, s);
      }
      if (cache.stg_level >= 0) {
        uint32_t* win = W.stage_win.get(((static_cast<size_t>(cache.stg_pitch) * cache.stg_rows + 3) & ~size_t(3)), s);
        build_stage_window(m->view, cache, win, s);
        cache.stg_win = win;
      }
      BBS_CUDA(cudaMemsetAsync(cache.info, 0xFF, slots * sizeof(int4), s));  // all kCacheEmpty
      BBS_CUDA(cudaMemsetAsync(cache.ctl, 0, kCacheCtl * sizeof(uint32_t), s));
      if (prebuild) {
        // fork: the histograms need only the scan, the map and the LUT, so
        // they build on a side stream while this stream selects and sorts
        // the root survivors (a host sync and small kernels: idle SMs)
        cache.pre_level = pl;
        if (!W.side) BBS_CUDA(cudaStreamCreateWithFlags(&W.side, cudaStreamNonBlocking));
        cudaEvent_t e0 = W.next_event();
        // the level's slots are marked BUILDING on this stream (so the first
        // flush's branch kernel never claims them) and listed in a list of
        // their own (the flush builds use cache.builds / ctl[2] meanwhile)
        RotCache pre = cache;
        pre.builds = W.cache_pre.get(pre_rot, s);
        pre.builds_w = W.cache_pre_w.get(pre_rot, s);
        launch_cache_prebuild_list(gv, pre, pl, static_cast<uint32_t>(pre_rot), s);
        BBS_CUDA(cudaEventRecord(ev_fork, s));
        BBS_CUDA(cudaStreamWaitEvent(W.side, ev_fork, 0));
        BBS_CUDA(cudaEventRecord(e0, W.side));
        launch_cache_prebuild(m->view, gv, sv, pre, static_cast<uint32_t>(pre_rot), W.side);
        BBS_CUDA(cudaEventRecord(ev_prebuilt, W.side));
        prebuild_pending = true;
        launches += 2;
        if (std::getenv("BBS_DEBUG_CACHE")) {
          BBS_CUDA(cudaEventSynchronize(ev_prebuilt));
          std::fprintf(stderr, "[cache] prebuild level %d: %llu rotations in %.3f ms\n", pl,
                       static_cast<unsigned long long>(pre_rot), elapsed(e0, ev_prebuilt));
        }
      }
    }
  }

  // (A/B on one box, 3 rounds: C2 0.936 vs 0.938 ms, C3 54.8 vs 55.1 ms, C1
  // 2.065 vs 2.046 ms for device vs host; between bench processes the same
  // path moves by ~1.5% with the buffers' placement, so the two are even on
  // latency; the device path has no host round trip, which frees the host
  // thread for concurrent searches)
  const bool dev_init = dev_init_ok;

  // exact mode: every rank gets every root score (unowned roots are -1)
  if (exact) xmax(root_scores, static_cast<size_t>(std::max<int64_t>(total, 0)));
  const uint64_t n_scored_roots = exact ? static_cast<uint64_t>(std::max<int64_t>(total, 0)) : n_own;

  // survivors >= threshold among own roots, in initial_nodes order
  const bool dbg_spec = std::getenv("BBS_DEBUG_SPEC") != nullptr;  // per-round state (stderr)
  const int E = (host_x || dump || dbg_spec) ? 1 : (g_group ? g_group->E : [] {
    const char* v = std::getenv("BBS_E");  // A/B: epochs per host check
    return v ? std::max(1, std::min(64, std::atoi(v))) : 8;
  }());  // epochs per host check
  unsigned long long root_probes = 0;
  int n_root_surv = 0;       // host path only
  unsigned long long* surv_idx = nullptr;
  uint64_t q_upper = 0;      // bound on the root survivors (queue / pool sizing)
  if (dev_init) {
    q_upper = static_cast<uint64_t>(total);
    BBS_CUDA(cudaEventRecord(ev_sel, s));
  } else {
    // survivor index buffer: the root count bounds it; huge root sets (TransOnly
    // searches: billions of roots) count the survivors first instead
    uint64_t surv_cap = std::max<uint64_t>(n_scored_roots, 1);
    if (total > 0 && n_scored_roots > (64ull << 20)) {
      unsigned long long* d_cnt = d_probes + 1;
      BBS_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), s));
      count_survivors_kernel<<<grid1(static_cast<uint64_t>(total)), 256, 0, s>>>(root_scores, static_cast<uint64_t>(total),
                                                                                 threshold, d_cnt);
      BBS_CUDA(cudaGetLastError());
      BBS_CUDA(cudaMemcpyAsync(&W.h_small[2], d_cnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
      BBS_CUDA(cudaStreamSynchronize(s));
      d2h += sizeof(unsigned long long);
      surv_cap = std::max<uint64_t>(W.h_small[2], 1);
      ++launches;
    }
    surv_idx = W.surv_idx.get(static_cast<size_t>(surv_cap), s);
    if (total > 0) {
      cub::CountingInputIterator<unsigned long long> cnt(0);
      size_t tb = 0;
      BBS_CUDA(cub::DeviceSelect::If(nullptr, tb, cnt, surv_idx, d_nsel, static_cast<int64_t>(total),
                                     RootSurvives{root_scores, threshold}, s));
      void* temp = W.temp.get(tb, s);
      BBS_CUDA(cub::DeviceSelect::If(temp, tb, cnt, surv_idx, d_nsel, static_cast<int64_t>(total),
                                     RootSurvives{root_scores, threshold}, s));
      BBS_CUDA(cudaMemcpyAsync(&W.h_small[0], d_probes, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
      BBS_CUDA(cudaMemcpyAsync(&W.h_small[1], d_nsel, sizeof(int), cudaMemcpyDeviceToHost, s));
      d2h += sizeof(unsigned long long) + sizeof(int);
      BBS_CUDA(cudaEventRecord(ev_sel, s));
      BBS_CUDA(cudaStreamSynchronize(s));
      n_root_surv = *reinterpret_cast<int*>(&W.h_small[1]);
      root_probes = W.h_small[0];
    } else {
      BBS_CUDA(cudaEventRecord(ev_sel, s));
    }
    q_upper = static_cast<uint64_t>(n_root_surv);
  }

  // queue buffers
  uint64_t qcap = q_upper + static_cast<uint64_t>(E + 1) * pend_cap;
  Queue q{};
  q.key[0] = W.qk0.get(qcap, s);
  q.key[1] = W.qk1.get(qcap, s);
  qcap = std::min(W.qk0.cap, W.qk1.cap);
  // node pool: one slot per push (seq), roots first in initial_nodes order
  uint64_t pool_cap = q_upper + static_cast<uint64_t>(E + 1) * pend_cap;
  q.pool = W.pool.get(pool_cap, s);
  pool_cap = W.pool.cap;
  BBS_CUDA(cudaEventRecord(ev_q0, s));

  // device path: the root kernels set the queue length, activity and prune
  // count of this state
  EpochState h0{};
  h0.best = threshold;
  h0.q_len = static_cast<uint32_t>(n_root_surv);
  h0.cur = 0;
  h0.seq = static_cast<unsigned long long>(n_root_surv);
  h0.nodes_generated = n_scored_roots;
  h0.nodes_pruned = n_scored_roots - static_cast<uint64_t>(n_root_surv);
  h0.batches_flushed = 1;
  h0.last_best_epoch = -1;
  h0.active = n_root_surv > 0 ? 1 : 0;
  h0.any_active = h0.active;
  h0.q_peak = h0.q_len;
  h0.spec_k = std::min(2, spec_k);  // the first round's depth; adapted per round
  h0.spec_kmax = static_cast<uint32_t>(spec_k);
  h0.tile_rank_min = [] {  // A/B and tests: BBS_TILE_RANK_MIN (survivors; 256 = always tiled)
    const char* v = std::getenv("BBS_TILE_RANK_MIN");
    return v ? static_cast<uint32_t>(std::max(256, std::atoi(v))) : 4096u;
  }();
  h0.merge_all = [] {
    const char* v = std::getenv("BBS_MERGE_IDLE");
    return v && v[0] == '0' ? 1u : 0u;
  }();
  EpochState* d_st = W.st.get(1, s);
  if (!dev_init) {
    *W.h_st = h0;
    BBS_CUDA(cudaMemcpyAsync(d_st, W.h_st, sizeof(h0), cudaMemcpyHostToDevice, s));
    h2d += sizeof(h0);
  }

  if (dev_init) {
    const uint32_t n = static_cast<uint32_t>(total);
    const uint32_t sel_tiles = (n + kRSTile - 1) / kRSTile;
    static const uint32_t sel_chunks = [] {  // A/B: BBS_SEL_CHUNKS
      const char* v = std::getenv("BBS_SEL_CHUNKS");
      return v ? std::max(1u, static_cast<uint32_t>(std::atoi(v))) : 592u;
    }();
    static const uint32_t root_pass_ctas = [] {  // A/B: BBS_PASS_CTAS
      const char* v = std::getenv("BBS_PASS_CTAS");
      return v ? std::max(1u, static_cast<uint32_t>(std::atoi(v))) : 148u;
    }();
    const uint32_t pass_tiles = (n + kRPTile - 1) / kRPTile;
    rinit.bkey = W.sk0.get(n, s);
    rinit.k1 = W.sk1.get(n, s);
    rinit.v1 = W.perm0.get(n, s);
    launch_pdl(root_select_kernel, std::min<uint32_t>(sel_tiles, sel_chunks), kRST, 0, s, d_st,
               static_cast<const int32_t*>(root_scores), n, static_cast<unsigned long long>(n_scored_roots),
               threshold, smax, bp, q.pool, rinit, h0);
    BBS_CUDA(cudaGetLastError());
    // the survivors (unknown here) are usually far fewer than the roots:
    // one CTA per SM claims the tiles (1184 CTAs were 2-3 waves of no work)
    const unsigned pgrid = std::min<uint32_t>(pass_tiles, root_pass_ctas);
    if (end_bit <= 8) {
      launch_pdl(root_pass_kernel<true>, pgrid, kRPT, 0, s, static_cast<const EpochState*>(d_st), rinit, 0u,
                 strategy, smax, L, static_cast<const uint32_t*>(rinit.bkey), static_cast<const uint32_t*>(nullptr),
                 static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr), q.key[0]);
      BBS_CUDA(cudaGetLastError());
      launches += 2;
    } else {
      launch_pdl(root_pass_kernel<false>, pgrid, kRPT, 0, s, static_cast<const EpochState*>(d_st), rinit, 0u,
                 strategy, smax, L, static_cast<const uint32_t*>(rinit.bkey), static_cast<const uint32_t*>(nullptr),
                 rinit.k1, rinit.v1, static_cast<unsigned long long*>(nullptr));
      BBS_CUDA(cudaGetLastError());
      launch_pdl(root_pass_kernel<true>, pgrid, kRPT, 0, s, static_cast<const EpochState*>(d_st), rinit, 1u,
                 strategy, smax, L, static_cast<const uint32_t*>(rinit.k1), static_cast<const uint32_t*>(rinit.v1),
                 static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr), q.key[0]);
      BBS_CUDA(cudaGetLastError());
      launches += 3;
    }
  } else if (n_root_surv > 0) {
    // nodes in initial_nodes order (seq = position), stable sort on the
    // score key over only the bits it spans, then gather nodes + queue keys
    uint32_t* sk0 = W.sk0.get(n_root_surv, s);
    uint32_t* sk1 = W.sk1.get(n_root_surv, s);
    bbs_node* n0 = q.pool;  // pool[seq] = root with rank seq among the survivors
    uint32_t* perm0 = W.perm0.get(n_root_surv, s);
    uint32_t* perm1 = W.perm1.get(n_root_surv, s);
    roots_to_queue_kernel<<<grid1(n_root_surv), 256, 0, s>>>(surv_idx, n_root_surv, root_scores, bp,
                                                             strategy, smax, sk0, perm0, n0);
    BBS_CUDA(cudaGetLastError());
    cub::DoubleBuffer<uint32_t> dk(sk0, sk1);
    cub::DoubleBuffer<uint32_t> dv(perm0, perm1);
    size_t tb = 0;
    BBS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, n_root_surv, 0, end_bit, s));
    void* temp = W.temp.get(tb, s);
    BBS_CUDA(cub::DeviceRadixSort::SortPairs(temp, tb, dk, dv, n_root_surv, 0, end_bit, s));
    queue_keys_kernel<<<grid1(n_root_surv), 256, 0, s>>>(dv.Current(), n0, strategy, q.key[0], n_root_surv);
    BBS_CUDA(cudaGetLastError());
    launches += 2;  // roots_to_queue, gather
  }
  BBS_CUDA(cudaEventRecord(ev_loop, s));

  bbs_node* pending = W.pending.get(pend_cap, s);
  int32_t* pscores = W.pscores.get(pend_cap, s);
  // exact mode: this rank's runs are scored from a compact copy
  RunSplit split{};
  if (exact) {
    const uint64_t own_cap = ((pend_cap / 8) / world + 2) * 8;
    split.pending_own = W.pending_own.get(own_cap, s);
    split.pscores_own = W.pscores_own.get(own_cap, s);
    split.rank = static_cast<uint32_t>(rank);
    split.world = static_cast<uint32_t>(world);
  }
  int32_t* d_x = W.xchg.get(2, s);
  const uint64_t n_surv_tiles = (pend_cap + kSTile - 1) / kSTile;
  unsigned long long* surv_tiles = W.surv_tiles.get(n_surv_tiles, s);
  BBS_CUDA(cudaMemsetAsync(surv_tiles, 0, n_surv_tiles * sizeof(unsigned long long), s));
  const unsigned surv_grid = static_cast<unsigned>(std::min<uint64_t>(n_surv_tiles, share_cap(148ull * 4)));
  const uint64_t exp_cap = pend_cap / 8 + 2;
  uint32_t* exp_parent = W.exp_parent.get(exp_cap, s);
  uint32_t* exp_off = W.exp_off.get(exp_cap, s);
  unsigned long long* s_key = W.s_key.get(pend_cap, s);
  unsigned long long* s_key2 = W.s_key2.get(pend_cap, s);
  size_t sort_temp_bytes = 0;
  void* sort_temp = nullptr;
  // survivors of one flush are at most pend_epoch: the rank sort up to
  // kRankSortMax of them (a speculative round keeps few), else a radix sort
  const bool rank_sorted = pend_epoch <= kRankSortMax;
  SpecRec* d_rec = spec_k > 1 ? reinterpret_cast<SpecRec*>(W.spec.get(kSpecMax * sizeof(SpecRec), s)) : nullptr;
  if (!rank_sorted) {
    BBS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, sort_temp_bytes, s_key, s_key2, static_cast<int64_t>(pend_cap),
                                            0, 64, s));
    sort_temp = W.sort_temp.get(sort_temp_bytes, s);
  }
  const uint64_t trace_cap = cfg.collect_trace ? std::max<uint64_t>(out->trace_capacity, 1) : 0;
  int32_t* d_trace = W.trace.get(std::max<uint64_t>(trace_cap, 1), s);
  // point tiles per run: one epoch's children, or a whole speculative round's
  const uint32_t ptiles_epoch = choose_ptiles((pend_epoch + 7) / 8, static_cast<uint32_t>(K));
  const uint32_t ptiles_round = choose_ptiles((pend_cap + 7) / 8, static_cast<uint32_t>(K));
  // the level L-1 prebuild ran on the side stream during the root survivor
  // selection and queue build
  // single searches wait for it only before the first flush's score
  // kernels: the first frontier and branch run meanwhile (co-batched
  // members wait here: the group waits on their stream)
  const bool prebuild_defer = prebuild_pending && !g_group && [] {
    const char* v = std::getenv("BBS_DEFER_PREBUILD");  // "0": wait before the first flush (A/B)
    return !(v && v[0] == '0');
  }();
  if (prebuild_pending && !prebuild_defer) BBS_CUDA(cudaStreamWaitEvent(s, ev_prebuilt, 0));

  // per-epoch-slot events of one batch; timings are harvested after each batch
  std::vector<cudaEvent_t> ev_pass(E), ev_s0(E), ev_s1(E);
  for (int e = 0; e < E; ++e) {
    ev_pass[e] = W.next_event();
    ev_s0[e] = W.next_event();
    ev_s1[e] = W.next_event();
  }
  std::vector<float> pass_ms;  // loop start -> end of each frontier pass
  double esm = 0.0;            // device time in the flush score kernels
  const uint32_t* d_nchild = reinterpret_cast<const uint32_t*>(
      reinterpret_cast<char*>(d_st) + (exact ? offsetof(EpochState, n_own) : offsetof(EpochState, n_children)));
  const size_t graph_after = [] {
    const char* v = std::getenv("BBS_GRAPH_AFTER");  // epochs before batches run as graphs
    return v ? static_cast<size_t>(std::atoi(v)) : static_cast<size_t>(0);
  }();
  bool capturing = false;
  // epoch 0 of every batch (a no-op once the prebuild is done; an external
  // event-wait node inside a captured batch)
  auto wait_prebuild = [&](int e) {
    if (!prebuild_defer || e != 0) return;
    BBS_CUDA(cudaStreamWaitEvent(s, ev_prebuilt, capturing ? cudaEventWaitExternal : 0));
  };
  auto record = [&](cudaEvent_t ev) {
    // External: a real record node when captured into the batch graph
    BBS_CUDA(capturing ? cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal)
                       : cudaEventRecord(ev, s));
  };
  // BBS_DEBUG_PHASES: per-phase in-stream times of every epoch (no graphs;
  // each event breaks the PDL overlap, so phases read ~2 us long)
  const bool dbg_phases = std::getenv("BBS_DEBUG_PHASES") != nullptr;
  std::vector<cudaEvent_t> ev_dbg(dbg_phases ? 3 * E : 0);
  for (auto& ev : ev_dbg) ev = W.next_event();
  double dbg_sum[6] = {0, 0, 0, 0, 0, 0};
  uint64_t dbg_n = 0;
  cudaEvent_t dbg_prev = ev_loop;
  // cached levels that can still claim a build (the prebuilt level cannot);
  // once the host sees all of them given up, the build launch is dropped
  uint32_t claimable = 0;
  if (cache.enabled)
    for (int l = 0; l < kMaxLevels; ++l)
      if (cache.base[l] != 0xFFFFFFFFu && l != cache.pre_level) claimable |= 1u << l;
  bool builds_live = claimable != 0;
  // one flush epoch (frontier -> branch -> score -> survivors -> sort -> merge)
  // speculative rounds start once the search outlives its first host check
  // (E single epochs): short searches (C2: 7 flushes, survivors that overtake
  // the next prefix every flush) keep the plain epoch chain
  // BBS_SPEC_AFTER=n (A/B): speculative rounds from the (n+1)-th host check
  const int spec_after = [] {
    const char* v = std::getenv("BBS_SPEC_AFTER");
    return v ? std::max(0, std::atoi(v)) : 1;
  }();
  int checks_done = 0;
  bool spec_on = spec_after == 0 && spec_k > 1;
  // direct runs (scored in the probe kernel's last phase) only in
  // speculative rounds: their probes carry enough histogram work to hide
  // them (C3 13.8 -> 13.3 ms), while a plain C2 epoch's probe is too short
  // and its 2 CTAs per SM score them slower than the cube kernel's 4
  // (C2 0.83 -> 0.88 ms)
  RotCache cache_plain = cache;
  cache_plain.direct_runs = nullptr;
  cache_plain.direct_flag = nullptr;
  auto epoch_cache = [&]() -> const RotCache& { return spec_on ? cache : cache_plain; };
  // device-switched rounds (frontier_auto_kernel ...): BFS single searches
  // with rank-sorted survivors; the host-switched schedule otherwise
  // (BBS_SPEC_AUTO=0: plain epochs for the first host check, then rounds)
  // merge grid cap (A/B: BBS_MERGE_CTAS; CTAs beyond the queue's output
  // tiles only take part in the sort tasks)
  const uint64_t merge_ctas = [] {
    const char* v = std::getenv("BBS_MERGE_CTAS");
    return v ? static_cast<uint64_t>(std::max(1, std::atoi(v))) : 148ull * 4;
  }();
  // the merge kernel does the rank sort (and the round's trim) itself
  // (BBS_FUSE_SORT=0: a rank-sort kernel before it)
  const bool fuse_sort = [] {
    const char* v = std::getenv("BBS_FUSE_SORT");
    return !(v && v[0] == '0');
  }();
  const bool spec_auto = spec_k > 1 && rank_sorted && !exact && !dbg_spec && [] {
    const char* v = std::getenv("BBS_SPEC_AUTO");
    return !(v && v[0] == '0');
  }();
  const int spec_votes_needed = [] {
    const char* v = std::getenv("BBS_SPEC_VOTES");  // consecutive plain epochs voting for rounds
    const char* k0 = std::getenv("BBS_SPEC_K0");  // depth of the first round after the switch (C1 1.43 -> 1.40, C3 12.7 -> 12.3 ms at 4; 8: C3 12.8)
    return (v ? std::max(1, std::atoi(v)) : 2) | ((k0 ? std::max(0, std::min(16, std::atoi(k0))) : 4) << 8);
  }();
  RotCache cache_auto = cache;
  cache_auto.direct_gate =
      reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(d_st) + offsetof(EpochState, spec_mode));
  auto enqueue_auto_epoch = [&](int e) {
    launch_pdl(frontier_auto_kernel, 1, kFT, 0, s, d_st, q, gv, cfg.batch_size, spec_k, exp_parent, exp_off, d_trace,
               trace_cap, strategy, cache.enabled ? cache.ctl : nullptr, d_rec);
    BBS_CUDA(cudaGetLastError());
    record(ev_pass[e]);
    launch_pdl(branch_kernel, grid1(pend_cap), 256, 0, s, d_st, q, gv, exp_parent, exp_off, pending, pscores,
               cache_auto, split);
    BBS_CUDA(cudaGetLastError());
    record(ev_s0[e]);
    wait_prebuild(e);
    launch_epoch_score(m->view, gv, sv, pending, d_nchild, static_cast<uint32_t>(pend_cap), ptiles_round, pscores,
                       cache_auto, s, builds_live);
    record(ev_s1[e]);
    launch_pdl(survivors_auto_kernel, surv_grid, kST, 0, s, d_st, q, strategy, static_cast<const bbs_node*>(pending),
               static_cast<const int32_t*>(pscores), s_key, surv_tiles, d_rec);
    BBS_CUDA(cudaGetLastError());
    if (dbg_phases) record(ev_dbg[3 * e]);
    if (!fuse_sort) {
      launch_pdl(rank_sort_auto_kernel, grid1(pend_cap, kRT), kRT, 0, s, d_st,
                 static_cast<const unsigned long long*>(s_key), s_key2, q, strategy);
      BBS_CUDA(cudaGetLastError());
      ++launches;
    }
    if (dbg_phases) record(ev_dbg[3 * e + 1]);
    launch_pdl(merge_auto_kernel,
               static_cast<unsigned>(std::min<uint64_t>((qcap + kMTile - 1) / kMTile, share_cap(merge_ctas))), kMT, 0,
               s, d_st, q, strategy, static_cast<const unsigned long long*>(s_key2),
               static_cast<const unsigned long long*>(s_key), spec_votes_needed, fuse_sort ? 1 : 0);
    BBS_CUDA(cudaGetLastError());
    if (dbg_phases) record(ev_dbg[3 * e + 2]);
    launches += 4 + (cache.enabled ? (builds_live ? 3 : 2) : 1);  // the score step: build + probe + cube
  };
  auto enqueue_epoch = [&](int e) {
    if (spec_auto && !roots_dev_x) {
      enqueue_auto_epoch(e);
      return;
    }
    if (spec_on)
      launch_pdl(frontier_spec_kernel, 1, kFT, 0, s, d_st, q, gv, cfg.batch_size, spec_k, exp_parent, exp_off,
                 d_trace, trace_cap, cache.enabled ? cache.ctl : nullptr, d_rec);
    else
      launch_pdl(frontier_kernel, 1, kFT, 0, s, d_st, q, gv, cfg.batch_size, exp_parent, exp_off, d_trace,
                 trace_cap, strategy, cache.enabled ? cache.ctl : nullptr);
    BBS_CUDA(cudaGetLastError());
    record(ev_pass[e]);
    launch_pdl(branch_kernel, grid1(pend_cap), 256, 0, s, d_st, q, gv, exp_parent, exp_off, pending, pscores,
               epoch_cache(), split);
    BBS_CUDA(cudaGetLastError());
    record(ev_s0[e]);
    wait_prebuild(e);
    if (exact) {
      launch_epoch_score(m->view, gv, sv, split.pending_own, d_nchild, static_cast<uint32_t>(pend_epoch),
                         ptiles_epoch, split.pscores_own, cache_plain, s, builds_live);
      record(ev_s1[e]);
      launch_pdl(scatter_own_kernel, grid1(pend_cap), 256, 0, s, d_st, split, pscores);
      BBS_CUDA(cudaGetLastError());
      ++launches;
      xmax(pscores, pend_cap);  // every rank: every score of the flush
    } else {
      launch_epoch_score(m->view, gv, sv, pending, d_nchild, static_cast<uint32_t>(spec_on ? pend_cap : pend_epoch),
                         spec_on ? ptiles_round : ptiles_epoch, pscores, epoch_cache(), s, builds_live);
      record(ev_s1[e]);
    }
    if (spec_on)  // survivors of the round + validation + commit of the kept epochs
      launch_pdl(survivors_spec_kernel, surv_grid, kST, 0, s, d_st, q, static_cast<const bbs_node*>(pending),
                 static_cast<const int32_t*>(pscores), s_key, surv_tiles, d_rec);
    else
      launch_pdl(survivors_kernel, surv_grid, kST, 0, s, d_st, q, strategy, pending, pscores, s_key,
                 surv_tiles);
    BBS_CUDA(cudaGetLastError());
    if (dbg_phases) record(ev_dbg[3 * e]);
    if (rank_sorted) {
      if (!fuse_sort) {
        launch_pdl(rank_sort_kernel, grid1(pend_cap, kRT), kRT, 0, s, d_st, s_key, s_key2, q,
                   spec_on ? strategy : -1);
        BBS_CUDA(cudaGetLastError());
        ++launches;
      }
    } else {
      launch_pdl(pad_keys_kernel, grid1(pend_cap), 256, 0, s, d_st, s_key, static_cast<uint64_t>(pend_cap), q,
                 spec_on ? strategy : -1);
      BBS_CUDA(cudaGetLastError());
      size_t tb = sort_temp_bytes;
      BBS_CUDA(cub::DeviceRadixSort::SortKeys(sort_temp, tb, s_key, s_key2, static_cast<int64_t>(pend_cap), 0, 64, s));
    }
    if (dbg_phases) record(ev_dbg[3 * e + 1]);
    launch_pdl(merge_kernel, static_cast<unsigned>(std::min<uint64_t>((qcap + kMTile - 1) / kMTile, share_cap(merge_ctas))),
               kMT, 0, s, d_st, q, strategy, static_cast<const unsigned long long*>(s_key2),
               static_cast<const unsigned long long*>(s_key),
               rank_sorted && fuse_sort ? (spec_on ? strategy : -1) : -3);
    BBS_CUDA(cudaGetLastError());
    if (dbg_phases) record(ev_dbg[3 * e + 2]);
    // frontier, branch, the score step (build + probe + cube), survivors, (pad + sort,) merge
    launches += (rank_sorted ? 4 : 5) + (cache.enabled ? (builds_live ? 3 : 2) : 1);
    if (roots_dev_x) {  // incumbent + activity over NCCL, no host round-trip
      xchg_pack_kernel<<<1, 1, 0, s>>>(d_st, d_x);
      BBS_CUDA(cudaGetLastError());
      comm_allreduce_max_i32(comm, d_x, 2, s);
      xchg_unpack_kernel<<<1, 1, 0, s>>>(d_st, d_x);
      BBS_CUDA(cudaGetLastError());
      launches += 2;
    }
  };
  // E epochs as one CUDA graph (all sizes live in EpochState, so the graph is
  // valid until the queue buffers are re-allocated).  The executable graph
  // lives in the workspace and is UPDATED in place (cudaGraphExecUpdate) for
  // every new capture -- across searches too -- so a search pays a capture
  // (host-side recording, overlapped with its root batch) but no instantiate.
  bool batch_ok = false;  // W.graph_exec holds this search's current capture
  uint64_t batch_qcap = 0;
  const bbs_node* batch_pool = nullptr;
  bool batch_builds = true, batch_spec = false;
  uint64_t batch_launches = 0;
  EpochState hs = h0;
  bool self_active = h0.active != 0;
  if (dev_init) {  // upper bounds until the first device state comes back
    hs.q_len = static_cast<uint32_t>(q_upper);
    hs.seq = q_upper;
    self_active = true;
  }
  bool others_active = false;
  auto exchange = [&]() {
    if (!roots_host_x) return;
    int64_t v[2] = {hs.best, self_active ? 1 : 0};
    if (shard->allreduce_max(v, 2, shard->user) != 0)
      throw Error(BBS_ERR_GENERIC, "search: incumbent all-reduce failed");
    others_active = v[1] != 0;
    if (v[0] > hs.best) {
      hs.best = static_cast<int32_t>(v[0]);
      W.h_st->best = hs.best;
      BBS_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(d_st) + offsetof(EpochState, best),
                               &W.h_st->best, sizeof(int32_t), cudaMemcpyHostToDevice, s));
      h2d += sizeof(int32_t);
      BBS_CUDA(cudaStreamSynchronize(s));
    }
  };
  exchange();  // after the root batch
  if (roots_dev_x) {
    xchg_pack_kernel<<<1, 1, 0, s>>>(d_st, d_x);
    BBS_CUDA(cudaGetLastError());
    comm_allreduce_max_i32(comm, d_x, 2, s);
    xchg_unpack_kernel<<<1, 1, 0, s>>>(d_st, d_x);
    BBS_CUDA(cudaGetLastError());
    BBS_CUDA(cudaMemcpyAsync(W.h_st, d_st, sizeof(EpochState), cudaMemcpyDeviceToHost, s));
    BBS_CUDA(cudaStreamSynchronize(s));
    d2h += sizeof(EpochState);
    hs = *W.h_st;
    others_active = hs.any_active != 0;
    launches += 2;
  }

  // concurrent searches (bbs_search_scans) wait on a blocking-sync event so
  // T waiting host threads do not spin on T cores
  auto host_wait = [&] {
    if (!g_blocking_sync) {
      BBS_CUDA(cudaStreamSynchronize(s));
      return;
    }
    if (!W.block_ev) BBS_CUDA(cudaEventCreateWithFlags(&W.block_ev, cudaEventBlockingSync | cudaEventDisableTiming));
    BBS_CUDA(cudaEventRecord(W.block_ev, s));
    BBS_CUDA(cudaEventSynchronize(W.block_ev));
  };
  // co-batched flushes (bbs_search_scans): a qualifying search runs its
  // epochs inside the group's launches (SearchGroup), else on its own stream
  SearchGroup* grp = g_group;
  if (grp && (shard || dump || dbg_phases || dbg_spec || !rank_sorted || strategy != grp->strategy ||
              cfg.batch_size != grp->b || E != grp->E))
    grp = nullptr;
  struct Member {
    SearchGroup* g = nullptr;
    uint32_t slot = 0;
    void leave() {
      if (g) g->leave(slot);
      g = nullptr;
    }
    ~Member() { leave(); }
  } member;
  if (grp && self_active) {
    // the group waits for this search's stream at every step: its root batch
    // and queue build finish first, so a joiner never stalls the others
    BBS_CUDA(cudaStreamSynchronize(s));
    member.slot = grp->join();
    member.g = grp;
  }
  // the root batch's counters are final: they ride along with the first
  // host check (no extra round trip after the loop)
  if (dev_init) {
    BBS_CUDA(cudaMemcpyAsync(&W.h_small[0], d_probes, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    d2h += sizeof(unsigned long long);
  }
  BBS_CUDA(cudaMemcpyAsync(&W.h_small[3], d_probes + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  d2h += sizeof(unsigned long long);
  bool state_fresh = false;  // W.h_st holds the device state after the last enqueued work
  const uint64_t trace_stage = cfg.collect_trace && out->best_score_trace
                                   ? std::min<uint64_t>({trace_cap, out->trace_capacity, kTraceStage})
                                   : 0;
  const auto t_loop = std::chrono::steady_clock::now();
  uint64_t group_checks = 0;
  tmark("loop");
  while (self_active || others_active) {
    // capacity: the queue grows by at most pend_cap per epoch
    if (static_cast<uint64_t>(hs.q_len) + static_cast<uint64_t>(E + 1) * pend_cap > qcap) {
      const uint64_t need = 2 * (static_cast<uint64_t>(hs.q_len) + static_cast<uint64_t>(E + 1) * pend_cap);
      // the live queue sits in buffer hs.cur; keep its contents
      q.key[0] = W.qk0.get(need, s, true, hs.cur == 0 ? hs.q_len : 0);
      q.key[1] = W.qk1.get(need, s, true, hs.cur == 1 ? hs.q_len : 0);
      qcap = std::min(W.qk0.cap, W.qk1.cap);
    }
    // the pool gains at most pend_cap nodes per epoch; slots [0, seq) are live
    if (hs.seq + static_cast<uint64_t>(E + 1) * pend_cap > pool_cap) {
      const uint64_t need = 2 * (hs.seq + static_cast<uint64_t>(E + 1) * pend_cap);
      if (need >= (1ull << 32)) throw Error(BBS_ERR_TOO_LARGE, "search: more than 2^32 queue pushes");
      q.pool = W.pool.get(need, s, true, hs.seq);
      pool_cap = W.pool.cap;
    }
    // device exchange: every rank runs the same number of epochs (and so
    // of collectives) per batch; the stop decision uses the reduced flag
    const int n_ep = (self_active || roots_dev_x) ? E : 1;
    NvtxRange nv_epochs("bbs::flush epochs");  // search.hpp:145-169, n_ep flushes per host check
    // graphs pay off for long searches (capture + instantiate ~0.2 ms)
    if (member.g) {
      SlotArgs sa{};
      sa.sc.G = gv;
      sa.sc.scan = sv;
      sa.sc.cache = epoch_cache();
      sa.sc.nodes = pending;
      sa.sc.d_n = d_nchild;
      sa.sc.scores = pscores;
      sa.sc.n_ptiles = spec_on ? ptiles_round : ptiles_epoch;
      sa.st = d_st;
      sa.q = q;
      sa.exp_parent = exp_parent;
      sa.exp_off = exp_off;
      sa.trace = d_trace;
      sa.trace_cap = trace_cap;
      sa.pending = pending;
      sa.pscores = pscores;
      sa.s_key = s_key;
      sa.s_key2 = s_key2;
      sa.surv_tiles = surv_tiles;
      sa.rec = d_rec;
      sa.k_max = spec_k;
      sa.spec = spec_on ? 1 : 0;
      member.g->step(member.slot, sa, s, d_st, W.h_st);
      launches += 6ull * E;
      ++group_checks;
    } else if (n_ep == E && E > 1 && pass_ms.size() >= graph_after && !dbg_phases) {
      if (!batch_ok || batch_qcap != qcap || batch_pool != q.pool || batch_builds != builds_live ||
          batch_spec != spec_on) {
        cudaGraph_t graph;
        BBS_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
        capturing = true;
        const uint64_t l0 = launches;
        for (int e = 0; e < E; ++e) enqueue_epoch(e);
        batch_launches = launches - l0;  // kernels per graph launch
        launches = l0;
        capturing = false;
        BBS_CUDA(cudaStreamEndCapture(s, &graph));
        struct GraphGuard {
          cudaGraph_t g;
          ~GraphGuard() { cudaGraphDestroy(g); }
        } gg{graph};
        bool updated = false;
        if (W.graph_exec) {
          cudaGraphExecUpdateResultInfo info{};
          updated = cudaGraphExecUpdate(W.graph_exec, graph, &info) == cudaSuccess;
          if (!updated) {
            (void)cudaGetLastError();  // a topology change: re-instantiate
            cudaGraphExecDestroy(W.graph_exec);
            W.graph_exec = nullptr;
          }
        }
        if (!updated) BBS_CUDA(cudaGraphInstantiate(&W.graph_exec, graph, 0));
        batch_ok = true;
        batch_qcap = qcap;
        batch_pool = q.pool;
        batch_builds = builds_live;
        batch_spec = spec_on;
      }
      BBS_CUDA(cudaGraphLaunch(W.graph_exec, s));
      launches += batch_launches;
      if (group_checks == 0 && pass_ms.empty()) tmark("first batch launched");
    } else {
      for (int e = 0; e < n_ep; ++e) enqueue_epoch(e);
    }
    if (!member.g) {
      BBS_CUDA(cudaMemcpyAsync(W.h_st, d_st, sizeof(EpochState), cudaMemcpyDeviceToHost, s));
      if (trace_stage) {  // the trace's head with the state: no round trip for it after the loop
        BBS_CUDA(cudaMemcpyAsync(W.h_small + 4, d_trace, trace_stage * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        d2h += trace_stage * sizeof(int32_t);
      }
      host_wait();
    }
    state_fresh = !member.g;
    d2h += sizeof(EpochState);
    // in the group the epochs are not timed one by one: host time since the
    // loop began stands for every pass of the check
    const float t_check =
        std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t_loop).count();
    for (int e = 0; e < n_ep; ++e) {
      if (member.g) {
        pass_ms.push_back(t_check);
        continue;
      }
      pass_ms.push_back(elapsed(ev_loop, ev_pass[e]));
      esm += elapsed(ev_s0[e], ev_s1[e]);
      if (dbg_phases) {
        const cudaEvent_t pts[7] = {dbg_prev, ev_pass[e], ev_s0[e], ev_s1[e], ev_dbg[3 * e], ev_dbg[3 * e + 1],
                                    ev_dbg[3 * e + 2]};
        float ph[6];
        for (int k = 0; k < 6; ++k) dbg_sum[k] += (ph[k] = elapsed(pts[k], pts[k + 1]));
        if (dbg_n < 16)
          std::fprintf(stderr, "[phases] epoch %llu: %.1f %.1f %.1f %.1f %.1f %.1f us\n",
                       static_cast<unsigned long long>(dbg_n), 1e3 * ph[0], 1e3 * ph[1], 1e3 * ph[2],
                       1e3 * ph[3], 1e3 * ph[4], 1e3 * ph[5]);
        ++dbg_n;
        dbg_prev = ev_dbg[3 * e + 2];
      }
    }
    if (dbg_phases && n_ep > 0) {
      // the next batch reuses the events: keep the last end time in its own event
      cudaEvent_t keep = W.next_event();
      BBS_CUDA(cudaEventRecord(keep, s));
      dbg_prev = keep;
    }
    hs = *W.h_st;
    if (dbg_spec)
      std::fprintf(stderr, "[spec] pass %u q_len %u best %d n_cons %u n_children %u n_surv %u spec_n %u acc %u k %u gen %llu pruned %llu flushed %llu trace %llu matched %d\n",
                   hs.pass, hs.q_len, hs.best, hs.n_cons, hs.n_children, hs.n_surv, hs.spec_n, hs.spec_acc, hs.spec_k,
                   hs.nodes_generated, hs.nodes_pruned, hs.batches_flushed, hs.trace_len, hs.matched);
    if (dump && hs.n_children > 0) {
      // this epoch's flushed batch: pending[0, n) and its scores (still in
      // place: the next epoch's branch kernel has not run)
      const uint32_t stride = std::max<uint32_t>(dump->epoch_stride, 1);
      if (dump_epoch % stride == 0) {
        const uint64_t n = hs.n_children, o = dump->flush_count;
        const uint64_t fit = o < dump->flush_capacity ? std::min<uint64_t>(n, dump->flush_capacity - o) : 0;
        if (fit && dump->flush_nodes)
          BBS_CUDA(cudaMemcpyAsync(dump->flush_nodes + o, pending, fit * sizeof(bbs_node), cudaMemcpyDeviceToHost, s));
        if (fit && dump->flush_scores)
          BBS_CUDA(cudaMemcpyAsync(dump->flush_scores + o, pscores, fit * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        BBS_CUDA(cudaStreamSynchronize(s));
        const uint64_t e = dump->epoch_count;
        if (e < dump->epoch_capacity) {
          if (dump->epoch_ids) dump->epoch_ids[e] = static_cast<uint32_t>(dump_epoch);
          if (dump->epoch_offsets) dump->epoch_offsets[e + 1] = o + n;
        }
        dump->flush_count = o + n;
        dump->epoch_count = e + 1;
      }
      ++dump_epoch;
    }
    self_active = hs.active != 0;
    builds_live = (claimable & ~hs.cache_raw) != 0;  // raw flags only ever get set
    // host-switched rounds from the second host check on (device-switched
    // searches keep the same batch graph)
    spec_on = !(spec_auto && !member.g) && spec_k > 1 && ++checks_done >= spec_after;
    if (roots_host_x)
      exchange();
    else
      others_active = roots_dev_x && hs.any_active != 0;
  }
  member.leave();  // the other members stop waiting for this one
  cudaEvent_t ev_end = W.next_event();
  BBS_CUDA(cudaEventRecord(ev_end, s));
  if (dbg_phases && total > 0) {
    std::fprintf(stderr, "[phases] init: roots %.1f us, select %.1f us, host sync gap %.1f us, queue %.1f us\n",
                 1e3 * elapsed(ev_roots0, ev_roots1), 1e3 * elapsed(ev_roots1, ev_sel), 1e3 * elapsed(ev_sel, ev_q0),
                 1e3 * elapsed(ev_q0, ev_loop));
  }
  if (dbg_phases && dbg_n) {
    static const char* names[6] = {"frontier", "branch", "score", "survivors", "rank_sort", "merge"};
    std::fprintf(stderr, "[phases] %llu epochs, us/epoch:", static_cast<unsigned long long>(dbg_n));
    for (int k = 0; k < 6; ++k) std::fprintf(stderr, " %s %.2f", names[k], 1e3 * dbg_sum[k] / dbg_n);
    std::fprintf(stderr, "\n");
  }
  if (!state_fresh || shard) {
    // the group path, a sharded search (its exchange may follow the last
    // check) or no check at all: read the final state once more
    BBS_CUDA(cudaMemcpyAsync(W.h_st, d_st, sizeof(EpochState), cudaMemcpyDeviceToHost, s));
    d2h += sizeof(EpochState);
    host_wait();
  } else {
    BBS_CUDA(cudaEventSynchronize(ev_end));  // nothing left on the stream: the event completes at once
  }
  hs = *W.h_st;
  if (dev_init) root_probes = W.h_small[0];
  out->root_words = W.h_small[3];
  out->root_col_ms = col_timed ? elapsed(ev_col0, ev_col1) : 0.0;

  tmark("state read");
  // ---- results ----
  std::memset(&out->stats, 0, sizeof(out->stats));
  out->scan_points = K;
  out->score_threshold = threshold;
  out->stats.nodes_generated = hs.nodes_generated;
  out->stats.nodes_pruned = hs.nodes_pruned;
  out->stats.batches_flushed = hs.batches_flushed;
  out->stats.initial_nodes_ms = elapsed(ev_start, ev_loop);
  const float loop_ms = elapsed(ev_loop, ev_end);
  if (hs.matched && hs.last_best_epoch >= 0 && hs.last_best_epoch < static_cast<int>(pass_ms.size())) {
    const float fb = pass_ms[static_cast<size_t>(hs.last_best_epoch)];
    out->stats.find_best_score_ms = fb;
    out->stats.pop_remaining_queue_ms = loop_ms - fb;
  } else {
    out->stats.find_best_score_ms = loop_ms;
    out->stats.pop_remaining_queue_ms = 0.0;
  }
  out->device_ms = elapsed(ev_start, ev_end);
  out->root_score_ms = elapsed(ev_roots0, ev_roots1);
  out->epoch_score_ms = esm;
  out->epochs = hs.epochs;
  out->root_nodes = n_own;  // roots this rank scored
  out->lookups = hs.nodes_generated * K;
  out->queue_peak = hs.q_peak;
  if (std::getenv("BBS_DEBUG_CACHE") && hs.seq > 0) {
    // dev aid: rotations (and level L-1 child rotations) the root survivors use
    const uint64_t np0 = std::min<uint64_t>(hs.seq, q_upper);
    std::vector<bbs_node> pn(np0);
    BBS_CUDA(cudaMemcpyAsync(pn.data(), q.pool, np0 * sizeof(bbs_node), cudaMemcpyDeviceToHost, s));
    BBS_CUDA(cudaStreamSynchronize(s));
    std::vector<char> used(nrot, 0);
    uint64_t nroot = 0;
    for (const auto& nd : pn)
      if (nd.level == L) {
        ++nroot;
        used[(static_cast<uint64_t>(nd.iroll) * bp.np + nd.ipitch) * bp.nw + nd.iyaw] = 1;
      }
    uint64_t nu = 0;
    for (char c : used) nu += c;
    std::fprintf(stderr, "[roots] survivors %llu of %llu, rotations used %llu of %u\n",
                 static_cast<unsigned long long>(nroot), static_cast<unsigned long long>(n_scored_roots),
                 static_cast<unsigned long long>(nu), nrot);
  }
  if (cache.enabled && std::getenv("BBS_DEBUG_CACHE")) {
    // dev aid: built histograms per level and their mean size
    const size_t ns = W.cache_info.cap;
    std::vector<int4> info(ns);
    BBS_CUDA(cudaMemcpyAsync(info.data(), cache.info, ns * sizeof(int4), cudaMemcpyDeviceToHost, s));
    BBS_CUDA(cudaStreamSynchronize(s));
    for (int l = 0; l <= L; ++l) {
      if (cache.base[l] == 0xFFFFFFFFu) continue;
      uint32_t end = static_cast<uint32_t>(ns);
      for (int l2 = 0; l2 <= L; ++l2)
        if (cache.base[l2] != 0xFFFFFFFFu && cache.base[l2] > cache.base[l]) end = std::min(end, cache.base[l2]);
      uint64_t ready = 0, none = 0, ent = 0, amb = 0;
      for (uint32_t i = cache.base[l]; i < end; ++i) {
        if (info[i].x == 0) {
          ++ready;
          ent += static_cast<uint32_t>(info[i].z);
          amb += static_cast<uint32_t>(info[i].w);
        } else if (info[i].x == -3) {
          ++none;
        }
      }
      std::fprintf(stderr, "[cache] level %d: slots %u built %llu failed %llu mean entries %.1f mean amb %.2f (K %zu)\n",
                   l, end - cache.base[l], static_cast<unsigned long long>(ready),
                   static_cast<unsigned long long>(none), ready ? double(ent) / ready : 0.0,
                   ready ? double(amb) / ready : 0.0, K);
    }
  }
  out->root_probes = root_probes;
  out->trace_length = cfg.collect_trace ? hs.trace_len : 0;
  if (cfg.collect_trace && out->best_score_trace && hs.trace_len) {
    const uint64_t nt = std::min<uint64_t>(hs.trace_len, out->trace_capacity);
    if (state_fresh && !shard && nt <= trace_stage) {
      std::memcpy(out->best_score_trace, W.h_small + 4, nt * sizeof(int32_t));  // staged with the last state
    } else {
      BBS_CUDA(cudaMemcpyAsync(out->best_score_trace, d_trace, nt * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      BBS_CUDA(cudaStreamSynchronize(s));
      d2h += nt * sizeof(int32_t);
    }
  }
  out->h2d_bytes = h2d;
  out->d2h_bytes = d2h;
  if (dbg_host) {
    tmark("results");
    std::fprintf(stderr, "[host]");
    for (const auto& m : th) std::fprintf(stderr, " %s %.1f", m.first, m.second);
    std::fprintf(stderr, " us (device %.1f us; frontier passes %u, rounds on %u, votes %u)\n", 1e3 * out->device_ms,
                 hs.pass, hs.spec_mode, hs.spec_votes);
  }
  out->kernel_launches = launches;
  out->group_checks = group_checks;
  for (int l = 0; l < kMaxLevels; ++l) out->evals_per_level[l] = hs.level_evals[l];
  out->evals_per_level[L] += n_scored_roots;  // the root batch
  int32_t best = hs.best;
  bbs_node best_node = hs.best_node;
  int matched = hs.matched;
  // winner election across ranks: max of (score, world-1-rank) among matched
  // (exact mode: every rank already holds the single-queue result)
  if (!exact && roots_dev_x && world > 1) {
    // over NCCL in int32 steps: top score, then the lowest rank holding it,
    // then that rank's node (same winner as the host protocol below)
    int32_t* d = W.xchg.get(8, s);
    int32_t* h = reinterpret_cast<int32_t*>(W.h_small);  // pinned, >= 32 B
    auto reduce = [&](int n) {
      BBS_CUDA(cudaMemcpyAsync(d, h, n * sizeof(int32_t), cudaMemcpyHostToDevice, s));
      comm_allreduce_max_i32(comm, d, n, s);
      BBS_CUDA(cudaMemcpyAsync(h, d, n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      BBS_CUDA(cudaStreamSynchronize(s));
    };
    h[0] = matched ? best : -1;
    reduce(1);
    const int32_t top = h[0];
    h[0] = (matched && best == top) ? world - 1 - rank : -1;
    reduce(1);
    const int winner = top < 0 ? -1 : world - 1 - h[0];
    const int32_t* f = reinterpret_cast<const int32_t*>(&best_node);
    for (int i = 0; i < 8; ++i) h[i] = rank == winner ? f[i] : INT32_MIN;
    reduce(8);
    if (winner >= 0) {
      std::memcpy(&best_node, h, sizeof(best_node));
      best = top;
      matched = 1;
    } else {
      matched = 0;
    }
  }
  if (!exact && roots_host_x && world > 1) {
    int64_t key[1] = {matched ? (static_cast<int64_t>(best) << 32) | static_cast<int64_t>(world - 1 - rank) : -1};
    if (shard->allreduce_max(key, 1, shard->user) != 0)
      throw Error(BBS_ERR_GENERIC, "search: winner election failed");
    const int winner = key[0] < 0 ? -1 : static_cast<int>(world - 1 - (key[0] & 0xffffffff));
    int64_t nv[8];
    const int32_t* f = reinterpret_cast<const int32_t*>(&best_node);
    for (int i = 0; i < 8; ++i) nv[i] = rank == winner ? static_cast<int64_t>(f[i]) : INT64_MIN;
    if (shard->allreduce_max(nv, 8, shard->user) != 0)
      throw Error(BBS_ERR_GENERIC, "search: winner broadcast failed");
    if (winner >= 0) {
      int32_t* bf = reinterpret_cast<int32_t*>(&best_node);
      for (int i = 0; i < 8; ++i) bf[i] = static_cast<int32_t>(nv[i]);
      best = static_cast<int32_t>(key[0] >> 32);
      matched = 1;
    } else {
      matched = 0;
    }
  }
  out->matched = matched;
  out->best_score = best;
  out->best_node = best_node;
  std::memset(&out->best_pose, 0, sizeof(out->best_pose));
  if (matched) {
    // node_pose(best).normalized(), search.hpp:183, nodes.hpp:33-43
    const double c = std::ldexp(cfg.min_resolution, best_node.level);
    out->best_pose.x = c * static_cast<double>(best_node.ix);
    out->best_pose.y = c * static_cast<double>(best_node.iy);
    out->best_pose.z = c * static_cast<double>(best_node.iz);
    out->best_pose.roll = grid.axis(0, best_node.level).angle(best_node.iroll);
    out->best_pose.pitch = grid.axis(1, best_node.level).angle(best_node.ipitch);
    const double two_pi = 6.283185307179586476925286766559;
    double y = std::fmod(grid.axis(2, best_node.level).angle(best_node.iyaw), two_pi);
    if (y < 0.0) y += two_pi;
    if (y >= two_pi) y = 0.0;
    out->best_pose.yaw = y;
  }
}

// batch_evaluate on device nodes (search.hpp:23-34).
void batch_evaluate_device(bbs_map* m, bbs_scan* scan, const bbs_search_config& cfg, double d_max,
                           bbs_node* d_nodes, uint64_t n, cudaStream_t s, const int32_t* lo,
                           const int32_t* hi) {
  StreamAllocs al(s);
  const GridView gv = upload_grid(cfg, d_max > 0 ? d_max : scan->d_max, lo, hi, s, al);
  batch_evaluate_device(m, scan, gv, d_nodes, n, s);
}

// The rotation LUT of (cfg, d_max) on the device (host libm, build_lut),
// allocated in `al` (freed with it).
GridView upload_grid(const bbs_search_config& cfg, double d_max, const int32_t* lo, const int32_t* hi,
                     cudaStream_t s, StreamAllocs& al) {
  const HostGrid grid = make_grid(cfg, d_max);
  GridView gv;
  const std::vector<double> lut = build_lut(grid, &gv, lo, hi);
  double2* d_lut = al.get<double2>(lut.size() / 2);
  BBS_CUDA(cudaMemcpyAsync(d_lut, lut.data(), lut.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  gv.lut = d_lut;
  return gv;
}

// batch_evaluate with a prebuilt device LUT (callers scoring many blocks).
void batch_evaluate_device(bbs_map* m, bbs_scan* scan, const GridView& gv, bbs_node* d_nodes, uint64_t n,
                           cudaStream_t s) {
  const uint64_t K = scan->k;
  const ScanView sv{scan->soa, scan->soa + K, scan->soa + 2 * K, static_cast<uint32_t>(K)};
  score_nodes_general(m->view, gv, sv, d_nodes, n, s);
}

}  // namespace bbs

bbs_scan::~bbs_scan() {
  if (soa && map) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(map->device);
    cudaFreeAsync(soa, map->stream);  // stream-ordered (searches using it have returned)
    cudaSetDevice(prev);
  }
}
