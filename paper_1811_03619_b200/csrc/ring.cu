// Fused compressed ring AllReduce kernel (sm_100a).
//
// Reference semantics: /root/reference/pkg/src/gradpipe/collective.py:77-139.
//   reduce-scatter step s: rank r sends block (r-s)%p to succ and folds
//     block (r-s-1)%p: acc = x_r[b] + D(C(partial_pred))          (:96-115)
//   allgather: owner (r+1)%p encodes its reduced block once; every rank
//     decodes the owner's exact bytes                              (:117-139)
// so block b is the left fold s_0 = x_b, s_k = fl(x_{b+k} + D(C(s_{k-1})))
// starting at rank b, and out[b] = D(C(s_{p-1})) on every rank.
//
// B200 mapping. One launch per rank per call (cooperative when all ranks
// are emulated on one GPU): up to G CTAs of 128 threads, every WARP an
// independent worker. A ring block is cut into chunks of `chunk` elements
// (multiple of 1024, origin = block start rounded down to 16); warps take
// chunk indices of each phase from a per-rank counter, and every chunk flows
// around the ring on its own:
//   lane 0 acquires flag(slot s, chunk c) -> the warp streams the chunk in
//   1024-element batches (each lane one 16-byte payload vector per group:
//   4 fp32 / 8 trunc16 / 16 quant8 elements) -> decode inbox + add local ->
//   encode -> st.global into succ's inbox over NVLink -> __syncwarp ->
//   lane 0: st.release.sys succ's flag.
// Small none/trunc16 blocks use the LL protocol instead (sequence number in
// every 8-byte word, no fence, no flag; see ll_put / ll_get).
// No CTA-wide barrier sits on the data path, so a warp waiting on its fence
// or flag never stalls the other warps of its SM.
// quant8 needs the block-wide max before any code can be emitted
// (compression.py:129-132): each of its hops is pass A (fold, park the
// partial sum in `out`, reduce the max), a rank-wide barrier carrying the
// max (per-warp atomics on the rank's control block), then pass B (encode
// with the block scale, push). The allgather is a direct owner->all-peers
// push over NVSwitch (the bytes the ring would forward, one hop not p-1).
// Emulation: with nlocal == p the same kernel runs all p ranks on one GPU
// in one cooperative launch (CTA group = rank) for parity tests at p > #GPUs.
#include <algorithm>
#include <cstdlib>

#include <cstdint>
#ifdef PIPESGD_CHECKED
namespace gp {
__device__ __noinline__ bool ring_access_ok(const void* p, uint64_t bytes, bool write);
__device__ __noinline__ void bounds_violation(uint64_t addr);
}  // namespace gp
#define GP_ACCESS_OK(p, bytes, write) ::gp::ring_access_ok((p), (bytes), (write))
#endif
#include "codec.cuh"
#include "ring.cuh"

namespace gp {

namespace {

constexpr int kWarps = kRingThreads / 32;
#ifndef PIPESGD_RING_BATCH
#define PIPESGD_RING_BATCH 1024
#endif
constexpr uint64_t kBatch = PIPESGD_RING_BATCH;  // elements per warp per batch (32 lanes x U x E)

// This call's sequence number, read from the rank's control block at entry.
// It lives on the device (not in the launch parameters) so a launch can be
// captured once in a CUDA graph and replayed: every replay is a new call.
__shared__ uint32_t s_seq;
__shared__ uint32_t s_bank;                 // ctl bank of this call (ring.cuh:CtlBank)
__shared__ unsigned long long s_calls;      // raw count of calls completed before this one
__shared__ unsigned long long s_abort;      // the abort word at kernel entry
__shared__ uint32_t s_iter;                 // iteration tag of this call (argument or device word)
// quant8 rank barriers, CTA-aggregated: the CTA's warps meet in shared
// memory, the last one to arrive makes the CTA's single global arrival and
// polls the rank counter, the others wait on s_bar_open (one barrier index k
// per rank barrier of the call, k < 16)
constexpr int kMaxBarriers = 16;
__shared__ unsigned s_bar_arrived[kMaxBarriers];
__shared__ unsigned s_bar_max[kMaxBarriers];
__shared__ float s_bar_vmax[kMaxBarriers];
__shared__ int s_bar_open[kMaxBarriers];    // 0 waiting, 1 open, 2 failed
#ifdef PIPESGD_CHECKED
__shared__ const RingParams* s_P;           // launch parameters (bounds checks)
#endif

__device__ __forceinline__ CtlBank* cb(Ctl* c) { return &c->bank[s_bank]; }

struct Blk {
  uint64_t start, len, A;
  uint32_t nch;
};

__device__ __forceinline__ Blk get_blk(const RingParams& P, int b) {
  Blk k;
  block_range(P.n, P.p, b, k.start, k.len);
  k.A = k.start & ~15ull;
  k.nch = k.len ? (uint32_t)((k.start + k.len - k.A + P.chunk - 1) / P.chunk) : 0u;
  return k;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ uint64_t* flag_ptr(uint8_t* inbox, const Layout& L, int slot, uint32_t c) {
#ifdef PIPESGD_CHECKED
  if (slot < 0 || (uint32_t)slot >= L.nslot || c >= L.max_chunks) {
    bounds_violation(((uint64_t)slot << 32) | c);
    slot = 0, c = 0;
  }
#endif
  return reinterpret_cast<uint64_t*>(inbox + L.off_flags) + (uint64_t)slot * L.max_chunks + c;
}
__device__ __forceinline__ SlotHdr* hdr_ptr(uint8_t* inbox, const Layout& L, int slot) {
#ifdef PIPESGD_CHECKED
  if (slot < 0 || (uint32_t)slot >= L.nslot) {
    bounds_violation((uint64_t)slot);
    slot = 0;
  }
#endif
  return reinterpret_cast<SlotHdr*>(inbox + L.off_hdr) + slot;
}
__device__ __forceinline__ uint8_t* slot_ptr(uint8_t* inbox, const Layout& L, int slot) {
  return inbox + L.off_payload + (uint64_t)slot * L.slot_bytes;
}

// ---- LL protocol (small blocks, ring.cuh:ll_payload_limit). A slot is a 32-byte
// header line then one 32-byte line per 16-byte payload group; every 8-byte
// word is {4 payload bytes, call sequence}, written with one 16-byte volatile
// store per half line. Aligned 8-byte accesses are single-copy atomic, so a
// word whose sequence half matches carries this call's payload half: the
// receiver polls the data itself, no fence and no flag store.
__device__ __forceinline__ uint8_t* ll_ptr(uint8_t* inbox, const Layout& L, int slot) {
  return inbox + L.off_ll + (uint64_t)slot * L.ll_slot_bytes;
}
__device__ __forceinline__ void st_vol_v4(uint4* p, uint4 v) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 ld_vol_v4(const uint4* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void ll_put(uint8_t* line, uint4 v) {
  if (!GP_ACCESS_OK(line, 32, true)) return;
  uint4* q = reinterpret_cast<uint4*>(line);
  st_vol_v4(q, make_uint4(v.x, s_seq, v.y, s_seq));
  st_vol_v4(q + 1, make_uint4(v.z, s_seq, v.w, s_seq));
}
// Poll one line; false if `give_up` turned true (timeout / abort seen).
template <typename G>
__device__ __forceinline__ bool ll_get(const uint8_t* line, uint4& out, G&& give_up) {
  if (!GP_ACCESS_OK(line, 32, false)) return false;
  const uint4* q = reinterpret_cast<const uint4*>(line);
  for (uint32_t it = 1;; ++it) {
    const uint4 a = ld_vol_v4(q), b = ld_vol_v4(q + 1);
    if (a.y == s_seq && a.w == s_seq && b.y == s_seq && b.w == s_seq) {
      out = make_uint4(a.x, a.z, b.x, b.z);
      return true;
    }
    if ((it & 255u) == 0 && give_up()) return false;
  }
}
template <int C>
__device__ __forceinline__ uint8_t* ll_line(uint8_t* llslot, uint64_t rel0) {
  return llslot + 32 + (rel0 / CodecT<C>::E) * 32;
}

// Abort on every rank: peers' spins see it and stop waiting, and the abort
// stays (ring.cuh:kAbortSticky), so later calls end at once too.
__device__ void broadcast_abort(const RingParams& P, const RankCtx& R) {
  abort_all(R.peer, P.p, P.L.off_ctl, s_seq, R.rank);
}

__device__ __forceinline__ bool aborted(const RingParams&, Ctl* ctl) { return comm_aborted(ctl); }

// Flag word: (call sequence << 32) | quant8 scale bits. Carrying the scale in
// the flag means no chunk has to read (or write) a shared header line.
__device__ __forceinline__ uint64_t flag_word(float scale) {
  return ((uint64_t)s_seq << 32) | __float_as_uint(scale);
}

// Lane 0 spins until the flag carries this call's sequence. Returns the
// flag word (0 on timeout or abort). Polls with relaxed loads and a short
// exponential back-off (thousands of warps poll at once; acquire loads in a
// tight loop would flood L2), then takes the acquire with one ld.acquire.
__device__ uint64_t spin_flag(const uint64_t* f, const RingParams& P, const RankCtx& R, Ctl* ctl,
                              ErrWord* err, int phase, int step, int block) {
  uint64_t v = ld_acquire_sys(f);
  if ((uint32_t)(v >> 32) == s_seq) return v;
  const uint64_t t0 = globaltimer();
  uint32_t ns = 32;
  for (uint32_t it = 1;; ++it) {
    if ((uint32_t)(ld_relaxed_sys(f) >> 32) == s_seq) return ld_acquire_sys(f);
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
    if ((it & 63u) == 0) {
      if (aborted(P, ctl)) {
        latch_error(err, kErrTimeout, phase, step, block, R.rank, kAbortConsequence);
        return 0;
      }
      if (globaltimer() - t0 > P.timeout_ns) {
        latch_error(err, kErrTimeout, phase, step, block, R.rank, 0);
        broadcast_abort(P, R);
        return 0;
      }
    }
  }
}

// Warp: wait for (slot, chunk) of this rank's inbox and take the scale from
// the flag word. With chunk 0 the slot header is validated like
// collective.py:_expect (:52-64, :109-114): block index, iteration tag and
// length must be what this rank expects.
__device__ bool warp_await(const RingParams& P, const RankCtx& R, Ctl* ctl, ErrWord* err, int slot,
                           uint32_t c, int phase, int step, int block, uint64_t len, float& scale) {
  int ok = 1;
  uint32_t sb = 0;
  if (lane_id() == 0) {
    const uint64_t v = spin_flag(flag_ptr(R.inbox, P.L, slot, c), P, R, ctl, err, phase, step, block);
    ok = v != 0;
    sb = (uint32_t)v;
    if (ok && c == 0) {
      const SlotHdr* h = hdr_ptr(R.inbox, P.L, slot);
      const uint32_t hb = __ldcg(&h->block), hi = __ldcg(&h->iteration), hn = __ldcg(&h->n_elems);
      if (hb != (uint32_t)block || hi != s_iter || hn != (uint32_t)len) {
        latch_error(err, kErrHeader, phase, step, block, R.rank, (int)hn);
        broadcast_abort(P, R);
        ok = 0;
      }
    }
  }
  __syncwarp();
  ok = __shfl_sync(0xffffffffu, ok, 0);
  scale = __uint_as_float(__shfl_sync(0xffffffffu, sb, 0));
  return ok;
}

__device__ __forceinline__ void write_hdr(const RingParams& P, uint8_t* dst, int slot, int block,
                                          uint64_t len, float scale) {
  SlotHdr* h = hdr_ptr(dst, P.L, slot);
  h->seq = s_seq;
  h->iteration = s_iter;
  h->block = (uint32_t)block;
  h->n_elems = (uint32_t)len;
  h->scale = scale;
}

// Warp: after this warp's payload stores to `dst`, release the chunk flag
// at system scope (chunk 0 also carries the slot header).
__device__ __forceinline__ void warp_publish(const RingParams& P, uint8_t* dst, int slot, uint32_t c,
                                             int block, uint64_t len, float scale) {
  __syncwarp();
  if (lane_id() == 0) {
    if (c == 0) write_hdr(P, dst, slot, block, len, scale);
#ifdef PIPESGD_EXP_NOFENCE  // timing experiment only (no ordering: results may be wrong)
    st_relaxed_sys(flag_ptr(dst, P.L, slot, c), flag_word(scale));
#else
    st_release_sys(flag_ptr(dst, P.L, slot, c), flag_word(scale));  // release: orders the warp's stores
#endif
  }
}

// Warp: publish chunk c of the owned block to every peer's allgather slot.
__device__ __forceinline__ void warp_publish_all(const RingParams& P, const RankCtx& R, int b, uint32_t c,
                                                 uint64_t len, float scale) {
  __syncwarp();
  if (lane_id() == 0) {
    if (c == 0)
      for (int d = 1; d < P.p; ++d) write_hdr(P, R.peer[(R.rank + d) % P.p], ag_slot(P.p, b), b, len, scale);
#ifndef PIPESGD_EXP_NOFENCE
    fence_sys();  // one system fence, then relaxed flag stores to every peer
#endif
    for (int d = 1; d < P.p; ++d)
      st_relaxed_sys(flag_ptr(R.peer[(R.rank + d) % P.p], P.L, ag_slot(P.p, b), c), flag_word(scale));
  }
}

// quant8: rank-wide barrier over all G CTAs of one rank carrying the block
// max. The CTA's warps meet in shared memory; the last warp of the CTA to
// arrive publishes the CTA max and one arrival to the rank's control block
// (4x fewer same-address atomics than per-warp arrivals, which serialised in
// L2) and polls for the rank count; the other warps spin on shared memory.
// Returns false on abort/timeout (a warp that left early never arrives: the
// rest time out, as everywhere else in the kernel).
__device__ bool warp_barrier_max(const RingParams& P, const RankCtx& R, Ctl* ctl, ErrWord* err, int k,
                                 uint32_t mymax, float& vmax, int step) {
  // every lane's earlier stores and the warp's global max-slot atomics are
  // ordered before its arrival: __syncwarp orders the lanes, and the fences
  // below are cumulative over what lane 0 has observed
  __syncwarp();
  const uint32_t m = warp_max_u32(mymax);
  int ok = 1;
  float v = 0.f;
  if (lane_id() == 0) {
    atomicMax(&s_bar_max[k], m);
    __threadfence();  // this warp's global writes (e.g. the pre-compress own-block max slot) before arriving
    const unsigned prev = atomicAdd(&s_bar_arrived[k], 1u);
    const uint64_t t0 = globaltimer();
    if (prev == (unsigned)kWarps - 1 && P.G == 1) {
      // a one-CTA launch (small calls): the CTA is the whole rank, so the
      // shared-memory meeting is the barrier -- no global arrival, fence or poll
      *(volatile float*)&s_bar_vmax[k] = __uint_as_float(*(volatile unsigned*)&s_bar_max[k]);
      __threadfence_block();
      *(volatile int*)&s_bar_open[k] = 1;
      v = *(volatile float*)&s_bar_vmax[k];
    } else if (prev == (unsigned)kWarps - 1) {  // last warp of the CTA: the CTA's global arrival
      atomicMax(&cb(ctl)->maxslot[k], ((unsigned long long)s_seq << 32) | *(volatile unsigned*)&s_bar_max[k]);
      __threadfence();
      atomicAdd(&cb(ctl)->bar, 1ull);
      const unsigned long long target = (unsigned long long)(k + 1) * P.G;
      for (uint32_t it = 1; ld_acquire_gpu(reinterpret_cast<uint64_t*>(&cb(ctl)->bar)) < target; ++it) {
        __nanosleep(32);
        if ((it & 63u) == 0) {
          if (aborted(P, ctl)) {
            latch_error(err, kErrTimeout, kPhBarrier, step, -1, R.rank, kAbortConsequence);
            ok = 0;
            break;
          }
          if (globaltimer() - t0 > P.timeout_ns) {
            latch_error(err, kErrTimeout, kPhBarrier, step, -1, R.rank, 0);
            broadcast_abort(P, R);
            ok = 0;
            break;
          }
        }
      }
      const unsigned long long w = ld_acquire_gpu(reinterpret_cast<uint64_t*>(&cb(ctl)->maxslot[k]));
      v = ((uint32_t)(w >> 32) == s_seq) ? __uint_as_float((uint32_t)w) : 0.f;
      *(volatile float*)&s_bar_vmax[k] = v;
      __threadfence_block();
      *(volatile int*)&s_bar_open[k] = ok ? 1 : 2;
    } else {
      int st;
      for (uint32_t it = 1; (st = *(volatile int*)&s_bar_open[k]) == 0; ++it) {
        __nanosleep(32);
        if ((it & 63u) == 0) {
          if (aborted(P, ctl)) {
            latch_error(err, kErrTimeout, kPhBarrier, step, -1, R.rank, kAbortConsequence);
            st = 2;
            break;
          }
          if (globaltimer() - t0 > P.timeout_ns) {
            latch_error(err, kErrTimeout, kPhBarrier, step, -1, R.rank, 0);
            broadcast_abort(P, R);
            st = 2;
            break;
          }
        }
      }
      __threadfence_block();
      ok = st == 1;
      v = *(volatile float*)&s_bar_vmax[k];
    }
  }
  __syncwarp();
  ok = __shfl_sync(0xffffffffu, ok, 0);
  vmax = __shfl_sync(0xffffffffu, v, 0);
  return ok;
}

// Iterate this lane's groups of chunk c of block B in 1024-element batches;
// all loads of a batch are issued before any of its stores.
#ifndef PIPESGD_Q8_UNROLL
#define PIPESGD_Q8_UNROLL 1
#endif
#ifndef PIPESGD_FLAG_STATIC
#define PIPESGD_FLAG_STATIC 0  // A/B knob: static chunk stride for the flag protocol too
#endif
// Direct reduce-scatter send jobs destination-fastest (job j -> peer j % (p-1),
// chunk j / (p-1)), so every moment's stores spread over all owners: p = 4
// codec none 64 MiB 202 -> 195 us, 256 MiB 686-724 -> 675 us
// (profiles/r02/direct_order_ab/); 0 = block-major.
#ifndef PIPESGD_DIRECT_INTERLEAVE
#define PIPESGD_DIRECT_INTERLEAVE 1
#endif
#ifndef PIPESGD_LL_STATIC
#define PIPESGD_LL_STATIC 1
#endif
#ifndef PIPESGD_LL_UNROLL
#define PIPESGD_LL_UNROLL 1
#endif
template <int C, bool LLM = false, typename L, typename S>
__device__ __forceinline__ void for_groups(const RingParams& P, const Blk& B, uint32_t c, L&& load, S&& use) {
  constexpr int E = CodecT<C>::E;
  // groups per lane per batch: 1024-element batches, except quant8 whose
  // 16-element groups and encode temporaries would spill at the 128-register
  // budget with two in flight, and the LL protocol: its chunks are 128
  // elements (one group per lane), and every unrolled copy of an LL poll +
  // encode + line store is instruction bytes a latency-bound call fetches
  // cold (the none kernel was 246 KB of SASS)
  constexpr int U = C == kQuant8 ? PIPESGD_Q8_UNROLL : LLM ? PIPESGD_LL_UNROLL : (int)kBatch / (32 * E);
  constexpr uint64_t kB = 32ull * E * U;
  const int lane = lane_id();
  const uint64_t cbase = B.A + (uint64_t)c * P.chunk;
  const uint64_t lo = max(B.start, cbase);
  const uint64_t hi = min(B.start + B.len, cbase + P.chunk);
  for (uint64_t b0 = cbase; b0 < hi; b0 += kB) {
    using T = decltype(load(b0, lo, hi, 0, E));
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t g0 = b0 + (uint64_t)(u * 32 + lane) * E;
      if (g0 < hi && g0 + E > lo) v[u] = load(g0, lo, hi, (int)(max(lo, g0) - g0), (int)(min(hi, g0 + E) - g0));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t g0 = b0 + (uint64_t)(u * 32 + lane) * E;
      if (g0 < hi && g0 + E > lo) use(g0, lo, hi, (int)(max(lo, g0) - g0), (int)(min(hi, g0 + E) - g0), v[u]);
    }
  }
}

// Optional timeline (debug/profiling): lane 0 of warp `wid` stamps slot k.
__device__ __forceinline__ void stamp(const RingParams& P, uint32_t wid, int lrank, int k) {
  if (P.trace != nullptr && (threadIdx.x & 31) == 0)
    P.trace[((uint64_t)lrank * P.G * kWarps + wid) * kTraceSlots + k] = globaltimer();
}

// p == 2 only (slots 4..13 belong to reduce-scatter steps s >= 1 otherwise):
// finer per-chunk stamps for the fold phase, first chunk of each warp.
__device__ __forceinline__ void stamp2(const RingParams& P, uint32_t wid, int lrank, int k, bool on) {
  if (on && P.p == 2) stamp(P, wid, lrank, kTrP2 + k - 4);
}

// Chunk scheduling: in every phase warp w first takes chunk w (no atomic,
// so a small call's warps never wait on the counter), then further chunks
// from a counter in the rank's control block (reset when the call closes),
// offset by the rank's warp count NW. Flags are per chunk, not per warp, so
// ranks need not agree on which warp handles which chunk; fast warps take
// more chunks, which evens out the unequal NVLink shares warps get under
// arbitration.
// Phases: 0 quant8 step-0 max, 1 step-0 send, 2+2s fold of step s,
// 3+2s quant8 push of step s, 20+k allgather of the k-th block.
__device__ __forceinline__ uint32_t grab(Ctl* ctl, int phase, uint32_t nw) {
  uint32_t c = 0;
  if ((threadIdx.x & 31) == 0) c = (uint32_t)atomicAdd(&cb(ctl)->next[phase], 1ull) + nw;
  return __shfl_sync(0xffffffffu, c, 0);
}

template <int E>
struct XIn {
  FV<E> x;
  uint4 in;
};

// Second max slot of a quant8 barrier (fused pre-compress: the own block's
// raw max). Each warp atomically maxes it before its barrier arrival, so it
// is complete once warp_barrier_max returned.
__device__ __forceinline__ float read_max_slot(Ctl* ctl, int idx) {
  uint32_t w = 0;
  if (lane_id() == 0) {
    const unsigned long long x = ld_acquire_gpu(reinterpret_cast<uint64_t*>(&cb(ctl)->maxslot[idx]));
    w = ((uint32_t)(x >> 32) == s_seq) ? (uint32_t)x : 0u;
  }
  return __uint_as_float(__shfl_sync(0xffffffffu, w, 0));
}

}  // namespace

#ifdef PIPESGD_CHECKED
// Bounds-checked build: every payload / vector / LL access of the ring must
// fall inside this rank's x (read only), out, slot output, or ONE region of
// some rank's inbox (the control area, a single payload slot, a single LL
// slot), so an indexing slip into a neighbouring slot is caught too. A
// refused access is skipped and latched as kErrBounds in the rank's error
// word (GP_FAIL_BOUNDS on the host).
namespace {
__device__ bool inbox_region_ok(const Layout& L, uint64_t off, uint64_t end) {
  if (end > L.total_bytes) return false;
  if (off < L.off_payload) return end <= L.off_payload;
  if (off < L.off_ll) return end <= L.off_payload + ((off - L.off_payload) / L.slot_bytes + 1) * L.slot_bytes;
  return end <= L.off_ll + ((off - L.off_ll) / L.ll_slot_bytes + 1) * L.ll_slot_bytes;
}
}  // namespace

__device__ __noinline__ void bounds_violation(uint64_t addr) {
  const RankCtx& R = s_P->rk[blockIdx.x / s_P->G];
  latch_error(reinterpret_cast<ErrWord*>(R.inbox + s_P->L.off_err), kErrBounds, kPhLocal, 0, -1, R.rank,
              (int)(uint32_t)addr);
}

__device__ __noinline__ bool ring_access_ok(const void* ptr, uint64_t bytes, bool write) {
  const RingParams& P = *s_P;
  const RankCtx& R = P.rk[blockIdx.x / P.G];
  const uint64_t a = reinterpret_cast<uint64_t>(ptr), b = a + bytes;
  const uint64_t w = P.codec == kNone ? 4 : P.codec == kTrunc16 ? 2 : 1;
  auto in = [&](const void* base, uint64_t len) {
    const uint64_t lo = reinterpret_cast<uint64_t>(base);
    return base != nullptr && a >= lo && b <= lo + len;
  };
  bool ok = (!write && in(R.x, 4 * P.n)) || in(R.out, 4 * P.n) || in(R.slot, w * P.n);
  for (int q = 0; q < P.p && !ok; ++q) {
    const uint64_t base = reinterpret_cast<uint64_t>(R.peer[q]);
    if (a >= base && a < base + P.L.total_bytes) {
      ok = inbox_region_ok(P.L, a - base, b - base);
      // the bytes a real run moves over NVLink: stores into another rank's inbox
      if (ok && write && q != R.rank)
        atomicAdd(&reinterpret_cast<Ctl*>(R.inbox + P.L.off_ctl)->wire_bytes, (unsigned long long)bytes);
    }
  }
  if (!ok) bounds_violation(a);
  return ok;
}
#endif

template <int C, bool LL, bool PRE>
__device__ __forceinline__ void ring_body(const RingParams& P) {
  constexpr int E = CodecT<C>::E;
  const int G = P.G;
  const int lr = blockIdx.x / G;
  const uint32_t wid = (blockIdx.x % G) * kWarps + (threadIdx.x >> 5);
  const uint32_t NW = (uint32_t)G * kWarps;  // this rank's warps in this launch
  const RankCtx& R = P.rk[lr];
  const int p = P.p, r = R.rank, succ = (r + 1) % p;
  Ctl* ctl = reinterpret_cast<Ctl*>(R.inbox + P.L.off_ctl);
  ErrWord* err = reinterpret_cast<ErrWord*>(R.inbox + P.L.off_err);
  const float* __restrict__ x = R.x;
  float* out = R.out;
  const bool slot_mode = R.slot != nullptr;
  int bad = 0;
  // Next chunk of a phase for this warp. The flag protocol takes it from the
  // phase counter (fast warps take more chunks: NVLink arbitration gives
  // warps unequal shares); the LL protocol strides statically -- its chunks
  // are short, so a shared counter meant thousands of same-address atomics
  // per phase on large LL blocks, and its warps wait on the data anyway.
  auto next = [&](int phase, uint32_t cur) -> uint32_t {
    if constexpr ((LL && PIPESGD_LL_STATIC) || PIPESGD_FLAG_STATIC) return cur + NW;
    else return grab(ctl, phase, NW);
  };
  stamp(P, wid, lr, 0);
#ifdef PIPESGD_CHECKED
  if (P.selftest && wid == 0 && out != nullptr) {  // negative control: one group past the end of out
    FV<4> z = {};
    store_fv<4>(out, P.n, P.n, P.n + 4, z);
  }
#endif
  // an earlier call failed on some rank: this one ends at once, reported as
  // a consequence of the peer's failure (no timeout wait)
  if (s_abort & kAbortSticky) {
    if (wid == 0 && lane_id() == 0) latch_error(err, kErrTimeout, kPhRS, 0, -1, r, 1);
    return;
  }

  // Local pre-compress fused into every load of x (engine.py:333, :355/:400:
  // the ring input is D(C(grad)) under the whole-vector codec). For quant8
  // its scale needs max|grad| over the whole vector: one extra read pass.
  Q8 q0 = q8_make(0.f);
  auto px = [&](FV<E> v) -> FV<E> {
    if constexpr (PRE) {
      if constexpr (C != kQuant8) {  // quant8: the whole-vector max pass already checked every x
#pragma unroll
        for (int i = 0; i < E; ++i) bad |= nonfinite(v.v[i]);
      }
      if constexpr (C == kTrunc16) {
#pragma unroll
        for (int i = 0; i < E; ++i) v.v[i] = t16_decode(t16_encode(v.v[i]));
      } else if constexpr (C == kQuant8) {
#pragma unroll
        for (int i = 0; i < E; ++i) v.v[i] = q8_decode(q8_encode(v.v[i], q0), q0.s);
      }
    }
    return v;
  };

  // LL protocol state (ring.cuh:ll_payload_limit): per-lane give-up flag for
  // polls (1 = this rank's timeout, 2 = a peer aborted the call). quant8's
  // block scale travels in the header line's 4th word (not in flags).
  constexpr bool ll = LL;
  uint64_t ll_t0 = 0;
  int ll_fail = 0;
  auto give_up = [&]() -> bool {
    if (ll_fail) return true;
    if (aborted(P, ctl)) {
      ll_fail = 2;  // an abort (this rank's or a peer's): a consequence
      return true;
    }
    const uint64_t now = globaltimer();
    if (!ll_t0) ll_t0 = now;
    else if (now - ll_t0 > P.timeout_ns) ll_fail = 1;
    return ll_fail != 0;
  };
  auto ll_load = [&](const uint8_t* llslot, uint64_t rel0) -> uint4 {
    uint4 v = make_uint4(0, 0, 0, 0);
    if (!ll_fail) ll_get(ll_line<C>(const_cast<uint8_t*>(llslot), rel0), v, give_up);
    return v;
  };
  // chunk 0 carries the slot header line (collective.py:_expect, :52-64)
  auto ll_hdr_put = [&](uint8_t* llslot, uint32_t c, int block, uint64_t len, float scale) {
    if (c == 0 && lane_id() == 0)
      ll_put(llslot, make_uint4((uint32_t)block, s_iter, (uint32_t)len, __float_as_uint(scale)));
  };
  // warp: any lane gave up -> latch like warp_await and leave
  auto ll_ok = [&](int phase, int step, int block) -> bool {
    const int any = __any_sync(0xffffffffu, ll_fail != 0), own = __any_sync(0xffffffffu, ll_fail == 1);
    if (!any) return true;
    if (lane_id() == 0) {
      latch_error(err, kErrTimeout, phase, step, block, r, own ? 0 : kAbortConsequence);
      if (own) broadcast_abort(P, R);
    }
    return false;
  };
  auto ll_hdr_get = [&](const uint8_t* llslot, uint32_t c, int phase, int step, int block, uint64_t len,
                        float& scale) -> bool {
    int ok = 1;
    uint32_t sb = 0;
    if ((c == 0 || C == kQuant8) && lane_id() == 0) {
      uint4 h;
      if (ll_get(const_cast<uint8_t*>(llslot), h, give_up)) {
        sb = h.w;
        if (c == 0 && (h.x != (uint32_t)block || h.y != s_iter || h.z != (uint32_t)len)) {
          latch_error(err, kErrHeader, phase, step, block, r, (int)h.z);
          broadcast_abort(P, R);
          ok = 0;
        }
      }
    }
    ok = __shfl_sync(0xffffffffu, ok, 0);
    scale = __uint_as_float(__shfl_sync(0xffffffffu, sb, 0));
    return ok && ll_ok(phase, step, block);
  };

  // ---- codec none, p >= 3: direct reduce-scatter over NVSwitch. The ring's
  // p-1 dependent hops become one: every rank pushes each block it does not
  // own straight to the block's owner (slot d = its fold position), and the
  // owner folds s_0 = x_b, s_k = fl(x_{b+k} + s_{k-1}) over the slots in the
  // reference's order (collective.py:99-115; D(C(.)) is the identity for
  // codec none, so the bits are the ring's). Same wire bytes per rank.
  const bool own_via_inbox = slot_mode && C == kQuant8;  // owner re-quantises later, with the global scale
  auto direct_rs = [&]() -> bool {
    const int own = (r + 1) % p;
    uint32_t NCH = 0;
    for (int b = 0; b < p; ++b) NCH = max(NCH, get_blk(P, b).nch);
    const Q8 q = q8_make(0.f);
    // send: block b = (r - d) % p goes to its owner (b - 1) % p, slot d
    for (uint32_t j = wid; j < (uint32_t)(p - 1) * NCH; j = next(1, j)) {
      const int d = PIPESGD_DIRECT_INTERLEAVE ? (int)(j % (uint32_t)(p - 1)) : (int)(j / NCH);
      const uint32_t c = PIPESGD_DIRECT_INTERLEAVE ? j / (uint32_t)(p - 1) : j % NCH;
      const int b = (r - d + p) % p;
      const Blk B = get_blk(P, b);
      if (c >= B.nch) continue;
      const int o = (b - 1 + p) % p;
      uint8_t* dst = slot_ptr(R.peer[o], P.L, rs_slot(d));
      uint8_t* lld = ll_ptr(R.peer[o], P.L, rs_slot(d));
      for_groups<C, LL>(P, B, c,
                    [&](uint64_t g0, uint64_t lo, uint64_t hi, int, int) { return load_fv<E>(x, g0, lo, hi); },
                    [&](uint64_t g0, uint64_t, uint64_t, int vlo, int vhi, const FV<E>& v) {
                      const uint4 pk = encode_v<C>(px(v), q, bad);
                      if (ll) ll_put(ll_line<C>(lld, g0 - B.A), pk);
                      else store_pay<C>(dst, g0 - B.A, vlo, vhi, pk);
                    });
      if (ll) ll_hdr_put(lld, c, b, B.len, 0.f);
      else warp_publish(P, R.peer[o], rs_slot(d), c, b, B.len, 0.f);
    }
    if (__any_sync(0xffffffffu, bad) && lane_id() == 0) latch_error(err, kErrNonFinite, kPhRS, 0, r, r, 0);
    bad = 0;
    stamp(P, wid, lr, 1);
    // fold the owned block over slots 0 .. p-2 and the own x, then push the
    // result to every peer's allgather slot (the ring's last hop)
    const Blk B = get_blk(P, own);
    constexpr int U = LL ? 1 : 2;  // groups per lane per batch: U x p loads in flight
    bool first = true;
    for (uint32_t c = wid; c < B.nch; c = next(2, c)) {
      if (ll) {
        float sdum;
        for (int d = 0; d < p - 1; ++d)
          if (!ll_hdr_get(ll_ptr(R.inbox, P.L, rs_slot(d)), c, kPhRS, d, own, B.len, sdum)) return false;
      } else {
        // lane d waits for slot d's chunk flag (p - 1 waits in parallel)
        int ok = 1;
        const int d = lane_id();
        if (d < p - 1) {
          const uint64_t v = spin_flag(flag_ptr(R.inbox, P.L, rs_slot(d), c), P, R, ctl, err, kPhRS, d, own);
          ok = v != 0;
          if (ok && c == 0) {
            const SlotHdr* h = hdr_ptr(R.inbox, P.L, rs_slot(d));
            const uint32_t hb = __ldcg(&h->block), hi = __ldcg(&h->iteration), hn = __ldcg(&h->n_elems);
            if (hb != (uint32_t)own || hi != s_iter || hn != (uint32_t)B.len) {
              latch_error(err, kErrHeader, kPhRS, d, own, r, (int)hn);
              broadcast_abort(P, R);
              ok = 0;
            }
          }
        }
        if (!__all_sync(0xffffffffu, ok)) return false;
      }
      if (first) stamp(P, wid, lr, tr_step(0, 0));
      first = false;
      const uint64_t cbase = B.A + (uint64_t)c * P.chunk;
      const uint64_t lo = max(B.start, cbase), hi = min(B.start + B.len, cbase + P.chunk);
      for (uint64_t b0 = cbase; b0 < hi; b0 += 32ull * E * U) {
        uint4 in[U][kMaxRanks - 1];
        FV<E> xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t g0 = b0 + (uint64_t)(u * 32 + lane_id()) * E;
          if (g0 < hi && g0 + E > lo) {
            const int vlo = (int)(max(lo, g0) - g0), vhi = (int)(min(hi, g0 + E) - g0);
            xv[u] = load_fv<E>(x, g0, lo, hi);
#pragma unroll
            for (int d = 0; d < kMaxRanks - 1; ++d)
              if (d < p - 1)
                in[u][d] = ll ? ll_load(ll_ptr(R.inbox, P.L, rs_slot(d)), g0 - B.A)
                              : load_pay<C>(slot_ptr(R.inbox, P.L, rs_slot(d)), g0 - B.A, vlo, vhi);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t g0 = b0 + (uint64_t)(u * 32 + lane_id()) * E;
          if (!(g0 < hi && g0 + E > lo)) continue;
          const int vlo = (int)(max(lo, g0) - g0), vhi = (int)(min(hi, g0 + E) - g0);
          FV<E> acc = decode_v<C>(in[u][0], 0.f);  // s_0 = x_b
#pragma unroll
          for (int d = 1; d < kMaxRanks - 1; ++d)
            if (d < p - 1) {
              (void)encode_v<C>(acc, q, bad);  // the reference compresses s_{d-1} (finite check)
              acc = add_v(decode_v<C>(in[u][d], 0.f), acc);
            }
          (void)encode_v<C>(acc, q, bad);
          acc = add_v(px(xv[u]), acc);  // s_{p-1} = x_own + s_{p-2}
          const uint4 pk = encode_v<C>(acc, q, bad);
          for (int k = 1; k < p; ++k) {
            if (ll) ll_put(ll_line<C>(ll_ptr(R.peer[(r + k) % p], P.L, ag_slot(p, own)), g0 - B.A), pk);
            else store_pay<C>(slot_ptr(R.peer[(r + k) % p], P.L, ag_slot(p, own)), g0 - B.A, vlo, vhi, pk);
          }
          if (slot_mode) store_pay<C>(R.slot, g0, vlo, vhi, pk);
          else store_fv<E>(out, g0, lo, hi, acc);
        }
      }
      if (ll && !ll_ok(kPhRS, p - 2, own)) return false;
      if (ll) {
        for (int k = 1; k < p; ++k) ll_hdr_put(ll_ptr(R.peer[(r + k) % p], P.L, ag_slot(p, own)), c, own, B.len, 0.f);
      } else {
        warp_publish_all(P, R, own, c, B.len, 0.f);
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane_id() == 0) latch_error(err, kErrNonFinite, kPhAG, 0, own, r, 0);
    bad = 0;
    stamp(P, wid, lr, tr_step(0, 3));
    return true;
  };

  if (C == kNone && P.direct) {
    if (!direct_rs()) return;
  } else {
    // ---- reduce-scatter step 0, send side: C(x_r[block r]) -> succ slot 0
    {
      const Blk B = get_blk(P, r);
      Q8 q = q8_make(0.f);
      if constexpr (C == kQuant8) {
        float vmax;
        if constexpr (!PRE) {
          uint32_t m = 0;
          const uint64_t keep = l2_evict_last();  // the send pass below re-reads the block
          for (uint32_t c = wid; c < B.nch; c = next(0, c))
            for_groups<C, LL>(P, B, c,
                          [&](uint64_t g0, uint64_t lo, uint64_t hi, int, int) {
                            return load_fv_pol<E>(x, g0, lo, hi, keep);
                          },
                          [&](uint64_t, uint64_t, uint64_t, int, int, const FV<E>& v) { m = max(m, absmax_bits(v)); });
          if (!warp_barrier_max(P, R, ctl, err, 0, m, vmax, 0)) return;
          if (nonfinite(vmax)) bad = 1;  // compress() rejects the block (compression.py:108-109)
        } else {
          // one pass over the whole local vector: max|x| (pre-compress scale)
          // and max|x| over the own block, whose D(C(.)) maximum is
          // D(C(max|x_r|)) because encode/decode are monotone in |x|
          Blk W;
          W.start = 0; W.len = P.n; W.A = 0;
          W.nch = P.n ? (uint32_t)((P.n + P.chunk - 1) / P.chunk) : 0u;
          uint32_t m = 0, mo = 0;
          for (uint32_t c = wid; c < W.nch; c = next(0, c))
            for_groups<C, LL>(P, W, c,
                          [&](uint64_t g0, uint64_t lo, uint64_t hi, int, int) { return load_fv<E>(x, g0, lo, hi); },
                          [&](uint64_t g0, uint64_t, uint64_t, int, int, const FV<E>& v) {
                            m = max(m, absmax_bits(v));
  #pragma unroll
                            for (int i = 0; i < E; ++i) {
                              const uint64_t g = g0 + i;
                              if (g >= B.start && g < B.start + B.len) mo = max(mo, __float_as_uint(v.v[i]) & 0x7FFFFFFFu);
                            }
                          });
          // own-block maximum goes through a second max slot before the
          // barrier arrival so it is complete when the barrier opens
          const uint32_t mow = warp_max_u32(mo);
          if (lane_id() == 0) atomicMax(&cb(ctl)->maxslot[8], ((unsigned long long)s_seq << 32) | mow);
          float xmax;
          if (!warp_barrier_max(P, R, ctl, err, 0, m, xmax, 0)) return;
          const float own = read_max_slot(ctl, 8);
          if (nonfinite(xmax)) bad = 1;  // reference compress() rejects the whole local vector
          q0 = q8_make(q8_scale(xmax));
          vmax = fabsf(q8_decode(q8_encode(own, q0), q0.s));
        }
        q = q8_make(q8_scale(vmax));
        stamp(P, wid, lr, kTrQ8Max);
      }
      uint8_t* dst = slot_ptr(R.peer[succ], P.L, rs_slot(0));
      uint8_t* lld = ll_ptr(R.peer[succ], P.L, rs_slot(0));
      bool first0 = true;
      for (uint32_t c = wid; c < B.nch; c = next(1, c)) {
        for_groups<C, LL>(P, B, c,
                      [&](uint64_t g0, uint64_t lo, uint64_t hi, int, int) { return load_fv<E>(x, g0, lo, hi); },
                      [&](uint64_t g0, uint64_t, uint64_t, int vlo, int vhi, const FV<E>& v) {
                        // quant8: finiteness is known from the block max
                        const uint4 pk = encode_v<C, C != kQuant8>(px(v), q, bad);
                        if (ll) ll_put(ll_line<C>(lld, g0 - B.A), pk);
                        else store_pay<C>(dst, g0 - B.A, vlo, vhi, pk);
                      });
        stamp2(P, wid, lr, 7, first0);
        if (ll) ll_hdr_put(lld, c, r, B.len, q.s);
        else warp_publish(P, R.peer[succ], rs_slot(0), c, r, B.len, q.s);
        stamp2(P, wid, lr, 8, first0);
        first0 = false;
      }
      if (__any_sync(0xffffffffu, bad) && lane_id() == 0) latch_error(err, kErrNonFinite, kPhRS, 0, r, r, 0);
      bad = 0;
      stamp(P, wid, lr, 1);
    }

    // ---- reduce-scatter steps: fold block (r-s-1)%p, forward (or own it)
    for (int s = 0; s < p - 1; ++s) {
      const int b = (r - s - 1 + p) % p;
      const Blk B = get_blk(P, b);
      const bool last = (s == p - 2);
      const uint8_t* in_slot = slot_ptr(R.inbox, P.L, rs_slot(s));
      uint8_t* fwd = last ? nullptr : slot_ptr(R.peer[succ], P.L, rs_slot(s + 1));
      const uint8_t* ll_in = ll_ptr(R.inbox, P.L, rs_slot(s));
      uint8_t* ll_fwd = last ? nullptr : ll_ptr(R.peer[succ], P.L, rs_slot(s + 1));
      auto load_xin = [&](uint64_t g0, uint64_t lo, uint64_t hi, int vlo, int vhi) {
        return XIn<E>{load_fv<E>(x, g0, lo, hi), ll ? ll_load(ll_in, g0 - B.A) : load_pay<C>(in_slot, g0 - B.A, vlo, vhi)};
      };
      auto emit = [&](uint64_t g0, uint64_t lo, uint64_t hi, int vlo, int vhi, const uint4& pk, float sc) {
        if (!last) {
          if (ll) ll_put(ll_line<C>(ll_fwd, g0 - B.A), pk);
          else store_pay<C>(fwd, g0 - B.A, vlo, vhi, pk);
        } else {
          for (int d = 1; d < p; ++d) {
            if (ll) ll_put(ll_line<C>(ll_ptr(R.peer[(r + d) % p], P.L, ag_slot(p, b)), g0 - B.A), pk);
            else store_pay<C>(slot_ptr(R.peer[(r + d) % p], P.L, ag_slot(p, b)), g0 - B.A, vlo, vhi, pk);
          }
          if (own_via_inbox) {
            if (ll) ll_put(ll_line<C>(ll_ptr(R.inbox, P.L, ag_slot(p, b)), g0 - B.A), pk);
            else store_pay<C>(slot_ptr(R.inbox, P.L, ag_slot(p, b)), g0 - B.A, vlo, vhi, pk);
          } else if (slot_mode)
            store_pay<C>(R.slot, g0, vlo, vhi, pk);  // none/trunc16: C(D(wire)) == wire
          else
            store_fv<E>(out, g0, lo, hi, decode_v<C>(pk, sc));
        }
      };
      auto publish_last = [&](uint32_t c, float sc) {
        if (ll) {
          for (int d = 1; d < p; ++d) ll_hdr_put(ll_ptr(R.peer[(r + d) % p], P.L, ag_slot(p, b)), c, b, B.len, sc);
          if (own_via_inbox) ll_hdr_put(ll_ptr(R.inbox, P.L, ag_slot(p, b)), c, b, B.len, sc);
          return;
        }
        warp_publish_all(P, R, b, c, B.len, sc);
        if (own_via_inbox && lane_id() == 0) {
          if (c == 0) write_hdr(P, R.inbox, ag_slot(p, b), b, B.len, sc);
          st_release_sys(flag_ptr(R.inbox, P.L, ag_slot(p, b), c), flag_word(sc));
        }
      };

      if constexpr (C != kQuant8) {
        const Q8 q = q8_make(0.f);
        bool first = true;
        for (uint32_t c = wid; c < B.nch; c = next(2 + 2 * s, c)) {
          float sin = 0.f;
          stamp2(P, wid, lr, 4, first);
          if (ll) {
            if (!ll_hdr_get(ll_in, c, kPhRS, s, b, B.len, sin)) return;
          } else if (!warp_await(P, R, ctl, err, rs_slot(s), c, kPhRS, s, b, B.len, sin)) {
            return;
          }
          if (first) stamp(P, wid, lr, tr_step(s, 0));
          for_groups<C, LL>(P, B, c, load_xin,
                        [&](uint64_t g0, uint64_t lo, uint64_t hi, int vlo, int vhi, const XIn<E>& v) {
                          emit(g0, lo, hi, vlo, vhi, encode_v<C>(add_v(px(v.x), decode_v<C>(v.in, sin)), q, bad),
                               0.f);
                        });
          if (ll && !ll_ok(kPhRS, s, b)) return;
          stamp2(P, wid, lr, 5, first);
          if (!last) {
            if (ll) ll_hdr_put(ll_fwd, c, b, B.len, 0.f);
            else warp_publish(P, R.peer[succ], rs_slot(s + 1), c, b, B.len, 0.f);
          } else {
            publish_last(c, 0.f);
          }
          stamp2(P, wid, lr, 6, first);
          first = false;
        }
      } else {
        // pass A: fold and reduce the block max. The partial sum is not
        // stored: pass B recomputes it from the same x and inbox bytes (the
        // same single fp32 add, so the same bits). pass A's loads mark their
        // lines L2 evict_last, so when the hop's x block and inbox fit the
        // 126 MB L2 (C3 at p >= 4: 61 + 15 MB) pass B re-reads them on chip
        // instead of a 4 B/elem partial written to HBM and read back.
        const uint64_t keep = l2_evict_last(), drop = l2_evict_first();
        auto load_xin_pol = [&](uint64_t g0, uint64_t lo, uint64_t hi, int vlo, int vhi, uint64_t pol) {
          return XIn<E>{load_fv_pol<E>(x, g0, lo, hi, pol),
                        ll ? ll_load(ll_in, g0 - B.A) : load_pay_pol<C>(in_slot, g0 - B.A, vlo, vhi, pol)};
        };
        uint32_t m = 0;
        bool first = true;
        for (uint32_t c = wid; c < B.nch; c = next(2 + 2 * s, c)) {
          float sin;
          if (ll) {
            if (!ll_hdr_get(ll_in, c, kPhRS, s, b, B.len, sin)) return;
          } else if (!warp_await(P, R, ctl, err, rs_slot(s), c, kPhRS, s, b, B.len, sin)) {
            return;
          }
          if (first) stamp(P, wid, lr, tr_step(s, 0));
          first = false;
          for_groups<C, LL>(P, B, c,
                        [&](uint64_t g0, uint64_t lo, uint64_t hi, int vlo, int vhi) {
                          return load_xin_pol(g0, lo, hi, vlo, vhi, keep);
                        },
                        [&](uint64_t, uint64_t, uint64_t, int, int, const XIn<E>& v) {
                          m = max(m, absmax_bits(add_v(px(v.x), decode_v<C>(v.in, sin))));
                        });
          if (ll && !ll_ok(kPhRS, s, b)) return;
        }
        float vmax;
        stamp(P, wid, lr, tr_step(s, 1));  // pass A done
        if (!warp_barrier_max(P, R, ctl, err, s + 1, m, vmax, s)) return;
        stamp(P, wid, lr, tr_step(s, 2));  // barrier open
        if (nonfinite(vmax)) bad = 1;  // pass A's block max covers every value pass B encodes
        const Q8 q = q8_make(q8_scale(vmax));
        // pass B: recompute the partial, encode it with the block scale and
        // push it. Any warp may take any chunk: the chunk's flag (or LL
        // lines) already carries this call's sequence, so the waits below
        // return at once and hand this warp the chunk's incoming scale.
        for (uint32_t c = wid; c < B.nch; c = next(3 + 2 * s, c)) {
          float sin;
          if (ll) {
            if (!ll_hdr_get(ll_in, c, kPhRS, s, b, B.len, sin)) return;
          } else if (!warp_await(P, R, ctl, err, rs_slot(s), c, kPhRS, s, b, B.len, sin)) {
            return;
          }
          for_groups<C, LL>(P, B, c,
                        [&](uint64_t g0, uint64_t lo, uint64_t hi, int vlo, int vhi) {
                          return load_xin_pol(g0, lo, hi, vlo, vhi, drop);
                        },
                        [&](uint64_t g0, uint64_t lo, uint64_t hi, int vlo, int vhi, const XIn<E>& v) {
                          const FV<E> acc = add_v(px(v.x), decode_v<C>(v.in, sin));
                          emit(g0, lo, hi, vlo, vhi, encode_v<C, false>(acc, q, bad), q.s);
                        });
          if (ll && !ll_ok(kPhRS, s, b)) return;
          if (!last) {
            if (ll) ll_hdr_put(ll_fwd, c, b, B.len, q.s);
            else warp_publish(P, R.peer[succ], rs_slot(s + 1), c, b, B.len, q.s);
          } else {
            publish_last(c, q.s);
          }
        }
      }
      if (__any_sync(0xffffffffu, bad) && lane_id() == 0)
        latch_error(err, kErrNonFinite, last ? kPhAG : kPhRS, last ? 0 : s + 1, b, r, 0);
      bad = 0;
      stamp(P, wid, lr, tr_step(s, 3));
    }
  }

  // ---- slot mode, quant8: the pipe re-compress (engine.py:407) needs the
  // whole-vector scale of the summed vector. Every block's codes reach 127,
  // so max|sum| = 127 * max_b s_b, known from the block scales in the
  // allgather flag words: no pass over the sum, and the result equals the
  // reference's compress(summed) scale exactly.
  Q8 qs = q8_make(0.f);
  if (own_via_inbox) {
    float vmax = 0.f;
    int ok = 1;
    if (lane_id() == 0) {
      for (int b = 0; b < p && ok; ++b) {
        const Blk B = get_blk(P, b);
        if (B.nch == 0) continue;
        uint32_t sb = 0;
        if (ll) {  // the block scale sits in the LL header line of the allgather slot
          uint4 h;
          ok = ll_get(ll_ptr(R.inbox, P.L, ag_slot(p, b)), h, give_up);
          sb = h.w;
        } else {
          const uint64_t v = spin_flag(flag_ptr(R.inbox, P.L, ag_slot(p, b), 0), P, R, ctl, err, kPhAG,
                                       (r - b + p) % p, b);
          ok = v != 0;
          sb = (uint32_t)v;
        }
        if (ok) vmax = fmaxf(vmax, __fmul_rn(127.f, __uint_as_float(sb)));
      }
    }
    __syncwarp();
    if (ll && !ll_ok(kPhAG, 0, -1)) return;
    if (!__shfl_sync(0xffffffffu, ok, 0)) return;
    qs = q8_make(q8_scale(__shfl_sync(0xffffffffu, vmax, 0)));
    if (wid == 0 && lane_id() == 0) *R.slot_scale = qs.s;
  } else if (slot_mode && wid == 0 && lane_id() == 0) {
    *R.slot_scale = 0.f;
  }

  // ---- allgather, receive side: every other owner's bytes (and, for the
  // quant8 slot, the own block) -> out (decoded) or the compressed slot
  for (int k = own_via_inbox ? 0 : 1; k < p; ++k) {
    const int b = (r + 1 + k) % p;  // own block is (r+1)%p
    const Blk B = get_blk(P, b);
    const int step = (r - b + p) % p;  // reference allgather step that delivers block b
    const uint8_t* in_slot = slot_ptr(R.inbox, P.L, ag_slot(p, b));
    const uint8_t* ll_in = ll_ptr(R.inbox, P.L, ag_slot(p, b));
    bool first = true;
    for (uint32_t c = wid; c < B.nch; c = next(20 + k, c)) {
      float sin = 0.f;
      stamp2(P, wid, lr, 9, first && k == 1);
      if (ll) {
        if (!ll_hdr_get(ll_in, c, kPhAG, step, b, B.len, sin)) return;
      } else if (!warp_await(P, R, ctl, err, ag_slot(p, b), c, kPhAG, step, b, B.len, sin)) {
        return;
      }
      if (k == 1 && first) stamp(P, wid, lr, kTrAgIn);
      first = false;
      for_groups<C, LL>(P, B, c,
                    [&](uint64_t g0, uint64_t, uint64_t, int vlo, int vhi) {
                      return ll ? ll_load(ll_in, g0 - B.A) : load_pay<C>(in_slot, g0 - B.A, vlo, vhi);
                    },
                    [&](uint64_t g0, uint64_t lo, uint64_t hi, int vlo, int vhi, const uint4& v) {
                      if (!slot_mode) {
                        store_fv<E>(out, g0, lo, hi, decode_v<C>(v, sin));
                      } else if constexpr (C == kQuant8) {
                        store_pay<C>(R.slot, g0, vlo, vhi, encode_v<C, false>(decode_v<C>(v, sin), qs, bad));
                      } else {
                        store_pay<C>(R.slot, g0, vlo, vhi, v);
                      }
                    });
      if (ll && !ll_ok(kPhAG, step, b)) return;
    }
  }
  stamp(P, wid, lr, kTrEnd);
}

#ifndef PIPESGD_RING_MINBLOCKS
#define PIPESGD_RING_MINBLOCKS (2048 / kRingThreads / 4 > 0 ? 2048 / kRingThreads / 4 : 1)
#endif
// PRE (the fused local pre-compress) is a template parameter like the codec
// and the protocol: each kernel carries only the code its calls execute, and
// a small call fetches that code cold (see for_groups).
template <int C, bool LL, bool PRE>
__global__ void __launch_bounds__(kRingThreads, PIPESGD_RING_MINBLOCKS)
    ring_allreduce_kernel(const __grid_constant__ RingParams P) {
  const int lr = blockIdx.x / P.G;
  Ctl* ctl = reinterpret_cast<Ctl*>(P.rk[lr].inbox + P.L.off_ctl);
  if (threadIdx.x == 0) {
#ifdef PIPESGD_CHECKED
    s_P = &P;
#endif
    const unsigned long long calls = ld_acquire_gpu(reinterpret_cast<uint64_t*>(&ctl->calls));
    s_calls = calls;
    s_seq = next_seq(calls);
    s_bank = (uint32_t)(calls & 1);
    s_abort = *(volatile unsigned long long*)&ctl->abort;
    // explicit branch + asm load: a volatile dereference inside a select here
    // built a kernel that faulted (even with a null pointer)
    uint32_t it = P.iteration;
    if (P.iteration_dev != nullptr) it = ld_relaxed_gpu_u32(P.iteration_dev);
    s_iter = it;
    for (int i = 0; i < kMaxBarriers; ++i) s_bar_arrived[i] = 0, s_bar_max[i] = 0, s_bar_open[i] = 0;
    if (blockIdx.x % P.G == 0) {  // the next call's bank starts from zero
      CtlBank* nb = &ctl->bank[(calls + 1) & 1];
      nb->bar = 0;
      nb->exits = 0;
      for (int i = 0; i < 32; ++i) nb->next[i] = 0;
      for (int i = 0; i < 16; ++i) nb->maxslot[i] = 0;
    }
  }
  __syncthreads();
  ring_body<C, LL, PRE>(P);  // returns early (per warp) on timeout / abort / header mismatch
  // The last warp of this rank to leave closes the call by advancing the call
  // count. The next call on this stream starts only after this kernel has
  // completed, which also makes the bank zeroing above visible to it.
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    const unsigned long long prev = atomicAdd(&cb(ctl)->exits, 1ull);
    if (prev == (unsigned long long)P.G * kWarps - 1) *(volatile unsigned long long*)&ctl->calls = s_calls + 1;
  }
}

// every ring kernel instantiation, indexed [codec][ll][pre]
#define GP_RING_FNS(C) \
  {{(const void*)ring_allreduce_kernel<C, false, false>, (const void*)ring_allreduce_kernel<C, false, true>}, \
   {(const void*)ring_allreduce_kernel<C, true, false>, (const void*)ring_allreduce_kernel<C, true, true>}}
static const void* const kRingFns[3][2][2] = {GP_RING_FNS(kNone), GP_RING_FNS(kTrunc16), GP_RING_FNS(kQuant8)};
#undef GP_RING_FNS

void launch_ring(const RingParams& P, int nlocal, cudaStream_t stream, cudaError_t* err) {
  void* args[] = {const_cast<RingParams*>(&P)};
  const dim3 grid(P.G * nlocal), block(kRingThreads);
  const void* fn = kRingFns[P.codec][P.ll ? 1 : 0][P.pre ? 1 : 0];
  // Emulated rings (nlocal > 1) need every CTA co-resident: cooperative
  // launch. A single rank per GPU only needs its G <= #SM CTAs to become
  // resident eventually (no CTA waits on a CTA of its own launch except the
  // quant8 rank barrier, and G CTAs always fit once other kernels drain), so
  // it can take the cheaper ordinary launch.
  static const int mode = [] {
    const char* e = std::getenv("PIPESGD_LAUNCH");
    return e ? std::atoi(e) : 1;
  }();
  if (nlocal > 1 || mode == 0) {
    *err = cudaLaunchCooperativeKernel(fn, grid, block, args, 0, stream);
  } else {
    *err = cudaLaunchKernel(fn, grid, block, args, 0, stream);
  }
}

int ring_warps_per_cta() { return kWarps; }

int ring_max_ctas_per_sm() {
  int m = 1 << 30;
  for (const auto& per_codec : kRingFns)
    for (const auto& per_ll : per_codec)
      for (const void* f : per_ll) {
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, f, kRingThreads, 0);
        m = std::min(m, std::max(b, 1));
      }
  return m;
}

}  // namespace gp
