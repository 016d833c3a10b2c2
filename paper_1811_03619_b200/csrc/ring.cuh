// Fused compressed ring AllReduce — shared declarations between the kernel
// (ring.cu) and the communicator (comm.cu).
#pragma once

#include "common.cuh"

namespace gp {

#ifndef PIPESGD_RING_THREADS
#define PIPESGD_RING_THREADS 128
#endif
constexpr int kRingThreads = PIPESGD_RING_THREADS;
constexpr int kRingWarps = kRingThreads / 32;
#ifndef PIPESGD_MIN_CHUNK
#define PIPESGD_MIN_CHUNK 1024
#endif
constexpr uint32_t kMinChunk = PIPESGD_MIN_CHUNK;  // elements per warp chunk; flags are sized for this
constexpr uint32_t kMaxChunk = 16384;  // default largest warp chunk (64 KiB of fp32)

// Per-rank inbox layout (identical on every rank of a communicator). Peers
// write payload, headers and flags here over NVLink; ctl/err are private.
// Low-latency (LL) protocol for small blocks: every 8-byte word carries 4
// payload bytes and the call's sequence number, so a receiver polls the data
// itself and no release fence / flag store is needed, at twice the bytes.
// A call of any codec takes it (quant8's block scale rides in the header
// line's fourth word) when its block payload (elements incl. the
// 16-element alignment slack x wire width) fits the 2 MiB LL slot. Measured
// (profiles/r02/ll_region_ab/, after the LL path's code shrank to one group
// per lane): 2 MiB blocks beat the flag protocol at p = 2 (codec none at
// C1's 2.6 MB 34 -> 25 us, trunc16 at 4 MiB 26 -> 19 us, quant8 at 8 MiB
// 43 -> 35 us) and at p = 4 (none at 6 MiB 70 -> 57 us, trunc16 at 12 MiB
// 67 -> 57 us); a 4 MiB slot lost at p = 4 (none at 12 MiB 79 -> 105 us).
// Compile-time constants, so every rank makes the same choice.
#ifndef PIPESGD_LL_HOP_BYTES
#define PIPESGD_LL_HOP_BYTES (1u << 20)
#endif
#ifndef PIPESGD_LL_REGION_BYTES
#define PIPESGD_LL_REGION_BYTES (2u << 20)
#endif
constexpr uint64_t kLLHopBytes = PIPESGD_LL_HOP_BYTES;
constexpr uint64_t kLLRegionBytes = PIPESGD_LL_REGION_BYTES;  // largest LL block payload (fixed: layouts agree)

// hop budget x (p - 1), twice it at p = 2, capped by the slot: 2 MiB for
// every p at the defaults
__host__ __device__ inline uint64_t ll_payload_limit(int p) {
  const uint64_t v = p == 2 ? 2 * kLLHopBytes : kLLHopBytes * (uint64_t)(p > 1 ? p - 1 : 1);
  return v < kLLRegionBytes ? v : kLLRegionBytes;
}

struct Layout {
  uint64_t off_ctl, off_err, off_hdr, off_flags, off_payload;
  uint64_t slot_bytes;   // payload bytes per slot
  uint64_t off_ll;       // LL region: nslot x ll_slot_bytes (32-byte header line + 2 x 16 B per group)
  uint64_t ll_slot_bytes;
  uint64_t ll_cap;       // largest block payload (bytes, incl. alignment slack) an LL slot holds
  uint64_t total_bytes;
  uint32_t max_chunks;   // flags per slot
  uint32_t nslot;        // 2p-1: p-1 reduce-scatter slots + p allgather slots
};

// Per-call scratch of the control block, double-banked: call k (k = the raw
// count of completed calls) uses bank k & 1 and zeroes bank (k + 1) & 1 at its
// start, so no call has to reset its counters (and fence) on the way out.
struct CtlBank {
  unsigned long long bar;          // quant8 barrier arrivals in the call
  unsigned long long exits;        // warps that finished the call
  unsigned long long next[32];     // per-phase chunk counters (dynamic chunk scheduling)
  unsigned long long maxslot[16];  // (seq << 32) | absmax bits, per quant8 barrier
};

struct Ctl {                   // rank-private control block (peers write abort / ack)
  unsigned long long calls;    // raw count of completed calls: seq = next_seq(calls)
  unsigned long long abort;    // kAbortSticky | rank + 1 | seq of the call that failed (0 = healthy)
  CtlBank bank[2];
  unsigned long long ack[kMaxRanks];  // star calls: == seq once rank q consumed this rank's data
  unsigned long long barflag[kMaxRanks];  // gp_comm_barrier: generation rank q reached (written by q)
  unsigned long long wire_bytes;          // bounds-checked build: payload bytes this rank stored into peers
};
static_assert(sizeof(Ctl) <= 2048, "ctl block: the p = 1 codec status lives at +2048");

// A failed call (timeout, header mismatch) poisons the communicator on every
// rank: the abort word keeps bit 63 set, so every later call -- not only the
// one that failed -- stops at once instead of waiting out its own timeout
// (the reference's run ends at the first failed recv, collective.py:157-161;
// the Python endpoint is unusable after a CollectiveError). Bits [39:32] hold
// the aborting rank + 1: a warp that sees its own rank's abort was waiting
// for the same missing peer (its own timeout), not for a failed peer.
constexpr unsigned long long kAbortSticky = 1ull << 63;

__device__ __forceinline__ unsigned long long abort_word(const Ctl* ctl) {
  return *(const volatile unsigned long long*)&ctl->abort;
}
__device__ __forceinline__ bool comm_aborted(const Ctl* ctl) { return (abort_word(ctl) & kAbortSticky) != 0; }
// A warp that stops on an abort latches a consequence (timeout kind, detail
// 1), whichever rank raised it: the warp that raised it has latched the cause
// itself (its own timeout, a header mismatch, ...) before broadcasting, and a
// cause outranks every consequence in the error word. (Reporting this rank's
// own abort as another timeout let it outrank a header mismatch at the same
// step, since timeout sorts first.)
constexpr int kAbortConsequence = 1;

// Poison this communicator on every rank (peers' ctl blocks over NVLink).
// Out of line: an error path, reached from every wait site.
inline __device__ __noinline__ void abort_all(uint8_t* const* peer, int p, uint64_t off_ctl, uint32_t seq, int rank) {
  const unsigned long long w = kAbortSticky | ((unsigned long long)((rank + 1) & 0xFF) << 32) | seq;
  for (int q = 0; q < p; ++q) {
    Ctl* c = reinterpret_cast<Ctl*>(peer[q] + off_ctl);
    atomicCAS(&c->abort, 0ull, w);  // the first abort names its rank
  }
  fence_sys();
}

// Call sequence numbers cycle through 1 .. 2^32 - 1: never 0 (the value of
// zero-initialised flags and LL words), and every check compares for
// equality, so the 32-bit sequence may wrap (a rank is never more than one
// call ahead of the data it reads). `calls` itself only counts up.
__host__ __device__ inline uint32_t next_seq(unsigned long long calls) {
  return (uint32_t)(calls % 0xFFFFFFFFull) + 1u;
}

struct SlotHdr {               // written by the sender before each chunk flag
  uint32_t seq, iteration, block, n_elems;
  float scale;
  uint32_t pad[11];
};

struct RankCtx {
  const float* x;              // this rank's input vector (n)
  float* out;                  // this rank's output vector (n); quant8 scratch in slot mode
  uint8_t* slot;               // slot mode: C(sum) payload (n * width bytes), else null
  float* slot_scale;           // slot mode: its whole-vector scale
  uint8_t* inbox;              // this rank's inbox (local HBM)
  uint8_t* peer[kMaxRanks];    // every rank's inbox as seen from this GPU
  int rank;
};

struct RingParams {
  RankCtx rk[kMaxRanks];       // one entry per rank in this launch (1, or p when emulated)
  Layout L;
  uint64_t n;
  uint64_t timeout_ns;
  uint32_t iteration;
  const uint32_t* iteration_dev;  // non-null: read the tag here at kernel entry (graph replays)
  uint32_t chunk;              // elements per chunk, multiple of 8, >= kMinChunk
  int p, codec, G;             // world size, codec tag, CTAs per rank (kRingWarps warp workers each)
  int pre;                     // x is the raw gradient: apply the local D(C(.)) on load
  int ll;                      // this call uses the LL protocol (see ll_payload_limit)
  int direct;                  // codec none, p >= 3: direct reduce-scatter (one hop, ring.cu)
  int selftest;                // bounds-checked build only: one deliberate store past `out` (negative control)
  unsigned long long* trace;   // optional timeline: kTraceSlots %globaltimer stamps per warp
};

// Ring timeline slots (per warp, %globaltimer ns): [0] start, [1] step-0 send
// done, [2] quant8 step-0 max barrier open, step s: [3+4s] first chunk in,
// [4+4s] quant8 pass A done, [5+4s] quant8 barrier open, [6+4s] step done;
// [35] allgather first in, [36] end; p = 2: [37-42] the first chunk's
// fold / send / allgather sub-stamps.
constexpr int kTraceSlots = 44;
constexpr int kTrQ8Max = 2, kTrAgIn = 35, kTrEnd = 36, kTrP2 = 37;
__host__ __device__ inline int tr_step(int s, int k) { return 3 + 4 * s + k; }

__host__ __device__ inline int rs_slot(int s) { return s; }
__host__ __device__ inline int ag_slot(int p, int b) { return p - 1 + b; }

// partition_blocks (collective.py:35-49)
__host__ __device__ inline void block_range(uint64_t n, int p, int b, uint64_t& start, uint64_t& len) {
  const uint64_t base = n / p, extra = n % p;
  start = (uint64_t)b * base + ((uint64_t)b < extra ? (uint64_t)b : extra);
  len = base + ((uint64_t)b < extra ? 1 : 0);
}

void launch_ring(const RingParams& P, int nlocal, cudaStream_t stream, cudaError_t* err);

// Star collectives (star.cu): gather-sum to a root / broadcast from a root.
struct StarLaunch {
  Layout L;
  uint64_t n, timeout_ns;
  int p, root, mode, zero_first, ctas, nlocal;
  int max_ctas;  // co-residency cap of one launch (SM count; emulated: all ranks' CTAs)
  const float* ins[kMaxRanks];
  float* outs[kMaxRanks];
  uint8_t* inboxes[kMaxRanks];
  uint8_t* peers[kMaxRanks];
  int ranks[kMaxRanks];
};
cudaError_t launch_star(const StarLaunch& S, cudaStream_t stream);
int ring_max_ctas_per_sm();  // occupancy of the ring kernel (worst codec)

}  // namespace gp
