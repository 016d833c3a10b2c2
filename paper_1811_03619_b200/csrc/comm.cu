// Communicator: inbox allocation, peer mapping (in-process peer access or
// CUDA IPC between torchrun processes), ring launch, traffic accounting and
// device error reporting. Replaces the reference transport for this path
// (transport.py:44-177) — send/recv disappear into the fused kernel; the
// endpoint bookkeeping (rank, world, timeout, stats) stays.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <string>

#include "../../include/pipesgd.h"
#include "ring.cuh"

using namespace gp;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const std::string& what) {
  return fail(GP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

uint64_t round_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

Layout make_layout(int p, uint64_t max_elems) {
  Layout L{};
  const uint64_t maxblk = (max_elems + p - 1) / p;
  L.nslot = (uint32_t)(2 * p - 1);
  L.slot_bytes = round_up((maxblk + 32) * 4, 256);
  L.max_chunks = (uint32_t)((maxblk + 16 + kMinChunk - 1) / kMinChunk + 1);
  L.off_ctl = 0;
  L.off_err = 4096;
  L.off_hdr = 4096 + 256;
  L.off_flags = round_up(L.off_hdr + (uint64_t)L.nslot * sizeof(SlotHdr), 256);
  L.off_payload = round_up(L.off_flags + (uint64_t)L.nslot * L.max_chunks * 8, 4096);
  // LL slot: a 32-byte header line + 2 x the payload of the largest block
  // (+ the launch's 16-element slack, fp32 worst case) up to kLLRegionBytes
  L.ll_cap = std::min<uint64_t>(4 * (maxblk + 16), kLLRegionBytes);
  L.ll_slot_bytes = round_up(32 + 2 * (L.ll_cap + 4 * 32), 256);
  L.off_ll = L.off_payload + (uint64_t)L.nslot * L.slot_bytes;
  L.total_bytes = L.off_ll + (uint64_t)L.nslot * L.ll_slot_bytes;
  return L;
}

}  // namespace

void gp_set_error_string(const std::string& m) { g_err = m; }

struct gp_comm {
  int rank = 0, world = 1, device = 0;
  uint64_t max_elems = 0;
  Layout L{};
  int nlocal = 1;                       // p when emulated
  int share = 1;                        // per-rank communicators launched on this comm's device
  uint8_t* inbox[kMaxRanks] = {};       // local allocations (1, or p when emulated)
  uint8_t* peer[kMaxRanks] = {};        // every rank's inbox as mapped on this device
  bool ipc_opened[kMaxRanks] = {};
  bool connected = false;
  uint32_t seq = 0;
  int G = 0;
  double timeout_s = 30.0;
  gp_stats stats[kMaxRanks] = {};
  unsigned long long* trace = nullptr;  // optional device timeline buffer
  const uint32_t* iteration_dev = nullptr;  // optional device-resident iteration tag
  uint64_t bar_gen = 0;                 // gp_comm_barrier generations issued
  uint64_t ll_max = ~0ull;              // gp_comm_set_protocol: largest LL block payload (bytes)
};

namespace {

int alloc_inbox(gp_comm* c, int i) {
  cudaError_t e = cudaMalloc(&c->inbox[i], c->L.total_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(inbox)");
  // Flags, headers, ctl, error word and the LL region (its words carry
  // sequence numbers) must start at zero; payload need not.
  e = cudaMemset(c->inbox[i], 0, c->L.off_payload);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemset(inbox)");
  e = cudaMemset(c->inbox[i] + c->L.off_ll, 0, c->L.total_bytes - c->L.off_ll);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemset(LL region)");
  e = cudaMemset(c->inbox[i] + c->L.off_err, 0xFF, sizeof(unsigned long long));  // no error
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemset(error word)");
  return GP_OK;
}

int sm_count(int device) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return sms;
}

// Default CTA budget: up to 16 warps per SM on every SM, never more CTAs
// than can be resident at once (the quant8 rank barrier needs all of them).
int default_ctas(int device) {
  return std::max(1, sm_count(device) * std::min(16 / kRingWarps, ring_max_ctas_per_sm()));
}

void count_message(gp_stats& s, int codec, uint64_t len) {
  const uint64_t w = codec == GP_CODEC_NONE ? 4 : codec == GP_CODEC_TRUNC16 ? 2 : 1;
  s.messages += 1;
  s.payload_bytes += len * w;
  s.frame_bytes += 11 + 9 + len * w;  // transport.py:37 frame + compression.py:33 header
}

// Reference accounting: rank r sends blocks (r-s)%p in reduce-scatter and
// (r+1-s)%p in allgather, s = 0..p-2 (collective.py:97-99, :125-127).
void account(gp_stats& s, int rank, int p, uint64_t n, int codec) {
  for (int st = 0; st < p - 1; ++st) {
    uint64_t off, len;
    block_range(n, p, ((rank - st) % p + p) % p, off, len);
    count_message(s, codec, len);
  }
  for (int st = 0; st < p - 1; ++st) {
    uint64_t off, len;
    block_range(n, p, ((rank + 1 - st) % p + p) % p, off, len);
    count_message(s, codec, len);
  }
}

uint64_t env_u64(const char* name, uint64_t dflt) {
  const char* e = std::getenv(name);
  return e ? std::strtoull(e, nullptr, 10) : dflt;
}

// Chunk size (elements) for one call: the block split over all warp workers,
// at least 1024 elements and at most 64 KiB of payload. A chunk is the unit
// of one system-scope release; measured on 2xB200 (profiles/), more parallel
// chunks beat fewer releases below 64 MB, and at 64 KiB per release the fence
// costs ~2% (tools/p2p_pattern_probe.py). Dynamic scheduling evens out the rest.
uint32_t pick_chunk(uint64_t n, int p, int G, int codec) {
  static const uint64_t min_bytes = env_u64("PIPESGD_MIN_CHUNK_BYTES", 0);
  static const uint64_t max_bytes = env_u64("PIPESGD_MAX_CHUNK_BYTES", 65536);
  static const uint64_t per_warp = std::max<uint64_t>(1, env_u64("PIPESGD_CHUNKS_PER_WARP", 1));
  const uint64_t w = codec == GP_CODEC_NONE ? 4 : codec == GP_CODEC_TRUNC16 ? 2 : 1;
  const uint64_t lo = std::max<uint64_t>(kMinChunk, round_up(min_bytes / w, kMinChunk));
  const uint64_t hi = std::max<uint64_t>(lo, round_up(max_bytes / w, kMinChunk));
  const uint64_t maxblk = (n + p - 1) / p + 16;
  // chunk indexing depends on G, so G is a communicator-wide setting (the
  // transports pass the same CTA budget on every rank and check it)
  const uint64_t workers = (uint64_t)G * kRingWarps * per_warp;
  const uint64_t ch = round_up((maxblk + workers - 1) / workers, kMinChunk);
  return (uint32_t)std::max(lo, std::min(hi, ch));
}

struct RingPlan {
  uint32_t chunk;  // elements per chunk (from the communicator-wide G: every rank agrees)
  int ctas;        // CTAs this call launches
  int ll;          // LL protocol
  uint64_t nch;    // chunks in the largest phase
  int direct;      // codec none, p >= 3: direct reduce-scatter (one hop instead of p - 1)
};

// Launch plan of one ring call. Launch only as many warps as the largest
// phase has chunks: the chunk size (and so every flag index) still follows
// the communicator-wide G, but small calls no longer start G CTAs whose warps
// would only hammer the phase counters (2p same-address atomics per idle
// warp). LL when the block payload fits ll_payload_limit(p) and the slot.
RingPlan plan_ring(uint64_t n, int p, int G, int codec, int pre, uint64_t ll_cap) {
  RingPlan r{};
  const uint64_t maxblk = (n + p - 1) / p + 16;
  const uint64_t w = codec == GP_CODEC_NONE ? 4 : codec == GP_CODEC_TRUNC16 ? 2 : 1;
  r.ll = (maxblk * w <= std::min<uint64_t>(ll_payload_limit(p), ll_cap)) ? 1 : 0;
  r.chunk = pick_chunk(n, p, G, codec);
  // LL uses no flags, so its chunk only sets how many warps share a block: a
  // receiving lane polls its lines one after another, so shorter chunks (more
  // warps, fewer polls each) cut the latency chain -- 128 elements for
  // none / trunc16 (p = 4: 16 KiB 45 -> 22 us, C1's 2.6 MB 51 -> 35 us), 256
  // for quant8 blocks up to 64 Ki elements; larger quant8 blocks keep the
  // flag-protocol chunk (every extra warp adds a rank-barrier arrival per hop).
  // profiles/r02/ll_chunk_ab/. PIPESGD_LL_CHUNK (elements) overrides.
  static const uint64_t ll_env = env_u64("PIPESGD_LL_CHUNK", 0);
  const uint64_t ll_chunk = ll_env ? ll_env
                            : codec != GP_CODEC_QUANT8 ? 128 : (maxblk <= 65552 ? 256 : 0);
  if (r.ll && ll_chunk) {
    const uint64_t workers = (uint64_t)G * kRingWarps;
    r.chunk = (uint32_t)std::max<uint64_t>(round_up(ll_chunk, 16), round_up((maxblk + workers - 1) / workers, 16));
  }
  r.nch = (maxblk + r.chunk - 1) / r.chunk;
  if (pre && codec == GP_CODEC_QUANT8) r.nch = std::max<uint64_t>(r.nch, (n + r.chunk - 1) / r.chunk);
  r.ctas = (int)std::min<uint64_t>((uint64_t)G, std::max<uint64_t>(1, (r.nch + kRingWarps - 1) / kRingWarps));
  // codec none folds D(C(.)) = identity, so the owner can fold every rank's
  // raw block in the ring's order after one NVSwitch hop: bit-identical
  // sums, identical wire bytes; PIPESGD_DIRECT=0 keeps the ring
  static const uint64_t direct_on = env_u64("PIPESGD_DIRECT", 1);
  r.direct = (direct_on && codec == GP_CODEC_NONE && p >= 3) ? 1 : 0;
  return r;
}

int check_common(gp_comm* c, uint64_t n, int codec) {
  if (!c) return fail(GP_ERR_ARG, "null communicator");
  if (codec < 0 || codec > 2) return fail(GP_ERR_ARG, "unknown codec " + std::to_string(codec));
  if (n > c->max_elems && c->world > 1)
    return fail(GP_ERR_ARG, "vector of " + std::to_string(n) + " elems exceeds communicator capacity " +
                                std::to_string(c->max_elems));
  if (n >= (1ull << 32) * (uint64_t)c->world) return fail(GP_ERR_ARG, "block exceeds 2^32 elements");
  return GP_OK;
}

bool misaligned(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) != 0; }

}  // namespace

extern "C" {

const char* gp_last_error_string(void) { return g_err.c_str(); }
int gp_version(void) { return 1; }

int gp_comm_create(int rank, int world, int device, uint64_t max_elems, gp_comm** out) {
  if (!out) return fail(GP_ERR_ARG, "null out");
  if (world < 1 || world > kMaxRanks) return fail(GP_ERR_ARG, "world size must be in [1, 8]");
  if (rank < 0 || rank >= world)
    return fail(GP_ERR_ARG, "rank " + std::to_string(rank) + " outside [0, " + std::to_string(world) + ")");
  DeviceGuard g(device);
  gp_comm* c = new gp_comm();
  c->rank = rank;
  c->world = world;
  c->device = device;
  c->max_elems = std::max<uint64_t>(max_elems, 1);
  c->L = make_layout(world, c->max_elems);
  c->G = default_ctas(device);
  int rc = alloc_inbox(c, 0);
  if (rc) { delete c; return rc; }
  c->peer[rank] = c->inbox[0];
  if (world == 1) c->connected = true;
  *out = c;
  return GP_OK;
}

int gp_comm_create_emulated(int world, int device, uint64_t max_elems, gp_comm** out) {
  if (!out) return fail(GP_ERR_ARG, "null out");
  if (world < 1 || world > kMaxRanks) return fail(GP_ERR_ARG, "world size must be in [1, 8]");
  DeviceGuard g(device);
  gp_comm* c = new gp_comm();
  c->world = world;
  c->device = device;
  c->nlocal = world;
  c->max_elems = std::max<uint64_t>(max_elems, 1);
  c->L = make_layout(world, c->max_elems);
  // all p x G CTAs of the single launch must be co-resident
  const int cap = sm_count(device) * ring_max_ctas_per_sm() / world;
  c->G = std::max(1, std::min(16 * 16 / kRingWarps, cap));
  for (int i = 0; i < world; ++i) {
    int rc = alloc_inbox(c, i);
    if (rc) { for (int k = 0; k < i; ++k) cudaFree(c->inbox[k]); delete c; return rc; }
    c->peer[i] = c->inbox[i];
  }
  c->connected = true;
  *out = c;
  return GP_OK;
}

int gp_comm_ipc_handle(gp_comm* c, void* handle_out) {
  if (!c || !handle_out) return fail(GP_ERR_ARG, "null argument");
  if (c->nlocal != 1) return fail(GP_ERR_STATE, "emulated communicator has no IPC handle");
  DeviceGuard g(c->device);
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, c->inbox[0]);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(handle_out, &h, 64);
  return GP_OK;
}

int gp_comm_connect_ipc(gp_comm* c, const void* handles) {
  if (!c || !handles) return fail(GP_ERR_ARG, "null argument");
  if (c->nlocal != 1) return fail(GP_ERR_STATE, "emulated communicator");
  DeviceGuard g(c->device);
  for (int q = 0; q < c->world; ++q) {
    if (q == c->rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const uint8_t*>(handles) + 64 * q, 64);
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle(rank " + std::to_string(q) + ")");
    c->peer[q] = static_cast<uint8_t*>(ptr);
    c->ipc_opened[q] = true;
  }
  c->connected = true;
  return GP_OK;
}

int gp_comm_connect_local(gp_comm* const* comms, int world) {
  if (!comms || world < 1 || world > kMaxRanks) return fail(GP_ERR_ARG, "bad communicator list");
  for (int i = 0; i < world; ++i)
    if (!comms[i] || comms[i]->world != world || comms[i]->rank != i || comms[i]->nlocal != 1)
      return fail(GP_ERR_ARG, "communicator list must hold ranks 0..world-1 of one world");
  // Ranks may share a GPU: each still gets its own inbox and its own ring
  // launch (cudaLaunchKernel on its own stream, the per-rank path of a real
  // multi-GPU run), and the device's SMs are split between them so that all
  // their launches are resident at once (they wait on each other's flags).
  for (int i = 0; i < world; ++i) {
    int share = 0;
    for (int k = 0; k < world; ++k) share += comms[k]->device == comms[i]->device;
    comms[i]->share = share;
  }
  int G = 1 << 30;
  for (int i = 0; i < world; ++i) {
    const int cap = std::max(1, sm_count(comms[i]->device) * ring_max_ctas_per_sm() / comms[i]->share);
    G = std::min(G, std::min(comms[i]->G, cap));
  }
  for (int i = 0; i < world; ++i) comms[i]->G = G;  // chunking follows G: every rank agrees
  for (int i = 0; i < world; ++i) {
    DeviceGuard g(comms[i]->device);
    for (int k = 0; k < world; ++k) {
      if (k == i) continue;
      comms[i]->peer[k] = comms[k]->inbox[0];
      if (comms[k]->device == comms[i]->device) continue;  // same device: plain pointers
      int can = 0;
      cudaDeviceCanAccessPeer(&can, comms[i]->device, comms[k]->device);
      if (!can)
        return fail(GP_ERR_UNSUPPORTED, "device " + std::to_string(comms[i]->device) +
                                            " cannot access device " + std::to_string(comms[k]->device));
      cudaError_t e = cudaDeviceEnablePeerAccess(comms[k]->device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (e != cudaSuccess) {
        return cuda_fail(e, "cudaDeviceEnablePeerAccess");
      }
    }
    comms[i]->connected = true;
  }
  return GP_OK;
}

int gp_comm_set_tuning(gp_comm* c, int ctas, double timeout_s) {
  if (!c) return fail(GP_ERR_ARG, "null communicator");
  if (ctas > 0) {
    // every CTA of one launch resident at once (emulated: all ranks' CTAs)
    const int cap = std::max(1, sm_count(c->device) * ring_max_ctas_per_sm() / (c->nlocal * c->share));
    c->G = std::min(ctas, cap);
  }
  if (timeout_s > 0) c->timeout_s = timeout_s;
  return GP_OK;
}

int gp_comm_set_protocol(gp_comm* c, uint64_t ll_max_bytes) {
  if (!c) return fail(GP_ERR_ARG, "null communicator");
  c->ll_max = ll_max_bytes;
  return GP_OK;
}

int gp_comm_set_iteration_source(gp_comm* c, const uint32_t* device_tag) {
  if (!c) return fail(GP_ERR_ARG, "null communicator");
  if (device_tag && (reinterpret_cast<uintptr_t>(device_tag) & 3u)) return fail(GP_ERR_ARG, "misaligned tag");
  c->iteration_dev = device_tag;
  return GP_OK;
}

int gp_comm_set_trace(gp_comm* c, void* device_buffer) {
  if (!c) return fail(GP_ERR_ARG, "null communicator");
  c->trace = static_cast<unsigned long long*>(device_buffer);
  return GP_OK;
}

int gp_comm_info(gp_comm* c, int64_t* o) {
  if (!c || !o) return fail(GP_ERR_ARG, "null argument");
  o[0] = c->rank; o[1] = c->world; o[2] = c->device; o[3] = (int64_t)c->max_elems;
  o[4] = c->G; o[5] = (int64_t)c->L.total_bytes; o[6] = c->seq; o[7] = c->nlocal > 1 ? 1 : (c->share > 1 ? 2 : 0);
  return GP_OK;
}

int gp_ring_plan(uint64_t n, int world, int ctas, int codec, int flags, uint64_t max_elems, int64_t* out) {
  if (!out) return fail(GP_ERR_ARG, "null out");
  if (world < 2 || world > kMaxRanks) return fail(GP_ERR_ARG, "world size must be in [2, 8]");
  if (codec < 0 || codec > 2) return fail(GP_ERR_ARG, "unknown codec " + std::to_string(codec));
  if (ctas < 1) return fail(GP_ERR_ARG, "ctas must be >= 1");
  const Layout L = make_layout(world, std::max<uint64_t>(max_elems, n));
  const RingPlan pl = plan_ring(n, world, ctas, codec, (flags & GP_RING_PRECOMPRESS) ? 1 : 0, L.ll_cap);
  out[0] = pl.chunk;
  out[1] = pl.ctas;
  out[2] = pl.ll;
  out[3] = (int64_t)pl.nch;
  out[4] = pl.direct;
  return GP_OK;
}

int gp_comm_set_call_counter(gp_comm* c, uint64_t calls) {
  if (!c) return fail(GP_ERR_ARG, "null communicator");
  if (calls > 0xFFFFFFFFull) return fail(GP_ERR_ARG, "call counter holds a 32-bit sequence number");
  DeviceGuard g(c->device);
  for (int i = 0; i < c->nlocal; ++i) {
    const unsigned long long v = calls;
    cudaError_t e = cudaMemcpy(c->inbox[i] + c->L.off_ctl + offsetof(Ctl, calls), &v, sizeof(v),
                               cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "set call counter");
    // the next call's bank follows the counter's parity: start both from zero
    e = cudaMemset(c->inbox[i] + c->L.off_ctl + offsetof(Ctl, bank), 0, sizeof(CtlBank) * 2);
    if (e != cudaSuccess) return cuda_fail(e, "reset ctl banks");
  }
  return GP_OK;
}

int gp_comm_destroy(gp_comm* c) {
  if (!c) return GP_OK;
  DeviceGuard g(c->device);
  for (int q = 0; q < kMaxRanks; ++q)
    if (c->ipc_opened[q]) cudaIpcCloseMemHandle(c->peer[q]);
  for (int i = 0; i < c->nlocal; ++i)
    if (c->inbox[i]) cudaFree(c->inbox[i]);
  delete c;
  return GP_OK;
}

// All-to-all flag barrier over NVSwitch, `rounds` times (the timing model's
// S, the reference's barrier probe harness.py:589-609): one thread per rank
// publishes generation g to every peer's ctl and waits until every peer's
// generation reached g. Writes the elapsed %globaltimer ns to ns_out.
struct PeerTable {
  uint8_t* peer[kMaxRanks];
};

__global__ void barrier_kernel(const __grid_constant__ PeerTable T, uint64_t off_ctl, int p, int rank, uint64_t base,
                               int rounds, uint64_t timeout_ns, unsigned long long* ns_out) {
  Ctl* mine = reinterpret_cast<Ctl*>(T.peer[rank] + off_ctl);
  const uint64_t t0 = globaltimer();
  for (int k = 1; k <= rounds; ++k) {
    const unsigned long long g = base + k;
    for (int q = 0; q < p; ++q)
      if (q != rank) st_release_sys(reinterpret_cast<uint64_t*>(&reinterpret_cast<Ctl*>(T.peer[q] + off_ctl)->barflag[rank]), g);
    for (int q = 0; q < p; ++q) {
      if (q == rank) continue;
      while (ld_acquire_sys(reinterpret_cast<const uint64_t*>(&mine->barflag[q])) < g) {
        if (globaltimer() - t0 > timeout_ns) {
          *ns_out = ~0ull;
          return;
        }
      }
    }
  }
  *ns_out = globaltimer() - t0;
}

__global__ void status_to_error_kernel(const gp_codec_status* st, ErrWord* e, int rank) {
  if (st->nonfinite) latch_error(e, kErrNonFinite, kPhRS, 0, rank, rank, 0);
}

// p == 1: the reference's ring is an identity copy (collective.py:153-154);
// the fused flags reduce to the whole-vector codec kernels.
static int launch_single(gp_comm* c, const float* in, float* out, void* slot, float* slot_scale, uint64_t n,
                         int codec, int flags, cudaStream_t st) {
  auto* status = reinterpret_cast<gp_codec_status*>(c->inbox[0] + c->L.off_ctl + 2048);
  auto* errw = reinterpret_cast<ErrWord*>(c->inbox[0] + c->L.off_err);
  int rc = GP_OK;
  if (flags & GP_RING_SLOT_OUT) {
    // C(D(C(x))) == C(x) for every codec (quant8: the scale snaps to itself)
    rc = gp_encode(codec, in, n, slot, status, st);
    if (rc) return rc;
    cudaError_t e = cudaMemcpyAsync(slot_scale, &status->scale, 4, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(slot scale)");
  } else if (flags & GP_RING_PRECOMPRESS) {
    rc = gp_roundtrip(codec, in, out, n, status, st);
    if (rc) return rc;
  } else {
    if (n) {
      cudaError_t e = cudaMemcpyAsync(out, in, n * 4, cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync");
    }
    return GP_OK;
  }
  status_to_error_kernel<<<1, 1, 0, st>>>(status, errw, c->rank);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GP_OK : cuda_fail(e, "status kernel");
}

static int launch(gp_comm* c, const float* const* ins, float* const* outs, void* const* slots,
                  float* const* slot_scales, uint64_t n, int codec, int flags, uint32_t iteration,
                  cudaStream_t st) {
  const int p = c->world;
  if (p == 1)
    return launch_single(c, ins[0], outs[0], slots ? slots[0] : nullptr, slot_scales ? slot_scales[0] : nullptr,
                         n, codec, flags, st);
  RingParams P{};
  P.L = c->L;
  P.n = n;
  P.p = p;
  P.codec = codec;
  P.G = c->G;
  P.pre = (flags & GP_RING_PRECOMPRESS) ? 1 : 0;
  ++c->seq;  // host-side count (info only); the kernel numbers calls on the device
  P.iteration = iteration;
  P.iteration_dev = c->iteration_dev;
  {
    const RingPlan pl = plan_ring(n, p, c->G, codec, P.pre, std::min(c->L.ll_cap, c->ll_max));
    P.chunk = pl.chunk;
    P.G = pl.ctas;
    P.ll = pl.ll;
    P.direct = pl.direct;
  }
  P.timeout_ns = (uint64_t)(c->timeout_s * 1e9);
  P.trace = c->trace;
#ifdef PIPESGD_CHECKED
  P.selftest = std::getenv("PIPESGD_CHECKED_SELFTEST") != nullptr;
#endif
  for (int i = 0; i < c->nlocal; ++i) {
    RankCtx& R = P.rk[i];
    R.x = ins[i];
    R.out = outs[i];
    R.slot = (flags & GP_RING_SLOT_OUT) ? static_cast<uint8_t*>(slots[i]) : nullptr;
    R.slot_scale = (flags & GP_RING_SLOT_OUT) ? slot_scales[i] : nullptr;
    R.rank = c->nlocal == 1 ? c->rank : i;
    R.inbox = c->inbox[i];
    for (int q = 0; q < p; ++q) R.peer[q] = c->peer[q];
  }
  cudaError_t e;
  launch_ring(P, c->nlocal, st, &e);
  if (e != cudaSuccess) return cuda_fail(e, "ring kernel launch");
  for (int i = 0; i < c->nlocal; ++i) account(c->stats[i], P.rk[i].rank, p, n, codec);
  return GP_OK;
}

static int check_flags(gp_comm* c, int flags, uint64_t n, const float* out, void* slot, float* slot_scale,
                       int codec) {
  if (flags & ~(GP_RING_PRECOMPRESS | GP_RING_SLOT_OUT)) return fail(GP_ERR_ARG, "unknown ring flags");
  if (flags & GP_RING_SLOT_OUT) {
    if (n && (!slot || !slot_scale)) return fail(GP_ERR_ARG, "slot output needs a payload and a scale");
    if (n && misaligned(slot)) return fail(GP_ERR_ARG, "slot payload must be 16-byte aligned");
    if (n && codec == GP_CODEC_QUANT8 && c->world > 1 && !out)
      return fail(GP_ERR_ARG, "quant8 slot output needs `out` as scratch");
  } else if (n && !out) {
    return fail(GP_ERR_ARG, "null output");
  }
  return GP_OK;
}

int gp_allreduce(gp_comm* c, const float* in, float* out, uint64_t n, int codec, uint32_t iteration,
                 void* stream) {
  return gp_allreduce_ex(c, in, out, nullptr, nullptr, n, codec, 0, iteration, stream);
}

int gp_allreduce_ex(gp_comm* c, const float* in, float* out, void* slot, float* slot_scale, uint64_t n,
                    int codec, int flags, uint32_t iteration, void* stream) {
  int rc = check_common(c, n, codec);
  if (rc) return rc;
  if (c->nlocal != 1) return fail(GP_ERR_STATE, "use gp_allreduce_emulated on an emulated communicator");
  if (!c->connected) return fail(GP_ERR_STATE, "communicator is not connected to its peers");
  if ((rc = check_flags(c, flags, n, out, slot, slot_scale, codec))) return rc;
  if (n && !in) return fail(GP_ERR_ARG, "null buffer");
  if (n && (misaligned(in) || (out && misaligned(out)))) return fail(GP_ERR_ARG, "buffers must be 16-byte aligned");
  if (n && out && in < out + n && out < in + n) return fail(GP_ERR_ARG, "input and output overlap");
  DeviceGuard g(c->device);
  return launch(c, &in, &out, &slot, &slot_scale, n, codec, flags, iteration, static_cast<cudaStream_t>(stream));
}

int gp_allreduce_emulated(gp_comm* c, const float* const* ins, float* const* outs, uint64_t n, int codec,
                          uint32_t iteration, void* stream) {
  return gp_allreduce_emulated_ex(c, ins, outs, nullptr, nullptr, n, codec, 0, iteration, stream);
}

int gp_allreduce_emulated_ex(gp_comm* c, const float* const* ins, float* const* outs, void* const* slots,
                             float* const* slot_scales, uint64_t n, int codec, int flags, uint32_t iteration,
                             void* stream) {
  int rc = check_common(c, n, codec);
  if (rc) return rc;
  if (c->nlocal == 1 && c->world > 1) return fail(GP_ERR_STATE, "not an emulated communicator");
  for (int i = 0; i < c->nlocal; ++i) {
    if ((rc = check_flags(c, flags, n, outs[i], slots ? slots[i] : nullptr, slot_scales ? slot_scales[i] : nullptr,
                          codec)))
      return rc;
    if (n && !ins[i]) return fail(GP_ERR_ARG, "null buffer");
    if (n && (misaligned(ins[i]) || (outs[i] && misaligned(outs[i]))))
      return fail(GP_ERR_ARG, "buffers must be 16-byte aligned");
  }
  DeviceGuard g(c->device);
  return launch(c, ins, outs, slots, slot_scales, n, codec, flags, iteration, static_cast<cudaStream_t>(stream));
}

// Reference accounting for the star: gather sends one n-element NONE message
// from every non-root rank (collective.py:227-233); broadcast sends one to
// every non-root rank from the root (:265-269).
static int star(gp_comm* c, const float* const* ins, float* const* outs, uint64_t n, int root, int mode,
                int zero_first, cudaStream_t st) {
  if (root < 0 || root >= c->world) return fail(GP_ERR_ARG, "root outside the communicator");
  if (n > c->max_elems) return fail(GP_ERR_ARG, "vector exceeds communicator capacity");
  StarLaunch S{};
  S.L = c->L;
  S.n = n;
  S.timeout_ns = (uint64_t)(c->timeout_s * 1e9);
  S.p = c->world;
  S.root = root;
  S.mode = mode;
  S.zero_first = zero_first;
  S.ctas = std::max(1, c->G / 4);
  S.max_ctas = std::max(1, sm_count(c->device) * std::max(1, 8 / c->nlocal));
  S.nlocal = c->nlocal;
  for (int i = 0; i < c->nlocal; ++i) {
    const int r = c->nlocal == 1 ? c->rank : i;
    if (n && !ins[i]) return fail(GP_ERR_ARG, "null buffer");
    const bool needs_out = mode == 1 || r == root;
    if (n && needs_out && !outs[i]) return fail(GP_ERR_ARG, "null output");
    if (n && (misaligned(ins[i]) || (outs[i] && misaligned(outs[i]))))
      return fail(GP_ERR_ARG, "buffers must be 16-byte aligned");
    S.ins[i] = ins[i];
    S.outs[i] = outs[i];
    S.inboxes[i] = c->inbox[i];
    S.ranks[i] = r;
  }
  for (int q = 0; q < c->world; ++q) S.peers[q] = c->peer[q];
  cudaError_t e = launch_star(S, st);
  if (e != cudaSuccess) return cuda_fail(e, "star kernel launch");
  ++c->seq;
  for (int i = 0; i < c->nlocal; ++i) {
    const int r = c->nlocal == 1 ? c->rank : i;
    if (mode == 0 && r != root) count_message(c->stats[i], GP_CODEC_NONE, n);
    if (mode == 1 && r == root)
      for (int q = 0; q < c->world - 1; ++q) count_message(c->stats[i], GP_CODEC_NONE, n);
  }
  return GP_OK;
}

int gp_gather_sum(gp_comm* c, const float* in, float* out, uint64_t n, int root, int zero_first,
                  uint32_t iteration, void* stream) {
  (void)iteration;
  if (!c || c->nlocal != 1 || !c->connected) return fail(GP_ERR_STATE, "not a connected per-rank communicator");
  DeviceGuard g(c->device);
  return star(c, &in, &out, n, root, 0, zero_first, static_cast<cudaStream_t>(stream));
}

int gp_broadcast(gp_comm* c, const float* in, float* out, uint64_t n, int root, uint32_t iteration,
                 void* stream) {
  (void)iteration;
  if (!c || c->nlocal != 1 || !c->connected) return fail(GP_ERR_STATE, "not a connected per-rank communicator");
  DeviceGuard g(c->device);
  return star(c, &in, &out, n, root, 1, 0, static_cast<cudaStream_t>(stream));
}

int gp_gather_sum_emulated(gp_comm* c, const float* const* ins, float* const* outs, uint64_t n, int root,
                           int zero_first, uint32_t iteration, void* stream) {
  (void)iteration;
  if (!c || (c->nlocal == 1 && c->world > 1)) return fail(GP_ERR_STATE, "not an emulated communicator");
  DeviceGuard g(c->device);
  return star(c, ins, outs, n, root, 0, zero_first, static_cast<cudaStream_t>(stream));
}

int gp_broadcast_emulated(gp_comm* c, const float* const* ins, float* const* outs, uint64_t n, int root,
                          uint32_t iteration, void* stream) {
  (void)iteration;
  if (!c || (c->nlocal == 1 && c->world > 1)) return fail(GP_ERR_STATE, "not an emulated communicator");
  DeviceGuard g(c->device);
  return star(c, ins, outs, n, root, 1, 0, static_cast<cudaStream_t>(stream));
}

int gp_comm_barrier(gp_comm* c, int rounds, void* ns_out, void* stream) {
  if (!c || !ns_out || rounds < 1) return fail(GP_ERR_ARG, "barrier needs a communicator, rounds >= 1, ns_out");
  if (c->nlocal != 1 || !c->connected) return fail(GP_ERR_STATE, "not a connected per-rank communicator");
  DeviceGuard g(c->device);
  PeerTable T{};
  for (int q = 0; q < kMaxRanks; ++q) T.peer[q] = c->peer[q];
  barrier_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(
      T, c->L.off_ctl, c->world, c->rank, c->bar_gen, rounds, (uint64_t)(c->timeout_s * 1e9),
      static_cast<unsigned long long*>(ns_out));
  c->bar_gen += (uint64_t)rounds;
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GP_OK : cuda_fail(e, "barrier kernel launch");
}

int gp_comm_wire_bytes(gp_comm* c, int rank, int reset, uint64_t* out) {
  if (!c || !out) return fail(GP_ERR_ARG, "null argument");
  const int i = c->nlocal == 1 ? 0 : rank;
  if (i < 0 || i >= c->nlocal) return fail(GP_ERR_ARG, "rank outside communicator");
  DeviceGuard g(c->device);
  uint8_t* p = c->inbox[i] + c->L.off_ctl + offsetof(Ctl, wire_bytes);
  cudaError_t e = cudaMemcpy(out, p, sizeof(uint64_t), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(wire bytes)");
  if (reset && (e = cudaMemset(p, 0, sizeof(uint64_t))) != cudaSuccess) return cuda_fail(e, "reset wire bytes");
  return GP_OK;
}

int gp_comm_poll_error(gp_comm* c, gp_error* out) {
  if (!c || !out) return fail(GP_ERR_ARG, "null argument");
  DeviceGuard g(c->device);
  std::memset(out, 0, sizeof(*out));
  unsigned long long best = ~0ull;
  for (int i = 0; i < c->nlocal; ++i) {
    ErrWord w;
    cudaError_t e = cudaMemcpy(&w, c->inbox[i] + c->L.off_err, sizeof(w), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(error word)");
    if (w.code != ~0ull) {
      best = std::min(best, w.code);
      const unsigned long long none = ~0ull;
      e = cudaMemcpy(c->inbox[i] + c->L.off_err, &none, sizeof(none), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(reset error word)");
    }
  }
  if (best != ~0ull) {
    static const int phases[4] = {kPhRS, kPhBarrier, kPhAG, kPhLocal};
    out->phase = phases[(best >> 60) & 0x7];  // bit 63: abort consequence (ordering only)
    out->step = (int)((best >> 53) & 0x7F);
    out->kind = (int)((best >> 48) & 0xF);
    out->block = (int)((best >> 40) & 0xFF) - 1;
    out->rank = (int)((best >> 32) & 0xFF);
    out->detail = (int)(uint32_t)best;
  }
  return GP_OK;
}

int gp_get_stats(gp_comm* c, int rank, gp_stats* out) {
  if (!c || !out) return fail(GP_ERR_ARG, "null argument");
  const int i = c->nlocal == 1 ? 0 : rank;
  if (i < 0 || i >= c->nlocal) return fail(GP_ERR_ARG, "rank outside communicator");
  *out = c->stats[i];
  return GP_OK;
}

int gp_reset_stats(gp_comm* c) {
  if (!c) return fail(GP_ERR_ARG, "null communicator");
  for (auto& s : c->stats) s = gp_stats{};
  return GP_OK;
}

}  // extern "C"
