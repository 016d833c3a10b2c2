// Star collectives over NVLink for the PS-Sync baseline.
//
// Reference: /root/reference/pkg/src/gradpipe/collective.py
//   gather_to_root      :215-252  root returns acc = local_root, then
//                                 acc += x_src for src in rank order (src != root)
//   broadcast_from_root :255-280  every rank gets a bit-exact copy of root's vector
// and the parameter server of engine.py:503-552, whose gather starts from its
// zero vector (acc = 0, then += x_0, x_1, ... in rank order).
//
// B200 mapping (pull): every rank stages its vector in its own inbox and
// releases per-chunk flags; the root's warps take chunks, acquire each
// source's flag over NVLink and fold the peers' bytes in rank order (remote
// loads), exactly the reference's order of fp32 additions. Broadcast is the
// mirror image: the root stages, everyone pulls. The root's NVLink ingress
// (gather) and egress (broadcast) carry (p-1) x n x 4 bytes: the parameter
// server bottleneck the paper measures against the ring.
#include <algorithm>

#include "../../include/pipesgd.h"
#include "common.cuh"
#include "ring.cuh"

namespace gp {

namespace {

constexpr int kStarThreads = 128;
constexpr int kStarWarps = kStarThreads / 32;

__shared__ uint32_t s_star_seq;
__shared__ uint32_t s_star_bank;
__shared__ unsigned long long s_star_calls;

struct StarRank {
  const float* in;
  float* out;
  uint8_t* inbox;
  uint8_t* peer[kMaxRanks];
  int rank;
};

struct StarParams {
  StarRank rk[kMaxRanks];
  Layout L;
  uint64_t n;
  uint64_t timeout_ns;
  uint32_t chunk;     // elements, multiple of 1024
  int p, G, root;
  int mode;           // 0 gather (sum to root), 1 broadcast
  int zero_first;     // gather: acc = 0 then every rank (server), else acc = x_root first
};

__device__ __forceinline__ uint64_t* star_flag(uint8_t* inbox, const Layout& L, int slot, uint32_t c) {
  return reinterpret_cast<uint64_t*>(inbox + L.off_flags) + (uint64_t)slot * L.max_chunks + c;
}
__device__ __forceinline__ float* staged(uint8_t* inbox, const Layout& L) {
  return reinterpret_cast<float*>(inbox + L.off_payload);
}

__device__ bool star_wait(const uint64_t* f, const StarParams& P, const StarRank& R, Ctl* ctl, ErrWord* err,
                          int phase, int src, int rank) {
  if ((uint32_t)(ld_acquire_sys(f) >> 32) == s_star_seq) return true;
  const uint64_t t0 = globaltimer();
  uint32_t ns = 64;
  for (uint32_t it = 1;; ++it) {
    if ((uint32_t)(ld_relaxed_sys(f) >> 32) == s_star_seq) {
      (void)ld_acquire_sys(f);
      return true;
    }
    __nanosleep(ns);
    if (ns < 512) ns <<= 1;
    if ((it & 31u) == 0) {
      if (comm_aborted(ctl)) {
        latch_error(err, kErrTimeout, phase, 0, src, rank, kAbortConsequence);
        return false;
      }
      if (globaltimer() - t0 > P.timeout_ns) {
        latch_error(err, kErrTimeout, phase, 0, src, rank, 0);
        abort_all(R.peer, P.p, P.L.off_ctl, s_star_seq, rank);  // peers stop waiting on this rank
        return false;
      }
    }
  }
}

__device__ __forceinline__ uint32_t star_grab(Ctl* ctl, int phase) {
  uint32_t c = 0;
  if ((threadIdx.x & 31) == 0) c = (uint32_t)atomicAdd(&ctl->bank[s_star_bank].next[phase], 1ull);
  return __shfl_sync(0xffffffffu, c, 0);
}

// Copy chunk c of `src` into `dst` (4 floats per lane, 8 in flight).
__device__ __forceinline__ void copy_chunk(float* dst, const float* src, uint64_t b, uint64_t e) {
  const int lane = threadIdx.x & 31;
  for (uint64_t g = b + 4ull * lane; g < e; g += 4ull * 32 * 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint64_t i = g + 4ull * 32 * u;
      if (i + 4 <= e) v[u] = __ldcg(reinterpret_cast<const float4*>(src + i));
      else if (i < e) {
        float t[4] = {0, 0, 0, 0};
        for (int k = 0; k < 4 && i + k < e; ++k) t[k] = __ldcg(src + i + k);
        v[u] = make_float4(t[0], t[1], t[2], t[3]);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint64_t i = g + 4ull * 32 * u;
      if (i + 4 <= e) *reinterpret_cast<float4*>(dst + i) = v[u];
      else if (i < e) {
        const float t[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
        for (int k = 0; k < 4 && i + k < e; ++k) dst[i + k] = t[k];
      }
    }
  }
}

__device__ void star_body(const StarParams& P) {
  const int lr = blockIdx.x / P.G;
  const StarRank& R = P.rk[lr];
  Ctl* ctl = reinterpret_cast<Ctl*>(R.inbox + P.L.off_ctl);
  ErrWord* err = reinterpret_cast<ErrWord*>(R.inbox + P.L.off_err);
  const int lane = threadIdx.x & 31;
  const uint64_t n = P.n;
  const uint32_t nch = n ? (uint32_t)((n + P.chunk - 1) / P.chunk) : 0u;
  const int slot = P.mode;  // flags: slot 0 gather staging, slot 1 broadcast staging
  const int phase = P.mode == 0 ? kPhRS : kPhAG;
  const bool root = R.rank == P.root;
  if (comm_aborted(ctl)) {  // an earlier call failed: end at once (ring.cuh:kAbortSticky)
    if (blockIdx.x % P.G == 0 && threadIdx.x == 0) latch_error(err, kErrTimeout, phase, 0, -1, R.rank, 1);
    return;
  }

  if ((P.mode == 0 && !root) || (P.mode == 1 && root)) {
    // stage my vector in my inbox and publish it chunk by chunk
    float* st = staged(R.inbox, P.L);
    for (uint32_t c = star_grab(ctl, 0); c < nch; c = star_grab(ctl, 0)) {
      const uint64_t b = (uint64_t)c * P.chunk, e = min(n, b + P.chunk);
      copy_chunk(st, R.in, b, e);
      if (P.mode == 1 && R.out != R.in) copy_chunk(R.out, R.in, b, e);
      __syncwarp();
      if (lane == 0 && P.p > 1) st_release_sys(star_flag(R.inbox, P.L, slot, c), (uint64_t)s_star_seq << 32);
    }
    return;
  }
  if (P.mode == 1) {
    // pull the root's staged chunks (broadcast receive)
    const float* src = staged(R.peer[P.root], P.L);
    for (uint32_t c = star_grab(ctl, 1); c < nch; c = star_grab(ctl, 1)) {
      int ok = 1;
      if (lane == 0) ok = star_wait(star_flag(R.peer[P.root], P.L, slot, c), P, R, ctl, err, phase, P.root, R.rank);
      __syncwarp();
      if (!__shfl_sync(0xffffffffu, ok, 0)) return;
      const uint64_t b = (uint64_t)c * P.chunk, e = min(n, b + P.chunk);
      copy_chunk(R.out, src, b, e);
    }
    return;
  }
  // gather at the root: fold the sources in the reference's order, one
  // streaming pass per source over the chunk (8 x 16 B loads in flight per
  // lane, remote sources read over NVLink, the running sum kept in `out`)
  for (uint32_t c = star_grab(ctl, 1); c < nch; c = star_grab(ctl, 1)) {
    int ok = 1;
    if (lane == 0)
      for (int s = 0; s < P.p && ok; ++s)
        if (s != R.rank) ok = star_wait(star_flag(R.peer[s], P.L, 0, c), P, R, ctl, err, phase, s, R.rank);
    __syncwarp();
    if (!__shfl_sync(0xffffffffu, ok, 0)) return;
    const uint64_t b = (uint64_t)c * P.chunk, e = min(n, b + P.chunk);
    // source order: [root, others ascending] (gather_to_root) or
    // [zero, 0, 1, ..., p-1] (the parameter server's zero vector first)
    const int nsrc = P.zero_first ? P.p : P.p;
    for (int k = 0; k < nsrc; ++k) {
      int s;
      if (P.zero_first) s = k;
      else s = (k == 0) ? R.rank : (k <= R.rank ? k - 1 : k);
      const float* src = (s == R.rank) ? R.in : staged(R.peer[s], P.L);
      const bool first = (k == 0);
      for (uint64_t g = b + 4ull * lane; g < e; g += 4ull * 32 * 8) {
        float4 v[8], a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint64_t i = g + 4ull * 32 * u;
          if (i + 4 <= e) {
            v[u] = __ldcg(reinterpret_cast<const float4*>(src + i));
            a[u] = first ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldcg(reinterpret_cast<const float4*>(R.out + i));
          } else if (i < e) {
            float t[4] = {0, 0, 0, 0}, o[4] = {0, 0, 0, 0};
            for (int q = 0; q < 4 && i + q < e; ++q) {
              t[q] = __ldcg(src + i + q);
              if (!first) o[q] = __ldcg(R.out + i + q);
            }
            v[u] = make_float4(t[0], t[1], t[2], t[3]);
            a[u] = make_float4(o[0], o[1], o[2], o[3]);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint64_t i = g + 4ull * 32 * u;
          if (i >= e) continue;
          float4 r;
          if (first && !P.zero_first) {
            r = v[u];  // gather_to_root: acc = copy(local_root)
          } else {   // fl(acc + x): with zero_first the first term is fl(0 + x_0)
            r = make_float4(__fadd_rn(a[u].x, v[u].x), __fadd_rn(a[u].y, v[u].y), __fadd_rn(a[u].z, v[u].z),
                            __fadd_rn(a[u].w, v[u].w));
          }
          if (i + 4 <= e) {
            *reinterpret_cast<float4*>(R.out + i) = r;
          } else {
            const float t[4] = {r.x, r.y, r.z, r.w};
            for (int q = 0; q < 4 && i + q < e; ++q) R.out[i + q] = t[q];
          }
        }
      }
      __syncwarp();  // this lane's next pass reads back what it wrote (same addresses)
    }
  }
}

// Lane 0: wait until ack word `a` carries this call's sequence.
__device__ bool star_wait_ack(unsigned long long* a, const StarParams& P, const StarRank& R, Ctl* ctl, ErrWord* err,
                              int phase, int src, int rank) {
  return star_wait(reinterpret_cast<const uint64_t*>(a), P, R, ctl, err, phase, src, rank);
}

// Close of a star call, run by the last warp of a rank: the side whose
// staged bytes were read waits until every reader acknowledged, so a rank
// never restages (next call) over data a peer is still reading.
//   gather:    the root, done folding, acks every source; sources wait.
//   broadcast: every receiver, done pulling, acks the root; the root waits.
__device__ void star_close_handshake(const StarParams& P, const StarRank& R, Ctl* ctl) {
  if (P.p < 2) return;
  ErrWord* err = reinterpret_cast<ErrWord*>(R.inbox + P.L.off_err);
  const int phase = P.mode == 0 ? kPhRS : kPhAG;
  const bool root = R.rank == P.root;
  const uint64_t ackw = (uint64_t)s_star_seq << 32;
  auto peer_ctl = [&](int q) { return reinterpret_cast<Ctl*>(R.peer[q] + P.L.off_ctl); };
  if (P.mode == 0) {
    if (root) {
      __threadfence_system();
      for (int q = 0; q < P.p; ++q)
        if (q != R.rank) st_release_sys(reinterpret_cast<uint64_t*>(&peer_ctl(q)->ack[R.rank]), ackw);
    } else {
      star_wait_ack(&ctl->ack[P.root], P, R, ctl, err, phase, P.root, R.rank);
    }
  } else {
    if (!root) {
      __threadfence_system();
      st_release_sys(reinterpret_cast<uint64_t*>(&peer_ctl(P.root)->ack[R.rank]), ackw);
    } else {
      for (int q = 0; q < P.p; ++q)
        if (q != R.rank && !star_wait_ack(&ctl->ack[q], P, R, ctl, err, phase, q, R.rank)) break;
    }
  }
}

__global__ void __launch_bounds__(kStarThreads) star_kernel(const __grid_constant__ StarParams P) {
  const int lr = blockIdx.x / P.G;
  Ctl* ctl = reinterpret_cast<Ctl*>(P.rk[lr].inbox + P.L.off_ctl);
  if (threadIdx.x == 0) {
    const unsigned long long calls = ld_acquire_gpu(reinterpret_cast<uint64_t*>(&ctl->calls));
    s_star_calls = calls;
    s_star_seq = next_seq(calls);
    s_star_bank = (uint32_t)(calls & 1);
    if (blockIdx.x % P.G == 0) {  // the next call's bank starts from zero (ring.cuh:CtlBank)
      CtlBank* nb = &ctl->bank[(calls + 1) & 1];
      nb->bar = 0;
      nb->exits = 0;
      for (int i = 0; i < 32; ++i) nb->next[i] = 0;
      for (int i = 0; i < 16; ++i) nb->maxslot[i] = 0;
    }
  }
  __syncthreads();
  star_body(P);
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {  // last warp of this rank closes the call (as the ring does)
    const unsigned long long prev = atomicAdd(&ctl->bank[s_star_bank].exits, 1ull);
    if (prev == (unsigned long long)P.G * kStarWarps - 1) {
      __threadfence();  // every warp of this rank is done with the staged data
      star_close_handshake(P, P.rk[lr], ctl);
      *(volatile unsigned long long*)&ctl->calls = s_star_calls + 1;
    }
  }
}

}  // namespace

cudaError_t launch_star(const StarLaunch& S, cudaStream_t stream) {
  StarParams P{};
  P.L = S.L;
  P.n = S.n;
  P.timeout_ns = S.timeout_ns;
  P.p = S.p;
  P.root = S.root;
  P.mode = S.mode;
  P.zero_first = S.zero_first;
  P.G = std::max(1, std::min(S.ctas, S.max_ctas));
  // full-vector staging in the inbox payload, chunk flags sized per slot
  const uint64_t want = (S.n + S.L.max_chunks - 1) / std::max<uint64_t>(1, S.L.max_chunks);
  P.chunk = (uint32_t)std::max<uint64_t>(4096, (want + 1023) / 1024 * 1024);
  for (int i = 0; i < S.nlocal; ++i) {
    P.rk[i].in = S.ins[i];
    P.rk[i].out = S.outs[i];
    P.rk[i].inbox = S.inboxes[i];
    P.rk[i].rank = S.ranks[i];
    for (int q = 0; q < S.p; ++q) P.rk[i].peer[q] = S.peers[q];
  }
  void* args[] = {&P};
  const dim3 grid(P.G * S.nlocal), block(kStarThreads);
  if (S.nlocal > 1) return cudaLaunchCooperativeKernel((const void*)star_kernel, grid, block, args, 0, stream);
  return cudaLaunchKernel((const void*)star_kernel, grid, block, args, 0, stream);
}

}  // namespace gp
