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
// B200 mapping. One cooperative launch per rank per call, G CTAs of 512
// threads. A block is cut into chunks of `chunk` elements aligned to
// multiples of 8 global indices; chunk c of every block belongs to CTA c%G
// on every rank, so each chunk flows around the ring independently:
//   wait flag(slot s, chunk c) -> decode inbox + add local -> encode ->
//   st.global into succ's inbox over NVLink -> st.release.sys succ's flag.
// quant8 needs the block-wide max before any code can be emitted
// (compression.py:129-132), so each of its hops is two passes around a
// rank-local barrier: pass A folds and reduces the max (partial sums parked
// in `out`, L2-resident), pass B encodes and pushes. The allgather is a
// direct owner->all-peers push over NVSwitch (same bytes the ring would
// forward, one hop instead of p-1).
// Emulation: with nlocal == p the same kernel runs all ranks of the ring on
// one GPU inside one cooperative launch (CTA group = rank), used for parity
// tests at p > #GPUs without separately-launched kernels that wait on each
// other.
#include "codec.cuh"
#include "ring.cuh"

namespace gp {

namespace {

struct Blk {
  uint64_t start, len, A;
  uint32_t nch;
};

__device__ __forceinline__ Blk get_blk(const RingParams& P, int b) {
  Blk k;
  block_range(P.n, P.p, b, k.start, k.len);
  k.A = k.start & ~7ull;
  k.nch = k.len ? (uint32_t)((k.start + k.len - k.A + P.chunk - 1) / P.chunk) : 0u;
  return k;
}

struct Sh {
  uint32_t red[kRingThreads / 32];
  int ok;
  float scale;
};

__device__ __forceinline__ uint64_t* flag_ptr(uint8_t* inbox, const Layout& L, int slot, uint32_t c) {
  return reinterpret_cast<uint64_t*>(inbox + L.off_flags) + (uint64_t)slot * L.max_chunks + c;
}
__device__ __forceinline__ SlotHdr* hdr_ptr(uint8_t* inbox, const Layout& L, int slot) {
  return reinterpret_cast<SlotHdr*>(inbox + L.off_hdr) + slot;
}
__device__ __forceinline__ uint8_t* slot_ptr(uint8_t* inbox, const Layout& L, int slot) {
  return inbox + L.off_payload + (uint64_t)slot * L.slot_bytes;
}

// Abort this call on every rank: peers' spins see it and stop waiting.
__device__ void broadcast_abort(const RingParams& P, const RankCtx& R) {
  for (int q = 0; q < P.p; ++q) {
    Ctl* c = reinterpret_cast<Ctl*>(R.peer[q] + P.L.off_ctl);
    atomicMax(&c->abort, (unsigned long long)P.seq);
  }
  fence_sys();
}

// Thread 0 spins until *f >= seq. Returns false on timeout or abort.
__device__ bool spin_flag(const uint64_t* f, const RingParams& P, const RankCtx& R, Ctl* ctl,
                          ErrWord* err, int phase, int step, int block) {
  if (ld_acquire_sys(f) >= P.seq) return true;
  const uint64_t t0 = globaltimer();
  for (uint32_t it = 1;; ++it) {
    if (ld_acquire_sys(f) >= P.seq) return true;
    if ((it & 255u) == 0) {
      if (*(volatile unsigned long long*)&ctl->abort >= P.seq) {
        latch_error(err, kErrTimeout, phase, step, block, R.rank, 1 /* peer aborted */);
        return false;
      }
      if (globaltimer() - t0 > P.timeout_ns) {
        latch_error(err, kErrTimeout, phase, step, block, R.rank, 0);
        broadcast_abort(P, R);
        return false;
      }
    }
  }
}

// All threads: wait for (slot, chunk) of this rank's inbox, validate the
// slot header like collective.py:_expect (:52-64, :109-114), fetch scale.
__device__ bool await_chunk(Sh& sh, const RingParams& P, const RankCtx& R, Ctl* ctl, ErrWord* err,
                            int slot, uint32_t c, int phase, int step, int block, uint64_t len,
                            float& scale) {
  if (threadIdx.x == 0) {
    bool ok = spin_flag(flag_ptr(R.inbox, P.L, slot, c), P, R, ctl, err, phase, step, block);
    if (ok) {
      const SlotHdr* h = hdr_ptr(R.inbox, P.L, slot);
      const uint32_t hb = __ldcg(&h->block), hi = __ldcg(&h->iteration), hn = __ldcg(&h->n_elems);
      if (hb != (uint32_t)block || hi != P.iteration || hn != (uint32_t)len) {
        latch_error(err, kErrHeader, phase, step, block, R.rank, (int)hn);
        broadcast_abort(P, R);
        ok = false;
      }
      sh.scale = __ldcg(&h->scale);
    }
    sh.ok = ok;
  }
  __syncthreads();
  scale = sh.scale;
  return sh.ok;
}

// All threads: after this CTA's payload stores to `dst_inbox`, write the
// slot header and release the chunk flag at system scope.
__device__ __forceinline__ void publish(const RingParams& P, uint8_t* dst_inbox, int slot, uint32_t c,
                                        int block, uint64_t len, float scale) {
  __syncthreads();
  if (threadIdx.x == 0) {
    SlotHdr* h = hdr_ptr(dst_inbox, P.L, slot);
    h->seq = P.seq;
    h->iteration = P.iteration;
    h->block = (uint32_t)block;
    h->n_elems = (uint32_t)len;
    h->scale = scale;
    fence_sys();
    st_release_sys(flag_ptr(dst_inbox, P.L, slot, c), P.seq);
  }
}

// quant8: rank-local barrier across the G CTAs of one rank, combined with
// the block max. Returns false on abort/timeout.
__device__ bool barrier_max(Sh& sh, const RingParams& P, const RankCtx& R, Ctl* ctl, ErrWord* err,
                            int k, uint32_t mymax, float& vmax, int step) {
  const uint32_t m = cta_max_u32<kRingThreads>(mymax, sh.red);
  if (threadIdx.x == 0) {
    atomicMax(&ctl->maxslot[k], ((unsigned long long)P.seq << 32) | m);
    __threadfence();
    atomicAdd(&ctl->bar, 1ull);
    const unsigned long long target = P.bar_base + (unsigned long long)(k + 1) * P.G;
    bool ok = true;
    const uint64_t t0 = globaltimer();
    for (uint32_t it = 1; ld_acquire_gpu(reinterpret_cast<uint64_t*>(&ctl->bar)) < target; ++it) {
      if ((it & 255u) == 0) {
        if (*(volatile unsigned long long*)&ctl->abort >= P.seq) { ok = false; break; }
        if (globaltimer() - t0 > P.timeout_ns) {
          latch_error(err, kErrTimeout, kPhBarrier, step, -1, R.rank, 0);
          broadcast_abort(P, R);
          ok = false;
          break;
        }
      }
    }
    const unsigned long long v = ld_acquire_gpu(reinterpret_cast<uint64_t*>(&ctl->maxslot[k]));
    sh.scale = ((uint32_t)(v >> 32) == P.seq) ? __uint_as_float((uint32_t)v) : 0.f;
    sh.ok = ok;
  }
  __syncthreads();
  vmax = sh.scale;
  return sh.ok;
}

__device__ __forceinline__ F8 add8(const F8& a, const F8& b) {
  F8 r;
#pragma unroll
  for (int i = 0; i < 8; ++i) r.v[i] = __fadd_rn(a.v[i], b.v[i]);
  return r;
}

// Iterate the 8-element groups of chunk c of block B owned by this thread.
template <typename Fn>
__device__ __forceinline__ void for_groups(const RingParams& P, const Blk& B, uint32_t c, Fn&& fn) {
  const uint64_t cbase = B.A + (uint64_t)c * P.chunk;
  const uint64_t lo = max(B.start, cbase);
  const uint64_t hi = min(B.start + B.len, cbase + P.chunk);
  for (uint64_t g0 = cbase + 8ull * threadIdx.x; g0 < hi; g0 += 8ull * kRingThreads) {
    const int vlo = (int)(max(lo, g0) - g0);
    const int vhi = (int)(min(hi, g0 + 8) - g0);
    fn(g0, lo, hi, vlo, vhi);
  }
}

}  // namespace

template <int C>
__global__ void __launch_bounds__(kRingThreads) ring_allreduce_kernel(const __grid_constant__ RingParams P) {
  __shared__ Sh sh;
  const int G = P.G;
  const int lr = blockIdx.x / G;
  const uint32_t j = blockIdx.x % G;
  const RankCtx& R = P.rk[lr];
  const int p = P.p, r = R.rank, succ = (r + 1) % p;
  Ctl* ctl = reinterpret_cast<Ctl*>(R.inbox + P.L.off_ctl);
  ErrWord* err = reinterpret_cast<ErrWord*>(R.inbox + P.L.off_err);
  const float* __restrict__ x = R.x;
  float* out = R.out;
  int bad = 0;

  // ---- reduce-scatter step 0, send side: C(x_r[block r]) -> succ slot 0
  {
    const Blk B = get_blk(P, r);
    Q8 q = q8_make(0.f);
    if constexpr (C == kQuant8) {
      uint32_t m = 0;
      for (uint32_t c = j; c < B.nch; c += G)
        for_groups(P, B, c, [&](uint64_t g0, uint64_t lo, uint64_t hi, int, int) {
          m = max(m, absmax8_bits(load_f8(x, g0, lo, hi)));
        });
      float vmax;
      if (!barrier_max(sh, P, R, ctl, err, 0, m, vmax, 0)) return;
      q = q8_make(q8_scale(vmax));
    }
    uint8_t* dst = slot_ptr(R.peer[succ], P.L, rs_slot(0));
    for (uint32_t c = j; c < B.nch; c += G) {
      for_groups(P, B, c, [&](uint64_t g0, uint64_t lo, uint64_t hi, int vlo, int vhi) {
        const Packed<C> pk = encode8<C>(load_f8(x, g0, lo, hi), q, bad);
        store_packed<C>(dst, g0 - B.A, vlo, vhi, pk);
      });
      publish(P, R.peer[succ], rs_slot(0), c, r, B.len, q.s);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) latch_error(err, kErrNonFinite, kPhRS, 0, r, r, 0);
    bad = 0;
  }

  // ---- reduce-scatter steps: fold block (r-s-1)%p, forward (or own it)
  for (int s = 0; s < p - 1; ++s) {
    const int b = (r - s - 1 + p) % p;
    const Blk B = get_blk(P, b);
    const bool last = (s == p - 2);
    uint8_t* in_slot = slot_ptr(R.inbox, P.L, rs_slot(s));
    uint8_t* fwd = last ? nullptr : slot_ptr(R.peer[succ], P.L, rs_slot(s + 1));

    if constexpr (C != kQuant8) {
      const Q8 q = q8_make(0.f);
      for (uint32_t c = j; c < B.nch; c += G) {
        float sin;
        if (!await_chunk(sh, P, R, ctl, err, rs_slot(s), c, kPhRS, s, b, B.len, sin)) return;
        for_groups(P, B, c, [&](uint64_t g0, uint64_t lo, uint64_t hi, int vlo, int vhi) {
          const F8 inc = decode8<C>(load_packed<C>(in_slot, g0 - B.A, vlo, vhi), sin);
          const F8 acc = add8(load_f8(x, g0, lo, hi), inc);
          const Packed<C> pk = encode8<C>(acc, q, bad);
          if (!last) {
            store_packed<C>(fwd, g0 - B.A, vlo, vhi, pk);
          } else {
            for (int d = 1; d < p; ++d)
              store_packed<C>(slot_ptr(R.peer[(r + d) % p], P.L, ag_slot(p, b)), g0 - B.A, vlo, vhi, pk);
            store_f8(out, g0, lo, hi, decode8<C>(pk, 0.f));
          }
        });
        if (!last) {
          publish(P, R.peer[succ], rs_slot(s + 1), c, b, B.len, 0.f);
        } else {
          __syncthreads();
          for (int d = 1; d < p; ++d) {
            uint8_t* dst = R.peer[(r + d) % p];
            if (threadIdx.x == 0) {
              SlotHdr* h = hdr_ptr(dst, P.L, ag_slot(p, b));
              h->seq = P.seq; h->iteration = P.iteration; h->block = (uint32_t)b;
              h->n_elems = (uint32_t)B.len; h->scale = 0.f;
            }
          }
          if (threadIdx.x == 0) {
            fence_sys();
            for (int d = 1; d < p; ++d)
              st_release_sys(flag_ptr(R.peer[(r + d) % p], P.L, ag_slot(p, b), c), P.seq);
          }
        }
      }
    } else {
      // pass A: fold into `out` (scratch for this block) and reduce the max
      uint32_t m = 0;
      for (uint32_t c = j; c < B.nch; c += G) {
        float sin;
        if (!await_chunk(sh, P, R, ctl, err, rs_slot(s), c, kPhRS, s, b, B.len, sin)) return;
        for_groups(P, B, c, [&](uint64_t g0, uint64_t lo, uint64_t hi, int vlo, int vhi) {
          const F8 inc = decode8<C>(load_packed<C>(in_slot, g0 - B.A, vlo, vhi), sin);
          const F8 acc = add8(load_f8(x, g0, lo, hi), inc);
          m = max(m, absmax8_bits(acc));
          store_f8(out, g0, lo, hi, acc);
        });
      }
      float vmax;
      if (!barrier_max(sh, P, R, ctl, err, s + 1, m, vmax, s)) return;
      const Q8 q = q8_make(q8_scale(vmax));
      // pass B: encode the partial with the block scale and push it
      for (uint32_t c = j; c < B.nch; c += G) {
        for_groups(P, B, c, [&](uint64_t g0, uint64_t lo, uint64_t hi, int vlo, int vhi) {
          const F8 acc = load_f8_cg(out, g0, lo, hi);
          const Packed<C> pk = encode8<C>(acc, q, bad);
          if (!last) {
            store_packed<C>(fwd, g0 - B.A, vlo, vhi, pk);
          } else {
            for (int d = 1; d < p; ++d)
              store_packed<C>(slot_ptr(R.peer[(r + d) % p], P.L, ag_slot(p, b)), g0 - B.A, vlo, vhi, pk);
            store_f8(out, g0, lo, hi, decode8<C>(pk, q.s));
          }
        });
        if (!last) {
          publish(P, R.peer[succ], rs_slot(s + 1), c, b, B.len, q.s);
        } else {
          __syncthreads();
          if (threadIdx.x == 0) {
            for (int d = 1; d < p; ++d) {
              SlotHdr* h = hdr_ptr(R.peer[(r + d) % p], P.L, ag_slot(p, b));
              h->seq = P.seq; h->iteration = P.iteration; h->block = (uint32_t)b;
              h->n_elems = (uint32_t)B.len; h->scale = q.s;
            }
            fence_sys();
            for (int d = 1; d < p; ++d)
              st_release_sys(flag_ptr(R.peer[(r + d) % p], P.L, ag_slot(p, b), c), P.seq);
          }
        }
      }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0)
      latch_error(err, kErrNonFinite, last ? kPhAG : kPhRS, last ? 0 : s + 1, b, r, 0);
    bad = 0;
  }

  // ---- allgather, receive side: decode every other owner's bytes
  for (int k = 1; k < p; ++k) {
    const int b = (r + 1 + k) % p;  // own block is (r+1)%p
    const Blk B = get_blk(P, b);
    const int step = (r - b + p) % p;  // reference allgather step that delivers block b
    uint8_t* in_slot = slot_ptr(R.inbox, P.L, ag_slot(p, b));
    for (uint32_t c = j; c < B.nch; c += G) {
      float sin;
      if (!await_chunk(sh, P, R, ctl, err, ag_slot(p, b), c, kPhAG, step, b, B.len, sin)) return;
      for_groups(P, B, c, [&](uint64_t g0, uint64_t lo, uint64_t hi, int vlo, int vhi) {
        store_f8(out, g0, lo, hi, decode8<C>(load_packed<C>(in_slot, g0 - B.A, vlo, vhi), sin));
      });
    }
  }
}

void launch_ring(const RingParams& P, int nlocal, cudaStream_t stream, cudaError_t* err) {
  void* args[] = {const_cast<RingParams*>(&P)};
  const dim3 grid(P.G * nlocal), block(kRingThreads);
  const void* fn = P.codec == kNone      ? (const void*)ring_allreduce_kernel<kNone>
                   : P.codec == kTrunc16 ? (const void*)ring_allreduce_kernel<kTrunc16>
                                         : (const void*)ring_allreduce_kernel<kQuant8>;
  *err = cudaLaunchCooperativeKernel(fn, grid, block, args, 0, stream);
}

}  // namespace gp
