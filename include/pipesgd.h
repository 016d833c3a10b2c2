/* pipesgd.h — C ABI of the B200-native Pipe-SGD communication hot path.
 *
 * libpipesgd.so (paper_1811_03619_b200/libpipesgd.so) exports exactly the
 * functions below: plain pointers, sizes and CUDA stream handles, no torch
 * types. Device pointers are CUDA device addresses on the communicator's
 * device (or the current device for the stateless codec/update calls);
 * `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *
 * Each entry replaces a function of the reference package `gradpipe`
 * (/root/reference/pkg/src/gradpipe):
 *   gp_allreduce            collective.py:143-163 ring_allreduce
 *                           collective.py:166-212 pipelined_allreduce (same bits)
 *   gp_allreduce_ex         the ring fused with the engine's local pre-compress
 *                           (engine.py:333) and pipe re-compress of the sum (engine.py:407)
 *   gp_allreduce_emulated   the same ring with all p ranks on one device
 *                           (collective.py:77-139 driven like tests/helpers.py:10-29)
 *   gp_gather_sum           collective.py:215-252 gather_to_root (+ the PS server's fold)
 *   gp_broadcast            collective.py:255-280 broadcast_from_root
 *   gp_comm_create/connect  transport.py:150-177 InProcTransport(world).endpoint(r)
 *                           transport.py:192-305 TcpEndpoint mesh set-up
 *   gp_get_stats/reset      transport.py:52-61, :85-91, :105-107 TrafficStats
 *   gp_comm_poll_error      collective.py:52-64, :157-161 CollectiveError,
 *                           compression.py:108-109 CodecError (non-finite)
 *   gp_encode / gp_decode   compression.py:103-136 compress, :141-151 decompress
 *   gp_roundtrip            engine.py:333 + :355/:400 decompress(compress(grad))
 *   gp_consume_update(_dev) engine.py:420-426 decompress -> engine.py:123-129
 *                           aggregate_mean -> models.py:198-204 sgd_update
 *   gp_calib_p2p_copy       harness.py:552-557 beta probe (flood), on NVLink
 *   gp_calib_pingpong       harness.py:547-550 alpha probe (1-byte ping), on NVLink
 *   gp_comm_set_tuning / _set_trace / _info / _set_call_counter, gp_ring_plan:
 *                           no reference counterpart (CTA budget + timeout,
 *                           timeline stamps, introspection, 32-bit sequence-wrap
 *                           test hook, launch-plan query)
 *
 * Return value: GP_OK (0) or a GP_ERR_* code; gp_last_error_string() gives
 * the calling thread's last message. Failures detected on the device
 * (non-finite values, ring timeouts, header mismatches) are latched in a
 * device error word and reported by gp_comm_poll_error / gp_codec_status.
 */
#ifndef PIPESGD_H_
#define PIPESGD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gp_comm gp_comm;

enum { GP_CODEC_NONE = 0, GP_CODEC_TRUNC16 = 1, GP_CODEC_QUANT8 = 2 };

enum {
  GP_OK = 0,
  GP_ERR_ARG = 1,         /* bad argument (codec, size, alignment, aliasing) */
  GP_ERR_CUDA = 2,        /* CUDA runtime failure */
  GP_ERR_STATE = 3,       /* communicator not connected / wrong mode */
  GP_ERR_UNSUPPORTED = 4  /* e.g. no peer access between two devices */
};

/* device failure kinds (gp_error.kind, gp_codec_status.nonfinite) */
enum { GP_FAIL_NONE = 0, GP_FAIL_NONFINITE = 1, GP_FAIL_TIMEOUT = 2, GP_FAIL_HEADER = 3,
       GP_FAIL_BOUNDS = 4 /* bounds-checked build only (libpipesgd_checked.so): an access outside its buffer or slot */ };
/* gp_error.phase */
enum { GP_PHASE_REDUCE_SCATTER = 0, GP_PHASE_ALLGATHER = 1, GP_PHASE_BARRIER = 2 };

typedef struct {
  int32_t kind;   /* GP_FAIL_* */
  int32_t phase;  /* GP_PHASE_* */
  int32_t step;   /* reference ring step within the phase */
  int32_t block;  /* block index (partition_blocks order), -1 if n/a */
  int32_t rank;   /* rank that observed the failure */
  int32_t detail; /* TIMEOUT: 1 = a peer aborted first; HEADER: advertised n_elems */
} gp_error;

typedef struct {
  uint64_t messages;      /* data messages sent: 2(p-1) per allreduce */
  uint64_t payload_bytes; /* codec payload bytes, 9-byte block header excluded */
  uint64_t frame_bytes;   /* payload + 9-byte block header + 11-byte frame header */
} gp_stats;

/* Device-resident status of a stateless codec call (16 bytes, device memory). */
typedef struct {
  uint32_t absmax_bits; /* bits of max|x| (quant8) */
  int32_t nonfinite;    /* != 0: a NaN/Inf was seen -> CodecError */
  float scale;          /* quant8 block scale written by gp_encode */
  uint32_t reserved;
} gp_codec_status;

/* ---- communicator (one per rank) ------------------------------------- */
int gp_comm_create(int rank, int world, int device, uint64_t max_elems, gp_comm** out);
int gp_comm_create_emulated(int world, int device, uint64_t max_elems, gp_comm** out);
int gp_comm_ipc_handle(gp_comm* comm, void* handle_out /* 64 bytes */);
int gp_comm_connect_ipc(gp_comm* comm, const void* handles /* world x 64 bytes, rank order */);
/* In-process peers (one thread per rank). Ranks may share a device: each keeps
 * its own inbox and its own per-rank ring launch, and the device's SMs are split
 * between them (every rank's CTA budget is capped so all launches co-reside). */
int gp_comm_connect_local(gp_comm* const* comms, int world);
int gp_comm_set_tuning(gp_comm* comm, int ctas_per_rank, double timeout_s);
/* Optional ring timeline for profiling: device buffer of nlocal x ctas x 4 warps
 * x 44 u64 %globaltimer stamps (see csrc/ring.cuh kTraceSlots); NULL disables. */
int gp_comm_set_trace(gp_comm* comm, void* device_buffer);
/* Iteration tag from device memory: ring launches made while `device_tag` is
 * set read the tag (the reference's message iteration, checked like
 * collective.py:_expect :52-64) from this device word at kernel entry instead
 * of the `iteration` argument, so a ring captured once in a CUDA graph still
 * carries and checks the real step t on every replay (the host writes t
 * before each replay). NULL restores the argument. */
int gp_comm_set_iteration_source(gp_comm* comm, const uint32_t* device_tag);
/* Wire protocol cap (NCCL_PROTO-like; every rank must pass the same value):
 * the LL protocol only for blocks whose payload is at most ll_max_bytes
 * (and the library's own 2 MiB limit); 0 = flag protocol for every call.
 * Default: no cap. Results are bit-identical either way. */
int gp_comm_set_protocol(gp_comm* comm, uint64_t ll_max_bytes);
int gp_comm_info(gp_comm* comm, int64_t* out /* [rank, world, device, max_elems, ctas, inbox_bytes, seq, mode (0 own GPU, 1 emulated, 2 per-rank launch on a shared GPU)] */);
int gp_comm_destroy(gp_comm* comm);
/* Test hook: set the device call counter of this communicator's inbox(es)
 * (sequence numbers cycle 1 .. 2^32-1; tests start near the wrap). Every rank
 * must set the same value while no call is in flight. */
int gp_comm_set_call_counter(gp_comm* comm, uint64_t calls);
/* Launch plan of a ring call (pure host logic, no GPU needed): out[0] chunk
 * elements, out[1] CTAs launched, out[2] 1 = LL protocol, out[3] chunks in
 * the largest phase, out[4] 1 = direct reduce-scatter (codec none, world >= 3:
 * every rank pushes each block straight to its owner, who folds them in the
 * ring's order), for n elements over `world` ranks, a communicator of
 * `ctas` CTAs and `max_elems` capacity. `out` holds 5 int64. */
int gp_ring_plan(uint64_t n, int world, int ctas, int codec, int flags, uint64_t max_elems, int64_t* out);

int gp_allreduce(gp_comm* comm, const float* in, float* out, uint64_t n, int codec,
                 uint32_t iteration, void* stream);
int gp_allreduce_emulated(gp_comm* comm, const float* const* ins, float* const* outs, uint64_t n,
                          int codec, uint32_t iteration, void* stream);
/* Fused variants. flags:
 *   GP_RING_PRECOMPRESS: `in` is the raw local gradient; the ring applies the
 *     engine's whole-vector D(C(.)) (engine.py:333, :355/:400) while loading it.
 *   GP_RING_SLOT_OUT: instead of the fp32 sum, write C(sum) with the whole-vector
 *     codec (engine.py:407) to `slot` (n * width bytes) and its scale to `slot_scale`
 *     (device f32); `out` is then scratch (quant8) and its contents undefined.
 * Results are bit-identical to ring_allreduce followed by compress/decompress. */
enum { GP_RING_PRECOMPRESS = 1, GP_RING_SLOT_OUT = 2 };
int gp_allreduce_ex(gp_comm* comm, const float* in, float* out, void* slot, float* slot_scale, uint64_t n,
                    int codec, int flags, uint32_t iteration, void* stream);
int gp_allreduce_emulated_ex(gp_comm* comm, const float* const* ins, float* const* outs, void* const* slots,
                             float* const* slot_scales, uint64_t n, int codec, int flags, uint32_t iteration,
                             void* stream);
/* Star collectives for the PS-Sync baseline (collective.py:215-280, engine.py:503-552):
 * gp_gather_sum: on `root`, out = x_root + x_0 + x_1 + ... (rank order, src != root) —
 *   the reference's gather_to_root — or, with zero_first, 0 + x_0 + x_1 + ... (the
 *   parameter server's fold from its zero vector); other ranks' `out` is untouched.
 * gp_broadcast: every rank's out = root's in (bit-exact). */
int gp_gather_sum(gp_comm* comm, const float* in, float* out, uint64_t n, int root, int zero_first,
                  uint32_t iteration, void* stream);
int gp_broadcast(gp_comm* comm, const float* in, float* out, uint64_t n, int root, uint32_t iteration,
                 void* stream);
int gp_gather_sum_emulated(gp_comm* comm, const float* const* ins, float* const* outs, uint64_t n, int root,
                           int zero_first, uint32_t iteration, void* stream);
int gp_broadcast_emulated(gp_comm* comm, const float* const* ins, float* const* outs, uint64_t n, int root,
                          uint32_t iteration, void* stream);
int gp_comm_poll_error(gp_comm* comm, gp_error* out); /* call after the stream completed; clears */
int gp_get_stats(gp_comm* comm, int rank, gp_stats* out);
int gp_reset_stats(gp_comm* comm);

/* ---- stateless codec / update kernels (current device) ---------------- */
int gp_encode(int codec, const float* in, uint64_t n, void* payload, gp_codec_status* status,
              void* stream);
int gp_decode(int codec, const void* payload, const float* scale /* device, quant8 */, uint64_t n,
              float* out, void* stream);
int gp_roundtrip(int codec, const float* in, float* out, uint64_t n, gp_codec_status* status,
                 void* stream);
int gp_consume_update(float* params, int codec, const void* slot, const float* slot_scale,
                      uint64_t n, float lr, int world, void* stream);
/* Same, with the learning rate read from device memory (one fp32): a CUDA
 * graph captures this call once and each replay uses the rate the host wrote
 * before it (models.py / engine.py:287-292 learning-rate decay under replay). */
int gp_consume_update_dev(float* params, int codec, const void* slot, const float* slot_scale,
                          uint64_t n, const float* lr, int world, void* stream);

/* ---- calibration (timing-model alpha/beta on NVLink) ------------------- */
int gp_calib_p2p_copy(void* dst, const void* src, uint64_t bytes, int ctas, int pull, void* stream);
/* mode: bit0 pull, bit1 contiguous chunks from a device counter, bit2 release a flag per chunk */
int gp_calib_p2p_copy_ex(void* dst, const void* src, uint64_t bytes, int ctas, int mode, uint64_t chunk_bytes,
                         void* counter /* device u64, zeroed */, void* flags /* device u64[] */, void* stream);
/* One reduce-scatter hop on one GPU for the timing model's gamma (the
 * reference calibrate()'s reduce_hop, harness.py:561-568): out = C(x + D(in))
 * with the block scale of the sum (quant8: two passes), scale into st; `grid`
 * lets the probe run on the ring's own thread budget. */
int gp_calib_hop(int codec, const float* x, const void* in, const float* in_scale, void* out, uint64_t n,
                 int grid /* CTAs of 256 threads; 0 = fill the GPU */, gp_codec_status* st, void* stream);
/* All-to-all flag barrier across the communicator's ranks, `rounds` times in
 * one launch (the timing model's S, the reference barrier probe
 * harness.py:589-609); every rank must call it; elapsed ns -> ns_out (device
 * u64, ~0 on timeout). */
int gp_comm_barrier(gp_comm* comm, int rounds, void* ns_out, void* stream);
/* Bounds-checked build (libpipesgd_checked.so) only: payload bytes the ring
 * kernels of `rank` stored into other ranks' inboxes since the last reset --
 * the bytes a multi-GPU run moves over NVLink, counted by the kernel itself.
 * Always 0 in the product build. */
int gp_comm_wire_bytes(gp_comm* comm, int rank, int reset, uint64_t* out);
int gp_calib_pingpong(void* mine, void* theirs, int iters, int initiator, uint64_t base,
                      void* ns_out /* device u64 */, void* stream);

const char* gp_last_error_string(void);
int gp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PIPESGD_H_ */
