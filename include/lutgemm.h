/*
 * lutgemm.h -- C ABI of the B200-native LUT-GEMM hot path (arXiv 2206.09557).
 *
 * The operation (Sec. 3.2, with the Eq. 3 bias):
 *
 *     y[beta][r] = sum_c ( sum_{i<q} alpha[r][c/g][i] * b_i[r][c] + z[r][c/g] ) * x[beta][c]
 *
 * for a q-bit extended-BCQ weight W (m rows, n reduction columns), binary
 * planes b_i in {-1,+1}, group-wise scales alpha shared by g consecutive columns
 * (Sec. 3.4), optional bias z (Eq. 3), and fp16 activations.  The
 * kernels evaluate it as the paper does: one lookup table of all 2^8 signed
 * partial sums per 8-column chunk of x, built in shared memory (mu = 8,
 * P:L192-199, App. B), indexed by the packed sign bits.
 *
 * Conventions (all calls):
 *  - Plain C.  fp16 values travel as uint16_t bit patterns (IEEE binary16).
 *  - "device" pointers are CUDA global-memory pointers on the current device;
 *    "host" pointers are CPU memory.  The library never allocates on the hot
 *    path; every buffer is caller-owned (the Python binding uses PyTorch
 *    tensors for this).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Every device call is asynchronous on that stream; launch errors return
 *    LUTGEMM_ERR_CUDA, execution errors surface at stream synchronisation.
 *  - No C++ exception crosses the ABI.  On any non-OK status,
 *    lutgemm_last_error() returns a thread-local description.
 *  - The library is stateless except for an explicit TP communicator and the
 *    thread-local error text; calls on distinct outputs/workspaces are
 *    thread-safe.
 *  - Supported shapes: n % 8 == 0, g % 8 == 0, n % g == 0
 *    (g is "an arbitrary number of weights"; g == n is row-wise,
 *    P:L496 '-' / P:L392 "g=m"); 1 <= q <= 8, m >= 1, 1 <= b <= 32.  Anything
 *    else returns LUTGEMM_ERR_INVALID_ARG.  A mu = 8 chunk never straddles a
 *    group under this rule (R13).  Groups that are not a multiple of
 *    32 columns (g % 32 != 0, e.g. 8, 24, 40) split a 32-column word: those
 *    weights store one scale entry per 8-column chunk and run the generic-q
 *    kernels (correct, untuned); the UNIFORM_COMPACT format and the
 *    quantizers need g % 32 == 0 (and the quantizers n % 32 == 0).
 *  - Requires an sm_100 device (B200); otherwise LUTGEMM_ERR_UNSUPPORTED.
 */
#ifndef LUTGEMM_H_
#define LUTGEMM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LUTGEMM_ABI_VERSION 1

typedef enum {
  LUTGEMM_OK = 0,
  LUTGEMM_ERR_INVALID_ARG = 1, /* shape rule above violated, NULL pointer, bad enum */
  LUTGEMM_ERR_MISALIGNED = 2,  /* a device pointer violates the stated alignment */
  LUTGEMM_ERR_WORKSPACE = 3,   /* ws too small (see lutgemm_workspace_bytes) */
  LUTGEMM_ERR_CUDA = 4,        /* CUDA runtime error (launch / attribute / device) */
  LUTGEMM_ERR_NCCL = 5,        /* NCCL error in a lutgemm_tp_* call */
  LUTGEMM_ERR_UNSUPPORTED = 6  /* current device is not sm_100 */
} lutgemm_status;

/* A packed weight in the kernel-native layout: ONE device buffer holding the
 * bit-planes, scales and (if has_offset) biases as a slice-major stream of
 * per-row-quad records (opaque byte order).
 * The struct lives on the host; `data` (lutgemm_packed_bytes() bytes,
 * 16-byte aligned) lives on the device and is owned by the caller. */
typedef struct {
  int32_t m, n, q, g;
  int32_t has_offset; /* 1: extended BCQ with bias z (Eq. 3); 0: z = 0 */
  int32_t format;     /* LUTGEMM_FMT_BCQ or LUTGEMM_FMT_UNIFORM_COMPACT (set by lutgemm_pack_bcq) */
  void* data;
} lutgemm_weight;

/* Stored-scale formats of a packed weight.
 *  BCQ: q fp16 scales alpha_i per (row, group) (+ z if has_offset) -- any
 *       extended-BCQ weight (Eq. 3, group-wise P:L296).
 *  UNIFORM_COMPACT: a uniform-quantized weight (App. C) keeps ONE
 *       fp16 scale s and the fp16 bias z per (row, group); the kernels derive
 *       alpha_i = 2^(i-1) s exactly (power-of-two scaling).  Same product as the
 *       BCQ conversion of the same source, with q-1 fewer scale loads per group
 *       (Table 5 counts one scale per group, R18). has_offset = 1. */
enum { LUTGEMM_FMT_BCQ = 0, LUTGEMM_FMT_UNIFORM_COMPACT = 1 };

/* UNIFORM_COMPACT: as UNIFORM, but packed into the UNIFORM_COMPACT format. */
enum { LUTGEMM_SRC_BCQ = 0, LUTGEMM_SRC_UNIFORM = 1, LUTGEMM_SRC_UNIFORM_COMPACT = 2 };

/* Source of a pack call, canonical layout, all device pointers.
 * BCQ (non-uniform, Eq. 3):
 *   planes : uint32 [q][m][n/32]; bit j of word w of row r of plane i is
 *            b_i[r][32w+j]; bit 1 means +1, bit 0 means -1 (R1, from
 *            b = 2*b_hat - 1).  Plane 0 first (R4).
 *   alpha  : fp16 [m][n/g][q]      (scale per row, group, plane; R7)
 *   offset : fp16 [m][n/g] or NULL (bias z per row and group; R5)
 * UNIFORM (App. C): w = s * code + z_hat (Eq. 6), converted on the
 * device to alpha_i = 2^(i-1) s, b_i = 2 * bit_i(code) - 1,
 * z = sum_i alpha_i + z_hat (Eq. 8), stored as fp16 (round to nearest even;
 * z is summed in fp64 before the single rounding, R17).
 *   codes  : uint8 [m][n], 0 <= code < 2^q
 *   scale  : fp16 [m][n/g]  (s)
 *   zero   : fp16 [m][n/g]  (z_hat, additive; an integer zero-point zp maps to
 *            z_hat = -s * zp, R16)
 * Source pointers need only their natural element alignment. */
typedef struct {
  int32_t kind; /* LUTGEMM_SRC_BCQ | LUTGEMM_SRC_UNIFORM */
  int32_t m, n, q, g;
  int32_t reserved;
  const uint32_t* planes;
  const uint16_t* alpha;
  const uint16_t* offset;
  const uint8_t* codes;
  const uint16_t* scale;
  const uint16_t* zero;
} lutgemm_pack_src;

/* Library ABI version (LUTGEMM_ABI_VERSION). */
int lutgemm_abi_version(void);

/* sha256 prefix (24 hex digits) of the sources and compile flags this library
 * was built from (paper_2206_09557_b200/_build.py); the Python binding refuses
 * to load a library whose hash differs from the tree it sits in. */
const char* lutgemm_source_hash(void);

/* Thread-local text for the last non-OK status returned on this thread. */
const char* lutgemm_last_error(void);

/* Byte size of the native buffer of an (m, n, q, g, has_offset) weight:
 * m4*n*q/8 bits + the stored scales/biases (+ 16-byte record padding), with
 * m4 = 4*ceil(m/4).  Pure host computation. */
lutgemm_status lutgemm_packed_bytes(int m, int n, int q, int g, int has_offset, size_t* bytes);

/* As lutgemm_packed_bytes for a given format (LUTGEMM_FMT_*); the
 * UNIFORM_COMPACT format implies has_offset = 1. */
lutgemm_status lutgemm_packed_bytes_fmt(int m, int n, int q, int g, int has_offset, int format, size_t* bytes);

/* Repack a canonical BCQ or uniform source into dst->data (which the caller
 * allocated with lutgemm_packed_bytes_fmt(..., has_offset, format) bytes:
 * has_offset = 1 for UNIFORM / UNIFORM_COMPACT, and for BCQ iff src->offset !=
 * NULL; format = UNIFORM_COMPACT for that source kind, else BCQ).  The call
 * fills dst->m, n, q, g, has_offset, format.  Offline step (App. C "two-step
 * methodology"); asynchronous on `stream`. */
lutgemm_status lutgemm_pack_bcq(const lutgemm_pack_src* src, lutgemm_weight* dst, void* stream);

/* Inverse of the BCQ pack (test-only): native -> canonical planes / alpha /
 * offset (offset may be NULL).  Bit-exact round trip.  A UNIFORM_COMPACT
 * weight unpacks to the alpha_i = 2^(i-1) s of its stored s (fp16-exact for
 * the normal s the generators draw), i.e. to the UNIFORM pack of the same source. */
lutgemm_status lutgemm_unpack_bcq(const lutgemm_weight* w, uint32_t* planes, uint16_t* alpha,
                                  uint16_t* offset, void* stream);

/* ---- Quantizers (the offline step before the path) ----
 * Input: a dense weight W, device fp16 [m][n] row-major; same shape rules as
 * every call plus n % 32 == 0 and g % 32 == 0.  Outputs are the canonical pack
 * sources above (device buffers, caller-owned), so a dense layer becomes a
 * packed weight with quantize_* followed by lutgemm_pack_bcq.  Offline,
 * asynchronous on `stream`, deterministic.
 *
 * RTN (the "RTN" baseline of Tables 3/6; conventions of SPEC S:L112-120): per
 * (row, group) s = fp16((max - min)/(2^q - 1)), z_hat = fp16(min) and
 * code = clamp(rint((w - z_hat)/s), 0, 2^q - 1) from the stored s and z_hat; a
 * constant group stores s = 1, codes 0.  Writes codes uint8 [m][n], scale and
 * zero fp16 [m][n/g] -- a LUTGEMM_SRC_UNIFORM(_COMPACT) source (App. C). */
lutgemm_status lutgemm_quantize_rtn(const uint16_t* W, int m, int n, int q, int g, uint8_t* codes, uint16_t* scale,
                                    uint16_t* zero, void* stream);

/* BCQ (Sec. 2.3; the "iterative solver" of App. E): greedy
 * residual fit per (row, group) -- b_i = sign(r) (sign(0) = +1), alpha_i =
 * fp16(mean |r|), r -= alpha_i b_i -- then `iters` alternating rounds (0 =
 * greedy only): alpha = least squares for the fixed signs (fp64 solve; a
 * singular B^T B keeps the previous alpha), then every element's signs = the
 * nearest of the 2^q levels sum_i +-alpha_i.  Writes planes uint32
 * [q][m][n/32] and alpha fp16 [m][n/g][q] -- a LUTGEMM_SRC_BCQ source.
 * LUTGEMM_ERR_INVALID_ARG if q * g / 8 + 2^(q+2) bytes exceed shared memory. */
lutgemm_status lutgemm_quantize_bcq(const uint16_t* W, int m, int n, int q, int g, int iters, uint32_t* planes,
                                    uint16_t* alpha, void* stream);

/* Workspace for a product with m rows, n columns, batch b: fp32 split-K
 * partials plus row-block arrival counters.  The workspace must be zeroed
 * once (lutgemm_workspace_init) before its first use; every successful call
 * leaves it ready for the next.  One workspace must not be used by two calls
 * that may run concurrently. */
size_t lutgemm_workspace_bytes(int m, int n, int b);
lutgemm_status lutgemm_workspace_init(void* ws, size_t ws_bytes, void* stream);

/* y = W x for one fp16 activation vector (b = 1), the paper's single-batch
 * case.  x: device fp16 [n], 16-byte aligned.  y: device fp16 [m],
 * 2-byte aligned, rounded to nearest even from an fp32 accumulation (R12).
 * ws: device, 16-byte aligned, >= lutgemm_workspace_bytes(m, n, 1).
 * Deterministic: fixed-order reductions, bitwise reproducible (R11). */
lutgemm_status lutgemm_gemv(const lutgemm_weight* w, const uint16_t* x, uint16_t* y, void* ws,
                            size_t ws_bytes, void* stream);

/* Y = X W^T for b activation rows (1 <= b <= 32): X device fp16 [b][n]
 * (16-byte aligned, rows contiguous), Y device fp16 [b][m].  Same LUT method,
 * one table bank per activation row sharing each key. */
lutgemm_status lutgemm_gemm_batched(const lutgemm_weight* w, const uint16_t* X, int b, uint16_t* Y,
                                    void* ws, size_t ws_bytes, void* stream);

/* As lutgemm_gemm_batched but writes the fp32 result Yf [b][m] (no fp16
 * rounding): the local partial of a column-split tensor-parallel shard. */
lutgemm_status lutgemm_gemm_batched_f32(const lutgemm_weight* w, const uint16_t* X, int b, float* Yf,
                                        void* ws, size_t ws_bytes, void* stream);

/* End-to-end call with HOST activations and outputs: copies X_host [b][n]
 * (fp16, ideally pinned) to the device staging area inside ws, runs the
 * product, delivers Y [b][m] to Y_host and synchronises `stream` before
 * returning.  When Y_host is page-locked and device-mapped (cudaHostAlloc,
 * torch pin_memory under UVA) the product's epilogue stores Y straight into
 * it; otherwise Y is staged in ws and copied back.  ws (device, 16-byte
 * aligned) must hold lutgemm_host_workspace_bytes(m, n, b) bytes and be
 * initialised like any workspace.  The weight stays resident on the device. */
size_t lutgemm_host_workspace_bytes(int m, int n, int b);
lutgemm_status lutgemm_gemm_host(const lutgemm_weight* w, const uint16_t* X_host, int b, uint16_t* Y_host,
                                 void* ws, size_t ws_bytes, void* stream);

/* Tracing (debug; not for the hot path).  Enabling clears the buffer; then every subsequent
 * product launch records a per-CTA %globaltimer timeline into a library-owned
 * device buffer (8 u64 per CTA, up to 1024 CTAs, last launch wins):
 * [0] CTA start, [1] x slice in hand (registers or staged), [2] first LUT built,
 * [3] PDL wait done, [4] all warps done with the first segment, [5] row group
 * complete (fused GEMV reducer CTAs), [6] CTA end (reduction share done),
 * [7] SM id (high word: segments processed).  lutgemm_trace_read copies up to
 * n values to host memory (synchronous) and returns how many it copied. */
lutgemm_status lutgemm_trace_enable(int on);
size_t lutgemm_trace_read(uint64_t* host, size_t n);

/* Number of product kernels (LUT-GEMV / LUT-GEMM and their reduction
 * kernels, not pack kernels) this process has launched through the library --
 * host-side count; a CUDA graph replay re-runs the launches captured in it
 * without counting them again.  For benchmark accounting. */
uint64_t lutgemm_launch_count(void);

/* ---------------- Tensor parallelism over NCCL (NVLink / NVSwitch) ----------------
 * The paper runs LUT-GEMM tensor-parallel on 1/2/4/8 GPUs (P:L378-385,
 * Table 2, Tables 3/4) and names communication as what limits it
 * (P:L411-413).  One process per GPU; the NCCL unique id is produced on rank
 * 0 and broadcast by the caller (the Python binding uses torch.distributed). */
typedef struct lutgemm_tp lutgemm_tp;

enum {
  LUTGEMM_TP_ROWS_LOCAL = 0,     /* shard = rows [r*m/P,(r+1)*m/P); x full; y = local rows only */
  LUTGEMM_TP_ROWS_ALLGATHER = 1, /* same shard; y = full [b][m] replicated via ncclAllGather */
  LUTGEMM_TP_COLS_ALLREDUCE = 2  /* shard = columns [r*n/P,(r+1)*n/P) (multiple of g); x = local
                                    slice [b][n/P]; fp32 partials ncclAllReduce(sum), then fp16 y [b][m] */
};

/* 128-byte opaque NCCL unique id, to be created on rank 0 only. */
lutgemm_status lutgemm_tp_unique_id(uint8_t id[128]);
/* Create the communicator (collective over all ranks; current CUDA device is used). */
lutgemm_status lutgemm_tp_init(int nranks, int rank, const uint8_t id[128], lutgemm_tp** out);
/* Workspace for lutgemm_tp_linear with this shard and mode. */
size_t lutgemm_tp_workspace_bytes(const lutgemm_tp* tp, int mode, int m_shard, int n_shard, int b);
/* One tensor-parallel linear: the shard's LUT-GEMM followed by the mode's
 * collective, all on `stream` (graph-capturable).  `shard` is this rank's
 * packed shard (m_shard x n_shard).  y layout per mode as above; for
 * ROWS_ALLGATHER y is [b][P*m_shard].  ws is >= lutgemm_tp_workspace_bytes. */
lutgemm_status lutgemm_tp_linear(lutgemm_tp* tp, int mode, const lutgemm_weight* shard,
                                 const uint16_t* x, int b, uint16_t* y, void* ws, size_t ws_bytes,
                                 void* stream);
lutgemm_status lutgemm_tp_destroy(lutgemm_tp* tp);
/* Failure detection (host polling): LUTGEMM_ERR_NCCL with the text of the error if the
 * communicator hit an asynchronous error (e.g. a peer died), else LUTGEMM_OK.  Poll it while
 * waiting for a stream that runs collectives, so a broken collective does not hang silently. */
lutgemm_status lutgemm_tp_async_error(lutgemm_tp* tp);
/* Abort the communicator (unblocks kernels stuck in its collectives) and free the handle. */
lutgemm_status lutgemm_tp_abort(lutgemm_tp* tp);
int lutgemm_tp_rank(const lutgemm_tp* tp);
int lutgemm_tp_nranks(const lutgemm_tp* tp);

/* ---------------- Tensor-parallel exchange fused into the GEMV ----------------
 * The collectives of lutgemm_tp_linear's ROWS_ALLGATHER and COLS_ALLREDUCE modes fused into
 * the GEMV's epilogue over peer memory (CUDA IPC mappings over NVLink / NVSwitch), no NCCL call;
 * one process per GPU (communication limits tensor parallelism once the matmul is
 * fast).  A call is ONE kernel on `stream`: the exchange runs in the fused GEMV's epilogue, in
 * the reducer CTAs, one thread per output row, as LL words (8-byte stores of 4 data bytes
 * and a 4-byte round stamp, polled by the reader: no fence or separate signal):
 *  - ROWS (m-split): each finished fp16 row pair of this rank's shard goes to y and into every
 *    peer's exchange window; each reducer then reads the peers' rows of its own share out of the
 *    local window into y (every rank runs the same reducer partition).
 *  - COLS (n-split): reduce-scatter + all-gather.  Rank o owns rows [o mb, (o+1) mb),
 *    mb = 8 ceil(ceil(m/P)/8); each fp32 row goes to its owner's window only; each rank sums its
 *    owned rows over the P slots in rank order (deterministic, bitwise identical on every rank,
 *    within tolerance of the 1-GPU result), rounds to fp16 and sends the row pairs to every
 *    peer, which copy them into y.  Every rank must own rows ((P - 1) mb < m), else
 *    LUTGEMM_ERR_INVALID_ARG.
 * The round number lives on the device, so calls are CUDA-graph capturable; each rank owns two
 * windows (double buffer by round parity).  Every rank must make the same sequence of calls on
 * a group.  y is complete when the call's kernel completes on the stream.  A reader that sees no
 * word from a peer for 30 s (env LUTGEMM_P2P_TIMEOUT_MS) traps: the launch fails (a sticky CUDA
 * error) instead of hanging. */
typedef struct lutgemm_p2p lutgemm_p2p;

/* Bytes of one exchange window for `mode` (LUTGEMM_TP_ROWS_ALLGATHER: m = rows of the gathered
 * output, P * m_shard; LUTGEMM_TP_COLS_ALLREDUCE: m = rows of the layer); 0 on bad arguments.
 * A group serves every call whose need is <= its window size. */
size_t lutgemm_p2p_window_bytes(int nranks, int mode, int m);
/* Allocate this rank's two windows (win_bytes each, device) and its (local) round word and write a 256-byte
 * exchange record (CUDA IPC handles, rank, sizes) that the caller gathers from all ranks, in rank
 * order, by any transport.  1 <= nranks <= 8.  Collective in the sense that every rank creates
 * one group with the same win_bytes. */
lutgemm_status lutgemm_p2p_create(int rank, int nranks, size_t win_bytes, lutgemm_p2p** out, uint8_t record[256]);
/* Open the peers' windows from the gathered records [nranks][256]; once per group (a second call
 * is rejected; on failure every mapping it opened is closed). */
lutgemm_status lutgemm_p2p_connect(lutgemm_p2p* g, const uint8_t* records);
/* ROWS: y [P * m_shard] (fp16, device, caller-owned, 2-byte aligned) = every rank's shard rows
 * times x.  shard: this rank's rows [r m_shard, (r+1) m_shard) of W, packed, m_shard % 8 == 0;
 * x [n] fp16 (16-byte aligned); ws >= lutgemm_workspace_bytes(m_shard, n, 1).  The shard must run
 * the fused GEMV mode (LUTGEMM_ERR_UNSUPPORTED otherwise: too few row quads for the J CTAs per
 * slice, or more slices than SMs).  Validated like lutgemm_gemv. */
lutgemm_status lutgemm_p2p_gemv_allgather(lutgemm_p2p* g, const lutgemm_weight* shard, const uint16_t* x, void* ws,
                                          size_t ws_bytes, void* stream, uint16_t* y);
/* COLS: y [m] (fp16, device) = sum over ranks of (shard_r [m][n/P]) x_r, x_r = this rank's slice of
 * x [n/P] (columns aligned to g).  Same requirements as above. */
lutgemm_status lutgemm_p2p_gemv_allreduce(lutgemm_p2p* g, const lutgemm_weight* shard, const uint16_t* x, void* ws,
                                          size_t ws_bytes, void* stream, uint16_t* y);
/* Synchronises the group's device, closes the peer mappings and frees the windows. */
lutgemm_status lutgemm_p2p_destroy(lutgemm_p2p* g);

#ifdef __cplusplus
}
#endif

#endif /* LUTGEMM_H_ */
