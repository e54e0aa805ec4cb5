/*
 * rf.h — C ABI of the B200-native random-features Gram / closed-form-kernel library
 * (arXiv 2110.01899, "Ternary Random Features").  Shared library: paper_2110_01899_b200/librf_b200.so
 *
 * Citations "P:<line>" are lines of the paper text.  Notation follows the paper:
 *   X = [x_1 … x_n] ∈ R^{p×n} data (P:5);  W ∈ R^{m×p} random projection, rows w_k;
 *   Σ = σ(WX) ∈ R^{m×n} random features (P:3);  G = (1/m) ΣᵀΣ ∈ R^{n×n} (Eq. def_Gram);
 *   Φ(x_i,x_j) = E_w σ(wᵀx_i)σ(wᵀx_j) approximated by the Taylor closed form EQ1;
 *   τ estimated by Lemma 1, τ̂ = (1/n)Σ‖x_i‖² (Algorithm 1 step 1 P:739).
 *
 * MEMORY LAYOUT (all row-major, element strides in ELEMENTS):
 *   X  : sample-major, X[i*ldx + l] = component l of sample x_i   (n rows of p values; = the paper's
 *        column-major p×n).  ldx ≥ p.
 *   W  : W[k*ldw + l] = component l of w_k                         (m_local rows of p values). ldw ≥ p.
 *   G, Φ : out[i*ld + j] = entry (i, j), 0 ≤ i, j < n.  ld ≥ n.
 *
 * DTYPES / PRECISION MODES (validated; no silent casts):
 *   RF_PREC_FP64   X, W f64 ; output f64 ; SIMT DFMA (small problems / reference mode)
 *   RF_PREC_FP32   X, W f32 ; output f32 ; SIMT FFMA, fp32-accurate
 *   RF_PREC_3XTF32 X, W f32 ; output f32 ; tcgen05 kind::tf32, hi·hi + hi·lo + lo·hi, fp32-accurate
 *   RF_PREC_TF32   X, W f32 ; output f32 ; tcgen05 kind::tf32, one pass (≈1e-3 class)
 *   RF_PREC_BF16   X, W bf16; output f32 ; tcgen05 kind::f16, Σ stored bf16, fp32 accumulation
 *
 * CONTEXT: every compute call takes an rf_ctx* first (NULL = this thread's default context of the current device):
 * it binds the call to a device, carries the tuning options and, once a collective is attached, the rank, the world
 * and the exchange resources of the multi-GPU G (rf_ctx_* below).  A context is not thread-safe: use one per thread.
 *
 * OWNERSHIP: the caller allocates every device buffer (inputs, outputs, workspace).  The library never
 * allocates device memory on a call path and keeps no pointer to a caller buffer after a call returns.  Only
 * context set-up allocates: rf_ctx_attach_peers (the staging buffer other ranks store G tiles into) and
 * rf_ctx_init_nccl / rf_ctx_attach_nccl (64 B of chunk counters); rf_ctx_destroy frees them.
 *
 * ASYNC: GPU work is enqueued on `stream` (a cudaStream_t passed as void*; NULL = legacy default stream)
 * and the call returns after enqueue, EXCEPT: rf_moments (host-only, synchronous); rf_estimate_tau and
 * rf_phi_closed_form with tau <= 0 (one 8-byte device→host copy + stream synchronize, because the
 * moments depend on τ).
 *
 * ERRORS: every argument is validated before any launch; on failure nothing is enqueued and the
 * status is returned with a message available from rf_last_error() (thread-local).  No C++ exception
 * crosses the ABI.  There is no CPU fallback: a device that is not sm_100 gives RF_E_UNSUPPORTED.
 */
#ifndef RF_B200_H
#define RF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RF_OK = 0,
  RF_E_INVALID = 1,      /* bad size / pointer / alignment / dtype-precision pair / τ <= 0 in rf_moments */
  RF_E_UNSUPPORTED = 2,  /* device is not sm_100 (B200) */
  RF_E_NONFINITE = 3,    /* σ non-finite at a quadrature node */
  RF_E_CUDA = 4,         /* a CUDA runtime/driver error (launch failure, earlier async fault) */
  RF_E_NCCL = 5,         /* NCCL missing from the process, or an NCCL call / the communicator's async error failed */
  RF_E_WORKSPACE = 6     /* workspace pointer NULL or smaller than rf_*_workspace_size() */
} rf_status;

/* σ ∈ {tanh, erf, sigmoid − 1/2}: the north star's activations (Assumption 3).
 * NEXT-3 adds the parameter-free activations of Table 2: ReLU max(0,t), |t|, sign(t), 1_{t>0},
 * cos t, sin t, t, t², the bump e^{−t²/2}.  Their derivatives are taken in the weak sense (Remark 2):
 * rf_moments evaluates ⟨k,d⟩ from σ alone through Stein's lemma (see rf_moments). */
typedef enum {
  RF_ACT_TANH = 0, RF_ACT_ERF = 1, RF_ACT_SIGMOID_HALF = 2,
  RF_ACT_RELU = 3, RF_ACT_ABS = 4, RF_ACT_SIGN = 5, RF_ACT_STEP = 6, RF_ACT_COS = 7, RF_ACT_SIN = 8,
  RF_ACT_IDENT = 9, RF_ACT_QUAD = 10, RF_ACT_BUMP = 11
} rf_act;
/* Table 2's two parametrised rows, registered at run time; the returned id is a valid rf_act for every
 * call (G through K3's runtime σ, moments through Stein as for the other Table-2 rows, Φ, TRF thresholds):
 *   rf_act_leaky_relu: σ(t) = a₊·max(0, t) + a₋·max(0, −t)   (ReLU: 1, 0;  |t|: 1, 1;  leaky ReLU slope s: 1, −s)
 *   rf_act_quadratic:  σ(t) = a₂t² + a₁t + a₀
 * Ids are RF_ACT_PARAM_BASE + k, process-wide and immutable; the same coefficients return the same id; at most
 * RF_ACT_PARAM_MAX registrations (then RF_E_INVALID).  Non-finite coefficients → RF_E_INVALID. */
#define RF_ACT_PARAM_BASE 64
#define RF_ACT_PARAM_MAX 64
rf_status rf_act_leaky_relu(double a_plus, double a_minus, rf_act* act);
rf_status rf_act_quadratic(double a0, double a1, double a2, rf_act* act);
typedef enum { RF_DT_F64 = 0, RF_DT_F32 = 1, RF_DT_BF16 = 2 } rf_dtype;
typedef enum { RF_PREC_FP64 = 0, RF_PREC_FP32 = 1, RF_PREC_3XTF32 = 2, RF_PREC_TF32 = 3, RF_PREC_BF16 = 4 } rf_prec;
/* UPPER: write only entries j >= i (the rest of the buffer is untouched).
 * FULL : write all n×n entries; the lower triangle mirrors the upper one (Φ: pivot = row, see below).
 * *_CENTERED (NEXT-2): the result is centered in place, K = P·A·P with P = I − (1/n)11ᵀ (Eq. (2)),
 *   as a post-pass (row sums of the symmetric matrix in fp64, then A_ij − r_i − r_j + s); it is linear, so per-rank
 *   partial G can each be centered.  Φ: only for the full row range.
 * PACKED_TRI: only the upper triangle's 256 × 256 tiles, contiguous: with T = ceil(n/256), tile (I, J ≥ I) (rows
 *   256I.., columns 256J..) starts at float offset 65536·(I·T − I(I−1)/2 + J − I) and is row-major with 256 floats
 *   per row; the buffer holds rf_packed_tri_elems(n) = 65536·T(T+1)/2 floats (≈ n²/2 + 128n) and must be 16-B
 *   aligned; ld is ignored.  Entries below the diagonal of diagonal tiles and entries past n are unspecified.
 *   Tensor-core precisions only (BF16, TF32, 3XTF32; rf_gram_ter); no centering.  It halves the bytes a host
 *   copy of G or Φ moves (the e2e path of bench.py).
 */
typedef enum {
  RF_OUT_UPPER = 0, RF_OUT_FULL = 1, RF_OUT_UPPER_CENTERED = 2, RF_OUT_FULL_CENTERED = 3, RF_OUT_PACKED_TRI = 4,
  RF_OUT_PACKED_TILES = 5   /* multi-GPU G: this rank's owned, SUMMED 256×256 tiles (rf_tile_map); rf_gram only */
} rf_out;
#define RF_OUT_CENTER 2
/* Number of floats of an RF_OUT_PACKED_TRI buffer for n samples (n > 0; else RF_E_INVALID). */
rf_status rf_packed_tri_elems(int64_t n, int64_t* elems);

/* Gaussian moments at τ (EQ1 coefficients P:1040; Theorem 1):
 *   kd[k][d] = E[(√τ ξ)^k σ^(d)(√τ ξ)], ξ ~ N(0,1), k = 0..4, d = 0..2
 *   e_sigma_sq = E[σ(√τ ξ)²]
 *   d0 = e_sigma_sq − kd[0][0]² − τ kd[0][1]²,  d1 = kd[0][1]²,  d2 = kd[0][2]²/4
 * method: 0 = Gauss–Hermite (Golub–Welsch, `nodes` points), 1 = composite trapezoid fallback. */
typedef struct {
  double tau;
  double kd[5][3];
  double e_sigma_sq;
  double d0, d1, d2;
  int32_t nodes;
  int32_t method;
  double quad_err_est;   /* |Q_N − Q_{N/2}| max over the table (GH), or the trapezoid h-halving change */
} rf_moments_t;

/* Thread-local text of the last error on this thread ("" after success). */
const char* rf_last_error(void);
const char* rf_version(void);

/* 1 if `device` is an sm_100 part this library's kernels run on, else 0 (no error text). */
int rf_device_supported(int device);

/* =============================================================================================
 * CONTEXT.  rf_ctx_create(device): a context bound to `device` (must be sm_100, else
 * RF_E_UNSUPPORTED); it owns a side stream (the concurrent tail launch of the K3/K4 multicast + pair hybrids) and
 * the options below.  rf_ctx_destroy releases everything the context allocated (NULL is a no-op); the caller must
 * have synchronized the streams it passed to calls on this context.
 * ============================================================================================= */
typedef struct rf_ctx rf_ctx;
rf_status rf_ctx_create(int device, rf_ctx** out);
void rf_ctx_destroy(rf_ctx* ctx);

/* Tuning options.  Defaults are the measured best; the alternatives exist for A/B measurement and
 * for the bit-exactness tests of the alternative kernels.  Value checks: RF_E_INVALID. */
typedef enum {
  RF_OPT_K3_HYBRID = 0,    /* 1: K3 as 4-CTA multicast clusters + pair clusters on the leftover SMs (n ≥ 32 row
                              tiles); 0: pair clusters only                                          default 1 */
  RF_OPT_K4_HYBRID = 1,    /* the same for K4 (n ≥ 64 row tiles)                                    default 1
                              Both hybrids' 4-CTA multicast kernels can hang when the GPU is time-sliced between
                              PROCESSES (compute preemption): set both to 0 when processes share a GPU.
                              One process per GPU never preempts them. */
  RF_OPT_K4_CL8 = 2,       /* 1: the K4 hybrid with 8-CTA clusters (2 × 2 pairs sharing A and B)     default 0 */
  RF_OPT_K4_SPLIT_R100 = 3,/* K4 hybrid work split: per-SM rate ratio multicast/pair × 100          default 111 */
  RF_OPT_K3_SPLIT_R100 = 4,/* K3 hybrid work split, as above                                        default 120 */
  RF_OPT_LOCK_W = 5,       /* K4 soft lockstep: allowed lead in K-blocks (0 = off)                  default 24 */
  RF_OPT_LOCK_KS = 6,      /* K4 soft lockstep: check period in K-blocks                            default 8 */
  RF_OPT_K5_WIDE = 7,      /* K5 epilogue warps: −1 auto (8), 0 → 8, 1 → 16                          default −1 */
  RF_OPT_EQ1_GENERAL = 8,  /* 1: the general EQ1 epilogue also for odd σ (A0, A2 kept)               default 0 */
  RF_OPT_KCHUNK = 9,       /* 3×TF32 K4 accumulation chunk in K-blocks (0 = whole K)                default 4 */
  RF_OPT_MAX_SMS = 10,     /* ≤ 0: all SMs; else the tensor-core kernels use at most this many       default 0 */
  RF_OPT_COMM_SMS = 11,    /* NCCL G5: SMs kept free of K4 for the overlapped reduce-scatter         default 8 */
  RF_OPT_VERBOSE = 12,     /* 1: print launch geometry to stderr                                     default 0 */
  RF_OPT_G5_PHASES = 13,   /* TEST HOOK, peers: which half of a collective rf_gram to enqueue — 1: K3 + K4 stores +
                              arrival flags, 2: the arrival waits + owner-side sums + release flags (on the caller's
                              stream), 3: the whole pipelined call (default).
                              Emulating R ranks on ONE GPU in one process: call phase 1 for every rank, then phase 2,
                              on one stream, so no stream-memory wait ever heads a queue its producer sits behind */
  RF_OPT_K4_DYNAMIC = 14,  /* 1: the K4 hybrid's two kernels pull 512 × 512 units of one raster from a shared device
                              counter (no static split); 0: the static split of RF_OPT_K4_SPLIT_R100     default 1 */
  RF_OPT_K5_ARES = 15,     /* K5 with A-panel residency (bf16, 256 < p ≤ 512): 0 off, 1 with 8, 2 with 16 (2-KB
                              staging), 3 with 12 epilogue warps                                      default 1 */
  RF_OPT_K5_DYNAMIC = 16,  /* 1: the A-resident K5 pulls its segments from a device counter (balanced last wave);
                              0: static round-robin                                                   default 1 */
  RF_OPT_G5_PIPE = 17,     /* peers: 1 = each chunk's owner-side sum on the context's reduce stream beside K4;
                              0 = all sums after K4 on the caller's stream                             default 1 */
  RF_OPT_COUNT = 18
} rf_opt;
rf_status rf_ctx_set_option(rf_ctx* ctx, rf_opt opt, int64_t value);
rf_status rf_ctx_get_option(const rf_ctx* ctx, rf_opt opt, int64_t* value);

/* =============================================================================================
 * G5 — the multi-GPU G.  G is a sum over the m features (Eq. def_Gram):
 * rank r holds W rows [m0, m1), computes the partial G_r = (1/m_total) Σ_{k ∈ its rows} σ(Xᵀw_k)σ(w_kᵀX), and
 * G = Σ_r G_r.  With a collective attached to the context, rf_gram(ctx, …, RF_OUT_PACKED_TILES, G = recv, …) is a
 * COLLECTIVE (every rank calls it with the same p, n, m_total, act, prec; its own W rows): K3 + K4 run on the rank's
 * features and K4's epilogue writes each upper-triangle 256×256 tile of the partial straight into its exchange
 * slot; the call returns (enqueued) with recv = this rank's owned tiles, SUMMED over all ranks.
 *
 * Tile ownership (rf_tile_map; a function of n and world only): the T = ⌈n/256⌉ row tiles are cut into C ≤ 16
 * chunks of whole 8-row-tile groups with near-equal triangle area; inside chunk c the upper 256-tiles (I, J ≥ I) are
 * numbered row-major, u = 0, 1, …, and tile u goes to owner u mod world at slot u div world.  recv holds, chunk after
 * chunk, chunk_slots[c] = ⌈tiles_c / world⌉ tiles of 65536 floats (row-major 256 × 256); slot s of the whole buffer
 * is the pair (I, J) rf_tile_map returns, or (−1, −1) for a padding slot (content unspecified).  Whole tiles are
 * stored: a diagonal tile also holds the mirror entries below the diagonal, entries with i or j ≥ n are 0.
 *
 * Two exchanges, chosen by what is attached:
 *   PEERS (the product path): each rank's context owns a staging buffer (world × recv floats + flags, one
 *     cudaMalloc); ranks exchange 64-byte CUDA IPC handles (rf_ctx_peer_handle / rf_ctx_open_peers) or, in one
 *     process, raw pointers (rf_ctx_peer_base / rf_ctx_connect_peers).  K4's epilogue stores every tile into its
 *     owner's staging buffer over NVLink as it finishes (the exchange overlaps the SYRK, no collective kernel), then
 *     device epoch flags (peer-mapped words written with system-scope release by a one-thread kernel, awaited with
 *     stream-memory waits) order the owner-side sum in rank order (deterministic) and the next call's stores —
 *     no host synchronization, no barrier.  Chunk-pipelined: K4 counts each chunk's finished pair tiles; on the
 *     context's comm stream chunk c's arrival flag goes to every owner as soon as its count is complete, and on the
 *     context's reduce stream chunk c is summed as soon as every source's flag for it is up — beside K4, which is
 *     still computing the later chunks (the caller's stream waits for both streams before the call's end).
 *   NCCL (the baseline): K4 writes a packed send buffer (in the workspace) chunk by chunk and bumps a per-chunk
 *     counter; on the context's communication stream each chunk's ncclReduceScatter waits (stream-memory wait) for
 *     its counter, so chunk c is reduced while K4 computes chunk c + 1.  K4 leaves RF_OPT_COMM_SMS SMs free.
 * rf_gram with RF_OUT_UPPER / RF_OUT_FULL on such a context computes the rank's PARTIAL G (no exchange).
 * ============================================================================================= */
#define RF_PACK_TILE 256
#define RF_MAX_PEERS 16
/* Host.  *tiles_owned = the receive slots of `rank` (padding included); ij_pairs (nullable, 2·slots int64): (I, J)
 * of each slot in recv order, (−1, −1) for padding.  tile must be 256.  n > 0, 1 ≤ world ≤ 4096, 0 ≤ rank < world. */
rf_status rf_tile_map(int64_t n, int32_t tile, int32_t world, int32_t rank, int64_t* tiles_owned, int64_t* ij_pairs);

/* NCCL.  rf_nccl_get_unique_id: a new ncclUniqueId (128 bytes) on one rank, to be broadcast by the caller's process
 * group; rf_ctx_init_nccl: every rank creates the communicator from it (ncclCommInitRank; owned by the context).
 * rf_ctx_attach_nccl: use a caller-owned ncclComm_t instead (kept until rf_ctx_destroy, not destroyed by it).
 * NCCL is taken from the process (dlopen "libnccl.so.2": the copy torch loads); absent → RF_E_NCCL.  Every collective
 * rf_gram first polls ncclCommGetAsyncError: an error → RF_E_NCCL. */
rf_status rf_nccl_get_unique_id(uint8_t id128[128]);
rf_status rf_ctx_init_nccl(rf_ctx* ctx, const uint8_t id128[128], int32_t rank, int32_t world);
rf_status rf_ctx_attach_nccl(rf_ctx* ctx, void* nccl_comm, int32_t rank, int32_t world);

/* Peers.  rf_ctx_attach_peers: allocate this rank's staging buffer for n ≤ n_max (world ≤ RF_MAX_PEERS; zero-filled).
 * rf_ctx_peer_handle: its 64-byte CUDA IPC handle (the handle names exactly that allocation).
 * rf_ctx_open_peers: map the other ranks' buffers from their handles (handles64 = world × 64 bytes, rank order; the
 *   own entry is ignored).  rf_ctx_peer_base / rf_ctx_connect_peers: the same with raw device pointers, for ranks
 *   that share one address space (several contexts in one process).  Every rank's context must be attached with
 *   the same world and n_max. */
rf_status rf_ctx_attach_peers(rf_ctx* ctx, int32_t rank, int32_t world, int64_t n_max);
rf_status rf_ctx_peer_handle(const rf_ctx* ctx, uint8_t handle64[64]);
rf_status rf_ctx_open_peers(rf_ctx* ctx, const uint8_t* handles64);
rf_status rf_ctx_peer_base(const rf_ctx* ctx, void** base);
rf_status rf_ctx_connect_peers(rf_ctx* ctx, void* const* bases);
/* rank, world and exchange of a context: *mode = 0 none, 1 NCCL, 2 peers (NULL outputs skipped). */
rf_status rf_ctx_collective(const rf_ctx* ctx, int32_t* rank, int32_t* world, int32_t* mode);

/* rf_workspace_size — bytes of workspace a call needs (op 0: rf_gram, 1: rf_phi_closed_form / rf_phi_eq2) for these
 * sizes on this context: rf_gram with RF_OUT_PACKED_TILES on an NCCL context also holds the packed send buffer. */
rf_status rf_workspace_size(const rf_ctx* ctx, int32_t op, int64_t p, int64_t n, int64_t m_local, rf_prec prec,
                            rf_out out, size_t* bytes);

/* ---------------------------------------------------------------------------------------------
 * rf_moments — host, synchronous.  Gauss–Hermite quadrature (probabilists' weight) by Golub–Welsch;
 * nodes = 0 → adaptive (N = 64, 128, 256, 512 until the table changes by < 1e-13, else trapezoid on
 * [−40, 40], h = 0.05).  nodes > 0 → exactly that many GH nodes (2 ≤ nodes ≤ 1024).
 * Errors: tau <= 0 or not finite → RF_E_INVALID; out == NULL → RF_E_INVALID; non-finite σ → RF_E_NONFINITE.
 */
rf_status rf_moments(rf_act act, double tau, int32_t nodes, rf_moments_t* out);
/* NEXT-3 activations (RF_ACT_RELU … RF_ACT_BUMP): nodes is ignored; M_j = E[ξ^j σ(√τξ)] (j ≤ 6) and E[σ²] by
 * composite Gauss–Legendre on [−L, 0] ∪ [0, L] (split at the kink / jump t = 0, L = 12, 48 panels × 24 nodes per
 * half), then ⟨k,0⟩ = τ^{k/2}M_k, ⟨k,1⟩ = τ^{(k−1)/2}(M_{k+1} − kM_{k−1}),
 * ⟨k,2⟩ = τ^{k/2−1}(M_{k+2} − (2k+1)M_k + k(k−1)M_{k−2}) (Stein once / twice); method = 2. */

/* ---------------------------------------------------------------------------------------------
 * rf_estimate_tau — Lemma 1: *tau_out = (1/n) Σ_i ‖x_i‖², fp64 accumulation, deterministic
 * order.  Device X (layout above, dtype x_dt), device workspace of rf_tau_workspace_size(n) bytes.
 * Synchronizes `stream` (8-byte D2H copy into *tau_out, a host pointer).
 */
rf_status rf_tau_workspace_size(int64_t n, size_t* bytes);
rf_status rf_estimate_tau(rf_ctx* ctx, const void* X, rf_dtype x_dt, int64_t ldx, int64_t p, int64_t n,
                          double* tau_out, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------
 * rf_round_bf16 — step G1 for RF_PREC_BF16 (X, W of P:470 in the north star's BF16 mode):
 *   dst[r·ldd + c] = bf16(src[r·lds + c]) for r < rows, c < cols, IEEE round to nearest, ties to even;
 *   ±inf stay ±inf, NaN stays a NaN (canonical payload), overflow past the bf16 range rounds to ±inf.
 *   src     device fp32, rows × cols, row stride lds ≥ cols elements, 4-B aligned
 *   dst     device bf16, rows × cols, row stride ldd ≥ cols elements, 2-B aligned; caller-owned
 *   Enqueued on `stream`; one launch (16-B vector path when cols, lds, ldd are multiples of 4 and the
 *   bases 16-B / 8-B aligned).  rows = 0 or cols = 0 → RF_OK, no launch.  Negative sizes, NULL
 *   buffers, ld < cols or misalignment → RF_E_INVALID.  Use it on X and W before rf_gram /
 *   rf_phi_closed_form in BF16 mode when the data are fp32.
 */
rf_status rf_round_bf16(rf_ctx* ctx, const float* src, int64_t lds, int64_t rows, int64_t cols, void* dst, int64_t ldd,
                        void* stream);

/* ---------------------------------------------------------------------------------------------
 * rf_gram — G = (1/m_total) Σ_{k < m_local} σ(w_kᵀx_i) σ(w_kᵀx_j)   (Eq. def_Gram)
 *   X       device, n × p (ldx), dtype per `prec`
 *   W_local device, m_local × p (ldw): this rank's rows of W (m_local = m_total on one GPU).  The
 *           sum over the rank's features is scaled by 1/m_total so that summing the partial G of all
 *           ranks (reduce-scatter / all-reduce) gives G.
 *   G       device, n × n (ldg), f64 in RF_PREC_FP64 else f32; `out` selects UPPER or FULL (or a centred form,
 *           or PACKED_TRI).  RF_OUT_PACKED_TILES (context with a collective attached, BF16 / TF32; 3XTF32 on NCCL
 *           only): G is this rank's receive buffer of rf_tile_map(n, 256, world, rank) slots × 65536 floats, ldg
 *           ignored, and the call is the collective described under G5 above.
 *   ws      device workspace ≥ rf_workspace_size(ctx, 0, p, n, m_local, prec, out) bytes, 256-B aligned
 *           (holds Σᵀ = σ(XᵀW_localᵀ), n × m_local, never written to HBM in fp32 in BF16 mode; and the NCCL send
 *           buffer).  rf_gram_workspace_size(p, n, m_local, prec) is the same number for a context without NCCL.
 * Pipeline: [3XTF32: K2 split X, W] → K3 fused Σᵀ = σ(X·Wᵀ) (tcgen05 GEMM, σ in the epilogue)
 *           → K4 upper-triangular SYRK G = ΣᵀΣ/m over 256×512 CTA-pair tiles with j ≥ i (3XTF32:
 *           256×256 tiles, K cut into chunks of 128 features whose partial sums are added in fp32, in TMEM, to
 *           bound the tensor pipe's truncating accumulation).
 * Alignment: X, W 16-B aligned with ldx·esize, ldw·esize multiples of 16 B (TMA); G aligned to its element
 *            size, any ldg ≥ n (16-B vector stores are used where rows allow); ws 256-B aligned.
 */
rf_status rf_gram_workspace_size(int64_t p, int64_t n, int64_t m_local, rf_prec prec, size_t* bytes);
rf_status rf_gram(rf_ctx* ctx, const void* X, int64_t ldx, const void* W_local, int64_t ldw,
                  int64_t p, int64_t n, int64_t m_local, int64_t m_total,
                  rf_act act, rf_prec prec, rf_out out, void* G, int64_t ldg,
                  void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------
 * rf_phi_closed_form — Φ(x_i, x_j) by EQ1 for every pair i ≤ j with i in the row range
 * [row_begin, row_end) (row_begin a multiple of 256, row_end = n or a multiple of 256; 0, n = all rows).
 *   Gram–Schmidt with x_i (the row) as pivot: u_a = ‖x_i‖, v_b = x_iᵀx_j/‖x_i‖,
 *   u_b = √max(0, ‖x_j‖² − (x_iᵀx_j)²/‖x_i‖²); diagonal: u_b = 0, v_b = u_a exactly.
 *   α = u_a/√τ − 1, β = u_b/√τ − 1, ν = v_b/√τ;  with ⟨k,d⟩ = mom->kd[k][d]
 *   Φ = A0(α)C0(β) + ν A1(α) C1(β) + (ν²/2) A2(α) ⟨0,2⟩,
 *   A_j(α) = ⟨j,0⟩ + α⟨j+1,1⟩ + (α²/2)⟨j+2,2⟩, C0(β) = ⟨0,0⟩ + β⟨1,1⟩ + (β²/2)⟨2,2⟩, C1(β) = ⟨0,1⟩ + β⟨1,2⟩
 *   (this is EQ1's 18 terms regrouped; DESIGN.md §4 lists the four corrected garbles).
 *   tau  > 0: used as given.  tau <= 0: τ̂ of Lemma 1 over ALL n rows (one stream sync).
 *   mom  != NULL: used as given (its tau must equal the τ used).  NULL: rf_moments(act, τ, 0).
 *   Phi  device, n × n (ldphi), f64 in RF_PREC_FP64 else f32.  UPPER writes j ≥ i of rows in range;
 *        FULL additionally writes the mirror Φ[j][i] = Φ[i][j] (only rows/cols the range covers).
 *   ws   ≥ rf_phi_workspace_size(p, n, prec) = rf_workspace_size(ctx, 1, p, n, 0, prec, out).
 * Pipeline: K1 row norms (fp64) [+ τ̂] → per-row coefficients → K5 fused XᵀX (tcgen05 CTA pairs,
 *           256×256 upper-triangle tiles) + EQ1 epilogue with TMA stores.
 * A zero-norm sample makes v_b undefined: with tau <= 0 (the call synchronizes anyway) it is detected →
 * RF_E_INVALID; with tau > 0 (asynchronous, no host check) a zero pivot x_i = 0 is taken as its Gram–Schmidt limit
 * (R23: v_b = 0, u_b = ‖x_j‖, diagonal u_a = v_b = u_b = 0), so every entry of Φ stays finite.
 */
rf_status rf_phi_workspace_size(int64_t p, int64_t n, rf_prec prec, size_t* bytes);
rf_status rf_phi_closed_form(rf_ctx* ctx, const void* X, int64_t ldx, int64_t p, int64_t n,
                             rf_act act, double tau, const rf_moments_t* mom,
                             rf_prec prec, rf_out out, int64_t row_begin, int64_t row_end,
                             void* Phi, int64_t ldphi, void* ws, size_t ws_bytes, void* stream);

/* rf_phi_eq2 — as rf_phi_closed_form with the six-term EQ2 instead of EQ1: the O(p^{-1}) truncation the
 * paper carries to Theorem 1 (NEXT-3):
 *   Φ2 = ⟨0,0⟩² + ⟨0,0⟩⟨1,1⟩(α + β) + ⟨1,1⟩²αβ + ⟨0,1⟩⟨1,0⟩ν + ⟨0,2⟩⟨2,0⟩ν²/2.
 * Same arguments, layouts, workspace (rf_phi_workspace_size) and errors. */
rf_status rf_phi_eq2(rf_ctx* ctx, const void* X, int64_t ldx, int64_t p, int64_t n, rf_act act, double tau,
                     const rf_moments_t* mom, rf_prec prec, rf_out out, int64_t row_begin, int64_t row_end,
                     void* Phi, int64_t ldphi, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------
 * rf_phi_row_split — row-block sharding of Φ over `world` ranks with no collective: returns the
 * range [*row_begin, *row_end) of rank `rank`, boundaries multiples of 256, balanced by upper-triangle
 * area (row i carries n − i entries).  Host only.
 */
rf_status rf_phi_row_split(int64_t n, int32_t world, int32_t rank, int64_t* row_begin, int64_t* row_end);

/* =============================================================================================
 * NEXT-2 — Theorem 1's asymptotic equivalent K̃ (EQ6):
 *   K̃ = P (d1·XᵀX + d2·V A Vᵀ + d0·I_n) P,   P = I_n − (1/n)11ᵀ,
 * for GMM data x_i = μ_a/√p + z_i (so Z + M Jᵀ/√p = X), V = [J/√p, φ] ∈ R^{n×(K+1)}, A = [[ttᵀ + 2T, t], [tᵀ, 1]]
 * (the caller forms V and A from its class statistics; d0, d1, d2 from rf_moments).  One tcgen05 pass: the XᵀX
 * mainloop of K5 with an epilogue d1·g + d2·u_iᵀv_j + d0·δ_ij − r'_i − r'_j, where u_i = A v_i and r'_i = r_i − s/2
 * come from the exact row means of the uncentred matrix (r_i = (d1·x_iᵀx̄ + d2·u_iᵀv̄ + d0)/n, s = mean r), so the
 * centring costs no extra pass over the n × n output.
 *   X   device n × p (ldx): bf16 for RF_PREC_BF16, f32 for RF_PREC_TF32 / RF_PREC_3XTF32.
 *   V   device f32 n × kv (ldv ≥ kv), 0 ≤ kv ≤ 8 (NULL if kv = 0);  A host f64 kv × kv row-major.
 *   out RF_OUT_UPPER or RF_OUT_FULL;  Kt device f32 n × n (ldk).  ws ≥ rf_ktilde_workspace_size(p, n, prec).
 * Async on `stream`. */
rf_status rf_ktilde_workspace_size(int64_t p, int64_t n, rf_prec prec, size_t* bytes);
rf_status rf_ktilde(rf_ctx* ctx, const void* X, int64_t ldx, int64_t p, int64_t n, const float* V, int64_t ldv, int32_t kv,
                    const double* A, double d0, double d1, double d2, rf_prec prec, rf_out out, float* Kt, int64_t ldk,
                    void* ws, size_t ws_bytes, void* stream);

/* =============================================================================================
 * NEXT-1 — Ternary Random Features (TRF): Eq. (3)-(5), Corollary 1 + Eq. (8),
 * Algorithm 1.  W^ter = c·T with T ∈ {−1, 0, +1} (P(0) = ε, P(±1) = (1−ε)/2) and c = (1−ε)^{-1/2};
 * σ^ter(t) = −1 if t < s−, +1 if t > s+, 0 otherwise; Σ^ter = σ^ter(W^ter X); G^ter = (1/m) Σ^terᵀ Σ^ter.
 * ============================================================================================= */

/* rf_trf_thresholds — host.  Algorithm 1 step 2: (s−, s+) whose ternary moments match Theorem 1's d1, d2
 * (P:539-541), from Eq. (5) with weak derivatives (Remark 2) — NOT Eq. (8) as printed, which contradicts Table 2's
 * sign(t) row (reading R15): E[σ^ter'] = (φ(a)+φ(b))/√τ, E[σ^ter''] = (aφ(a)+bφ(b))/τ, a = s−/√τ,
 * b = s+/√τ.  sign2 (±1) picks the sign of E[σ^ter''] (the mirror solution (−s+, −s−) has the same d1, d2).
 * Errors: tau <= 0, negative / non-finite d → RF_E_INVALID; unreachable targets (√(τd1) > 2φ(0), i.e. more than
 * sign(t), or 2τ√d2 > 2φ(1)) → RF_E_INVALID with the residual in rf_last_error(). */
rf_status rf_trf_thresholds(double d1, double d2, double tau, int32_t sign2, double* s_minus, double* s_plus);
/* The same for the d1, d2 of a north-star σ at τ (rf_moments, sign2 = sign of E[σ'']; odd σ → s− = −s+). */
rf_status rf_trf_thresholds_for(rf_act act, double tau, double* s_minus, double* s_plus);

/* rf_ter_features — Algorithm 1 step 4, features only (also the test hook for the decisions):
 *   features[i*ldf + k] = FP8 E4M3 code of σ^ter(c·x_iᵀt_k): 0x38 (+1), 0xB8 (−1), 0x00 (0).
 *   X device bf16 n × p (ldx); T device bf16 m_local × p (ldt) with entries exactly −1, 0, +1 (not checked).
 *   The projection z = x_iᵀt_k is accumulated in fp32 on the tensor cores (bf16 × {−1,0,1} products are
 *   exact) and compared with t± = s±/c rounded to fp32; an entry whose exact z lies within the fp32 rounding
 *   of z of a threshold may decide either way (the tests bound that band).
 *   features: device, 16-B aligned, ldf ≥ m_local bytes, ldf % 16 == 0.  Async on `stream`. */
rf_status rf_ter_features(rf_ctx* ctx, const void* X, int64_t ldx, const void* T, int64_t ldt, int64_t p, int64_t n,
                          int64_t m_local, double eps, double s_minus, double s_plus, void* features, int64_t ldf,
                          void* stream);
/* rf_gram_ter — G^ter = (1/m_total) Σ^terᵀ Σ^ter over this rank's m_local features (UPPER / FULL like rf_gram).
 * Pipeline: K3^ter (bf16 tcgen05 GEMM X·Tᵀ, σ^ter in the epilogue → fp8 codes, 1 byte per feature instead of the
 * paper's 32 bits) → K4^ter (fp8 kind::f8f6f4 SYRK, 256×512 CTA-pair tiles, soft lockstep): the ±1
 * products and their sums are exact in fp32 (m_local ≤ 2^24), so m_total·G^ter is an exact integer count of the
 * decided features.  ws ≥ rf_gram_ter_workspace_size(p, n, m_local). */
rf_status rf_gram_ter_workspace_size(int64_t p, int64_t n, int64_t m_local, size_t* bytes);
rf_status rf_gram_ter(rf_ctx* ctx, const void* X, int64_t ldx, const void* T, int64_t ldt, int64_t p, int64_t n, int64_t m_local,
                      int64_t m_total, double eps, double s_minus, double s_plus, rf_out out, float* G, int64_t ldg,
                      void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------
 * TEST HOOK (not a step of the method): C = A·Bᵀ on the same tcgen05 mainloop the G/Φ kernels use,
 * raw fp32 accumulator, rectangular pair tiles (256 × 256).  A: M × K (lda), B: N × K (ldb), dtype per
 * prec ∈ {BF16 (bf16 inputs), TF32, 3XTF32 (f32 inputs)}; C: M × N fp32 (ldc).  kchunk > 0 cuts the K
 * reduction into chunks of kchunk K-blocks (64 bf16 / 32 fp32 elements each) whose partial sums are added
 * in fp32 in the epilogue; 0 = one chunk.  ws ≥ rf_debug_gemm_workspace_size() (3XTF32 split operands).
 */
rf_status rf_debug_gemm_workspace_size(int64_t M, int64_t N, int64_t K, rf_prec prec, size_t* bytes);
rf_status rf_debug_gemm_nt(rf_ctx* ctx, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                           rf_prec prec, int32_t kchunk, float* C, int64_t ldc, void* ws, size_t ws_bytes,
                           void* stream);

/* ---------------------------------------------------------------------------------------------
 * NEXT-4: random-features kernel ridge regression on G (the paper's downstream use of G: Section 5 P:757-761,
 * App. A; the estimator is the textbook one, R20).  For each γ in gammas:
 *     α_γ = (G_train + γ·I)^{-1} Y        (fp64 blocked Cholesky of G_train + γI, then two triangular solves)
 *     Ŷ_γ = G_cross · α_γ                 (G_cross[t][i] = the Gram of test sample t and training sample i)
 * G_train and G_cross are read from ONE Gram over the stacked samples [X_train; X_test] (n_all = n_train + n_test
 * rows), as rf_gram / rf_gram_ter write it: only entries j ≥ i are read (UPPER or FULL layout, ld = ldg ≥ n_all).
 *   G       device f32, n_all × n_all (ldg), 4-B aligned
 *   gammas  HOST, n_gamma values, each finite and > 0
 *   Y       device f64, n_train × nrhs row-major (ldy ≥ nrhs): the training targets
 *   alpha   device f64, n_gamma blocks of n_train × nrhs (row-major, ld nrhs), block g for gammas[g]
 *   Yhat    device f64, n_gamma blocks of n_test × nrhs (ld nrhs); may be NULL when n_test = 0
 *   ws      ≥ rf_ridge_workspace_size(n_train) bytes, 256-B aligned (one fp64 factor and its diagonal-block
 *           inverses); a workspace of 256 + k·(rf_ridge_workspace_size(n_train) − 256) bytes lets k ≤ 16 γ values
 *           be factored concurrently (one set of launches per batch)
 * Synchronous at the end (one event wait, through mapped host memory) to report the factorisation:
 * G_train + γI not positive definite (a non-positive pivot) → RF_E_NONFINITE. */
rf_status rf_ridge_workspace_size(int64_t n_train, size_t* bytes);
rf_status rf_ridge(rf_ctx* ctx, const float* G, int64_t ldg, int64_t n_train, int64_t n_test, const double* gammas,
                   int32_t n_gamma, const double* Y, int64_t ldy, int32_t nrhs, double* alpha, double* Yhat,
                   void* ws, size_t ws_bytes, void* stream);

/* Number of kernel launches the last successful rf_gram / rf_phi_closed_form call on this thread
 * enqueued (for bench accounting). */
int32_t rf_last_launch_count(void);

/* Launch tracing.  rf_profile_enable(1): from now on every kernel launch of this library is bracketed by
 * two CUDA events recorded on the launching stream (negligible cost; process-wide switch).
 * rf_profile_read: waits for the recorded events, writes up to max_records entries — names[32*k] is a
 * NUL-terminated kernel name (e.g. "K4_syrk"), ms[k] its device duration — sets *count to the number of
 * records taken (may exceed max_records; the excess is dropped) and clears the record list. */
rf_status rf_profile_enable(int on);
rf_status rf_profile_read(int32_t max_records, char* names, float* ms, int32_t* count);
/* rf_profile_timeline: as rf_profile_read, plus start_ms[k] = the launch's start relative to the earliest recorded
 * start (records on several streams — a collective's flag / sum kernels beside K4 — on one device time line). */
rf_status rf_profile_timeline(int32_t max_records, char* names, float* start_ms, float* ms, int32_t* count);

#ifdef __cplusplus
}
#endif
#endif /* RF_B200_H */
