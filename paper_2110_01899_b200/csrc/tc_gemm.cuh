// Warp-specialised persistent tcgen05 GEMM for sm_100a on CTA PAIRS (cta_group::2), shared by the three
// tensor-core kernels of the path:
//   K3  Σᵀ = σ(X·Wᵀ)          rectangular pair tiles, σ in the epilogue          (Σ = σ(WX))
//   K4  G  = ΣᵀΣ / m          upper-triangular pair tiles, scale in the epilogue (Eq. def_Gram)
//   K5  Φ  = EQ1(XᵀX, …)      upper-triangular pair tiles, EQ1 in the epilogue
// D[i][j] = Σ_k A[i][k]·B[j][k]; A (rows i) and B (rows j) are both K-major in HBM, so
// both UMMA operands are K-major 128-B-swizzled smem tiles written by TMA.
//
// Pair tile 256 (M) × BN (N = 256 or 512).  CTA r of the pair loads A rows [M0+128r, +128) and, for each
// 256-wide N sub-tile s, B rows [N0+256s+128r, +128); the leader (r = 0) issues
// tcgen05.mma.cta_group::2 (M = 256, N = 256) per sub-tile and K-step; CTA r's TMEM receives rows
// M0+128r.. of the accumulator.  Per SM this moves (16 + 16·BN/256) KB of operands per
// 256·BN·64 MACs — half (BN=256) or a third (BN=512) of the 1-CTA 128×256 tile's L2 traffic per flop.
// K-block = one 128-byte swizzle row (64 bf16 / 32 fp32).
//
// Warp roles (128 + 32·kEpiW threads per CTA): w0 TMA producer, w1 MMA issuer (leader CTA, one thread), w2 TMEM
// allocator, w3 column-vector loader (kColVec epilogues; else idle), w4.. epilogue (warp w: TMEM lane quarter w%4; with 8 epilogue warps column half (w-4)/4,
// with 12 / 16 the 32-column chunks ≡ (w-4)/4 mod 3 / 4).
// Pipelines: smem ring (full barrier in the leader, empty barriers in both CTAs) TMA→MMA; TMEM
// accumulator slots (2 × 256 columns for BN = 256, 1 × 512 for BN = 512) MMA→epilogue.
//
// K-chunked accumulation (kchunk k-blocks): the K range of a tile is cut into chunks whose partial sums
// start from zero in TMEM slot 0 and are added in fp32 (round-to-nearest) into a running sum in TMEM slot 1
// by the epilogue warps; the functor sees the final sum once.  The tensor pipe's
// accumulation into TMEM loses up to ~2^-23 relative per MMA (measured: 3×TF32 SYRK error grows
// linearly with K), so long-K fp32-accurate results need short chunks.
// 3×TF32 (kSplit = 3): each stage holds A_hi, A_lo, B_hi, B_lo; per K-step three MMAs lo·hi, hi·lo,
// hi·hi accumulate into the same accumulator (small terms first).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <type_traits>

#include "ptx_sm100.cuh"
#include "rf_common.cuh"

namespace rfk {

// kStg: 4-KB TMA-store staging buffers per epilogue warp (-1 = default: 1 if stages are large, else 2;
// 0 for epilogues that store directly from registers, e.g. K3).
// kCl: CTAs per cluster.  2 = one CTA pair per cluster.  4 = two pairs computing vertically adjacent tiles
// (row tiles 2I, 2I+1, same column tile).  BN = 256: each CTA loads one 64-row half of its rank's B rows (through
// the 64-row-box map passed as tmB_lo) and multicasts it to the same rank of both pairs.  BN = 512: each CTA
// loads its own A half and ONE of the NSUB B sub-tiles for its
// rank-in-pair and TMA-multicasts it to the same rank of both pairs, so a B sub-tile leaves L2 once per cluster
// instead of once per pair (a third less L2 → SM traffic per flop for BN = 512, a quarter for BN = 256).
// Requires kSplit == 1.
// kAres: A-panel residency (K5 with K ≤ 8 K-blocks): each CTA keeps its 128 A rows over the whole K in shared memory
// for a run of column tiles of the same row tile (segment schedule, Sched::seg_len), so only B streams per tile.
template <int kFmt /*1 = bf16 (kind::f16), 2 = tf32, 3 = fp8 e4m3 (kind::f8f6f4)*/, int kSplit /*1 or 3*/,
          int kBN /*256 or 512*/, int kStg = -1, int kCl = 2, int kEpiW = 8, int kAres = 0>
struct TcCfg {
  static constexpr int CL = kCl;
  static constexpr bool ARES = kAres != 0;
  static_assert(!kAres || (kSplit == 1 && kCl == 2 && kBN == 256), "A residency: one operand split, pairs, BN 256");
  static_assert(kCl == 2 || (kCl == 4 && kSplit == 1) || (kCl == 8 && kSplit == 1 && kBN == 512),
                "4-CTA clusters: one operand split; 8-CTA clusters: BN = 512");
  static constexpr int BM = 256, BN = kBN;      // pair tile
  static constexpr int NSUB = kBN / 256;        // N=256 MMAs per K-step
  static constexpr int ESZ = kFmt == 1 ? 2 : (kFmt == 3 ? 1 : 4);
  static constexpr int BK = 128 / ESZ;          // elements per K-block (one 128-B swizzle row)
  static constexpr int UK = 32 / ESZ;           // K per tcgen05.mma (16 bf16 / 8 tf32 / 32 fp8) = 32 bytes
  static constexpr int NOPS = kSplit == 3 ? 2 : 1;
  static constexpr int A_BYTES = 128 * 128;     // per CTA: 128 rows × 128 B
  static constexpr int B_BYTES = 128 * 128;     // per CTA per N sub-tile
  static constexpr int ARES_KB = 8;              // resident K-blocks (K ≤ 512 bf16)
  static constexpr int ARES_BYTES = kAres ? ARES_KB * A_BYTES : 0;
  static constexpr int STAGE_BYTES = NOPS * ((kAres ? 0 : A_BYTES) + NSUB * B_BYTES);
  static constexpr int ACC_COLS = kBN;
  static constexpr int ACC_SLOTS = 512 / kBN;
  // 8 epilogue warps (two per TMEM lane quarter, each owning half of the accumulator columns), or 12 / 16 (three /
  // four per quarter, 32-column chunks dealt round-robin; unpipelined TMEM loads to fit 128 / 96 registers)
  static constexpr int EPI_WARPS = kEpiW;
  static_assert(kEpiW == 8 || kEpiW == 12 || kEpiW == 16, "8, 12 or 16 epilogue warps");
  static constexpr int THREADS = 128 + 32 * kEpiW;
  static constexpr int STG_BUFS = kStg >= 0 ? kStg : ((kSplit == 3 || kBN == 512) ? 1 : 2);   // per epi warp
  // 16 epilogue warps with A residency: 2-KB staging buffers (32 × 16 boxes, 64-B swizzle) keep four B stages
  static constexpr bool HALF_STG = kAres && kEpiW == 16;
  static constexpr int STG_BUF_BYTES = HALF_STG ? 2048 : 4096;
  static constexpr int STG_BYTES = EPI_WARPS * STG_BUFS * STG_BUF_BYTES;
  // per-column vector of the tile (epilogues with kColVec, e.g. ‖x_j‖²/τ of K5), double-buffered with the accumulator
  static constexpr int COL_BYTES = kBN == 256 ? 2 * 256 * 4 : 0;
  static constexpr int BAR_BYTES = 512;             // mbarriers, the TMEM address word, the unit ring
  static constexpr int SMEM_MAX = 227 * 1024;       // opt-in dynamic shared memory per CTA
  static constexpr int FIXED = ARES_BYTES + STG_BYTES + COL_BYTES + BAR_BYTES;
  static constexpr int STAGES = (SMEM_MAX - FIXED) / STAGE_BYTES;
  // room left to align the dynamic window to 1024 B (the base is 1024-aligned in practice: the kernel checks)
  static constexpr int SLACK = SMEM_MAX - STAGES * STAGE_BYTES - FIXED < 1024 ? SMEM_MAX - STAGES * STAGE_BYTES - FIXED
                                                                              : 1024;
  static constexpr size_t SMEM_BYTES = (size_t)SLACK + (size_t)STAGES * STAGE_BYTES + FIXED;
  static_assert(8 * (2 * STAGES + 6 + 2 * 4 + 2) + 4 + 4 * 4 <= BAR_BYTES, "barrier area");
  static constexpr uint32_t IDESC = ptx::idesc_f32acc(kFmt == 3 ? 0u : (uint32_t)kFmt, 256, 256);
  static_assert(STAGES >= 2, "pipeline too shallow");
  static_assert(SMEM_BYTES <= 227 * 1024, "smem budget");
};

// Epilogues that read a per-column vector (one float per accumulator column, e.g. K5's ‖x_j‖²/τ) declare
// kColVec = 1 and `col_src` (global, padded to whole tiles): the TMA producer of each CTA bulk-copies the tile's slice
// into shared memory (double-buffered like the accumulator) when the tile starts, so the epilogue reads it with
// LDS.128 broadcasts instead of waiting on a global load per 32-column chunk.
template <class E, class = void>
struct ColVecOf {
  static constexpr bool value = false;
};
template <class E>
struct ColVecOf<E, decltype(void(E::kColVec))> {
  static constexpr bool value = E::kColVec != 0;
};
// Epilogues with an interior fast path declare kFast = 1 and provide fast_tile(ti, tj) (every chunk of the tile is
// needed, off the diagonal band and stored whole by TMA) and fast<kSlot>(…): the kernel's 8-warp loop then runs the
// tile with no per-chunk predicates and a static staging-batch slot (chunk cc goes to buffer cc & 1).
template <class E, class = void>
struct FastOf {
  static constexpr bool value = false;
};
template <class E>
struct FastOf<E, decltype(void(E::kFast))> {
  static constexpr bool value = E::kFast != 0;
};

// Pair-tile scheduler.  Rows of 256, columns of BN.  Rectangular: row tiles [row_tile0, row_tile1) × all
// column tiles.  Triangular: row tile I needs the column tiles J ≥ floor(256 I / BN) (every tile holding
// an entry j ≥ i).  Work item = (tile, K-chunk); a cluster processes all chunks of a tile in order.
//
// L2-aware order: row tiles are taken in groups of `gm`; inside a group the walk is column-major (down
// the gm rows, then the next column), so the ~74 tiles in flight at once cover gm row panels × ~74/gm
// column panels instead of 1 × 74.  Measured on configs[3] (K4): the row-major walk re-read Σᵀ ≈ 155×
// from DRAM (1.33 TB per launch); grouping bounds the re-reads to one pass of the column panels per
// group (and all clusters advance through K in near lockstep, so only K-slices need to stay in L2).
struct Sched {
  int tri;
  int shift;            // log2(BN/256)
  int tiles_n;
  int row_tile0, row_tile1;
  int num_tiles;
  int num_kb;           // K-blocks of the whole reduction
  int kchunk;           // K-blocks per chunk
  int nchunks;
  int gm;               // row tiles per raster group
  // Soft lockstep (K4): every `lock_ks` K-blocks the leader CTA's producer publishes its cluster's
  // K-block count in prog[cluster] and waits (bounded, ≤ 50 µs per check) until the slowest cluster is
  // within `lock_w` K-blocks.  Tiles of one raster wave share Σᵀ panels, but a K-block row slice stays in
  // L2 only ~25 µs at the kernel's fill rate; unsynchronised clusters drift further apart than that and
  // re-read the shared panels from DRAM (measured: 1.16 TB of DRAM reads per configs[3] launch for 8.6 GB
  // of Σᵀ).  prog == nullptr disables it.  The wait is bounded, so co-residency of all clusters is not
  // required for progress.
  uint32_t* prog;
  int lock_w, lock_ks;
  // L2 policies: operand loads (0 = evict_normal, 1 = evict_last: operands re-read by many tiles, e.g. X in
  // K5) and epilogue TMA stores (0 = normal, 1 = evict_first: a streamed output must not evict them).
  int load_pol, store_pol;
  uint32_t* started;    // non-null: the first CTA writes 1 here when the kernel starts (hybrid K4 launch order)
  // Dynamic units (TileSeq): queue != nullptr → the cluster pulls work items ("units" = tiles of this schedule) from
  // the counter *queue, shared with the other kernel of a hybrid launch; a 2-CTA-cluster kernel processes a unit as
  // nsub row tiles (2I, 2I + 1; rows ≥ sub_rows skipped), a 4-CTA-cluster kernel as one row tile per pair (2I + pi).
  uint32_t* queue;
  int nsub, sub_rows;
  // Segment schedule (A residency, seg_len > 0): work item = segment (row tile I, column tiles [J0, J1)), column-block
  // major: for column block b (tiles [b·L, (b+1)·L) ∩ [0, T)) every row tile I ∈ [row_tile0, min(row_tile1, (b+1)L, T))
  // in order, J0 = max(b·L, I).  Concurrent segments share the block's B panels; a cluster reloads A once per segment.
  int seg_len;
  __host__ __device__ __forceinline__ long long seg_rows(int b) const {   // segments of column block b
    const int hi = min(min(row_tile1, (b + 1) * seg_len), tiles_n);
    return hi > row_tile0 ? hi - row_tile0 : 0;
  }
  __host__ __device__ __forceinline__ long long seg_prefix(int b) const {   // segments of blocks [0, b)
    // blocks whose row bound is (b'+1)L (before the bound saturates at U = min(row_tile1, T)) contribute an
    // arithmetic series, the rest U − row_tile0 each
    const long long U = min(row_tile1, tiles_n), L = seg_len, r0 = row_tile0;
    const long long bsat = U / L;               // blocks b' < bsat have (b'+1)L ≤ U
    long long tot = 0;
    const long long b1 = b < bsat ? b : bsat;
    long long blo = r0 / L;                     // first block with (b'+1)L > r0
    if (blo < b1) {                             // Σ_{b'=blo}^{b1−1} ((b'+1)L − r0)
      const long long cnt = b1 - blo;
      tot += L * ((blo + 1 + b1) * cnt / 2) - r0 * cnt;
    }
    if (b > bsat && U > r0) tot += (long long)(b - bsat) * (U - r0);
    return tot;
  }
  __host__ __device__ __forceinline__ void seg_get(long long sidx, int& I, int& J0, int& J1) const {
    const int nb = (tiles_n + seg_len - 1) / seg_len;
    int lo = 0, hi = nb;                        // largest b with seg_prefix(b) ≤ sidx
    while (hi - lo > 1) {
      const int mid = (lo + hi) / 2;
      if (seg_prefix(mid) <= sidx) lo = mid; else hi = mid;
    }
    I = row_tile0 + (int)(sidx - seg_prefix(lo));
    J0 = max(lo * seg_len, I);
    J1 = min((lo + 1) * seg_len, tiles_n);
  }

  struct Group {
    int I0, I1, J0, Jf;
    long long P, cnt;
  };
  __host__ __device__ __forceinline__ Group group(int I0) const {
    Group g;
    g.I0 = I0;
    g.I1 = I0 + gm < row_tile1 ? I0 + gm : row_tile1;
    const long long rows = g.I1 - g.I0;
    if (!tri) {
      g.J0 = g.Jf = 0;
      g.P = 0;
      g.cnt = rows * tiles_n;
      return g;
    }
    g.J0 = I0 >> shift;
    const int jf = (g.I1 - 1) >> shift;     // first column where every row of the group is needed
    g.Jf = jf < tiles_n ? jf : tiles_n;
    const long long a = g.J0, b = g.Jf;
    g.P = ((b * (b + 1) - a * (a + 1)) / 2 << shift) - (b - a) * (long long)I0;   // partial columns [J0, Jf)
    g.cnt = g.P + (tiles_n - g.Jf) * rows;
    return g;
  }
  // tile (ti, tj) of index u inside group g
  __host__ __device__ __forceinline__ void in_group(const Group& g, long long u, int& ti, int& tj) const {
    if (u < g.P) {
      int J = g.J0;
      for (;;) {
        const long long rv = ((long long)(J + 1) << shift) - g.I0;
        if (u < rv) break;
        u -= rv;
        ++J;
      }
      ti = g.I0 + (int)u;
      tj = J;
      return;
    }
    u -= g.P;
    const int rows = g.I1 - g.I0;
    tj = g.Jf + (int)(u / rows);
    ti = g.I0 + (int)(u % rows);
  }
  static Sched make(int tri, int bn, int row_tile0, int row_tile1, int tiles_n, int num_kb, int kchunk, int gm = 8) {
    Sched s;
    s.tri = tri;
    s.shift = bn == 512 ? 1 : 0;
    s.tiles_n = tiles_n;
    s.row_tile0 = row_tile0;
    s.row_tile1 = row_tile1;
    s.num_kb = num_kb;
    s.kchunk = (kchunk <= 0 || kchunk > num_kb) ? (num_kb > 0 ? num_kb : 1) : kchunk;
    s.nchunks = num_kb > 0 ? (num_kb + s.kchunk - 1) / s.kchunk : 1;
    s.gm = gm > 0 ? gm : 1;
    s.prog = nullptr;
    s.lock_w = 0;
    s.lock_ks = 8;
    s.load_pol = 0;
    s.store_pol = 0;
    s.started = nullptr;
    s.queue = nullptr;
    s.nsub = 1;
    s.sub_rows = 0;
    s.seg_len = 0;
    long long tot = 0;
    for (int I0 = row_tile0; I0 < row_tile1; I0 += s.gm) tot += s.group(I0).cnt;
    s.num_tiles = (int)tot;
    return s;
  }
};

// Monotone cursor over the tile order (each cluster visits t = cid, cid + ncl, … in increasing order, so
// advancing group by group is amortised O(1)).  The group is held in scalar registers (a struct passed by reference
// was placed in local memory: 8 STL + 8 LDL per tile and warp).
struct TileCursor {
  const Sched* s;
  int I0, I1, J0, Jf;
  long long P, cnt, base;
  __device__ __forceinline__ void load(int i0) {
    const Sched::Group g = s->group(i0);
    I0 = g.I0; I1 = g.I1; J0 = g.J0; Jf = g.Jf; P = g.P; cnt = g.cnt;
  }
  __device__ __forceinline__ void init(const Sched* sp) {
    s = sp;
    base = 0;
    load(s->row_tile0);
  }
  __device__ __forceinline__ void get(long long t, int& ti, int& tj) {
    while (t >= base + cnt) {
      base += cnt;
      load(I1);
    }
    long long u = t - base;
    if (u < P) {   // partial columns [J0, Jf): column J holds rows I0 .. min(I1, (J + 1)·2^shift) − 1
      int J = J0;
      for (;;) {
        const long long rv = ((long long)(J + 1) << s->shift) - I0;
        if (u < rv) break;
        u -= rv;
        ++J;
      }
      ti = I0 + (int)u;
      tj = J;
      return;
    }
    u -= P;
    const int rows = I1 - I0;
    tj = Jf + (int)(u / rows);
    ti = I0 + (int)(u % rows);
  }
};

// Tile sequence of one warp role of a cluster (every role walks the same sequence).  Static: tiles t = cid, cid + ncl, …
// of the schedule.  Dynamic (sched.queue): the cluster's fetcher — the producer warp of cluster rank 0 — takes the next
// unit with an atomicAdd on the counter every cluster of the launch shares (both kernels of the K4 hybrid), writes it
// into a kRing-deep ring in every CTA of the cluster (st.shared::cluster) and arrives (release, cluster scope) on
// that CTA's ring_full; every other role waits there (acquire), reads the unit and arrives on the fetcher's
// ring_empty, which the fetcher waits on before it reuses the slot.  A unit past the end is published as ~0u (stop).
constexpr int kRing = 4;
struct TileSeq {
  const Sched* s;
  TileCursor cur;
  long long t;
  int ncl, cl, pi;
  bool dyn, fetcher;
  uint32_t lane, ring_s, rfull_s, rempty_s, rempty_c;
  int k, sub, nsub, ui, uj;
  long long u;
  int sI, sJ, sJ1;       // segment mode: current segment and next column tile
  bool seg_first;        // the tile just returned starts a segment (a new A panel)
  __device__ __forceinline__ void init(const Sched* sp, int cid, int ncl_, int cl_, int pi_, bool fetcher_,
                                       uint32_t lane_, uint32_t ring_s_, uint32_t rfull_s_, uint32_t rempty_s_,
                                       uint32_t rempty_c_) {
    s = sp;
    cur.init(sp);
    t = cid;
    ncl = ncl_;
    cl = cl_;
    pi = pi_;
    dyn = sp->queue != nullptr;
    fetcher = fetcher_;
    lane = lane_;
    ring_s = ring_s_;
    rfull_s = rfull_s_;
    rempty_s = rempty_s_;
    rempty_c = rempty_c_;
    k = 0;
    nsub = cl_ == 2 ? sp->nsub : 1;
    sub = nsub;
    ui = uj = 0;
    u = 0;
    sI = sJ = sJ1 = 0;
    seg_first = false;
  }
  __device__ __forceinline__ long long fetch() {
    const int slot = k % kRing;
    const uint32_t par = (uint32_t)(k / kRing) & 1u;
    ++k;
    uint32_t v = 0;
    if (fetcher) {
      if (lane == 0) {
        ptx::mbar_wait_cluster(rempty_s + 8 * slot, par ^ 1u);
        v = atomicAdd(s->queue, 1u);
        if (v >= (uint32_t)s->num_tiles) v = 0xFFFFFFFFu;
        for (int r = 0; r < cl; ++r) {
          ptx::st_shared_cluster_u32(ptx::mapa(ring_s + 4 * slot, (uint32_t)r), v);
          ptx::mbar_arrive_release_cluster(ptx::mapa(rfull_s + 8 * slot, (uint32_t)r));
        }
      }
      v = __shfl_sync(0xFFFFFFFFu, v, 0);
    } else {
      ptx::mbar_wait_cluster(rfull_s + 8 * slot, par);
      v = ptx::ld_shared_u32(ring_s + 4 * slot);
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_release_cluster(rempty_c + 8 * slot);
    }
    return v == 0xFFFFFFFFu ? -1 : (long long)v;
  }
  // next tile of this role: (schedule index / unit, row tile, column tile) with the cluster's CTA placement applied.
  // kDyn = false (every kernel but the K4 hybrid's and the A-resident K5): the static walk only, so the ring state
  // costs no registers.
  template <bool kDyn, bool kSeg = false>
  __device__ __forceinline__ bool next(long long& tt, int& ti, int& tj) {
    if (kSeg) {               // segment schedule (A residency configurations only)
      seg_first = false;
      if (sJ >= sJ1) {
        if (kDyn && dyn) {    // dynamic: the next segment from the shared counter (keeps the last wave balanced)
          u = fetch();
          if (u < 0) return false;
        } else {
          if (t >= s->num_tiles) return false;
          u = t;
          t += ncl;
        }
        s->seg_get(u, sI, sJ, sJ1);
        seg_first = true;
      }
      tt = u;
      ti = sI;
      tj = sJ++;
      return true;
    }
    if (!kDyn || !dyn) {
      if (t >= s->num_tiles) return false;
      cur.get(t, ti, tj);
      tt = t;
      t += ncl;
      if (cl == 4) ti = 2 * ti + pi;       // 4-CTA clusters walk 512-row super tiles
      if (cl == 8) {                       // … 8-CTA clusters also 1024-column super tiles
        ti = 2 * ti + (pi & 1);
        tj = 2 * tj + (pi >> 1);
      }
      return true;
    }
    for (;;) {
      if (sub >= nsub) {
        u = fetch();
        if (u < 0) return false;
        cur.get(u, ui, uj);
        sub = 0;
      }
      const int row = 2 * ui + (cl == 4 ? pi : sub);
      ++sub;
      if (cl == 2 && row >= s->sub_rows) continue;   // the odd last super row has one row tile
      tt = u;
      ti = row;
      tj = uj;
      return true;
    }
  }
};

// ------------------------------------------------------------------------------------------
// Epilogue store helpers.  A warp owns 32 rows (lanes) × 32 columns per call.
// ------------------------------------------------------------------------------------------
template <int kBufs, bool kHalf = false>
struct EpiCtx {
  const CUtensorMap* tm;   // fp32 output map: box 32 × 32, 128-B swizzle, bounds = the n×n matrix
  uint8_t* sbuf;           // this warp's staging buffers (kBufs × 4 KB, 1024-B aligned)
  uint32_t sbuf_s;         // … as a 32-bit shared address (STS, never a generic store)
  uint32_t col_s;          // kColVec epilogues: shared address of the current tile's column vector
  int cur;
  uint32_t lane;
  int hint;                // 1: stores carry the L2 evict_first hint `pol`
  uint64_t pol;

  // Whole 32×32 block → smem (128-B swizzle: 16-B chunk c of row r at chunk c ^ (r & 7), conflict-free)
  // → TMA store (rows/cols beyond the matrix are clipped by the tensor map).  With two staging buffers the
  // blocks are batched in pairs: both are staged, then ONE proxy fence and two TMA stores (the fence waits for
  // the warp's shared stores; one per block cost ≈ 10 % of a store-bound epilogue, scripts/store_probe.cu).
  int nst;                 // blocks staged in the open batch (kBufs == 2)
  int32_t pc0, pr0;        // coordinates of the first staged block
  __device__ __forceinline__ void issue(const uint8_t* b, int32_t c0, int32_t r0) {
    if (hint)
      ptx::tma_store_2d_hint(tm, b, c0, r0, pol);
    else
      ptx::tma_store_2d(tm, b, c0, r0);
  }
  // stg_x = sbuf_s + 128·lane with the lane's 128-B-swizzle XOR folded in: chunk c of the lane's row sits at
  // stg_x ^ (c << 4) (bits 4..6 of sbuf_s + 128·lane are zero: 1024-B aligned buffers), buffer b at + 4096·b.
  uint32_t stg_x;
  __device__ __forceinline__ void set_stg_x() { stg_x = (sbuf_s + lane * 128) | ((lane & 7) << 4); }
  template <int kOff>
  __device__ __forceinline__ void stage_x(const float (&v)[32]) {
#pragma unroll
    for (int c = 0; c < 8; ++c) ptx::sts128((stg_x ^ (c << 4)) + kOff, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  }
  // Interior tiles: with two buffers the warp's chunks pair up as (even, odd) = (buffer 0, buffer 1) of one batch
  // (the odd chunk's block is 32 columns right of the even one's, so the batch needs no saved coordinates).
  template <int kSlot>
  __device__ __forceinline__ void store_static(int32_t r0, int32_t c0, const float (&v)[32]) {
    static_assert(kBufs == 1 || kBufs == 2, "one or two 4-KB staging buffers");
    if constexpr (kBufs == 1) {   // one buffer: wait until the previous block has been read out, stage, store
      if (lane == 0) ptx::bulk_wait_read<0>();
      __syncwarp();
      stage_x<0>(v);
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        issue(sbuf, c0, r0);
        ptx::bulk_commit();
      }
    } else if constexpr (kSlot == 0) {
      if (lane == 0) ptx::bulk_wait_read<0>();
      __syncwarp();
      stage_x<0>(v);
    } else {
      stage_x<4096>(v);
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        issue(sbuf, c0 - 32, r0);
        issue(sbuf + 4096, c0, r0);
        ptx::bulk_commit();
      }
    }
  }
  __device__ __forceinline__ void stage(uint32_t b, const float (&v)[32]) {
    const uint32_t row = b + lane * 128;
#pragma unroll
    for (int c = 0; c < 8; ++c) ptx::sts128(row + ((c ^ (lane & 7)) << 4), v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  }
  // kHalf: one 2-KB buffer per warp, the block goes out as two 32-row × 16-column boxes (64-B swizzle: 16-B chunk c of
  // row r at c ^ ((r >> 1) & 3), conflict-free for the 8-lane phases of STS.128); the second half waits until the
  // first has been read out of shared memory.
  __device__ __forceinline__ void stage_half(uint32_t b, const float (&v)[32], int hf) {
    const uint32_t row = b + lane * 64;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int q = 4 * hf + c;
      ptx::sts128(row + ((c ^ ((lane >> 1) & 3)) << 4), v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  }
  __device__ __forceinline__ void store_block(int64_t row_lo, int64_t col0, const float (&v)[32]) {
    static_assert(kBufs >= 1, "store_block needs staging buffers");
    if constexpr (kHalf) {
      static_assert(kBufs == 1, "half-width staging: one buffer per warp");
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        if (lane == 0) ptx::bulk_wait_read<0>();
        __syncwarp();
        stage_half(sbuf_s, v, hf);
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          issue(sbuf, (int32_t)col0 + 16 * hf, (int32_t)row_lo);
          ptx::bulk_commit();
        }
      }
      return;
    }
    if (kBufs == 2) {
      if (nst == 0) {
        if (lane == 0) ptx::bulk_wait_read<0>();       // the previous batch has been read out of smem
        __syncwarp();
        stage(sbuf_s, v);
        pc0 = (int32_t)col0;
        pr0 = (int32_t)row_lo;
        nst = 1;
      } else {
        stage(sbuf_s + 4096, v);
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          issue(sbuf, pc0, pr0);
          issue(sbuf + 4096, (int32_t)col0, (int32_t)row_lo);
          ptx::bulk_commit();
        }
        nst = 0;
      }
      return;
    }
    uint8_t* b = sbuf + cur * 4096;
    if (lane == 0) ptx::bulk_wait_read<kBufs - 1>();
    __syncwarp();
    stage(sbuf_s + cur * 4096, v);
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      issue(b, (int32_t)col0, (int32_t)row_lo);
      ptx::bulk_commit();
    }
    cur = (cur + 1 == kBufs) ? 0 : cur + 1;
  }
  // Issue a half-filled batch (end of a tile).
  __device__ __forceinline__ void flush() {
    if (kBufs == 2 && nst == 1) {
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        issue(sbuf, pc0, pr0);
        ptx::bulk_commit();
      }
      nst = 0;
    }
  }
};

// Direct masked stores of row `row`, columns [col0, col0+32) ∩ [lo, n) into a row-major fp32 matrix.
__device__ __forceinline__ void store_row_masked(float* M, int64_t ld, int64_t n, int64_t row, int64_t col0, int64_t lo,
                                                 const float (&v)[32]) {
  RF_DCHECK(row >= 0 && col0 >= 0 && col0 < n && ld >= n, "row %lld col0 %lld n %lld ld %lld", (long long)row,
            (long long)col0, (long long)n, (long long)ld);   // n: the column bound (rows are bounded by the caller)
  float* dst = M + row * ld + col0;
  if (col0 >= lo && col0 + 32 <= n && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      reinterpret_cast<float4*>(dst)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  } else {
#pragma unroll
    for (int e = 0; e < 32; ++e)
      if (col0 + e >= lo && col0 + e < n) dst[e] = v[e];
  }
}
// Mirror (FULL output): M[j][row] = v[j - col0] for j > row; for fixed e the 32 lanes write 32
// consecutive floats of row col0+e (coalesced).
__device__ __forceinline__ void store_mirror(float* M, int64_t ld, int64_t n, int64_t row, int64_t col0,
                                             const float (&v)[32]) {
  if (row >= n) return;
#pragma unroll
  for (int e = 0; e < 32; ++e)
    if (col0 + e > row && col0 + e < n) M[(col0 + e) * ld + row] = v[e];
}

// RF_OUT_PACKED_TRI (include/rf.h): 256×256 tile (I, J ≥ I) of the T × T tile grid stored contiguously at tile
// index I·T − I(I−1)/2 + (J − I), row-major inside the tile.  The TMA map of such a buffer is (tiles·256) × 256.
__device__ __forceinline__ int64_t tri_tile_index(int64_t I, int64_t J, int64_t T) {
  return I * T - I * (I - 1) / 2 + (J - I);
}
template <class Ctx>
__device__ __forceinline__ void tri_store(Ctx& cx, float* P, int64_t n, int64_t T, int use_tma, int64_t row_lo,
                                          int64_t col0, const float (&v)[32]) {
  const int64_t ti = row_lo >> 8, tj = col0 >> 8;
  const int64_t u = tri_tile_index(ti, tj, T);
  RF_DCHECK(tj >= ti && tj < T && u < T * (T + 1) / 2, "packed tile (%lld, %lld) of T %lld", (long long)ti, (long long)tj,
            (long long)T);
  const int64_t lr = row_lo & 255, lc = col0 & 255;
  if (use_tma && col0 >= row_lo + 31) {
    cx.store_block(u * 256 + lr, lc, v);
    return;
  }
  if (row_lo + cx.lane >= n) return;
  const int64_t nloc = n - (tj << 8) < 256 ? n - (tj << 8) : 256;
  const int64_t lo = tj == ti ? lr + cx.lane : 0;                 // j ≥ i inside a diagonal tile
  store_row_masked(P + u * 65536, 256, nloc, lr + cx.lane, lc, lo, v);
}

// ------------------------------------------------------------------------------------------
// Epilogue functors: operator()(ctx, row_lo, col0, r[32], chunk, nchunks, t) for the warp's rows
// [row_lo, row_lo+32) (row = row_lo + lane) and accumulator columns [col0, col0+32).  r is the tile's complete
// accumulator: with K-chunked accumulation the kernel sums the chunks in TMEM first and calls the functor once
// (chunk = 0, nchunks = 1).
// ------------------------------------------------------------------------------------------

// K3: Σᵀ[i][k] = σ(z), z = x_iᵀw_k.  kOut: 0 = bf16, 1 = fp32, 2 = fp32 hi/lo split (3×TF32).
// kAct = rf_act (compile time), or −1: the runtime `act` (the Table-2 activations of NEXT-3).
template <int kOut, int kAct>
struct EpiSigma {
  void* out0;
  void* out1;
  int64_t ld;       // elements
  int64_t M, N;     // n rows (samples), m_local columns (features)
  int act;          // used when kAct < 0
  ActRt ap;         // kAct < 0 and ap.kind > 0: a parametrised Table-2 σ (leaky ReLU, quadratic)
  __device__ __forceinline__ bool chunk_needed(int64_t row_lo, int64_t col0) const { return col0 < N && row_lo < M; }
  __device__ __forceinline__ void tile_done(int, uint32_t) const {}
  struct Pre {};
  __device__ __forceinline__ Pre prefetch(int64_t, int64_t, uint32_t) const { return Pre{}; }
  template <class Ctx>
  __device__ __forceinline__ void operator()(Ctx& cx, int64_t row_lo, int64_t col0, const uint32_t (&r)[32], int,
                                             int, long long, const Pre&) const {
    const int64_t row = row_lo + cx.lane;
    if (row >= M) return;
    RF_DCHECK(col0 >= 0 && col0 < N, "K3 col0 %lld N %lld", (long long)col0, (long long)N);
    float s[32];
#pragma unroll
    for (int e = 0; e < 32; ++e)
      s[e] = kAct < 0 ? (ap.kind ? act_param<float>(ap, __uint_as_float(r[e])) : act_f32(act, __uint_as_float(r[e])))
                      : (kOut == 0 ? act_bf16out<kAct>(__uint_as_float(r[e])) : act_fixed<kAct>(__uint_as_float(r[e])));
    const bool full = col0 + 32 <= N;
    if (kOut == 0) {
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(out0) + row * ld + col0;
      if (full) {
        uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint32_t w[4];
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(s[v * 8 + 2 * h], s[v * 8 + 2 * h + 1]);
            w[h] = *reinterpret_cast<uint32_t*>(&b2);
          }
          d4[v] = make_uint4(w[0], w[1], w[2], w[3]);
        }
      } else {
        for (int e = 0; e < 32; ++e)
          if (col0 + e < N) dst[e] = __float2bfloat16_rn(s[e]);
      }
    } else {
      float* d0 = reinterpret_cast<float*>(out0) + row * ld + col0;
      float* d1 = kOut == 2 ? reinterpret_cast<float*>(out1) + row * ld + col0 : nullptr;
      if (full) {
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          float4 a = make_float4(s[4 * v], s[4 * v + 1], s[4 * v + 2], s[4 * v + 3]);
          if (kOut == 2) {
            float4 h = make_float4(tf32_hi(a.x), tf32_hi(a.y), tf32_hi(a.z), tf32_hi(a.w));
            float4 l = make_float4(a.x - h.x, a.y - h.y, a.z - h.z, a.w - h.w);
            reinterpret_cast<float4*>(d0)[v] = h;
            reinterpret_cast<float4*>(d1)[v] = l;
          } else {
            reinterpret_cast<float4*>(d0)[v] = a;
          }
        }
      } else {
        for (int e = 0; e < 32; ++e) {
          if (col0 + e < N) {
            if (kOut == 2) {
              const float h = tf32_hi(s[e]);
              d0[e] = h;
              d1[e] = s[e] - h;
            } else {
              d0[e] = s[e];
            }
          }
        }
      }
    }
  }
};

// K3^ter (NEXT-1, Algorithm 1 step 4): Σ^terᵀ[i][k] = σ^ter(c·z), z = x_iᵀt_k, W^ter = c·T, c = (1−ε)^{-1/2}
// (Eq. (4)); σ^ter(v) = −1 if v < s−, +1 if v > s+, else 0 (Eq. (5)).  The comparison is made on z against
// t± = s±/c (rounded once on the host), so no product is formed per entry.  Stored as FP8 E4M3 codes
// (+1 = 0x38, −1 = 0xB8, 0 = 0x00): exact operands for the fp8 SYRK that forms G^ter.
struct EpiSigmaTer {
  uint8_t* out;
  int64_t ld;       // bytes
  int64_t M, N;     // n rows (samples), m_local columns (features)
  float t_minus, t_plus;
  __device__ __forceinline__ bool chunk_needed(int64_t row_lo, int64_t col0) const { return col0 < N && row_lo < M; }
  __device__ __forceinline__ void tile_done(int, uint32_t) const {}
  struct Pre {};
  __device__ __forceinline__ Pre prefetch(int64_t, int64_t, uint32_t) const { return Pre{}; }
  template <class Ctx>
  __device__ __forceinline__ void operator()(Ctx& cx, int64_t row_lo, int64_t col0, const uint32_t (&r)[32], int,
                                             int, long long, const Pre&) const {
    const int64_t row = row_lo + cx.lane;
    if (row >= M) return;
    uint32_t w[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const float z = __uint_as_float(r[4 * q + b]);
        const uint32_t code = z > t_plus ? 0x38u : (z < t_minus ? 0xB8u : 0u);
        word |= code << (8 * b);
      }
      w[q] = word;
    }
    uint8_t* dst = out + row * ld + col0;
    if (col0 + 32 <= N) {
      reinterpret_cast<uint4*>(dst)[0] = make_uint4(w[0], w[1], w[2], w[3]);
      reinterpret_cast<uint4*>(dst)[1] = make_uint4(w[4], w[5], w[6], w[7]);
    } else {
      for (int e = 0; e < 32; ++e)
        if (col0 + e < N) dst[e] = (uint8_t)(w[e >> 2] >> (8 * (e & 3)));
    }
  }
};

// K4: G[i][j] = scale · Σᵀ_iᵀΣᵀ_j for j ≥ i (and the mirror for FULL); chunked: G += scale·partial.
struct EpiSyrk {
  float* G;
  int64_t ld, n;
  float scale;
  int full;
  int use_tma;      // the output tensor map is valid (16-B aligned rows)
  int64_t tri_T;    // > 0: RF_OUT_PACKED_TRI with T = ceil(n/256)
  __device__ __forceinline__ bool chunk_needed(int64_t row_lo, int64_t col0) const {
    return col0 < n && row_lo < n && col0 + 31 >= row_lo;
  }
  __device__ __forceinline__ void tile_done(int, uint32_t) const {}
  struct Pre {};
  __device__ __forceinline__ Pre prefetch(int64_t, int64_t, uint32_t) const { return Pre{}; }
  template <class Ctx>
  __device__ __forceinline__ void operator()(Ctx& cx, int64_t row_lo, int64_t col0, const uint32_t (&r)[32],
                                             int, int, long long, const Pre&) const {
    const int64_t row = row_lo + cx.lane;
    float v[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]) * scale;
    if (tri_T > 0) {
      tri_store(cx, G, n, tri_T, use_tma, row_lo, col0, v);
      return;
    }
    if (use_tma && col0 >= row_lo + 31) {
      cx.store_block(row_lo, col0, v);
    } else {
      if (row >= n) return;
      store_row_masked(G, ld, n, row, col0, row, v);
    }
    if (full) store_mirror(G, ld, n, row, col0, v);
  }
};

// K4 with PACKED output: the multi-GPU G5 (include/rf.h).  Tile ownership is canonical (rf_tile_map): the row tiles
// are cut into chunks (crow[c] .. crow[c+1]); inside chunk c the upper 256-tiles (I, J ≥ I) are numbered row-major
// from u = 0, and tile u goes to owner u mod world, slot u div world.  Every 256×256 tile of the upper triangle is
// stored whole; 256-tiles a pair tile covers below the diagonal (J < I) or past the matrix (J ≥ T) are skipped.
//   NCCL:  send + soff[c] + (owner·slots[c] + slot)·65536         (chunk-major, owner-major: one ReduceScatter per chunk)
//   PEERS: peer[owner] + self·recv_elems + roff[c] + slot·65536   (the owner's staging buffer, over NVLink)
constexpr int kMaxP2P = RF_MAX_PEERS;
constexpr int kMaxChunks = 16;
struct PackDev {
  int32_t T;                                 // 256-tiles per side
  int32_t nchunks, world, self, p2p;
  int32_t crow[kMaxChunks + 1];              // first row tile of chunk c
  int64_t slots[kMaxChunks];
  int64_t soff[kMaxChunks + 1];
  int64_t roff[kMaxChunks + 1];
  int64_t recv_elems;
  float* send;                               // NCCL send buffer (workspace)
  uint32_t* sync;                            // NCCL: per-chunk count of finished (pair tile, epilogue warp)s; else null
  float* peer[kMaxP2P];
};
struct EpiSyrkPacked {
  float scale;
  PackDev pk;
  __device__ __forceinline__ bool chunk_needed(int64_t row_lo, int64_t col0) const {
    return (col0 >> 8) >= (row_lo >> 8) && (col0 >> 8) < pk.T;
  }
  struct Pre {};
  __device__ __forceinline__ Pre prefetch(int64_t, int64_t, uint32_t) const { return Pre{}; }
  __device__ __forceinline__ int chunk_of(int ti) const {
    int c = 0;
    while (c + 1 < pk.nchunks && ti >= pk.crow[c + 1]) ++c;
    return c;
  }
  template <class Ctx>
  __device__ __forceinline__ void operator()(Ctx& cx, int64_t row_lo, int64_t col0, const uint32_t (&r)[32],
                                             int, int, long long, const Pre&) const {
    const int64_t I = row_lo >> 8, J = col0 >> 8;
    const int c = chunk_of((int)I);
    const int64_t r0 = pk.crow[c];
    const int64_t u = (I - r0) * pk.T - (I * (I - 1) - r0 * (r0 - 1)) / 2 + (J - I);   // row-major in the chunk
    const int64_t owner = u % pk.world, slot = u / pk.world;
    RF_DCHECK(J >= I && J < pk.T && c >= 0 && c < pk.nchunks && I >= pk.crow[c] && I < pk.crow[c + 1] && u >= 0 &&
                  slot < pk.slots[c] && (!pk.p2p || pk.peer[owner] != nullptr),
              "G5 tile (%lld, %lld) chunk %d u %lld slot %lld", (long long)I, (long long)J, c, (long long)u,
              (long long)slot);
    float* tile = pk.p2p ? pk.peer[owner] + (int64_t)pk.self * pk.recv_elems + pk.roff[c] +
                               slot * (int64_t)(RF_PACK_TILE * RF_PACK_TILE)
                         : pk.send + pk.soff[c] + (owner * pk.slots[c] + slot) * (int64_t)(RF_PACK_TILE * RF_PACK_TILE);
    float v[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]) * scale;
    // Whole 32-B sectors: four 256-bit stores per lane (its row's 128 B), so over NVLink (the peer path) every store
    // carries full sectors rather than 16-B halves, and the warp issues half the store instructions.  (Staging the
    // block through shared memory for whole 128-B lines made the K4 epilogue slower beside the co-resident G5 sums:
    // R = 8 emulation 31.2 vs 29.4 ms per call.)
    float* dst = tile + ((row_lo & 255) + cx.lane) * RF_PACK_TILE + (col0 & 255);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      ptx::stg256(dst + 8 * q, v[8 * q], v[8 * q + 1], v[8 * q + 2], v[8 * q + 3], v[8 * q + 4], v[8 * q + 5],
                  v[8 * q + 6], v[8 * q + 7]);
  }
  // After the warp's last store of a pair tile in row tile ti, publish it to the chunk counter (system-scope fence,
  // one atomic per epilogue warp: the library waits for 2 · EPI_WARPS · (pair tiles of the chunk) — NCCL: before the
  // chunk's reduce-scatter; peers: before the chunk's arrival flags).
  __device__ __forceinline__ void tile_done(int ti, uint32_t lane) const {
    if (!pk.sync) return;
    __syncwarp();
    if (lane == 0) {
      __threadfence_system();
      atomicAdd(pk.sync + chunk_of(ti), 1u);
    }
  }
};

// K5: Φ[i][j] = EQ1 with x_i as pivot (DESIGN.md §4 R6), j ≥ i.  Off-diagonal chunks evaluate EQ1 on fp32
// pairs (eq1_pair); kOdd selects the odd-σ form Φ = ν·A1(α)·C1(s) (A0 = A2 = 0 for odd σ).
template <bool kOdd>
struct EpiEq1 {
  static constexpr int kColVec = 1;   // ‖x_j‖²/τ staged per tile in shared memory by the producer (ColVecOf)
  static constexpr int kFast = 1;     // interior tiles: fast<kSlot> (FastOf)
  float* Phi;
  int64_t ld, n;
  const RowCoef* rc;     // per row
  const float* col_src;  // ‖x_j‖²/τ per column, padded to whole 256-column tiles
  float e0, e1, e2, f0, f1;
  int full;
  int use_tma;
  int64_t tri_T;          // > 0: RF_OUT_PACKED_TRI
  __device__ __forceinline__ bool chunk_needed(int64_t row_lo, int64_t col0) const {
    return col0 < n && row_lo < n && col0 + 31 >= row_lo;
  }
  __device__ __forceinline__ void tile_done(int, uint32_t) const {}
  // The row's coefficient record does not depend on the accumulator: loaded before the TMEM wait.
  struct Pre {
    RowCoef c;
  };
  __device__ __forceinline__ Pre prefetch(int64_t row_lo, int64_t, uint32_t lane) const {
    const int64_t row = row_lo + lane;
    return Pre{rc[row < n ? row : n - 1]};
  }
  // A 256×256 tile strictly right of the diagonal tile and inside the n×n matrix, stored by TMA into the plain
  // upper triangle: every 32×32 chunk is needed and off the diagonal.
  __device__ __forceinline__ bool fast_tile(int ti, int tj) const {
#if defined(K5_EXP)
    return false;   // timing experiments run the general path
#endif
    return tri_T == 0 && !full && use_tma && tj > ti && (int64_t)(tj + 1) * 256 <= n;
  }
  template <int kSlot, class Ctx>
  __device__ __forceinline__ void fast(Ctx& cx, int32_t row_lo, int32_t col0, const uint32_t (&r)[32],
                                       const Pre& pf) const {
    RF_DCHECK(col0 >= row_lo + 32 && (int64_t)col0 + 32 <= n, "fast chunk row_lo %d col0 %d n %lld", row_lo, col0,
              (long long)n);
    const RowCoef& c = pf.c;
    float nj[32];
    const uint32_t ca = cx.col_s + (uint32_t)(col0 & 255) * 4;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 t = ptx::lds128(ca + 16 * q);
      nj[4 * q] = t.x; nj[4 * q + 1] = t.y; nj[4 * q + 2] = t.z; nj[4 * q + 3] = t.w;
    }
    float v[32];
    if (kOdd) {
      const float P = c.c * c.a1 * f0, Q = c.c * c.a1 * f1;
      const uint64_t c2 = pk2(c.c, c.c), p2 = pk2(P, P), q2 = pk2(Q, Q);
#pragma unroll
      for (int e = 0; e < 32; e += 2)
        eq1_pair_odd(__uint_as_float(r[e]), __uint_as_float(r[e + 1]), nj[e], nj[e + 1], c2, p2, q2, v[e], v[e + 1]);
    } else {
      const uint64_t c2 = pk2(c.c, c.c), a0_2 = pk2(c.a0, c.a0), a1_2 = pk2(c.a1, c.a1), a2h_2 = pk2(c.a2h, c.a2h);
      const uint64_t e0_2 = pk2(e0, e0), e1_2 = pk2(e1, e1), e2_2 = pk2(e2, e2), f0_2 = pk2(f0, f0), f1_2 = pk2(f1, f1);
#pragma unroll
      for (int e = 0; e < 32; e += 2)
        eq1_pair<kOdd>(__uint_as_float(r[e]), __uint_as_float(r[e + 1]), nj[e], nj[e + 1], c2, a0_2, a1_2, a2h_2, e0_2,
                       e1_2, e2_2, f0_2, f1_2, v[e], v[e + 1]);
    }
    cx.template store_static<kSlot>(row_lo, col0, v);
  }
  template <class Ctx>
  __device__ __forceinline__ void operator()(Ctx& cx, int64_t row_lo, int64_t col0, const uint32_t (&r)[32], int,
                                             int, long long, const Pre& pf) const {
    const int64_t row = row_lo + cx.lane;
    const RowCoef& c = pf.c;
    float nj[32];   // columns past n hold padding; their results are never stored
    const uint32_t ca = cx.col_s + (uint32_t)(col0 & 255) * 4;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 t = ptx::lds128(ca + 16 * q);
      nj[4 * q] = t.x; nj[4 * q + 1] = t.y; nj[4 * q + 2] = t.z; nj[4 * q + 3] = t.w;
    }
    float v[32];
#if defined(K5_EXP) && K5_EXP == 3
    if (true) {
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]) + nj[e];
    } else
#endif
    if (col0 + 31 >= row_lo && col0 <= row_lo + 31) {   // chunk holds diagonal entries (warp-uniform)
#pragma unroll
      for (int e = 0; e < 32; ++e)
        v[e] = eq1_entry<float>(__uint_as_float(r[e]), c.a0, c.a1, c.a2h, c.c, nj[e], col0 + e == row, c.nu_diag, e0,
                                e1, e2, f0, f1);
    } else if (kOdd) {
      const float P = c.c * c.a1 * f0, Q = c.c * c.a1 * f1;
      const uint64_t c2 = pk2(c.c, c.c), p2 = pk2(P, P), q2 = pk2(Q, Q);
#pragma unroll
      for (int e = 0; e < 32; e += 2)
        eq1_pair_odd(__uint_as_float(r[e]), __uint_as_float(r[e + 1]), nj[e], nj[e + 1], c2, p2, q2, v[e], v[e + 1]);
    } else {
      const uint64_t c2 = pk2(c.c, c.c), a0_2 = pk2(c.a0, c.a0), a1_2 = pk2(c.a1, c.a1), a2h_2 = pk2(c.a2h, c.a2h);
      const uint64_t e0_2 = pk2(e0, e0), e1_2 = pk2(e1, e1), e2_2 = pk2(e2, e2), f0_2 = pk2(f0, f0), f1_2 = pk2(f1, f1);
#pragma unroll
      for (int e = 0; e < 32; e += 2)
        eq1_pair<kOdd>(__uint_as_float(r[e]), __uint_as_float(r[e + 1]), nj[e], nj[e + 1], c2, a0_2, a1_2, a2h_2, e0_2,
                       e1_2, e2_2, f0_2, f1_2, v[e], v[e + 1]);
    }
#if defined(K5_EXP)   // timing experiments only (scripts): 1 = no store at all, 2 = STS staging but no TMA store
    if (K5_EXP == 1 || K5_EXP == 2) {
      if (K5_EXP == 2) {
        cx.stage(cx.sbuf_s, v);
        ptx::fence_proxy_async_smem();
      }
      float acc = 0.f;
#pragma unroll
      for (int e = 0; e < 32; ++e) acc += v[e];
      if (acc == 1.2345e-30f) Phi[0] = acc;
      return;
    }
#endif
#if defined(K5_EXP) && K5_EXP == 6   // timing experiment: each lane stores its row's 32 floats as four full sectors
    if (tri_T == 0 && !full && col0 >= row_lo + 31 && col0 + 32 <= n && row < n && ((ld & 7) == 0)) {
      float* dst = Phi + row * ld + col0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        ptx::stg256(dst + 8 * q, v[8 * q], v[8 * q + 1], v[8 * q + 2], v[8 * q + 3], v[8 * q + 4], v[8 * q + 5],
                    v[8 * q + 6], v[8 * q + 7]);
      return;
    }
#endif
    if (tri_T > 0) {
      tri_store(cx, Phi, n, tri_T, use_tma, row_lo, col0, v);
      return;
    }
    if (use_tma && col0 >= row_lo + 31) {
      cx.store_block(row_lo, col0, v);
    } else {
      if (row >= n) return;
      store_row_masked(Phi, ld, n, row, col0, row, v);
    }
    if (full) store_mirror(Phi, ld, n, row, col0, v);
  }
};

// NEXT-2: Theorem 1's K̃ (EQ6) from the Gram XᵀX, centred in the same pass:
//   K̃_ij = d1·g_ij + d2·u_iᵀv_j + d0·δ_ij − r'_i − r'_j,   u_i = A v_i,  g = x_iᵀx_j,  r'_i = r_i − s/2,
// with r_i = (1/n)(d1·x_iᵀx̄ + d2·u_iᵀv̄ + d0) the row means of the uncentred matrix (x̄ = Σ_j x_j, v̄ = Σ_j v_j)
// and s their mean: P(M)P = M − r1ᵀ − 1rᵀ + s11ᵀ for the symmetric M = d1XᵀX + d2VAVᵀ + d0I.
// Per-row data: u (n × 8, zero-padded), r' (n); per-column data: Vt (8 × n), r'.  kv ≤ 8 columns of V.
struct EpiKtilde {
  float* Kt;
  int64_t ld, n;
  const float* u;     // n × 8
  const float* vt;    // 8 × nvt (rows 16-B aligned)
  int64_t nvt;
  const float* r;     // n: r'_i = r_i − s/2
  float d0, d1, d2;
  int kv;
  int full;
  int use_tma;
  __device__ __forceinline__ bool chunk_needed(int64_t row_lo, int64_t col0) const {
    return col0 < n && row_lo < n && col0 + 31 >= row_lo;
  }
  __device__ __forceinline__ void tile_done(int, uint32_t) const {}
  struct Pre {
    float u[8];
    float r;
  };
  __device__ __forceinline__ Pre prefetch(int64_t row_lo, int64_t, uint32_t lane) const {
    Pre pf;
    const int64_t row = row_lo + lane;
    const int64_t rr = row < n ? row : n - 1;
    const float4 a = __ldg(reinterpret_cast<const float4*>(u + rr * 8));
    const float4 b = __ldg(reinterpret_cast<const float4*>(u + rr * 8) + 1);
    pf.u[0] = a.x; pf.u[1] = a.y; pf.u[2] = a.z; pf.u[3] = a.w;
    pf.u[4] = b.x; pf.u[5] = b.y; pf.u[6] = b.z; pf.u[7] = b.w;
    pf.r = __ldg(r + rr);
    return pf;
  }
  template <class Ctx>
  __device__ __forceinline__ void operator()(Ctx& cx, int64_t row_lo, int64_t col0, const uint32_t (&acc)[32], int,
                                             int, long long, const Pre& pf) const {
    const int64_t row = row_lo + cx.lane;
    const bool colfull = col0 + 32 <= n;
    float v[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = fmaf(d1, __uint_as_float(acc[e]), -pf.r);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float rj[4];
      if (colfull) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(r + col0) + q);
        rj[0] = t.x; rj[1] = t.y; rj[2] = t.z; rj[3] = t.w;
      } else {
#pragma unroll
        for (int b = 0; b < 4; ++b) rj[b] = (col0 + 4 * q + b < n) ? __ldg(r + col0 + 4 * q + b) : 0.f;
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) v[4 * q + b] -= rj[b];
    }
    for (int k = 0; k < kv; ++k) {
      const float uk = d2 * pf.u[k];
      const float* vk = vt + (int64_t)k * nvt + col0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float vj[4];
        if (colfull) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(vk) + q);
          vj[0] = t.x; vj[1] = t.y; vj[2] = t.z; vj[3] = t.w;
        } else {
#pragma unroll
          for (int b = 0; b < 4; ++b) vj[b] = (col0 + 4 * q + b < n) ? __ldg(vk + 4 * q + b) : 0.f;
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) v[4 * q + b] = fmaf(uk, vj[b], v[4 * q + b]);
      }
    }
    if (col0 <= row_lo + 31 && row_lo <= col0 + 31) {            // chunk crosses the diagonal: the d0·I term
#pragma unroll
      for (int e = 0; e < 32; ++e)
        if (col0 + e == row) v[e] += d0;
    }
    if (use_tma && col0 >= row_lo + 31) {
      cx.store_block(row_lo, col0, v);
    } else {
      if (row >= n) return;
      store_row_masked(Kt, ld, n, row, col0, row, v);
    }
    if (full) store_mirror(Kt, ld, n, row, col0, v);
  }
};

// Raw accumulator D = A·Bᵀ (rectangular, fp32, chunk-accumulated) — the mainloop test hook behind
// rf_debug_gemm_nt.
struct EpiRaw {
  float* C;
  int64_t ld, M, N;
  __device__ __forceinline__ bool chunk_needed(int64_t row_lo, int64_t col0) const { return col0 < N && row_lo < M; }
  __device__ __forceinline__ void tile_done(int, uint32_t) const {}
  struct Pre {};
  __device__ __forceinline__ Pre prefetch(int64_t, int64_t, uint32_t) const { return Pre{}; }
  template <class Ctx>
  __device__ __forceinline__ void operator()(Ctx& cx, int64_t row_lo, int64_t col0, const uint32_t (&r)[32],
                                             int, int, long long, const Pre&) const {
    const int64_t row = row_lo + cx.lane;
    if (row >= M) return;
    float v[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]);
    store_row_masked(C, ld, N, row, col0, 0, v);
  }
};

// ------------------------------------------------------------------------------------------
// The kernel.  Launch: grid = 2 × (#clusters), cluster dims (2,1,1), 384 threads, Cfg::SMEM_BYTES.
// ------------------------------------------------------------------------------------------
template <class Cfg, class Epi>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmA_lo, const __grid_constant__ CUtensorMap tmB_lo,
                   const __grid_constant__ CUtensorMap tmOut, const Sched sched, const Epi epi) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  constexpr int STAGES = Cfg::STAGES, NOPS = Cfg::NOPS, NSUB = Cfg::NSUB;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment by an offset from the __shared__ array (not an integer round trip), so the compiler keeps the
  // shared address space and the epilogue's staging stores compile to STS, not generic ST
  const uint32_t pad = (1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u;
  if (pad > (uint32_t)Cfg::SLACK) __trap();   // never seen: the dynamic window starts 1024-aligned
  uint8_t* smem = smem_raw + pad;
  uint8_t* sA = smem;                       // [STAGES][NOPS][A_BYTES], or (A residency) [ARES_KB][A_BYTES]
  uint8_t* sB = sA + (Cfg::ARES ? (size_t)Cfg::ARES_BYTES : (size_t)STAGES * NOPS * Cfg::A_BYTES);   // [STAGES][NOPS][NSUB][B_BYTES]
  uint8_t* sStg = sB + (size_t)STAGES * NOPS * NSUB * Cfg::B_BYTES;      // [EPI_WARPS][STG_BUFS][4096]
  float* sCol = reinterpret_cast<float*>(sStg + Cfg::STG_BYTES);          // [2][BN] column vectors (kColVec)
  uint64_t* full = reinterpret_cast<uint64_t*>(sStg + Cfg::STG_BYTES + Cfg::COL_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* colfull = tempty + 2;
  uint64_t* colempty = colfull + 2;
  uint64_t* rfull = colempty + 2;       // dynamic-unit ring (TileSeq)
  uint64_t* rempty = rfull + kRing;
  uint64_t* afull = rempty + kRing;     // A residency: the resident A panel has landed / its last MMAs completed
  uint64_t* aempty = afull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + 1);
  uint32_t* ring = tmem_slot + 1;
  constexpr bool kCol = ColVecOf<Epi>::value;
  static_assert(!kCol || (Cfg::COL_BYTES > 0 && Cfg::CL == 2), "column vectors: 256-wide pair tiles, clusters of 2");

  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();
  const uint32_t crank = ptx::cluster_ctarank();
  const uint32_t rank = crank & 1u;                    // rank inside the CTA pair
  const uint32_t pi = crank >> 1;                      // pair index inside the cluster (kCl = 4)
  const uint32_t leader = crank & ~1u;                 // cluster rank of this pair's MMA-issuing CTA
  const int cid = (int)ptx::cluster_id_x();
  const int ncl = (int)ptx::ncluster_x();

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    if (NOPS == 2 || Cfg::CL >= 4) {
      ptx::prefetch_tmap(&tmA_lo);
      ptx::prefetch_tmap(&tmB_lo);
    }
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      // released by the MMA commit of every pair whose smem this CTA's loads fill: itself (CL 2), both pairs
      // (CL 4), itself + its A partner + its B partner (CL 8)
      ptx::mbar_init(&empty[s], Cfg::CL == 8 ? 3 : Cfg::CL / 2);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 2 * Cfg::EPI_WARPS);
      ptx::mbar_init(&colfull[a], 1);
      ptx::mbar_init(&colempty[a], Cfg::EPI_WARPS);
    }
    // ring consumers per cluster: the other CTAs' producers, one MMA warp per pair, every epilogue warp (and, with
    // a column vector, every CTA's column loader)
    for (int a = 0; a < kRing; ++a) {
      ptx::mbar_init(&rfull[a], 1);
      ptx::mbar_init(&rempty[a], (Cfg::CL - 1) + Cfg::CL / 2 + Cfg::CL * Cfg::EPI_WARPS + (kCol ? Cfg::CL : 0));
    }
    ptx::mbar_init(afull, 1);
    ptx::mbar_init(aempty, 1);
    ptx::fence_mbarrier_init();
  }
  if (sched.started && blockIdx.x == 0 && threadIdx.x == 0) ptx::st_relaxed_gpu(sched.started, 1u);
  if (warp == 2) ptx::tmem_alloc_cg2(tmem_slot, 512);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
#if defined(RF_DEBUG)
  // the pair allocates all 512 columns of each CTA's TMEM: the base must be lane 0, column 0 (a leaked or
  // concurrent allocation would show up here)
  if (tmem_base != 0u) {
    printf("[rf debug] TMEM allocation base 0x%x (expected 0) block %d\n", tmem_base, (int)blockIdx.x);
    __trap();
  }
#endif
  const int kchunk = sched.kchunk, nchunks = sched.nchunks, num_kb = sched.num_kb;
  // dynamic units only for the K4 hybrid's configurations (512-wide pair tiles) and the A-resident K5 (segments);
  // the host never sets sched.queue else
  constexpr bool kDyn = (Cfg::BN == 512 && Cfg::CL <= 4 && !kCol) || Cfg::ARES;
  const uint32_t ring_s = ptx::smem_u32(ring), rfull_s = ptx::smem_u32(&rfull[0]), rempty_s = ptx::smem_u32(&rempty[0]);
  const uint32_t rempty_c = ptx::mapa(rempty_s, 0);   // the fetcher's (cluster rank 0) ring_empty
  auto make_seq = [&](bool fetcher) {
    TileSeq q;
    q.init(&sched, cid, ncl, Cfg::CL, (int)pi, fetcher, lane, ring_s, rfull_s, rempty_s, rempty_c);
    return q;
  };

  if (warp == 0) {
    // ===== TMA producer (both CTAs; completion bytes land on the leader's full barrier) =====
    // The whole warp walks the loop (lane 0 issues); the leader's warp also runs the lockstep check.
    const bool lock = sched.prog != nullptr && crank == 0;
    const uint64_t pol = sched.load_pol ? ptx::policy_evict_last() : ptx::policy_evict_normal();
    const uint32_t full0 = ptx::mapa(ptx::smem_u32(&full[0]), leader);
    // kCl = 4: barrier operand of the multicast B load in the CTA-relative form with the pair bit cleared,
    // so each destination's bytes are counted on its own pair leader's full barrier.
    const uint32_t full_rel0 = ptx::smem_u32(&full[0]) & 0xFEFFFFFFu;
    const uint16_t mc_mask = (uint16_t)((1u << rank) | (1u << (2 + rank)));
    // CL 8: pair pi = di + 2·dj computes row tile 2I + di, column tile 2J + dj; A (row tile) is shared with pair
    // (di, 1 − dj), B (column tile) with pair (1 − di, dj)
    const uint32_t di = pi & 1u, dj = pi >> 1;
    const uint16_t mcA8 = (uint16_t)((1u << (2 * di + rank)) | (1u << (2 * (di + 2) + rank)));
    const uint16_t mcB8 = (uint16_t)((1u << (2 * (2 * dj) + rank)) | (1u << (2 * (1 + 2 * dj) + rank)));
    int stage = 0;
    uint32_t phase = 0;
    uint32_t step = 0;
    TileSeq seq = make_seq(crank == 0);
    long long t;
    int ti, tj;
    uint32_t tiles_done = 0;
    const uint32_t afull_c = ptx::mapa(ptx::smem_u32(afull), leader);
    while (seq.template next<kDyn, Cfg::ARES>(t, ti, tj)) {
      const int ra = ti * Cfg::BM + (int)rank * 128;
      const int rb = tj * Cfg::BN + (int)rank * 128;
      if constexpr (Cfg::ARES) {
        // a new segment: reload this CTA's 128-row A panel over the whole K once the MMAs of the previous tile (the
        // last reader of the old panel) have completed; completion bytes of both CTAs on the leader's afull
        if (seq.seg_first && lane == 0) {
          if (tiles_done > 0) ptx::mbar_wait(aempty, (tiles_done - 1) & 1u);
          if (rank == 0) ptx::mbar_arrive_expect_tx(afull, 2u * (uint32_t)num_kb * Cfg::A_BYTES);
          for (int kb = 0; kb < num_kb; ++kb)
            ptx::tma_load_2d_cg2(sA + (size_t)kb * Cfg::A_BYTES, &tmA, afull_c, kb * Cfg::BK, ra, pol);
        }
        __syncwarp();
        ++tiles_done;
      }
      for (int c = 0; c < nchunks; ++c) {
        const int kb1 = min(num_kb, (c + 1) * kchunk);
        for (int kb = c * kchunk; kb < kb1; ++kb, ++step) {
          if (lock && (step % (uint32_t)sched.lock_ks) == 0) {
            if (lane == 0) ptx::st_relaxed_gpu(sched.prog + cid, step);
            const uint32_t need = step > (uint32_t)sched.lock_w ? step - (uint32_t)sched.lock_w : 0u;
            const uint64_t t0 = ptx::globaltimer_ns();
            for (;;) {
              uint32_t mn = 0xFFFFFFFFu;
              for (int q = (int)lane; q < ncl; q += 32) mn = min(mn, ptx::ld_relaxed_gpu(sched.prog + q));
              mn = __reduce_min_sync(0xFFFFFFFFu, mn);
              if (mn >= need || ptx::globaltimer_ns() - t0 > 50000ull) break;
              __nanosleep(256);
            }
          }
#if defined(K5_EXP) && K5_EXP == 5
          constexpr bool kSkipA = kCol;   // timing experiment: no A operand loads (stale smem, wrong results)
#else
          constexpr bool kSkipA = false;
#endif
          if (lane == 0) {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            if (rank == 0)   // both CTAs' bytes
              ptx::mbar_arrive_expect_tx(&full[stage], 2 * (Cfg::STAGE_BYTES - (kSkipA ? Cfg::A_BYTES : 0)));
            const uint32_t fb = full0 + stage * 8;
            const int k = kb * Cfg::BK;
            uint8_t* a = sA + (size_t)(stage * NOPS) * Cfg::A_BYTES;
            uint8_t* b = sB + (size_t)(stage * NOPS * NSUB) * Cfg::B_BYTES;
            if (Cfg::CL == 8) {
              // A: the 64-row half dj of this CTA's 128 A rows (tmA_lo: 64-row box) to rank r of pairs (di, 0/1);
              // B: sub-tile di of the column tile to rank r of pairs (0/1, dj)
              ptx::tma_load_2d_cg2_mc(a + dj * (Cfg::A_BYTES / 2), &tmA_lo, full_rel0 + stage * 8, k, ra + 64 * (int)dj,
                                      mcA8, pol);
              ptx::tma_load_2d_cg2_mc(b + di * Cfg::B_BYTES, &tmB, full_rel0 + stage * 8, k, rb + 256 * (int)di, mcB8,
                                      pol);
            } else if (!kSkipA && !Cfg::ARES) {
              ptx::tma_load_2d_cg2(a, &tmA, fb, k, ra, pol);
            }
            if (Cfg::CL == 8) {
            } else if (Cfg::CL == 4 && NSUB == 2) {
              ptx::tma_load_2d_cg2_mc(b + pi * Cfg::B_BYTES, &tmB, full_rel0 + stage * 8, k, rb + 256 * (int)pi, mc_mask,
                                      pol);
            } else if (Cfg::CL == 4) {
              // 256-wide tiles: the pair's B tile is one sub-tile; CTA (pi, r) loads the 64-row half pi of its rank's
              // 128 rows (tmB_lo: the same operand with a 64-row box) and multicasts it to rank r of both pairs
              ptx::tma_load_2d_cg2_mc(b + pi * (Cfg::B_BYTES / 2), &tmB_lo, full_rel0 + stage * 8, k, rb + 64 * (int)pi,
                                      mc_mask, pol);
            } else {
#pragma unroll
              for (int s = 0; s < NSUB; ++s)
                ptx::tma_load_2d_cg2(b + s * Cfg::B_BYTES, &tmB, fb, k, rb + 256 * s, pol);
            }
            if (NOPS == 2) {
              ptx::tma_load_2d_cg2(a + Cfg::A_BYTES, &tmA_lo, fb, k, ra, pol);
#pragma unroll
              for (int s = 0; s < NSUB; ++s)
                ptx::tma_load_2d_cg2(b + (NSUB + s) * Cfg::B_BYTES, &tmB_lo, fb, k, rb + 256 * s, pol);
            }
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    if (lock && lane == 0) ptx::st_relaxed_gpu(sched.prog + cid, 0xFFFFFFFFu);   // done: never the minimum
  } else if (warp == 1) {
    if (rank == 0) {
      // ===== MMA issuer (leader CTA).  The whole warp walks the loop so that stage addresses and UMMA
      // descriptors stay warp-uniform (uniform datapath, no per-MMA R2UR broadcasts); one elected lane
      // issues the k-block's MMAs and commits.
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      uint16_t empty_mask = Cfg::CL == 4 ? 0xF : 0x3;
      if (Cfg::CL == 8) {   // this pair, its A partner (di, 1 − dj) and its B partner (1 − di, dj)
        const uint32_t di = pi & 1u, dj = pi >> 1;
        const uint32_t pa = di + 2 * (1 - dj), pb = (1 - di) + 2 * dj;
        empty_mask = (uint16_t)((0x3u << (2 * pi)) | (0x3u << (2 * pa)) | (0x3u << (2 * pb)));
      }
      TileSeq seq = make_seq(false);
      long long t;
      int ti, tj;
      uint32_t segs = 0;
      while (seq.template next<kDyn, Cfg::ARES>(t, ti, tj)) {
        if constexpr (Cfg::ARES) {
          if (seq.seg_first) {   // the segment's A panel has landed in both CTAs
            ptx::mbar_wait(afull, segs & 1u);
            ++segs;
          }
        }
        for (int c = 0; c < nchunks; ++c, ++it) {
          // K-chunked accumulation: every chunk goes to slot 0; the epilogue keeps the running fp32 sum in slot 1
          const bool dbl = Cfg::ACC_SLOTS == 2 && nchunks == 1;
          const int slot = dbl ? (it & 1) : 0;
          const uint32_t acc_phase = (dbl ? (it >> 1) : it) & 1;
          ptx::mbar_wait(&tempty[slot], acc_phase ^ 1);
          ptx::tc_fence_after();
          const uint32_t d = tmem_base + slot * Cfg::ACC_COLS;
          const int kb0 = c * kchunk, kb1 = min(num_kb, (c + 1) * kchunk);
          for (int kb = kb0; kb < kb1; ++kb) {
            ptx::mbar_wait(&full[stage], phase);
            ptx::tc_fence_after();
            const uint32_t a_s = ptx::smem_u32(sA + (Cfg::ARES ? (size_t)kb * Cfg::A_BYTES
                                                              : (size_t)(stage * NOPS) * Cfg::A_BYTES));
            const uint32_t b_s = ptx::smem_u32(sB + (size_t)(stage * NOPS * NSUB) * Cfg::B_BYTES);
            const uint64_t ad = ptx::sdesc_k128(a_s);
            if (ptx::elect_one()) {
#pragma unroll
              for (int k = 0; k < Cfg::BK / Cfg::UK; ++k) {
                const uint64_t off = (uint64_t)((k * 32) >> 4);   // +32 B along K inside the swizzle row
                const uint32_t accum = (kb != kb0 || k != 0) ? 1u : 0u;
#pragma unroll
                for (int s = 0; s < NSUB; ++s) {
                  const uint64_t bd = ptx::sdesc_k128(b_s + s * Cfg::B_BYTES);
                  const uint32_t ds = d + s * 256;
                  if (NOPS == 2) {
                    const uint64_t adl = ptx::sdesc_k128(a_s + Cfg::A_BYTES);
                    const uint64_t bdl = ptx::sdesc_k128(b_s + (NSUB + s) * Cfg::B_BYTES);
                    ptx::mma_tf32_cg2(ds, adl + off, bd + off, Cfg::IDESC, accum);
                    ptx::mma_tf32_cg2(ds, ad + off, bdl + off, Cfg::IDESC, 1u);
                    ptx::mma_tf32_cg2(ds, ad + off, bd + off, Cfg::IDESC, 1u);
                  } else if (Cfg::ESZ == 2) {
                    ptx::mma_bf16_cg2(ds, ad + off, bd + off, Cfg::IDESC, accum);
                  } else if (Cfg::ESZ == 1) {
                    ptx::mma_f8_cg2(ds, ad + off, bd + off, Cfg::IDESC, accum);
                  } else {
                    ptx::mma_tf32_cg2(ds, ad + off, bd + off, Cfg::IDESC, accum);
                  }
                }
              }
              ptx::mma_commit_cg2_mc(&empty[stage], empty_mask);   // every CTA that fed the stage
            }
            __syncwarp();
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          if (ptx::elect_one()) ptx::mma_commit_cg2_mc(&tfull[slot], (uint16_t)(0x3u << (2 * pi)));
          __syncwarp();
        }
        // A residency: this tile's MMAs — the last readers so far of the resident A panel — complete → aempty
        if (Cfg::ARES && ptx::elect_one()) ptx::mma_commit_cg2_mc(aempty, (uint16_t)0x3u);
        __syncwarp();
      }
    }
  } else if (warp == 3) {
    if constexpr (kCol) {
      // ===== Column-vector loader: tile k's slice of the per-column vector into sCol[k & 1] once the epilogue has
      // released the buffer (tile k − 2), a 1-D bulk copy completing on colfull.  A warp of its own, so the operand
      // producer never waits on the epilogue.
      TileSeq seq = make_seq(false);   // static, segment or dynamic-segment schedules
      long long t;
      int ti, tj;
      for (int tcount = 0; seq.template next<kDyn, Cfg::ARES>(t, ti, tj); ++tcount) {
        if (lane == 0) {
          const int cs = tcount & 1;
          ptx::mbar_wait(&colempty[cs], ((tcount >> 1) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&colfull[cs], Cfg::BN * 4);
          ptx::bulk_load_1d(sCol + cs * Cfg::BN, epi.col_src + (int64_t)tj * Cfg::BN, Cfg::BN * 4, &colfull[cs]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ===== Epilogue: TMEM → registers → fused op → global (8 warps) =====
    const uint32_t q = warp & 3;               // TMEM lane quarter this warp may access
    const uint32_t h = (warp - 4) >> 2;        // column share of the accumulator (0 .. EPI_WARPS/4 − 1)
    EpiCtx<Cfg::STG_BUFS, Cfg::HALF_STG> cx;
    cx.tm = &tmOut;
    cx.sbuf = sStg + (size_t)(warp - 4) * Cfg::STG_BUFS * Cfg::STG_BUF_BYTES;
    cx.sbuf_s = ptx::smem_u32(cx.sbuf);
    cx.col_s = 0;
    cx.cur = 0;
    cx.nst = 0;
    cx.pc0 = cx.pr0 = 0;
    cx.lane = lane;
    cx.set_stg_x();
    cx.hint = sched.store_pol;
    cx.pol = ptx::policy_evict_first();
    const uint32_t tempty0 = ptx::mapa(ptx::smem_u32(&tempty[0]), leader);
    constexpr int HALF = Cfg::ACC_COLS / 2;
    int it = 0;
    int tcount = 0;
    TileSeq seq = make_seq(false);
    long long t;
    int ti, tj;
    for (; seq.template next<kDyn, Cfg::ARES>(t, ti, tj); ++tcount) {
      if constexpr (kCol) {   // the tile's column vector (bulk-copied by this CTA's producer when the tile started)
        ptx::mbar_wait(&colfull[tcount & 1], (tcount >> 1) & 1);
        cx.col_s = ptx::smem_u32(sCol + (tcount & 1) * Cfg::BN);
      }
      const int64_t row_lo = (int64_t)ti * Cfg::BM + rank * 128 + q * 32;
      const int64_t colb = (int64_t)tj * Cfg::BN + h * HALF;
      if (Cfg::ACC_SLOTS == 2 && Cfg::EPI_WARPS == 8 && nchunks > 1) {
        // K-chunked accumulation (3×TF32; the tensor pipe truncates long accumulations, DESIGN.md §6 finding 4):
        // chunk c's partial arrives in slot 0; the warp adds it to the running sum in slot 1 in fp32
        // (round-to-nearest) through registers, then frees slot 0 so the MMA of chunk c + 1 starts while the
        // last chunk's sum goes out through the functor.  TMEM traffic only: no read-modify-write of G in HBM.
        const uint32_t tA = tmem_base + ((q * 32) << 16) + h * HALF;
        const uint32_t tS = tA + Cfg::ACC_COLS;
        constexpr int NCH = HALF / 32;
        const typename Epi::Pre pf = epi.prefetch(row_lo, colb, lane);
        for (int c = 0; c < nchunks; ++c, ++it) {
          ptx::mbar_wait(&tfull[0], (uint32_t)it & 1u);
          ptx::tc_fence_after();
#pragma unroll 1
          for (int cc = 0; cc < NCH; ++cc) {
            uint32_t a[32], sm[32];
            ptx::tmem_ld_32x32b_x32(tA + cc * 32, a);
            if (c > 0) ptx::tmem_ld_32x32b_x32(tS + cc * 32, sm);
            ptx::tmem_ld_wait();
            if (c > 0) {
#pragma unroll
              for (int e = 0; e < 32; ++e) a[e] = __float_as_uint(__uint_as_float(a[e]) + __uint_as_float(sm[e]));
            }
            ptx::tmem_st_32x32b_x32(tS + cc * 32, a);
          }
          ptx::tmem_st_wait();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_cluster(tempty0);
        }
        ptx::tc_fence_after();
#pragma unroll 1
        for (int cc = 0; cc < NCH; ++cc) {
          uint32_t a[32];
          ptx::tmem_ld_32x32b_x32(tS + cc * 32, a);
          ptx::tmem_ld_wait();
          const int64_t col0 = colb + cc * 32;
          if (epi.chunk_needed(row_lo, col0)) epi(cx, row_lo, col0, a, 0, 1, (long long)t, pf);
        }
        cx.flush();
        epi.tile_done(ti, lane);
        if constexpr (kCol) {
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&colempty[tcount & 1]);
        }
        continue;
      }
      for (int c = 0; c < nchunks; ++c, ++it) {
        const int slot = Cfg::ACC_SLOTS == 2 ? (it & 1) : 0;
        const uint32_t acc_phase = (Cfg::ACC_SLOTS == 2 ? (it >> 1) : it) & 1;
        const uint32_t tbase = tmem_base + ((q * 32) << 16) + slot * Cfg::ACC_COLS + h * HALF;
        if constexpr (Cfg::EPI_WARPS != 8) {
          // three (four) warps per lane quarter: 32-column chunks cc ≡ h (mod 3 (4)) of the accumulator row
          const int64_t col_t = (int64_t)tj * Cfg::BN;
          const uint32_t tb = tmem_base + ((q * 32) << 16) + slot * Cfg::ACC_COLS;
          const typename Epi::Pre pf = epi.prefetch(row_lo, col_t, lane);
          ptx::mbar_wait(&tfull[slot], acc_phase);
          ptx::tc_fence_after();
          uint32_t ra[32];
          constexpr int STEP = Cfg::EPI_WARPS / 4;
#pragma unroll 1
          for (int cc = (int)h; cc < Cfg::ACC_COLS / 32; cc += STEP) {
            ptx::tmem_ld_32x32b_x32(tb + cc * 32, ra);
            ptx::tmem_ld_wait();
            if (cc + STEP >= Cfg::ACC_COLS / 32) {
              // the warp's last chunk is in registers: hand the accumulator back to the MMA now, before its
              // transform and store, so the next tile's MMAs into this slot start one chunk earlier
              ptx::tc_fence_before();
              __syncwarp();
              if (lane == 0) ptx::mbar_arrive_cluster(tempty0 + slot * 8);
            }
            const int64_t col0 = col_t + cc * 32;
            if (epi.chunk_needed(row_lo, col0)) epi(cx, row_lo, col0, ra, c, nchunks, (long long)t, pf);
          }
          continue;
        }
        const typename Epi::Pre pf = epi.prefetch(row_lo, colb, lane);   // per-row inputs: before the wait
        ptx::mbar_wait(&tfull[slot], acc_phase);
        ptx::tc_fence_after();
        // Software pipeline over the warp's 32-column chunks: the TMEM load of chunk cc+1 is in flight while
        // chunk cc is transformed and stored (tcgen05.wait::ld waits for all of a thread's loads, so the
        // next load is issued only after the current one has been waited for).
        constexpr int NCH = HALF / 32;
        static_assert(NCH % 2 == 0, "even number of 32-column chunks");
        uint32_t ra[32], rb[32];
        auto step = [&](int cc, uint32_t(&cur)[32], uint32_t(&nxt)[32]) __attribute__((always_inline)) {
          const int64_t col0 = colb + cc * 32;
          ptx::tmem_ld_wait();
          if (cc + 1 < NCH) {
            ptx::tmem_ld_32x32b_x32(tbase + (cc + 1) * 32, nxt);
          } else {   // all of the warp's accumulator columns are in registers: release the slot before the last chunk
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(tempty0 + slot * 8);
          }
          if (epi.chunk_needed(row_lo, col0)) epi(cx, row_lo, col0, cur, c, nchunks, (long long)t, pf);
        };
        ptx::tmem_ld_32x32b_x32(tbase, ra);
        if constexpr (FastOf<Epi>::value && !Cfg::HALF_STG && (Cfg::STG_BUFS == 1 || Cfg::STG_BUFS == 2)) {
          if (nchunks == 1 && epi.fast_tile(ti, tj)) {
            // interior tile: the same pipeline with no per-chunk predicates; chunk cc → staging buffer cc & 1
            const int32_t r32 = (int32_t)row_lo, c32 = (int32_t)colb;
            auto fstep = [&](auto kslot, int cc, uint32_t(&cur)[32], uint32_t(&nxt)[32]) __attribute__((always_inline)) {
              ptx::tmem_ld_wait();
              if (cc + 1 < NCH) {
                ptx::tmem_ld_32x32b_x32(tbase + (cc + 1) * 32, nxt);
              } else {
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive_cluster(tempty0 + slot * 8);
              }
              epi.template fast<decltype(kslot)::value>(cx, r32, c32 + cc * 32, cur, pf);
            };
#pragma unroll 1
            for (int cc = 0; cc < NCH; cc += 2) {
              fstep(std::integral_constant<int, 0>{}, cc, ra, rb);
              fstep(std::integral_constant<int, 1>{}, cc + 1, rb, ra);
            }
            continue;
          }
        }
#pragma unroll 1
        for (int cc = 0; cc < NCH; cc += 2) {
          step(cc, ra, rb);
          step(cc + 1, rb, ra);
        }
      }
      cx.flush();
      epi.tile_done(ti, lane);
      if constexpr (kCol) {   // done reading this tile's column vector
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&colempty[tcount & 1]);
      }
    }
    if (lane == 0) ptx::bulk_wait_all();
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg2(tmem_base, 512);
  }
#endif
}

}  // namespace rfk
