// prefill.cu — a2 + a3: causal prefill attention of one layer with the paged
// K/V write fused in (tcgen05 / TMEM / TMA, sm_100a).
//
// What it computes (§2.1; App. A "attention only
// operates among the tokens in the same request"; readings R1 scale, R2 causal):
//   out[i] = sum_{j<=i} softmax_j(scale * q[i].k[j]) v[j]     per (sequence, head)
//   cache[layer][K|V][bt[r][t/16]][h][t%16] = k|v[t][h]       (a3)
//
// B200 design — one grid CTA per (128-row q tile, head, sequence), TWO CTAs per
// SM, run persistently: a CTA that finishes an item takes over the next CTA that
// has not launched yet (cluster launch control), so each SM slot streams items
// back to back with the next item's loads overlapping this item's tail:
//   * kv tiles of 64 keys: smem holds Q (32 KiB) + 2 K stages + 2 V stages
//     (4 x 16 KiB, 128B-swizzled, TMA-fed) = 96 KiB at head_dim 128; TMEM holds
//     256 columns = S0 | S1 (64 fp32 columns each, double-buffered) | O (128).
//     N = 64 MMAs run at the same per-MAC rate as N = 128; the 64-key tiles buy
//     double buffering of K, V and S inside the 2-CTA/SM budget, so S_{j+1}
//     and the K/V loads of tile j+1 overlap the softmax of tile j, and the two
//     co-resident CTAs interleave their softmax and MMA phases.
//   * warp 4  TMA producer: Q once; K_j / V_j into stage j%2 as soon as S_{j-2}
//             / P_{j-2}V_{j-2} released it. Afterwards it writes the two
//             diagonal K/V tiles (the only ones this CTA owns) to the paged
//             cache with TMA tensor stores, one 16-token page per store (a3).
//   * warp 5  MMA issuer (one elected lane): S_j = Q K_j^T (SS, fp32 in TMEM
//             buffer j%2), then O += P_{j-1} V_{j-1} (TS: P read from TMEM, V
//             MN-major from smem).
//   * warps 0-3 softmax: thread t owns q row t (TMEM lane t): tcgen05.ld S row,
//             online base-2 softmax (scale*log2 e folded into one FFMA), P
//             rounded to bf16 and written back over its S buffer in TMEM
//             (tcgen05.st), lazy warp-uniform O rescale in TMEM, final
//             O / l -> bf16 -> global.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace ds {
namespace {

constexpr int kBM = 128, kBN = 64;  // q rows per CTA, keys per kv tile
constexpr int kCompactSeqs = kPrefillCompactSeqs;
constexpr int kThreads = 192;
constexpr uint32_t kChunkBytes128 = 128 * 128;  // Q: 128 rows x 128 B (64 bf16) per SW128 column block
constexpr uint32_t kChunkBytes64 = 64 * 128;    // K/V tile: 64 rows x 128 B per SW128 column block
constexpr uint32_t kTmemCols = 256;             // S0 [0,64) S1 [64,128) O [128, 128+D)
constexpr float kRescaleLog2 = 8.f;             // move the exponent base only past 2^8 growth
#ifndef DS_PF_POLY_EVERY
#define DS_PF_POLY_EVERY 8
#endif
#ifndef DS_PF_SLEEP_NS  // suspend hint of the producer / MMA waits (0: plain try_wait spin)
#define DS_PF_SLEEP_NS 0
#endif
constexpr int kPolyEvery = DS_PF_POLY_EVERY;    // 1 in kPolyEvery exp2 on the FMA pipe (ex2_poly)

// Tail ordering. Launch order keeps a (sequence, head)'s q tiles together, heaviest
// first, so their K/V re-reads hit L2 — but then the last groups' heavy tiles start
// just before the end and the kernel ends on a tail (config 5, 8 x ~1.8k tokens x 24
// heads: SM activity avg / max 0.90 under ncu). The LAST groups of the launch order
// — as many as keep their K/V within DS_PF_BAND_MB of L2, at most kBandSeqs sequences
// — are launched level-major instead: every band group's q tile i before any q tile
// i-1 (tiles of a level by sequence length, descending, then head), so the heavy
// tiles start first and the light ones fill the tail.
#ifndef DS_PF_BAND_MB
#define DS_PF_BAND_MB 48
#endif
constexpr int kBandSeqs = 32, kBandLevels = 64;
struct Band {
  int item0;   // first band item in launch order (n_loc * pref[num_seqs]: no band)
  int levels;  // q-tile levels of the band (its longest sequence's tile count)
  int seq[kBandSeqs], hlo[kBandSeqs];  // band sequences, tile count descending; first band head
  int lvl[kBandLevels];                // band items of the levels above level i
};

template <int D>
struct Smem {
  static constexpr uint32_t kQTile = kBM * D * 2;
  static constexpr uint32_t kKVTile = kBN * D * 2;
  static constexpr uint32_t Q = 0;
  static constexpr uint32_t K0 = Q + kQTile;           // 2 stages
  static constexpr uint32_t V0 = K0 + 2 * kKVTile;     // 2 stages
  static constexpr uint32_t OST = V0 + 2 * kKVTile;    // epilogue staging: 4 warps x 32 rows x 32 dims bf16
  static constexpr uint32_t PREF = OST + 4 * 2048;     // int[kCompactSeqs + 1] tile prefix + 8 warp totals
  static constexpr uint32_t BAND = PREF + (kCompactSeqs + 1 + 8) * 4;  // struct Band (tail ordering)
  static constexpr uint32_t CLC = (BAND + sizeof(Band) + 15) / 16 * 16;  // 2 x 16-B work-stealing responses
  static constexpr uint32_t BAR = CLC + 32;
  static constexpr uint32_t kBars = 21;
  static constexpr uint32_t TMEM_SLOT = BAR + kBars * 8;
  static constexpr uint32_t TOTAL = TMEM_SLOT + 16;
  static constexpr uint32_t ALLOC = TOTAL + 1024;  // slack for 1024-B alignment
};

// barrier indices ([2] = per stage / per S buffer / per response slot)
enum {
  B_Q = 0,      // Q tile landed (once per item)
  B_QE = 1,     // Q no longer read: the item's last S MMA completed
  B_KF = 2,     // [2] K stage full
  B_VF = 4,     // [2] V stage full
  B_KE = 6,     // [2] K stage consumed by S MMA
  B_VE = 8,     // [2] V stage consumed by P.V MMA
  B_SF = 10,    // [2] S buffer written by the MMA
  B_P = 12,     // [2] P written over S buffer (128 softmax threads)
  B_O = 14,     // [2] O += P_g V_g completed, per S buffer (g & 1)
  B_OE = 16,    // O read out by the epilogue (128 softmax threads, once per item)
  B_CLC = 17,   // [2] work-stealing response landed
  B_CLCE = 19,  // [2] response read by all 6 warps
};

// Persistent via cluster launch control: the grid keeps one CTA per (q tile, head,
// sequence) — the hardware's launch order keeps the q tiles of one (sequence, head)
// together, so their K/V re-reads hit L2 — but a running CTA takes over CTAs that
// have not launched yet (clusterlaunchcontrol.try_cancel) and runs their items back
// to back: the producer loads item k+1's Q and K/V while item k's last tiles and
// epilogue run, so no CTA start-up latency is exposed. All per-tile barrier phases
// run on a CTA-wide tile counter g (stage = g & 1, phase = (g >> 1) & 1).
// Measured (tools/kernel_bench.py, vs one item per CTA): 64 x 128 -12 %, 64 x 512
// -8 %, 16 x 2048 -3 %, 4 x 4096 -5 %, chunked prefill -5..7 %. (The MMA and
// producer roles must stay under elect.sync: with a plain lane test the compiler
// loses the uniform datapath for the UMMA operands and every length got slower.)
#ifdef DS_TRACE
// Timeline tracing (A/B builds only, tools/ab.sh trace "-DDS_TRACE"): clock64 stamps
// of the role events of the CTAs that run on SM 0, read back with
// ds_debug_prefill_trace (not part of the public ABI). Each recording thread owns a
// region and a register counter, so a record is two plain stores (no atomics on
// the timed path).
constexpr int kTrSlots = 8, kTrRecorders = 8, kTrCap = 32768;
__device__ unsigned long long g_pf_trace[kTrSlots * kTrRecorders * kTrCap * 2];
__device__ unsigned int g_pf_slot;
struct Tracer {
  unsigned long long *base = nullptr;
  uint32_t n = 0;
  DS_DEVICE void rec(uint32_t ev, uint32_t cta, uint32_t g) {
    if (base && n < kTrCap) {
      base[2 * n] = clock64();
      base[2 * n + 1] = ((uint64_t)ev << 56) | ((uint64_t)cta << 32) | g;
      ++n;
    }
  }
};
#define TRACE(ev, g) tracer.rec((ev), cta_id, (g))
#else
#define TRACE(ev, g) ((void)0)
#endif
enum { T_SM_WAIT_S = 1, T_SM_GOT_S, T_SM_P_DONE, T_MMA_S, T_MMA_WAIT_P, T_MMA_PV, T_SM_EPI_DONE, T_LD_K, T_LD_V,
       T_SM_EPI_PV, T_EPI_LD = 32 /* 32 + 2*chunk: TMEM chunk loaded; +1: chunk stored */,
       T_SM_WARP_P = 16 /* + warp (< 32) */ };

// Launch order of the work items (q tile i, head h, sequence r): sequences in order,
// their heads in order, and the q tiles of one (sequence, head) adjacent, heaviest
// first (their K/V re-reads hit L2). With a.compact the item space holds only the
// tiles that exist: pref[r] = sum of ceil(len/128) over the sequences before r (built
// in smem once per CTA), so a batch of mixed lengths launches no empty items — each
// costs a persistent CTA ~0.5 us to skip (64 x 128-token prompts launched with a
// 2048-token bound: 85 -> 144 us). Items past the last tile come back as i = -1.
// Without it (num_seqs > kCompactSeqs) the grid is num_q_tiles x n_loc x num_seqs.
DS_DEVICE void item_coords(const PrefillArgs &a, const int *pref, const Band &bd, int item, int &i, int &h,
                           int &r) {
  if (!a.compact) {
    const int Q = a.num_q_tiles, g = item / Q;
    i = Q - 1 - (item - g * Q);
    r = g / a.n_loc;
    h = g - r * a.n_loc;
    return;
  }
  const int n = a.n_loc;
  if (item >= n * pref[a.num_seqs]) {
    i = -1;
    r = h = 0;
    return;
  }
  if (item >= bd.item0) {  // the band: level-major (see Band)
    int k = item - bd.item0, lo = 0, hi = bd.levels - 1;  // smallest level with lvl[level] <= k
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (bd.lvl[mid] <= k) hi = mid;
      else lo = mid + 1;
    }
    i = lo;
    k -= bd.lvl[lo];
    for (int s = 0;; ++s) {  // the level's sequences are a prefix of the length-sorted band
      const int hs = n - bd.hlo[s];
      if (k < hs) {
        r = bd.seq[s];
        h = bd.hlo[s] + k;
        return;
      }
      k -= hs;
    }
  }
  int lo = 0, hi = a.num_seqs - 1;  // largest r with n * pref[r] <= item
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (n * pref[mid] <= item) lo = mid;
    else hi = mid - 1;
  }
  r = lo;
  const int tr = pref[r + 1] - pref[r], k = item - n * pref[r];
  h = k / tr;
  i = tr - 1 - (k - h * tr);
}

// pref[r] = sum_{r' < r} ceil(len_r' / 128), r in [0, num_seqs], by all threads of
// the CTA (per-thread runs, warp shuffle scan, one pass over the warp totals)
DS_DEVICE void build_tile_prefix(const PrefillArgs &a, int *pref, int *warp_tot) {
  const int B = a.num_seqs, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int per = (B + kThreads - 1) / kThreads;
  const int b0 = min(B, t * per), b1 = min(B, b0 + per);
  int sum = 0;
  for (int b = b0; b < b1; ++b) sum += (a.cu_seqlens[b + 1] - a.cu_seqlens[b] + kBM - 1) / kBM;
  int inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < warp; ++w) base += warp_tot[w];
  int run = base + inc - sum;
  for (int b = b0; b < b1; ++b) {
    pref[b] = run;
    run += (a.cu_seqlens[b + 1] - a.cu_seqlens[b] + kBM - 1) / kBM;
  }
  if (t == kThreads - 1) pref[B] = base + inc;
}

// The band (see Band), by one warp once pref is complete: lane t looks at sequence
// num_seqs-1-t; the band takes whole sequences from the end (and the last heads of one
// more) while their K/V bytes (chunked prefill: with the cached prefix) fit the
// budget; ranks by tile count sort them; level counts and their suffix sums give lvl.
DS_DEVICE void build_band(const PrefillArgs &a, const int *pref, Band &bd, int head_dim) {
  const int B = a.num_seqs, n = a.n_loc, lane = threadIdx.x & 31, r = B - 1 - lane;
  const int64_t per_token = 4LL * head_dim;  // K + V bytes of one head
  const int len = r >= 0 ? a.cu_seqlens[r + 1] - a.cu_seqlens[r] : 0;
  const int tr = r >= 0 ? pref[r + 1] - pref[r] : 0;
  // K/V a group re-reads: its own tokens, plus the cached prefix in chunked prefill
  const int64_t kv_len = len + (r >= 0 && a.prefix_lens ? a.prefix_lens[r] : 0);
  const int64_t sb = (int64_t)n * kv_len * per_token;
  int64_t inc = sb;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  const int64_t budget = (int64_t)DS_PF_BAND_MB << 20, before = inc - sb;
  int heads = 0;
  if (r >= 0 && len > 0 && before < budget) heads = (int)min((int64_t)n, (budget - before) / (kv_len * per_token));
  const unsigned in = __ballot_sync(0xffffffffu, heads > 0);  // a prefix of the lanes
  const int nseq = in == 0xffffffffu ? 32 : __ffs(~in) - 1;
  int levels = heads > 0 ? tr : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) levels = max(levels, __shfl_xor_sync(0xffffffffu, levels, o));
  if (nseq == 0 || levels > kBandLevels) {
    if (lane == 0) {
      bd.item0 = n * pref[B];
      bd.levels = 0;
    }
    return;
  }
  int rank = 0, items = heads * tr, cnt_lo = 0, cnt_hi = 0;
  for (int t = 0; t < nseq; ++t) {
    const int tr_t = __shfl_sync(0xffffffffu, tr, t), h_t = __shfl_sync(0xffffffffu, heads, t);
    if (tr_t > tr || (tr_t == tr && t > lane)) ++rank;  // longer first; ties in launch order
    if (tr_t > lane) cnt_lo += h_t;                      // items of level `lane`
    if (tr_t > lane + 32) cnt_hi += h_t;                 // items of level `lane + 32`
  }
  if (lane < nseq) {
    bd.seq[rank] = r;
    bd.hlo[rank] = n - heads;
  }
  // lvl[i] = sum of the level counts above i (suffix sums over lanes, hi levels first)
  int suf_hi = cnt_hi, suf_lo = cnt_lo;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int yh = __shfl_down_sync(0xffffffffu, suf_hi, o), yl = __shfl_down_sync(0xffffffffu, suf_lo, o);
    if (lane + o < 32) {
      suf_hi += yh;
      suf_lo += yl;
    }
  }
  const int tot_hi = __shfl_sync(0xffffffffu, suf_hi, 0);
  bd.lvl[lane + 32] = suf_hi - cnt_hi;
  bd.lvl[lane] = suf_lo - cnt_lo + tot_hi;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) items += __shfl_xor_sync(0xffffffffu, items, o);
  if (lane == 0) {
    bd.item0 = n * pref[B] - items;
    bd.levels = levels;
  }
}

// waits of the producer and MMA threads
DS_DEVICE void ctl_wait(uint64_t *bar, uint32_t parity) {
  if (DS_PF_SLEEP_NS > 0)
    mbar_wait_sleep(bar, parity, DS_PF_SLEEP_NS);
  else
    mbar_wait(bar, parity);
}

// kPush: the fused push migration — every K/V page the kernel writes also goes,
// from the same smem tile, to the destination pool (a peer GPU's pool mapped
// through CUDA IPC, or another pool of this GPU) with a second TMA tensor store.
template <int D, bool kChunked, bool kPush>
__global__ void __launch_bounds__(kThreads, 2)
    prefill_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv,
                   const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_cache,
                   const __grid_constant__ CUtensorMap tm_o, const __grid_constant__ CUtensorMap tm_dst,
                   const PrefillArgs a) {
  using S = Smem<D>;
  constexpr int kChunks = D / 64;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t *smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  const uint32_t sbase = smem_u32(smem);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + S::BAR);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + S::TMEM_SLOT);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int b = 0; b < (int)S::kBars; ++b) {
      const bool per_thread = b == B_P || b == B_P + 1 || b == B_OE;
      mbar_init(&bars[b], per_thread ? 128 : (b == B_CLCE || b == B_CLCE + 1) ? kThreads / 32 : 1);
    }
    fence_barrier_init();
  }
  if (warp == 5) {
    tmem_alloc<kTmemCols>(tmem_slot);
    tmem_relinquish();
  }
  int *pref = reinterpret_cast<int *>(smem + S::PREF);
  Band &band = *reinterpret_cast<Band *>(smem + S::BAND);
  if (a.compact) {
    build_tile_prefix(a, pref, pref + kCompactSeqs + 1);
    __syncthreads();
    // (prompts of at most 2 q tiles have no heavy items to reorder: skip the band)
    if (warp == 0) {
      if (a.num_q_tiles > 2)
        build_band(a, pref, band, D);
      else if (lane == 0)
        band.item0 = a.n_loc * pref[a.num_seqs];
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem + 128;
  if (warp == 4 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_kv);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_cache);
    tma_prefetch_desc(&tm_o);
    if (kPush) tma_prefetch_desc(&tm_dst);
  }

  int item = blockIdx.x;  // current item (linear launch index, see item_coords)
#ifdef DS_TRACE
  const uint32_t cta_id = blockIdx.x;
  Tracer tracer;
  {
    int &tr_slot = *reinterpret_cast<int *>(smem + S::TMEM_SLOT + 8);  // spare bytes of the slot
    if (threadIdx.x == 0) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      tr_slot = smid == 0 ? (int)atomicAdd(&g_pf_slot, 1u) : -1;
    }
    __syncthreads();
    const int rcd = warp < 4 ? warp : warp == 4 ? 4 : 5;  // softmax warps 0-3, producer, MMA
    if (tr_slot >= 0 && tr_slot < kTrSlots && (lane == 0 || warp >= 4))
      tracer.base = g_pf_trace + ((size_t)(tr_slot * kTrRecorders + rcd) * kTrCap) * 2;
  }
#endif
  uint32_t g0 = 0;  // kv tiles of earlier items (CTA-wide tile counter)
  uint32_t it = 0;  // non-empty items before the current one
  bool store_pending = false;  // producer: paged TMA stores may still read a stage
  for (uint32_t q = 0;; ++q) {
    if (a.persistent && warp == 4 && lane == 0) {  // ask for the next item now; the answer is needed at the end
      if (q >= 2) mbar_wait(&bars[B_CLCE + (q & 1)], ((q >> 1) - 1) & 1);
      fence_proxy_async_smem();  // the generic reads of this slot precede the async write
      mbar_arrive_expect_tx(&bars[B_CLC + (q & 1)], 16);
      clc_try_cancel(sbase + S::CLC + (q & 1) * 16, &bars[B_CLC + (q & 1)]);
    }
    int i, h, r;
    item_coords(a, pref, band, item, i, h, r);
    const int seq_start = a.cu_seqlens[r];
    const int len = a.cu_seqlens[r + 1] - seq_start;
    if (i >= 0 && i * kBM < len) {
      // chunked prefill (NEXT-3): the sequence already holds c0 tokens in the paged
      // cache; kv tiles [0, npt) are that prefix (read from the pages), tiles
      // [npt, ntiles) are the chunk's own keys 0 .. 2i+1 (64 keys each; the second
      // diagonal tile is skipped when it lies wholly past the end of the chunk)
      const int c0 = kChunked ? a.prefix_lens[r] : 0;
      const int npt = kChunked ? (c0 + kBN - 1) / kBN : 0;
      const int ntiles = npt + 2 * i + 1 + (len - i * kBM > kBN ? 1 : 0);
      const uint32_t gl = g0 + ntiles - 1;  // last tile of this item

      if (warp == 4) {
        // ------------------------------------------------------------ producer
        __syncwarp();  // elect.sync needs the whole warp converged (lane 0 issued the CLC request)
        if (elect_one()) {
          if (it > 0) ctl_wait(&bars[B_QE], (it - 1) & 1);  // the previous item's S MMAs are done with Q
          mbar_arrive_expect_tx(&bars[B_Q], S::kQTile);
#pragma unroll
          for (int c = 0; c < kChunks; ++c)
            tma_load_3d(smem + S::Q + c * kChunkBytes128, &tm_q, &bars[B_Q], c * 64, h, seq_start + i * kBM);
          if (store_pending) {  // the previous item's paged stores read the stages we refill now
            bulk_wait_group_read0();
            store_pending = false;
          }
          const int32_t *btr = a.block_table + (size_t)r * a.max_blocks;
          for (int j = 0; j < ntiles; ++j) {
            const uint32_t g = g0 + j;
            const int st = g & 1;
            const uint32_t ph_free = ((g >> 1) - 1) & 1;  // release of tile g-2 from this stage
            if (kChunked && j < npt) {
              // prefix tile: 4 pages of 16 cached tokens straight from the pool. A tail
              // tile with np < 4 prefix pages fills its remaining page slots with its
              // last prefix page again: their keys are masked (p = 0 or ~2^-126), but
              // the V rows still enter the P.V MMA, so they must be finite — stale smem
              // (e.g. NaN patterns left by an earlier kernel) would poison the row.
              const int p0 = 4 * j, np = min(4, (c0 + 15) / 16 - p0);
              const uint32_t bytes = 4u * 16 * D * 2;
#pragma unroll
              for (int kv = 0; kv < 2; ++kv) {
                if (g >= 2) ctl_wait(&bars[(kv ? B_VE : B_KE) + st], ph_free);
                uint64_t *full = &bars[(kv ? B_VF : B_KF) + st];
                mbar_arrive_expect_tx(full, bytes);
                for (int p = 0; p < 4; ++p)
#pragma unroll
                  for (int c = 0; c < kChunks; ++c)
                    tma_load_4d(smem + (kv ? S::V0 : S::K0) + st * S::kKVTile + c * kChunkBytes64 + p * 16 * 128,
                                &tm_cache, full, c * 64, 0, h,
                                (a.layer * 2 + kv) * a.num_blocks + btr[p0 + min(p, np - 1)]);
              }
              continue;
            }
            const int kv0 = seq_start + (j - npt) * kBN;
            if (g >= 2) ctl_wait(&bars[B_KE + st], ph_free);  // S_{g-2} has consumed the K stage
            mbar_arrive_expect_tx(&bars[B_KF + st], S::kKVTile);
#pragma unroll
            for (int c = 0; c < kChunks; ++c)
              tma_load_3d(smem + S::K0 + st * S::kKVTile + c * kChunkBytes64, &tm_kv, &bars[B_KF + st], c * 64, h,
                          kv0);
            TRACE(T_LD_K, g);
            if (g >= 2) ctl_wait(&bars[B_VE + st], ph_free);  // PV_{g-2} has consumed the V stage
            mbar_arrive_expect_tx(&bars[B_VF + st], S::kKVTile);
#pragma unroll
            for (int c = 0; c < kChunks; ++c)
              tma_load_3d(smem + S::V0 + st * S::kKVTile + c * kChunkBytes64, &tm_v, &bars[B_VF + st], c * 64, h,
                          kv0);
            TRACE(T_LD_V, g);
          }
          // a3: the diagonal K/V tiles 2i (pages 8i..8i+3) and 2i+1 (8i+4..8i+7) -> paged
          // cache (chunked mode appends the chunk with ds' append kernel instead: the
          // chunk need not start on a page boundary)
          const int npg = kChunked ? 0 : min(8, (len - i * kBM + 15) >> 4);
          const int32_t *bt = btr + i * 8;
          const int32_t *dbt = kPush ? a.dst_block_table + (size_t)r * a.dst_max_blocks + i * 8 : nullptr;
          for (int t = npt + 2 * i; npg > 0 && t < ntiles; ++t) {
            const uint32_t g = g0 + t;
            const int st = g & 1;
            ctl_wait(&bars[B_KF + st], (g >> 1) & 1);
            ctl_wait(&bars[B_VF + st], (g >> 1) & 1);
            for (int p = (t - npt - 2 * i) * 4; p < min(npg, (t - npt - 2 * i) * 4 + 4); ++p) {
              const int blk = bt[p];
              const int dblk = kPush ? dbt[p] : 0;
#pragma unroll
              for (int kv = 0; kv < 2; ++kv)
#pragma unroll
                for (int c = 0; c < kChunks; ++c) {
                  const uint8_t *src =
                      smem + (kv ? S::V0 : S::K0) + st * S::kKVTile + c * kChunkBytes64 + (p & 3) * 16 * 128;
                  if (!kPush || a.write_local)
                    tma_store_4d(&tm_cache, src, c * 64, 0, h, (a.layer * 2 + kv) * a.num_blocks + blk);
                  if (kPush)
                    tma_store_4d(&tm_dst, src, c * 64, 0, a.dst_head0 + h,
                                 (a.dst_layer * 2 + kv) * a.dst_num_blocks + dblk);
                }
            }
          }
          if (npg > 0) {
            bulk_commit_group();
            store_pending = true;
          }
        }
        __syncwarp();
      } else if (warp == 5) {
        // ------------------------------------------------------------ MMA issuer
        // Order per tile g: S_g = Q K_g^T, then O += P_{g-1} V_{g-1} (within an item).
        // P.V completions are tracked per S buffer (B_O[g & 1]) for the softmax warps;
        // this thread never waits on them (in-order tcgen05.mma execution orders every
        // S_g after the P_{g-2} V_{g-2} that reads its buffer).
        __syncwarp();
        if (elect_one()) {
          constexpr uint32_t idesc_s = idesc_bf16_f32(kBM, kBN, 0, 0);
          constexpr uint32_t idesc_o = idesc_bf16_f32(kBM, D, 0, 1);
          ctl_wait(&bars[B_Q], it & 1);
          auto issue_pv = [&](uint32_t g, bool first) {  // O (+)= P_g V_g
            const int st = g & 1;
            TRACE(T_MMA_WAIT_P, g);
            ctl_wait(&bars[B_P + st], (g >> 1) & 1);
            ctl_wait(&bars[B_VF + st], (g >> 1) & 1);
            if (first && it > 0) ctl_wait(&bars[B_OE], (it - 1) & 1);  // previous item's O read out
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < kBN / 16; ++kk)  // 16 keys = 8 packed P columns per step
              umma_ts(tO, tmem + st * kBN + kk * 8,
                      smem_desc_sw128(sbase + S::V0 + st * S::kKVTile + kk * 16 * 128, kChunkBytes64, 1024),
                      idesc_o, (!first || kk > 0));
            umma_commit(&bars[B_O + st]);
            umma_commit(&bars[B_VE + st]);
            TRACE(T_MMA_PV, g);
          };
          for (int j = 0; j < ntiles; ++j) {
            const uint32_t g = g0 + j;
            const int st = g & 1;
            ctl_wait(&bars[B_KF + st], (g >> 1) & 1);
            // S buffer st still holds P_{g-2}, read by P_{g-2} V_{g-2}: that MMA was
            // issued before this one by this thread, and tcgen05.mma ops of one thread
            // execute in issue order, so S_g cannot overwrite P_{g-2} before it is read
            // (no wait: the tensor pipe never drains between tiles)
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
              umma_ss(tmem + st * kBN,
                      smem_desc_sw128(sbase + S::Q + (kk >> 2) * kChunkBytes128 + (kk & 3) * 32, 16, 1024),
                      smem_desc_sw128(sbase + S::K0 + st * S::kKVTile + (kk >> 2) * kChunkBytes64 + (kk & 3) * 32,
                                      16, 1024),
                      idesc_s, kk > 0);
            umma_commit(&bars[B_SF + st]);
            umma_commit(&bars[B_KE + st]);
            TRACE(T_MMA_S, g);
            if (j == ntiles - 1) umma_commit(&bars[B_QE]);
            if (j >= 1) issue_pv(g - 1, j == 1);
          }
          issue_pv(gl, ntiles == 1);
        }
        __syncwarp();
      } else {
        // ------------------------------------------------------------ softmax warps 0-3
        const int row = threadIdx.x;  // TMEM lane == q row within the tile
        const int q_pos = i * kBM + row;
        const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
        const float sl2 = a.scale_log2;
        float m = -__int_as_float(0x7f800000), l = 0.f;
        // P_k V_k complete (B_O[k & 1]). Parity waits are exact only if this thread
        // has seen the previous phase of that barrier and the next cannot complete yet:
        // it waits on P_{g-2} V_{g-2} at every tile g before publishing P_g (so every
        // phase of both barriers in order, one tile of slack), and on P_{g-1} V_{g-1}
        // only to rescale O, and on the last P.V in the epilogue.
        auto wait_pv = [&](uint32_t k) { mbar_wait(&bars[B_O + (k & 1)], (k >> 1) & 1); };
        for (int j = 0; j < ntiles; ++j) {
          const uint32_t g = g0 + j;
          const int st = g & 1;
          if (threadIdx.x == 0) TRACE(T_SM_WAIT_S, g);
          mbar_wait(&bars[B_SF + st], (g >> 1) & 1);
          if (threadIdx.x == 0) TRACE(T_SM_GOT_S, g);
          tc_fence_after();
          uint32_t sr[2][32];
          tmem_ld32(tmem + lane_off + st * kBN, sr[0]);
          tmem_ld32(tmem + lane_off + st * kBN + 32, sr[1]);
          tmem_wait_ld();
          // row max on the raw scores (scale > 0 preserves order); prefix tiles: keys at
          // or beyond c0 are not cached yet (masked); chunk tiles: causal within the
          // chunk (key position > query position masked) — only the diagonal tiles
          // row max on the raw scores; four independent 3-input max chains (the
          // softmax is latency-bound with two softmax warps per SMSP, so ILP matters)
          const float ninf = -__int_as_float(0x7f800000);
          float mxv[4] = {ninf, ninf, ninf, ninf};
          const bool prefix_tail = kChunked && j == npt - 1 && (c0 % kBN) != 0;
          if (prefix_tail || j - npt >= 2 * i) {
            const int lim = prefix_tail ? c0 - 1 - j * kBN : q_pos - (j - npt) * kBN;  // last visible column
#pragma unroll
            for (int cc = 0; cc < 2; ++cc)
#pragma unroll
              for (int e = 0; e < 32; ++e)
                if (cc * 32 + e > lim) sr[cc][e] = 0xff800000u;  // -inf
          }
#pragma unroll
          for (int cc = 0; cc < 2; ++cc)
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              float &mk = mxv[(cc * 16 + e / 2) & 3];
              mk = fmaxf(mk, fmaxf(__uint_as_float(sr[cc][e]), __uint_as_float(sr[cc][e + 1])));
            }
          const float mx = fmaxf(fmaxf(mxv[0], mxv[1]), fmaxf(mxv[2], mxv[3]));
          // Conditional rescaling: the exponent base m only moves when this tile's row
          // max exceeds it by more than kRescaleLog2 (p <= 2^8 in between, exact in
          // fp32/bf16 range); softmax is invariant to the base, so the result is the
          // same function — most tiles then skip the O rescale AND the wait on the
          // previous P.V MMA.
          const float m_tile = mx * sl2;
          const bool grow = m_tile > m + kRescaleLog2;
          const float m_new = grow ? m_tile : m;
          const float alpha = grow ? ex2(m - m_new) : 1.f;
          // p = 2^(s*scale*log2e - m): one FFMA + one MUFU ex2 per element; P is rounded
          // to bf16 (the P operand of the P.V MMA), the row sum stays fp32.
          uint32_t pk[32];
          const uint64_t sl2x2 = f2_pack(sl2, sl2), negm2 = f2_pack(-m_new, -m_new);
          uint64_t rs2[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) rs2[u] = f2_pack(0.f, 0.f);
#pragma unroll
          for (int cc = 0; cc < 2; ++cc)
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              // exponent arguments two at a time (FFMA2); kPolyEvery-th exponentials on
              // the FMA pipe, the rest on MUFU; the fp32 row sum two at a time (FADD2)
              // in four independent accumulators
              float x0, x1;
              f2_unpack(f2_fma(f2_pack(__uint_as_float(sr[cc][e]), __uint_as_float(sr[cc][e + 1])), sl2x2, negm2),
                        x0, x1);
#if DS_PF_FAKE_EXP  // timing experiment only (wrong results): exp replaced by a clamp
              const float p0 = fminf(x0, 1.f), p1 = fminf(x1, 1.f);
#else
              const float p0 = (e % kPolyEvery) == 0 ? ex2_poly(x0) : ex2(x0);
              const float p1 = ((e + 1) % kPolyEvery) == 0 ? ex2_poly(x1) : ex2(x1);
#endif
              uint64_t &rk = rs2[(cc * 16 + e / 2) & 3];
              rk = f2_add(rk, f2_pack(p0, p1));
              pk[cc * 16 + e / 2] = pack_bf16(p0, p1);
            }
          float rs0, rs1;
          f2_unpack(f2_add(f2_add(rs2[0], rs2[1]), f2_add(rs2[2], rs2[3])), rs0, rs1);
          l = l * alpha + (rs0 + rs1);
          m = m_new;
          if (j > 0 && __any_sync(0xffffffffu, grow)) {  // warp-uniform O rescale, only when a base moved
            wait_pv(g - 1);                              // O is not in use by P_{g-1} V_{g-1} any more
            tc_fence_after();
#pragma unroll
            for (int cc = 0; cc < D / 32; ++cc) {
              uint32_t o[32];
              tmem_ld32(tO + lane_off + cc * 32, o);
              tmem_wait_ld();
              const uint64_t a2 = f2_pack(alpha, alpha), z2 = f2_pack(0.f, 0.f);
#pragma unroll
              for (int e = 0; e < 32; e += 2) {
                float lo, hi;
                f2_unpack(f2_fma(f2_pack(__uint_as_float(o[e]), __uint_as_float(o[e + 1])), a2, z2), lo, hi);
                o[e] = __float_as_uint(lo);
                o[e + 1] = __float_as_uint(hi);
              }
              tmem_st32(tO + lane_off + cc * 32, o);
            }
          }
          if (g >= 2) wait_pv(g - 2);  // keep the observed phases contiguous (normally long complete)
          // P (bf16 pairs, low half = even key) over the first 32 columns of S buffer st
          tmem_st32(tmem + lane_off + st * kBN, pk);
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&bars[B_P + st]);
          if (lane == 0) TRACE(T_SM_WARP_P + warp, g);
        }
        // epilogue: O / l -> bf16 -> global. Each warp stages its 32 rows x 32 dims
        // chunk in smem (2 KiB in the 64-B swizzle of the TMA box: conflict-free
        // STS) and one lane TMA-stores it: per-thread row stores (32 rows, 10 KB
        // apart, per instruction) took ~5000 cycles per item on the LSU path. A
        // warp whose rows run past the sequence end stores its valid rows directly
        // (a TMA box would overwrite the next sequence's rows).
        wait_pv(gl);
        if (threadIdx.x == 0) TRACE(T_SM_EPI_PV, gl);
        tc_fence_after();
        const float inv_l = 1.f / l;
        const int row0 = i * kBM + warp * 32;
        const bool boxed = row0 + 32 <= len;  // warp-uniform
        uint8_t *stg = smem + S::OST + warp * 2048;
        uint16_t *orow = reinterpret_cast<uint16_t *>(a.out) + ((size_t)(seq_start + q_pos) * a.n_loc + h) * D;
        const uint64_t inv2 = f2_pack(inv_l, inv_l), zero2 = f2_pack(0.f, 0.f);
        auto store_chunk = [&](const uint32_t (&o)[32], int cc) {
          uint4 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float lo, hi;
              f2_unpack(f2_fma(f2_pack(__uint_as_float(o[u * 8 + 2 * e]), __uint_as_float(o[u * 8 + 2 * e + 1])),
                               inv2, zero2),
                        lo, hi);
              w[e] = pack_bf16(lo, hi);
            }
            v[u] = make_uint4(w[0], w[1], w[2], w[3]);
          }
          if (boxed) {
            // (a second staging buffer per warp measured no faster; per-thread 32-B
            // STG.256 row stores 1-5 % slower, profiles/r02/prefill_band_ab)
            if (lane == 0) bulk_wait_group_read0();  // the previous chunk's store has read the buffer
            __syncwarp();
#pragma unroll
            for (int u = 0; u < 4; ++u)  // SWIZZLE_64B layout of the box: conflict-free STS
              *reinterpret_cast<uint4 *>(stg + lane * 64 + ((u ^ ((lane >> 1) & 3)) << 4)) = v[u];
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_3d(&tm_o, stg, cc * 32, h, seq_start + row0);
              bulk_commit_group();
            }
          } else if (q_pos < len) {
#pragma unroll
            for (int u = 0; u < 4; ++u) *reinterpret_cast<uint4 *>(orow + cc * 32 + u * 8) = v[u];
          }
          if (threadIdx.x == 0) TRACE(T_EPI_LD + 2 * cc + 1, gl);
        };
        // TMEM loads run one chunk ahead of the stores (two register buffers)
        uint32_t oa[32], ob[32];
        tmem_ld32(tO + lane_off, oa);
        tmem_ld32(tO + lane_off + 32, ob);
        tmem_wait_ld();
        if (threadIdx.x == 0) TRACE(T_EPI_LD, gl);
        store_chunk(oa, 0);
        if constexpr (D == 128) {
          tmem_ld32(tO + lane_off + 64, oa);
          store_chunk(ob, 1);
          tmem_wait_ld();
          tmem_ld32(tO + lane_off + 96, ob);
          store_chunk(oa, 2);
          tmem_wait_ld();
          store_chunk(ob, 3);
        } else {
          store_chunk(ob, 1);
        }
        tc_fence_before();
        mbar_arrive(&bars[B_OE]);  // the next item's first P.V may overwrite O
        if (threadIdx.x == 0) TRACE(T_SM_EPI_DONE, gl);
      }
      g0 += ntiles;
      ++it;
    }
    if (!a.persistent) break;
    // next item: the work-stealing response (every warp reads it, then releases the slot)
    mbar_wait(&bars[B_CLC + (q & 1)], (q >> 1) & 1);
    int nx, ny, nz;
    const bool more = clc_query(smem + S::CLC + (q & 1) * 16, nx, ny, nz);
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars[B_CLCE + (q & 1)]);
    if (!more) break;
    item = nx;
  }

  if (warp < 4 && lane == 0) bulk_wait_group0();  // the epilogue's O stores are complete
  if (warp == 4 && lane == 0 && g0 > 0) {
    // observe the last stage releases too (every mbarrier phase is waited on; also
    // guarantees the final MMAs have drained before the CTA retires)
    for (uint32_t t = g0 >= 2 ? g0 - 2 : 0; t < g0; ++t) {
      mbar_wait(&bars[B_KE + (t & 1)], (t >> 1) & 1);
      mbar_wait(&bars[B_VE + (t & 1)], (t >> 1) & 1);
    }
    bulk_wait_group_read0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

template <int D, bool C, bool P>
static cudaError_t set_prefill_smem_once() {
  static cudaError_t st = cudaFuncSetAttribute(prefill_kernel<D, C, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)Smem<D>::ALLOC);
  return st;
}

template <int D, bool C, bool P>
static cudaError_t launch_one(const PrefillArgs &a, const CUtensorMap &tq, const CUtensorMap &tk,
                              const CUtensorMap &tv, const CUtensorMap &tc, const CUtensorMap &to,
                              const CUtensorMap &tdst, cudaStream_t stream) {
  cudaError_t e = set_prefill_smem_once<D, C, P>();
  if (e != cudaSuccess) return e;
  prefill_kernel<D, C, P><<<(unsigned)a.grid_items, kThreads, Smem<D>::ALLOC, stream>>>(
      tq, tk, tv, tc, to, tdst, a);
  return cudaGetLastError();
}

}  // namespace

#ifdef DS_TRACE
// copies the whole trace buffer (zero clock = empty record) and optionally clears it
extern "C" __attribute__((visibility("default"))) int ds_debug_prefill_trace(unsigned long long *host, int cap_records,
                                                                             int reset) {
  const int total = kTrSlots * kTrRecorders * kTrCap;
  cudaDeviceSynchronize();
  if (host && cap_records >= total) cudaMemcpyFromSymbol(host, g_pf_trace, sizeof(g_pf_trace));
  if (reset) {
    void *p = nullptr;
    cudaGetSymbolAddress(&p, g_pf_trace);
    cudaMemset(p, 0, sizeof(g_pf_trace));
    const unsigned int z = 0;
    cudaMemcpyToSymbol(g_pf_slot, &z, sizeof(z));
    cudaDeviceSynchronize();
  }
  return total;
}
#endif

void prefill_set_grid(PrefillArgs &a, int64_t total_tokens) {
  a.compact = a.num_seqs <= kCompactSeqs;
  a.grid_items = a.compact ? (int64_t)a.n_loc * ((total_tokens + (int64_t)(kBM - 1) * a.num_seqs) / kBM)
                           : (int64_t)a.num_q_tiles * a.n_loc * a.num_seqs;
}

bool prefill_persistent(int /*max_len*/) {
  // always (faster at every measured length); DS_PREFILL_PERSISTENT=0 runs one
  // item per CTA for A/B measurements and the parity test of that mode
  static const bool on = [] {
    const char *e = getenv("DS_PREFILL_PERSISTENT");
    return e ? atoi(e) != 0 : true;
  }();
  return on;
}

size_t prefill_smem_bytes(int head_dim) {
  return head_dim == 128 ? Smem<128>::ALLOC : Smem<64>::ALLOC;
}

cudaError_t launch_prefill(const PrefillArgs &a, const CUtensorMap &tm_q, const CUtensorMap &tm_k,
                           const CUtensorMap &tm_v, const CUtensorMap &tm_cache, const CUtensorMap &tm_o,
                           const CUtensorMap *tm_dst, int head_dim, cudaStream_t stream) {
  const bool chunked = a.prefix_lens != nullptr;
  if (tm_dst) {  // fused push (regular prefill only)
    if (chunked) return cudaErrorInvalidValue;
    return head_dim == 128 ? launch_one<128, false, true>(a, tm_q, tm_k, tm_v, tm_cache, tm_o, *tm_dst, stream)
                           : launch_one<64, false, true>(a, tm_q, tm_k, tm_v, tm_cache, tm_o, *tm_dst, stream);
  }
  if (head_dim == 128)
    return chunked ? launch_one<128, true, false>(a, tm_q, tm_k, tm_v, tm_cache, tm_o, tm_o, stream)
                   : launch_one<128, false, false>(a, tm_q, tm_k, tm_v, tm_cache, tm_o, tm_o, stream);
  return chunked ? launch_one<64, true, false>(a, tm_q, tm_k, tm_v, tm_cache, tm_o, tm_o, stream)
                 : launch_one<64, false, false>(a, tm_q, tm_k, tm_v, tm_cache, tm_o, tm_o, stream);
}

}  // namespace ds
