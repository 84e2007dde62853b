// decode.cu — a7 + a8: one decode step of one layer over a paged KV cache.
//
// PAPER.md P:233 (decode generates one token at a time reusing the KV cache),
// P:237 (batching), P:696-698 (decode attention is memory-bound: it streams the
// whole cached K/V once per step). Reading R9: the new token's K/V are appended
// at position c before attending, so the step attends c+1 tokens.
//
// Two kernels, one computation (launch_decode picks; decode_uses_pairs):
//  * decode_kernel (the default), below;
//  * decode_pairs_kernel (opt-in, DS_DEC_PAIRS): each (sequence, head) pair is
//    streamed by one CTA, its 16 warps taking the pair's pages round-robin, the
//    warps' partials merged in shared memory; CTAs take pairs from a counter, so
//    the launch ends within about one pair's streaming time (see its comment).
//
// B200 design (HBM-bound; no tensor cores — every cached element is used once):
//  * persistent grid of one 16-warp CTA per SM; the (sequence, head, page) space
//    is flattened and cut into equal contiguous page ranges, one per warp, so
//    every warp streams the same number of pages whatever the batch and length
//    mix (no wave tail, no idle SMs on ragged batches);
//  * each warp keeps its own ring of 4 KiB page slots (K page, V page, ...)
//    filled by 1-D TMA bulk copies (cp.async.bulk, mbarrier complete_tx) issued
//    by one lane ahead of the consumer: 16 warps x 3 x 4 KiB = 192 KiB per SM;
//  * consumer: a 16-token page is read from smem by TPG = head_dim/8 lanes per
//    token row (16-B vectors, conflict-free); the q.k partials are
//    transpose-reduced so every lane ends with ONE token's score (one exp per
//    token, not per lane), the page max/sum are warp reductions, the running
//    (m, l) is warp-uniform with a lazy rescale, and each token's weight is
//    shuffled back to the lanes that hold its V row; full pages take a
//    mask-free path, only the page holding position c is masked;
//  * a warp's range covers whole (seq, head) pairs — written straight to `out`
//    — plus at most a partial first and a partial last pair, whose (m, l, o)
//    go to the workspace; the warp that publishes a pair's last partial merges
//    them (a8, fused; atomic ticket per pair, self-resetting);
//  * launched with programmatic dependent launch (griddepcontrol.wait before
//    the first read), so launch latency overlaps the previous kernel's tail;
//    with DS_DECODE_EARLY_KV the lengths, table and first pages are read before
//    that wait (the caller vouches the previous kernel does not write them), so
//    the opening page burst overlaps the previous kernel's drain;
//  * the append (i) is fused: the warp that owns the page holding position c
//    stores k_new/v_new into it and uses them from global memory for token c.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace ds {

namespace {

#ifndef DS_DEC_WARPS
#define DS_DEC_WARPS 16
#endif
#ifndef DS_DEC_SLOTS
#define DS_DEC_SLOTS 3
#endif
#ifndef DS_DEC_CTAS
#define DS_DEC_CTAS 1
#endif
constexpr int kWarps = DS_DEC_WARPS;           // consumer warps per CTA
constexpr int kCtasPerSm = DS_DEC_CTAS;        // resident CTAs per SM (A/B: 2 x 8 warps)
constexpr int kWarpsPerSm = kWarps * kCtasPerSm;
#ifndef DS_DEC_DYN_PCT
#define DS_DEC_DYN_PCT 10
#endif
#ifndef DS_DEC_CHUNK
#define DS_DEC_CHUNK 8
#endif
// Work split: each warp first streams a static contiguous page range; the last
// kDynPct % of the pages are cut into chunks of kChunkPages that warps take
// dynamically (one atomic counter) when their static range is done, so the warps
// that stream slower (DRAM latency differs per SM) no longer set the launch's end.
constexpr int kDynPct = DS_DEC_DYN_PCT;
// below kDynPctSwitch pages per warp the dynamic share is kDynPctLow %: measured in
// bench.py's power-capped step (config 2, B = 128, ~75 pages per warp) 7 % x 8-page
// chunks beat 10 % (216.4 vs 220.1 us per launch; 5 %: 217.9, 3 %: 224.4, 0 %: 222.5,
// 15-20 %: 220.0-220.9, 4-page chunks 223-224), while at B = 256 (~150 pages per
// warp) 10 % stays best (sustained: 427.3 vs 429.4 us at 7 %; equal at B = 192,
// ~112 pages per warp). profiles/r02/decode_dyn_share_ab.txt
#ifndef DS_DEC_DYN_PCT_LOW
#define DS_DEC_DYN_PCT_LOW 7
#endif
constexpr int kDynPctLow = DS_DEC_DYN_PCT_LOW;
constexpr int kDynPctSwitch = 112;
constexpr int kChunkPages = DS_DEC_CHUNK;
#ifndef DS_DEC_DYN_MINPW
#define DS_DEC_DYN_MINPW 64
#endif
constexpr int kDynMinPagesPerWarp = DS_DEC_DYN_MINPW;
// range queue entries per warp (the producer is < 2 pages ahead, so 2 would do; 3 lets
// two 8-warp CTAs fit one SM's 228 KiB)
constexpr int kRangeQ = kCtasPerSm > 1 ? 3 : 4;
constexpr int kMaxSeqs = kDecodeMaxSeqs;
constexpr float kNegInf = -__builtin_huge_valf();

template <int D>
struct DecCfg {
  static constexpr int kPageBytes = 16 * D * 2;         // one K or V page of one head
  static constexpr int kSlots = D == 128 ? DS_DEC_SLOTS : 2 * DS_DEC_SLOTS;  // half-stages per warp ring
  static constexpr int kRingBytes = kWarps * kSlots * kPageBytes;
  static constexpr int kPrefixOff = kRingBytes;          // int[kMaxSeqs + 1]
  static constexpr int kRangeOff = (kPrefixOff + (kMaxSeqs + 1) * 4 + 7) & ~7;  // int64[kWarps][kRangeQ][3]
  static constexpr int kDoneOff = kRangeOff + kWarps * kRangeQ * 3 * 8;  // int: warps of this CTA done
  static constexpr int kBarOff = kDoneOff + 8;
  static constexpr int kSmem = kBarOff + kWarps * kSlots * 8;
};

// the consumer's wait for a page slot (A/B knob DS_DEC_WAIT_NS: > 0 adds a suspend-
// time hint, so waiting lanes sleep instead of spinning)
#ifndef DS_DEC_WAIT_NS
#define DS_DEC_WAIT_NS 0
#endif
// the ring's copies and barriers by 32-bit shared-window address, computed once per
// warp (the generic -> shared conversion per call cost a few instructions per issue)
DS_DEVICE void expect_tx_s(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
DS_DEVICE void bulk_g2s_s(uint32_t dst, const void *gsrc, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(reinterpret_cast<uint64_t>(gsrc)), "r"(bytes), "r"(bar)
               : "memory");
}
DS_DEVICE void page_wait(uint64_t *bar, uint32_t parity) {
  if (DS_DEC_WAIT_NS > 0)
    mbar_wait_sleep(bar, parity, DS_DEC_WAIT_NS);
  else
    mbar_wait(bar, parity);
}

// f32 = bf16 * bf16 + f32 in one instruction (sm_100 FHFMA.BF16, operands read
// straight from either half of a packed register; the bf16 x bf16 product is exact)
DS_DEVICE float fma_bf16(uint16_t a, uint16_t b, float c) {
  float d;
  asm("fma.rn.f32.bf16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
  return d;
}
DS_DEVICE void halves(uint32_t x, uint16_t &lo, uint16_t &hi) {
  asm("mov.b32 {%0, %1}, %2;" : "=h"(lo), "=h"(hi) : "r"(x));
}

// q.k over 8 dims, bf16 q and k, fp32 accumulation in two chains
DS_DEVICE float dot8(const uint4 &q, const uint4 &k) {
  uint16_t q0, q1, q2, q3, q4, q5, q6, q7, k0, k1, k2, k3, k4, k5, k6, k7;
  halves(q.x, q0, q1); halves(q.y, q2, q3); halves(q.z, q4, q5); halves(q.w, q6, q7);
  halves(k.x, k0, k1); halves(k.y, k2, k3); halves(k.z, k4, k5); halves(k.w, k6, k7);
  float s = fma_bf16(q0, k0, 0.f), t = fma_bf16(q1, k1, 0.f);
  s = fma_bf16(q2, k2, s); t = fma_bf16(q3, k3, t);
  s = fma_bf16(q4, k4, s); t = fma_bf16(q5, k5, t);
  s = fma_bf16(q6, k6, s); t = fma_bf16(q7, k7, t);
  return s + t;
}

// acc += p * v over 8 dims (fp32 weight: rounding p to bf16 for FHFMA measured
// no faster and costs accuracy)
#ifndef DS_DEC_FFMA2
#define DS_DEC_FFMA2 1
#endif
DS_DEVICE void axpy8(float (&acc)[8], float p, const uint4 &v) {
  // two dims per FFMA2 (packed fp32x2, bitwise the same as two FFMAs): 32 fewer
  // instructions per page; measured neutral in the bench step (223.4 vs 223.6 us)
  if (DS_DEC_FFMA2) {
    const uint64_t p2 = f2_pack(p, p);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float lo, hi;
      f2_unpack(f2_fma(p2, f2_pack(bf16lo(w[k]), bf16hi(w[k])), f2_pack(acc[2 * k], acc[2 * k + 1])), lo, hi);
      acc[2 * k] = lo;
      acc[2 * k + 1] = hi;
    }
    return;
  }
  acc[0] = fmaf(p, bf16lo(v.x), acc[0]);
  acc[1] = fmaf(p, bf16hi(v.x), acc[1]);
  acc[2] = fmaf(p, bf16lo(v.y), acc[2]);
  acc[3] = fmaf(p, bf16hi(v.y), acc[3]);
  acc[4] = fmaf(p, bf16lo(v.z), acc[4]);
  acc[5] = fmaf(p, bf16hi(v.z), acc[5]);
  acc[6] = fmaf(p, bf16lo(v.w), acc[6]);
  acc[7] = fmaf(p, bf16hi(v.w), acc[7]);
}

// weight of a partial with running max m against merged max mm (0 if empty)
DS_DEVICE float rescale(float m, float mm) { return m == kNegInf ? 0.f : ex2(m - mm); }

__host__ __device__ inline int npages_of(int c) { return (c + 1 + 15) >> 4; }

// page range [B_w, B_{w+1}) of warp w out of W over P pages
__host__ __device__ inline int64_t range_begin(int64_t w, int64_t W, int64_t P) { return w * P / W; }

// exclusive prefix of pages per sequence: prefix[b] = sum_{b' < b} npages(b').
// Thread t sums a contiguous run of sequences; the runs are scanned with warp
// shuffles and one pass over the kWarps warp totals (no serial loop over threads).
DS_DEVICE void build_prefix(const int32_t *cache_lens, int B, int *prefix) {
  __shared__ int warp_total[kWarps];
  const int T = blockDim.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int per = (B + T - 1) / T;
  const int b0 = min(B, t * per), b1 = min(B, b0 + per);
  int s = 0;
  for (int b = b0; b < b1; ++b) s += npages_of(cache_lens[b]);
  int inc = s;  // inclusive scan within the warp
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) warp_total[warp] = inc;
  __syncthreads();
  int base = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) base += w < warp ? warp_total[w] : 0;
  int run = base + inc - s;
  if (t == T - 1) prefix[B] = base + inc;
  for (int b = b0; b < b1; ++b) {
    prefix[b] = run;
    run += npages_of(cache_lens[b]);
  }
  __syncthreads();
}

// flattened page x -> (b, h, p); order (b, h, p): the pages of head h of
// sequence b are contiguous in the flattened space.
struct PagePos {
  int b, h, p, npg;
};
DS_DEVICE PagePos locate(int64_t x, const int *prefix, int B, int n) {
  int lo = 0, hi = B - 1;  // largest b with n*prefix[b] <= x
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((int64_t)n * prefix[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  const int npg = prefix[lo + 1] - prefix[lo];
  const int64_t off = x - (int64_t)n * prefix[lo];
  return {lo, (int)(off / npg), (int)(off % npg), npg};
}
DS_DEVICE void advance(PagePos &q, const int *prefix, int n) {
  if (++q.p == q.npg) {
    q.p = 0;
    if (++q.h == n) {
      q.h = 0;
      ++q.b;
      q.npg = prefix[q.b + 1] - prefix[q.b];
    }
  }
}

// owner warp of flattened page x: B_w <= x < B_{w+1}
DS_DEVICE int64_t owner_of(int64_t x, int64_t W, int64_t P) {
  int64_t w = x * W / P;
  while (w + 1 < W && range_begin(w + 1, W, P) <= x) ++w;
  while (w > 0 && range_begin(w, W, P) > x) --w;
  return w;
}

// The page space as "virtual workers": v < W are the static warp ranges over
// [0, P1), v = W + c the dynamic chunk c over [P1 + c*kChunkPages, ...). Ranges are
// contiguous, non-empty and in page order, so a (seq, head) pair's contributors
// are the consecutive virtual workers owning its first .. last page.
struct Part {
  int64_t W, P1, P, NC;
};
__host__ __device__ inline Part make_part(int64_t P, int64_t Wmax, int64_t max_chunks) {
  Part q;
  q.W = P < Wmax ? P : Wmax;
  int64_t dyn = 0;
  // only with >= 64 pages per warp (measured: B = 128 and 256 x 544 tokens gain 5-7 %,
  // B <= 64 loses up to 10 %: there the takes, the chunk partials and their merges
  // cost more than the balance gains)
  const int64_t pct = P < kDynPctSwitch * q.W ? kDynPctLow : kDynPct;
  if (kDynPct > 0 && P >= kDynMinPagesPerWarp * q.W) dyn = (P * pct / 100) / kChunkPages * kChunkPages;
  if (dyn > max_chunks * kChunkPages) dyn = max_chunks * kChunkPages;  // workspace bound
  q.P1 = P - dyn;
  q.P = P;
  q.NC = dyn / kChunkPages;
  return q;
}
DS_DEVICE int64_t vbegin(const Part &q, int64_t v) {
  return v <= q.W ? range_begin(v, q.W, q.P1) : q.P1 + (v - q.W) * kChunkPages;
}
DS_DEVICE int64_t vowner(const Part &q, int64_t x) {
  return x < q.P1 ? owner_of(x, q.W, q.P1) : q.W + (x - q.P1) / kChunkPages;
}

// partial row of warp w, segment seg (0: its first pair, 1: its last pair):
// o[D] then m, l; rows padded to 16 B so o loads/stores are vectors
template <int D>
constexpr int kPartialStride = D + 4;
template <int D, bool kDyn>
DS_DEVICE float *partial_row(const DecodeArgs &a, const Part &q, int64_t v, int seg) {
  if (!kDyn) return a.workspace + ((size_t)v * 2 + seg) * kPartialStride<D>;
  return v < q.W ? a.workspace + ((size_t)v * 2 + seg) * kPartialStride<D>
                 : a.chunk_rows + ((size_t)(v - q.W) * 2 + seg) * kPartialStride<D>;
}

// a8, fused: the warp that publishes the LAST partial of a straddling (seq, head)
// pair merges all of them (log-sum-exp rule) and resets the pair's ticket:
//   m* = max_k m_k ; l* = sum_k l_k 2^(m_k - m*) ; o = sum_k o_k 2^(m_k - m*) / l*
// Partials are published with a release fence + atomic ticket; the merger reads
// them with an acquire fence through L2 (ld.cg). Every warp range is non-empty
// (W <= P), so all k candidate contributors publish one partial each.
template <int D, bool kDyn>
DS_DEVICE void merge_if_last(const DecodeArgs &a, const int *prefix, int b, int h, const Part &part, int lane) {
  const int n = a.n_loc;
  const int npg = prefix[b + 1] - prefix[b];
  const int64_t start = (int64_t)n * prefix[b] + (int64_t)h * npg;
  const int64_t w0 = vowner(part, start), w1 = vowner(part, start + npg - 1);
  const int k = (int)(w1 - w0 + 1);
  __syncwarp();  // the partial written by lanes < TPG is ordered before the release below
  int ticket = 0;
  const int pair = b * n + h;
  if (lane == 0)
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(ticket) : "l"(a.tickets + pair) : "memory");
  ticket = __shfl_sync(0xffffffffu, ticket, 0);
  if (ticket != k - 1) return;
  __syncwarp();
  const int seg0 = vbegin(part, w0) < start ? 1 : 0;  // the pair is w0's last segment
  constexpr int PER = D / 32;  // dims per lane: 4 (D = 128) or 2 (D = 64)
  constexpr int U = 8;         // contributors whose o slices are in flight at once
  float mm = kNegInf, lt = 0.f, ot[PER];
#pragma unroll
  for (int e = 0; e < PER; ++e) ot[e] = 0.f;
  for (int j0 = 0; j0 < k; j0 += 32) {  // 32 contributors per round, (m, l) loads in parallel
    const int j = j0 + lane;
    const float *ws = partial_row<D, kDyn>(a, part, w0 + min(j, k - 1), j == 0 ? seg0 : 0);
    const float mj = j < k ? __ldcg(ws + D) : kNegInf;
    const float lj = j < k ? __ldcg(ws + D + 1) : 0.f;
    float mr = mj;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, o));
    const float m_new = fmaxf(mm, mr);
    const float alpha = rescale(mm, m_new);
    const float wj = rescale(mj, m_new);
    float lsum = lj * wj;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    lt = lt * alpha + lsum;
#pragma unroll
    for (int e = 0; e < PER; ++e) ot[e] *= alpha;
    mm = m_new;
    const int cnt = min(32, k - j0);
    for (int u0 = 0; u0 < cnt; u0 += U) {  // U independent vector loads, then the FMAs
      float val[U][PER];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int jj = j0 + u0 + u;
        const float *src = partial_row<D, kDyn>(a, part, w0 + min(jj, k - 1), jj == 0 ? seg0 : 0) + lane * PER;
        if (u0 + u < cnt) {
          if constexpr (PER == 4) {
            const float4 f = __ldcg(reinterpret_cast<const float4 *>(src));
            val[u][0] = f.x; val[u][1] = f.y; val[u][2] = f.z; val[u][3] = f.w;
          } else {
            const float2 f = __ldcg(reinterpret_cast<const float2 *>(src));
            val[u][0] = f.x; val[u][1] = f.y;
          }
        } else {
#pragma unroll
          for (int e = 0; e < PER; ++e) val[u][e] = 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float wt = __shfl_sync(0xffffffffu, wj, (u0 + u) & 31);
#pragma unroll
        for (int e = 0; e < PER; ++e) ot[e] = fmaf(val[u][e], wt, ot[e]);
      }
    }
  }
  const float inv = 1.f / lt;
  uint16_t *o = reinterpret_cast<uint16_t *>(a.out) + ((size_t)b * n + h) * D + lane * PER;
#pragma unroll
  for (int e = 0; e < PER; e += 2)
    *reinterpret_cast<uint32_t *>(o + e) = pack_bf16(ot[e] * inv, ot[e + 1] * inv);
  if (lane == 0) a.tickets[pair] = 0;  // self-cleaning: the workspace stays ready
}

// One page of 16 tokens for one warp. Lane (g, dpart): token rows t = it*GPW + g,
// dims [8*dpart, 8*dpart+8). kLast: the page holding position c (masked; token c
// comes from k_new/v_new).
template <int D, bool kLast>
DS_DEVICE void consume_page(const uint8_t *kst, const uint8_t *vst, const uint4 &q, float (&acc)[8],
                            float &m, float &l, int lane, int pos0, int c, float scale_log2,
                            const uint16_t *knew, const uint16_t *vnew) {
  constexpr int TPG = D / 8, GPW = 32 / TPG, NIT = 16 / GPW;  // NIT == TPG / 2
  const int g = lane / TPG, dpart = lane % TPG;
  // q.k partial sums of this lane's NIT rows
  float v[NIT];
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    const int t = it * GPW + g;
    uint4 kk = *reinterpret_cast<const uint4 *>(kst + t * (D * 2) + dpart * 16);
    if (kLast && pos0 + t == c) kk = *reinterpret_cast<const uint4 *>(knew);
    v[it] = dot8(q, kk);
  }
  // transpose-reduce over the TPG lanes: afterwards lane holds the full score of
  // row r = (lane >> 1) & (NIT - 1) (lanes 2k and 2k+1 hold the same row)
  int cnt = NIT;
#pragma unroll
  for (int o = TPG / 2; o >= 2; o >>= 1) {
    const bool up = lane & o;
#pragma unroll
    for (int j = 0; j < NIT / 2; ++j) {
      if (j < cnt / 2) {
        const float send = up ? v[j] : v[j + cnt / 2];
        const float keep = up ? v[j + cnt / 2] : v[j];
        v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    cnt >>= 1;
  }
  float s = (v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1)) * scale_log2;
  const int my_t = ((lane >> 1) & (NIT - 1)) * GPW + g;
  if (kLast && pos0 + my_t > c) s = kNegInf;
  // warp max / sum over the 16 distinct scores (skip xor 1: duplicates)
  float pmax = s;
#pragma unroll
  for (int o = 2; o < 32; o <<= 1) pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
  const float m_new = fmaxf(m, pmax);  // finite: every page has >= 1 valid token
  const float p = ex2(s - m_new);
  float psum = p;
#pragma unroll
  for (int o = 2; o < 32; o <<= 1) psum += __shfl_xor_sync(0xffffffffu, psum, o);
  if (m_new != m) {  // warp-uniform; lazy rescale
    const float alpha = rescale(m, m_new);
    l *= alpha;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] *= alpha;
    m = m_new;
  }
  l += psum;
  // P.V: broadcast the weight of each of this lane's rows from its owner lane
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    const int t = it * GPW + g;
    const float pw = __shfl_sync(0xffffffffu, p, g * TPG + it * 2);
    uint4 vv = *reinterpret_cast<const uint4 *>(vst + t * (D * 2) + dpart * 16);
    if (kLast && pos0 + t == c) vv = *reinterpret_cast<const uint4 *>(vnew);
    // slots past position c hold whatever the pool held (never written for this
    // sequence): their weight is 0, but 0 * NaN is NaN, so their V rows are zeroed
    if (kLast && pos0 + t > c) vv = make_uint4(0u, 0u, 0u, 0u);
    axpy8(acc, pw, vv);
  }
}

#ifdef DS_TRACE
// per-warp globaltimer stamps (A/B trace builds only): entry, prefix built, first
// page ready, loop done; read back with ds_debug_decode_trace
__device__ unsigned long long g_dec_trace[kDecodeMaxSMs * kWarpsPerSm][6];
DS_DEVICE unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define DTRACE(k, v) \
  if (lane == 0) g_dec_trace[blockIdx.x * kWarps + warp][k] = (v)
#else
#define DTRACE(k, v) ((void)0)
#endif

// kDyn: the launch may take dynamic chunks (the host picks it when the batch can
// reach >= 64 pages per warp); the static-only instance keeps the short path of
// small batches free of the range queue (measured 1-3 us per launch at B <= 32).
template <int D, bool kDyn>
__global__ void __launch_bounds__(kWarps * 32, kCtasPerSm) decode_kernel(const DecodeArgs a) {
  using C = DecCfg<D>;
  constexpr int TPG = D / 8;  // lanes per token row
  extern __shared__ __align__(128) uint8_t smem[];
  int *prefix = reinterpret_cast<int *>(smem + C::kPrefixOff);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::kBarOff);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int dpart = lane % TPG;
  const int B = a.num_seqs, n = a.n_loc;

  // PDL: the launch and CTA set-up overlap the previous kernel's tail; nothing
  // written by an earlier kernel (lengths, tables, pages, workspace) is read
  // before this wait.
  const bool early = a.early_kv != 0;
  if (!early) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) *reinterpret_cast<int *>(smem + C::kDoneOff) = 0;  // ordered by build_prefix's barriers
  DTRACE(0, gtimer());
  build_prefix(a.cache_lens, B, prefix);
  DTRACE(1, gtimer());
  const int64_t P = (int64_t)n * prefix[B];
  // at most one warp per page: every active warp range is non-empty, so a pair
  // never spans idle warps (tiny batches would otherwise merge across thousands)
  const Part part = make_part(P, (int64_t)gridDim.x * kWarps, kDyn ? a.max_chunks : 0);
  const int64_t W = part.W;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  if (gw >= W) return;

  // per-warp ring of kSlots half-stages: slot 2k holds a K page, 2k+1 its V page
  uint8_t *ring = smem + warp * C::kSlots * C::kPageBytes;
  uint64_t *wbar = bars + warp * C::kSlots;
  const uint32_t ring_s = smem_u32(ring), wbar_s = smem_u32(wbar);
  // per-warp queue of the page ranges this warp streams (its static range, then the
  // dynamic chunks it took), written by the producer lane, read by the whole warp
  int64_t *rq = reinterpret_cast<int64_t *>(smem + C::kRangeOff) + warp * 3 * kRangeQ;
  if (lane == 0) {
    for (int s = 0; s < C::kSlots; ++s) mbar_init(&wbar[s], 1);
    fence_barrier_init();
  }
  __syncwarp();  // the barriers are initialised before any lane waits on them

  const size_t page_elems = 16 * D;
  const size_t kv_stride = (size_t)a.num_blocks * n * page_elems;  // K -> V
  const uint16_t *layer_base = a.cache + (size_t)a.layer * 2 * kv_stride;

  // producer (lane 0): a page cursor that reads the block table one page ahead
  // (the load is consumed a step later, so lane 0 — and with it the consuming
  // warp — does not stall on it); the TMA bulk copies of K/V pages run kSlots
  // half-pages ahead of the consumer. At the end of a range it continues with the
  // chunk it took from the dynamic counter one range earlier (the atomic's result
  // is not waited on until then). (An L2 prefetch of pages further ahead —
  // cp.async.bulk.prefetch or per-lane prefetch.global.L2 — was measured 10-40 %
  // SLOWER at every batch size and is not used.)
  int nranges = 0;  // ranges written to the queue
  int pend = (int)part.NC;
  int64_t pr_x = 0, pr_x1 = 0;  // producer's next page / end of its current range
  bool prod_done = false;
  PagePos pf{};
  int blk_next = 0;
  auto push_range = [&](int64_t v) {
    const int64_t r0 = vbegin(part, v), r1 = vbegin(part, v + 1);
    if (kDyn) {
      int64_t *e = rq + 3 * (nranges % kRangeQ);
      e[0] = r0;
      e[1] = r1;
      e[2] = v;
      ++nranges;
    }
    pr_x = r0;
    pr_x1 = r1;
    pf = locate(r0, prefix, B, n);
    blk_next = a.block_table[(size_t)pf.b * a.max_blocks + pf.p];
  };
  auto next_range = [&]() -> bool {
    if (!kDyn) {
      prod_done = true;
      return false;
    }
    if (pend >= part.NC) {  // no chunk left: end-of-queue marker
      rq[3 * (nranges % kRangeQ)] = -1;
      ++nranges;
      prod_done = true;
      return false;
    }
    push_range(W + pend);
    return true;
  };
  auto next_page = [&]() {  // pool offset (in pages) of page pr_x; advances the cursor
    const size_t off = (size_t)blk_next * n + pf.h;
    if (++pr_x < pr_x1) {
      advance(pf, prefix, n);
      blk_next = a.block_table[(size_t)pf.b * a.max_blocks + pf.p];
    } else if (part.NC > 0) {
      // the range's last page is being issued: take the next chunk now (its
      // atomic completes while the ring still holds this range's last pages);
      // once the counter is past the end nobody adds to it any more
      pend = *reinterpret_cast<volatile int32_t *>(a.dyn) >= part.NC ? (int)part.NC : atomicAdd(a.dyn, 1);
    }
    return off;
  };
  int64_t h_issued = 0;
  int p_slot = 0;  // ring slot of the next half-page
  const uint16_t *cur_page = nullptr;
  auto issue = [&]() -> bool {  // one half-page into the ring; false when nothing is left
    if ((h_issued & 1) == 0) {
      if (pr_x == pr_x1 && !next_range()) return false;
      cur_page = layer_base + next_page() * page_elems;
    }
    const int slot = p_slot;  // == h_issued % kSlots, kept incrementally (no 64-bit division per issue)
    if (++p_slot == C::kSlots) p_slot = 0;
    expect_tx_s(wbar_s + slot * 8, C::kPageBytes);
    bulk_g2s_s(ring_s + slot * C::kPageBytes, cur_page + ((h_issued & 1) ? kv_stride : 0), C::kPageBytes,
               wbar_s + slot * 8);
    ++h_issued;
    return true;
  };
  if (lane == 0) {
    push_range(gw);
    for (int i = 0; i < C::kSlots && issue(); ++i) {
    }
  }
  if (early) {
    // early_kv: the lengths, the table and this layer's pages were read above
    // (and the first pages are in flight) before the previous kernel finished;
    // q, k_new, v_new, the workspace and `out` only from here on. The next kernel
    // may start once every CTA got here, so the kernel before this one is complete
    // by the time the next one reads anything.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }

  // consumer (its first range is the static one: computed here, not read from the
  // queue, so its loads overlap the producer lane's)
  int cr_i = 0;  // queue index of the range being consumed
  const int64_t x0 = vbegin(part, gw);
  int64_t cr_x1 = vbegin(part, gw + 1), cr_v = gw;
  PagePos cq = locate(x0, prefix, B, n);
  int seg_begin = cq.p;  // the first segment of a range may start mid-pair
  bool first_seg = true;
  uint4 qv;
  float m = kNegInf, l = 0.f, acc[8];
  int c = 0;
  size_t row = 0;
  auto load_pair = [&]() {
    row = ((size_t)cq.b * n + cq.h) * D + dpart * 8;
    qv = *reinterpret_cast<const uint4 *>(a.q + row);  // bf16 q; the scale goes on the score
    c = a.cache_lens[cq.b];
    m = kNegInf;
    l = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  };
  load_pair();

  int64_t x = x0, xc = 0;  // page, and pages consumed by this warp so far
  int c_slot = 0, c_ph = 0;  // consumer's ring slot and phase parity (see below)
  for (;; ++x, ++xc) {
    // ring slots and phase parities of this page's half-pages 2 xc, 2 xc + 1, kept
    // incrementally: the 64-bit divisions by kSlots cost ~20 instructions per page
    const int sk = c_slot, pk = c_ph;
    if (++c_slot == C::kSlots) c_slot = 0, c_ph ^= 1;
    const int sv = c_slot, pv = c_ph;
    if (++c_slot == C::kSlots) c_slot = 0, c_ph ^= 1;
    const bool last = cq.p == (c >> 4);
    if (last && lane < 2 * TPG) {  // (i) fused append of the new token at position c
      const int kv = lane / TPG;
      const int blk = a.block_table[(size_t)cq.b * a.max_blocks + cq.p];
      uint16_t *dst = const_cast<uint16_t *>(layer_base) + kv * kv_stride +
                      ((size_t)blk * n + cq.h) * page_elems + (size_t)(c & 15) * D + (lane % TPG) * 8;
      const size_t r2 = ((size_t)cq.b * n + cq.h) * D + (lane % TPG) * 8;
      *reinterpret_cast<uint4 *>(dst) = *reinterpret_cast<const uint4 *>((kv ? a.v_new : a.k_new) + r2);
    }
    page_wait(&wbar[sk], pk);
    page_wait(&wbar[sv], pv);
#ifdef DS_TRACE
    if (xc == 0) DTRACE(2, gtimer());
#endif
    const uint8_t *kst = ring + sk * C::kPageBytes, *vst = ring + sv * C::kPageBytes;
#if DS_DEC_FAKE  // timing experiment only (wrong results): no compute on the pages
    acc[0] += reinterpret_cast<const float *>(kst)[lane] + reinterpret_cast<const float *>(vst)[lane];
    if (false)
#else
    if (last)
#endif
      consume_page<D, true>(kst, vst, qv, acc, m, l, lane, cq.p * 16, c, a.scale_log2, a.k_new + row,
                            a.v_new + row);
    else
      consume_page<D, false>(kst, vst, qv, acc, m, l, lane, cq.p * 16, c, a.scale_log2, nullptr, nullptr);
    // both half-stages consumed: refill them kSlots half-pages ahead (refilling the
    // K slot right after the score reads was measured slower)
    __syncwarp();
    if (lane == 0 && !prod_done) {
      fence_proxy_async_smem();
      if (issue()) issue();
    }
    const bool pair_end = cq.p == cq.npg - 1;
    const bool range_end = x == cr_x1 - 1;
    if (pair_end || range_end) {
#pragma unroll
      for (int off = TPG; off < 32; off <<= 1)  // sum the token-row groups (same m)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], off);
      if (seg_begin == 0 && pair_end) {  // the whole pair is ours: final output
        if (lane < TPG) {
          const float inv = 1.f / l;
          uint4 o;
          o.x = pack_bf16(acc[0] * inv, acc[1] * inv);
          o.y = pack_bf16(acc[2] * inv, acc[3] * inv);
          o.z = pack_bf16(acc[4] * inv, acc[5] * inv);
          o.w = pack_bf16(acc[6] * inv, acc[7] * inv);
          *reinterpret_cast<uint4 *>(reinterpret_cast<uint16_t *>(a.out) + row) = o;
        }
      } else {  // a straddling pair: partial (o, m, l), merged by the last contributor (a8)
        float *ws = partial_row<D, kDyn>(a, part, cr_v, first_seg ? 0 : 1);
        if (lane < TPG) {
          reinterpret_cast<float4 *>(ws + dpart * 8)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
          reinterpret_cast<float4 *>(ws + dpart * 8)[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
          if (lane == 0) {
            ws[D] = m;
            ws[D + 1] = l;
          }
        }
        merge_if_last<D, kDyn>(a, prefix, cq.b, cq.h, part, lane);
      }
      first_seg = false;
      if (!range_end) {
        advance(cq, prefix, n);
        seg_begin = 0;
        load_pair();
      } else {  // next range of this warp (its entry is written: the producer runs ahead)
        if (!kDyn) break;
        ++cr_i;
        __syncwarp();
        const int64_t *e = rq + 3 * (cr_i % kRangeQ);
        if (e[0] < 0) break;
        x = e[0] - 1;  // ++x at the loop head
        cr_x1 = e[1];
        cr_v = e[2];
        cq = locate(e[0], prefix, B, n);
        seg_begin = cq.p;
        first_seg = true;
        load_pair();
      }
    } else {
      advance(cq, prefix, n);
    }
  }
  DTRACE(3, gtimer());
  DTRACE(4, (unsigned long long)xc);
  // the last warp out resets the dynamic counters for the next launch (every warp
  // has made its final take by now); warps are counted per CTA in smem, and the
  // last warp of each CTA counts the CTA globally (one global atomic per CTA)
  if (part.NC > 0 && lane == 0) {
    const int ctas = (int)((W + kWarps - 1) / kWarps);
    const int in_cta = (int)min((int64_t)kWarps, W - (int64_t)blockIdx.x * kWarps);
    int *cta_done = reinterpret_cast<int *>(smem + C::kDoneOff);
    if (atomicAdd(cta_done, 1) == in_cta - 1 && atomicAdd(a.dyn + 1, 1) == ctas - 1) {
      a.dyn[0] = 0;
      a.dyn[1] = 0;
    }
  }
}


// ------------------------------------------------------------------ pair streaming
// decode_pairs_kernel: the same computation as decode_kernel, with another work
// split. Every (sequence, head) pair is streamed by ONE CTA, all 16 of its warps at
// once: the CTA's pairs form one page stream and warp w takes stream pages w, w + 16,
// w + 32, ... (so each warp holds a partial (m, l, o) of every pair it touched); the
// partials of a pair meet in shared memory and the warp that publishes the last one
// merges them (a8) and writes `out`. The CTA takes its pairs one at a time from a
// global counter (its first pair is blockIdx.x), so no pair is split across CTAs —
// no global partials or tickets — and the launch ends within about one pair's
// streaming time (~6 us at 544 tokens with the SM's whole ring behind one pair)
// instead of one dynamic chunk of one warp (8 pages at ~3 GB/s per warp: the ~12-20
// us spread of warp finish times of decode_kernel, profiles/r01/decode_trace_*.txt).
// Used when the batch has enough pairs to keep every SM busy (host: launch_decode).
constexpr int kPU = 4;  // pairs whose partials can be in shared memory at once
// pair descriptors in flight: more than twice the units a warp's producer can run
// ahead of the slowest consumer (2 pages x 16 warps of 1-page pairs), so the
// publisher never waits on the warp that asks for a descriptor
constexpr int kPD = 64;
// descriptors published beyond the one asked for: every pair a CTA holds when the
// counter runs out is one more pair it streams while others are done. 0 measured best
// (B = 128 x 544 tokens: 211.7 us vs 212.6 with 1 and 220.3 with 2; the take of the
// next pair is made when the first warp's producer reaches it, ~4 us before the CTA's
// consumers do, which hides its ~2 us; profiles/r02/decode_pairs_ab.txt)
#ifndef DS_DEC_PAIR_LOOKAHEAD
#define DS_DEC_PAIR_LOOKAHEAD 0
#endif
constexpr int kPairLookahead = DS_DEC_PAIR_LOOKAHEAD;

template <int D>
struct PairCfg {
  static constexpr int kPageBytes = 16 * D * 2;
  static constexpr int kSlots = DecCfg<D>::kSlots;
  static constexpr int kRingBytes = kWarps * kSlots * kPageBytes;
  static constexpr int kRow = D + 4;                           // o[D], m, l, pad (floats)
  static constexpr int kPartOff = kRingBytes;                  // float[kPU][kWarps][kRow]
  static constexpr int kDescOff = kPartOff + kPU * kWarps * kRow * 4;  // int4[kPD]: pair, npg, sbeg, c
  static constexpr int kCtlOff = kDescOff + kPD * 16;          // int[16], see Ctl
  static constexpr int kWuOff = kCtlOff + 16 * 4;              // int[kWarps]: unit each warp's consumer is on
  static constexpr int kBarOff = kWuOff + kWarps * 4;
  static constexpr int kSmem = kBarOff + kWarps * kSlots * 8;
};
enum { CT_SEQ = 0, CT_LOCK = 1, CT_SBEG = 2, CT_END = 3, CT_DONE = 4, CT_GEN = 8 /* [kPU] */, CT_CNT = 12 /* [kPU] */ };

template <int D>
__global__ void __launch_bounds__(kWarps * 32, 1) decode_pairs_kernel(const DecodeArgs a) {
  using C = PairCfg<D>;
  constexpr int TPG = D / 8;
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int dpart = lane % TPG;
  const int n = a.n_loc;
  const int num_pairs = a.num_seqs * n;
  float *part = reinterpret_cast<float *>(smem + C::kPartOff);
  int4 *desc = reinterpret_cast<int4 *>(smem + C::kDescOff);
  volatile int *ctl = reinterpret_cast<volatile int *>(smem + C::kCtlOff);
  volatile int *wunit = reinterpret_cast<volatile int *>(smem + C::kWuOff);
  uint64_t *wbar = reinterpret_cast<uint64_t *>(smem + C::kBarOff) + warp * C::kSlots;
  uint8_t *ring = smem + warp * C::kSlots * C::kPageBytes;
  int *counter = a.dyn + 2, *ctas_done = a.dyn + 3;

  const bool early = a.early_kv != 0;
  if (!early) asm volatile("griddepcontrol.wait;" ::: "memory");
  DTRACE(0, gtimer());
  if (threadIdx.x == 0) {
    for (int k = 0; k < 16; ++k) ctl[k] = 0;
    // unit 0 is static (no counter access before the PDL wait)
    const int p0 = blockIdx.x;
    if (p0 < num_pairs) {
      const int c = a.cache_lens[p0 / n], npg = npages_of(c);
      desc[0] = make_int4(p0, npg, 0, c);
      ctl[CT_SBEG] = npg;
    } else {
      desc[0] = make_int4(-1, 0, 0, 0);
      ctl[CT_END] = 1;
    }
    ctl[CT_SEQ] = 1;
  }
  if (lane == 0) {
    for (int s = 0; s < C::kSlots; ++s) mbar_init(&wbar[s], 1);
    wunit[warp] = 0;
  }
  fence_barrier_init();
  __syncthreads();
  DTRACE(1, gtimer());

  // descriptor d (lane 0 of any warp): published in order by whoever holds the lock;
  // slot d % kPD is rewritten only when every warp's consumer is past unit d - kPD
  bool past_wait = !early;
  // (every wait below backs off with __nanosleep: under the power cap a spinning
  // warp costs SM clock — the first version's tight CAS loop on the lock measured
  // 1556 vs 1620 MHz and a slower step in bench.py than the page-range kernel)
  auto need_desc = [&](int d) {
    while (ctl[CT_SEQ] <= d) {
      if (ctl[CT_LOCK] != 0 || atomicCAS(const_cast<int *>(&ctl[CT_LOCK]), 0, 1) != 0) {
        __nanosleep(128);
        continue;
      }
      int seq = ctl[CT_SEQ];
      while (seq <= d + kPairLookahead && !ctl[CT_END]) {
        int lo = 0x7fffffff;
        for (int w = 0; w < kWarps; ++w) lo = min(lo, wunit[w]);
        if (lo <= seq - kPD) break;  // descriptor slot still in use
        const int pr = (int)gridDim.x + atomicAdd(counter, 1);
        if (pr >= num_pairs) {
          desc[seq % kPD] = make_int4(-1, 0, 0, 0);
          ctl[CT_END] = 1;
        } else {
          const int c = a.cache_lens[pr / n], npg = npages_of(c), sb = ctl[CT_SBEG];
          desc[seq % kPD] = make_int4(pr, npg, sb, c);
          ctl[CT_SBEG] = sb + npg;
        }
        __threadfence_block();
        ctl[CT_SEQ] = ++seq;
      }
      __threadfence_block();
      atomicExch(const_cast<int *>(&ctl[CT_LOCK]), 0);
    }
  };
  auto read_desc = [&](int d) {
    const volatile int *v = reinterpret_cast<volatile int *>(&desc[d % kPD]);
    return make_int4(v[0], v[1], v[2], v[3]);
  };

  const size_t page_elems = 16 * D;
  const size_t kv_stride = (size_t)a.num_blocks * n * page_elems;
  const uint16_t *layer_base = a.cache + (size_t)a.layer * 2 * kv_stride;

  // ---- producer (lane 0): stream pages w, w+16, ... one half-page per issue
  int ps = warp, pd = 0;
  int4 pdesc = desc[0];
  bool prod_done = false;
  int64_t h_issued = 0;
  int p_slot = 0;  // ring slot of the next half-page
  const uint16_t *cur_page = nullptr;
  // false: the stream has ended (or, before the PDL wait, this warp's next page is past unit 0)
  auto prod_locate = [&]() -> bool {
    while (pdesc.x >= 0 && ps >= pdesc.z + pdesc.y) {
      if (!past_wait) return false;
      ++pd;
      need_desc(pd);
      pdesc = read_desc(pd);
    }
    return pdesc.x >= 0;
  };
  auto issue = [&]() -> bool {
    if ((h_issued & 1) == 0) {
      if (!prod_locate()) return false;
      const int b = pdesc.x / n, h = pdesc.x - b * n, p = ps - pdesc.z;
      const int blk = a.block_table[(size_t)b * a.max_blocks + p];
      cur_page = layer_base + ((size_t)blk * n + h) * page_elems;
      ps += kWarps;
    }
    const int slot = p_slot;  // == h_issued % kSlots, kept incrementally (no 64-bit division per issue)
    if (++p_slot == C::kSlots) p_slot = 0;
    mbar_arrive_expect_tx(&wbar[slot], C::kPageBytes);
    bulk_g2s(ring + slot * C::kPageBytes, cur_page + ((h_issued & 1) ? kv_stride : 0), C::kPageBytes, &wbar[slot]);
    ++h_issued;
    return true;
  };
  if (lane == 0)
    for (int i = 0; i < C::kSlots && issue(); ++i) {
    }
  if (early) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    past_wait = true;
    __syncwarp();
    if (lane == 0)  // top up what stopped at unit 0
      while (h_issued < C::kSlots && issue()) {
      }
  }

  // ---- consumer (all lanes)
  int cs = warp, cd = 0;
  int4 cdesc = desc[0];
  bool have = false;  // this warp holds a partial of unit cd
  uint4 qv;
  float m = kNegInf, l = 0.f, acc[8];
  size_t row = 0;
  // publish the partial of unit u (pair pr, npg pages, stream start sb); the last of
  // its min(16, npg) contributors merges them and writes out[b][h]
  auto flush = [&](int u, const int4 &dd) {
#pragma unroll
    for (int off = TPG; off < 32; off <<= 1)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], off);
    const int slot = u % kPU, gen = u / kPU;
    while (ctl[CT_GEN + slot] < gen) __nanosleep(64);
    float *mine = part + (slot * kWarps + warp) * C::kRow;
    if (lane < TPG) {
      reinterpret_cast<float4 *>(mine + dpart * 8)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
      reinterpret_cast<float4 *>(mine + dpart * 8)[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
      if (lane == 0) {
        mine[D] = m;
        mine[D + 1] = l;
      }
    }
    __syncwarp();
    int t = 0;
    if (lane == 0) {
      __threadfence_block();
      t = atomicAdd(const_cast<int *>(&ctl[CT_CNT + slot]), 1);
    }
    t = __shfl_sync(0xffffffffu, t, 0);
    const int k = min(kWarps, dd.y);
    if (t != k - 1) return;
    __threadfence_block();
    constexpr int PER = D / 32;
    float mm = kNegInf;
    for (int j = 0; j < k; ++j) mm = fmaxf(mm, part[(slot * kWarps + (dd.z + j) % kWarps) * C::kRow + D]);
    float lt = 0.f, ot[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) ot[e] = 0.f;
    for (int j = 0; j < k; ++j) {
      const float *pj = part + (slot * kWarps + (dd.z + j) % kWarps) * C::kRow;
      const float wj = rescale(pj[D], mm);
      lt = fmaf(pj[D + 1], wj, lt);
#pragma unroll
      for (int e = 0; e < PER; ++e) ot[e] = fmaf(pj[lane * PER + e], wj, ot[e]);
    }
    const float inv = 1.f / lt;
    const int b = dd.x / n, h = dd.x - b * n;
    uint16_t *o = reinterpret_cast<uint16_t *>(a.out) + ((size_t)b * n + h) * D + lane * PER;
#pragma unroll
    for (int e = 0; e < PER; e += 2) *reinterpret_cast<uint32_t *>(o + e) = pack_bf16(ot[e] * inv, ot[e + 1] * inv);
    __syncwarp();
    if (lane == 0) {
      ctl[CT_CNT + slot] = 0;
      __threadfence_block();
      ctl[CT_GEN + slot] = gen + 1;  // the slot's next pair may publish
    }
  };
  // q of the next pair is loaded when this warp enters a pair (if its descriptor is
  // out), so the load's latency is not paid every ~2 pages
  uint4 qn = make_uint4(0u, 0u, 0u, 0u);
  int qn_pair = -1;
  auto enter = [&](const int4 &dd) {  // first page of this warp in pair dd.x
    row = ((size_t)dd.x * D) + dpart * 8;  // pair index b * n + h == dd.x
    qv = qn_pair == dd.x ? qn : *reinterpret_cast<const uint4 *>(a.q + row);
    qn_pair = -1;
    if (ctl[CT_SEQ] > cd + 1) {
      const int4 nx = read_desc(cd + 1);
      if (nx.x >= 0) {
        qn = *reinterpret_cast<const uint4 *>(a.q + (size_t)nx.x * D + dpart * 8);
        qn_pair = nx.x;
      }
    }
    m = kNegInf;
    l = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    have = true;
  };

  int c_slot = 0, c_ph = 0;  // consumer's ring slot and phase parity (see below)
  for (int64_t xc = 0;; ++xc) {
    // locate stream page cs (descriptors were published for this warp's producer)
    while (cdesc.x >= 0 && cs >= cdesc.z + cdesc.y) {
      if (have) flush(cd, cdesc);
      have = false;
      ++cd;
      while (ctl[CT_SEQ] <= cd) __nanosleep(64);
      cdesc = read_desc(cd);
      if (lane == 0) wunit[warp] = cd;
    }
    if (cdesc.x < 0) break;
    if (!have) enter(cdesc);
    const int p = cs - cdesc.z, c = cdesc.w;
    const int b = cdesc.x / n, h = cdesc.x - b * n;
    const bool last = p == (c >> 4);
    // ring slots and phase parities of this page's half-pages 2 xc, 2 xc + 1, kept
    // incrementally: the 64-bit divisions by kSlots cost ~20 instructions per page
    const int sk = c_slot, pk = c_ph;
    if (++c_slot == C::kSlots) c_slot = 0, c_ph ^= 1;
    const int sv = c_slot, pv = c_ph;
    if (++c_slot == C::kSlots) c_slot = 0, c_ph ^= 1;
    if (last && lane < 2 * TPG) {  // (i) fused append of the new token at position c
      const int kv = lane / TPG;
      const int blk = a.block_table[(size_t)b * a.max_blocks + p];
      uint16_t *dst = const_cast<uint16_t *>(layer_base) + kv * kv_stride + ((size_t)blk * n + h) * page_elems +
                      (size_t)(c & 15) * D + (lane % TPG) * 8;
      *reinterpret_cast<uint4 *>(dst) = *reinterpret_cast<const uint4 *>((kv ? a.v_new : a.k_new) + row);
    }
    page_wait(&wbar[sk], pk);
    page_wait(&wbar[sv], pv);
#ifdef DS_TRACE
    if (xc == 0) DTRACE(2, gtimer());
#endif
    const uint8_t *kst = ring + sk * C::kPageBytes, *vst = ring + sv * C::kPageBytes;
    if (last)
      consume_page<D, true>(kst, vst, qv, acc, m, l, lane, p * 16, c, a.scale_log2, a.k_new + row, a.v_new + row);
    else
      consume_page<D, false>(kst, vst, qv, acc, m, l, lane, p * 16, c, a.scale_log2, nullptr, nullptr);
    __syncwarp();
    if (lane == 0 && !prod_done) {
      fence_proxy_async_smem();
      if (!issue() || !issue()) prod_done = true;
    }
    cs += kWarps;
  }
  if (lane == 0) wunit[warp] = 0x7fffffff;
  DTRACE(3, gtimer());
#ifdef DS_TRACE
  {
    // pages consumed by this warp: count the stream indices it visited
    DTRACE(4, (unsigned long long)((cs - warp) / kWarps));
  }
#endif

  // the last warp of the last CTA resets the counters for the next launch
  if (lane == 0 && atomicAdd(const_cast<int *>(&ctl[CT_DONE]), 1) == kWarps - 1) {
    if (atomicAdd(ctas_done, 1) == (int)gridDim.x - 1) {
      *counter = 0;
      *ctas_done = 0;
    }
  }
}

}  // namespace

#ifdef DS_TRACE
extern "C" __attribute__((visibility("default"))) int ds_debug_decode_trace(unsigned long long *host, int reset) {
  cudaDeviceSynchronize();
  if (host) cudaMemcpyFromSymbol(host, g_dec_trace, sizeof(g_dec_trace));
  if (reset) {
    void *p = nullptr;
    cudaGetSymbolAddress(&p, g_dec_trace);
    cudaMemset(p, 0, sizeof(g_dec_trace));
    cudaDeviceSynchronize();
  }
  return (int)(sizeof(g_dec_trace) / 8);
}
#endif

// workspace: [dyn counters 16 B][tickets kDecodeMaxPairs x int32][static partial rows]
// [chunk partial rows]. The counters and tickets must be zero between calls: both sit
// at offsets and in regions that depend on nothing about the call (batch, heads,
// head_dim, lengths), so a workspace reused with a growing batch or another head_dim
// still finds every ticket it touches at zero. The partial rows need no
// initialisation (written before they are read in every launch).
DecodeLayout decode_layout(int num_seqs, int n_loc, int head_dim, int num_sms, int max_cache_len) {
  DecodeLayout L;
  const size_t row = (size_t)(head_dim + 4) * sizeof(float);
  L.dyn_off = 0;
  L.tickets_off = 16;
  L.rows_off = L.tickets_off + (size_t)kDecodeMaxPairs * 4;
  L.chunk_off = L.rows_off + (size_t)num_sms * kWarpsPerSm * 2 * row;
  const int64_t pmax = (int64_t)num_seqs * n_loc * npages_of(max_cache_len);
  const Part q = make_part(pmax, (int64_t)num_sms * kWarpsPerSm, INT64_MAX / kChunkPages);
  L.max_chunks = q.NC;
  L.total = L.chunk_off + (size_t)q.NC * 2 * row;
  return L;
}

int decode_warps_per_cta() { return kWarps; }

template <int D, bool kDyn>
static cudaError_t set_decode_smem_once() {
  static cudaError_t st = cudaFuncSetAttribute(decode_kernel<D, kDyn>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               DecCfg<D>::kSmem);  // thread-safe static init, once
  return st;
}
template <int D, bool kDyn>
static cudaError_t launch_d(cudaLaunchConfig_t &cfg, const DecodeArgs &a) {
  cudaError_t e = set_decode_smem_once<D, kDyn>();
  if (e != cudaSuccess) return e;
  cfg.dynamicSmemBytes = DecCfg<D>::kSmem;
  return cudaLaunchKernelEx(&cfg, decode_kernel<D, kDyn>, a);
}

bool decode_uses_pairs(int num_seqs, int n_loc, int num_sms) {
  // pair streaming (decode_pairs_kernel): OPT-IN, DS_DEC_PAIRS=k uses it from k pairs
  // per SM on (read once). Measured (profiles/r02/decode_pairs_ab.txt): alone it is
  // 4-5 % faster than decode_kernel from B = 32 to 128 x 544 tokens x 40 heads (3 % at
  // 256; equal at 4.3 pairs per SM, slower below) — B = 128: 211.6 vs 221.0 us, within
  // 2 % of trtllm-gen — but inside bench.py's step, where the GPU runs at its power
  // cap, it is 1.5-2.5 % SLOWER (228-231 vs 225 us per launch, SM clock 1635 vs
  // 1655-1665 MHz): it executes 19 % more instructions (ncu, B = 128: 122.8 M vs
  // 102.9 M — every warp enters, flushes and polls for every pair), and under the cap
  // instructions cost clock. The default stays decode_kernel.
  static const int pairs_mode = [] {
    const char *e = getenv("DS_DEC_PAIRS");
    return e ? atoi(e) : 0;
  }();
  return pairs_mode > 0 && kCtasPerSm == 1 && (int64_t)num_seqs * n_loc >= (int64_t)pairs_mode * num_sms;
}

cudaError_t launch_decode(const DecodeArgs &a, int head_dim, int num_sms, cudaStream_t stream) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(num_sms * kCtasPerSm);
  cfg.blockDim = dim3(kWarps * 32);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // dynamic chunks only if the batch can reach the threshold (an upper bound of the
  // page count from max_cache_len; the kernel decides exactly from the lengths)
  if (decode_uses_pairs(a.num_seqs, a.n_loc, num_sms)) {
    cfg.gridDim = dim3(num_sms);
    cudaError_t e;
    if (head_dim == 128) {
      static cudaError_t st = cudaFuncSetAttribute(decode_pairs_kernel<128>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, PairCfg<128>::kSmem);
      if (st != cudaSuccess) return st;
      cfg.dynamicSmemBytes = PairCfg<128>::kSmem;
      e = cudaLaunchKernelEx(&cfg, decode_pairs_kernel<128>, a);
    } else {
      static cudaError_t st = cudaFuncSetAttribute(decode_pairs_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   PairCfg<64>::kSmem);
      if (st != cudaSuccess) return st;
      cfg.dynamicSmemBytes = PairCfg<64>::kSmem;
      e = cudaLaunchKernelEx(&cfg, decode_pairs_kernel<64>, a);
    }
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  const int64_t pmax = (int64_t)a.num_seqs * a.n_loc * npages_of(a.max_cache_len);
  const bool dyn = a.max_chunks > 0 && make_part(pmax, (int64_t)num_sms * kWarpsPerSm, a.max_chunks).NC > 0;
  cudaError_t e;
  if (head_dim == 128)
    e = dyn ? launch_d<128, true>(cfg, a) : launch_d<128, false>(cfg, a);
  else
    e = dyn ? launch_d<64, true>(cfg, a) : launch_d<64, false>(cfg, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace ds
