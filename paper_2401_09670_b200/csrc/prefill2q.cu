// prefill2q.cu — EXPERIMENTAL a2 + a3 variant (DS_PREFILL_KERNEL=2q): one CTA
// per PAIR of 128-row q tiles (256 query rows) of one (sequence, head),
// FA4-style ping-pong with 128-key tiles. Parity-tested; still slower than
// prefill.cu's two CTAs per SM (4 x 4096: 700 us vs 647-680 us, after the FA4
// issue order and the TMA-store epilogue took it from 821 us): one CTA per SM
// runs one item at a time (no persistence), so item start-up and the drain are
// exposed, and each 128-column softmax tile is a long latency chain.
//
// Same computation as prefill.cu (§2.1, App. A;
// readings R1, R2; a3 page write P:102):
//   out[i] = sum_{j<=i} softmax_j(scale * q[i].k[j]) v[j];  cache[..][t] = k|v[t]
//
// Why a second kernel: with one q tile per CTA the S -> softmax -> P.V chain of
// a tile is serial, and two independent CTAs on an SM do not coordinate who
// uses the tensor pipe. Here two q tiles A and B share every K/V tile (half
// the K/V smem/L2 traffic per query row) and one MMA warp interleaves them:
//     S_A(j)  S_B(j)  [P_A(j) ready] PV_A(j)  [P_B(j) ready] PV_B(j)  S_A(j+1) ...
// so the tensor pipe computes one tile's MMAs while the other tile's softmax
// warpgroup runs (MUFU and tensor are both ~2048 clk per 128-key tile here).
//   warps 0-3 softmax A, 4-7 softmax B (thread = q row = TMEM lane),
//   warp 8 TMA producer (+ paged store of the CTA's 256 diagonal keys),
//   warp 9 MMA issuer (+ TMEM allocation: S_A | O_A | S_B | O_B = 512 columns).
// smem: Q_A, Q_B, 2 K stages, 2 V stages of 128 keys = 192 KiB at head_dim 128.
#include "common.cuh"
#include "kernels.h"

namespace ds {
namespace {

constexpr int kBM = 128, kBN = 128;
constexpr int kThreads = 320;
constexpr uint32_t kChunk = 128 * 128;  // 128 rows x 128 B: one SW128 column block
constexpr float kRescaleLog2 = 8.f;     // exponent base moves only past 2^8 growth
constexpr int kPolyEvery = 4;           // 1 in 4 exp2 on the FMA pipe: MUFU is the co-bottleneck here

template <int D>
struct Smem2 {
  static constexpr uint32_t kTile = 128 * D * 2;
  static constexpr uint32_t QA = 0, QB = kTile;
  static constexpr uint32_t K0 = 2 * kTile;  // 2 stages
  static constexpr uint32_t V0 = K0 + 2 * kTile;
  static constexpr uint32_t OST = V0 + 2 * kTile;  // epilogue staging: 8 warps x 32 rows x 32 dims bf16
  static constexpr uint32_t BAR = OST + 8 * 2048;
  static constexpr uint32_t kBars = 16;
  static constexpr uint32_t TMEM_SLOT = BAR + kBars * 8;
  static constexpr uint32_t ALLOC = TMEM_SLOT + 16 + 1024;
};

enum { B_Q = 0, B_KF = 1, B_VF = 3, B_KE = 5, B_VE = 7, B_SF = 9, B_PF = 11, B_OD = 13 };  // [2]: stage / tile

DS_DEVICE void ctl_wait2(uint64_t *bar, uint32_t parity) { mbar_wait(bar, parity); }

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    prefill2q_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_cache,
                     const __grid_constant__ CUtensorMap tm_o, const PrefillArgs a) {
  using S = Smem2<D>;
  constexpr int kChunks = D / 64;
  const int h = blockIdx.y, r = blockIdx.z;
  const int i = a.num_q_tiles - 1 - (int)blockIdx.x;  // q-tile PAIR index, heaviest first
  const int seq_start = a.cu_seqlens[r];
  const int len = a.cu_seqlens[r + 1] - seq_start;
  if (i * 2 * kBM >= len) return;
  const bool has_b = i * 2 * kBM + kBM < len;
  // key tiles per q tile: A (rows 256i..) needs 0..2i, B (rows 256i+128..) 0..2i+1
  const int n_a = 2 * i + 1, n_b = has_b ? 2 * i + 2 : 0;
  auto n_t = [&](int t) { return t ? n_b : n_a; };
  const int ntiles = has_b ? 2 * i + 2 : 2 * i + 1;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t *smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  const uint32_t sbase = smem_u32(smem);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + S::BAR);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + S::TMEM_SLOT);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int b = 0; b < (int)S::kBars; ++b) mbar_init(&bars[b], (b == B_PF || b == B_PF + 1) ? 128 : 1);
    fence_barrier_init();
  }
  if (warp == 9) {
    tmem_alloc<512>(tmem_slot);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // S_t at t*256, O_t at t*256 + 128
  auto tS = [&](int t) { return tmem + t * 256; };
  auto tO = [&](int t) { return tmem + t * 256 + 128; };

  if (warp == 8) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      tma_prefetch_desc(&tm_cache);
      const int q0 = seq_start + i * 2 * kBM;
      mbar_arrive_expect_tx(&bars[B_Q], S::kTile * (has_b ? 2 : 1));
#pragma unroll
      for (int c = 0; c < kChunks; ++c) {
        tma_load_3d(smem + S::QA + c * kChunk, &tm_q, &bars[B_Q], c * 64, h, q0);
        if (has_b) tma_load_3d(smem + S::QB + c * kChunk, &tm_q, &bars[B_Q], c * 64, h, q0 + kBM);
      }
      for (int j = 0; j < ntiles; ++j) {
        const int st = j & 1, kv0 = seq_start + j * kBN;
        if (j >= 2) mbar_wait(&bars[B_KE + st], ((j >> 1) - 1) & 1);
        mbar_arrive_expect_tx(&bars[B_KF + st], S::kTile);
#pragma unroll
        for (int c = 0; c < kChunks; ++c)
          tma_load_3d(smem + S::K0 + st * S::kTile + c * kChunk, &tm_k, &bars[B_KF + st], c * 64, h, kv0);
        if (j >= 2) mbar_wait(&bars[B_VE + st], ((j >> 1) - 1) & 1);
        mbar_arrive_expect_tx(&bars[B_VF + st], S::kTile);
#pragma unroll
        for (int c = 0; c < kChunks; ++c)
          tma_load_3d(smem + S::V0 + st * S::kTile + c * kChunk, &tm_v, &bars[B_VF + st], c * 64, h, kv0);
      }
      // a3: the CTA owns keys [256i, 256i+256) = key tiles 2i, 2i+1 = pages 16i .. 16i+15
      const int npg = min(16, (len - i * 2 * kBM + 15) >> 4);
      const int32_t *bt = a.block_table + (size_t)r * a.max_blocks + i * 16;
      for (int t = 2 * i; t < ntiles; ++t) {
        const int st = t & 1;
        mbar_wait(&bars[B_KF + st], (t >> 1) & 1);
        mbar_wait(&bars[B_VF + st], (t >> 1) & 1);
        for (int p = (t - 2 * i) * 8; p < min(npg, (t - 2 * i) * 8 + 8); ++p) {
          const int blk = bt[p];
#pragma unroll
          for (int kv = 0; kv < 2; ++kv)
#pragma unroll
            for (int c = 0; c < kChunks; ++c)
              tma_store_4d(&tm_cache, smem + (kv ? S::V0 : S::K0) + st * S::kTile + c * kChunk + (p & 7) * 16 * 128,
                           c * 64, 0, h, (a.layer * 2 + kv) * a.num_blocks + blk);
        }
      }
      bulk_commit_group();
      for (int t = max(0, ntiles - 2); t < ntiles; ++t) {  // observe the last stage releases
        mbar_wait(&bars[B_KE + (t & 1)], (t >> 1) & 1);
        mbar_wait(&bars[B_VE + (t & 1)], (t >> 1) & 1);
      }
      bulk_wait_group_read0();
    }
    __syncwarp();
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(kBM, kBN, 0, 0);
      constexpr uint32_t idesc_o = idesc_bf16_f32(kBM, D, 0, 1);
      // FA4-style order: S_A(0) S_B(0) | PV_A(j) S_A(j+1) PV_B(j) S_B(j+1) | ...
      // so each tile's softmax overlaps the other tile's P.V and S MMAs (two MMA
      // blocks). S_t(j+1) overwrites P_t(j) right after P_t(j) V_t(j) was issued:
      // tcgen05.mma ops of one thread execute in issue order, so no wait is needed.
      auto issue_s = [&](int t, int j) {
        const int st = j & 1;
        if (t == 0 || j >= n_t(0)) ctl_wait2(&bars[B_KF + st], (j >> 1) & 1);  // first user of K_j waits
        tc_fence_after();
        const uint32_t qb = t ? S::QB : S::QA;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kChunk + (kk & 3) * 32;
          umma_ss(tS(t), smem_desc_sw128(sbase + qb + off, 16, 1024),
                  smem_desc_sw128(sbase + S::K0 + st * S::kTile + off, 16, 1024), idesc_s, kk > 0);
        }
        umma_commit(&bars[B_SF + t]);
        if (t == 1 || j >= n_t(1)) umma_commit(&bars[B_KE + st]);  // last user of K_j releases it
      };
      auto issue_pv = [&](int t, int j) {
        const int st = j & 1;
        ctl_wait2(&bars[B_PF + t], j & 1);
        if (t == 0 || j >= n_t(0)) ctl_wait2(&bars[B_VF + st], (j >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk)
          umma_ts(tO(t), tS(t) + kk * 8, smem_desc_sw128(sbase + S::V0 + st * S::kTile + kk * 16 * 128, kChunk, 1024),
                  idesc_o, (j > 0 || kk > 0));
        if (j == n_t(t) - 1) umma_commit(&bars[B_OD + t]);        // once per tile: O_t final
        if (t == 1 || j >= n_t(1)) umma_commit(&bars[B_VE + st]);  // last user of V_j releases it
      };
      ctl_wait2(&bars[B_Q], 0);
      issue_s(0, 0);
      if (n_t(1) > 0) issue_s(1, 0);
      for (int j = 0; j < ntiles; ++j) {
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          if (j >= n_t(t)) continue;
          issue_pv(t, j);
          if (j + 1 < n_t(t)) issue_s(t, j + 1);
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ softmax warpgroup t
    const int t = warp >> 2;
    const int row = threadIdx.x & 127;
    const int q_pos = i * 2 * kBM + t * kBM + row;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const float sl2 = a.scale_log2;
    float m = -__int_as_float(0x7f800000), l = 0.f;
    for (int j = 0; j < n_t(t); ++j) {
      // S_t(j) ready; it was issued after P_t(j-1) V_t(j-1), and in-order MMA
      // execution means that P.V is complete too, so O_t is stable
      mbar_wait(&bars[B_SF + t], j & 1);
      tc_fence_after();
      uint32_t sr[4][32];
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) tmem_ld32(tS(t) + lane_off + cc * 32, sr[cc]);
      tmem_wait_ld();
      float mx = -__int_as_float(0x7f800000);
      if (j == 2 * i + t) {  // diagonal key tile: key column > query row is masked
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            if (cc * 32 + e > row) sr[cc][e] = 0xff800000u;
            mx = fmaxf(mx, __uint_as_float(sr[cc][e]));
          }
      } else {
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
#pragma unroll
          for (int e = 0; e < 32; ++e) mx = fmaxf(mx, __uint_as_float(sr[cc][e]));
      }
      const float m_tile = mx * sl2;
      const bool grow = m_tile > m + kRescaleLog2;  // conditional rescaling (see prefill.cu)
      const float m_new = grow ? m_tile : m;
      const float alpha = grow ? ex2(m - m_new) : 1.f;
      const uint64_t sl2x2 = f2_pack(sl2, sl2), negm2 = f2_pack(-m_new, -m_new);
      uint64_t rs2 = f2_pack(0.f, 0.f);
      uint32_t pk[2][32];
#pragma unroll
      for (int cc = 0; cc < 4; ++cc)
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float x0, x1;
          f2_unpack(f2_fma(f2_pack(__uint_as_float(sr[cc][e]), __uint_as_float(sr[cc][e + 1])), sl2x2, negm2), x0,
                    x1);
          const float p0 = (e % kPolyEvery) == 0 ? ex2_poly(x0) : ex2(x0);
          const float p1 = ex2(x1);
          rs2 = f2_add(rs2, f2_pack(p0, p1));
          pk[cc >> 1][(cc & 1) * 16 + e / 2] = pack_bf16(p0, p1);
        }
      float rs0, rs1;
      f2_unpack(rs2, rs0, rs1);
      l = l * alpha + (rs0 + rs1);
      m = m_new;
      if (j > 0 && __any_sync(0xffffffffu, grow)) {
        const uint64_t a2 = f2_pack(alpha, alpha), z2 = f2_pack(0.f, 0.f);
#pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) {
          uint32_t o[32];
          tmem_ld32(tO(t) + lane_off + cc * 32, o);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            float lo, hi;
            f2_unpack(f2_fma(f2_pack(__uint_as_float(o[e]), __uint_as_float(o[e + 1])), a2, z2), lo, hi);
            o[e] = __float_as_uint(lo);
            o[e + 1] = __float_as_uint(hi);
          }
          tmem_st32(tO(t) + lane_off + cc * 32, o);
        }
      }
      tmem_st32(tS(t) + lane_off + 0, pk[0]);  // P (bf16 pairs) over the first 64 columns of S_t
      tmem_st32(tS(t) + lane_off + 32, pk[1]);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bars[B_PF + t]);
    }
    if (n_t(t) > 0) {
      // epilogue as in prefill.cu: each warp stages its 32 rows x 32 dims chunks in
      // smem (64-B swizzle of the TMA box) and one lane TMA-stores them; a warp whose
      // rows run past the sequence end stores its valid rows directly
      mbar_wait(&bars[B_OD + t], 0);  // committed once, after O_t's last P.V
      tc_fence_after();
      const float inv_l = 1.f / l;
      const int row0 = i * 2 * kBM + t * kBM + (warp & 3) * 32;
      const bool boxed = row0 + 32 <= len;
      uint8_t *stg = smem + S::OST + warp * 2048;
      uint16_t *orow = reinterpret_cast<uint16_t *>(a.out) + ((size_t)(seq_start + q_pos) * a.n_loc + h) * D;
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t o[32];
        tmem_ld32(tO(t) + lane_off + cc * 32, o);
        tmem_wait_ld();
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          v[u].x = pack_bf16(__uint_as_float(o[u * 8 + 0]) * inv_l, __uint_as_float(o[u * 8 + 1]) * inv_l);
          v[u].y = pack_bf16(__uint_as_float(o[u * 8 + 2]) * inv_l, __uint_as_float(o[u * 8 + 3]) * inv_l);
          v[u].z = pack_bf16(__uint_as_float(o[u * 8 + 4]) * inv_l, __uint_as_float(o[u * 8 + 5]) * inv_l);
          v[u].w = pack_bf16(__uint_as_float(o[u * 8 + 6]) * inv_l, __uint_as_float(o[u * 8 + 7]) * inv_l);
        }
        if (boxed) {
          if (lane == 0) bulk_wait_group_read0();
          __syncwarp();
#pragma unroll
          for (int u = 0; u < 4; ++u)
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
      }
      if (lane == 0) bulk_wait_group0();
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int D>
static cudaError_t launch2(const PrefillArgs &a, const CUtensorMap &tq, const CUtensorMap &tk,
                           const CUtensorMap &tv, const CUtensorMap &tc, const CUtensorMap &to,
                           cudaStream_t stream) {
  static cudaError_t attr = cudaFuncSetAttribute(prefill2q_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)Smem2<D>::ALLOC);
  if (attr != cudaSuccess) return attr;
  prefill2q_kernel<D><<<dim3(a.num_q_tiles, a.n_loc, a.num_seqs), kThreads, Smem2<D>::ALLOC, stream>>>(tq, tk, tv,
                                                                                                       tc, to, a);
  return cudaGetLastError();
}

}  // namespace

// a.num_q_tiles = number of q-tile PAIRS (256 rows); K/V maps with 128-row boxes
cudaError_t launch_prefill2q(const PrefillArgs &a, const CUtensorMap &tm_q, const CUtensorMap &tm_k,
                             const CUtensorMap &tm_v, const CUtensorMap &tm_cache, const CUtensorMap &tm_o,
                             int head_dim, cudaStream_t stream) {
  return head_dim == 128 ? launch2<128>(a, tm_q, tm_k, tm_v, tm_cache, tm_o, stream)
                         : launch2<64>(a, tm_q, tm_k, tm_v, tm_cache, tm_o, stream);
}

}  // namespace ds
