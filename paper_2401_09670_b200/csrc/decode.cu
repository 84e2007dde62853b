// decode.cu — a7 + a8: one decode step of one layer over a paged KV cache.
//
// PAPER.md P:233 (decode generates one token at a time reusing the KV cache),
// P:237 (batching), P:696-698 (decode attention is memory-bound: it streams the
// whole cached K/V once per step). Reading R9: the new token's K/V are appended
// at position c before attending, so the step attends c+1 tokens.
//
// B200 design (HBM-bound, no tensor cores — each cached element is used once):
//  * one CTA of 4 warps per (sequence, head, split); a split is a contiguous
//    range of 16-token pages; splits are only used when B*n_loc cannot fill the
//    148 SMs, and their partials are merged by a log-sum-exp combine (a8);
//  * each warp owns whole pages: its lanes form 32/TPG token groups of TPG =
//    head_dim/8 lanes; a lane loads 16 B (8 bf16) of a K row and of a V row
//    with 128-bit non-allocating loads, all 2x(16/ (32/TPG)) loads of a page
//    issued before use (one page of K and V = 8 KiB in flight per warp);
//  * q.k partial dots are reduced with xor-shuffles inside the TPG-lane group;
//    online softmax in base 2 (scale*log2 e folded into q), one rescale per
//    page; groups, warps and splits are merged with the same (m, l, o) rule.
//  * the append (i) is fused: the CTA whose split holds position c writes
//    k_new/v_new into the page and uses them from registers for token c.
#include "common.cuh"
#include "kernels.h"

namespace ds {

namespace {

constexpr int kWarps = 4;
constexpr float kNegInf = -__builtin_huge_valf();

DS_DEVICE uint4 ld_nc_v4(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

DS_DEVICE float dot8(const float (&q)[8], const uint4 &k) {
  float s = q[0] * bf16lo(k.x);
  s = fmaf(q[1], bf16hi(k.x), s);
  s = fmaf(q[2], bf16lo(k.y), s);
  s = fmaf(q[3], bf16hi(k.y), s);
  s = fmaf(q[4], bf16lo(k.z), s);
  s = fmaf(q[5], bf16hi(k.z), s);
  s = fmaf(q[6], bf16lo(k.w), s);
  s = fmaf(q[7], bf16hi(k.w), s);
  return s;
}

DS_DEVICE void axpy8(float (&acc)[8], float p, const uint4 &v) {
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

template <int D>
__global__ void __launch_bounds__(kWarps * 32)
    decode_split_kernel(const DecodeArgs a) {
  constexpr int TPG = D / 8;        // lanes per token row
  constexpr int GPW = 32 / TPG;     // token groups per warp
  constexpr int NIT = 16 / GPW;     // loads per lane per page (K and V each)
  const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / TPG, dpart = lane % TPG;

  const int c = a.cache_lens[b];
  const int npages = (c + 1 + 15) >> 4;
  const int p_begin = split * a.pages_per_split;
  const int p_end = min(npages, p_begin + a.pages_per_split);
  if (p_begin >= p_end) return;  // empty split (combine skips it)

  const int n = a.n_loc;
  const size_t row_off = ((size_t)b * n + h) * D;  // [B][n][D]
  const size_t page_elems = 16 * D;
  const size_t kv_stride = (size_t)a.num_blocks * n * page_elems;  // K -> V
  const uint16_t *layer_base = a.cache + (size_t)a.layer * 2 * kv_stride;
  const int *bt = a.block_table + (size_t)b * a.max_blocks;
  const int c_page = c >> 4;

  // (i) fused append of the new token's K/V at position c (R9)
  if (c_page >= p_begin && c_page < p_end && warp == 0 && lane < 2 * TPG) {
    const int kv = lane / TPG, part = lane % TPG;
    const uint16_t *src = (kv ? a.v_new : a.k_new) + row_off + part * 8;
    uint16_t *dst = const_cast<uint16_t *>(layer_base) + kv * kv_stride +
                    ((size_t)bt[c_page] * n + h) * page_elems + (size_t)(c & 15) * D + part * 8;
    *reinterpret_cast<uint4 *>(dst) = *reinterpret_cast<const uint4 *>(src);
  }

  float q[8];
  {
    const uint4 qv = *reinterpret_cast<const uint4 *>(a.q + row_off + dpart * 8);
    const float s = a.scale_log2;
    q[0] = bf16lo(qv.x) * s; q[1] = bf16hi(qv.x) * s;
    q[2] = bf16lo(qv.y) * s; q[3] = bf16hi(qv.y) * s;
    q[4] = bf16lo(qv.z) * s; q[5] = bf16hi(qv.z) * s;
    q[6] = bf16lo(qv.w) * s; q[7] = bf16hi(qv.w) * s;
  }
  const uint16_t *knew = a.k_new + row_off + dpart * 8;
  const uint16_t *vnew = a.v_new + row_off + dpart * 8;

  float m = kNegInf, l = 0.f, acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;

  for (int p = p_begin + warp; p < p_end; p += kWarps) {
    const size_t pg = ((size_t)bt[p] * n + h) * page_elems;
    const uint16_t *kp = layer_base + pg + dpart * 8;
    const uint16_t *vp = layer_base + kv_stride + pg + dpart * 8;
    uint4 kr[NIT], vr[NIT];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int t = it * GPW + g, pos = p * 16 + t;
      const bool is_new = pos == c;
      kr[it] = is_new ? *reinterpret_cast<const uint4 *>(knew)
                      : ld_nc_v4(kp + (size_t)t * D);
    }
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int t = it * GPW + g, pos = p * 16 + t;
      const bool is_new = pos == c;
      vr[it] = is_new ? *reinterpret_cast<const uint4 *>(vnew)
                      : ld_nc_v4(vp + (size_t)t * D);
    }
    float s[NIT];
    float pmax = kNegInf;
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      float x = dot8(q, kr[it]);
#pragma unroll
      for (int off = TPG / 2; off >= 1; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
      const int pos = p * 16 + it * GPW + g;
      s[it] = pos <= c ? x : kNegInf;
      pmax = fmaxf(pmax, s[it]);
    }
    const float m_new = fmaxf(m, pmax);
    if (m_new != kNegInf) {
      const float alpha = rescale(m, m_new);
      l *= alpha;
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] *= alpha;
#pragma unroll
      for (int it = 0; it < NIT; ++it) {
        if (s[it] != kNegInf) {
          const float pr = ex2(s[it] - m_new);
          l += pr;
          axpy8(acc, pr, vr[it]);
        }
      }
      m = m_new;
    }
  }

  // merge the GPW token groups of the warp (lanes with equal ds)
#pragma unroll
  for (int off = TPG; off < 32; off <<= 1) {
    const float mo = __shfl_xor_sync(0xffffffffu, m, off);
    const float lo = __shfl_xor_sync(0xffffffffu, l, off);
    const float mm = fmaxf(m, mo);
    const float wa = rescale(m, mm), wb = rescale(mo, mm);
    l = l * wa + lo * wb;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float ao = __shfl_xor_sync(0xffffffffu, acc[e], off);
      acc[e] = acc[e] * wa + ao * wb;
    }
    m = mm;
  }

  // merge the warps through shared memory
  __shared__ float s_o[kWarps][D];
  __shared__ float s_ml[kWarps][2];
  if (lane < TPG) {
#pragma unroll
    for (int e = 0; e < 8; ++e) s_o[warp][dpart * 8 + e] = acc[e];
    if (lane == 0) {
      s_ml[warp][0] = m;
      s_ml[warp][1] = l;
    }
  }
  __syncthreads();
  if (threadIdx.x < D) {
    const int t = threadIdx.x;
    float mm = kNegInf;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) mm = fmaxf(mm, s_ml[w][0]);
    float lt = 0.f, ot = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float wt = rescale(s_ml[w][0], mm);
      lt += s_ml[w][1] * wt;
      ot += s_o[w][t] * wt;
    }
    if (a.num_splits == 1) {
      reinterpret_cast<__nv_bfloat16 *>(a.out)[row_off + t] = __float2bfloat16_rn(ot / lt);
    } else {
      float *ws = a.workspace + (((size_t)b * n + h) * a.num_splits + split) * (D + 2);
      ws[t] = ot;
      if (t == 0) {
        ws[D] = mm;
        ws[D + 1] = lt;
      }
    }
  }
}

// a8: log-sum-exp merge of the split partials:
//   m* = max_k m_k ; l* = sum_k l_k 2^(m_k - m*) ; o = sum_k o_k 2^(m_k - m*) / l*
template <int D>
__global__ void __launch_bounds__(D) decode_combine_kernel(const DecodeArgs a) {
  const int h = blockIdx.x, b = blockIdx.y, t = threadIdx.x;
  const int c = a.cache_lens[b];
  const int npages = (c + 1 + 15) >> 4;
  const int active = (npages + a.pages_per_split - 1) / a.pages_per_split;
  const float *ws = a.workspace + ((size_t)b * a.n_loc + h) * a.num_splits * (D + 2);
  float mm = kNegInf;
  for (int k = 0; k < active; ++k) mm = fmaxf(mm, ws[k * (D + 2) + D]);
  float lt = 0.f, ot = 0.f;
  for (int k = 0; k < active; ++k) {
    const float w = rescale(ws[k * (D + 2) + D], mm);
    lt += ws[k * (D + 2) + D + 1] * w;
    ot += ws[k * (D + 2) + t] * w;
  }
  reinterpret_cast<__nv_bfloat16 *>(a.out)[((size_t)b * a.n_loc + h) * D + t] =
      __float2bfloat16_rn(ot / lt);
}

}  // namespace

cudaError_t launch_decode(const DecodeArgs &a, int head_dim, cudaStream_t stream) {
  dim3 grid(a.num_splits, a.n_loc, a.num_seqs);
  if (head_dim == 128) {
    decode_split_kernel<128><<<grid, kWarps * 32, 0, stream>>>(a);
    if (a.num_splits > 1)
      decode_combine_kernel<128><<<dim3(a.n_loc, a.num_seqs), 128, 0, stream>>>(a);
  } else {
    decode_split_kernel<64><<<grid, kWarps * 32, 0, stream>>>(a);
    if (a.num_splits > 1)
      decode_combine_kernel<64><<<dim3(a.n_loc, a.num_seqs), 64, 0, stream>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace ds
