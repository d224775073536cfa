// Fresh-patch attention over a stage's full-sequence K/V buffer (tcgen05).
//
// Replaces `attention_rows` (/root/reference/proj/src/toy_model.cpp:104-143):
// per query row and head, softmax(q.k / sqrt(dh)) over ALL kv rows of the
// buffer (rows of other patches are stale or fresh depending on the pipeline
// position; zero rows are real rows, never masked), times V.
//
// Layout (HBM, per stage and local layer; dhp = dh rounded up to 16, padding
// columns are zero):
//   Q  [heads][P][dhp]  bf16   K-major A operand of S = Q K^T
//   K  [heads][P][dhp]  bf16   K-major B operand of S = Q K^T
//   V  [heads][P][dhp]  bf16   MN-major B operand of O = P V (no transpose)
//   out[P][hs]          bf16   row-major, column head*dh + d
// Q/K/V tiles arrive by TMA as dhp/16 column chunks of [128 rows x 32 B]
// (SWIZZLE_32B atoms), which serve both as K-major (Q, K) and MN-major (V)
// UMMA operands.
//
// One CTA = 128 query rows x one head x one kv split. Roles (256 threads):
//   warp 0      TMA producer: Q once, then K_i and V_i in separate rings
//   warp 1      MMA issuer: S_i = Q K_i^T into TMEM (double-buffered), then
//               O += P_{i-1} V_{i-1} (TMEM accumulator); K slots are released
//               as soon as S_i completes, V slots after PV_i
//   warp 2      TMEM allocator
//   warps 4..7  softmax: one query row per thread; online softmax in fp32 with
//               lazy rescaling (O and l are rescaled only when the running max
//               grows by more than 2^8), P written as bf16 into a
//               double-buffered 128B-swizzled smem tile.
// With kv_splits > 1 each split writes an unnormalised partial (O, m, l) in
// fp32 and `attn_combine_kernel` merges the splits in a fixed order.
#pragma once

#include "sm100_ptx.cuh"

namespace pf {

constexpr int kAttnBM = 128;   // query rows per CTA
constexpr int kAttnBN = 128;   // kv rows per block

template <int DHP>
struct AttnSmem {
  static constexpr int kStages = DHP <= 80 ? 3 : 2;
  static constexpr uint32_t kTileBytes = kAttnBM * DHP * 2;  // Q, K or V tile
  static constexpr uint32_t kPBytes = kAttnBM * kAttnBN * 2;  // 32 KB
  static constexpr uint32_t kQOff = 0;
  static constexpr uint32_t kKOff = (kTileBytes + 1023) & ~1023u;
  static constexpr uint32_t kVOff = kKOff + kStages * kKOff;
  static constexpr uint32_t kPOff = kVOff + kStages * kKOff;
  static constexpr uint32_t kBarOff = kPOff + 2 * kPBytes;
  static constexpr uint32_t kTotal = kBarOff + 512 + 1024;
  static_assert(DHP % 16 == 0 && DHP <= 128, "head dim padding");
  static_assert(kTotal <= 232448, "attention smem budget");
};

struct AttnParams {
  int P;            // kv rows in the buffer (= sequence length)
  int rows;         // query rows this launch
  int row0;         // first query row
  int heads, dh, hs;
  float scale_log2; // log2(e) / sqrt(dh)
  int kv_splits;    // >= 1
  int blocks_per_split;
  __nv_bfloat16* out;  // [P][hs]   (used when kv_splits == 1)
  float* part_o;       // [splits][heads][rows_pad][DHP] (kv_splits > 1)
  float* part_ml;      // [splits][heads][rows_pad][2]
  int rows_pad;        // q_tiles * 128
};

template <int DHP>
__global__ void __launch_bounds__(256, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q,
                    const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, AttnParams prm) {
  using L = AttnSmem<DHP>;
  constexpr int S = L::kStages;
  constexpr int kChunks = DHP / 16;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + L::kQOff;
  uint8_t* sK = smem + L::kKOff;
  uint8_t* sV = smem + L::kVOff;
  uint8_t* sP = smem + L::kPOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;       // [S]
  uint64_t* k_empty = k_full + S;    // [S]
  uint64_t* v_full = k_empty + S;    // [S]
  uint64_t* v_empty = v_full + S;    // [S]
  uint64_t* s_full = v_empty + S;    // [2]
  uint64_t* s_empty = s_full + 2;    // [2]
  uint64_t* p_full = s_empty + 2;    // [2]
  uint64_t* pv_done = p_full + 2;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = ptx::lane_id();
  const int qt = blockIdx.x;
  const int head = blockIdx.y;
  const int split = blockIdx.z;
  const int total_blocks = (prm.P + kAttnBN - 1) / kAttnBN;
  const int blk_begin = split * prm.blocks_per_split;
  int blk_end = blk_begin + prm.blocks_per_split;
  if (blk_end > total_blocks) blk_end = total_blocks;
  const int nblk = blk_end - blk_begin;  // >= 1 by construction

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tm_q);
    ptx::prefetch_tmap(&tm_k);
    ptx::prefetch_tmap(&tm_v);
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&k_full[s], 1);
      ptx::mbar_init(&k_empty[s], 1);
      ptx::mbar_init(&v_full[s], 1);
      ptx::mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&s_full[b], 1);
      ptx::mbar_init(&s_empty[b], 128);
      ptx::mbar_init(&p_full[b], 128);
      ptx::mbar_init(&pv_done[b], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tmem_o = tmem_base + 256;

  if (warp == 0) {
    if (lane == 0) {
      const int qrow = head * prm.P + prm.row0 + qt * kAttnBM;
      ptx::mbar_arrive_expect_tx(q_full, L::kTileBytes);
#pragma unroll
      for (int c = 0; c < kChunks; ++c)
        ptx::tma_load_2d(sQ + c * (kAttnBM * 32), &tm_q, q_full, c * 16, qrow);
      for (int i = 0; i < nblk; ++i) {
        const int s = i % S;
        const uint32_t ph = ((i / S) & 1) ^ 1;
        const int kvrow = head * prm.P + (blk_begin + i) * kAttnBN;
        ptx::mbar_wait(&k_empty[s], ph);
        ptx::mbar_arrive_expect_tx(&k_full[s], L::kTileBytes);
#pragma unroll
        for (int c = 0; c < kChunks; ++c)
          ptx::tma_load_2d(sK + s * L::kKOff + c * (kAttnBN * 32), &tm_k, &k_full[s],
                           c * 16, kvrow);
        ptx::mbar_wait(&v_empty[s], ph);
        ptx::mbar_arrive_expect_tx(&v_full[s], L::kTileBytes);
#pragma unroll
        for (int c = 0; c < kChunks; ++c)
          ptx::tma_load_2d(sV + s * L::kKOff + c * (kAttnBN * 32), &tm_v, &v_full[s],
                           c * 16, kvrow);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(kAttnBM, kAttnBN);
      constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(kAttnBM, DHP, /*b_mn_major=*/true);
      const uint32_t q_base = ptx::smem_u32(sQ);
      const uint32_t k_base = ptx::smem_u32(sK);
      const uint32_t v_base = ptx::smem_u32(sV);
      const uint32_t p_base = ptx::smem_u32(sP);
      ptx::mbar_wait(q_full, 0);

      auto issue_pv = [&](int j) {
        const int b = j & 1;
        const int s = j % S;
        ptx::mbar_wait(&v_full[s], (j / S) & 1);
        ptx::mbar_wait(&p_full[b], (j >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t pb = p_base + b * L::kPBytes;
        const uint32_t vb = v_base + s * L::kKOff;
#pragma unroll
        for (int k = 0; k < kAttnBN / 16; ++k) {
          // A: P rows x 16 kv (SW128 K-major, 64 kv per atom column)
          // B: V 16 kv rows x DHP (SW32 MN-major: LBO = next 16-col chunk,
          //    SBO = next 8 kv rows)
          ptx::umma_bf16_ss(tmem_o,
                            ptx::desc_kmajor_sw128(pb + (k >> 2) * (kAttnBM * 128) + (k & 3) * 32),
                            ptx::desc_mnmajor_sw32(vb + k * 16 * 32, kAttnBN * 32, 256),
                            idesc_o, (j | k) != 0);
        }
        ptx::umma_commit(&pv_done[b]);
        ptx::umma_commit(&v_empty[s]);
      };

      for (int i = 0; i < nblk; ++i) {
        const int s = i % S;
        const int b = i & 1;
        ptx::mbar_wait(&k_full[s], (i / S) & 1);
        if (i >= 2) ptx::mbar_wait(&s_empty[b], ((i >> 1) - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t kb = k_base + s * L::kKOff;
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
          ptx::umma_bf16_ss(tmem_base + b * kAttnBN,
                            ptx::desc_kmajor_sw32(q_base + c * (kAttnBM * 32)),
                            ptx::desc_kmajor_sw32(kb + c * (kAttnBN * 32)),
                            idesc_s, c != 0);
        }
        ptx::umma_commit(&s_full[b]);
        ptx::umma_commit(&k_empty[s]);
        if (i >= 1) issue_pv(i - 1);
      }
      issue_pv(nblk - 1);
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int trow = 32 * q + int(lane);  // row within the tile == TMEM lane
    const uint32_t lane_off = uint32_t(32 * q) << 16;
    const float sc = prm.scale_log2;
    float m_ref = -INFINITY;  // running (lazy) max, scaled log2 domain
    float l_sum = 0.f;
    for (int i = 0; i < nblk; ++i) {
      const int b = i & 1;
      const int kv0 = (blk_begin + i) * kAttnBN;
      ptx::mbar_wait(&s_full[b], (i >> 1) & 1);
      ptx::tc_fence_after();
      uint32_t sr[kAttnBN];
#pragma unroll
      for (int c = 0; c < kAttnBN / 32; ++c)
        ptx::tmem_ld32(tmem_base + lane_off + b * kAttnBN + 32 * c,
                       *reinterpret_cast<uint32_t(*)[32]>(&sr[32 * c]));
      ptx::tmem_wait_ld();
      // S buffer b may be overwritten by S_{i+2} now.
      ptx::tc_fence_before();
      ptx::mbar_arrive(&s_empty[b]);

      float* s = reinterpret_cast<float*>(sr);
      if (kv0 + kAttnBN > prm.P) {  // kv rows past the buffer end are masked
        const int valid = prm.P - kv0;
#pragma unroll
        for (int e = 0; e < kAttnBN; ++e)
          if (e >= valid) s[e] = -INFINITY;
      }
      float bm0 = s[0], bm1 = s[1];
#pragma unroll
      for (int e = 2; e < kAttnBN; e += 2) {
        bm0 = fmaxf(bm0, s[e]);
        bm1 = fmaxf(bm1, s[e + 1]);
      }
      const float bm = fmaxf(bm0, bm1) * sc;
      const bool need = bm > m_ref + 8.0f;
      const float m_new = need ? bm : m_ref;
      const float alpha = need ? ptx::ex2_approx(m_ref - m_new) : 1.0f;  // 0 on first block
      if (__any_sync(0xffffffffu, need) && i > 0) {
        // O accumulated through PV_{i-1}: wait for it, then rescale in TMEM.
        ptx::mbar_wait(&pv_done[(i - 1) & 1], ((i - 1) >> 1) & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
          uint32_t r[16];
          ptx::tmem_ld16(tmem_o + lane_off + 16 * c, r);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
          ptx::tmem_st16(tmem_o + lane_off + 16 * c, r);
        }
        ptx::tmem_wait_st();
      }
      l_sum *= alpha;
      m_ref = m_new;

      // P_{i-2} (same smem buffer) must have been consumed by PV_{i-2}.
      if (i >= 2) ptx::mbar_wait(&pv_done[b], ((i - 2) >> 1) & 1);
      uint8_t* pbuf = sP + b * L::kPBytes;
      float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int e0 = 64 * h + 8 * c;
          float p[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) p[e] = ptx::ex2_approx(fmaf(s[e0 + e], sc, -m_new));
          ls0 += (p[0] + p[1]) + (p[2] + p[3]);
          ls1 += (p[4] + p[5]) + (p[6] + p[7]);
          uint4 v;
          v.x = ptx::pack_bf16x2(p[0], p[1]);
          v.y = ptx::pack_bf16x2(p[2], p[3]);
          v.z = ptx::pack_bf16x2(p[4], p[5]);
          v.w = ptx::pack_bf16x2(p[6], p[7]);
          const int chunk = c ^ (trow & 7);
          *reinterpret_cast<uint4*>(pbuf + h * (kAttnBM * 128) + trow * 128 + chunk * 16) = v;
        }
      }
      l_sum += ls0 + ls1;
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&p_full[b]);
    }

    // Epilogue: wait for the last PV, read O, normalise, store.
    ptx::mbar_wait(&pv_done[(nblk - 1) & 1], ((nblk - 1) >> 1) & 1);
    ptx::tc_fence_after();
    const bool row_ok = qt * kAttnBM + trow < prm.rows;
    const int grow = prm.row0 + qt * kAttnBM + trow;  // global query row
    if (prm.kv_splits == 1) {
      const float inv_l = 1.0f / l_sum;
      __nv_bfloat16* orow = prm.out + size_t(grow) * prm.hs + size_t(head) * prm.dh;
      const bool vec = (prm.dh % 8 == 0) && (prm.hs % 8 == 0);
#pragma unroll
      for (int c = 0; c < kChunks; ++c) {
        uint32_t r[16];
        ptx::tmem_ld16(tmem_o + lane_off + 16 * c, r);
        ptx::tmem_wait_ld();
        if (row_ok) {
          if (vec) {
#pragma unroll
            for (int e = 0; e < 16; e += 8) {
              const int d = 16 * c + e;
              if (d < prm.dh) {
                uint4 v;
                v.x = ptx::pack_bf16x2(__uint_as_float(r[e]) * inv_l, __uint_as_float(r[e + 1]) * inv_l);
                v.y = ptx::pack_bf16x2(__uint_as_float(r[e + 2]) * inv_l, __uint_as_float(r[e + 3]) * inv_l);
                v.z = ptx::pack_bf16x2(__uint_as_float(r[e + 4]) * inv_l, __uint_as_float(r[e + 5]) * inv_l);
                v.w = ptx::pack_bf16x2(__uint_as_float(r[e + 6]) * inv_l, __uint_as_float(r[e + 7]) * inv_l);
                *reinterpret_cast<uint4*>(orow + d) = v;
              }
            }
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int d = 16 * c + e;
              if (d < prm.dh) orow[d] = __float2bfloat16_rn(__uint_as_float(r[e]) * inv_l);
            }
          }
        }
      }
    } else {
      const size_t prow = (size_t(split) * prm.heads + head) * prm.rows_pad + qt * kAttnBM + trow;
      float* po = prm.part_o + prow * DHP;
#pragma unroll
      for (int c = 0; c < kChunks; ++c) {
        uint32_t r[16];
        ptx::tmem_ld16(tmem_o + lane_off + 16 * c, r);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; e += 4)
          *reinterpret_cast<float4*>(po + 16 * c + e) =
              make_float4(__uint_as_float(r[e]), __uint_as_float(r[e + 1]),
                          __uint_as_float(r[e + 2]), __uint_as_float(r[e + 3]));
      }
      prm.part_ml[prow * 2 + 0] = m_ref;
      prm.part_ml[prow * 2 + 1] = l_sum;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem_base);
  }
}

// Merge kv splits in ascending split order (deterministic).
// One thread per (query row, head, 16-column chunk).
template <int DHP>
__global__ void attn_combine_kernel(AttnParams prm) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int chunks = DHP / 16;
  const int total = prm.rows * prm.heads * chunks;
  if (idx >= total) return;
  const int c = idx % chunks;
  const int head = (idx / chunks) % prm.heads;
  const int r = idx / (chunks * prm.heads);
  float m = -INFINITY;
  for (int sp = 0; sp < prm.kv_splits; ++sp) {
    const size_t prow = (size_t(sp) * prm.heads + head) * prm.rows_pad + r;
    m = fmaxf(m, prm.part_ml[prow * 2]);
  }
  float acc[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) acc[e] = 0.f;
  float l = 0.f;
  for (int sp = 0; sp < prm.kv_splits; ++sp) {
    const size_t prow = (size_t(sp) * prm.heads + head) * prm.rows_pad + r;
    const float w = ptx::ex2_approx(prm.part_ml[prow * 2] - m);
    l += w * prm.part_ml[prow * 2 + 1];
    const float* po = prm.part_o + prow * DHP + 16 * c;
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] += w * po[e];
  }
  const float inv_l = 1.0f / l;
  __nv_bfloat16* orow = prm.out + size_t(prm.row0 + r) * prm.hs + size_t(head) * prm.dh;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int d = 16 * c + e;
    if (d < prm.dh) orow[d] = __float2bfloat16_rn(acc[e] * inv_l);
  }
}

}  // namespace pf
