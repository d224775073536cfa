// Attention with the score buffers triple-buffered in tensor memory (padded
// head dims <= 80: C2 / C3 / PixArt dh 72, SD3 dh 64).
//
// Same contract, layouts, stream-K schedule, segment epilogues and partial
// formats as attn_fwd_kernel (attn_sm100.cuh, which documents them); the
// difference is the pipeline between the MMA warp and the softmax warps.
// There, each query tile owns one 128-column S buffer: S_{t,i+1} can only be
// computed after the softmax of block i stored P_{t,i} over S_{t,i}, so every
// block the softmax waits ~650 clk for the MMA (measured, tools/attn_trace.py)
// and the tensor pipe idles during the exp section. Here the KV block is 112
// rows and the two tiles share THREE 112-column S buffers in rotation (the
// global sequence n = 2 i + t of (block, tile) pairs uses buffer n % 3), so
// the MMA warp computes the scores of the next (block, tile) while the
// softmax of the current one runs; TMEM = 3 x 112 S + 2 x 80 O <= 512
// columns. Because S_{n+3} is issued before PV_{n+1}, an O rescale waits for
// the previous block's PV explicitly (pv_done).
#pragma once

#include "attn_sm100.cuh"

namespace pf {

constexpr int kAttn3Buf = 3;   // S buffers
// kv rows per block: the widest multiple of 16 with 3 S buffers + 2 O tiles
// in the 512 TMEM columns (dhp <= 80: 112; dhp 96 / 112 / 128: 96 / 80 / 64)
__host__ __device__ constexpr int attn3_bn(int dhp) {
  return dhp <= 80 ? 112 : ((512 - 2 * dhp) / 3) / 16 * 16;
}
constexpr int kAttn3BN = 112;  // dhp <= 80

template <int DHP>
struct Attn3Smem {
  static constexpr int BN = attn3_bn(DHP);
  static constexpr int NT = 2;
  static constexpr uint32_t kQBytes = kAttnBM * DHP * 2;
  static constexpr uint32_t kQAlloc = (kQBytes + 1023) & ~1023u;
  static constexpr uint32_t kKVBytes = BN * DHP * 2;
  static constexpr uint32_t kKVAlloc = (kKVBytes + 1023) & ~1023u;
  static constexpr uint32_t kBudget = 232448 - 1024 - 512 - 16 * kAttnMaxSegs;
  static constexpr int kStagesMax = int((kBudget - NT * kQAlloc) / (2 * kKVAlloc));
  static constexpr int kStages = kStagesMax > 6 ? 6 : kStagesMax;
  static constexpr uint32_t kQOff = 0;
  static constexpr uint32_t kKOff = NT * kQAlloc;
  static constexpr uint32_t kVOff = kKOff + kStages * kKVAlloc;
  static constexpr uint32_t kBarOff = kVOff + kStages * kKVAlloc;
  static constexpr uint32_t kSegOff = kBarOff + 512;
  static constexpr uint32_t kTotal = kSegOff + 16 * kAttnMaxSegs + 1024;
  static constexpr int kThreads = 128 + 128 * NT;
  // TMEM columns: S buffer b at BN b, O_t at kOCol + kOW t
  static constexpr uint32_t kOW = DHP <= 80 ? 80 : DHP;
  static constexpr uint32_t kOCol = 512 - 2 * kOW;
  static_assert(DHP % 16 == 0 && DHP <= 128 && BN % 16 == 0 && BN >= 32, "attn3 shapes");
  static_assert(kOCol + 2 * kOW <= 512 && kAttn3Buf * BN <= int(kOCol), "TMEM budget");
  static_assert(kStages >= 2, "attention smem budget");
  static_assert(kTotal <= 232448, "attention smem budget");
};

template <int DHP, int kPoly, bool kSumCol>
__global__ void __launch_bounds__(384, 1)
    attn3_fwd_kernel(const __grid_constant__ CUtensorMap tm_q,
                     const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, AttnParams prm) {
  using L = Attn3Smem<DHP>;
  constexpr int NT = 2;
  constexpr int S = L::kStages;
  constexpr int BN = L::BN;
  constexpr int kChunks = DHP / 16;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + L::kQOff;
  uint8_t* sK = smem + L::kKOff;
  uint8_t* sV = smem + L::kVOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;                 // [S]
  uint64_t* k_empty = k_full + S;              // [S]
  uint64_t* v_full = k_empty + S;              // [S]
  uint64_t* v_empty = v_full + S;              // [S]
  uint64_t* s_full = v_empty + S;              // [3]   S buffer b written
  // [NT][2] P_t of a block stored (softmax -> MMA), by block parity: with the
  // next block's scores already computed, a fast warp may finish block i + 1
  // before a slow one finished block i, and its arrivals must not complete
  // block i's phase (it cannot get two blocks ahead: S of block i + 2 is
  // issued after PV of block i)
  uint64_t* p_full = s_full + kAttn3Buf;
  uint64_t* pv_done = p_full + 2 * NT;         // [NT]  PV_t of a block complete
  uint64_t* o_done = pv_done + NT;             // [NT]  last PV_t of a segment complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + NT);
  int* nseg_slot = reinterpret_cast<int*>(tmem_slot + 1);
  int4* segs = reinterpret_cast<int4*>(smem + L::kSegOff);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = ptx::lane_id();
  struct Seg {
    int x, b0, n;
  };
  const int B = prm.blocks;
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tm_q);
    ptx::prefetch_tmap(&tm_k);
    ptx::prefetch_tmap(&tm_v);
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&k_full[s], 1);
      ptx::mbar_init(&k_empty[s], 1);
      ptx::mbar_init(&v_full[s], 1);
      ptx::mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < kAttn3Buf; ++b) ptx::mbar_init(&s_full[b], 1);
    for (int t = 0; t < NT; ++t) {
      ptx::mbar_init(&p_full[2 * t], 128);
      ptx::mbar_init(&p_full[2 * t + 1], 128);
      ptx::mbar_init(&pv_done[t], 1);
      ptx::mbar_init(&o_done[t], 1);
    }
    ptx::fence_barrier_init();
    const long long u0 = prm.strided ? 0 : attn_unit_start(prm, blockIdx.x);
    const long long u1 = prm.strided ? 0 : attn_unit_start(prm, blockIdx.x + 1);
    int n = 0;
    if (prm.strided)
      for (long long x = blockIdx.x; x < prm.units / B && n < kAttnMaxSegs; x += prm.grid)
        segs[n++] = make_int4(int(x), 0, B, 0);
    for (long long u = u0; u < u1 && n < kAttnMaxSegs; ++n) {
      const int x = int(u / B);
      const int b0 = int(u - (long long)x * B);
      const int len = int(u1 - u < B - b0 ? u1 - u : B - b0);
      segs[n] = make_int4(x, b0, len, 0);
      u += len;
    }
    if (prm.fused)
      for (int i = 0; i < n / 2; ++i) {
        const int4 tmp = segs[i];
        segs[i] = segs[n - 1 - i];
        segs[n - 1 - i] = tmp;
      }
    *nseg_slot = n;
  }
  if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int nseg = *nseg_slot;
  const bool rev = prm.fused != 0;
  ptx::pdl_wait();
  ptx::pdl_launch();

  if (warp < 4) {
    ptx::setmaxnreg_dec<56>();
    if (warp == 0 && lane == 0) {
      // ------------------------------------------------------------ TMA
      int g = 0;
      for (int sgi = 0; sgi < nseg; ++sgi) {
        const int4 sg4 = segs[sgi];
        const Seg sg{sg4.x, sg4.y, sg4.z};
        const int head = sg.x / prm.nq;
        const int qt = sg.x - head * prm.nq;
        if (sgi > 0) ptx::mbar_wait(q_empty, (sgi - 1) & 1);
        const int qrow = head * prm.q_stride + prm.row0 + qt * (NT * kAttnBM);
        ptx::mbar_arrive_expect_tx(q_full, NT * L::kQBytes);
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int c = 0; c < kChunks; ++c)
            ptx::tma_load_2d(sQ + t * L::kQAlloc + c * (kAttnBM * 32), &tm_q, q_full, c * 16,
                             qrow + t * kAttnBM);
        for (int i = 0; i < sg.n; ++i, ++g) {
          const int s = g % S;
          const uint32_t ph = ((g / S) & 1) ^ 1;
          const int kvrow = head * prm.P + (sg.b0 + i) * BN;
          ptx::mbar_wait(&k_empty[s], ph);
          ptx::mbar_arrive_expect_tx(&k_full[s], L::kKVBytes);
#pragma unroll
          for (int c = 0; c < kChunks; ++c)
            ptx::tma_load_2d(sK + s * L::kKVAlloc + c * (BN * 32), &tm_k, &k_full[s], c * 16,
                             kvrow);
          ptx::mbar_wait(&v_empty[s], ph);
          ptx::mbar_arrive_expect_tx(&v_full[s], L::kKVBytes);
#pragma unroll
          for (int c = 0; c < kChunks; ++c)
            ptx::tma_load_2d(sV + s * L::kKVAlloc + c * (BN * 32), &tm_v, &v_full[s], c * 16,
                             kvrow);
        }
      }
    } else if (warp == 1 && lane == 0) {
      // ------------------------------------------------------------ MMA
      // Per segment the (block, tile) pairs n = 2 i + t run in order; S of
      // pair n + 3 is issued right after PV of pair n (it reuses n's buffer,
      // and tcgen05.mma from one thread execute in issue order).
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(kAttnBM, BN);
      constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(kAttnBM, DHP, /*b_mn_major=*/true);
      const uint32_t q_base = ptx::smem_u32(sQ);
      const uint32_t k_base = ptx::smem_u32(sK);
      const uint32_t v_base = ptx::smem_u32(sV);
      int gb = 0;    // global block counter (K/V ring, per-tile p_full parity)
      int gn = 0;    // global (block, tile) counter (S buffer rotation)
      for (int sgi = 0; sgi < nseg; ++sgi) {
        const int4 sg4 = segs[sgi];
        const int nb = sg4.z;
        const int N = 2 * nb;
        ptx::mbar_wait(q_full, sgi & 1);
        ptx::tc_fence_after();
        auto issue_s = [&](int n) {  // S of local pair n into buffer (gn + n) % 3
          const int i = n >> 1, t = n & 1;
          const int kg = gb + i;
          if (t == 0) {
            ptx::mbar_wait(&k_full[kg % S], (kg / S) & 1);
            ptx::tc_fence_after();
          }
          const uint32_t kb = k_base + (kg % S) * L::kKVAlloc;
          const uint32_t qb = q_base + t * L::kQAlloc;
          const uint32_t d = tmem_base + uint32_t(((gn + n) % kAttn3Buf) * BN);
#pragma unroll
          for (int c = 0; c < kChunks; ++c)
            ptx::umma_bf16_ss(d, ptx::desc_kmajor_sw32(qb + c * (kAttnBM * 32)),
                              ptx::desc_kmajor_sw32(kb + c * (BN * 32)), idesc_s, c != 0);
          ptx::umma_commit(&s_full[(gn + n) % kAttn3Buf]);
          if (t == 1) ptx::umma_commit(&k_empty[kg % S]);
          if (n == N - 1) ptx::umma_commit(q_empty);  // every S of the segment issued
        };
        for (int n = 0; n < 3 && n < N; ++n) issue_s(n);
        for (int n = 0; n < N; ++n) {
          const int i = n >> 1, t = n & 1;
          const int vg = gb + i;
          if (t == 0) {
            ptx::mbar_wait(&v_full[vg % S], (vg / S) & 1);
          }
          ptx::mbar_wait(&p_full[2 * t + (vg & 1)], (vg >> 1) & 1);
          ptx::tc_fence_after();
          const uint32_t vb = v_base + (vg % S) * L::kKVAlloc;
          const uint32_t pt = tmem_base + uint32_t(((gn + n) % kAttn3Buf) * BN) + BN / 2;
          const uint32_t od = tmem_base + L::kOCol + L::kOW * uint32_t(t);
#pragma unroll
          for (int k = 0; k < BN / 16; ++k)
            ptx::umma_bf16_ts(od, pt + 8 * k,
                              ptx::desc_mnmajor_sw32(vb + k * 16 * 32, BN * 32, 256), idesc_o,
                              !(i == 0 && k == 0));
          ptx::umma_commit(&pv_done[t]);
          if (t == 1) ptx::umma_commit(&v_empty[vg % S]);
          if (i == nb - 1) ptx::umma_commit(&o_done[t]);
          if (n + 3 < N) issue_s(n + 3);
        }
        gb += nb;
        gn += N;
      }
    }
  } else {
    ptx::setmaxnreg_inc<224>();
    // -------------------------------------------------------------- softmax
    const int t = (warp - 4) >> 2;
    const int q = warp & 3;
    const int trow = 32 * q + int(lane);
    const uint32_t lane_off = uint32_t(32 * q) << 16;
    const uint32_t tmem_o = tmem_base + L::kOCol + L::kOW * uint32_t(t) + lane_off;
    const float sc = prm.scale_log2;
    int gb = 0, gn = 0;
    int* pending_flag = nullptr;
    for (int sgi = 0; sgi < nseg; ++sgi) {
      const int4 sg4 = segs[sgi];
      const Seg sg{sg4.x, sg4.y, sg4.z};
      float m_ref = -INFINITY;
      float l_sum = 0.f;
      for (int i = 0; i < sg.n; ++i) {
        const int gnn = gn + 2 * i + t;
        const int buf = gnn % kAttn3Buf;
        const uint32_t tmem_s = tmem_base + uint32_t(buf * BN) + lane_off;
        const int kv0 = (sg.b0 + i) * BN;
        const bool tr = gb + i < 256;
        if (tr) attn_trace(prm, 2048 * t + 8 * (gb + i) + 0);
        ptx::mbar_wait(&s_full[buf], (gnn / kAttn3Buf) & 1);
        if (tr) attn_trace(prm, 2048 * t + 8 * (gb + i) + 1);
        ptx::tc_fence_after();
        uint32_t sr[BN];
#pragma unroll
        for (int c = 0; c + 32 <= BN; c += 32)
          ptx::tmem_ld32(tmem_s + c, *reinterpret_cast<uint32_t(*)[32]>(&sr[c]));
        if constexpr (BN % 32 == 16)
          ptx::tmem_ld16(tmem_s + (BN - 16), *reinterpret_cast<uint32_t(*)[16]>(&sr[BN - 16]));
        ptx::tmem_wait_ld();
        float* s = reinterpret_cast<float*>(sr);
        if (kv0 + BN > prm.P) {
          const int valid = prm.P - kv0;
#pragma unroll
          for (int e = 0; e < BN; ++e)
            if (e >= valid) s[e] = -INFINITY;
        }
        // row max: 8 chains of BN / 8 columns with FMNMX3
        float bm[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          bm[a] = s[a];
#pragma unroll
          for (int e = 8; e + 8 < BN; e += 16) bm[a] = ptx::fmax3(bm[a], s[e + a], s[e + 8 + a]);
          if constexpr ((BN / 8) % 2 == 0) bm[a] = fmaxf(bm[a], s[BN - 8 + a]);
        }
        const float bmax = fmaxf(ptx::fmax3(bm[0], bm[1], bm[2]),
                                 ptx::fmax3(bm[3], ptx::fmax3(bm[4], bm[5], bm[6]), bm[7])) * sc;
        const bool need = bmax > m_ref + 8.0f;
        const float m_new = need ? bmax : m_ref;
        const float alpha = need ? ptx::ex2_approx(m_ref - m_new) : 1.0f;
        if (tr) attn_trace(prm, 2048 * t + 8 * (gb + i) + 2);
        // the previous block's PV has landed in O (needed before a rescale;
        // waited every block so each pv_done phase is observed -- it is long
        // complete by now: S load and row max take longer than one tile's PV)
        if (gb + i > 0) ptx::mbar_wait(&pv_done[t], (gb + i - 1) & 1);
        if (i > 0 && __any_sync(0xffffffffu, need)) {
          ptx::tc_fence_after();
#pragma unroll
          for (int c = 0; c < kChunks; ++c) {
            uint32_t r[16];
            ptx::tmem_ld16(tmem_o + 16 * c, r);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
            ptx::tmem_st16(tmem_o + 16 * c, r);
          }
        }
        if (tr) attn_trace(prm, 2048 * t + 8 * (gb + i) + 3);
        // P = exp2(s sc - m) packed to bf16 pairs over the upper half of S
        const float2 sc2 = make_float2(sc, sc);
        const float2 nm2 = make_float2(-m_new, -m_new);
        const uint32_t tmem_p = tmem_s + BN / 2;
        constexpr int kParts = (BN + 31) / 32;  // 32 scores per part (the last may be 16)
#pragma unroll
        for (int part = 0; part < kParts; ++part) {
          const int plen = (32 * part + 32 <= BN) ? 32 : BN - 32 * part;
          uint32_t pk[16];
#pragma unroll
          for (int gg = 0; gg < 8; ++gg) {
            if (4 * gg >= plen) break;
            const int e = 32 * part + 4 * gg;
            const int grp = (e / 4) & 7;
            const float2 x0 = ptx::ffma2(make_float2(s[e], s[e + 1]), sc2, nm2);
            const float2 x1 = ptx::ffma2(make_float2(s[e + 2], s[e + 3]), sc2, nm2);
            float2 p0, p1;
            if ((kPoly >> grp) & 1) {
              p0 = ptx::ex2_poly2(x0);
              p1 = ptx::ex2_poly2(x1);
            } else {
              p0 = make_float2(ptx::ex2_approx(x0.x), ptx::ex2_approx(x0.y));
              p1 = make_float2(ptx::ex2_approx(x1.x), ptx::ex2_approx(x1.y));
            }
            if constexpr (!kSumCol) {
              s[e] = p0.x; s[e + 1] = p0.y; s[e + 2] = p1.x; s[e + 3] = p1.y;
            }
            pk[2 * gg] = ptx::pack_bf16x2(p0.x, p0.y);
            pk[2 * gg + 1] = ptx::pack_bf16x2(p1.x, p1.y);
          }
          if (plen == 32) {
            ptx::tmem_st16(tmem_p + 16 * part, pk);
          } else {
            ptx::tmem_st8(tmem_p + 16 * part, *reinterpret_cast<const uint32_t(*)[8]>(&pk[0]));
          }
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&p_full[2 * t + ((gb + i) & 1)]);
        if (pending_flag) {
          __syncwarp();
          if (lane == 0) ptx::st_release_gpu(pending_flag, 1);
          pending_flag = nullptr;
        }
        if (tr) attn_trace(prm, 2048 * t + 8 * (gb + i) + 4);
        if constexpr (!kSumCol) {
          float2 a0 = make_float2(0.f, 0.f), a1 = a0;
#pragma unroll
          for (int e = 0; e < BN; e += 4) {
            a0 = ptx::fadd2(a0, make_float2(s[e], s[e + 1]));
            a1 = ptx::fadd2(a1, make_float2(s[e + 2], s[e + 3]));
          }
          a0 = ptx::fadd2(a0, a1);
          l_sum = l_sum * alpha + (a0.x + a0.y);
        }
        m_ref = m_new;
        if (tr) attn_trace(prm, 2048 * t + 8 * (gb + i) + 5);
      }
      gb += sg.n;
      gn += 2 * sg.n;

      // Segment epilogue (as attn_fwd_kernel)
      ptx::mbar_wait(&o_done[t], sgi & 1);
      ptx::tc_fence_after();
      if constexpr (kSumCol) {
        uint32_t r[16];
        ptx::tmem_ld16(tmem_o + 16 * (prm.dh / 16), r);
        ptx::tmem_wait_ld();
        const int cd = prm.dh % 16;
        float lv = 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (j == cd) lv = __uint_as_float(r[j]);
        l_sum = lv;
      }
      const int head = sg.x / prm.nq;
      const int qt = sg.x - head * prm.nq;
      const int lrow = qt * (NT * kAttnBM) + t * kAttnBM + trow;
      const bool row_ok = lrow < prm.rows;
      const bool vec = (prm.dh % 8 == 0) && (prm.hs % 8 == 0);
      __nv_bfloat16* orow = prm.out + size_t(prm.row0 + lrow) * prm.hs + size_t(head) * prm.dh;
      auto store16 = [&](int c, const float (&o)[16]) {
        if (!row_ok) return;
        if (vec) {
#pragma unroll
          for (int e = 0; e < 16; e += 8) {
            const int d = 16 * c + e;
            if (d < prm.dh) {
              uint4 v;
              v.x = ptx::pack_bf16x2(o[e], o[e + 1]);
              v.y = ptx::pack_bf16x2(o[e + 2], o[e + 3]);
              v.z = ptx::pack_bf16x2(o[e + 4], o[e + 5]);
              v.w = ptx::pack_bf16x2(o[e + 6], o[e + 7]);
              *reinterpret_cast<uint4*>(orow + d) = v;
            }
          }
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int d = 16 * c + e;
            if (d < prm.dh) orow[d] = __float2bfloat16_rn(o[e]);
          }
        }
      };
      if (sg.n == B) {
        const float inv_l = 1.0f / l_sum;
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
          uint32_t r[16];
          ptx::tmem_ld16(tmem_o + 16 * c, r);
          ptx::tmem_wait_ld();
          float o[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) o[j] = __uint_as_float(r[j]) * inv_l;
          store16(c, o);
        }
      } else if (rev && sg.b0 > 0) {
        const int c0 = int(blockIdx.x);
        const int wflag = (c0 - 1) * kAttnFlagsPerCta + (warp - 4);
        if (lane == 0) {
          while (ptx::ld_acquire_gpu(prm.flags + wflag) == 0) __nanosleep(32);
          prm.flags[wflag] = 0;
        }
        __syncwarp();
        const int prow = t * kAttnBM + trow;
        const size_t sbase = size_t(2 * (c0 - 1) + 1);
        const float m2 = prm.part_ml[(sbase * 2 + 0) * (NT * kAttnBM) + prow];
        const float l2 = prm.part_ml[(sbase * 2 + 1) * (NT * kAttnBM) + prow];
        const float mm = fmaxf(m_ref, m2);
        const float w1 = ptx::ex2_approx(m_ref - mm), w2 = ptx::ex2_approx(m2 - mm);
        const float inv_l = 1.0f / (w1 * l_sum + w2 * l2);
        const float a1 = w1 * inv_l, a2 = w2 * inv_l;
        const float* po = prm.part_o + sbase * DHP * (NT * kAttnBM) + prow;
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
          uint32_t r[16];
          ptx::tmem_ld16(tmem_o + 16 * c, r);
          float pv[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) pv[j] = po[size_t(16 * c + j) * (NT * kAttnBM)];
          ptx::tmem_wait_ld();
          float o[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) o[j] = a1 * __uint_as_float(r[j]) + a2 * pv[j];
          store16(c, o);
        }
      } else {
        const int slot = 2 * int(blockIdx.x) + (sgi == 0 && !rev ? 0 : 1);
        const int prow = t * kAttnBM + trow;
        float* po = prm.part_o + size_t(slot) * DHP * (NT * kAttnBM) + prow;
        uint32_t r[kChunks][16];
#pragma unroll
        for (int c = 0; c < kChunks; ++c) ptx::tmem_ld16(tmem_o + 16 * c, r[c]);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < kChunks; ++c)
#pragma unroll
          for (int e = 0; e < 16; ++e)
            po[size_t(16 * c + e) * (NT * kAttnBM)] = __uint_as_float(r[c][e]);
        prm.part_ml[(size_t(slot) * 2 + 0) * (NT * kAttnBM) + prow] = m_ref;
        prm.part_ml[(size_t(slot) * 2 + 1) * (NT * kAttnBM) + prow] = l_sum;
        if (rev) pending_flag = prm.flags + int(blockIdx.x) * kAttnFlagsPerCta + (warp - 4);
      }
    }
    if (pending_flag) {
      __syncwarp();
      if (lane == 0) ptx::st_release_gpu(pending_flag, 1);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace pf
