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
// Work item = NT = 2 query tiles of 128 rows (sharing every K/V tile, which
// halves the L2->SM operand traffic per FLOP) x one head; its units are the
// item's 128-row KV blocks. Stream-K schedule: the items x blocks units are
// cut into `grid` equal contiguous ranges, one persistent CTA per range (one
// per SM), so no SM idles in a partial last wave (C2: 256 items over 148 SMs
// would otherwise take 2 full waves for 1.73 waves of work). A CTA walks its
// range as segments (item, [b0, b1)): a segment covering a whole item writes
// the normalised output; a cut segment writes an unnormalised fp32 partial
// (O, m, l) into slot 2c (the CTA's first segment) or 2c + 1 (its last), and
// `attn_streamk_combine_kernel` merges each cut item's partials in CTA order.
// When every range spans at least one item (`fused`: each item meets at most
// two CTAs) the merge happens in this kernel instead: CTAs walk their
// segments in reverse, so the head of a cut item (CTA c-1's last segment) is
// computed first and published (partial + release flag), and the tail
// (CTA c's first segment) is computed last and merged with it in the
// epilogue -- the flag is long set by then, and no CTA waits on a later one.
// The same in-kernel merge serves "halves" grids (exactly two CTAs per item,
// one head and one tail, for full sequences with few items), and patches
// whose items fit one wave run one CTA per item (no cuts); attn_grid
// (kernels.cu) picks the schedule from the shape only. Partials are stored column-major
// ([slot][d][row]: one 128-byte line per warp store), and each softmax warp
// releases its own flag one KV block after its stores were issued.
// Roles (384 threads):
//   warp 0        TMA producer: Q tiles once, then K_i and V_i in two rings
//   warp 1        MMA issuer: S_{t,i} = Q_t K_i^T (SS: both operands in smem)
//                 into TMEM, O_t += P_{t,i} V_i (TS: P read from TMEM)
//   warp 2        TMEM allocator (S_t at column 128 t, P_t = S_t + 64,
//                 O_t at 256 + 128 t)
//   warps 4..11   one softmax warpgroup per tile: one query row per thread;
//                 online softmax in fp32 with lazy rescaling (O and l are
//                 rescaled only when the running max grows by more than 2^8);
//                 P is packed to bf16 and stored into TMEM over the consumed
//                 scores, so P never touches shared memory (the SS-mode MMAs
//                 and TMA already use most of the smem bandwidth). exp2 is
//                 split 3:1 between MUFU.EX2 and an FMA-pipe polynomial
//                 (measured alternatives: 1:1, 1:0, packed f16x2 MUFU exp --
//                 all slower on B200, whose f16x2 ex2 issues two MUFU ops).
//
// Measured at C2 (dh 72 -> 80, 4096 x 4096 x 16 heads): ~2900 clk per
// 128-row KV block per CTA, the softmax exp section being the largest part
// (MUFU ~80 % busy inside it, idle during max / row sum). A variant with
// double-buffered 64-column S buffers per tile (S_{j+1} computed during the
// softmax of S_j) was 8 % slower: the softmax is not waiting on the MMA.
// Before the stream-K schedule, merging uniform kv splits inside the kernel
// (the last-arriving CTA of each query tile group) was 1.75x slower than a
// separate merge kernel at 512-row patches: the merge then ran on one CTA
// per (tiles, head) at the end of the critical path.
#pragma once

#include "kernels.h"  // kAttnFlagsPerCta
#include "sm100_ptx.cuh"

namespace pf {

constexpr int kAttnBM = 128;   // query rows per tile
constexpr int kAttnBN = 128;   // kv rows per block

constexpr int kAttnMaxSegs = 64;  // segments per CTA (attn_grid keeps within)

// NT query tiles (of 128 rows) per CTA share every K/V tile.
// kW softmax warps per query-row quadrant of a tile (1: one thread per row
// owns all 128 scores of a KV block; 2: two warps split the block's columns
// and exchange their partial row maxima through shared memory).
template <int DHP, int NT, int kW = 1>
struct AttnSmem {
  static constexpr uint32_t kTileBytes = kAttnBM * DHP * 2;  // Q, K or V tile
  static constexpr uint32_t kTileAlloc = (kTileBytes + 1023) & ~1023u;
  static constexpr uint32_t kXBytes = kW == 2 ? 2 * NT * 4 * 2 * 32 * 4 : 0;  // max exchange
  static constexpr uint32_t kBudget = 232448 - 1024 - 512 - 16 * kAttnMaxSegs - kXBytes;
  static constexpr int kStagesMax = int((kBudget - NT * kTileAlloc) / (2 * kTileAlloc));
  static constexpr int kStages = kStagesMax > 4 ? 4 : kStagesMax;
  static constexpr uint32_t kQOff = 0;
  static constexpr uint32_t kKOff = NT * kTileAlloc;
  static constexpr uint32_t kVOff = kKOff + kStages * kTileAlloc;
  static constexpr uint32_t kBarOff = kVOff + kStages * kTileAlloc;
  static constexpr uint32_t kSegOff = kBarOff + 512;  // int4 segment table
  static constexpr uint32_t kXOff = kSegOff + 16 * kAttnMaxSegs;  // [2][NT][4][2][32] fp32
  static constexpr uint32_t kTotal = kXOff + kXBytes + 1024;
  static constexpr int kThreads = 128 + 128 * NT * kW;
  static_assert(DHP % 16 == 0 && DHP <= 128, "head dim padding");
  static_assert(kStages >= 2, "attention smem budget");
  static_assert(kTotal <= 232448, "attention smem budget");
};

// Two query tiles per CTA for every supported head dim: with P kept in
// tensor memory the smem holds only Q and the K/V rings.
__host__ __device__ constexpr int attn_tiles_per_cta(int /*dhp*/) { return 2; }

struct AttnParams {
  int P;            // kv rows per head in the K/V buffers (= sequence length)
  int q_stride;     // rows per head of the Q buffer (= P for self-attention)
  int fresh_lo, fresh_hi;  // kv rows [lo, hi) (128-aligned) read from tm_k2/tm_v2
  int rows;         // query rows this launch
  int row0;         // first query row
  int heads, dh, hs;
  float scale_log2; // log2(e) / sqrt(dh)
  int nq;           // query-tile groups per head (item = head * nq + group)
  int blocks;       // kv blocks per item
  long long units;  // items * blocks
  int grid;         // persistent CTAs; CTA c owns units [c U / grid, (c+1) U / grid)
  __nv_bfloat16* out;  // [P][hs]
  float* part_o;       // [2 grid][DHP][NT * 128]  partials of cut items (column-major)
  float* part_ml;      // [2 grid][2][NT * 128]    (m, l)
  int* flags;          // [grid][kAttnFlagsPerCta] head partial published, per softmax
                       // warp (fused merge; cleared by the reading warp)
  int fused;           // merge cut items in-kernel (every range >= one item)
  int strided;         // whole items c, c + grid, ... per CTA (no cuts; AttnSchedule)
  // L2 prefetch of the weights the next kernels stream (the CTAs split every
  // region; issued by the otherwise idle warp 3 before the PDL wait)
  const char* pf_ptr[kAttnPrefetchRegions];
  unsigned long long pf_bytes[kAttnPrefetchRegions];
  // Debug timeline (clock64) of CTA (0,0,0); null in production. Slots:
  // [0, 4096) softmax t: 2048 t + 8 i + event; [4096, 6144) MMA: 8 i + event;
  // [6144, 8192) TMA: 8 i + event.
  unsigned long long* trace;
};

__device__ __forceinline__ void attn_trace(const AttnParams& prm, int slot) {
  if (prm.trace && blockIdx.x == 0 && (threadIdx.x & 31) == 0) prm.trace[slot] = clock64();
}

__host__ __device__ __forceinline__ long long attn_unit_start(const AttnParams& prm, int c) {
  return (long long)c * prm.units / prm.grid;
}

// kPoly: bit (g & 7) set -> 4-element group g of a score row takes the
// FMA-pipe exp2 polynomial instead of MUFU.EX2. kPingPong: serialise the two
// softmax warpgroups' exp sections (named barriers 1/2).
// kSumCol: V column dh (< DHP) is 1.0 in every kv row, so O column dh
// accumulates the softmax row sum in the PV MMA (of the bf16 P it multiplies
// V with) and the softmax warps skip their per-element row sum.
template <int DHP, int NT, int kPoly = 0x88, bool kPingPong = false, bool kSumCol = false,
          int kW = 1>
__global__ void __launch_bounds__(128 + 128 * NT * kW, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q,
                    const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v,
                    const __grid_constant__ CUtensorMap tm_k2,
                    const __grid_constant__ CUtensorMap tm_v2, AttnParams prm) {
  using L = AttnSmem<DHP, NT, kW>;
  constexpr int S = L::kStages;
  constexpr int kChunks = DHP / 16;
  static_assert(kW == 1 || (kW == 2 && kSumCol && !kPingPong), "split softmax needs kSumCol");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + L::kQOff;
  uint8_t* sK = smem + L::kKOff;
  uint8_t* sV = smem + L::kVOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;       // [S]
  uint64_t* k_empty = k_full + S;    // [S]
  uint64_t* v_full = k_empty + S;    // [S]
  uint64_t* v_empty = v_full + S;    // [S]
  uint64_t* s_full = v_empty + S;    // [NT]  S_t ready (and PV_{t,i-1} done)
  uint64_t* p_full = s_full + NT;    // [NT]  P_t written to TMEM, S_t consumed
  uint64_t* o_done = p_full + NT;    // [NT]  last PV_t of a segment complete
  uint64_t* q_empty = o_done + NT;   // every S MMA of a segment complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_empty + 1);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = ptx::lane_id();
  int4* segs = reinterpret_cast<int4*>(smem + L::kSegOff);  // {item, b0, n, -}
  struct Seg {
    int x, b0, n;  // item, kv blocks [b0, b0 + n)
  };
  int* nseg_slot = reinterpret_cast<int*>(tmem_slot + 1);
  const int B = prm.blocks;
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tm_q);
    ptx::prefetch_tmap(&tm_k);
    ptx::prefetch_tmap(&tm_v);
    if (prm.fresh_lo < prm.fresh_hi) {
      ptx::prefetch_tmap(&tm_k2);
      ptx::prefetch_tmap(&tm_v2);
    }
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&k_full[s], 1);
      ptx::mbar_init(&k_empty[s], 1);
      ptx::mbar_init(&v_full[s], 1);
      ptx::mbar_init(&v_empty[s], 1);
    }
    for (int t = 0; t < NT; ++t) {
      ptx::mbar_init(&s_full[t], 1);
      ptx::mbar_init(&p_full[t], 128 * kW);
      ptx::mbar_init(&o_done[t], 1);
    }
    ptx::fence_barrier_init();
    // Segment table of this CTA's unit range [u0, u1): natural order, or
    // reversed when cut items are merged in-kernel (see header).
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
  // TMEM columns: S_t = [128 t, 128 t + 128) fp32, P_t = S_t + 64 (64 columns
  // of packed bf16 pairs, written over consumed scores), O_t = 256 + 128 t.
  if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int nseg = *nseg_slot;
  const bool rev = prm.fused != 0;
  if (warp == 3) {
    for (int rgn = 0; rgn < kAttnPrefetchRegions; ++rgn) {
      const unsigned long long bytes = prm.pf_bytes[rgn];
      if (!bytes) continue;
      const unsigned long long per = ((bytes + gridDim.x - 1) / gridDim.x + 15) & ~15ull;
      const unsigned long long beg = per * blockIdx.x;
      const unsigned long long end = beg + per < bytes ? beg + per : bytes;
      constexpr unsigned long long kChunk = 32768;
      for (unsigned long long off = beg + lane * kChunk; off < end; off += 32 * kChunk)
        ptx::prefetch_l2_bulk(prm.pf_ptr[rgn] + off,
                              uint32_t(end - off < kChunk ? end - off : kChunk));
    }
  }
  const bool cta_trace = prm.trace && threadIdx.x == 0 && blockIdx.x < 1024;
  if (cta_trace) prm.trace[8192 + 4 * blockIdx.x] = ptx::globaltimer();
  ptx::pdl_wait();    // predecessor's outputs (A operand, residual, K/V) complete
  ptx::pdl_launch();  // successor may start its prologue as our CTAs retire
  if (cta_trace) {
    prm.trace[8192 + 4 * blockIdx.x + 1] = ptx::globaltimer();
    prm.trace[8192 + 4 * blockIdx.x + 3] = ptx::smid();
  }

  // With NT = 2 (384 threads) registers move from the producer warpgroup
  // (TMA, MMA, allocator) to the two softmax warpgroups.
  if (warp < 4) {
    if constexpr (NT == 2) ptx::setmaxnreg_dec<56>();
    if (warp == 0 && lane == 0) {
      // ------------------------------------------------------------ TMA
      int g = 0;  // blocks loaded so far (K/V ring position)
      int sgi = 0;
      for (; sgi < nseg; ++sgi) {
        const int4 sg4 = segs[sgi];
        const Seg sg{sg4.x, sg4.y, sg4.z};
        const int head = sg.x / prm.nq;
        const int qt = sg.x - head * prm.nq;
        // Q of the previous segment is free once all its S MMAs completed
        if (sgi > 0) ptx::mbar_wait(q_empty, (sgi - 1) & 1);
        if (g < 256) attn_trace(prm, 6144 + 8 * g + 3);
        const int qrow = head * prm.q_stride + prm.row0 + qt * (NT * kAttnBM);
        ptx::mbar_arrive_expect_tx(q_full, NT * L::kTileBytes);
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int c = 0; c < kChunks; ++c)
            ptx::tma_load_2d(sQ + t * L::kTileAlloc + c * (kAttnBM * 32), &tm_q, q_full,
                             c * 16, qrow + t * kAttnBM);
        for (int i = 0; i < sg.n; ++i, ++g) {
          const int s = g % S;
          const uint32_t ph = ((g / S) & 1) ^ 1;
          const int kvr = (sg.b0 + i) * kAttnBN;
          const int kvrow = head * prm.P + kvr;
          // DistriFusion: the worker's own (fresh) rows come from a second buffer
          const bool fresh = kvr >= prm.fresh_lo && kvr < prm.fresh_hi;
          const CUtensorMap* km = fresh ? &tm_k2 : &tm_k;
          const CUtensorMap* vm = fresh ? &tm_v2 : &tm_v;
          if (g < 256) attn_trace(prm, 6144 + 8 * g + 0);
          ptx::mbar_wait(&k_empty[s], ph);
          if (g < 256) attn_trace(prm, 6144 + 8 * g + 1);
          ptx::mbar_arrive_expect_tx(&k_full[s], L::kTileBytes);
#pragma unroll
          for (int c = 0; c < kChunks; ++c)
            ptx::tma_load_2d(sK + s * L::kTileAlloc + c * (kAttnBN * 32), km, &k_full[s],
                             c * 16, kvrow);
          ptx::mbar_wait(&v_empty[s], ph);
          if (g < 256) attn_trace(prm, 6144 + 8 * g + 2);
          ptx::mbar_arrive_expect_tx(&v_full[s], L::kTileBytes);
#pragma unroll
          for (int c = 0; c < kChunks; ++c)
            ptx::tma_load_2d(sV + s * L::kTileAlloc + c * (kAttnBN * 32), vm, &v_full[s],
                             c * 16, kvrow);
        }
      }
    } else if (warp == 1 && lane == 0) {
      // ------------------------------------------------------------ MMA
      // Issue order: S_{0,0} S_{1,0} | PV_{0,0} S_{0,1} PV_{1,0} S_{1,1} | ...
      // PV_{t,i} reads P_t from the S_t columns and S_{t,i+1} overwrites them
      // afterwards: tcgen05.mma from one thread execute in issue order.
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(kAttnBM, kAttnBN);
      constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(kAttnBM, DHP, /*b_mn_major=*/true);
      const uint32_t q_base = ptx::smem_u32(sQ);
      const uint32_t k_base = ptx::smem_u32(sK);
      const uint32_t v_base = ptx::smem_u32(sV);

      auto issue_s = [&](int t, int g) {
        const uint32_t kb = k_base + (g % S) * L::kTileAlloc;
        const uint32_t qb = q_base + t * L::kTileAlloc;
#pragma unroll
        for (int c = 0; c < kChunks; ++c)
          ptx::umma_bf16_ss(tmem_base + 128 * t, ptx::desc_kmajor_sw32(qb + c * (kAttnBM * 32)),
                            ptx::desc_kmajor_sw32(kb + c * (kAttnBN * 32)), idesc_s, c != 0);
        ptx::umma_commit(&s_full[t]);
      };
      auto issue_pv = [&](int t, int g, bool first) {
        const uint32_t vb = v_base + (g % S) * L::kTileAlloc;
        const uint32_t pt = tmem_base + 128 * t + 64;
#pragma unroll
        for (int k = 0; k < kAttnBN / 16; ++k)
          // A: P_t columns (8 per 16 kv); B: V 16 kv rows x DHP (SW32
          // MN-major: LBO = next 16-column chunk, SBO = next 8 kv rows)
          ptx::umma_bf16_ts(tmem_base + 256 + 128 * t, pt + 8 * k,
                            ptx::desc_mnmajor_sw32(vb + k * 16 * 32, kAttnBN * 32, 256),
                            idesc_o, !(first && k == 0));
      };

      int g = 0;
      int sgi = 0;
      for (; sgi < nseg; ++sgi) {
        const int4 sg4 = segs[sgi];
        const Seg sg{sg4.x, sg4.y, sg4.z};
        ptx::mbar_wait(q_full, sgi & 1);
        if (g < 256) attn_trace(prm, 4096 + 8 * g + 6);
        ptx::mbar_wait(&k_full[g % S], (g / S) & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int t = 0; t < NT; ++t) issue_s(t, g);
        ptx::umma_commit(&k_empty[g % S]);
        if (sg.n == 1) ptx::umma_commit(q_empty);
        for (int i = 0; i < sg.n; ++i, ++g) {
          const int s = g % S;
          const bool more = i + 1 < sg.n;
          if (g < 256) attn_trace(prm, 4096 + 8 * g + 0);
          ptx::mbar_wait(&v_full[s], (g / S) & 1);
          if (g < 256) attn_trace(prm, 4096 + 8 * g + 1);
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            ptx::mbar_wait(&p_full[t], g & 1);
            if (g < 256) attn_trace(prm, 4096 + 8 * g + 2 + 2 * t);
            ptx::tc_fence_after();
            issue_pv(t, g, i == 0);
            if (more) {
              if (t == 0) {
                ptx::mbar_wait(&k_full[(g + 1) % S], ((g + 1) / S) & 1);
                ptx::tc_fence_after();
              }
              issue_s(t, g + 1);
              if (g < 256) attn_trace(prm, 4096 + 8 * g + 3 + 2 * t);
            } else {
              ptx::umma_commit(&o_done[t]);
            }
          }
          ptx::umma_commit(&v_empty[s]);
          if (more) ptx::umma_commit(&k_empty[(g + 1) % S]);
          if (i + 2 == sg.n) ptx::umma_commit(q_empty);  // last S of the segment issued
        }
      }
    }
  } else if constexpr (kW == 2) {
    ptx::setmaxnreg_inc<104>();
    // ------------------------------------------------ softmax, two warps per row
    // Warps 4 + 8 t + 4 h + q own rows 32 q .. 32 q + 31 of tile t (TMEM lane
    // quadrant q) and KV columns [64 h, 64 h + 64) of each block: half the
    // scores per thread, twice the warps per SM sub-partition to overlap the
    // MUFU exp2 with the FMA-pipe polynomial and the TMEM traffic. The two
    // warps of a row quadrant exchange partial block maxima through shared
    // memory (double-buffered by block parity) and agree on every rescale
    // decision; O's column chunks, the epilogue stores and the merge partials
    // are split between them (chunk c belongs to half c % 2). The row sum is
    // O column dh (kSumCol).
    const int idx = warp - 4;
    const int t = idx >> 3;
    const int half = (idx >> 2) & 1;
    const int q = warp & 3;
    const int trow = 32 * q + int(lane);
    const uint32_t lane_off = uint32_t(32 * q) << 16;
    const uint32_t tmem_s = tmem_base + 128 * t + lane_off;
    const uint32_t tmem_p = tmem_s + 64;
    const uint32_t tmem_o = tmem_base + 256 + 128 * t + lane_off;
    const float sc = prm.scale_log2;
    float* xmax = reinterpret_cast<float*>(smem + L::kXOff);
    const uint32_t bar_id = uint32_t(3 + 4 * t + q);
    int g = 0;
    int sgi = 0;
    int* pending_flag = nullptr;
    for (; sgi < nseg; ++sgi) {
      const int4 sg4 = segs[sgi];
      const Seg sg{sg4.x, sg4.y, sg4.z};
      float m_ref = -INFINITY;
      for (int i = 0; i < sg.n; ++i, ++g) {
        const int kv0 = (sg.b0 + i) * kAttnBN + 64 * half;
        const bool tr = g < 256;
        if (tr) attn_trace(prm, 2048 * t + 8 * g + 0);
        ptx::mbar_wait(&s_full[t], g & 1);
        if (tr) attn_trace(prm, 2048 * t + 8 * g + 1);
        ptx::tc_fence_after();
        uint32_t sr[64];
        ptx::tmem_ld32(tmem_s + 64 * half, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
        ptx::tmem_ld32(tmem_s + 64 * half + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
        ptx::tmem_wait_ld();
        float* s = reinterpret_cast<float*>(sr);
        if (kv0 + 64 > prm.P) {
          const int valid = prm.P - kv0;
#pragma unroll
          for (int e = 0; e < 64; ++e)
            if (e >= valid) s[e] = -INFINITY;
        }
        float bm[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          bm[a] = ptx::fmax3(s[a], s[a + 8], s[a + 16]);
          bm[a] = ptx::fmax3(bm[a], s[a + 24], s[a + 32]);
          bm[a] = ptx::fmax3(bm[a], s[a + 40], s[a + 48]);
          bm[a] = fmaxf(bm[a], s[a + 56]);
        }
        const float pm = fmaxf(ptx::fmax3(bm[0], bm[1], bm[2]),
                               ptx::fmax3(bm[3], ptx::fmax3(bm[4], bm[5], bm[6]), bm[7]));
        // exchange with the other half (the barrier also orders this warp's
        // P stores after the other warp's score loads of the shared columns)
        float* xs = xmax + ((size_t(g & 1) * NT + t) * 4 + q) * 64;
        xs[32 * half + int(lane)] = pm;
        ptx::named_bar_sync(bar_id, 64);
        const float po = xs[32 * (half ^ 1) + int(lane)];
        const float bmax = (half == 0 ? fmaxf(pm, po) : fmaxf(po, pm)) * sc;
        const bool need = bmax > m_ref + 8.0f;
        const float m_new = need ? bmax : m_ref;
        const float alpha = need ? ptx::ex2_approx(m_ref - m_new) : 1.0f;
        if (tr) attn_trace(prm, 2048 * t + 8 * g + 2);
        if (i > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll
          for (int c = half; c < kChunks; c += 2) {
            uint32_t r[16];
            ptx::tmem_ld16(tmem_o + 16 * c, r);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
            ptx::tmem_st16(tmem_o + 16 * c, r);
          }
        }
        if (tr) attn_trace(prm, 2048 * t + 8 * g + 3);
        const float2 sc2 = make_float2(sc, sc);
        const float2 nm2 = make_float2(-m_new, -m_new);
#pragma unroll
        for (int hq = 0; hq < 2; ++hq) {  // 32 scores -> 16 packed bf16 pairs per store
          uint32_t pk[16];
#pragma unroll
          for (int gg = 0; gg < 8; ++gg) {
            const int e = 32 * hq + 4 * gg;
            const int grp = 8 * hq + gg;
            const float2 x0 = ptx::ffma2(make_float2(s[e], s[e + 1]), sc2, nm2);
            const float2 x1 = ptx::ffma2(make_float2(s[e + 2], s[e + 3]), sc2, nm2);
            float2 p0, p1;
            if ((kPoly >> (grp & 7)) & 1) {
              p0 = ptx::ex2_poly2(x0);
              p1 = ptx::ex2_poly2(x1);
            } else {
              p0 = make_float2(ptx::ex2_approx(x0.x), ptx::ex2_approx(x0.y));
              p1 = make_float2(ptx::ex2_approx(x1.x), ptx::ex2_approx(x1.y));
            }
            pk[2 * gg] = ptx::pack_bf16x2(p0.x, p0.y);
            pk[2 * gg + 1] = ptx::pack_bf16x2(p1.x, p1.y);
          }
          ptx::tmem_st16(tmem_p + 32 * half + 16 * hq, pk);
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&p_full[t]);
        if (pending_flag) {
          __syncwarp();
          if (lane == 0) ptx::st_release_gpu(pending_flag, 1);
          pending_flag = nullptr;
        }
        if (tr) attn_trace(prm, 2048 * t + 8 * g + 4);
        m_ref = m_new;
        if (tr) attn_trace(prm, 2048 * t + 8 * g + 5);
      }

      // Segment epilogue: this warp's column chunks of O.
      ptx::mbar_wait(&o_done[t], sgi & 1);
      ptx::tc_fence_after();
      float l_sum;
      {
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
        for (int c = half; c < kChunks; c += 2) {
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
        const int wflag = (c0 - 1) * kAttnFlagsPerCta + idx;
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
        for (int c = half; c < kChunks; c += 2) {
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
#pragma unroll
        for (int c = half; c < kChunks; c += 2) {
          uint32_t r[16];
          ptx::tmem_ld16(tmem_o + 16 * c, r);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e)
            po[size_t(16 * c + e) * (NT * kAttnBM)] = __uint_as_float(r[e]);
        }
        prm.part_ml[(size_t(slot) * 2 + 0) * (NT * kAttnBM) + prow] = m_ref;
        prm.part_ml[(size_t(slot) * 2 + 1) * (NT * kAttnBM) + prow] = l_sum;
        if (rev) pending_flag = prm.flags + int(blockIdx.x) * kAttnFlagsPerCta + idx;
      }
    }
    if (pending_flag) {
      __syncwarp();
      if (lane == 0) ptx::st_release_gpu(pending_flag, 1);
    }
  } else {
    if constexpr (NT == 2) ptx::setmaxnreg_inc<224>();
    // -------------------------------------------------------------- softmax
    const int t = (warp - 4) >> 2;        // query tile of this warpgroup
    const int q = warp & 3;
    const int trow = 32 * q + int(lane);  // row within the tile == TMEM lane
    const uint32_t lane_off = uint32_t(32 * q) << 16;
    const uint32_t tmem_s = tmem_base + 128 * t + lane_off;
    const uint32_t tmem_p = tmem_s + 64;
    const uint32_t tmem_o = tmem_base + 256 + 128 * t + lane_off;
    const float sc = prm.scale_log2;
    // Warpgroup 0 takes the first exp turn.
    constexpr bool pp = NT == 2 && kPingPong;
    if (pp && t == 1) ptx::named_bar_arrive(1, 256);
    int g = 0;
    int sgi = 0;
    // fused merge: this warp's head-partial flag is released one block after
    // its stores were issued, so the release does not stall on their acks
    int* pending_flag = nullptr;
    for (; sgi < nseg; ++sgi) {
    const int4 sg4 = segs[sgi];
    const Seg sg{sg4.x, sg4.y, sg4.z};
    float m_ref = -INFINITY;  // running (lazy) max, scaled log2 domain
    float l_sum = 0.f;
    for (int i = 0; i < sg.n; ++i, ++g) {
      const int kv0 = (sg.b0 + i) * kAttnBN;
      // S_{t,i} complete; so is PV_{t,i-1} (issued before it), hence O_t is
      // stable until P_{t,i} is published.
      const bool tr = g < 256;
      if (tr) attn_trace(prm, 2048 * t + 8 * g + 0);
      ptx::mbar_wait(&s_full[t], g & 1);
      if (tr) attn_trace(prm, 2048 * t + 8 * g + 1);
      ptx::tc_fence_after();
      uint32_t sr[kAttnBN];
#pragma unroll
      for (int c = 0; c < kAttnBN / 32; ++c)
        ptx::tmem_ld32(tmem_s + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&sr[32 * c]));
      ptx::tmem_wait_ld();

      float* s = reinterpret_cast<float*>(sr);
      if (kv0 + kAttnBN > prm.P) {  // kv rows past the buffer end are masked
        const int valid = prm.P - kv0;
#pragma unroll
        for (int e = 0; e < kAttnBN; ++e)
          if (e >= valid) s[e] = -INFINITY;
      }
      // row max with three-input FMNMX3: 8 chains over 16 columns each
      static_assert(kAttnBN == 128, "row-max chains");
      float bm[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        bm[a] = ptx::fmax3(s[a], s[a + 8], s[a + 16]);
#pragma unroll
        for (int e = 24; e < 120; e += 16) bm[a] = ptx::fmax3(bm[a], s[e + a], s[e + 8 + a]);
        bm[a] = fmaxf(bm[a], s[120 + a]);
      }
      const float bmax = fmaxf(ptx::fmax3(bm[0], bm[1], bm[2]),
                               ptx::fmax3(bm[3], ptx::fmax3(bm[4], bm[5], bm[6]), bm[7])) * sc;
      const bool need = bmax > m_ref + 8.0f;
      const float m_new = need ? bmax : m_ref;
      const float alpha = need ? ptx::ex2_approx(m_ref - m_new) : 1.0f;  // 0 on first block
      // Optional ping-pong of the exp-heavy section between the two softmax
      // warpgroups (named barriers 1/2). Off by default: letting both
      // warpgroups exponentiate concurrently measured 4 % faster at dh 72.
      if (tr) attn_trace(prm, 2048 * t + 8 * g + 2);
      if (pp) ptx::named_bar_sync(1 + t, 256);
      if (tr) attn_trace(prm, 2048 * t + 8 * g + 3);
      if (i > 0 && __any_sync(0xffffffffu, need)) {
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
      // P = exp2(s * sc - m): packed fp32x2 FMAs; 1 of every 4 pairs of
      // pairs goes through the FMA-pipe polynomial, the rest through
      // MUFU.EX2; P is packed to bf16 pairs and stored into TMEM over S.
      const float2 sc2 = make_float2(sc, sc);
      const float2 nm2 = make_float2(-m_new, -m_new);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t pk[32];
#pragma unroll
        for (int g = 0; g < 16; ++g) {
          const int e = 64 * h + 4 * g;
          const float2 x0 = ptx::ffma2(make_float2(s[e], s[e + 1]), sc2, nm2);
          const float2 x1 = ptx::ffma2(make_float2(s[e + 2], s[e + 3]), sc2, nm2);
          float2 p0, p1;
          if ((kPoly >> (g & 7)) & 1) {
            p0 = ptx::ex2_poly2(x0);
            p1 = ptx::ex2_poly2(x1);
          } else {
            p0 = make_float2(ptx::ex2_approx(x0.x), ptx::ex2_approx(x0.y));
            p1 = make_float2(ptx::ex2_approx(x1.x), ptx::ex2_approx(x1.y));
          }
          s[e] = p0.x; s[e + 1] = p0.y; s[e + 2] = p1.x; s[e + 3] = p1.y;
          pk[2 * g] = ptx::pack_bf16x2(p0.x, p0.y);
          pk[2 * g + 1] = ptx::pack_bf16x2(p1.x, p1.y);
        }
        if (h == 1 && pp) ptx::named_bar_arrive(2 - t, 256);  // hand the turn over
        ptx::tmem_st32(tmem_p + 32 * h, pk);
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&p_full[t]);
      if (pending_flag) {
        __syncwarp();
        if (lane == 0) ptx::st_release_gpu(pending_flag, 1);
        pending_flag = nullptr;
      }
      if (tr) attn_trace(prm, 2048 * t + 8 * g + 4);
      if constexpr (!kSumCol) {
        // Row sum off the critical path (the PV MMA is already running).
        float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
#pragma unroll
        for (int e = 0; e < kAttnBN; e += 8) {
          a0 = ptx::fadd2(a0, make_float2(s[e], s[e + 1]));
          a1 = ptx::fadd2(a1, make_float2(s[e + 2], s[e + 3]));
          a2 = ptx::fadd2(a2, make_float2(s[e + 4], s[e + 5]));
          a3 = ptx::fadd2(a3, make_float2(s[e + 6], s[e + 7]));
        }
        a0 = ptx::fadd2(ptx::fadd2(a0, a1), ptx::fadd2(a2, a3));
        l_sum = l_sum * alpha + (a0.x + a0.y);
      }
      m_ref = m_new;
      if (tr) attn_trace(prm, 2048 * t + 8 * g + 5);
    }

    // Segment epilogue: wait for the last PV, read O, normalise, store.
    ptx::mbar_wait(&o_done[t], sgi & 1);
    if (g - 1 < 256) attn_trace(prm, 2048 * t + 8 * (g - 1) + 6);
    ptx::tc_fence_after();
    if constexpr (kSumCol) {  // the row sum is O column dh (rescaled with O)
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
    const int lrow = qt * (NT * kAttnBM) + t * kAttnBM + trow;  // row within the launch
    const bool row_ok = lrow < prm.rows;
    if (sg.n == B) {
      const float inv_l = 1.0f / l_sum;
      __nv_bfloat16* orow =
          prm.out + size_t(prm.row0 + lrow) * prm.hs + size_t(head) * prm.dh;
      const bool vec = (prm.dh % 8 == 0) && (prm.hs % 8 == 0);
#pragma unroll
      for (int c = 0; c < kChunks; ++c) {
        uint32_t r[16];
        ptx::tmem_ld16(tmem_o + 16 * c, r);
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
    } else if (rev && sg.b0 > 0) {
      // fused merge: tail of a cut item + its head, published by the same
      // warp of CTA c-1 (per-warp flag; this warp consumes and clears it)
      const int c = int(blockIdx.x);
      const int wflag = (c - 1) * kAttnFlagsPerCta + (warp - 4);
      if (lane == 0) {
        while (ptx::ld_acquire_gpu(prm.flags + wflag) == 0) __nanosleep(32);
        prm.flags[wflag] = 0;  // the next launch is stream-ordered after this one
      }
      __syncwarp();
      const int prow = t * kAttnBM + trow;
      const size_t sbase = size_t(2 * (c - 1) + 1);
      const float m2 = prm.part_ml[(sbase * 2 + 0) * (NT * kAttnBM) + prow];
      const float l2 = prm.part_ml[(sbase * 2 + 1) * (NT * kAttnBM) + prow];
      const float mm = fmaxf(m_ref, m2);
      const float w1 = ptx::ex2_approx(m_ref - mm), w2 = ptx::ex2_approx(m2 - mm);
      const float inv_l = 1.0f / (w1 * l_sum + w2 * l2);
      const float a1 = w1 * inv_l, a2 = w2 * inv_l;
      const float* po = prm.part_o + sbase * DHP * (NT * kAttnBM) + prow;
      __nv_bfloat16* orow =
          prm.out + size_t(prm.row0 + lrow) * prm.hs + size_t(head) * prm.dh;
#pragma unroll
      for (int c2 = 0; c2 < kChunks; ++c2) {
        uint32_t r[16];
        ptx::tmem_ld16(tmem_o + 16 * c2, r);
        float pv[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) pv[j] = po[size_t(16 * c2 + j) * (NT * kAttnBM)];
        ptx::tmem_wait_ld();
        float o[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) o[j] = a1 * __uint_as_float(r[j]) + a2 * pv[j];
        if (row_ok) {
          if ((prm.dh % 8 == 0) && (prm.hs % 8 == 0)) {
#pragma unroll
            for (int e = 0; e < 16; e += 8) {
              const int d = 16 * c2 + e;
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
              const int d = 16 * c2 + e;
              if (d < prm.dh) orow[d] = __float2bfloat16_rn(o[e]);
            }
          }
        }
      }
    } else {
      // cut item: partial into slot 2c (first segment) or 2c + 1 (last; the
      // head of a cut item in fused mode). Column-major [slot][d][row]: each
      // warp store is one contiguous 128-byte line.
      const int slot = 2 * int(blockIdx.x) + (sgi == 0 && !rev ? 0 : 1);
      const int prow = t * kAttnBM + trow;
      float* po = prm.part_o + size_t(slot) * DHP * (NT * kAttnBM) + prow;
      const int ep = 12288 + 64 * t + 8 * (sgi & 7);  // debug probes (CTA 0)
      uint32_t r[kChunks][16];
#pragma unroll
      for (int c = 0; c < kChunks; ++c) ptx::tmem_ld16(tmem_o + 16 * c, r[c]);
      ptx::tmem_wait_ld();
      attn_trace(prm, ep + 0);
#pragma unroll
      for (int c = 0; c < kChunks; ++c)
#pragma unroll
        for (int e = 0; e < 16; ++e) po[size_t(16 * c + e) * (NT * kAttnBM)] = __uint_as_float(r[c][e]);
      attn_trace(prm, ep + 1);
      prm.part_ml[(size_t(slot) * 2 + 0) * (NT * kAttnBM) + prow] = m_ref;
      prm.part_ml[(size_t(slot) * 2 + 1) * (NT * kAttnBM) + prow] = l_sum;
      // publish this warp's rows of the head partial to CTA c+1
      if (rev) pending_flag = prm.flags + int(blockIdx.x) * kAttnFlagsPerCta + (warp - 4);
    }
    // O_t is read: the next segment's first PV (after its P_{t,0}) may overwrite it
    if (g - 1 < 256) attn_trace(prm, 2048 * t + 8 * (g - 1) + 7);
    }
    if (pending_flag) {
      __syncwarp();
      if (lane == 0) ptx::st_release_gpu(pending_flag, 1);
    }
    // Balance the ping-pong: warpgroup 0 consumes warpgroup 1's last hand-off.
    if (pp && t == 0) ptx::named_bar_sync(1, 256);
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (cta_trace) prm.trace[8192 + 4 * blockIdx.x + 2] = ptx::globaltimer();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem_base);
  }
}

// Merge the partials of every cut item in CTA order (deterministic).
// blockIdx.x + 1 = interior range boundary c; the first boundary inside an
// item merges it, over CTAs c-1 .. (last CTA whose range meets the item).
// blockIdx.y = 256-element slice of the item's (row, 16-column chunk)
// elements; each thread issues all its partials' loads before reducing (the
// merge is L2-latency bound, not bandwidth bound).
constexpr int kAttnMaxParts = 8;  // attn_grid keeps every item within 8 CTAs

template <int DHP, int NT>
__global__ void __launch_bounds__(256)
    attn_streamk_combine_kernel(AttnParams prm) {
  __shared__ int s_slot[kAttnMaxParts];
  __shared__ int s_np;
  ptx::pdl_wait();
  ptx::pdl_launch();
  const int c = int(blockIdx.x) + 1;
  const long long B = prm.blocks;
  const long long s = attn_unit_start(prm, c);
  if (s % B == 0) return;  // boundary on an item edge
  const int x = int(s / B);
  const long long x0 = (long long)x * B, x1 = x0 + B;
  if (attn_unit_start(prm, c - 1) > x0) return;  // an earlier boundary merges this item
  if (threadIdx.x == 0) {
    int np = 0;
    for (int k = c - 1; k < prm.grid && np < kAttnMaxParts; ++k) {
      const long long st = attn_unit_start(prm, k);
      if (st >= x1) break;
      s_slot[np++] = 2 * k + (st >= x0 ? 0 : 1);
    }
    s_np = np;
  }
  __syncthreads();
  const int np = s_np;
  constexpr int kChunks = DHP / 16;
  const int e = int(blockIdx.y) * 256 + int(threadIdx.x);
  if (e >= NT * kAttnBM * kChunks) return;
  const int r = e % (NT * kAttnBM);  // row within the item (consecutive threads: rows)
  const int cc = e / (NT * kAttnBM);
  const int head = x / prm.nq;
  const int qt = x - head * prm.nq;
  const int lrow = qt * (NT * kAttnBM) + r;
  if (lrow >= prm.rows) return;
  constexpr int R = NT * kAttnBM;
  float2 ml[kAttnMaxParts];
#pragma unroll
  for (int p = 0; p < kAttnMaxParts; ++p)
    if (p < np)
      ml[p] = make_float2(prm.part_ml[(size_t(s_slot[p]) * 2 + 0) * R + r],
                          prm.part_ml[(size_t(s_slot[p]) * 2 + 1) * R + r]);
  float m = -INFINITY;
#pragma unroll
  for (int p = 0; p < kAttnMaxParts; ++p)
    if (p < np) m = fmaxf(m, ml[p].x);
  float acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = 0.f;
  float l = 0.f;
#pragma unroll
  for (int p = 0; p < kAttnMaxParts; ++p) {
    if (p < np) {
      const float w = ptx::ex2_approx(ml[p].x - m);
      l += w * ml[p].y;
      const float* po = prm.part_o + (size_t(s_slot[p]) * DHP + 16 * cc) * R + r;
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = po[size_t(j) * R];
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] += w * v[j];
    }
  }
  const float inv_l = 1.0f / l;
  __nv_bfloat16* orow = prm.out + size_t(prm.row0 + lrow) * prm.hs + size_t(head) * prm.dh;
  const bool vec = (prm.dh % 8 == 0) && (prm.hs % 8 == 0);
  if (vec) {
#pragma unroll
    for (int j = 0; j < 16; j += 8) {
      const int d = 16 * cc + j;
      if (d < prm.dh) {
        uint4 v;
        v.x = ptx::pack_bf16x2(acc[j] * inv_l, acc[j + 1] * inv_l);
        v.y = ptx::pack_bf16x2(acc[j + 2] * inv_l, acc[j + 3] * inv_l);
        v.z = ptx::pack_bf16x2(acc[j + 4] * inv_l, acc[j + 5] * inv_l);
        v.w = ptx::pack_bf16x2(acc[j + 6] * inv_l, acc[j + 7] * inv_l);
        *reinterpret_cast<uint4*>(orow + d) = v;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int d = 16 * cc + j;
      if (d < prm.dh) orow[d] = __float2bfloat16_rn(acc[j] * inv_l);
    }
  }
}

}  // namespace pf
