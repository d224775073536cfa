// Persistent warp-specialised tcgen05 GEMM for the toy DiT block:
//   D[rows x N] = A[rows x K] . B[N x K]^T      (bf16 operands, fp32 in TMEM)
// followed by a fused epilogue functor (K/V scatter, residual add, tanh).
//
// This is the sm_100a replacement of the reference's `matmul_rows`
// (/root/reference/proj/src/toy_model.cpp:93-102): out = x . w with w stored
// here pre-transposed (N x K, K-major) so both operands are K-major.
//
// Roles (256 threads):
//   warp 0      TMA producer (one elected lane)
//   warp 1      tcgen05.mma issuer (one elected lane)
//   warp 2      TMEM allocator / deallocator
//   warps 4..7  epilogue: TMEM -> registers -> functor (warp w reads lanes
//               32*(w%4) .. +31, i.e. one accumulator row per thread)
// Pipelines: STAGES-deep smem ring (TMA <-> MMA) and a 2-deep TMEM
// accumulator ring (MMA <-> epilogue) so a tile's epilogue overlaps the next
// tile's main loop.
#pragma once

#include <type_traits>

#include "sm100_ptx.cuh"

namespace pf {

// Debug timeline of the 1-SM GEMM kernel (null in production): 8 slots per
// CTA (blockIdx.x < 256): globaltimer at entry, after the PDL wait, first
// stage landed (MMA issuer), last MMA issued, first accumulator ready
// (epilogue), exit; SM id.
__device__ unsigned long long* g_gemm_trace = nullptr;


constexpr int kGemmBM = 128;
constexpr int kGemmBK = 64;  // 64 bf16 = 128 B = one SW128 atom row

// Epilogue functors may carry per-row state computed once per tile before
// the accumulator is ready (e.g. LayerNorm statistics of the A rows):
// `typename E::RowState E::row_state(int row) const` and
// `E::operator()(row, col0, v, nvalid, const RowState&)`.
struct NoRowState {};
template <class E, class = void>
struct epi_row_state {
  static constexpr bool value = false;
  using type = NoRowState;
};
template <class E>
struct epi_row_state<E, std::void_t<typename E::RowState>> {
  static constexpr bool value = true;
  using type = typename E::RowState;
};

// Epilogues may also declare `static constexpr int kColVecs` per-column fp32
// vectors (`const float* colvec(int v) const`, null = zeros). The epilogue
// warps stage the tile's BN columns of each vector in shared memory before
// waiting for the accumulator (double-buffered by tile parity) and pass a
// ColView to `operator()(row, col0, v, nvalid, rs, cv)`: cv.p[k * cv.stride + e]
// is vector k at column col0 + e.
struct ColView {
  const float* p;
  int stride;
};
template <class E, class = void>
struct epi_colvecs {
  static constexpr int value = 0;
};
template <class E>
struct epi_colvecs<E, std::void_t<decltype(E::kColVecs)>> {
  static constexpr int value = E::kColVecs;
};
constexpr int kMaxColVecs = 2;

// Stage the tile's columns [n0, n0 + BN) of the epilogue's column vectors
// into `dst` ([NV][BN] fp32); the 128 epilogue threads (tid 0..127) then
// synchronise on named barrier 2.
template <int BN, class Epi>
__device__ __forceinline__ void stage_colvecs(const Epi& epi, float* dst, int n0, int N,
                                              int tid) {
  constexpr int NV = epi_colvecs<Epi>::value;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const float* src = epi.colvec(v);
    for (int c = tid; c < BN; c += 128)
      dst[v * BN + c] = (src && n0 + c < N) ? __ldg(src + n0 + c) : 0.f;
  }
  ptx::named_bar_sync(2, 128);
}

// One 32-column chunk of a non-preloading epilogue.
template <int BN, class Epi, class RS>
__device__ __forceinline__ void epilogue_chunk(const Epi& epi, const uint32_t (&r)[32], int c,
                                               int grow, bool row_ok, int n0, int N,
                                               const RS& rs, const float* colbuf) {
  const int col0 = n0 + 32 * c;
  if (!row_ok || col0 >= N) return;
  const int nvalid = (N - col0) < 32 ? (N - col0) : 32;
  float v[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]);
  if constexpr (epi_colvecs<Epi>::value > 0) {
    epi(grow, col0, v, nvalid, rs, ColView{colbuf + 32 * c, BN});
  } else if constexpr (epi_row_state<Epi>::value) {
    epi(grow, col0, v, nvalid, rs);
  } else {
    epi(grow, col0, v, nvalid);
  }
}

// The tile's BN / 32 chunks, not unrolled (the functor bodies are large and
// a fully unrolled tile overflows the instruction cache), with the TMEM load
// of chunk c + 1 in flight while chunk c is processed.
template <int BN, class Epi, class RS>
__device__ __forceinline__ void epilogue_chunks(const Epi& epi, uint32_t taddr, int grow,
                                                bool row_ok, int n0, int N, const RS& rs,
                                                const float* colbuf) {
  constexpr int NC = BN / 32;
  static_assert(NC % 2 == 0, "chunk pairs");
  uint32_t ra[32], rb[32];
  ptx::tmem_ld32(taddr, ra);
  ptx::tmem_wait_ld();
#pragma unroll 1
  for (int c = 0; c < NC; c += 2) {
    ptx::tmem_ld32(taddr + 32 * (c + 1), rb);
    epilogue_chunk<BN>(epi, ra, c, grow, row_ok, n0, N, rs, colbuf);
    ptx::tmem_wait_ld();
    if (c + 2 < NC) ptx::tmem_ld32(taddr + 32 * (c + 2), ra);
    epilogue_chunk<BN>(epi, rb, c + 1, grow, row_ok, n0, N, rs, colbuf);
    ptx::tmem_wait_ld();
  }
}

template <int BN, int STAGES>
struct GemmSmem {
  static constexpr uint32_t kABytes = kGemmBM * kGemmBK * 2;
  static constexpr uint32_t kBBytes = BN * kGemmBK * 2;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr uint32_t kBarOffset = STAGES * kStageBytes;
  static constexpr uint32_t kColOffset = kBarOffset + 256;  // [2][kMaxColVecs][BN] fp32
  static constexpr uint32_t kTotal = kColOffset + 2 * kMaxColVecs * BN * 4 + 1024;
  static constexpr uint32_t kTmemCols = (2 * BN <= 32)    ? 32
                                        : (2 * BN <= 64)  ? 64
                                        : (2 * BN <= 128) ? 128
                                        : (2 * BN <= 256) ? 256
                                                          : 512;
};

// Deterministic split-K for skinny problems (few output tiles, long K): the
// K loop of every tile is cut into `splits` ranges processed by different
// CTAs; each stores its fp32 partial tile to `ws`, and the CTA that finishes
// a tile last (per-tile counter) sums the partials in split order and runs
// the epilogue. splits == 1 is the ordinary persistent kernel.
struct SplitK {
  int splits = 1;
  float* ws = nullptr;     // [tiles][splits][128][BN] fp32 (in-kernel fixup)
  int* counters = nullptr; // [tiles], zero between launches
  // partials only: split s writes rows x N fp32 at ws + s * rows * N (row-major)
  // and no epilogue runs; a separate reduction kernel finishes the output
  bool partials_only = false;
};

template <int BN, int STAGES, class Epi>
__global__ void __launch_bounds__(256, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap tma_a,
                        const __grid_constant__ CUtensorMap tma_b, int rows,
                        int row0, int N, int K, Epi epi, SplitK sk) {
  const long long t_entry = clock64();
  using L = GemmSmem<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_last = reinterpret_cast<int*>(smem + L::kBarOffset + 248);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = ptx::lane_id();
  const int m_tiles = (rows + kGemmBM - 1) / kGemmBM;
  const int n_tiles = (N + BN - 1) / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int kblocks = (K + kGemmBK - 1) / kGemmBK;
  const int splits = sk.splits;
  const int num_units = num_tiles * splits;
  const int kb_per = (kblocks + splits - 1) / splits;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tma_a);
    ptx::prefetch_tmap(&tma_b);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 128);
    }
    ptx::fence_barrier_init();
  }
  const long long t_pre_alloc = clock64();
  if (warp == 2) ptx::tmem_alloc<L::kTmemCols>(tmem_slot);
  const long long t_post_alloc = clock64();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  unsigned long long* trc = g_gemm_trace && blockIdx.x < 128 ? g_gemm_trace + 16 * blockIdx.x
                                                              : nullptr;
  if (trc && threadIdx.x == 0) trc[7] = t_entry;
  if (trc && threadIdx.x == 0) trc[0] = clock64();
  if (trc && threadIdx.x == 64) {
    trc[9] = t_pre_alloc;
    trc[10] = t_post_alloc;
  }
  // The B operand is always a weight matrix (never written by a preceding
  // kernel): the producer puts the first stages' B tiles in flight before the
  // PDL wait, overlapping their latency with the predecessor's tail.
  int preloaded = 0;
  if (warp == 0 && lane == 0 && int(blockIdx.x) < num_units) {
    const int split = int(blockIdx.x) % splits;
    const int nt = (int(blockIdx.x) / splits) / m_tiles;
    const int kb0 = split * kb_per;
    preloaded = min(STAGES, min(kblocks, kb0 + kb_per) - kb0);
    for (int j = 0; j < preloaded; ++j) {
      ptx::mbar_arrive_expect_tx(&full[j], L::kStageBytes);
      ptx::tma_load_2d(smem + j * L::kStageBytes + L::kABytes, &tma_b, &full[j],
                       (kb0 + j) * kGemmBK, nt * BN);
    }
  }
  ptx::pdl_wait();    // predecessor's outputs (A operand, residual, K/V) complete
  ptx::pdl_launch();  // successor may start its prologue as our CTAs retire
  if (trc && threadIdx.x == 0) {
    trc[1] = clock64();
    trc[6] = ptx::smid();
  }

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x) {
        const int tile = unit / splits;
        const int split = unit - tile * splits;
        const int mt = tile % m_tiles;
        const int nt = tile / m_tiles;
        const int kb0 = split * kb_per;
        const int kb1 = min(kblocks, kb0 + kb_per);
        for (int kb = kb0; kb < kb1; ++kb) {
          uint8_t* sa = smem + stage * L::kStageBytes;
          uint8_t* sb = sa + L::kABytes;
          if (preloaded > 0) {  // B already in flight (first unit, first stages)
            --preloaded;
            if (trc && kb == kb0) trc[8] = clock64();
            ptx::tma_load_2d(sa, &tma_a, &full[stage], kb * kGemmBK, row0 + mt * kGemmBM);
          } else {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            ptx::mbar_arrive_expect_tx(&full[stage], L::kStageBytes);
            ptx::tma_load_2d(sa, &tma_a, &full[stage], kb * kGemmBK,
                             row0 + mt * kGemmBM);
            ptx::tma_load_2d(sb, &tma_b, &full[stage], kb * kGemmBK, nt * BN);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(kGemmBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x) {
        const int split = unit % splits;
        const int kb0 = split * kb_per;
        const int kb1 = min(kblocks, kb0 + kb_per);
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          if (trc && kb == kb0 && unit == int(blockIdx.x)) trc[2] = clock64();
          ptx::tc_fence_after();
          const uint32_t a_base = ptx::smem_u32(smem + stage * L::kStageBytes);
          const uint32_t b_base = a_base + L::kABytes;
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k) {
            ptx::umma_bf16_ss(d_tmem, ptx::desc_kmajor_sw128(a_base + k * 32),
                              ptx::desc_kmajor_sw128(b_base + k * 32), idesc,
                              (kb != kb0 || k != 0));
          }
          ptx::umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::umma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
      if (trc) trc[3] = clock64();
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int tid = int(threadIdx.x) - 128;  // 0..127 = accumulator row within the tile
    int acc = 0;
    uint32_t acc_phase = 0;
    int tile_count = 0;
    for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x) {
      const int tile = unit / splits;
      const int split = unit - tile * splits;
      const int mt = tile % m_tiles;
      const int nt = tile / m_tiles;
      const int local_row = mt * kGemmBM + 32 * q + int(lane);
      const bool row_ok = local_row < rows;
      const uint32_t taddr = tmem_base + (uint32_t(32 * q) << 16) + acc * BN;
      constexpr int kNV = epi_colvecs<Epi>::value;
      float* colbuf = reinterpret_cast<float*>(smem + L::kColOffset) +
                      (tile_count & 1) * kMaxColVecs * BN;
      if (splits > 1 && sk.partials_only) {
        // ---- partial tile -> [split][rows][N] workspace, reduced elsewhere
        ptx::mbar_wait(&tfull[acc], acc_phase);
        ptx::tc_fence_after();
        float* wrow = sk.ws + (size_t(split) * rows + local_row) * N;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          ptx::tmem_ld32(taddr + 32 * c, r);
          ptx::tmem_wait_ld();
          const int col0 = nt * BN + 32 * c;
          if (row_ok && col0 + 32 <= N) {
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              *reinterpret_cast<float4*>(wrow + col0 + e) =
                  make_float4(__uint_as_float(r[e]), __uint_as_float(r[e + 1]),
                              __uint_as_float(r[e + 2]), __uint_as_float(r[e + 3]));
          } else if (row_ok) {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (col0 + e < N) wrow[col0 + e] = __uint_as_float(r[e]);
          }
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        continue;
      }
      if (splits > 1) {
        // ---- partial tile -> workspace; the last CTA of the tile reduces
        float* wsp = sk.ws + ((size_t(tile) * splits + split) * kGemmBM + tid) * BN;
        ptx::mbar_wait(&tfull[acc], acc_phase);
        ptx::tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          ptx::tmem_ld32(taddr + 32 * c, r);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<float4*>(wsp + 32 * c + e) =
                make_float4(__uint_as_float(r[e]), __uint_as_float(r[e + 1]),
                            __uint_as_float(r[e + 2]), __uint_as_float(r[e + 3]));
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        __threadfence();
        ptx::named_bar_sync(1, 128);
        if (tid == 0) *s_last = atomicAdd(sk.counters + tile, 1) == splits - 1;
        ptx::named_bar_sync(1, 128);
        if (!*s_last) continue;
        __threadfence();
        typename epi_row_state<Epi>::type rs{};
        if constexpr (epi_row_state<Epi>::value) {
          if (row_ok) rs = epi.row_state(row0 + local_row);
        }
        if constexpr (kNV > 0) stage_colvecs<BN>(epi, colbuf, nt * BN, N, tid);
        ++tile_count;
        const float* wst = sk.ws + (size_t(tile) * splits * kGemmBM + tid) * BN;
        const size_t sstride = size_t(kGemmBM) * BN;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          const int col0 = nt * BN + 32 * c;
          if (!row_ok || col0 >= N) continue;
          const int nvalid = (N - col0) < 32 ? (N - col0) : 32;
          float v[32];
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const float4 a = __ldcg(reinterpret_cast<const float4*>(wst + 32 * c + e));
            v[e] = a.x; v[e + 1] = a.y; v[e + 2] = a.z; v[e + 3] = a.w;
          }
          for (int sp = 1; sp < splits; ++sp) {
#pragma unroll
            for (int e = 0; e < 32; e += 4) {
              const float4 a =
                  __ldcg(reinterpret_cast<const float4*>(wst + sp * sstride + 32 * c + e));
              v[e] += a.x; v[e + 1] += a.y; v[e + 2] += a.z; v[e + 3] += a.w;
            }
          }
          if constexpr (Epi::kPreload) {
            float pre[32];
            epi.preload(row0 + local_row, col0, pre, nvalid);
            epi.apply(row0 + local_row, col0, v, pre, nvalid);
          } else if constexpr (kNV > 0) {
            epi(row0 + local_row, col0, v, nvalid, rs, ColView{colbuf + 32 * c, BN});
          } else if constexpr (epi_row_state<Epi>::value) {
            epi(row0 + local_row, col0, v, nvalid, rs);
          } else {
            epi(row0 + local_row, col0, v, nvalid);
          }
        }
        if (tid == 0) sk.counters[tile] = 0;  // ready for the next launch / graph replay
        continue;
      }
      // Epilogues that read an existing output (the residual stream) issue
      // those loads before waiting for the accumulator, so they overlap the
      // tile's main loop instead of sitting on the critical path.
      float pre[Epi::kPreload ? BN / 32 : 1][32];
      if constexpr (Epi::kPreload) {
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          const int col0 = nt * BN + 32 * c;
          if (row_ok && col0 < N)
            epi.preload(row0 + local_row, col0, pre[c], (N - col0) < 32 ? (N - col0) : 32);
        }
      }
      typename epi_row_state<Epi>::type rs{};
      if constexpr (epi_row_state<Epi>::value) {
        if (row_ok) rs = epi.row_state(row0 + local_row);
      }
      if constexpr (kNV > 0) stage_colvecs<BN>(epi, colbuf, nt * BN, N, tid);
      ++tile_count;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      if (trc && tid == 0 && tile_count == 1) trc[4] = clock64();
      ptx::tc_fence_after();
      if constexpr (Epi::kPreload) {
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          const int col0 = nt * BN + 32 * c;
          if (col0 >= N) break;
          uint32_t r[32];
          ptx::tmem_ld32(taddr + 32 * c, r);
          ptx::tmem_wait_ld();
          if (row_ok) {
            const int nvalid = (N - col0) < 32 ? (N - col0) : 32;
            float v[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]);
            epi.apply(row0 + local_row, col0, v, pre[c], nvalid);
          }
        }
      } else {
        epilogue_chunks<BN>(epi, taddr, row0 + local_row, row_ok, nt * BN, N, rs, colbuf);
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (trc && threadIdx.x == 0) trc[5] = clock64();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<L::kTmemCols>(tmem_base);
  }
}


// ---------------------------------------------------------------------------
// 2-SM variant (cluster of 2 CTAs on one TPC, tcgen05.mma.cta_group::2):
// one 256 x BN output tile per CTA pair. CTA r TMA-loads A rows
// [m0 + 128 r, +128) and B rows [n0 + BN/2 r, +BN/2); the even CTA issues
// the M = 256 MMAs, whose B operand is read half from each CTA. Per SM this
// halves the shared-memory operand traffic of the 1-SM 128 x BN kernel
// (SS-mode MMA + TMA writes otherwise exceed the 128 B/clk smem bandwidth).
template <int BN, int STAGES>
struct Gemm2SmSmem {
  static constexpr uint32_t kABytes = kGemmBM * kGemmBK * 2;        // 16 KB
  static constexpr uint32_t kBBytes = (BN / 2) * kGemmBK * 2;       // half of B
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr uint32_t kBarOffset = STAGES * kStageBytes;
  static constexpr uint32_t kColOffset = kBarOffset + 256;  // [2][kMaxColVecs][BN] fp32
  static constexpr uint32_t kTotal = kColOffset + 2 * kMaxColVecs * BN * 4 + 1024;
  static constexpr uint32_t kTmemCols = (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  static_assert(BN % 32 == 0 && BN <= 256, "2-SM tile N");
  static_assert(((BN / 2) * 128) % 1024 == 0, "B half must keep 1024-B aligned stages");
};

// NP = 2: a cluster of two CTA pairs computing N-adjacent tiles of the same
// 256 rows. Each CTA loads half of its 128-row A tile (a 64-row box,
// tma_a_half) and multicasts it to itself and its counterpart in the other
// pair, so every A tile leaves L2 once per cluster instead of once per pair:
// the layer GEMMs move ~8-9 TB/s of operands L2 -> SM over all SMs, and this
// cuts that traffic by 25-33 %. A stage may be refilled only when both
// pairs' MMAs released it: the empty barriers count one multicast commit
// from each pair. Opt-in (kernels.cu): only 33 4-CTA clusters fit on the
// 148 SMs, and the lost wave outweighs the ~8 % per-tile gain measured.
template <int BN, int STAGES, class Epi, int NP = 1>
__global__ void __cluster_dims__(2 * NP, 1, 1) __launch_bounds__(256, 1)
    gemm2sm_bf16_tn_kernel(const __grid_constant__ CUtensorMap tma_a,
                           const __grid_constant__ CUtensorMap tma_b, int rows, int row0,
                           int N, int K, Epi epi,
                           const __grid_constant__ CUtensorMap tma_a_half) {
  using L = Gemm2SmSmem<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = ptx::lane_id();
  const uint32_t crank = ptx::cluster_ctarank();
  const uint32_t rank = crank & 1;          // position in the CTA pair
  const int pr = int(crank >> 1);           // pair within the cluster (N offset)
  const bool leader = rank == 0;
  const int cluster = blockIdx.x / (2 * NP);
  const int nclusters = gridDim.x / (2 * NP);
  const int m_tiles = (rows + 2 * kGemmBM - 1) / (2 * kGemmBM);
  const int n_tiles = (N + BN - 1) / BN;   // NP = 2: even (host checks)
  const int num_tiles = m_tiles * (n_tiles / NP);
  const int kblocks = (K + kGemmBK - 1) / kGemmBK;
  const uint16_t pair_mask = uint16_t(0x3u << (2 * pr));

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tma_a);
    ptx::prefetch_tmap(&tma_b);
    if constexpr (NP == 2) ptx::prefetch_tmap(&tma_a_half);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], NP);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 2);  // one elected arrival per CTA of the pair
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_2sm<L::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  ptx::pdl_wait();    // predecessor's outputs (A operand, residual, K/V) complete
  ptx::pdl_launch();  // successor may start its prologue as our CTAs retire

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cluster; tile < num_tiles; tile += nclusters) {
        const int mt = tile % m_tiles;
        const int nt = (tile / m_tiles) * NP + pr;
        for (int kb = 0; kb < kblocks; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * L::kStageBytes;
          uint8_t* sb = sa + L::kABytes;
          if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * L::kStageBytes);
          if constexpr (NP == 2) {
            // rows [64 pr, +64) of this CTA's A tile, to both pairs
            ptx::tma_load_2d_2sm_mc(sa + pr * (L::kABytes / 2), &tma_a_half, &full[stage],
                                    kb * kGemmBK,
                                    row0 + mt * 2 * kGemmBM + int(rank) * kGemmBM + 64 * pr,
                                    uint16_t(0x5u << rank));
          } else {
            ptx::tma_load_2d_2sm(sa, &tma_a, &full[stage], kb * kGemmBK,
                                 row0 + mt * 2 * kGemmBM + int(rank) * kGemmBM);
          }
          ptx::tma_load_2d_2sm(sb, &tma_b, &full[stage], kb * kGemmBK,
                               nt * BN + int(rank) * (BN / 2));
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(2 * kGemmBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = cluster; tile < num_tiles; tile += nclusters) {
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_base = ptx::smem_u32(smem + stage * L::kStageBytes);
          const uint32_t b_base = a_base + L::kABytes;
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k)
            ptx::umma2_bf16_ss(d_tmem, ptx::desc_kmajor_sw128(a_base + k * 32),
                               ptx::desc_kmajor_sw128(b_base + k * 32), idesc, (kb | k) != 0);
          // the stage's A also holds the other pair's multicast half: release
          // it to every CTA of the cluster
          ptx::umma2_commit_mc(&empty[stage], NP == 2 ? uint16_t(0xF) : pair_mask);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::umma2_commit_mc(&tfull[acc], pair_mask);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const uint32_t tempty_leader0 =
        ptx::mapa_shared(ptx::smem_u32(&tempty[0]), uint32_t(2 * pr));
    int acc = 0;
    uint32_t acc_phase = 0;
    int tile_count = 0;
    for (int tile = cluster; tile < num_tiles; tile += nclusters) {
      const int mt = tile % m_tiles;
      const int nt = (tile / m_tiles) * NP + pr;
      const int local_row = mt * 2 * kGemmBM + int(rank) * kGemmBM + 32 * q + int(lane);
      const bool row_ok = local_row < rows;
      float pre[Epi::kPreload ? BN / 32 : 1][32];
      if constexpr (Epi::kPreload) {
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          const int col0 = nt * BN + 32 * c;
          if (row_ok && col0 < N)
            epi.preload(row0 + local_row, col0, pre[c], (N - col0) < 32 ? (N - col0) : 32);
        }
      }
      typename epi_row_state<Epi>::type rs{};
      if constexpr (epi_row_state<Epi>::value) {
        if (row_ok) rs = epi.row_state(row0 + local_row);
      }
      constexpr int kNV = epi_colvecs<Epi>::value;
      float* colbuf = reinterpret_cast<float*>(smem + L::kColOffset) +
                      (tile_count & 1) * kMaxColVecs * BN;
      if constexpr (kNV > 0) stage_colvecs<BN>(epi, colbuf, nt * BN, N, int(threadIdx.x) - 128);
      ++tile_count;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const uint32_t taddr = tmem_base + (uint32_t(32 * q) << 16) + acc * BN;
      if constexpr (Epi::kPreload) {
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          const int col0 = nt * BN + 32 * c;
          if (col0 >= N) break;
          uint32_t r[32];
          ptx::tmem_ld32(taddr + 32 * c, r);
          ptx::tmem_wait_ld();
          if (row_ok) {
            const int nvalid = (N - col0) < 32 ? (N - col0) : 32;
            float v[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]);
            epi.apply(row0 + local_row, col0, v, pre[c], nvalid);
          }
        }
      } else {
        epilogue_chunks<BN>(epi, taddr, row0 + local_row, row_ok, nt * BN, N, rs, colbuf);
      }
      // All four epilogue warps of this CTA have drained accumulator `acc`:
      // one elected thread tells the pair's MMA issuer (in the even CTA).
      ptx::tc_fence_before();
      ptx::named_bar_sync(1, 128);
      if (warp == 4 && lane == 0)
        ptx::mbar_arrive_cluster(tempty_leader0 + acc * 8);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_2sm<L::kTmemCols>(tmem_base);
  }
}


// ---------------------------------------------------------------------------
// Residual-stream GEMM with a TMA epilogue (1 SM, 128 x 128 tiles):
//   h32[rows, N] += A . B^T;  hb = bf16(h32);  non-finite -> flag
// The producer warp TMA-loads the fp32 residual tile into a 128B-swizzled
// smem buffer once the tile's k-loop is issued; the epilogue warps add the
// TMEM accumulator in smem, write the bf16 copy next to it, and one thread
// TMA-stores both tiles. Global traffic is bulk and coalesced instead of
// one row per thread. Requires rows % 128 == 0 (whole row tiles: stores must
// not touch rows of other patches) and N % 32 == 0.
// The residual tile is loaded through tma_h32 and stored through
// tma_h32_out / tma_hb_out: the same buffers normally, another GPU's landing
// buffers when the last layer of a pipeline stage writes its output straight
// to the next stage (rank mode).
struct ResidTmaArgs {
  float* h;        // for the finite check only
  int* flag;
  int code;
  // PixArt block (kMod kernels only):
  //   h += gate[n] * (acc + bias[n])            (null gate -> 1, null bias -> 0)
  //   hb = bf16(h * (1 + colscale[n]))          (null colscale -> bf16(h)): the
  //        next LayerNorm consumer's adaLN scale, folded into its A operand
  //   stats[(n / 32) * stats_ld + row] = (sum h, sum h^2) over the 32 columns
  const float* bias = nullptr;
  const float* gate = nullptr;
  const float* colscale = nullptr;
  float2* stats = nullptr;
  int stats_ld = 0;
  // rows at or past row_end belong to another stream / patch (a partial last
  // tile: the output tensor maps end at row_end and clip the TMA stores);
  // their statistics and finite checks are skipped. INT_MAX: whole tiles.
  int row_end = 0x7fffffff;
  // Stream-K schedule (gemm2sm_resid_tma_kernel only; null: tiles round-robin
  // over the pairs). Pair c owns the (tile, K block) units [c U / P, (c+1) U / P);
  // requires tiles >= pairs, so a tile spans at most two pairs. sk_ws holds one
  // fp32 head partial [BN cols][128 rows] per CTA, sk_flags one flag per CTA
  // (zero between launches: the reader clears it).
  float* sk_ws = nullptr;
  int* sk_flags = nullptr;
};

// Stream-K walk of a pair's unit range in REVERSE: the pair's last segment
// (the head of a tile the next pair finishes) comes first, so its partial is
// published long before the next pair needs it; the pair's first segment (the
// tail of a tile whose head the previous pair computed) comes last.
struct SkWalk {
  int u, u0, kblocks;
  __device__ __forceinline__ bool next(int& tile, int& kb0, int& kb1) {
    if (u <= u0) return false;
    tile = (u - 1) / kblocks;
    const int ts = tile * kblocks;
    const int s = ts > u0 ? ts : u0;
    kb0 = s - ts;
    kb1 = u - ts;
    u = s;
    return true;
  }
};

// Segments of one CTA pair: the round-robin tile walk (every tile whole) or
// the stream-K walk.
struct ResidTiles {
  bool sk;
  int cluster, nclusters, num_tiles, kblocks;
  int t;       // round-robin: next tile
  SkWalk w;    // stream-K
  __device__ __forceinline__ ResidTiles(bool sk_, int c, int nc, int nt, int kb)
      : sk(sk_), cluster(c), nclusters(nc), num_tiles(nt), kblocks(kb), t(c) {
    const long long units = (long long)nt * kb;
    w.u0 = int(units * c / nc);
    w.u = int(units * (c + 1) / nc);
    w.kblocks = kb;
  }
  __device__ __forceinline__ bool next(int& tile, int& kb0, int& kb1) {
    if (sk) return w.next(tile, kb0, kb1);
    if (t >= num_tiles) return false;
    tile = t;
    kb0 = 0;
    kb1 = kblocks;
    t += nclusters;
    return true;
  }
};

__device__ __forceinline__ float4 ldg4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}

// One thread's 32-column chunk of the TMA residual epilogue: fp32 residual
// tile (SW128, 4 x [128 rows x 32 fp32]) updated in place, bf16 copy written
// into the SW128 bf16 tile (2 x [128 rows x 64 bf16]). Returns "non-finite".
template <bool kMod>
__device__ __forceinline__ bool resid_chunk(uint8_t* sC, uint8_t* sD, int r, int c,
                                            const uint32_t (&v)[32], int col0, int grow,
                                            const ResidTmaArgs& args) {
  const uint32_t sw = uint32_t(r & 7);
  uint8_t* crow = sC + c * 16384 + r * 128;
  uint8_t* drow = sD + (c >> 1) * 16384 + r * 128;
  bool bad = false;
  float s = 0.f, ss = 0.f;
#pragma unroll
  for (int g = 0; g < 8; ++g) {  // 16-byte piece g of the 32 fp32 columns
    float4* pc = reinterpret_cast<float4*>(crow + ((uint32_t(g) ^ sw) << 4));
    float4 x = *pc;
    float4 a = make_float4(__uint_as_float(v[4 * g + 0]), __uint_as_float(v[4 * g + 1]),
                           __uint_as_float(v[4 * g + 2]), __uint_as_float(v[4 * g + 3]));
    float4 y;
    if constexpr (kMod) {
      const int n = col0 + 4 * g;
      if (args.bias) {
        const float4 b = ldg4(args.bias + n);
        a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
      }
      if (args.gate) {
        const float4 gt = ldg4(args.gate + n);
        a.x *= gt.x; a.y *= gt.y; a.z *= gt.z; a.w *= gt.w;
      }
      x.x += a.x; x.y += a.y; x.z += a.z; x.w += a.w;
      s += (x.x + x.y) + (x.z + x.w);
      ss += (x.x * x.x + x.y * x.y) + (x.z * x.z + x.w * x.w);
      y = x;
      if (args.colscale) {
        const float4 cs = ldg4(args.colscale + n);
        y.x *= 1.f + cs.x; y.y *= 1.f + cs.y; y.z *= 1.f + cs.z; y.w *= 1.f + cs.w;
      }
    } else {
      x.x += a.x; x.y += a.y; x.z += a.z; x.w += a.w;
      y = x;
    }
    *pc = x;
    bad |= !(isfinite(x.x) && isfinite(x.y) && isfinite(x.z) && isfinite(x.w));
    // bf16 copy: columns 32c + 4g .. +3 -> byte 64 (c&1) + 8 g of the row
    const uint32_t byte = uint32_t(64 * (c & 1) + 8 * g);
    uint2* pd = reinterpret_cast<uint2*>(drow + ((((byte >> 4) ^ sw) << 4) | (byte & 15)));
    *pd = make_uint2(ptx::pack_bf16x2(y.x, y.y), ptx::pack_bf16x2(y.z, y.w));
  }
  if (grow >= args.row_end) return false;
  if constexpr (kMod) {
    if (args.stats) args.stats[size_t(col0 >> 5) * args.stats_ld + grow] = make_float2(s, ss);
  }
  return bad;
}

template <int STAGES>
struct GemmResSmem {
  static constexpr int BN = 128;
  static constexpr uint32_t kABytes = kGemmBM * kGemmBK * 2;
  static constexpr uint32_t kBBytes = BN * kGemmBK * 2;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr uint32_t kCOff = STAGES * kStageBytes;       // fp32 tile: 4 x 16 KB
  static constexpr uint32_t kDOff = kCOff + 4 * 16384;          // bf16 tile: 2 x 16 KB
  static constexpr uint32_t kBarOffset = kDOff + 2 * 16384;
  static constexpr uint32_t kTotal = kBarOffset + 256 + 1024;
  static_assert(kTotal <= 232448, "residual GEMM smem budget");
};

template <int STAGES, bool kMod>
__global__ void __launch_bounds__(256, 1)
    gemm_resid_tma_kernel(const __grid_constant__ CUtensorMap tma_a,
                          const __grid_constant__ CUtensorMap tma_b,
                          const __grid_constant__ CUtensorMap tma_h32,
                          const __grid_constant__ CUtensorMap tma_hb,
                          const __grid_constant__ CUtensorMap tma_h32_out,
                          const __grid_constant__ CUtensorMap tma_hb_out, int rows, int row0,
                          int N, int K, ResidTmaArgs args) {
  using L = GemmResSmem<STAGES>;
  constexpr int BN = L::BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sC = smem + L::kCOff;
  uint8_t* sD = smem + L::kDOff;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* c_full = tempty + 2;
  uint64_t* c_empty = c_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(c_empty + 1);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = ptx::lane_id();
  const int m_tiles = (rows + kGemmBM - 1) / kGemmBM;  // partial last tile: clipped maps
  const int n_tiles = (N + BN - 1) / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int kblocks = (K + kGemmBK - 1) / kGemmBK;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tma_a);
    ptx::prefetch_tmap(&tma_b);
    ptx::prefetch_tmap(&tma_h32);
    ptx::prefetch_tmap(&tma_hb);
    ptx::prefetch_tmap(&tma_h32_out);
    ptx::prefetch_tmap(&tma_hb_out);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 128);
    }
    ptx::mbar_init(c_full, 1);
    ptx::mbar_init(c_empty, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<256>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // weights (B) in flight before the PDL wait (see gemm_bf16_tn_kernel)
  int preloaded = 0;
  if (warp == 0 && lane == 0 && int(blockIdx.x) < num_tiles) {
    const int nt = int(blockIdx.x) / m_tiles;
    preloaded = min(STAGES, kblocks);
    for (int j = 0; j < preloaded; ++j) {
      ptx::mbar_arrive_expect_tx(&full[j], L::kStageBytes);
      ptx::tma_load_2d(smem + j * L::kStageBytes + L::kABytes, &tma_b, &full[j],
                       j * kGemmBK, nt * BN);
    }
  }
  ptx::pdl_wait();    // predecessor's outputs (A operand, residual, K/V) complete
  ptx::pdl_launch();  // successor may start its prologue as our CTAs retire

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int mt = tile % m_tiles;
        const int nt = tile / m_tiles;
        for (int kb = 0; kb < kblocks; ++kb) {
          uint8_t* sa = smem + stage * L::kStageBytes;
          uint8_t* sb = sa + L::kABytes;
          if (preloaded > 0) {
            --preloaded;
            ptx::tma_load_2d(sa, &tma_a, &full[stage], kb * kGemmBK, row0 + mt * kGemmBM);
          } else {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            ptx::mbar_arrive_expect_tx(&full[stage], L::kStageBytes);
            ptx::tma_load_2d(sa, &tma_a, &full[stage], kb * kGemmBK, row0 + mt * kGemmBM);
            ptx::tma_load_2d(sb, &tma_b, &full[stage], kb * kGemmBK, nt * BN);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 3) {
    // residual tiles on their own warp: the operand producer never waits for
    // the previous tile's epilogue stores
    if (lane == 0) {
      uint32_t c_phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int mt = tile % m_tiles;
        const int nt = tile / m_tiles;
        ptx::mbar_wait(c_empty, c_phase ^ 1);  // previous tile's stores drained sC
        ptx::mbar_arrive_expect_tx(c_full, 4 * 16384);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          ptx::tma_load_2d(sC + c * 16384, &tma_h32, c_full, nt * BN + 32 * c,
                           row0 + mt * kGemmBM);
        c_phase ^= 1;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(kGemmBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_base = ptx::smem_u32(smem + stage * L::kStageBytes);
          const uint32_t b_base = a_base + L::kABytes;
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k)
            ptx::umma_bf16_ss(d_tmem, ptx::desc_kmajor_sw128(a_base + k * 32),
                              ptx::desc_kmajor_sw128(b_base + k * 32), idesc, (kb | k) != 0);
          ptx::umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::umma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int r = 32 * q + int(lane);  // row within the tile == TMEM lane
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t c_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int mt = tile % m_tiles;
      const int nt = tile / m_tiles;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::mbar_wait(c_full, c_phase);
      ptx::tc_fence_after();
      bool bad = false;
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        ptx::tmem_ld32(tmem_base + (uint32_t(32 * q) << 16) + acc * BN + 32 * c, v);
        ptx::tmem_wait_ld();
        bad |= resid_chunk<kMod>(sC, sD, r, c, v, nt * BN + 32 * c,
                                 row0 + mt * kGemmBM + r, args);
      }
      if (bad && args.flag) atomicMin(args.flag, args.code);
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
      ptx::fence_proxy_async_smem();
      ptx::named_bar_sync(1, 128);
      if (warp == 4 && lane == 0) {
        const int gr = row0 + mt * kGemmBM;
#pragma unroll
        for (int c = 0; c < 4; ++c) ptx::tma_store_2d(&tma_h32_out, sC + c * 16384, nt * BN + 32 * c, gr);
#pragma unroll
        for (int c = 0; c < 2; ++c) ptx::tma_store_2d(&tma_hb_out, sD + c * 16384, nt * BN + 64 * c, gr);
        ptx::tma_store_commit();
        ptx::tma_store_wait_read();
        ptx::mbar_arrive(c_empty);
      }
      c_phase ^= 1;
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    // outstanding stores must complete before the CTA exits
    if (warp == 4 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<256>(tmem_base);
  }
}


// ---------------------------------------------------------------------------
// CTA-pair residual GEMM with the TMA epilogue, 256 x 128 pair tiles, whole-
// tile epilogue buffer (measured faster than the part-streamed kernel below
// at this width): the 2-SM main loop of gemm2sm_bf16_tn_kernel and the smem
// residual epilogue of gemm_resid_tma_kernel, each CTA handling its own 128
// rows.
template <int STAGES>
struct Gemm2SmRes128Smem {
  static constexpr int BN = 128;
  static constexpr uint32_t kABytes = kGemmBM * kGemmBK * 2;
  static constexpr uint32_t kBBytes = (BN / 2) * kGemmBK * 2;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr uint32_t kCOff = STAGES * kStageBytes;
  static constexpr uint32_t kDOff = kCOff + 4 * 16384;
  static constexpr uint32_t kBarOffset = kDOff + 2 * 16384;
  static constexpr uint32_t kTotal = kBarOffset + 256 + 1024;
  static_assert(kTotal <= 232448, "2-SM residual GEMM smem budget");
};

template <int STAGES, bool kMod>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    gemm2sm_resid128_tma_kernel(const __grid_constant__ CUtensorMap tma_a,
                             const __grid_constant__ CUtensorMap tma_b,
                             const __grid_constant__ CUtensorMap tma_h32,
                             const __grid_constant__ CUtensorMap tma_hb,
                             const __grid_constant__ CUtensorMap tma_h32_out,
                             const __grid_constant__ CUtensorMap tma_hb_out, int rows, int row0,
                             int N, int K, ResidTmaArgs args) {
  using L = Gemm2SmRes128Smem<STAGES>;
  constexpr int BN = L::BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sC = smem + L::kCOff;
  uint8_t* sD = smem + L::kDOff;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* c_full = tempty + 2;
  uint64_t* c_empty = c_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(c_empty + 1);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = ptx::lane_id();
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;
  const int m_tiles = rows / (2 * kGemmBM);
  const int n_tiles = (N + BN - 1) / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int kblocks = (K + kGemmBK - 1) / kGemmBK;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tma_a);
    ptx::prefetch_tmap(&tma_b);
    ptx::prefetch_tmap(&tma_h32);
    ptx::prefetch_tmap(&tma_hb);
    ptx::prefetch_tmap(&tma_h32_out);
    ptx::prefetch_tmap(&tma_hb_out);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 2);
    }
    ptx::mbar_init(c_full, 1);
    ptx::mbar_init(c_empty, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_2sm<256>(tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  ptx::pdl_wait();    // predecessor's outputs (A operand, residual, K/V) complete
  ptx::pdl_launch();  // successor may start its prologue as our CTAs retire

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t c_phase = 0;
      for (int tile = cluster; tile < num_tiles; tile += nclusters) {
        const int mt = tile % m_tiles;
        const int nt = tile / m_tiles;
        const int my_row = row0 + mt * 2 * kGemmBM + int(rank) * kGemmBM;
        for (int kb = 0; kb < kblocks; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * L::kStageBytes;
          uint8_t* sb = sa + L::kABytes;
          if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * L::kStageBytes);
          ptx::tma_load_2d_2sm(sa, &tma_a, &full[stage], kb * kGemmBK, my_row);
          ptx::tma_load_2d_2sm(sb, &tma_b, &full[stage], kb * kGemmBK,
                               nt * BN + int(rank) * (BN / 2));
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::mbar_wait(c_empty, c_phase ^ 1);
        ptx::mbar_arrive_expect_tx(c_full, 4 * 16384);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          ptx::tma_load_2d(sC + c * 16384, &tma_h32, c_full, nt * BN + 32 * c, my_row);
        c_phase ^= 1;
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(2 * kGemmBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = cluster; tile < num_tiles; tile += nclusters) {
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_base = ptx::smem_u32(smem + stage * L::kStageBytes);
          const uint32_t b_base = a_base + L::kABytes;
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k)
            ptx::umma2_bf16_ss(d_tmem, ptx::desc_kmajor_sw128(a_base + k * 32),
                               ptx::desc_kmajor_sw128(b_base + k * 32), idesc, (kb | k) != 0);
          ptx::umma2_commit_mc(&empty[stage], 0x3);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::umma2_commit_mc(&tfull[acc], 0x3);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int r = 32 * q + int(lane);
    const uint32_t tempty_leader0 = ptx::mapa_shared(ptx::smem_u32(&tempty[0]), 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t c_phase = 0;
    for (int tile = cluster; tile < num_tiles; tile += nclusters) {
      const int mt = tile % m_tiles;
      const int nt = tile / m_tiles;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::mbar_wait(c_full, c_phase);
      ptx::tc_fence_after();
      bool bad = false;
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        ptx::tmem_ld32(tmem_base + (uint32_t(32 * q) << 16) + acc * BN + 32 * c, v);
        ptx::tmem_wait_ld();
        bad |= resid_chunk<kMod>(sC, sD, r, c, v, nt * BN + 32 * c,
                                 row0 + mt * 2 * kGemmBM + int(rank) * kGemmBM + r, args);
      }
      if (bad && args.flag) atomicMin(args.flag, args.code);
      ptx::tc_fence_before();
      ptx::fence_proxy_async_smem();
      ptx::named_bar_sync(1, 128);
      if (warp == 4 && lane == 0) {
        ptx::mbar_arrive_cluster(tempty_leader0 + acc * 8);
        const int gr = row0 + mt * 2 * kGemmBM + int(rank) * kGemmBM;
#pragma unroll
        for (int c = 0; c < 4; ++c) ptx::tma_store_2d(&tma_h32_out, sC + c * 16384, nt * BN + 32 * c, gr);
#pragma unroll
        for (int c = 0; c < 2; ++c) ptx::tma_store_2d(&tma_hb_out, sD + c * 16384, nt * BN + 64 * c, gr);
        ptx::tma_store_commit();
        ptx::tma_store_wait_read();
        ptx::mbar_arrive(c_empty);
      }
      c_phase ^= 1;
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (warp == 4 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_2sm<256>(tmem_base);
  }
}

// ---------------------------------------------------------------------------
// CTA-pair residual GEMM with the TMA epilogue (256 x BN pair tiles, BN 128 or
// 192): the 2-SM main loop of gemm2sm_bf16_tn_kernel and the smem residual
// epilogue of gemm_resid_tma_kernel, each CTA handling its own 128 rows.
// Wider pair tiles cut the L2 -> SM traffic of the A operand (each A row tile
// is re-read N / BN times). The epilogue streams the tile in 64-column parts
// through two smem buffers (fp32 residual 2 x [128 x 32], bf16 copy
// [128 x 64]): warp 3 TMA-loads part g + 1's residual while part g is added
// and TMA-stored.
template <int BN_, int STAGES>
struct Gemm2SmResSmem {
  static constexpr int BN = BN_;
  static constexpr int kParts = BN / 64;
  static constexpr uint32_t kABytes = kGemmBM * kGemmBK * 2;
  static constexpr uint32_t kBBytes = (BN / 2) * kGemmBK * 2;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr uint32_t kPartBytes = 2 * 16384 + 16384;  // fp32 2 x 16 KB + bf16 16 KB
  static constexpr uint32_t kCOff = STAGES * kStageBytes;
  static constexpr uint32_t kBarOffset = kCOff + 2 * kPartBytes;
  static constexpr uint32_t kTotal = kBarOffset + 256 + 1024;
  static constexpr uint32_t kTmemCols = 2 * BN <= 256 ? 256 : 512;
  static_assert(BN % 64 == 0 && BN <= 256, "residual pair tile");
  static_assert(((BN / 2) * 128) % 1024 == 0 || BN == 192, "B half alignment");
  static_assert(kTotal <= 232448, "2-SM residual GEMM smem budget");
};

template <int BN, int STAGES, bool kMod>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    gemm2sm_resid_tma_kernel(const __grid_constant__ CUtensorMap tma_a,
                             const __grid_constant__ CUtensorMap tma_b,
                             const __grid_constant__ CUtensorMap tma_h32,
                             const __grid_constant__ CUtensorMap tma_hb,
                             const __grid_constant__ CUtensorMap tma_h32_out,
                             const __grid_constant__ CUtensorMap tma_hb_out, int rows, int row0,
                             int N, int K, ResidTmaArgs args) {
  using L = Gemm2SmResSmem<BN, STAGES>;
  constexpr int kParts = L::kParts;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sE = smem + L::kCOff;  // 2 x part buffers: [fp32 32 KB | bf16 16 KB]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* c_full = tempty + 2;   // [2]
  uint64_t* c_empty = c_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(c_empty + 2);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = ptx::lane_id();
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;
  const int m_tiles = rows / (2 * kGemmBM);
  const int n_tiles = (N + BN - 1) / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int kblocks = (K + kGemmBK - 1) / kGemmBK;
  const bool sk = args.sk_ws != nullptr;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tma_a);
    ptx::prefetch_tmap(&tma_b);
    ptx::prefetch_tmap(&tma_h32);
    ptx::prefetch_tmap(&tma_hb);
    ptx::prefetch_tmap(&tma_h32_out);
    ptx::prefetch_tmap(&tma_hb_out);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 2);
      ptx::mbar_init(&c_full[a], 1);
      ptx::mbar_init(&c_empty[a], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_2sm<L::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  ptx::pdl_wait();    // predecessor's outputs (A operand, residual, K/V) complete
  ptx::pdl_launch();  // successor may start its prologue as our CTAs retire

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      ResidTiles it(sk, cluster, nclusters, num_tiles, kblocks);
      for (int tile, kb0, kb1; it.next(tile, kb0, kb1);) {
        const int mt = tile % m_tiles;
        const int nt = tile / m_tiles;
        const int my_row = row0 + mt * 2 * kGemmBM + int(rank) * kGemmBM;
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * L::kStageBytes;
          uint8_t* sb = sa + L::kABytes;
          if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * L::kStageBytes);
          ptx::tma_load_2d_2sm(sa, &tma_a, &full[stage], kb * kGemmBK, my_row);
          ptx::tma_load_2d_2sm(sb, &tma_b, &full[stage], kb * kGemmBK,
                               nt * BN + int(rank) * (BN / 2));
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 3) {
    // residual parts, one ahead of the epilogue (double-buffered)
    if (lane == 0) {
      int g = 0;
      ResidTiles it(sk, cluster, nclusters, num_tiles, kblocks);
      for (int tile, kb0, kb1; it.next(tile, kb0, kb1);) {
        if (kb1 < kblocks) continue;  // head partial: no residual
        const int mt = tile % m_tiles;
        const int nt = tile / m_tiles;
        const int my_row = row0 + mt * 2 * kGemmBM + int(rank) * kGemmBM;
        for (int part = 0; part < kParts; ++part, ++g) {
          const int b = g & 1;
          uint8_t* sc = sE + b * L::kPartBytes;
          ptx::mbar_wait(&c_empty[b], ((g >> 1) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&c_full[b], 2 * 16384);
#pragma unroll
          for (int c = 0; c < 2; ++c)
            ptx::tma_load_2d(sc + c * 16384, &tma_h32, &c_full[b], nt * BN + 64 * part + 32 * c,
                             my_row);
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(2 * kGemmBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      ResidTiles it(sk, cluster, nclusters, num_tiles, kblocks);
      for (int tile, kb0, kb1; it.next(tile, kb0, kb1);) {
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_base = ptx::smem_u32(smem + stage * L::kStageBytes);
          const uint32_t b_base = a_base + L::kABytes;
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k)
            ptx::umma2_bf16_ss(d_tmem, ptx::desc_kmajor_sw128(a_base + k * 32),
                               ptx::desc_kmajor_sw128(b_base + k * 32), idesc,
                               (kb != kb0) || (k != 0));
          ptx::umma2_commit_mc(&empty[stage], 0x3);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::umma2_commit_mc(&tfull[acc], 0x3);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int r = 32 * q + int(lane);
    const uint32_t tempty_leader0 = ptx::mapa_shared(ptx::smem_u32(&tempty[0]), 0);
    const bool elect = warp == 4 && lane == 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int g = 0;
    const int my_cta = int(blockIdx.x);
    ResidTiles it(sk, cluster, nclusters, num_tiles, kblocks);
    for (int tile, kb0, kb1; it.next(tile, kb0, kb1);) {
      const int mt = tile % m_tiles;
      const int nt = tile / m_tiles;
      const int gr = row0 + mt * 2 * kGemmBM + int(rank) * kGemmBM;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      if (kb1 < kblocks) {
        // head of a tile the next pair finishes: publish the fp32 partial
        // ([BN cols][128 rows] per CTA: coalesced over the rows of a warp)
        float* ws = args.sk_ws + size_t(my_cta) * BN * kGemmBM + r;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t v[32];
          ptx::tmem_ld32(tmem_base + (uint32_t(32 * q) << 16) + acc * BN + 32 * c, v);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) __stcg(ws + size_t(32 * c + j) * kGemmBM, __uint_as_float(v[j]));
        }
        ptx::tc_fence_before();
        __threadfence();
        ptx::named_bar_sync(1, 128);
        if (elect) {
          ptx::mbar_arrive_cluster(tempty_leader0 + acc * 8);
          ptx::st_release_gpu(args.sk_flags + my_cta, 1);
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        continue;
      }
      const float* pws = nullptr;  // head partial of this tile (previous pair)
      if (kb0 > 0) {
        const int src = my_cta - 2;
        if (elect) {
          while (ptx::ld_acquire_gpu(args.sk_flags + src) == 0) __nanosleep(64);
          args.sk_flags[src] = 0;
        }
        ptx::named_bar_sync(1, 128);
        pws = args.sk_ws + size_t(src) * BN * kGemmBM + r;
      }
      bool bad = false;
      for (int part = 0; part < kParts; ++part, ++g) {
        const int b = g & 1;
        uint8_t* sc = sE + b * L::kPartBytes;
        uint8_t* sd = sc + 2 * 16384;
        uint32_t v0[32], v1[32];
        const uint32_t tcol = tmem_base + (uint32_t(32 * q) << 16) + acc * BN + 64 * part;
        ptx::tmem_ld32(tcol, v0);
        ptx::tmem_ld32(tcol + 32, v1);
        if (pws) {
          float p0[32], p1[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            p0[j] = __ldcg(pws + size_t(64 * part + j) * kGemmBM);
            p1[j] = __ldcg(pws + size_t(64 * part + 32 + j) * kGemmBM);
          }
          ptx::tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            v0[j] = __float_as_uint(__uint_as_float(v0[j]) + p0[j]);
            v1[j] = __float_as_uint(__uint_as_float(v1[j]) + p1[j]);
          }
        }
        ptx::mbar_wait(&c_full[b], (g >> 1) & 1);
        ptx::tmem_wait_ld();
        if (part == kParts - 1) {
          // every TMEM column of this accumulator is in registers
          ptx::tc_fence_before();
          ptx::named_bar_sync(1, 128);
          if (elect) ptx::mbar_arrive_cluster(tempty_leader0 + acc * 8);
        }
        bad |= resid_chunk<kMod>(sc, sd, r, 0, v0, nt * BN + 64 * part, gr + r, args);
        bad |= resid_chunk<kMod>(sc, sd, r, 1, v1, nt * BN + 64 * part + 32, gr + r, args);
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(1, 128);
        if (elect) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
            ptx::tma_store_2d(&tma_h32_out, sc + c * 16384, nt * BN + 64 * part + 32 * c, gr);
          ptx::tma_store_2d(&tma_hb_out, sd, nt * BN + 64 * part, gr);
          ptx::tma_store_commit();
          // release the buffer to the loader as soon as the stores have read
          // it (the other epilogue threads meanwhile load the next part)
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          ptx::mbar_arrive(&c_empty[b]);
        }
      }
      if (bad && args.flag) atomicMin(args.flag, args.code);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (elect) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_2sm<L::kTmemCols>(tmem_base);
  }
}

}  // namespace pf
