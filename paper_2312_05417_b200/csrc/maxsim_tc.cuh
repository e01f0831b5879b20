// maxsim_tc.cuh -- K2: fused gather + MaxSim on the sm_100a tensor cores.
//
// Restates maxsim_score (proj/include/espn/scoring.hpp:7-10) for
// a whole batch of (query, candidate) pairs, fused with the candidate gather of
// StoreHandle::fetch_batch (store.hpp:91-94) and with no score matrix in HBM.
//
// Mapping:
//   * A work unit is (query b, up to `unit_docs` consecutive needed candidates).
//     Each doc's t token rows are packed into a stream of 8-aligned "slots"
//     (the last row is duplicated into the pad slots, which leaves the max
//     unchanged); a stage holds 4 quarters x NQC slots.
//   * Producer warps gather rows HBM -> SMEM with 16-byte cp.async straight into
//     the UMMA K-major core-matrix layout (no staging copy, no register hop).
//   * One thread issues tcgen05.mma (M=128, N<=NQC, K=16) per quarter and K-step.
//     A is a 128-row window over [96 zero rows | Q (32 rows) | 96 zero rows]
//     whose offset puts the query tokens on TMEM lanes 32w..32w+31 for quarter
//     w ("block-diagonal" A), so all four lane quarters -- and all four
//     epilogue warps -- get useful work from every MMA.
//   * Epilogue warp w reads its lanes with tcgen05.ld: thread i holds query
//     token i's dot products against the quarter's doc tokens along columns,
//     so max over doc tokens is an in-register running max; per-doc partial
//     maxima go to SMEM and one thread per doc sums the q maxima in ascending
//     query-token order (the oracle's summation order).
#pragma once
#include "common.cuh"
#include "ptx.cuh"

namespace espn_k {

template <int D>
struct TcCfg;
template <> struct TcCfg<16>  { static constexpr int NQC = 128, NS = 4, UNITMAX = 64, P = 2; };
template <> struct TcCfg<32>  { static constexpr int NQC = 128, NS = 4, UNITMAX = 64, P = 2; };
template <> struct TcCfg<64>  { static constexpr int NQC = 64,  NS = 3, UNITMAX = 64, P = 2; };
template <> struct TcCfg<128> { static constexpr int NQC = 32,  NS = 3, UNITMAX = 32, P = 2; };

template <int D>
struct TcLayout {
  using C = TcCfg<D>;
  static constexpr int NQC = C::NQC, NS = C::NS, UNITMAX = C::UNITMAX, P = C::P;
  static constexpr int CH = D / 8;                 // 16-byte chunks per token row
  static constexpr int SBO = CH * 128;             // bytes between 8-row core-matrix groups
  static constexpr int LBO = 128;                  // bytes between K-adjacent core matrices
  static constexpr int KSTEPS = D / 16;
  static constexpr int STAGE_SLOTS = 4 * NQC;
  static constexpr int QBYTES = NQC * D * 2;       // one quarter of a stage
  static constexpr int STAGE_BYTES = 4 * QBYTES;
  static constexpr int A_ROWS = 96 + 2 * 128;      // zeros | Q0 | zeros | Q1 | zeros
  static constexpr int A_BYTES = A_ROWS * D * 2;
  static constexpr int MAX_SLOTS = UNITMAX * 64;   // slot budget of one unit
  static constexpr int MAXW = MAX_SLOTS / 8 / 32;  // bitmap words (one bit per 8-slot group)
  static constexpr int PM_STRIDE = UNITMAX + 1;    // padded: conflict-free emits and combine
  static constexpr int PM_FLOATS = 4 * 32 * PM_STRIDE;
  static constexpr int NBUF = (512 / NQC) < 4 ? (512 / NQC) : 4;
  static constexpr uint32_t TMEM_COLS = NBUF * NQC <= 32 ? 32 : NBUF * NQC <= 64 ? 64
                                      : NBUF * NQC <= 128 ? 128 : NBUF * NQC <= 256 ? 256 : 512;
  static constexpr int NWARPS = 5 + P;             // 4 epilogue, 1 MMA, P producers
  static constexpr int NTHREADS = NWARPS * 32;

  struct Unit {
    uint32_t b, j0, nd, S;
    uint32_t bitmap[MAXW];
    uint32_t wprefix[MAXW];
    uint64_t row[UNITMAX];
    uint32_t t[UNITMAX];
    uint32_t slot[UNITMAX];
  };
  // Byte offsets inside dynamic shared memory (1024-aligned base).
  static constexpr int OFF_B = 0;
  static constexpr int OFF_A = OFF_B + NS * STAGE_BYTES;
  static constexpr int OFF_PM = OFF_A + A_BYTES;
  static constexpr int OFF_UNIT = OFF_PM + PM_FLOATS * 4;
  static constexpr int OFF_BAR = (OFF_UNIT + 2 * (int)sizeof(Unit) + 7) / 8 * 8;
  static constexpr int N_BARS = 2 * NS + 2 * NBUF + 4;
  static constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
  static constexpr int SMEM_BYTES = OFF_TMEM + 16;
};

template <int D>
__global__ void __launch_bounds__(TcLayout<D>::NTHREADS, 1)
maxsim_tc_kernel(const MaxSimParams p) {
  using L = TcLayout<D>;
  using namespace espn_ptx;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sB = smem + L::OFF_B;
  uint8_t* sA = smem + L::OFF_A;
  float* pm = reinterpret_cast<float*>(smem + L::OFF_PM);
  typename L::Unit* units = reinterpret_cast<typename L::Unit*>(smem + L::OFF_UNIT);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* full_bar = bars;                       // [NS]  producers -> MMA
  uint64_t* empty_bar = bars + L::NS;              // [NS]  MMA commit -> producers
  uint64_t* tfull_bar = bars + 2 * L::NS;          // [NBUF] MMA commit -> epilogue
  uint64_t* tempty_bar = tfull_bar + L::NBUF;      // [NBUF] epilogue -> MMA
  uint64_t* ufull_bar = tempty_bar + L::NBUF;      // [2] producers -> MMA, epilogue
  uint64_t* uempty_bar = ufull_bar + 2;            // [2] epilogue -> producers
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  // ---- one-time setup: zero operand tiles (stale NaN bit patterns would leak
  // into other quarters through the zero rows of A), barriers, TMEM ----------
  {
    uint4* z = reinterpret_cast<uint4*>(smem);
    const int n16 = (L::OFF_PM) / 16;
    for (int i = tid; i < n16; i += L::NTHREADS) z[i] = make_uint4(0, 0, 0, 0);
  }
  fence_proxy_async_smem();
  if (tid == 0) {
    for (int i = 0; i < L::NS; ++i) {
      mbar_init(&full_bar[i], L::P * 32);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < L::NBUF; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&ufull_bar[i], 1);
      mbar_init(&uempty_bar[i], 1);
    }
    mbar_fence_init();
  }
  if (warp == 4) tmem_alloc<L::TMEM_COLS>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const uint32_t n_units = p.n_units;

  if (warp >= 5) {
    // =========================== PRODUCERS ===================================
    const int pw = warp - 5;
    uint32_t gs = 0;  // global stage counter
    for (uint32_t it = 0;; ++it) {
      const uint32_t ug = blockIdx.x + it * gridDim.x;
      if (ug >= n_units) break;
      const uint32_t us = it & 1;
      typename L::Unit& U = units[us];
      mbar_wait(&uempty_bar[us], ((it >> 1) & 1) ^ 1);
      // Locate the unit: query b owns units [unit_off[b], unit_off[b+1]).
      uint32_t lo = 0, hi = p.n_queries;  // find b with unit_off[b] <= ug < unit_off[b+1]
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(&p.unit_off[mid]) <= ug) lo = mid; else hi = mid;
      }
      const uint32_t b = lo;
      const uint32_t chunk = ug - __ldg(&p.unit_off[b]);
      const uint64_t c0 = __ldg(&p.cand_off[b]);
      const uint32_t n_needed = __ldg(&p.needed[b]);
      const uint32_t j0 = chunk * p.unit_docs;
      const uint32_t nd = min(p.unit_docs, n_needed - j0);
      if (pw == 0) {
        // doc info + slot prefix sum (warp scan) + doc-start bitmap
        for (int i = lane; i < L::MAXW; i += 32) U.bitmap[i] = 0;
        __syncwarp();
        uint32_t carry = 0;
        for (uint32_t k0 = 0; k0 < nd; k0 += 32) {
          const uint32_t k = k0 + lane;
          uint32_t t = 0;
          uint64_t r0 = 0;
          if (k < nd) {
            const uint64_t loc = shard_local(__ldg(&p.cand_ids[c0 + j0 + k]), p.shard_count,
                                             p.shard_index, p.n_docs);
            if (loc != ~0ull) {
              r0 = __ldg(&p.row_ptr[loc]);
              t = (uint32_t)(__ldg(&p.row_ptr[loc + 1]) - r0);
            } else {
              atomicOr(p.err, ERR_UNKNOWN_DOC);
            }
          }
          const uint32_t pad = (t + 7u) & ~7u;
          uint32_t incl = pad;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
          }
          const uint32_t start = carry + incl - pad;
          if (k < nd) {
            U.row[k] = r0;
            U.t[k] = t;
            U.slot[k] = start;
            if (t > 0 && start < (uint32_t)L::MAX_SLOTS)
              atomicOr(&U.bitmap[start >> 8], 1u << ((start >> 3) & 31));
          }
          carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (carry > (uint32_t)L::MAX_SLOTS) {
          if (lane == 0) atomicOr(p.err, ERR_UNIT_TOO_LARGE);
          carry = 0;  // skip the unit's MMA work; the call fails on the host
        }
        __syncwarp();
        if (lane == 0) {
          uint32_t acc = 0;
          for (int i = 0; i < L::MAXW; ++i) {
            U.wprefix[i] = acc;
            acc += __popc(U.bitmap[i]);
          }
          U.b = b;
          U.j0 = (uint32_t)(c0 + j0);
          U.nd = nd;
          U.S = carry;
        }
      }
      if (pw == L::P - 1) {
        // Query tokens -> A slot `us` (rows 96+128*us .. +32), converted to the
        // table dtype; rows >= nq stay zero.
        const float* q = p.q32 + (size_t)b * p.nq * D;
        const int abase = 96 + 128 * (int)us;
        for (int e = lane; e < 32 * L::CH; e += 32) {
          const int i = e / L::CH, c = e % L::CH;
          uint32_t w4[4] = {0, 0, 0, 0};
          if ((uint32_t)i < p.nq) {
            bool bad = false;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const float x0 = __ldg(&q[i * D + c * 8 + 2 * h]);
              const float x1 = __ldg(&q[i * D + c * 8 + 2 * h + 1]);
              const uint16_t h0 = f32_to_code(x0, p.bf16), h1 = f32_to_code(x1, p.bf16);
              bad |= !isfinite(code_to_f32(h0, p.bf16)) || !isfinite(code_to_f32(h1, p.bf16));
              w4[h] = (uint32_t)h0 | ((uint32_t)h1 << 16);
            }
            if (bad) atomicOr(p.err, ERR_NONFINITE_QUERY);
          }
          const int r = abase + i;
          *reinterpret_cast<uint4*>(sA + (r >> 3) * L::SBO + c * L::LBO + (r & 7) * 16) =
              make_uint4(w4[0], w4[1], w4[2], w4[3]);
        }
        fence_proxy_async_smem();
      }
      named_bar_sync(1, L::P * 32);
      if (pw == 0 && lane == 0) mbar_arrive(&ufull_bar[us]);

      const uint32_t S = U.S;
      const uint32_t n_st = (S + L::STAGE_SLOTS - 1) / L::STAGE_SLOTS;
      uint32_t kcur = 0;  // first doc overlapping the current stage
      for (uint32_t st = 0; st < n_st; ++st, ++gs) {
        const uint32_t s = gs % L::NS;
        mbar_wait(&empty_bar[s], ((gs / L::NS) & 1) ^ 1);
        const uint32_t x0 = st * L::STAGE_SLOTS, x1 = x0 + L::STAGE_SLOTS;
        while (kcur < nd && U.slot[kcur] + ((U.t[kcur] + 7u) & ~7u) <= x0) ++kcur;
        const uint32_t sbase = smem_u32(sB + s * L::STAGE_BYTES);
        for (uint32_t k = kcur + pw; k < nd; k += L::P) {
          const uint32_t sk = U.slot[k];
          if (sk >= x1) break;
          const uint32_t t = U.t[k];
          const uint32_t pad = (t + 7u) & ~7u;
          const uint32_t a = max(sk, x0), e_ = min(sk + pad, x1);
          if (a >= e_) continue;
          const uint16_t* src_doc = p.rows + U.row[k] * D;
          const uint32_t n_copies = (e_ - a) * L::CH;
          for (uint32_t e = lane; e < n_copies; e += 32) {
            const uint32_t sl = a + e / L::CH, c = e % L::CH;
            const uint32_t tok = min(sl - sk, t - 1u);
            const uint32_t rel = sl - x0;
            const uint32_t w = rel / L::NQC, n = rel % L::NQC;
            const uint32_t dst = sbase + w * L::QBYTES + (n >> 3) * L::SBO + c * L::LBO + (n & 7) * 16;
            cp_async_16(dst, src_doc + (size_t)tok * D + c * 8);
          }
        }
        cp_async_mbar_arrive_noinc(&full_bar[s]);
      }
    }
    cp_async_wait_all();
  } else if (warp == 4) {
    // ============================ MMA ISSUER ==================================
    if (lane == 0) {
      uint32_t gs = 0;
      const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
      for (uint32_t it = 0;; ++it) {
        const uint32_t ug = blockIdx.x + it * gridDim.x;
        if (ug >= n_units) break;
        const uint32_t us = it & 1;
        mbar_wait(&ufull_bar[us], (it >> 1) & 1);
        const uint32_t S = units[us].S;
        const uint32_t n_st = (S + L::STAGE_SLOTS - 1) / L::STAGE_SLOTS;
        for (uint32_t st = 0; st < n_st; ++st, ++gs) {
          const uint32_t s = gs % L::NS, buf = gs % L::NBUF;
          mbar_wait(&full_bar[s], (gs / L::NS) & 1);
          mbar_wait(&tempty_bar[buf], ((gs / L::NBUF) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + buf * L::NQC;
          const uint32_t x0 = st * L::STAGE_SLOTS;
          uint32_t acc = 0;
#pragma unroll 1
          for (int w = 0; w < 4; ++w) {
            const int rem = (int)S - (int)(x0 + w * L::NQC);
            if (rem <= 0) break;
            const uint32_t nv = rem < L::NQC ? (uint32_t)rem : (uint32_t)L::NQC;
            const uint32_t n_mma = (nv + 15u) & ~15u;
            const uint32_t idesc = umma_idesc_f16(128, n_mma, p.bf16);
            const uint32_t a_row0 = 96 + 128 * us - 32 * w;
            const uint32_t a_addr = a_base + (a_row0 >> 3) * L::SBO;
            const uint32_t b_addr = b_base + s * L::STAGE_BYTES + w * L::QBYTES;
#pragma unroll
            for (int ks = 0; ks < L::KSTEPS; ++ks) {
              const uint64_t ad = umma_desc_kmajor(a_addr + ks * 2 * L::LBO, L::LBO, L::SBO);
              const uint64_t bd = umma_desc_kmajor(b_addr + ks * 2 * L::LBO, L::LBO, L::SBO);
              umma_f16(d_tmem, ad, bd, idesc, acc);
              acc = 1;
            }
          }
          umma_commit(&empty_bar[s]);
          umma_commit(&tfull_bar[buf]);
        }
      }
    }
    __syncwarp();
  } else {
    // ============================ EPILOGUE (warps 0-3) ===========================
    const int w = warp;  // TMEM lane quarter == query-token quarter
    float* my_pm = pm + (w * 32 + lane) * L::PM_STRIDE;
    uint32_t gs = 0;
    for (uint32_t it = 0;; ++it) {
      const uint32_t ug = blockIdx.x + it * gridDim.x;
      if (ug >= n_units) break;
      const uint32_t us = it & 1;
      const typename L::Unit& U = units[us];
      mbar_wait(&ufull_bar[us], (it >> 1) & 1);
      const uint32_t S = U.S, nd = U.nd, j0 = U.j0;
      for (uint32_t k = 0; k < nd; ++k) my_pm[k] = -INFINITY;
      const uint32_t n_st = (S + L::STAGE_SLOTS - 1) / L::STAGE_SLOTS;
      for (uint32_t st = 0; st < n_st; ++st, ++gs) {
        const uint32_t buf = gs % L::NBUF;
        mbar_wait(&tfull_bar[buf], (gs / L::NBUF) & 1);
        tc_fence_after();
        const uint32_t xw = st * L::STAGE_SLOTS + w * L::NQC;
        const int remv = (int)S - (int)xw;
        if (remv > 0) {
          const uint32_t nv = remv < L::NQC ? (uint32_t)remv : (uint32_t)L::NQC;
          const uint32_t G0 = xw >> 3;
          int doc = (int)(U.wprefix[G0 >> 5] + __popc(U.bitmap[G0 >> 5] & ((2u << (G0 & 31)) - 1u))) - 1;
          float m = -INFINITY;
          const uint32_t taddr0 = tmem_base + ((uint32_t)(w * 32) << 16) + buf * L::NQC;
          for (uint32_t c0 = 0; c0 < nv; c0 += 32) {
            float v[32];
            tmem_ld_32x32b_x32(taddr0 + c0, v);
            const uint32_t G = (xw + c0) >> 3;  // multiple of 4
            const uint32_t bits = (U.bitmap[G >> 5] >> (G & 31)) & 0xFu;
            tmem_ld_wait();
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              if (c0 + 8 * g < nv) {
                float gm = fmaxf(fmaxf(fmaxf(v[8 * g + 0], v[8 * g + 1]), fmaxf(v[8 * g + 2], v[8 * g + 3])),
                                 fmaxf(fmaxf(v[8 * g + 4], v[8 * g + 5]), fmaxf(v[8 * g + 6], v[8 * g + 7])));
                if (((bits >> g) & 1u) && (c0 + 8 * g) > 0) {
                  my_pm[doc] = fmaxf(my_pm[doc], m);
                  ++doc;
                  m = gm;
                } else {
                  m = fmaxf(m, gm);
                }
              }
            }
          }
          my_pm[doc] = fmaxf(my_pm[doc], m);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[buf]);
      }
      // ---- combine: bow(doc) = sum_i max_w pm[w][i][doc], i ascending ----
      named_bar_sync(2, 128);
      for (uint32_t k = tid; k < nd; k += 128) {
        float s = 0.0f;
        for (uint32_t i = 0; i < p.nq; ++i) {
          const float a0 = pm[(0 * 32 + i) * L::PM_STRIDE + k];
          const float a1 = pm[(1 * 32 + i) * L::PM_STRIDE + k];
          const float a2 = pm[(2 * 32 + i) * L::PM_STRIDE + k];
          const float a3 = pm[(3 * 32 + i) * L::PM_STRIDE + k];
          s = __fadd_rn(s, fmaxf(fmaxf(a0, a1), fmaxf(a2, a3)));
        }
        p.bow_out[j0 + k] = s;
      }
      named_bar_sync(2, 128);
      if (tid == 0) mbar_arrive(&uempty_bar[us]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc<L::TMEM_COLS>(tmem_base);
  }
}

}  // namespace espn_k
