// maxsim_tc.cuh -- K2: fused gather + MaxSim on the sm_100a tensor cores.
//
// Restates maxsim_score (proj/include/espn/scoring.hpp:7-10) for
// a whole batch of (query, candidate) pairs, fused with the candidate gather of
// StoreHandle::fetch_batch (store.hpp:91-94) and with no score matrix in HBM.
//
// Mapping:
//   * A work unit is (query b, up to `unit_docs` consecutive needed candidates).
//     Each doc's t token rows occupy ceil8(t) consecutive 8-aligned "slots";
//     a stage holds 4 quarters x NQC slots.
//   * The table is stored in the HBM tile layout (RowLayout, common.cuh), so a
//     document is one contiguous byte range per K-panel that ONE 1-D
//     cp.async.bulk (TMA engine, UBLKCP) lands directly in the UMMA K-major
//     SWIZZLE_{32,64,128}B operand layout -- no per-element address math, no
//     register hop.  Pad slots of a doc's last 8-row group are not copied; the
//     epilogue masks those columns.
//   * Warp roles: 0-3 epilogue, 4 MMA issuer (one thread), 5 bulk-copy
//     producer, 6 unit loader (candidate ids -> row offsets, slot plan, query
//     tile) running NU-1 units ahead so the dependent id->row_ptr loads are off
//     the copy path.
//   * tcgen05.mma (M=128, N<=NQC, K=16) per quarter and K-step.  A is a 128-row
//     window over [96 zero rows | Q (32 rows) | 96 zero rows ...] whose offset
//     puts the query tokens on TMEM lanes 32w..32w+31 for quarter w
//     ("block-diagonal" A), so all four lane quarters -- and all four epilogue
//     warps -- get useful work from every MMA into one accumulator buffer.
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
template <> struct TcCfg<16>  { static constexpr int NQC = 128, NS = 6, UNITMAX = 64, NU = 3; };
template <> struct TcCfg<32>  { static constexpr int NQC = 128, NS = 4, UNITMAX = 64, NU = 3; };
template <> struct TcCfg<64>  { static constexpr int NQC = 64,  NS = 3, UNITMAX = 64, NU = 3; };
template <> struct TcCfg<128> { static constexpr int NQC = 32,  NS = 3, UNITMAX = 32, NU = 2; };

template <int D>
struct TcLayout {
  using C = TcCfg<D>;
  using RL = RowLayout<D>;
  static constexpr int NQC = C::NQC, NS = C::NS, UNITMAX = C::UNITMAX, NU = C::NU;
  static constexpr int ROWB = RL::ROWB, PW = RL::PW, NP = RL::NP;
  static constexpr uint32_t SWZ = PW == 128 ? 2u : PW == 64 ? 4u : 6u;  // UMMA layout code
  static constexpr int KSTEPS = D / 16;
  static constexpr int STAGE_SLOTS = 4 * NQC;
  static constexpr int PANEL_BYTES = STAGE_SLOTS * PW;  // one K-panel of a stage
  static constexpr int STAGE_BYTES = NP * PANEL_BYTES;
  // A (query) operand: K-major SWIZZLE_NONE core matrices
  static constexpr int CH = D / 8;                 // 16-byte chunks per query row
  static constexpr int A_SBO = CH * 128;
  static constexpr int A_LBO = 128;
  static constexpr int A_ROWS = 96 + NU * 128;     // zeros | Q0 | zeros | Q1 | ...
  static constexpr int A_BYTES = A_ROWS * D * 2;
  static constexpr int MAX_SLOTS = UNITMAX * 64;   // slot budget of one unit
  static constexpr int NG = MAX_SLOTS / 8;         // 8-slot groups
  static constexpr int MAXW = NG / 32;             // bitmap words (one bit per group)
  static constexpr int MAX_STAGES = MAX_SLOTS / STAGE_SLOTS;  // stages of a full unit
  static constexpr int PM_STRIDE = UNITMAX + 1;    // padded: conflict-free emits and combine
  static constexpr int PM_FLOATS = NU * 32 * PM_STRIDE;  // per unit slot: [query token][doc] keys
  static constexpr int NBUF = (512 / NQC) < 4 ? (512 / NQC) : 4;
  static constexpr uint32_t TMEM_COLS = NBUF * NQC <= 32 ? 32 : NBUF * NQC <= 64 ? 64
                                      : NBUF * NQC <= 128 ? 128 : NBUF * NQC <= 256 ? 256 : 512;
  static constexpr int NPROD = 2;                  // bulk-copy producer warps
  static constexpr int NEPI = 8;                   // epilogue warps: 4 lane quarters x 2 column halves
  static constexpr int MMA_WARP = NEPI;
  static constexpr int PROD_WARP0 = NEPI + 1;
  static constexpr int LOADER_WARP = PROD_WARP0 + NPROD;
  static constexpr int COMBINE_WARP = LOADER_WARP + 1;
  static constexpr int NWARPS = COMBINE_WARP + 1;
  static constexpr int HALF = NQC / 2;             // columns per epilogue warp per stage
  static constexpr int LW = HALF < 32 ? HALF : 32; // tcgen05.ld width (columns)
  static constexpr int NLD = HALF / LW;            // loads per epilogue warp per stage
  static constexpr int NGH = HALF / 8;             // 8-slot groups per epilogue warp per stage
  static constexpr int NTHREADS = NWARPS * 32;

  struct Unit {
    uint32_t b, nd, S, pad_;
    uint64_t cfirst;            // candidate index of the unit's first doc
    uint32_t bitmap[MAXW];      // bit g: a doc starts at group g
    uint32_t wprefix[MAXW];     // docs starting before word w
    uint64_t src[UNITMAX];      // address of the doc's rows (table or staging buffer)
    uint32_t t[UNITMAX];
    uint32_t slot[UNITMAX];
    uint8_t gvalid[NG];         // valid (non-pad) columns of group g, 1..8
    uint32_t kbeg[MAX_STAGES];  // docs [kbeg, kend) have rows in stage st
    uint32_t kend[MAX_STAGES];
  };
  // Byte offsets inside dynamic shared memory (1024-aligned base).
  static constexpr int OFF_B = 0;
  static constexpr int OFF_A = OFF_B + NS * STAGE_BYTES;
  static constexpr int OFF_PM = OFF_A + A_BYTES;
  static constexpr int OFF_UNIT = OFF_PM + PM_FLOATS * 4;
  static constexpr int OFF_BAR = (OFF_UNIT + NU * (int)sizeof(Unit) + 7) / 8 * 8;
  static constexpr int N_BARS = 2 * NS + 2 * NBUF + 3 * NU;
  static constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
  static constexpr int SMEM_BYTES = OFF_TMEM + 16 + 1024;  // + alignment slack
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  static_assert(STAGE_BYTES % 1024 == 0 && A_BYTES % 16 == 0, "alignment");
};

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// ESPN_DEBUG bit 8: CTA 0 records a per-unit timeline of its roles and prints it.
#define ESPN_STRACE(slot, g)                                                     \
  do {                                                                           \
    if ((p.dbg & 8u) && blockIdx.x == 0 && (g) < 16) strace[(slot) * 16 + (g)] = gtimer(); \
  } while (0)
#define ESPN_TRACE(slot, it)                                                     \
  do {                                                                           \
    if ((p.dbg & 8u) && blockIdx.x == 0 && (it) < 8) trace[(slot) * 8 + (it)] = gtimer(); \
  } while (0)

template <int D>
__global__ void __launch_bounds__(TcLayout<D>::NTHREADS, 1)
maxsim_tc_kernel(const MaxSimParams p) {
  __shared__ uint64_t trace[8 * 8];
  __shared__ uint64_t strace[6 * 16];  // per-stage: producer, MMA full, MMA tempty, epilogue
  using L = TcLayout<D>;
  using namespace espn_ptx;
  // swizzled operand atoms need 1024-byte aligned stage bases: align manually
  extern __shared__ __align__(1024) uint8_t tc_smem_raw[];
  uint8_t* smem = tc_smem_raw + ((1024u - (smem_u32(tc_smem_raw) & 1023u)) & 1023u);
  uint8_t* sB = smem + L::OFF_B;
  uint8_t* sA = smem + L::OFF_A;
  float* pm = reinterpret_cast<float*>(smem + L::OFF_PM);
  typename L::Unit* units = reinterpret_cast<typename L::Unit*>(smem + L::OFF_UNIT);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* full_bar = bars;                       // [NS]  producer (expect_tx) -> MMA
  uint64_t* empty_bar = bars + L::NS;              // [NS]  MMA commit -> producer
  uint64_t* tfull_bar = bars + 2 * L::NS;          // [NBUF] MMA commit -> epilogue
  uint64_t* tempty_bar = tfull_bar + L::NBUF;      // [NBUF] epilogue -> MMA
  uint64_t* ufull_bar = tempty_bar + L::NBUF;      // [NU] loader -> producer, MMA, epilogue
  uint64_t* uempty_bar = ufull_bar + L::NU;        // [NU] combine -> loader
  uint64_t* edone_bar = uempty_bar + L::NU;        // [NU] epilogue (all lanes) -> combine
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  if (p.prof && tid == 0) atomicMin(&p.prof[2], (unsigned long long)gtimer());

  // ---- one-time setup: zero operand tiles (stale NaN bit patterns would leak
  // into other quarters through the zero rows of A), barriers, TMEM ----------
  {
    uint4* z = reinterpret_cast<uint4*>(smem);
    const int n16 = (L::OFF_PM) / 16;
    for (int i = tid; i < n16; i += L::NTHREADS) z[i] = make_uint4(0, 0, 0, 0);
  }
  {
    int* pmk = reinterpret_cast<int*>(smem + L::OFF_PM);
    for (int i = tid; i < L::PM_FLOATS; i += L::NTHREADS) pmk[i] = ord_key(-INFINITY);
  }
  fence_proxy_async_smem();
  if (tid == 0) {
    for (int i = 0; i < L::NS; ++i) {
      mbar_init(&full_bar[i], L::NPROD);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < L::NBUF; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], L::NEPI);
    }
    for (int i = 0; i < L::NU; ++i) {
      mbar_init(&ufull_bar[i], 1);
      mbar_init(&uempty_bar[i], 1);
      mbar_init(&edone_bar[i], 32 * L::NEPI);
    }
    mbar_fence_init();
  }
  if (warp == L::MMA_WARP) tmem_alloc<L::TMEM_COLS>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const uint64_t t_start = gtimer();
  // let the dependent top-k grid launch now: its dedup prologue reads only
  // candidate ids and then waits (griddepcontrol.wait) for this grid to finish
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  const uint32_t n_units = *p.n_units;  // planned on the device (plan_kernel)

  if (warp == L::LOADER_WARP) {
    // ============================ UNIT LOADER ===================================
    for (uint32_t it = 0;; ++it) {
      const uint32_t ug = blockIdx.x + it * gridDim.x;
      if (ug >= n_units) break;
      const uint32_t us = it % L::NU;
      typename L::Unit& U = units[us];
      // Unit table entry (host-planned): query b, doc count, first candidate.
      if (lane == 0) ESPN_TRACE(0, it);
      const uint4 ue = __ldg(&p.unit_tab[ug]);
      const uint32_t b = ue.x, nd = ue.y;
      const uint64_t cfirst = (uint64_t)ue.z | ((uint64_t)ue.w << 32);
      // Issue every independent global load of the unit up front: candidate
      // ids (<= 2 per lane), then the query tile, then the dependent row_ptr.
      uint32_t idk[L::UNITMAX / 32];
#pragma unroll
      for (int r = 0; r < L::UNITMAX / 32; ++r) {
        const uint32_t k = r * 32 + lane;
        idk[r] = k < nd ? __ldg(&p.cand_ids[cfirst + k]) : 0u;
      }
      mbar_wait(&uempty_bar[us], ((it / L::NU) & 1) ^ 1);
      if (lane == 0) ESPN_TRACE(1, it);
      for (int i = lane; i < L::MAXW; i += 32) U.bitmap[i] = 0;
      for (int i = lane; i < L::MAX_STAGES; i += 32) {
        U.kbeg[i] = 0xFFFFFFFFu;
        U.kend[i] = 0;
      }
      __syncwarp();
      // doc info + slot prefix sum (warp scan) + group plan
      uint32_t carry = 0;
#pragma unroll
      for (int r = 0; r < L::UNITMAX / 32; ++r) {
        const uint32_t k = r * 32 + lane;
        uint32_t t = 0;
        uint64_t r0 = 0;
        uint64_t srcaddr = 0;
        if (k < nd) {
          const uint64_t loc = shard_local(idk[r], p.shard_count, p.shard_index, p.n_docs);
          if (loc != ~0ull) {
            r0 = __ldg(&p.row_ptr[loc]);
            t = (uint32_t)(__ldg(&p.row_ptr[loc + 1]) - r0);
            srcaddr = p.cand_src ? __ldg(&p.cand_src[cfirst + k])  // tiered: staged / resident address
                                 : (uint64_t)(p.rows + r0 * D);
            if (srcaddr == 0) t = 0;  // not staged (staging overflow, reported by stage_kernel)
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
          U.src[k] = srcaddr;
          U.t[k] = t;
          U.slot[k] = start;
          if (t > 0 && start + pad <= (uint32_t)L::MAX_SLOTS) {
            atomicOr(&U.bitmap[start >> 8], 1u << ((start >> 3) & 31));
            const uint32_t g0 = start >> 3, ng = pad >> 3;
            for (uint32_t g = 0; g + 1 < ng; ++g) U.gvalid[g0 + g] = 8;
            U.gvalid[g0 + ng - 1] = (uint8_t)(t - 8 * (ng - 1));
            // stages holding this doc's rows (a doc spans at most a few)
            for (uint32_t st = start / L::STAGE_SLOTS; st <= (start + t - 1) / L::STAGE_SLOTS; ++st) {
              atomicMin(&U.kbeg[st], k);
              atomicMax(&U.kend[st], k + 1);
            }
          }
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (carry > (uint32_t)L::MAX_SLOTS) {
        if (lane == 0) atomicOr(p.err, ERR_UNIT_TOO_LARGE);
        carry = 0;  // skip the unit's MMA work; the call fails on the host
      }
      // Query tokens -> A slot `us` (rows 96+128*us .. +32), converted to the
      // table dtype; rows >= nq stay zero.  Item e = (row i, 8-value chunk c);
      // batches of 4 items per lane keep all their loads in flight together.
      {
        const float* q = p.q32 + (size_t)b * p.nq * D;
        const int abase = 96 + 128 * (int)us;
        constexpr int ITEMS = 32 * L::CH / 32;  // per lane
        constexpr int BATCH = ITEMS < 4 ? ITEMS : 4;
#pragma unroll
        for (int i0 = 0; i0 < ITEMS; i0 += BATCH) {
          float4 x[BATCH][2];
#pragma unroll
          for (int u = 0; u < BATCH; ++u) {
            const int e = (i0 + u) * 32 + lane;
            const int i = e / L::CH, c = e % L::CH;
            if ((uint32_t)i < p.nq) {
              const float4* src = reinterpret_cast<const float4*>(q + i * D + c * 8);
              x[u][0] = __ldg(src);
              x[u][1] = __ldg(src + 1);
            } else {
              x[u][0] = x[u][1] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
          bool bad = false;
#pragma unroll
          for (int u = 0; u < BATCH; ++u) {
            const int e = (i0 + u) * 32 + lane;
            const int i = e / L::CH, c = e % L::CH;
            const float f[8] = {x[u][0].x, x[u][0].y, x[u][0].z, x[u][0].w,
                                x[u][1].x, x[u][1].y, x[u][1].z, x[u][1].w};
            uint32_t w4[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const uint16_t h0 = f32_to_code(f[2 * h], p.bf16), h1 = f32_to_code(f[2 * h + 1], p.bf16);
              bad |= !isfinite(code_to_f32(h0, p.bf16)) || !isfinite(code_to_f32(h1, p.bf16));
              w4[h] = (uint32_t)h0 | ((uint32_t)h1 << 16);
            }
            const int r = abase + i;
            *reinterpret_cast<uint4*>(sA + (r >> 3) * L::A_SBO + c * L::A_LBO + (r & 7) * 16) =
                make_uint4(w4[0], w4[1], w4[2], w4[3]);
          }
          if (bad) atomicOr(p.err, ERR_NONFINITE_QUERY);
        }
      }
      __syncwarp();
      if (lane == 0) {
        uint32_t acc = 0;
        for (int i = 0; i < L::MAXW; ++i) {
          U.wprefix[i] = acc;
          acc += __popc(U.bitmap[i]);
        }
        U.b = b;
        U.cfirst = cfirst;
        U.nd = nd;
        U.S = carry;
      }
      fence_proxy_async_smem();  // A tile is read by the tensor core (async proxy)
      __syncwarp();
      if (lane == 0) { ESPN_TRACE(2, it); mbar_arrive(&ufull_bar[us]); }
    }
  } else if (warp >= L::PROD_WARP0 && warp < L::PROD_WARP0 + L::NPROD) {
    // ====================== BULK-COPY PRODUCERS (NPROD warps) ======================
    // Producer pw takes docs kbeg + pw*32 + lane, stride 32*NPROD; each warp
    // arrives on the stage's full barrier with its own expect_tx byte count.
    const uint32_t pw = warp - L::PROD_WARP0;
    const uint64_t policy = l2_policy_evict_first();
    uint32_t gs = 0;  // global stage counter
    for (uint32_t it = 0;; ++it) {
      const uint32_t ug = blockIdx.x + it * gridDim.x;
      if (ug >= n_units) break;
      const uint32_t us = it % L::NU;
      const typename L::Unit& U = units[us];
      mbar_wait(&ufull_bar[us], (it / L::NU) & 1);
      if (lane == 0 && pw == 0) ESPN_TRACE(3, it);
      const uint32_t S = U.S;
      const uint32_t n_st = (S + L::STAGE_SLOTS - 1) / L::STAGE_SLOTS;
      for (uint32_t st = 0; st < n_st; ++st, ++gs) {
        const uint32_t s = gs % L::NS;
        const uint32_t x0 = st * L::STAGE_SLOTS, x1 = x0 + L::STAGE_SLOTS;
        // docs [kbeg, kend) (loader-planned) contribute rows [max(x0,slot), min(x1,slot+t))
        const uint32_t kcur = U.kbeg[st], kend = U.kend[st];
        uint32_t bytes = 0;
        for (uint32_t k = kcur + pw * 32 + lane; k < kend; k += 32 * L::NPROD) {
          const uint32_t a = max(U.slot[k], x0), e = min(U.slot[k] + U.t[k], x1);
          bytes += e > a ? (e - a) * (uint32_t)L::ROWB : 0u;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
        mbar_wait(&empty_bar[s], ((gs / L::NS) & 1) ^ 1);
        if (lane == 0 && pw == 0) ESPN_STRACE(0, gs);
        if (p.dbg & 4u) bytes = 0;
        if (lane == 0) mbar_arrive_expect_tx(&full_bar[s], bytes);
        __syncwarp();
        if (p.dbg & 4u) continue;
        const uint32_t sbase = smem_u32(sB + s * L::STAGE_BYTES);
        for (uint32_t k = kcur + pw * 32 + lane; k < kend; k += 32 * L::NPROD) {
          const uint32_t sk = U.slot[k], t = U.t[k];
          const uint32_t a = max(sk, x0), e = min(sk + t, x1);
          if (e <= a) continue;
          const uint32_t ja = a - sk, n = e - a;
          const uint8_t* src = reinterpret_cast<const uint8_t*>(U.src[k]);
#pragma unroll
          for (int pn = 0; pn < L::NP; ++pn)
            bulk_g2s(sbase + pn * L::PANEL_BYTES + (a - x0) * L::PW,
                     src + ((size_t)pn * t + ja) * L::PW, n * L::PW, &full_bar[s], policy);
        }
      }
    }
  } else if (warp == L::MMA_WARP) {
    // ============================ MMA ISSUER ==================================
    if (lane == 0) {
      uint32_t gs = 0;
      const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
      for (uint32_t it = 0;; ++it) {
        const uint32_t ug = blockIdx.x + it * gridDim.x;
        if (ug >= n_units) break;
        const uint32_t us = it % L::NU;
        mbar_wait(&ufull_bar[us], (it / L::NU) & 1);
        const uint32_t S = units[us].S;
        const uint32_t n_st = (S + L::STAGE_SLOTS - 1) / L::STAGE_SLOTS;
        for (uint32_t st = 0; st < n_st; ++st, ++gs) {
          const uint32_t s = gs % L::NS, buf = gs % L::NBUF;
          mbar_wait(&full_bar[s], (gs / L::NS) & 1);
          ESPN_STRACE(1, gs);
          mbar_wait(&tempty_bar[buf], ((gs / L::NBUF) & 1) ^ 1);
          ESPN_STRACE(2, gs);
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
            if ((p.dbg & 2u) || ((p.dbg & 64u) && w > 0)) break;
            const uint32_t idesc = umma_idesc_f16(128, n_mma, p.bf16);
            const uint32_t a_row0 = 96 + 128 * us - 32 * w;
            const uint32_t a_addr = a_base + (a_row0 >> 3) * L::A_SBO;
            const uint32_t b_addr = b_base + s * L::STAGE_BYTES + w * L::NQC * L::PW;
#pragma unroll
            for (int ks = 0; ks < L::KSTEPS; ++ks) {
              const uint32_t kb = ks * 32;  // K offset in bytes
              const uint64_t ad = umma_desc_kmajor(a_addr + ks * 2 * L::A_LBO, L::A_LBO, L::A_SBO);
              const uint64_t bd = umma_desc_sw(b_addr + (kb / L::PW) * L::PANEL_BYTES + (kb % L::PW),
                                               8 * L::PW, L::SWZ);
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
  } else if (warp < L::NEPI) {
    // ==================== EPILOGUE (warps 0..NEPI-1) ===========================
    // warp = h*4 + w: TMEM lane quarter w (== query-token quarter), column half h.
    // pm holds order-preserving int keys of the per-doc partial maxima; the two
    // halves of a quarter may both flush a doc straddling the split, so
    // flushes are shared-memory atomicMax (a few per stage).
    const int w = warp & 3, h = warp >> 2;
    uint32_t gs = 0;
    for (uint32_t it = 0;; ++it) {
      const uint32_t ug = blockIdx.x + it * gridDim.x;
      if (ug >= n_units) break;
      const uint32_t us = it % L::NU;
      const typename L::Unit& U = units[us];
      mbar_wait(&ufull_bar[us], (it / L::NU) & 1);
      if (tid == 0) ESPN_TRACE(4, it);
      const uint32_t S = U.S;
      int* my_pm = reinterpret_cast<int*>(pm) + (us * 32 + lane) * L::PM_STRIDE;
      const uint32_t n_st = (S + L::STAGE_SLOTS - 1) / L::STAGE_SLOTS;
      for (uint32_t st = 0; st < n_st; ++st, ++gs) {
        const uint32_t buf = gs % L::NBUF;
        mbar_wait(&tfull_bar[buf], (gs / L::NBUF) & 1);
        if (tid == 0) ESPN_STRACE(3, gs);
        tc_fence_after();
        const uint32_t xw = st * L::STAGE_SLOTS + w * L::NQC + h * L::HALF;
        const int remv = (p.dbg & 1u) ? 0 : (int)S - (int)xw;
        if (remv > 0) {
          // All TMEM loads of this warp's columns first, then the TMEM buffer
          // is released and the group maxima are computed with full ILP; only
          // the short doc-boundary scan over NGH groups is sequential.
          const uint32_t nv = remv < L::HALF ? (uint32_t)remv : (uint32_t)L::HALF;
          const uint32_t taddr0 = tmem_base + ((uint32_t)(w * 32) << 16) + buf * L::NQC + h * L::HALF;
          float v[L::NLD][L::LW];
#pragma unroll
          for (int c = 0; c < L::NLD; ++c) {
            if (p.dbg & 16u) {
#pragma unroll
              for (int j = 0; j < L::LW; ++j) v[c][j] = (float)j;
            } else if (c == 0 || (uint32_t)(L::LW * c) < nv) {
              tmem_ld_32x32b<L::LW>(taddr0 + L::LW * c, v[c]);
            }
          }
          const uint32_t G0 = xw >> 3;  // multiple of NGH
          const uint32_t bw = U.bitmap[G0 >> 5];
          const uint32_t sbits = (bw >> (G0 & 31)) & ((1u << L::NGH) - 1u);
          int doc = (int)(U.wprefix[G0 >> 5] + __popc(bw & ((2u << (G0 & 31)) - 1u))) - 1;
          uint32_t gvw[(L::NGH + 3) / 4];
          if constexpr (L::NGH % 4 == 0) {
#pragma unroll
            for (int c = 0; c < L::NGH / 4; ++c) gvw[c] = *reinterpret_cast<const uint32_t*>(&U.gvalid[G0 + 4 * c]);
          } else {  // G0 is only NGH-aligned: byte loads
            gvw[0] = 0;
#pragma unroll
            for (int q = 0; q < L::NGH; ++q) gvw[0] |= (uint32_t)U.gvalid[G0 + q] << (8 * q);
          }
          tmem_ld_wait();
          if (tid == 0) ESPN_STRACE(4, gs);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[buf]);
          if (p.dbg & 32u) continue;
          // group maxima over the valid (non-pad) columns, branch-free
          float gm[L::NGH];
#pragma unroll
          for (int q = 0; q < L::NGH; ++q) {
            const float* x = &v[(8 * q) / L::LW][(8 * q) % L::LW];
            const uint32_t nval = (gvw[q / 4] >> (8 * (q % 4))) & 0xFFu;
            const float x0 = x[0];
            const float x1 = sel_gt(nval, 1, x[1], x0), x2 = sel_gt(nval, 2, x[2], x0);
            const float x3 = sel_gt(nval, 3, x[3], x0), x4 = sel_gt(nval, 4, x[4], x0);
            const float x5 = sel_gt(nval, 5, x[5], x0), x6 = sel_gt(nval, 6, x[6], x0);
            const float x7 = sel_gt(nval, 7, x[7], x0);
            gm[q] = fmaxf(fmax3(x0, x1, x2), fmax3(fmax3(x3, x4, x5), x6, x7));
          }
          float m = -INFINITY;
#pragma unroll
          for (int q = 0; q < L::NGH; ++q) {
            if ((uint32_t)(8 * q) < nv) {
              if (q > 0 && ((sbits >> q) & 1u)) {
                atomicMax(&my_pm[doc], ord_key(m));
                ++doc;
                m = gm[q];
              } else {
                m = fmaxf(m, gm[q]);
              }
            }
          }
          atomicMax(&my_pm[doc], ord_key(m));
          if (tid == 0) ESPN_STRACE(5, gs);
        } else {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[buf]);
        }
      }
      // all lanes' flushes of this unit are done: hand the slot to the combiner
      if (tid == 0) ESPN_TRACE(5, it);
      mbar_arrive(&edone_bar[us]);
    }
  } else if (warp == L::COMBINE_WARP) {
    // ============================ COMBINE ========================================
    // bow(doc) = sum_i pm[us][i][doc] (max over the doc's tokens, reduced by the
    // epilogue's atomicMax), i ascending (the oracle's summation order); then
    // the slot's keys are reset and the unit slot is released to the loader.
    // Runs concurrently with the epilogue of the next units.
    for (uint32_t it = 0;; ++it) {
      const uint32_t ug = blockIdx.x + it * gridDim.x;
      if (ug >= n_units) break;
      const uint32_t us = it % L::NU;
      const typename L::Unit& U = units[us];
      mbar_wait(&edone_bar[us], (it / L::NU) & 1);
      const uint32_t nd = U.nd;
      const uint64_t j0 = U.cfirst;
      int* pmu = reinterpret_cast<int*>(pm) + us * 32 * L::PM_STRIDE;
      for (uint32_t k = lane; k < nd; k += 32) {
        float s = 0.0f;
        for (uint32_t i = 0; i < p.nq; ++i) s = __fadd_rn(s, key_ord(pmu[i * L::PM_STRIDE + k]));
        p.bow_out[j0 + k] = s;
#pragma unroll 8
        for (uint32_t i = 0; i < 32; ++i) pmu[i * L::PM_STRIDE + k] = ord_key(-INFINITY);
      }
      __syncwarp();
      if (lane == 0) { ESPN_TRACE(6, it); mbar_arrive(&uempty_bar[us]); }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == L::MMA_WARP) {
    tc_fence_after();
    tmem_dealloc<L::TMEM_COLS>(tmem_base);
  }
  if (p.prof && tid == 0) {
    __threadfence();
    if (atomicAdd(&p.prof[3], 1ull) == gridDim.x - 1) {  // last CTA out
      const unsigned long long t0 = atomicAdd(&p.prof[2], 0ull);
      atomicAdd(&p.prof[0], (unsigned long long)gtimer() - t0);
      atomicAdd(&p.prof[1], 1ull);
      p.prof[2] = ~0ull;
      p.prof[3] = 0;
    }
  }
  if ((p.dbg & 8u) && blockIdx.x == 0 && tid == 0) {
    const char* nm[7] = {"ld.start", "ld.slot", "ld.ready", "pr.start", "ep.start", "ep.mmadone", "ep.done"};
    printf("CTA0 units=%u end=%.2fus\n", (n_units + gridDim.x - 1) / gridDim.x, (gtimer() - t_start) / 1e3);
    for (int e = 0; e < 7; ++e) {
      printf("%-11s", nm[e]);
      for (int u = 0; u < 8 && blockIdx.x + u * gridDim.x < n_units; ++u)
        printf(" %8.2f", ((int64_t)(trace[e * 8 + u] - t_start)) / 1e3);
      printf("\n");
    }
    const char* sn[6] = {"P.empty", "M.full", "M.tempty", "E.tfull", "E.ldone", "E.proc"};
    for (int e = 0; e < 6; ++e) {
      printf("%-9s", sn[e]);
      for (int g = 0; g < 16; ++g) printf(" %6.2f", ((int64_t)(strace[e * 16 + g] - t_start)) / 1e3);
      printf("\n");
    }
  }
}

}  // namespace espn_k
