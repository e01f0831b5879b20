// espn_gpu.cu -- C-ABI implementation (include/espn_gpu.h): table / workspace
// lifetime, batch orchestration (H2D -> K2 MaxSim -> K3 top-k -> D2H) and the
// standalone gather / merge / synth entry points.  Pure CUDA runtime; no torch.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is loaded at run time (nccl_api below)

#include <algorithm>
#include <type_traits>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/espn_gpu.h"
#include "common.cuh"
#include "kernels_misc.cuh"
#include "maxsim_tc.cuh"
#include "shard.cuh"
#include "small.cuh"

using namespace espn_k;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define ESPN_CUDA_TRY(expr)                                                                  \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fail(ESPN_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));          \
  } while (0)

int err_bits_to_status(uint32_t bits) {
  if (!bits) return ESPN_OK;
  std::string m = "device-side validation failed:";
  if (bits & ERR_UNKNOWN_DOC) m += " candidate doc id not in the table (store lacks a candidate);";
  if (bits & ERR_NONFINITE_QUERY) m += " query token not finite in the table dtype;";
  if (bits & ERR_NONFINITE_CLS) m += " non-finite cls_score;";
  if (bits & ERR_DUPLICATE) m += " duplicate candidate doc id;";
  if (bits & ERR_NONFINITE_SCORE) m += " non-finite aggregate score;";
  if (bits & ERR_UNIT_TOO_LARGE) m += " internal: work unit slot budget exceeded;";
  if (bits & ERR_BAD_OFFSETS) m += " cand_offsets must start at 0 and be non-decreasing;";
  if (bits & ERR_CAPACITY) m += " batch exceeds workspace capacity;";
  if (bits & ERR_STAGING) m += " host-tier rows of the batch exceed the staging buffer (raise staging_bytes);";
  if (bits & ERR_SERVER) m += " the persistent re-rank server did not complete the batch (stopped or stalled);";
  if (bits & ERR_NOT_PREFETCHED)
    m += " a needed doc of the disk tier was not staged by espn_gpu_prefetch_rows before this PREFETCHED batch;";
  g_last_error = m;
  if (bits & ERR_UNKNOWN_DOC) return ESPN_E_DATA_INTEGRITY;
  if (bits & ERR_UNIT_TOO_LARGE) return ESPN_E_INVALID_STATE;
  if (bits & ERR_STAGING) return ESPN_E_INVALID_CONFIG;
  if (bits & ERR_SERVER) return ESPN_E_INVALID_STATE;
  if (bits & ERR_NOT_PREFETCHED) return ESPN_E_INVALID_STATE;
  return ESPN_E_INVALID_INPUT;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    // a non-sticky error left pending by an earlier, unrelated runtime call of
    // this thread would otherwise surface at this call's first launch check
    (void)cudaGetLastError();
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int check_device(int dev, int* num_sms, bool* tc_ok) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    return fail(ESPN_E_CUDA, "no CUDA device available (the re-rank path has no CPU fallback)");
  if (dev < 0 || dev >= n) return fail(ESPN_E_INVALID_INPUT, "device ordinal out of range");
  cudaDeviceProp prop;
  ESPN_CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
  *num_sms = prop.multiProcessorCount;
  *tc_ok = prop.major == 10 && prop.minor == 0;
  return ESPN_OK;
}

constexpr int kMinUnitDocs = 8;
constexpr int kExclusiveUnitDocs = 64;  // longest unit of a non-served tcgen05 launch
// internal re-rank flag: device cand_offsets are a query slice of a larger
// batch (cand_offsets[0] may be nonzero; REPLICA placement of the sharded call)
constexpr uint32_t kFlagBaseOffsets = 0x80000000u;  // shortest work unit (small batches, see espn_gpu_rerank)

template <int D, bool S>
constexpr int tc_unit_docs(uint32_t max_t) {
  using L = TcLayout<D, S>;
  const uint32_t pad = (max_t + 7u) & ~7u;
  const uint32_t u = pad ? (uint32_t)L::MAX_SLOTS / pad : 0;
  return (int)std::min<uint32_t>(u, (uint32_t)L::UNITMAX);
}

// longest doc one work unit holds (UNITMAX x 64 slots; the split-query layout
// of d = 32 has shorter units than the rounded-query one)
int tc_max_tokens_rt(uint32_t d, bool split) {
  switch (d * 2 + (split ? 1 : 0)) {
    case 32: return TcLayout<16, false>::MAX_SLOTS;
    case 33: return TcLayout<16, true>::MAX_SLOTS;
    case 64: return TcLayout<32, false>::MAX_SLOTS;
    case 65: return TcLayout<32, true>::MAX_SLOTS;
    case 128: return TcLayout<64, false>::MAX_SLOTS;
    case 129: return TcLayout<64, true>::MAX_SLOTS;
    case 256: return TcLayout<128, false>::MAX_SLOTS;
    case 257: return TcLayout<128, true>::MAX_SLOTS;
    default: return 0;
  }
}

int tc_unit_docs_rt(uint32_t d, uint32_t max_t, bool split) {
  switch (d * 2 + (split ? 1 : 0)) {
    case 32: return tc_unit_docs<16, false>(max_t);
    case 33: return tc_unit_docs<16, true>(max_t);
    case 64: return tc_unit_docs<32, false>(max_t);
    case 65: return tc_unit_docs<32, true>(max_t);
    case 128: return tc_unit_docs<64, false>(max_t);
    case 129: return tc_unit_docs<64, true>(max_t);
    case 256: return tc_unit_docs<128, false>(max_t);
    case 257: return tc_unit_docs<128, true>(max_t);
    default: return 0;
  }
}

// cudaFuncSetAttribute is per DEVICE: one process may drive several GPUs
// through the C-ABI, so each (kernel, device) pair is configured once.
template <typename K>
cudaError_t smem_attr_once(K* kern, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

template <int D, bool SPLIT>
cudaError_t launch_tc(const MaxSimParams& p, int num_sms, cudaStream_t s, bool pdl) {
  using L = TcLayout<D, SPLIT>;
  static std::atomic<uint64_t> attr_set{0};
  {
    cudaError_t e = smem_attr_once(maxsim_tc_kernel<D, SPLIT>, L::SMEM_BYTES, attr_set);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(maxsim_tc_kernel<D, SPLIT>, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
  }
  // persistent: one CTA per SM; the unit count is read on the device.  As a
  // programmatic dependent of plan_kernel (pdl) its prologue overlaps the plan.
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(num_sms);
  lc.blockDim = dim3(L::NTHREADS);
  lc.dynamicSmemBytes = L::SMEM_BYTES;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&lc, maxsim_tc_kernel<D, SPLIT>, p);
}

cudaError_t launch_tc_rt(uint32_t d, bool split, const MaxSimParams& p, int num_sms, cudaStream_t s, bool pdl) {
  switch (d * 2 + (split ? 1 : 0)) {
    case 32: return launch_tc<16, false>(p, num_sms, s, pdl);
    case 33: return launch_tc<16, true>(p, num_sms, s, pdl);
    case 64: return launch_tc<32, false>(p, num_sms, s, pdl);
    case 65: return launch_tc<32, true>(p, num_sms, s, pdl);
    case 128: return launch_tc<64, false>(p, num_sms, s, pdl);
    case 129: return launch_tc<64, true>(p, num_sms, s, pdl);
    case 256: return launch_tc<128, false>(p, num_sms, s, pdl);
    case 257: return launch_tc<128, true>(p, num_sms, s, pdl);
    default: return cudaErrorInvalidValue;
  }
}

// Query precision of the tcgen05 path (ESPN_RERANK_QUERY_* in espn_gpu.h).
bool tc_query_split(uint32_t d, uint32_t dtype, uint32_t flags) {
  if (flags & ESPN_RERANK_QUERY_ROUNDED) return false;
  if (flags & ESPN_RERANK_QUERY_SPLIT) return true;
  (void)d;
  // bf16 needs the split (a bf16-rounded query is off by ~3e-3 relative); an
  // f16-rounded one stays within ~5e-4, and the second MMA costs ~17% of the
  // C2 step (46.4 vs 39.8 us, profiles/query_split_r2_{split,rounded}.json), so f16 rounds
  return dtype == ESPN_DTYPE_BF16;
}

template <int D>
cudaError_t launch_simt(const MaxSimParams& p, int num_sms, cudaStream_t s) {
  maxsim_simt_kernel<D><<<num_sms * 8, 256, 0, s>>>(p);  // 64 warps per SM, grid-stride
  return cudaGetLastError();
}

cudaError_t launch_simt_rt(uint32_t d, const MaxSimParams& p, int num_sms, cudaStream_t s) {
  switch (d) {
    case 8: return launch_simt<8>(p, num_sms, s);
    case 16: return launch_simt<16>(p, num_sms, s);
    case 32: return launch_simt<32>(p, num_sms, s);
    case 48: return launch_simt<48>(p, num_sms, s);
    case 64: return launch_simt<64>(p, num_sms, s);
    case 96: return launch_simt<96>(p, num_sms, s);
    case 128: return launch_simt<128>(p, num_sms, s);
    default: return cudaErrorInvalidValue;
  }
}

bool simt_supported(uint32_t d) {
  return d == 8 || d == 16 || d == 32 || d == 48 || d == 64 || d == 96 || d == 128;
}
bool tc_supported(uint32_t d) { return d == 16 || d == 32 || d == 64 || d == 128; }

size_t topk_smem_bytes() {
  return (size_t)kTopkSort * 8 + (size_t)kMaxK * 8 + (size_t)kTopkHash * 4;
}

cudaError_t ensure_topk_attr() {
  static std::atomic<uint64_t> d1{0}, d2{0}, d3{0}, d4{0}, d5{0};
  cudaError_t e = smem_attr_once(topk_kernel, (int)topk_smem_bytes(), d1);
  if (e == cudaSuccess) e = smem_attr_once(merge_packed_kernel, (int)topk_smem_bytes(), d5);
  if (e == cudaSuccess) e = smem_attr_once(merge_topk_kernel, (int)topk_smem_bytes(), d2);
  if (e == cudaSuccess) e = smem_attr_once(topk_cta_kernel<16>, 8192 * 8 + 8 * 32 * 8, d3);
  if (e == cudaSuccess) e = smem_attr_once(topk_cta_kernel<32>, 8192 * 8 + 8 * 32 * 8, d4);
  return e;
}


// ---- NCCL, loaded at run time ------------------------------------------------
// The C-ABI does not link NCCL: torch (or the integrator) may already have a
// libnccl.so.2 loaded, and that copy must be the one whose communicators we
// are handed, so dlopen(RTLD_NOLOAD) first, then the default search path.
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommCuDevice)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.why = std::string("NCCL not loadable (libnccl.so.2): ") + (e ? e : "?");
      return a;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) all = false;
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommInitAll, "ncclCommInitAll");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.CommCount, "ncclCommCount");
    sym(a.CommUserRank, "ncclCommUserRank");
    sym(a.CommCuDevice, "ncclCommCuDevice");
    sym(a.AllGather, "ncclAllGather");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    a.ok = all;
    if (!all) a.why = "libnccl.so.2 lacks an expected symbol";
    return a;
  }();
  return api;
}
#define ESPN_NCCL_TRY(expr)                                                                   \
  do {                                                                                        \
    const ncclResult_t r_ = (expr);                                                           \
    if (r_ != ncclSuccess)                                                                    \
      return fail(ESPN_E_CUDA, std::string(#expr) + ": " + nccl_api().GetErrorString(r_));    \
  } while (0)


bool layout_tiled(uint32_t d) { return d == 16 || d == 32 || d == 64 || d == 128; }

// plain CSR rows (device) -> HBM tile layout (device), both n_tokens * d codes
cudaError_t tile_rows(uint32_t d, const uint16_t* plain, const uint64_t* row_ptr, uint64_t n_docs,
                      uint16_t* tiled, int num_sms) {
  const int blocks = num_sms * 8;
  switch (d) {
    case 16: tile_rows_kernel<16><<<blocks, 256>>>(plain, row_ptr, n_docs, tiled); break;
    case 32: tile_rows_kernel<32><<<blocks, 256>>>(plain, row_ptr, n_docs, tiled); break;
    case 64: tile_rows_kernel<64><<<blocks, 256>>>(plain, row_ptr, n_docs, tiled); break;
    case 128: tile_rows_kernel<128><<<blocks, 256>>>(plain, row_ptr, n_docs, tiled); break;
    default: return cudaSuccess;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return cudaDeviceSynchronize();
}

}  // namespace

struct espn_gpu_table {
  int device = 0;
  int num_sms = 0;
  bool tc_ok = false;
  uint64_t n_docs = 0, n_tokens = 0;
  uint32_t d = 0, dtype = 0, d_cls = 0, value_width = 2, alignment = 1;
  uint32_t max_t = 0, min_t = 0;
  uint32_t shard_count = 1, shard_index = 0;
  bool owned = false;       // row_ptr owned
  bool owned_rows = false;  // rows owned
  uint64_t* row_ptr = nullptr;
  uint16_t* rows = nullptr;
  // tiered store (desc->resident): HBM compact rows in `rows`, pinned host tier
  bool tiered = false;
  uint64_t* doc_loc = nullptr;   // device: per-doc row address | tier bit
  uint8_t* host_rows = nullptr;  // pinned, mapped
  uint64_t hbm_row_bytes = 0, host_row_bytes = 0, resident_docs = 0;
  // ESPN_TABLE_STREAMED: filled in doc order by espn_gpu_table_load_rows
  bool streamed = false;
  bool disk_tier = false;  // ESPN_TABLE_DISK_TIER: non-resident docs have no in-memory copy
  uint64_t loaded_docs = 0;
  std::vector<uint64_t> h_row_ptr;  // host copies used while filling
  std::vector<uint64_t> h_loc;      // tiered: per-doc address | tier bit
  uint8_t* host_dev = nullptr;      // device alias of host_rows
  // persistent re-rank server (espn_gpu_server_start)
  ServerQueue* server = nullptr;      // device queue (NULL: no server)
  cudaStream_t server_stream = nullptr;
  uint32_t* server_alive_h = nullptr;  // mapped pinned: 1 while the kernel runs
  bool server_split = false;
  uint32_t server_dbg = 0;
  uint64_t server_idle_ns = 0;
  uint64_t server_launches = 0;
};

struct espn_gpu_workspace {
  espn_gpu_table* table = nullptr;
  uint32_t max_queries = 0, max_candidates = 0, max_nq = 0;
  uint32_t* unit_off = nullptr;
  uint32_t* needed = nullptr;
  uint4* unit_tab = nullptr;    // tcgen05 work units {b, n_docs, first candidate}
  uint64_t max_units = 0;
  uint32_t* n_units = nullptr;    // planned unit count (device)
  uint32_t max_list = 0;          // longest candidate list the top-k hash is sized for
  // fused top-k (tcgen05 path, final_k <= kFusedMaxK)
  unsigned long long* unit_top = nullptr;  // max_units x kFusedMaxK keys
  uint32_t* dedup = nullptr;               // 2 x B x hash_slots (0xFF.. = empty), by batch parity
  uint32_t* ff_seen = nullptr;             // 2 x B
  uint32_t* fused_state = nullptr;         // {epoch, rows used by parity 0, parity 1}
  uint32_t hash_slots = 0;
  uint32_t* small_arrive = nullptr;        // single-launch small batches: per-query arrival counters,
  unsigned long long* small_top = nullptr; // per-CTA best-k lists (kSmallMaxCtas x kFusedMaxK),
  uint32_t* small_hash = nullptr;          // per-query duplicate hashes (kSmallMaxB x kSmallHashSlots)
  uint32_t* small_ff = nullptr;            // and their empty-code flags
  unsigned long long* kprof = nullptr;  // device-timed MaxSim {sum_ns, launches, start, done}
  // tiered tables: two staging slots (one scoring, one being prefetched)
  struct Stage {
    uint8_t* buf = nullptr;
    uint64_t* cand_src = nullptr;
    uint8_t* cand_status = nullptr;        // per needed candidate (StageParams::cand_status)
    unsigned long long* cursor = nullptr;
    unsigned long long* qstats = nullptr;  // B x 6
    uint64_t* off = nullptr;               // device copy of the batch offsets (prefetch, host offsets)
    uint32_t* need = nullptr;
    uint64_t* off_h = nullptr;             // pinned staging of host offsets
    uint32_t* need_h = nullptr;
    cudaEvent_t done = nullptr;            // staging finished
    cudaEvent_t free_ev = nullptr;         // last MaxSim reading this slot finished
    bool used = false;
    uint32_t hint_epoch = 0;               // != 0: filled by espn_gpu_prefetch_hints (doc-keyed)
    uint32_t* hint_ids = nullptr;          // device copy of host hint ids (lazy, max_candidates)
    uint32_t* hint_ids_h = nullptr;        // its pinned staging
    uint8_t* ext_buf = nullptr;            // espn_gpu_prefetch_rows: the caller's rows on the device (lazy)
    uint64_t ext_cap = 0;
    uint64_t* ext_off = nullptr;           // per hint: byte offset of its rows in ext_buf (lazy)
    uint64_t* ext_off_h = nullptr;         // its pinned staging
  } stage[2];
  uint64_t* hint_map = nullptr;            // per local doc: epoch << 32 | staged offset / 16 (lazy)
  uint32_t hint_epoch = 0;
  uint64_t staging_bytes = 0;
  int pf_q[2] = {-1, -1};  // FIFO of prefetched slots awaiting their PREFETCHED batch
  int pf_count = 0;
  int next_slot = 0;
  int last_slot = -1;  // staging slot of the last re-ranked batch (espn_gpu_workspace_cand_status)
  unsigned long long* h_qstats = nullptr;  // pinned B x 6
  float* bow = nullptr;
  uint32_t* out_ids = nullptr;
  float* out_scores = nullptr;
  uint32_t* out_counts = nullptr;
  uint32_t* err = nullptr;
  // Pinned host staging for the small per-batch tables, as a ring: an ASYNC
  // caller may enqueue batch n+1 before batch n's H2D copies ran, so each
  // call stages into its own slot, reused only after its copy-done event.
  static constexpr int kSlots = 8;
  struct Slot {
    uint64_t* cand_off = nullptr;
    uint32_t* needed = nullptr;
    cudaEvent_t copied = nullptr;
    bool used = false;
  } slots[kSlots];
  uint64_t calls = 0;
  // Host-I/O batches: inputs staged on a copy stream into one of two device
  // slots, so batch n+1's H2D overlaps batch n's kernels (ASYNC callers).
  cudaStream_t cs = nullptr;
  struct IoSlot {
    float* q32 = nullptr;
    uint32_t* ids = nullptr;
    float* cls = nullptr;
    uint64_t* cand_off = nullptr;
    uint32_t* needed_in = nullptr;
    cudaEvent_t in_ready = nullptr;  // H2D done (copy stream)
    cudaEvent_t done = nullptr;      // last kernel reading the slot done (compute stream)
    uint8_t* in_h = nullptr;         // pinned staging of pageable host inputs (pack layout)
    uint8_t* dpack = nullptr;        // device pack (synchronous pageable calls)
    size_t pack_bytes = 0;
    bool used = false;
  } io[2];
  uint8_t* opack = nullptr;          // device: err | out ids | scores | counts
  // synchronous pageable-buffer calls of a repeating shape replay one CUDA
  // graph (H2D pack -> plan -> MaxSim -> finalize -> D2H pack) on the caller's stream
  cudaStream_t gs = nullptr;         // capture stream
  cudaGraphExec_t sg_exec = nullptr;
  uint64_t sg_key[5] = {0, 0, 0, 0, 0};
  uint64_t sg_seen[5] = {0, 0, 0, 0, 0};  // last shape run eagerly (captured on its second call)
  bool capturing = false;            // a capture left open by an error return
  // host input pointers last checked for pinned memory (q32, ids, cls)
  bool in_pinned[3] = {false, false, false};  // this call's q32 / ids / cls
  uint8_t* out_h = nullptr;  // pinned bounce of pageable host outputs (synchronous calls)
  uint64_t io_calls = 0;
  // zero-copy outputs: last output pointers checked for pinned host memory
  void* zc_dev[3] = {nullptr, nullptr, nullptr};
  // Host pointers seen by this workspace -> pinned? (and the device alias of
  // mapped pinned memory): callers rotate a few buffer sets, so a small cache
  // keeps cudaPointerGetAttributes off the per-call path.
  struct PtrCache {
    static constexpr int N = 64;
    const void* key[N] = {};
    void* dev[N] = {};
    bool pinned[N] = {};
    int next = 0;
    bool lookup(const void* p, void** devptr) {
      for (int i = 0; i < N; ++i)
        if (key[i] == p && p) {
          *devptr = dev[i];
          return pinned[i];
        }
      cudaPointerAttributes at{};
      const bool pin = cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost;
      cudaGetLastError();  // clear a sticky "invalid value" for unregistered memory
      key[next] = p;
      pinned[next] = pin;
      dev[next] = pin ? at.devicePointer : nullptr;
      next = (next + 1) % N;
      *devptr = pin ? at.devicePointer : nullptr;
      return pin;
    }
  } ptrs;
  uint32_t* h_err = nullptr;
  bool async_pending = false;  // device err word carries bits of un-synced ASYNC calls
  // PROFILE: event triples around MaxSim / top-k, drained lazily
  static constexpr int kProf = 64;
  struct Prof {
    cudaEvent_t e[3] = {nullptr, nullptr, nullptr};
    bool pending = false;
  } prof[kProf];
  uint64_t prof_calls = 0;
  espn_counters counters{};
  uint32_t* done_flag = nullptr;  // persistent server: batch done (server -> server_wait_kernel)
  uint32_t* plan_done = nullptr;  // persistent server: plan CTAs finished (plan_kernel's submitter)
  // multi-GPU (espn_gpu_rerank_sharded): the global batch staged from host
  // arrays, this shard's own lists, the packed exchange blocks.  Grown on the
  // first sharded call of a shape (never inside a stream capture).
  struct Shard {
    float* g_q = nullptr;
    uint32_t* g_ids = nullptr;
    float* g_cls = nullptr;
    uint64_t* g_off = nullptr;
    uint32_t* g_need = nullptr;
    uint32_t* loc_ids = nullptr;
    float* loc_cls = nullptr;
    uint64_t* loc_off = nullptr;
    uint32_t* loc_need = nullptr;
    int32_t* send = nullptr;
    int32_t* recv = nullptr;
    uint64_t send_cap = 0, recv_cap = 0;  // int32 words
    bool lists = false;
  } sh;
};

namespace {
void drain_prof(espn_gpu_workspace* w, int i) {
  auto& p = w->prof[i];
  if (!p.pending) return;
  cudaEventSynchronize(p.e[2]);
  float a = 0.f, b = 0.f;
  cudaEventElapsedTime(&a, p.e[0], p.e[1]);
  cudaEventElapsedTime(&b, p.e[1], p.e[2]);
  w->counters.maxsim_ms += a;
  w->counters.topk_ms += b;
  w->counters.profiled_batches += 1;
  p.pending = false;
}
}  // namespace

namespace {
const char* const kDiskGather =
    "gather of a disk-tier table: its non-resident docs exist only in the store file (espn_store_fetch)";
// Calls that read rows need every doc of a streamed table loaded.
int require_loaded(const espn_gpu_table* t) {
  if (t && t->streamed && t->loaded_docs != t->n_docs)
    return fail(ESPN_E_INVALID_STATE, "streamed table: " + std::to_string(t->n_docs - t->loaded_docs) +
                                          " docs not loaded yet (espn_gpu_table_load_rows)");
  return ESPN_OK;
}
// ---- ESPN_TABLE_STREAMED: allocation from row_ptr, fill in doc order ----
int open_streamed(espn_gpu_table* t, const espn_table_desc* desc) {
  const uint64_t* rp = desc->row_ptr;
  const uint64_t n = desc->n_docs;
  if (rp[0] != 0) return fail(ESPN_E_INVALID_INPUT, "row_ptr[0] must be 0");
  uint32_t mn = UINT32_MAX, mx = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (rp[i + 1] <= rp[i]) return fail(ESPN_E_INVALID_INPUT, "doc " + std::to_string(i) + " has t < 1 (types.hpp:64-68)");
    const uint64_t len = rp[i + 1] - rp[i];
    mn = (uint32_t)std::min<uint64_t>(mn, len);
    mx = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(mx, len), UINT32_MAX);
  }
  t->min_t = mn;
  t->max_t = mx;
  t->n_tokens = rp[n];
  t->streamed = true;
  t->h_row_ptr.assign(rp, rp + n + 1);
  ESPN_CUDA_TRY(cudaMalloc(&t->row_ptr, (n + 1) * sizeof(uint64_t)));
  t->owned = true;
  ESPN_CUDA_TRY(cudaMemcpy(t->row_ptr, rp, (n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice));
  const uint64_t rowb = (uint64_t)t->d * 2;
  if (!desc->resident) {  // all in HBM, exactly the table's bytes
    ESPN_CUDA_TRY(cudaMalloc(&t->rows, std::max<uint64_t>(t->n_tokens * rowb, 16)));
    t->owned_rows = true;
    t->resident_docs = n;
    return ESPN_OK;
  }
  t->disk_tier = (desc->flags & ESPN_TABLE_DISK_TIER) != 0;
  uint64_t hb = 0, sb = 0, nres = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t bytes = (rp[i + 1] - rp[i]) * rowb;
    if (desc->resident[i]) { hb += bytes; ++nres; } else if (!t->disk_tier) { sb += bytes; }
  }
  uint8_t* hbm = nullptr;
  ESPN_CUDA_TRY(cudaMalloc(&hbm, std::max<uint64_t>(hb, 16)));
  t->rows = reinterpret_cast<uint16_t*>(hbm);
  t->owned_rows = true;
  ESPN_CUDA_TRY(cudaHostAlloc(&t->host_rows, std::max<uint64_t>(sb, 16), cudaHostAllocMapped | cudaHostAllocPortable));
  ESPN_CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&t->host_dev), t->host_rows, 0));
  ESPN_CUDA_TRY(cudaMalloc(&t->doc_loc, n * 8));
  t->h_loc.resize(n);
  uint64_t oh = 0, os = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t bytes = (rp[i + 1] - rp[i]) * rowb;
    if (desc->resident[i]) { t->h_loc[i] = reinterpret_cast<uint64_t>(hbm + oh); oh += bytes; }
    else if (t->disk_tier) { t->h_loc[i] = kLocHost | kLocDisk; }  // no address: staged only by prefetch_rows
    else { t->h_loc[i] = reinterpret_cast<uint64_t>(t->host_dev + os) | kLocHost; os += bytes; }
  }
  ESPN_CUDA_TRY(cudaMemcpy(t->doc_loc, t->h_loc.data(), n * 8, cudaMemcpyHostToDevice));
  t->tiered = true;
  t->hbm_row_bytes = hb;
  t->host_row_bytes = sb;
  t->resident_docs = nres;
  return ESPN_OK;
}

template <int D>
void tile_doc_host(const uint8_t* src, uint32_t t, uint8_t* dst) {
  using RL = RowLayout<D>;
  for (uint32_t j = 0; j < t; ++j)
    for (uint32_t c = 0; c < (uint32_t)RL::CH; ++c) std::memcpy(dst + RL::off(t, j, c), src + ((uint64_t)j * RL::CH + c) * 16, 16);
}
void tile_doc_host_rt(uint32_t d, const uint8_t* src, uint32_t t, uint8_t* dst) {
  switch (d) {
    case 16: tile_doc_host<16>(src, t, dst); break;
    case 32: tile_doc_host<32>(src, t, dst); break;
    case 64: tile_doc_host<64>(src, t, dst); break;
    case 128: tile_doc_host<128>(src, t, dst); break;
    default: std::memcpy(dst, src, (uint64_t)t * d * 2); break;  // plain-row dims
  }
}

int load_streamed(espn_gpu_table* t, uint64_t b0, uint64_t n, const uint16_t* rows) {
  const uint64_t rowb = (uint64_t)t->d * 2;
  const uint64_t* rp = t->h_row_ptr.data();
  const uint8_t* src = reinterpret_cast<const uint8_t*>(rows);
  // HBM docs go through a bounded bounce: pinned chunk -> device chunk -> tile kernel
  constexpr uint64_t kChunk = 64ull << 20;
  uint8_t* h_chunk = nullptr;
  uint8_t* d_chunk = nullptr;
  TileJob* h_jobs = nullptr;
  TileJob* d_jobs = nullptr;
  const uint64_t max_jobs = std::max<uint64_t>(kChunk / rowb, 1);
  auto cleanup = [&] { cudaFreeHost(h_chunk); cudaFree(d_chunk); cudaFreeHost(h_jobs); cudaFree(d_jobs); };
  bool have_hbm = false;
  for (uint64_t i = b0; i < b0 + n && !have_hbm; ++i) have_hbm = !t->tiered || !(t->h_loc[i] & 1ull);
  if (have_hbm) {
    if (cudaHostAlloc(&h_chunk, kChunk, cudaHostAllocDefault) != cudaSuccess || cudaMalloc(&d_chunk, kChunk) != cudaSuccess ||
        cudaHostAlloc(&h_jobs, max_jobs * sizeof(TileJob), cudaHostAllocDefault) != cudaSuccess ||
        cudaMalloc(&d_jobs, max_jobs * sizeof(TileJob)) != cudaSuccess) {
      cleanup();
      return fail(ESPN_E_CUDA, "streamed load: bounce allocation failed");
    }
  }
  uint64_t used = 0, nj = 0;
  auto flush = [&]() -> cudaError_t {
    if (!nj) return cudaSuccess;
    cudaError_t e = cudaMemcpy(d_chunk, h_chunk, used, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_jobs, h_jobs, nj * sizeof(TileJob), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
      const int blocks = (int)std::min<uint64_t>((nj + 7) / 8, (uint64_t)t->num_sms * 8);
      switch (t->d) {
        case 16: tile_jobs_kernel<16><<<blocks, 256>>>(d_chunk, d_jobs, (uint32_t)nj); break;
        case 32: tile_jobs_kernel<32><<<blocks, 256>>>(d_chunk, d_jobs, (uint32_t)nj); break;
        case 64: tile_jobs_kernel<64><<<blocks, 256>>>(d_chunk, d_jobs, (uint32_t)nj); break;
        case 128: tile_jobs_kernel<128><<<blocks, 256>>>(d_chunk, d_jobs, (uint32_t)nj); break;
        default:
          for (uint64_t j = 0; j < nj && e == cudaSuccess; ++j)
            e = cudaMemcpy(reinterpret_cast<void*>(h_jobs[j].dst), d_chunk + h_jobs[j].src, (uint64_t)h_jobs[j].t * rowb,
                           cudaMemcpyDeviceToDevice);
          break;
      }
      if (e == cudaSuccess) e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
    }
    used = 0;
    nj = 0;
    return e;
  };
  for (uint64_t i = b0; i < b0 + n; ++i) {
    const uint32_t tt = (uint32_t)(rp[i + 1] - rp[i]);
    const uint64_t bytes = (uint64_t)tt * rowb;
    const uint8_t* s = src + (rp[i] - rp[b0]) * rowb;
    if (t->tiered && (t->h_loc[i] & kLocDisk)) continue;  // disk tier: stays in the file
    const bool host_tier = t->tiered && (t->h_loc[i] & 1ull);
    if (host_tier) {  // tile straight into the pinned tier
      const uint64_t a = (t->h_loc[i] & ~1ull) - reinterpret_cast<uint64_t>(t->host_dev);
      tile_doc_host_rt(t->d, s, tt, t->host_rows + a);
      continue;
    }
    if (bytes > kChunk) { cleanup(); return fail(ESPN_E_INVALID_INPUT, "a document larger than the 64 MB bounce"); }
    if (used + bytes > kChunk || nj == max_jobs) {
      const cudaError_t e = flush();
      if (e != cudaSuccess) { cleanup(); return fail(ESPN_E_CUDA, std::string("streamed load: ") + cudaGetErrorString(e)); }
    }
    std::memcpy(h_chunk + used, s, bytes);
    const uint64_t dst = t->tiered ? t->h_loc[i] : reinterpret_cast<uint64_t>(t->rows) + rp[i] * rowb;
    h_jobs[nj++] = TileJob{used, dst, tt, 0};
    used += bytes;
  }
  const cudaError_t e = flush();
  cleanup();
  if (e != cudaSuccess) return fail(ESPN_E_CUDA, std::string("streamed load: ") + cudaGetErrorString(e));
  return ESPN_OK;
}

// Staging slots of a tiered workspace: pf_q lists the slots holding a
// prefetch not yet consumed by its PREFETCHED batch; any other staging must
// use the other slot, or it would overwrite that prefetch.
int peek_free_slot(const espn_gpu_workspace* w) {
  if (w->pf_count >= 2) return -1;
  int s = w->next_slot;
  if (w->pf_count == 1 && w->pf_q[0] == s) s ^= 1;
  return s;
}
int take_free_slot(espn_gpu_workspace* w) {
  const int s = peek_free_slot(w);
  if (s >= 0) w->next_slot = s ^ 1;
  return s;
}
// Splits an open table into an HBM tier (resident docs, compacted) and a
// pinned-host tier (the rest), both in the tile layout; see espn_table_desc.
int tier_table(espn_gpu_table* t, const uint8_t* resident, const uint64_t* host_row_ptr) {
  const uint32_t rowb = t->d * 2;
  std::vector<uint64_t> rp;
  if (!host_row_ptr) {
    rp.resize(t->n_docs + 1);
    ESPN_CUDA_TRY(cudaMemcpy(rp.data(), t->row_ptr, (t->n_docs + 1) * 8, cudaMemcpyDeviceToHost));
    host_row_ptr = rp.data();
  }
  uint64_t hb = 0, sb = 0, nres = 0;
  for (uint64_t i = 0; i < t->n_docs; ++i) {
    const uint64_t bytes = (host_row_ptr[i + 1] - host_row_ptr[i]) * rowb;
    if (resident[i]) { hb += bytes; ++nres; } else { sb += bytes; }
  }
  uint8_t* hbm = nullptr;
  uint8_t* host = nullptr;
  uint64_t* dloc = nullptr;
  auto undo = [&] { cudaFree(hbm); cudaFreeHost(host); cudaFree(dloc); };
  if (cudaMalloc(&hbm, std::max<uint64_t>(hb, 16)) != cudaSuccess ||
      cudaHostAlloc(&host, std::max<uint64_t>(sb, 16), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
      cudaMalloc(&dloc, t->n_docs * 8) != cudaSuccess) {
    undo();
    return fail(ESPN_E_CUDA, "tiered table: allocation failed (HBM or pinned host)");
  }
  uint8_t* host_dev = nullptr;
  if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&host_dev), host, 0) != cudaSuccess) {
    undo();
    return fail(ESPN_E_CUDA, "tiered table: host tier not mappable");
  }
  std::vector<uint64_t> loc(t->n_docs);
  uint64_t oh = 0, os = 0;
  for (uint64_t i = 0; i < t->n_docs; ++i) {
    const uint64_t bytes = (host_row_ptr[i + 1] - host_row_ptr[i]) * rowb;
    if (resident[i]) { loc[i] = reinterpret_cast<uint64_t>(hbm + oh); oh += bytes; }
    else { loc[i] = reinterpret_cast<uint64_t>(host_dev + os) | 1ull; os += bytes; }
  }
  cudaError_t e = cudaMemcpy(dloc, loc.data(), t->n_docs * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    relocate_rows_kernel<<<t->num_sms * 8, 256>>>(reinterpret_cast<const uint8_t*>(t->rows), t->row_ptr, dloc,
                                                   t->n_docs, rowb);
    e = cudaDeviceSynchronize();
  }
  if (e != cudaSuccess) {
    undo();
    return fail(ESPN_E_CUDA, std::string("tiered table: relocation failed: ") + cudaGetErrorString(e));
  }
  if (t->owned_rows) cudaFree(t->rows);
  t->rows = reinterpret_cast<uint16_t*>(hbm);
  t->owned_rows = true;
  t->host_rows = host;
  t->doc_loc = dloc;
  t->tiered = true;
  t->hbm_row_bytes = hb;
  t->host_row_bytes = sb;
  t->resident_docs = nres;
  return ESPN_OK;
}
// Stage the host-tier rows of one batch into workspace slot `slot` on stream s.
int launch_stage(espn_gpu_table* t, espn_gpu_workspace* w, int slot, const uint64_t* dev_off,
                 const uint32_t* dev_need, const uint32_t* dev_ids, uint32_t B, uint32_t R, cudaStream_t s,
                 bool prefetch) {
  auto& st = w->stage[slot];
  // consumer of espn_gpu_prefetch_hints: keep the hinted rows, the cursor and
  // the prefetch byte counts, append the misses
  const bool hinted = !prefetch && st.hint_epoch != 0;
  if (!hinted) {
    if (st.used) ESPN_CUDA_TRY(cudaStreamWaitEvent(s, st.free_ev, 0));  // previous reader done
    ESPN_CUDA_TRY(cudaMemsetAsync(st.cursor, 0, sizeof(unsigned long long), s));
    ESPN_CUDA_TRY(cudaMemsetAsync(st.qstats, 0, (size_t)B * 6 * sizeof(unsigned long long), s));
  }
  StageParams sp{};
  sp.row_ptr = t->row_ptr;
  sp.doc_loc = t->doc_loc;
  sp.n_docs = t->n_docs;
  sp.shard_count = t->shard_count;
  sp.shard_index = t->shard_index;
  sp.cand_ids = dev_ids;
  sp.cand_off = dev_off;
  sp.needed_in = dev_need;
  sp.rerank_count = R;
  sp.n_queries = B;
  sp.max_candidates = w->max_candidates;
  sp.row_bytes = t->d * 2;
  sp.prefetch = prefetch ? 1u : 0u;
  sp.cand_src = st.cand_src;
  sp.stage = st.buf;
  sp.stage_cap = w->staging_bytes;
  sp.cursor = st.cursor;
  sp.qstats = st.qstats;
  sp.err = w->err;
  sp.hint_map = hinted ? w->hint_map : nullptr;
  sp.hint_epoch = hinted ? st.hint_epoch : 0u;
  sp.cand_status = st.cand_status;
  stage_kernel<<<B, kStageThreads, 0, s>>>(sp);
  ESPN_CUDA_TRY(cudaGetLastError());
  ESPN_CUDA_TRY(cudaEventRecord(st.done, s));
  return ESPN_OK;
}
}  // namespace


namespace {
constexpr unsigned long long kServerWaitNs = 30ull * 1000 * 1000 * 1000;  // a batch that takes > 30 s fails

// (Re)launch the persistent MaxSim kernel of table t on its server stream:
// the previous launch (if any) has exited; the queue is reset and fully
// written before the kernel starts and before this returns, so work the
// caller enqueues afterwards sees the fresh queue.
int server_launch(espn_gpu_table* t) {
  ESPN_CUDA_TRY(cudaStreamSynchronize(t->server_stream));  // the old kernel is gone
  ServerQueue init{};
  init.idle_ns = t->server_idle_ns;
  init.alive_host = nullptr;
  uint32_t* alive_dev = nullptr;
  ESPN_CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&alive_dev), t->server_alive_h, 0));
  init.alive_host = alive_dev;
  ESPN_CUDA_TRY(cudaMemsetAsync(t->server, 0, sizeof(ServerQueue), t->server_stream));
  ESPN_CUDA_TRY(cudaMemcpyAsync(t->server, &init, offsetof(ServerQueue, slot), cudaMemcpyHostToDevice, t->server_stream));
  ESPN_CUDA_TRY(cudaStreamSynchronize(t->server_stream));
  *reinterpret_cast<volatile uint32_t*>(t->server_alive_h) = 1u;
  MaxSimParams p{};
  p.server = t->server;
  p.dbg = t->server_dbg;
  const cudaError_t e = launch_tc_rt(t->d, t->server_split, p, t->num_sms, t->server_stream, false);
  if (e != cudaSuccess) {
    *reinterpret_cast<volatile uint32_t*>(t->server_alive_h) = 0u;
    return fail(ESPN_E_CUDA, std::string("server launch: ") + cudaGetErrorString(e));
  }
  ++t->server_launches;
  return ESPN_OK;
}

// Before a served batch: relaunch a server that exited (idle or paused).
// Inside a stream capture nothing is launched: the captured plan submits to
// whatever server runs when the graph is replayed (none: ERR_SERVER).
int server_ensure(espn_gpu_table* t, cudaStream_t s) {
  if (*reinterpret_cast<volatile uint32_t*>(t->server_alive_h)) return ESPN_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  ESPN_CUDA_TRY(cudaStreamIsCapturing(s, &cs));
  if (cs != cudaStreamCaptureStatusNone) return ESPN_OK;
  return server_launch(t);
}

// The SM's shared-memory carveout is fixed while CTAs are resident: a CTA
// whose kernel prefers another split cannot join an SM the server occupies.
// The per-batch kernels therefore ask for the server's (maximum) carveout.
cudaError_t server_carveouts() {
  cudaError_t e = cudaFuncSetAttribute(plan_kernel<16>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(server_wait_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
  return e;
}

// Stop the kernel once the queue is drained (the table stays attached).
void server_halt(espn_gpu_table* t) {
  cudaStream_t cs = nullptr;
  if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess) {
    static const uint32_t one = 1u;
    cudaMemcpyAsync(&t->server->stop_req, &one, sizeof(uint32_t), cudaMemcpyHostToDevice, cs);
    cudaStreamSynchronize(cs);
    cudaStreamDestroy(cs);
  }
  cudaStreamSynchronize(t->server_stream);
}
}  // namespace

extern "C" {

int espn_gpu_server_start(espn_gpu_table* t, uint32_t flags, uint32_t idle_us) {
  if (!t) return fail(ESPN_E_INVALID_INPUT, "null table");
  DeviceGuard g(t->device);
  if (t->server) return server_ensure(t, nullptr);
  if (!t->tc_ok || !tc_supported(t->d))
    return fail(ESPN_E_INVALID_CONFIG, "the persistent server runs the tcgen05 MaxSim: needs sm_100 and d in {16,32,64,128}");
  if (t->tiered) return fail(ESPN_E_INVALID_CONFIG, "the persistent server serves HBM-resident (untiered) tables");
  const bool split = tc_query_split(t->d, t->dtype, flags);
  // the per-batch plan and wait kernels must fit on an SM beside a server CTA
  {
    int smem_sm = 0, reserved = 0, regs_sm = 0;
    ESPN_CUDA_TRY(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, t->device));
    ESPN_CUDA_TRY(cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, t->device));
    ESPN_CUDA_TRY(cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, t->device));
    cudaFuncAttributes fp{}, fw{};
    ESPN_CUDA_TRY(cudaFuncGetAttributes(&fp, plan_kernel<16>));
    ESPN_CUDA_TRY(cudaFuncGetAttributes(&fw, server_wait_kernel));
    int tc_smem = 0, tc_threads = 0, tc_regs = 0;
    switch (t->d * 2 + (split ? 1 : 0)) {
#define ESPN_SZ(DD, SS)                                                                    \
  case DD * 2 + SS: {                                                                      \
    cudaFuncAttributes fa{};                                                               \
    ESPN_CUDA_TRY(cudaFuncGetAttributes(&fa, maxsim_tc_kernel<DD, (bool)SS>));             \
    tc_smem = TcLayout<DD, (bool)SS>::SMEM_BYTES + (int)fa.sharedSizeBytes;                \
    tc_threads = TcLayout<DD, (bool)SS>::NTHREADS;                                         \
    tc_regs = fa.numRegs;                                                                  \
  } break;
      ESPN_SZ(16, 0) ESPN_SZ(16, 1) ESPN_SZ(32, 0) ESPN_SZ(32, 1) ESPN_SZ(64, 0) ESPN_SZ(64, 1) ESPN_SZ(128, 0)
      ESPN_SZ(128, 1)
#undef ESPN_SZ
    }
    const int need_smem = tc_smem + reserved + (int)fp.sharedSizeBytes + reserved;
    // registers come from the SM's 4 sub-partitions (16K each); a CTA's warps
    // are spread over all four, so the busiest sub-partition (ceil(17/4) = 5
    // server warps) must still hold a plan (or wait) warp
    auto warp_regs = [](int r) { return (r * 32 + 255) / 256 * 256; };
    const int tc_warps = tc_threads / 32;
    const int need_regs = ((tc_warps + 3) / 4) * warp_regs(tc_regs) + std::max(warp_regs(fp.numRegs), warp_regs(fw.numRegs));
    if (need_smem > smem_sm || need_regs > regs_sm / 4)
      return fail(ESPN_E_INVALID_CONFIG, "persistent server: the plan kernel would not fit beside a server CTA (smem " +
                                             std::to_string(need_smem) + "/" + std::to_string(smem_sm) + ", regs " +
                                             std::to_string(need_regs) + "/" + std::to_string(regs_sm / 4) + " per sub-partition)");
  }
  ESPN_CUDA_TRY(server_carveouts());
  ServerQueue* q = nullptr;
  uint32_t* alive = nullptr;
  cudaStream_t st = nullptr;
  if (cudaMalloc(&q, sizeof(ServerQueue)) != cudaSuccess ||
      cudaHostAlloc(&alive, sizeof(uint32_t), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
      cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
    cudaFree(q);
    cudaFreeHost(alive);
    if (st) cudaStreamDestroy(st);
    return fail(ESPN_E_CUDA, "persistent server: allocation failed");
  }
  *alive = 0;
  t->server = q;
  t->server_alive_h = alive;
  t->server_stream = st;
  t->server_split = split;
  t->server_idle_ns = (uint64_t)(idle_us ? idle_us : 50000u) * 1000ull;
  static const uint32_t dbg = [] {
    const char* e = getenv("ESPN_DEBUG");
    return e ? (uint32_t)strtoul(e, nullptr, 0) : 0u;
  }();
  t->server_dbg = dbg;
  const int rc = server_launch(t);
  if (rc) {
    const std::string why = g_last_error;
    espn_gpu_server_stop(t);
    return fail(rc, why);
  }
  return ESPN_OK;
}

int espn_gpu_server_pause(espn_gpu_table* t) {
  if (!t || !t->server) return ESPN_OK;
  DeviceGuard g(t->device);
  server_halt(t);
  return ESPN_OK;
}

int espn_gpu_server_stop(espn_gpu_table* t) {
  if (!t || !t->server) return ESPN_OK;
  DeviceGuard g(t->device);
  server_halt(t);  // the kernel stops once the queue is drained
  cudaStreamDestroy(t->server_stream);
  cudaFree(t->server);
  cudaFreeHost(t->server_alive_h);
  t->server = nullptr;
  t->server_stream = nullptr;
  t->server_alive_h = nullptr;
  return ESPN_OK;
}

int espn_gpu_server_debug(const espn_gpu_table* t, uint64_t* out8) {
  if (!t || !t->server || !out8) return fail(ESPN_E_INVALID_INPUT, "no server");
  DeviceGuard g(t->device);
  cudaStream_t cs = nullptr;
  ESPN_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  ServerQueue h;
  ESPN_CUDA_TRY(cudaMemcpyAsync(&h, t->server, sizeof h, cudaMemcpyDeviceToHost, cs));
  ESPN_CUDA_TRY(cudaStreamSynchronize(cs));
  cudaStreamDestroy(cs);
  out8[0] = h.state;
  out8[1] = h.stop_req;
  out8[2] = h.exited;
  out8[3] = h.idle_ns;
  out8[4] = h.slot[0].ready;
  out8[5] = h.slot[0].done;
  out8[6] = (uint64_t)h.slot[0].done_count | ((uint64_t)h.slot[0].merge_count << 32);
  out8[7] = *reinterpret_cast<volatile uint32_t*>(t->server_alive_h) | (t->server_launches << 8);
  return ESPN_OK;
}

int espn_gpu_server_running(const espn_gpu_table* t) {
  return (t && t->server && *reinterpret_cast<volatile uint32_t*>(t->server_alive_h)) ? 1 : 0;
}

}  // extern "C"

extern "C" {

const char* espn_last_error(void) { return g_last_error.c_str(); }
int espn_abi_version(void) { return ESPN_GPU_ABI_VERSION; }

int espn_gpu_table_open(const espn_table_desc* desc, espn_gpu_table** out) {
  if (!desc || !out) return fail(ESPN_E_INVALID_INPUT, "null argument");
  *out = nullptr;
  if (desc->d == 0 || desc->d % 8 != 0 || desc->d > 256)
    return fail(ESPN_E_INVALID_INPUT, "token dim d must be a multiple of 8 in [8, 256]");
  if (desc->dtype > ESPN_DTYPE_BF16) return fail(ESPN_E_INVALID_INPUT, "dtype must be f16 or bf16");
  if (desc->value_width != 2 && desc->value_width != 4)
    return fail(ESPN_E_INVALID_INPUT, "value_width must be 2 or 4 (store.hpp:27)");
  if (desc->alignment != 1 && desc->alignment != 512 && desc->alignment != 4096)
    return fail(ESPN_E_INVALID_INPUT, "alignment must be 1, 512 or 4096 (store.hpp:28)");
  if (desc->n_docs == 0) return fail(ESPN_E_INVALID_INPUT, "empty table");
  const bool streamed = (desc->flags & ESPN_TABLE_STREAMED) != 0;
  if (!desc->row_ptr || (!desc->rows && !streamed)) return fail(ESPN_E_INVALID_INPUT, "null row_ptr/rows");
  if (streamed && (desc->flags & ESPN_TABLE_DEVICE_BORROWED))
    return fail(ESPN_E_INVALID_INPUT, "a streamed table takes a HOST row_ptr");
  if ((desc->flags & ESPN_TABLE_DISK_TIER) && !(streamed && desc->resident))
    return fail(ESPN_E_INVALID_INPUT, "ESPN_TABLE_DISK_TIER needs ESPN_TABLE_STREAMED and a resident mask");
  int sms = 0;
  bool tc = false;
  int st = check_device(desc->device, &sms, &tc);
  if (st) return st;
  DeviceGuard g(desc->device);
  auto* t = new espn_gpu_table();
  t->device = desc->device;
  t->num_sms = sms;
  t->tc_ok = tc;
  t->n_docs = desc->n_docs;
  t->d = desc->d;
  t->dtype = desc->dtype;
  t->d_cls = desc->d_cls;
  t->value_width = desc->value_width;
  t->alignment = desc->alignment;
  t->shard_count = desc->shard_count > 1 ? desc->shard_count : 1;
  t->shard_index = desc->shard_count > 1 ? desc->shard_index : 0;
  if (t->shard_index >= t->shard_count) { delete t; return fail(ESPN_E_INVALID_INPUT, "shard_index >= shard_count"); }
  const bool borrowed = (desc->flags & ESPN_TABLE_DEVICE_BORROWED) != 0;
  if (streamed) {
    const int ss = open_streamed(t, desc);
    if (ss) {
      espn_gpu_table_close(t);
      return ss;
    }
    *out = t;
    return ESPN_OK;
  }
  if (!borrowed) {
    // host tables: validate (types.hpp:64-68: t >= 1), then upload
    const uint64_t* rp = desc->row_ptr;
    if (rp[0] != 0) { delete t; return fail(ESPN_E_INVALID_INPUT, "row_ptr[0] must be 0"); }
    uint32_t mn = UINT32_MAX, mx = 0;
    for (uint64_t i = 0; i < desc->n_docs; ++i) {
      if (rp[i + 1] <= rp[i]) {
        delete t;
        return fail(ESPN_E_INVALID_INPUT, "doc " + std::to_string(i) + " has t < 1 (types.hpp:64-68)");
      }
      const uint64_t len = rp[i + 1] - rp[i];
      mn = (uint32_t)std::min<uint64_t>(mn, len);
      mx = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(mx, len), UINT32_MAX);
    }
    t->min_t = mn;
    t->max_t = mx;
    t->n_tokens = rp[desc->n_docs];
    cudaError_t e1 = cudaMalloc(&t->row_ptr, (desc->n_docs + 1) * sizeof(uint64_t));
    cudaError_t e2 = cudaMalloc(&t->rows, std::max<uint64_t>(1, t->n_tokens * t->d) * sizeof(uint16_t));
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
      cudaFree(t->row_ptr);
      cudaFree(t->rows);
      delete t;
      return fail(ESPN_E_CUDA, "cudaMalloc failed for the HBM table");
    }
    t->owned = true;
    t->owned_rows = true;
    cudaMemcpy(t->row_ptr, rp, (desc->n_docs + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice);
    const size_t row_bytes = t->n_tokens * t->d * sizeof(uint16_t);
    cudaError_t e3;
    if (layout_tiled(t->d) && !(desc->flags & ESPN_TABLE_ROWS_TILED)) {
      // upload plain rows to a staging buffer, then tile into the table
      uint16_t* plain = nullptr;
      e3 = cudaMalloc(&plain, std::max<size_t>(row_bytes, 16));
      if (e3 == cudaSuccess) e3 = cudaMemcpy(plain, desc->rows, row_bytes, cudaMemcpyHostToDevice);
      if (e3 == cudaSuccess) e3 = tile_rows(t->d, plain, t->row_ptr, t->n_docs, t->rows, t->num_sms);
      cudaFree(plain);
    } else {
      e3 = cudaMemcpy(t->rows, desc->rows, row_bytes, cudaMemcpyHostToDevice);
    }
    if (e3 != cudaSuccess) {
      espn_gpu_table_close(t);
      return fail(ESPN_E_CUDA, std::string("table upload: ") + cudaGetErrorString(e3));
    }
  } else {
    t->row_ptr = const_cast<uint64_t*>(desc->row_ptr);
    t->rows = const_cast<uint16_t*>(desc->rows);
    unsigned long long* mm = nullptr;
    ESPN_CUDA_TRY(cudaMalloc(&mm, 3 * sizeof(unsigned long long)));
    unsigned long long init[3] = {~0ull, 0ull, 0ull};
    cudaMemcpy(mm, init, sizeof init, cudaMemcpyHostToDevice);
    minmax_len_kernel<<<sms * 4, 256>>>(t->row_ptr, t->n_docs, mm);
    unsigned long long res[3];
    uint64_t first = 1, last = 0;
    cudaMemcpy(res, mm, sizeof res, cudaMemcpyDeviceToHost);
    cudaMemcpy(&first, t->row_ptr, sizeof(uint64_t), cudaMemcpyDeviceToHost);
    cudaError_t e = cudaMemcpy(&last, t->row_ptr + t->n_docs, sizeof(uint64_t), cudaMemcpyDeviceToHost);
    cudaFree(mm);
    if (e != cudaSuccess) { delete t; return fail(ESPN_E_CUDA, cudaGetErrorString(e)); }
    if (first != 0 || res[2] != 0) {
      delete t;
      return fail(ESPN_E_INVALID_INPUT, "row_ptr must start at 0 and give every doc t >= 1");
    }
    t->min_t = (uint32_t)res[0];
    t->max_t = (uint32_t)std::min<unsigned long long>(res[1], UINT32_MAX);
    t->n_tokens = last;
    if (layout_tiled(t->d) && !(desc->flags & ESPN_TABLE_ROWS_TILED)) {
      // borrowed plain rows: the table keeps its own tiled copy
      uint16_t* tiled = nullptr;
      cudaError_t e4 = cudaMalloc(&tiled, std::max<size_t>(t->n_tokens * t->d * sizeof(uint16_t), 16));
      if (e4 == cudaSuccess) e4 = tile_rows(t->d, t->rows, t->row_ptr, t->n_docs, tiled, t->num_sms);
      if (e4 != cudaSuccess) {
        cudaFree(tiled);
        delete t;
        return fail(ESPN_E_CUDA, std::string("table tiling: ") + cudaGetErrorString(e4));
      }
      t->rows = tiled;
      t->owned_rows = true;
    }
  }
  if (desc->resident) {
    const int ts = tier_table(t, desc->resident, borrowed ? nullptr : desc->row_ptr);
    if (ts) {
      espn_gpu_table_close(t);
      return ts;
    }
  } else {
    t->resident_docs = t->n_docs;
  }
  *out = t;
  return ESPN_OK;
}

int espn_gpu_table_close(espn_gpu_table* t) {
  if (!t) return ESPN_OK;
  espn_gpu_server_stop(t);
  DeviceGuard g(t->device);
  if (t->owned) cudaFree(t->row_ptr);
  if (t->owned_rows) cudaFree(t->rows);
  cudaFree(t->doc_loc);
  if (t->host_rows) cudaFreeHost(t->host_rows);
  delete t;
  return ESPN_OK;
}

int espn_gpu_table_load_rows(espn_gpu_table* t, uint64_t doc_begin, uint64_t n, const uint16_t* rows) {
  if (!t) return fail(ESPN_E_INVALID_INPUT, "null table");
  if (!t->streamed) return fail(ESPN_E_INVALID_STATE, "not a streamed table (ESPN_TABLE_STREAMED)");
  if (doc_begin != t->loaded_docs) return fail(ESPN_E_INVALID_INPUT, "streamed docs must be loaded in order");
  if (n == 0) return ESPN_OK;
  if (doc_begin + n > t->n_docs) return fail(ESPN_E_INVALID_INPUT, "doc range beyond the table");
  if (!rows) return fail(ESPN_E_INVALID_INPUT, "null rows");
  DeviceGuard g(t->device);
  const int st = load_streamed(t, doc_begin, n, rows);
  if (st) return st;
  t->loaded_docs += n;
  if (t->loaded_docs == t->n_docs) {  // complete: drop the fill-time host copies
    std::vector<uint64_t>().swap(t->h_loc);
    if (!t->disk_tier) std::vector<uint64_t>().swap(t->h_row_ptr);  // (disk tier: espn_gpu_prefetch_rows checks)
  }
  return ESPN_OK;
}

int espn_gpu_table_info(const espn_gpu_table* t, espn_table_info* out) {
  if (!t || !out) return fail(ESPN_E_INVALID_INPUT, "null argument");
  out->n_docs = t->n_docs;
  out->n_tokens = t->n_tokens;
  out->d = t->d;
  out->dtype = t->dtype;
  out->max_tokens = t->max_t;
  out->min_tokens = t->min_t;
  out->hbm_bytes = (t->owned ? (t->n_docs + 1) * 8 : 0) +
                   (t->tiered ? t->hbm_row_bytes + t->n_docs * 8 : (t->owned_rows ? t->n_tokens * t->d * 2 : 0));
  out->host_bytes = t->host_row_bytes;
  out->resident_docs = t->resident_docs;
  return ESPN_OK;
}

int espn_gpu_workspace_create(espn_gpu_table* t, const espn_workspace_desc* desc,
                              espn_gpu_workspace** out) {
  if (!t || !desc || !out) return fail(ESPN_E_INVALID_INPUT, "null argument");
  *out = nullptr;
  if (desc->max_queries == 0 || desc->max_candidates == 0)
    return fail(ESPN_E_INVALID_INPUT, "workspace capacities must be positive");
  if (desc->max_query_tokens == 0 || desc->max_query_tokens > 32)
    return fail(ESPN_E_INVALID_INPUT, "max_query_tokens must be in [1, 32]");
  DeviceGuard g(t->device);
  auto* w = new espn_gpu_workspace();
  w->table = t;
  w->max_queries = desc->max_queries;
  w->max_candidates = desc->max_candidates;
  w->max_nq = desc->max_query_tokens;
  const size_t B = desc->max_queries, C = desc->max_candidates;
  cudaError_t e = cudaSuccess;
  auto al = [&](void** p, size_t bytes) {
    if (e == cudaSuccess) e = cudaMalloc(p, std::max<size_t>(bytes, 16));
  };
  al((void**)&w->unit_off, (B + 1) * sizeof(uint32_t));
  al((void**)&w->needed, B * sizeof(uint32_t));
  // work-unit table capacity: every query may end in a partial unit
  {
    // (the shorter of the two layouts' units that fit the longest doc: the
    // query precision picks one per call)
    const int ur = t->tc_ok ? tc_unit_docs_rt(t->d, t->max_t, false) : 0;
    const int us = t->tc_ok ? tc_unit_docs_rt(t->d, t->max_t, true) : 0;
    int ud = (ur > 0 && us > 0) ? std::min(ur, us) : std::max(ur, us);
    if (ud > kMinUnitDocs) ud = kMinUnitDocs;  // small batches use units down to kMinUnitDocs docs
    w->max_units = ud > 0 ? (C + ud - 1) / ud + 2 * B : 0;  // + partial units (needed, tail)
  }
  al((void**)&w->unit_tab, w->max_units * sizeof(uint4));
  al((void**)&w->n_units, sizeof(uint32_t));
  al((void**)&w->kprof, 4 * sizeof(unsigned long long));
  al((void**)&w->done_flag, sizeof(uint32_t));
  al((void**)&w->plan_done, sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(w->done_flag, 0, sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(w->plan_done, 0, sizeof(uint32_t));
  if (t->tiered) {
    w->staging_bytes = desc->staging_bytes ? desc->staging_bytes : (64ull << 20);
    for (auto& st : w->stage) {
      al((void**)&st.buf, w->staging_bytes);
      al((void**)&st.cand_src, C * sizeof(uint64_t));
      al((void**)&st.cand_status, C);
      al((void**)&st.cursor, sizeof(unsigned long long));
      al((void**)&st.qstats, B * 6 * sizeof(unsigned long long));
      al((void**)&st.off, (B + 1) * sizeof(uint64_t));
      al((void**)&st.need, B * sizeof(uint32_t));
      if (e == cudaSuccess) e = cudaMallocHost(&st.off_h, (B + 1) * sizeof(uint64_t));
      if (e == cudaSuccess) e = cudaMallocHost(&st.need_h, (B + 1) * sizeof(uint32_t));
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&st.done, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&st.free_ev, cudaEventDisableTiming);
    }
  }
  if (e == cudaSuccess) e = cudaMallocHost(&w->h_qstats, B * 6 * sizeof(unsigned long long));
  // same size as opack ([err 16 B | ids | scores | counts]): the bounce receives the whole pack
  if (e == cudaSuccess) e = cudaMallocHost(&w->out_h, 16 + (size_t)B * kMaxK * 8 + (size_t)B * 4);
  w->max_list = desc->max_list ? desc->max_list : (uint32_t)std::min<size_t>(C, 4096);
  // fused top-k state; the dedup hash is 8x the declared list (one-probe
  // inserts), at most 32K slots (lists up to 16K candidates)
  w->hash_slots = 128;
  while (w->hash_slots < 8ull * w->max_list && w->hash_slots < (1u << 15)) w->hash_slots <<= 1;
  if (w->max_units && 2ull * w->max_list <= w->hash_slots) {
    al((void**)&w->unit_top, w->max_units * kFusedMaxK * sizeof(unsigned long long));
    al((void**)&w->dedup, 2 * B * (size_t)w->hash_slots * sizeof(uint32_t));
    al((void**)&w->ff_seen, 2 * B * sizeof(uint32_t));
    al((void**)&w->fused_state, 4 * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(w->ff_seen, 0, 2 * B * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(w->fused_state, 0, 4 * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(w->dedup, 0xFF, 2 * B * (size_t)w->hash_slots * sizeof(uint32_t));
  }
  // single-launch small batches (ESPN_KERNEL_SMALL): arrival counters (zero
  // between batches; each query's last CTA resets its own) and per-CTA lists
  al((void**)&w->small_arrive, kSmallMaxB * sizeof(uint32_t));
  al((void**)&w->small_top, (size_t)kSmallMaxCtas * kFusedMaxK * sizeof(unsigned long long));
  al((void**)&w->small_hash, (size_t)kSmallMaxB * kSmallHashSlots * sizeof(uint32_t));
  al((void**)&w->small_ff, kSmallMaxB * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(w->small_arrive, 0, kSmallMaxB * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(w->small_ff, 0, kSmallMaxB * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(w->small_hash, 0xFF, (size_t)kSmallMaxB * kSmallHashSlots * sizeof(uint32_t));
  al((void**)&w->bow, C * sizeof(float));
  // outputs and the error word in ONE allocation: [err 16 B | ids | scores |
  // counts], so a synchronous call reads everything back with one copy
  al((void**)&w->opack, 16 + (size_t)B * kMaxK * 8 + (size_t)B * 4);
  if (e == cudaSuccess) {
    w->err = reinterpret_cast<uint32_t*>(w->opack);
    w->out_ids = reinterpret_cast<uint32_t*>(w->opack + 16);
    w->out_scores = reinterpret_cast<float*>(w->out_ids + (size_t)B * kMaxK);
    w->out_counts = reinterpret_cast<uint32_t*>(w->out_scores + (size_t)B * kMaxK);
  }
  for (auto& io : w->io) {
    al((void**)&io.q32, B * w->max_nq * t->d * sizeof(float));
    al((void**)&io.ids, C * sizeof(uint32_t));
    al((void**)&io.cls, C * sizeof(float));
    al((void**)&io.cand_off, (B + 1) * sizeof(uint64_t));
    al((void**)&io.needed_in, B * sizeof(uint32_t));
    // packed inputs of synchronous pageable-buffer calls: [offsets | needed |
    // q32 | ids | cls], 16-byte aligned pieces, one H2D per call
    io.pack_bytes = ((B + 1) * 8 + 15) / 16 * 16 + (B * 4 + 15) / 16 * 16 +
                    ((size_t)B * w->max_nq * t->d * 4 + 15) / 16 * 16 + (C * 4 + 15) / 16 * 16 + C * 4;
    al((void**)&io.dpack, io.pack_bytes);
    if (e == cudaSuccess) e = cudaMallocHost(&io.in_h, io.pack_bytes);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&io.in_ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&io.done, cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&w->cs, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&w->gs, cudaStreamNonBlocking);
  for (auto& sl : w->slots) {
    if (e == cudaSuccess) e = cudaMallocHost(&sl.cand_off, (B + 1) * sizeof(uint64_t));
    if (e == cudaSuccess) e = cudaMallocHost(&sl.needed, (B + 1) * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sl.copied, cudaEventDisableTiming);
  }
  for (auto& pr : w->prof)
    for (auto& ev : pr.e)
      if (e == cudaSuccess) e = cudaEventCreate(&ev);
  if (e == cudaSuccess) e = cudaMallocHost(&w->h_err, sizeof(uint32_t));
  // the whole output pack starts defined: a synchronous call copies it back in
  // one piece, including the slots beyond a query's count (unspecified, 0 here)
  if (e == cudaSuccess) e = cudaMemset(w->opack, 0, 16 + (size_t)B * kMaxK * 8 + (size_t)B * 4);
  if (e == cudaSuccess) {
    const unsigned long long init[4] = {0ull, 0ull, ~0ull, 0ull};
    e = cudaMemcpy(w->kprof, init, sizeof init, cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    espn_gpu_workspace_destroy(w);
    return fail(ESPN_E_CUDA, std::string("workspace allocation: ") + cudaGetErrorString(e));
  }
  *out = w;
  return ESPN_OK;
}

int espn_gpu_workspace_destroy(espn_gpu_workspace* w) {
  if (!w) return ESPN_OK;
  DeviceGuard g(w->table->device);
  for (auto& io : w->io) {
    if (io.done) cudaEventSynchronize(io.done);
    cudaFree(io.q32); cudaFree(io.ids); cudaFree(io.cls); cudaFree(io.cand_off); cudaFree(io.needed_in);
    cudaFreeHost(io.in_h); cudaFree(io.dpack);
    if (io.in_ready) cudaEventDestroy(io.in_ready);
    if (io.done) cudaEventDestroy(io.done);
  }
  if (w->cs) { cudaStreamSynchronize(w->cs); cudaStreamDestroy(w->cs); }
  if (w->sg_exec) cudaGraphExecDestroy(w->sg_exec);
  if (w->gs) cudaStreamDestroy(w->gs);
  cudaFree(w->unit_off); cudaFree(w->needed); cudaFree(w->unit_tab); cudaFree(w->n_units);
  cudaFree(w->kprof);
  cudaFree(w->done_flag);
  cudaFree(w->plan_done);
  cudaFree(w->unit_top); cudaFree(w->dedup); cudaFree(w->ff_seen); cudaFree(w->fused_state);
  cudaFree(w->small_arrive); cudaFree(w->small_top); cudaFree(w->small_hash); cudaFree(w->small_ff);
  for (auto& st : w->stage) {
    if (st.done) cudaEventSynchronize(st.done);
    if (st.free_ev) cudaEventSynchronize(st.free_ev);
    cudaFree(st.buf); cudaFree(st.cand_src); cudaFree(st.cand_status); cudaFree(st.cursor); cudaFree(st.qstats); cudaFree(st.off);
    cudaFree(st.need); cudaFreeHost(st.off_h); cudaFreeHost(st.need_h);
    cudaFree(st.hint_ids); cudaFreeHost(st.hint_ids_h);
    cudaFree(st.ext_buf); cudaFree(st.ext_off); cudaFreeHost(st.ext_off_h);
    st.hint_epoch = 0;
    if (st.done) cudaEventDestroy(st.done);
    if (st.free_ev) cudaEventDestroy(st.free_ev);
  }
  cudaFree(w->hint_map);
  cudaFreeHost(w->h_qstats); cudaFreeHost(w->out_h); cudaFree(w->bow); cudaFree(w->opack);
  for (auto& sl : w->slots) {
    if (sl.copied) cudaEventSynchronize(sl.copied);
    cudaFreeHost(sl.cand_off); cudaFreeHost(sl.needed);
    if (sl.copied) cudaEventDestroy(sl.copied);
  }
  for (auto& pr : w->prof)
    for (auto& ev : pr.e)
      if (ev) { cudaEventSynchronize(ev); cudaEventDestroy(ev); }
  cudaFreeHost(w->h_err);
  {
    auto& h = w->sh;
    cudaFree(h.g_q); cudaFree(h.g_ids); cudaFree(h.g_cls); cudaFree(h.g_off); cudaFree(h.g_need);
    cudaFree(h.loc_ids); cudaFree(h.loc_cls); cudaFree(h.loc_off); cudaFree(h.loc_need);
    cudaFree(h.send); cudaFree(h.recv);
  }
  delete w;
  return ESPN_OK;
}

int espn_gpu_rerank(espn_gpu_table* t, espn_gpu_workspace* w, const espn_rerank_args* a,
                    espn_rerank_out* o, void* stream_v) {
  if (!t || !w || !a || !o) return fail(ESPN_E_INVALID_INPUT, "null argument");
  if (w->table != t) return fail(ESPN_E_INVALID_STATE, "workspace belongs to another table");
  if (const int ls = require_loaded(t)) return ls;
  cudaStream_t s = static_cast<cudaStream_t>(stream_v);
  const uint32_t B = a->n_queries, nq = a->n_query_tokens, k = a->final_k;
  // ---- host-side validation (pipeline.hpp:31-32) ----
  if (B > w->max_queries) return fail(ESPN_E_INVALID_INPUT, "n_queries exceeds workspace capacity");
  if (nq < 1 || nq > w->max_nq) return fail(ESPN_E_INVALID_INPUT, "n_query_tokens must be in [1, workspace max <= 32]");
  if (k < 1 || k > (uint32_t)kMaxK) return fail(ESPN_E_INVALID_INPUT, "final_k must be in [1, 1024]");
  if (!std::isfinite(a->alpha)) return fail(ESPN_E_INVALID_INPUT, "alpha must be finite");
  const bool partial = (a->flags & ESPN_RERANK_PARTIAL) != 0;
  if (!partial && a->rerank_count < k)
    return fail(ESPN_E_INVALID_INPUT, "rerank_count < final_k requires partial re-ranking (SPEC.md:265)");
  if (B == 0) return ESPN_OK;
  if (!a->cand_offsets || !a->query_tokens || !o->ids || !o->scores || !o->counts)
    return fail(ESPN_E_INVALID_INPUT, "null array argument");
  const bool dev_io = (a->flags & ESPN_RERANK_DEVICE_IO) != 0;
  const bool dev_off = (a->flags & ESPN_RERANK_DEVICE_OFFSETS) != 0;
  if (dev_off && !dev_io) return fail(ESPN_E_INVALID_INPUT, "DEVICE_OFFSETS requires DEVICE_IO");
  uint64_t C = 0;          // total candidates (host-offset mode only)
  uint64_t max_list = 0;   // longest scored list (hash sizing)
  if (!dev_off) {
    const uint64_t* off = a->cand_offsets;
    if (off[0] != 0) return fail(ESPN_E_INVALID_INPUT, "cand_offsets[0] must be 0");
    for (uint32_t b = 0; b < B; ++b) {
      if (off[b + 1] < off[b]) return fail(ESPN_E_INVALID_INPUT, "cand_offsets must be non-decreasing");
      const uint64_t n = off[b + 1] - off[b];
      const uint64_t need = std::min<uint64_t>(n, a->needed_counts ? a->needed_counts[b] : a->rerank_count);
      max_list = std::max<uint64_t>(max_list, partial ? n : need);
    }
    C = off[B];
    if (C > w->max_candidates) return fail(ESPN_E_INVALID_INPUT, "candidates exceed workspace capacity");
    if (C > 0 && (!a->cand_ids || !a->cand_cls)) return fail(ESPN_E_INVALID_INPUT, "null candidate arrays");
  } else {
    max_list = w->max_list;  // device offsets: the workspace's declared bound
  }
  DeviceGuard g(t->device);

  // ---- kernel choice (tcgen05 when the dim has a tensor-core tiling) ----
  uint32_t kern = a->kernel;
  // (the query precision the tcgen05 path would use picks the unit layout)
  const bool split_if_tc = tc_query_split(t->d, t->dtype, a->flags);
  const int layout_docs = t->tc_ok ? tc_unit_docs_rt(t->d, t->max_t, split_if_tc) : 0;
  // size the units so that the batch is a whole number of rounds over the
  // SMs: with units of at most `cap` docs, how many rounds does the batch
  // take?  Then spread each query over as many (shorter) units as those rounds
  // hold.  C2 (64 x 1000, 148 SMs, cap 96): 704 units of 91 docs = 4.8
  // rounds; C1 (1 x 1000): 125 units of 8 docs, one per SM.
  auto size_units = [&](int cap) -> int {
    if (cap <= kMinUnitDocs || a->n_queries == 0) return cap;
    const uint64_t Bq = a->n_queries;
    const uint64_t per_q = std::max<uint64_t>(1, std::min<uint64_t>(std::max<uint32_t>(a->rerank_count, 1u), max_list));
    const uint64_t sms = (uint64_t)t->num_sms;
    const uint64_t n_long = Bq * ((per_q + cap - 1) / cap);
    const uint64_t upq = std::max<uint64_t>(1, ((n_long + sms - 1) / sms) * sms / Bq);  // units per query
    return (int)std::max<uint64_t>(kMinUnitDocs, std::min<uint64_t>((uint64_t)cap, (per_q + upq - 1) / upq));
  };
  int unit_docs = size_units(layout_docs);
  // single-launch small batches (K5, small.cuh): a few queries, short lists,
  // fused-size k, table in HBM.  Opt-in only: its CUDA-core arithmetic on the
  // fp32 query is exact, the tcgen05 path rounds the query (f16) or splits it
  // (bf16), so AUTO never switches arithmetic with the batch size -- a query's
  // scores do not depend on the batch it arrives in.
  const bool small_ok = k <= (uint32_t)kFusedMaxK && !t->tiered && simt_supported(t->d) && B <= (uint32_t)kSmallMaxB &&
                        max_list <= (uint64_t)kSmallMaxList && !(a->flags & ESPN_RERANK_PREFETCHED);
  if (kern == ESPN_KERNEL_SMALL && !small_ok)
    return fail(ESPN_E_INVALID_CONFIG, "single-launch small batches need n_queries <= 16, scored lists <= 2048, "
                                       "final_k <= 32, an HBM-resident table and d in {8,16,32,48,64,96,128}");
  const bool small = kern == ESPN_KERNEL_SMALL;
  const uint32_t small_P = small ? small_ctas_per_query(max_list, B) : 0u;
  if (small) unit_docs = (int)small_P;  // (graph key: the grid shape)
  if (kern == ESPN_KERNEL_AUTO) kern = (tc_supported(t->d) && unit_docs > 0) ? ESPN_KERNEL_TCGEN05 : ESPN_KERNEL_SIMT;
  if (kern == ESPN_KERNEL_TCGEN05 && (!t->tc_ok || !tc_supported(t->d) || unit_docs <= 0))
    return fail(ESPN_E_INVALID_CONFIG, "tcgen05 MaxSim needs an sm_100 device, d in {16,32,64,128} and docs of at most " +
                                           std::to_string(tc_max_tokens_rt(t->d, split_if_tc)) + " tokens at d=" + std::to_string(t->d) +
                                           " (longest doc here: " + std::to_string(t->max_t) + ")");
  if (kern == ESPN_KERNEL_SIMT && !simt_supported(t->d))
    return fail(ESPN_E_INVALID_CONFIG, "CUDA-core MaxSim supports d in {8,16,32,48,64,96,128}");
  const bool tc = kern == ESPN_KERNEL_TCGEN05;

  static const uint32_t dbg = [] {
    const char* e = getenv("ESPN_DEBUG");
    return e ? (uint32_t)strtoul(e, nullptr, 0) : 0u;
  }();
  const bool profile_dev = (a->flags & ESPN_RERANK_PROFILE) != 0;
  // host CUDA events only outside stream capture (device offsets = graph-capturable
  // mode); the MaxSim kernel times itself on the device in both modes
  const bool profile = profile_dev && !dev_off;
  // Fused aggregate + top-k (and duplicate check) inside the tcgen05 MaxSim
  // kernel when final_k <= 32 and the workspace's dedup hash covers the
  // lists; ESPN_DEBUG bit 512 / ESPN_RERANK_SEPARATE_TOPK: separate top-k kernel.
  const bool fused = tc && k <= (uint32_t)kFusedMaxK && w->dedup != nullptr && 2ull * max_list <= w->hash_slots &&
                     !(a->flags & ESPN_RERANK_SEPARATE_TOPK) && !(dbg & 512u);
  // ---- persistent server (espn_gpu_server_start): the batch is submitted to
  // the running MaxSim kernel by the plan and awaited by a one-thread kernel ----
  const bool qsplit = tc && tc_query_split(t->d, t->dtype, a->flags);
  const bool served = t->server != nullptr && tc && fused && !t->tiered && qsplit == t->server_split;
  // any other kernel would wait for SM resources the running server holds
  // (every SM is occupied by one server CTA) until the server idles out
  if (t->server && !served)
    return fail(ESPN_E_INVALID_STATE, "a persistent re-rank server runs on this table: only fused tcgen05 batches "
                                      "(final_k <= 32, the server's query precision) can be served; stop it first");
  if (served) {
    const int ss = server_ensure(t, s);
    if (ss) return ss;
  }
  // a launch of its own runs one batch alone: its last round is not hidden
  // behind the next batch's units as in the served queue, so shorter units
  // (C2: 46 -> 42 us per launch; served, the 96-doc units are 8% faster)
  if (tc && !served && layout_docs > kExclusiveUnitDocs) unit_docs = size_units(kExclusiveUnitDocs);
  // dedup hash of the separate top-k kernel, sized by the longest scored list
  // (part of the graph key: a captured launch bakes it in)
  uint32_t topk_hs = 64;
  while (topk_hs < 2 * max_list) topk_hs <<= 1;
  const int pslot = (int)(w->prof_calls % espn_gpu_workspace::kProf);
  if (profile) drain_prof(w, pslot);

  const bool sync_call = !(a->flags & ESPN_RERANK_ASYNC);
  // Outputs: device pointers (DEVICE_IO); pinned host buffers are written
  // directly by the kernels (zero-copy, no D2H); other host buffers get a
  // D2H from the workspace's output arrays.
  uint32_t* out_ids_k = w->out_ids;
  float* out_scores_k = w->out_scores;
  uint32_t* out_counts_k = w->out_counts;
  bool out_direct = dev_io;
  bool out_bounce = false;  // synchronous pageable outputs: compact [err | ids | scores | counts], one D2H
  if (dev_io) {
    out_ids_k = o->ids;
    out_scores_k = o->scores;
    out_counts_k = o->counts;
  } else {
    const void* key[3] = {o->ids, o->scores, o->counts};
    bool zc_ok = true;
    for (int i = 0; i < 3; ++i) zc_ok = w->ptrs.lookup(key[i], &w->zc_dev[i]) && w->zc_dev[i] && zc_ok;
    if (zc_ok) {
      out_ids_k = static_cast<uint32_t*>(w->zc_dev[0]);
      out_scores_k = static_cast<float*>(w->zc_dev[1]);
      out_counts_k = static_cast<uint32_t*>(w->zc_dev[2]);
      out_direct = true;
    } else if (sync_call && w->out_h) {
      out_bounce = true;
      out_ids_k = w->out_ids;  // == opack + 16
      out_scores_k = reinterpret_cast<float*>(w->out_ids + (size_t)B * k);
      out_counts_k = reinterpret_cast<uint32_t*>(out_scores_k + (size_t)B * k);
    }
  }
  // ---- inputs -> device ----
  const uint64_t* cand_off = a->cand_offsets;
  const uint32_t* needed_in = a->needed_counts;
  const float* q32 = a->query_tokens;
  const uint32_t* ids = a->cand_ids;
  const float* cls = a->cand_cls;
  // Host-staged inputs go through I/O slot io_slot on the workspace's copy
  // stream: the slot's previous batch must be done with it, and the compute
  // stream waits for the H2D -- batch n+1's copies overlap batch n's kernels.
  int io_slot = -1;
  if (!dev_io) {  // which caller buffers are pinned (cached per pointer)
    const void* key[3] = {q32, ids, cls};
    void* dummy = nullptr;
    for (int i = 0; i < 3; ++i) w->in_pinned[i] = w->ptrs.lookup(key[i], &dummy);
  }
  const bool all_pinned = !dev_io && w->in_pinned[0] && (C == 0 || (w->in_pinned[1] && w->in_pinned[2]));
  const bool packed = sync_call && !dev_io && !dev_off && !all_pinned;
  // per-shape CUDA graph of the packed synchronous path (everything the graph
  // bakes in is in the key; the data it reads lives in fixed pinned/device buffers)
  const bool graph_ok = packed && out_bounce && !t->tiered && !profile_dev && !o->bow_scores && !w->async_pending &&
                        !(a->flags & (ESPN_RERANK_WRITE_BOW | ESPN_RERANK_PREFETCHED)) && !(dbg & 0x40000u);
  uint32_t alpha_bits;
  std::memcpy(&alpha_bits, &a->alpha, 4);
  const uint64_t gkey[5] = {(uint64_t)B | ((uint64_t)nq << 32), C, (uint64_t)k | ((uint64_t)a->rerank_count << 32),
                            (uint64_t)alpha_bits | ((uint64_t)a->flags << 32),
                            (uint64_t)kern | ((uint64_t)fused << 8) | ((uint64_t)(a->needed_counts != nullptr) << 9) |
                                ((uint64_t)(uint32_t)unit_docs << 16) | ((uint64_t)__builtin_ctz(topk_hs) << 32) |
                                ((uint64_t)served << 40) |
                                ((uint64_t)(o->fetch_stats != nullptr) << 48)};
  const bool replay = graph_ok && w->sg_exec && std::equal(gkey, gkey + 5, w->sg_key);
  const bool capture = graph_ok && !replay && std::equal(gkey, gkey + 5, w->sg_seen);
  if (graph_ok && !replay && !capture) std::copy(gkey, gkey + 5, w->sg_seen);
  cudaStream_t user_s = s;
  if (w->capturing) {  // an earlier call failed inside its capture: close it, drop the graph
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(w->gs, &g);
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    w->capturing = false;
  }
  if (packed) {
    // synchronous call with pageable buffers: pack every input into the I/O
    // slot's pinned buffer and move it with ONE copy on the compute stream
    io_slot = graph_ok ? 0 : (int)(w->io_calls++ % 2);  // a graph always uses slot 0
    auto& io = w->io[io_slot];
    if (io.used) ESPN_CUDA_TRY(cudaEventSynchronize(io.done));  // an earlier batch is done with it
    auto a16 = [](size_t x) { return (x + 15) / 16 * 16; };
    const size_t qb = (size_t)B * nq * t->d * sizeof(float), ib = C * sizeof(uint32_t), cb = C * sizeof(float);
    const size_t o_need = a16((B + 1) * 8), o_q = o_need + a16(B * 4), o_ids = o_q + a16(qb),
                 o_cls = o_ids + a16(ib), total = o_cls + cb;
    std::memcpy(io.in_h, a->cand_offsets, (B + 1) * sizeof(uint64_t));
    if (a->needed_counts) std::memcpy(io.in_h + o_need, a->needed_counts, B * sizeof(uint32_t));
    std::memcpy(io.in_h + o_q, q32, qb);
    if (C) {
      std::memcpy(io.in_h + o_ids, ids, ib);
      std::memcpy(io.in_h + o_cls, cls, cb);
    }
    if (replay) {
      ESPN_CUDA_TRY(cudaGraphLaunch(w->sg_exec, s));
      ESPN_CUDA_TRY(cudaEventRecord(io.done, s));
      io.used = true;
      ESPN_CUDA_TRY(cudaStreamSynchronize(s));
      const size_t ob_ids = (size_t)B * k * sizeof(uint32_t), ob_sc = (size_t)B * k * sizeof(float);
      std::memcpy(w->h_err, w->out_h, sizeof(uint32_t));
      std::memcpy(o->ids, w->out_h + 16, ob_ids);
      std::memcpy(o->scores, w->out_h + 16 + ob_ids, ob_sc);
      std::memcpy(o->counts, w->out_h + 16 + ob_ids + ob_sc, (size_t)B * sizeof(uint32_t));
      if (*w->h_err) {
        ESPN_CUDA_TRY(cudaMemsetAsync(w->err, 0, sizeof(uint32_t), s));
        ESPN_CUDA_TRY(cudaStreamSynchronize(s));
      }
      if (o->fetch_stats)
        for (uint32_t b = 0; b < B; ++b) {  // HBM-resident table: every needed row is resident
          const uint64_t n = a->cand_offsets[b + 1] - a->cand_offsets[b];
          const uint64_t need = std::min<uint64_t>(n, a->needed_counts ? a->needed_counts[b] : a->rerank_count);
          o->fetch_stats[b] = espn_fetch_stats{need, need, 0, 0, 0, 0};
        }
      w->counters.batches += 1;
      w->counters.queries += B;
      w->counters.kernel_launches += small ? 1 : served ? 2 : 3;
      return err_bits_to_status(*w->h_err);
    }
    if (capture) {
      ESPN_CUDA_TRY(cudaStreamBeginCapture(w->gs, cudaStreamCaptureModeRelaxed));
      w->capturing = true;
      s = w->gs;
    }
    ESPN_CUDA_TRY(cudaMemcpyAsync(io.dpack, io.in_h, total, cudaMemcpyHostToDevice, s));
    cand_off = reinterpret_cast<const uint64_t*>(io.dpack);
    if (a->needed_counts) needed_in = reinterpret_cast<const uint32_t*>(io.dpack + o_need);
    q32 = reinterpret_cast<const float*>(io.dpack + o_q);
    ids = reinterpret_cast<const uint32_t*>(io.dpack + o_ids);
    cls = reinterpret_cast<const float*>(io.dpack + o_cls);
  } else if (!dev_off || !dev_io) {
    io_slot = (int)(w->io_calls++ % 2);
    auto& io = w->io[io_slot];
    if (io.used) ESPN_CUDA_TRY(cudaStreamWaitEvent(w->cs, io.done, 0));
    if (!dev_off) {
      // the small per-batch tables via a pinned ring slot (an ASYNC caller may
      // enqueue batch n+1 before batch n's H2D copies ran)
      auto& sl = w->slots[w->calls % espn_gpu_workspace::kSlots];
      if (sl.used) ESPN_CUDA_TRY(cudaEventSynchronize(sl.copied));
      std::memcpy(sl.cand_off, a->cand_offsets, (B + 1) * sizeof(uint64_t));
      ESPN_CUDA_TRY(cudaMemcpyAsync(io.cand_off, sl.cand_off, (B + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, w->cs));
      if (a->needed_counts) {
        std::memcpy(sl.needed, a->needed_counts, B * sizeof(uint32_t));
        ESPN_CUDA_TRY(cudaMemcpyAsync(io.needed_in, sl.needed, B * sizeof(uint32_t), cudaMemcpyHostToDevice, w->cs));
        needed_in = io.needed_in;
      }
      ESPN_CUDA_TRY(cudaEventRecord(sl.copied, w->cs));
      sl.used = true;
      ++w->calls;
      cand_off = io.cand_off;
    }
    if (!dev_io) {
      // pinned caller buffers are copied directly (truly async); pageable ones
      // are staged through the slot's pinned buffer first (a pageable
      // cudaMemcpyAsync is a synchronous driver copy per array)
      const size_t qb = (size_t)B * nq * t->d * sizeof(float), ib = C * sizeof(uint32_t), cb = C * sizeof(float);
      if (!(w->in_pinned[0] && w->in_pinned[1] && w->in_pinned[2]) && io.used)
        ESPN_CUDA_TRY(cudaEventSynchronize(io.in_ready));  // the slot's previous H2D has read in_h
      uint8_t* hq = io.in_h;
      uint8_t* hi = io.in_h + qb;
      uint8_t* hc = hi + ib;
      const void* srcq = w->in_pinned[0] ? (const void*)q32 : (std::memcpy(hq, q32, qb), (const void*)hq);
      ESPN_CUDA_TRY(cudaMemcpyAsync(io.q32, srcq, qb, cudaMemcpyHostToDevice, w->cs));
      if (C) {
        const void* srci = w->in_pinned[1] ? (const void*)ids : (std::memcpy(hi, ids, ib), (const void*)hi);
        const void* srcc = w->in_pinned[2] ? (const void*)cls : (std::memcpy(hc, cls, cb), (const void*)hc);
        ESPN_CUDA_TRY(cudaMemcpyAsync(io.ids, srci, ib, cudaMemcpyHostToDevice, w->cs));
        ESPN_CUDA_TRY(cudaMemcpyAsync(io.cls, srcc, cb, cudaMemcpyHostToDevice, w->cs));
      }
      q32 = io.q32;
      ids = io.ids;
      cls = io.cls;
    }
    ESPN_CUDA_TRY(cudaEventRecord(io.in_ready, w->cs));
    ESPN_CUDA_TRY(cudaStreamWaitEvent(s, io.in_ready, 0));
  }
  // the device error word is sticky across un-synced ASYNC batches; it is
  // read and cleared by the synchronising call (or espn_gpu_workspace_sync)

  // bow scores are defined for the needed prefix of each list only: the rest
  // of the returned array reads as 0 (not as the previous batch's values)
  if ((a->flags & ESPN_RERANK_WRITE_BOW) && o->bow_scores && C)
    ESPN_CUDA_TRY(cudaMemsetAsync(w->bow, 0, C * sizeof(float), s));
  // ---- MaxSim parameters (also the server's batch descriptor) ----
  MaxSimParams mp{};
  mp.rows = t->rows;
  mp.doc_loc = t->doc_loc;
  mp.cand_src = nullptr;  // tiered: set once the staging slot is known
  mp.row_ptr = t->row_ptr;
  mp.n_docs = t->n_docs;
  mp.shard_count = t->shard_count;
  mp.shard_index = t->shard_index;
  mp.q32 = q32;
  mp.cand_ids = ids;
  mp.cand_off = cand_off;
  mp.unit_off = w->unit_off;
  mp.unit_tab = w->unit_tab;
  mp.needed = w->needed;
  mp.bow_out = w->bow;
  mp.err = w->err;
  mp.n_queries = B;
  mp.nq = nq;
  mp.rerank_count = a->rerank_count;
  mp.unit_docs = (uint32_t)std::max(unit_docs, 1);
  mp.n_units = w->n_units;
  mp.bf16 = t->dtype == ESPN_DTYPE_BF16;
  mp.qround = (a->flags & ESPN_RERANK_QUERY_ROUNDED) ? 1u : 0u;
  mp.dbg = dbg;
  mp.prof = (profile_dev && tc && !served) ? w->kprof : nullptr;
  mp.done_flag = w->done_flag;
  if (fused) {
    mp.cand_cls = cls;
    mp.alpha = a->alpha;
    mp.k = k;
    mp.out_ids = out_ids_k;
    mp.out_scores = out_scores_k;
    mp.out_counts = out_counts_k;
    mp.unit_top = w->unit_top;
    mp.dedup = w->dedup;
    mp.ff_seen = w->ff_seen;
    mp.fused_state = w->fused_state;
    mp.hash_slots = w->hash_slots;
    mp.max_queries = w->max_queries;
  }
  int slot = -1;
  bool hint_consumed = false;
  if (small) {
    // ---- K5: the whole batch in one launch ----
    SmallParams sp{};
    sp.m = mp;
    sp.m.cand_cls = cls;
    sp.m.alpha = a->alpha;
    sp.m.k = k;
    sp.m.out_ids = out_ids_k;
    sp.m.out_scores = out_scores_k;
    sp.m.out_counts = out_counts_k;
    sp.m.unit_top = w->small_top;
    sp.m.prof = profile_dev ? w->kprof : nullptr;
    sp.needed_in = needed_in;
    sp.max_candidates = w->max_candidates;
    sp.partial = partial ? 1u : 0u;
    sp.P = small_P;
    sp.base_ok = (dev_off && (a->flags & kFlagBaseOffsets)) ? 1u : 0u;
    sp.arrive = w->small_arrive;
    sp.hash = w->small_hash;
    sp.ff_seen = w->small_ff;
    if (profile) ESPN_CUDA_TRY(cudaEventRecord(w->prof[pslot].e[0], s));
    const cudaError_t se = launch_small_rt(t->d, sp, B, s);
    if (se != cudaSuccess) return fail(ESPN_E_CUDA, std::string("small-batch launch: ") + cudaGetErrorString(se));
    if (profile) ESPN_CUDA_TRY(cudaEventRecord(w->prof[pslot].e[1], s));
  } else {
    // ---- K0: batch plan on the device ----
    PlanParams pp{};
    pp.cand_off = cand_off;
    pp.needed_in = needed_in;
    pp.needed = w->needed;
    pp.unit_off = w->unit_off;
    pp.unit_tab = w->unit_tab;
    pp.n_units = w->n_units;
    pp.err = w->err;
    pp.max_candidates = w->max_candidates;
    pp.max_units = tc ? w->max_units : ~0ull;
    pp.n_queries = B;
    pp.rerank_count = a->rerank_count;
    pp.unit_docs = tc ? (uint32_t)unit_docs : 1u;
    pp.write_tab = tc ? 1u : 0u;
    pp.tail_units = (fused && partial) ? 1u : 0u;
    pp.out_counts = fused ? out_counts_k : nullptr;
    pp.fused_state = fused ? w->fused_state : nullptr;
    pp.base_ok = (dev_off && (a->flags & kFlagBaseOffsets)) ? 1u : 0u;
    pp.dbg = dbg;
    ServerSubmit sb{};
    if (served) {
      sb.server = t->server;
      sb.plan_done = w->plan_done;
      sb.msp = mp;
    }
    if (served)
      plan_kernel<16><<<(B + kPlanThreads - 1) / kPlanThreads, kPlanThreads, 0, s>>>(pp, sb);
    else
      plan_kernel<1><<<(B + kPlanThreads - 1) / kPlanThreads, kPlanThreads, 0, s>>>(pp, sb);
    ESPN_CUDA_TRY(cudaGetLastError());

    // ---- tiered table: host-tier rows staged into HBM (prefetched or now) ----
    if (t->tiered) {
      if (a->flags & ESPN_RERANK_PREFETCHED) {
        if (w->pf_count == 0) return fail(ESPN_E_INVALID_STATE, "PREFETCHED batch without a pending espn_gpu_prefetch");
        slot = w->pf_q[0];
        w->pf_q[0] = w->pf_q[1];
        --w->pf_count;
        ESPN_CUDA_TRY(cudaStreamWaitEvent(s, w->stage[slot].done, 0));
        if (w->stage[slot].hint_epoch) {  // doc-keyed hints: resolve this batch's needed rows now
          hint_consumed = true;
          const int ss = launch_stage(t, w, slot, cand_off, needed_in, ids, B, a->rerank_count, s, false);
          w->stage[slot].hint_epoch = 0;
          if (ss) return ss;
        }
      } else {
        slot = take_free_slot(w);
        if (slot < 0) return fail(ESPN_E_INVALID_STATE, "both staging slots hold pending prefetches");
        const int ss = launch_stage(t, w, slot, cand_off, needed_in, ids, B, a->rerank_count, s, false);
        if (ss) return ss;
      }
    }

    mp.cand_src = slot >= 0 ? w->stage[slot].cand_src : nullptr;
    w->last_slot = slot;
    if (profile) ESPN_CUDA_TRY(cudaEventRecord(w->prof[pslot].e[0], s));
    cudaError_t e = served ? (server_wait_kernel<<<1, 32, 0, s>>>(w->done_flag, w->err, kServerWaitNs), cudaGetLastError())
                    : tc   ? launch_tc_rt(t->d, qsplit, mp, t->num_sms, s, /*pdl=*/slot < 0 && !profile)
                           : launch_simt_rt(t->d, mp, t->num_sms, s);
    if (e != cudaSuccess) return fail(ESPN_E_CUDA, std::string("MaxSim launch: ") + cudaGetErrorString(e));
    if (slot >= 0) {  // the slot may be re-staged once this MaxSim finished
      ESPN_CUDA_TRY(cudaEventRecord(w->stage[slot].free_ev, s));
      w->stage[slot].used = true;
    }
    if (profile) ESPN_CUDA_TRY(cudaEventRecord(w->prof[pslot].e[1], s));

    if (fused && !served) {  // (served: the server's dedup warps merged the lists)
      // ---- K3': merge of the per-unit top-k lists (programmatic dependent) ----
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3((B + kFinalizeWarps - 1) / kFinalizeWarps);
      lc.blockDim = dim3(kFinalizeWarps * 32);
      lc.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = (dbg & 0x10000u) ? 1 : 0;  // plain launch: as a programmatic dependent its CTAs
                                               // crowd onto the first SMs MaxSim frees
      ESPN_CUDA_TRY(cudaLaunchKernelEx(&lc, finalize_kernel, mp));
    }

    // ---- K3: aggregate + top-k (unless fused into MaxSim) ----
    if (!fused) {
    ESPN_CUDA_TRY(ensure_topk_attr());
    TopKParams tp{};
    tp.bow = w->bow;
    tp.cand_ids = ids;
    tp.cand_cls = cls;
    tp.cand_off = cand_off;
    tp.needed = w->needed;
    tp.out_ids = out_ids_k;
    tp.out_scores = out_scores_k;
    tp.out_counts = out_counts_k;
    tp.err = w->err;
    tp.n_queries = B;
    tp.rerank_count = a->rerank_count;
    tp.k = k;
    tp.partial = partial ? 1u : 0u;
    tp.alpha = a->alpha;
    tp.dbg = dbg;
    {
      // CTA-per-query fast path when final_k <= 32 and the dedup hash fits;
      // launched as a programmatic dependent of MaxSim (its id-only dedup
      // prologue overlaps the MaxSim tail)
      const uint32_t hs = topk_hs;
      if (k <= 32 && hs <= 8192) {
        const size_t smem = (size_t)hs * 8 + 8 * 32 * 8;
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(B);
        lc.blockDim = dim3(kTopkCtaThreads);
        lc.dynamicSmemBytes = smem;
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        ESPN_CUDA_TRY(k <= 16 ? cudaLaunchKernelEx(&lc, topk_cta_kernel<16>, tp, hs)
                              : cudaLaunchKernelEx(&lc, topk_cta_kernel<32>, tp, hs));
      } else {
        topk_kernel<<<B, kTopkThreads, topk_smem_bytes(), s>>>(tp);
        ESPN_CUDA_TRY(cudaGetLastError());
      }
    }
    }
  }
  if (profile) {
    ESPN_CUDA_TRY(cudaEventRecord(w->prof[pslot].e[2], s));
    w->prof[pslot].pending = true;
    ++w->prof_calls;
  }

  if (io_slot >= 0 && !capture) {  // every kernel reading the I/O slot is enqueued
    ESPN_CUDA_TRY(cudaEventRecord(w->io[io_slot].done, s));
    w->io[io_slot].used = true;
  }
  // pageable host outputs of a synchronous call: the compact output pack
  // (error word included) comes back with ONE copy into the pinned bounce and
  // is copied out after the sync below (ASYNC callers get direct copies)
  const size_t ob_ids = (size_t)B * k * sizeof(uint32_t), ob_sc = (size_t)B * k * sizeof(float);
  if (out_bounce) {
    ESPN_CUDA_TRY(cudaMemcpyAsync(w->out_h, w->opack, 16 + ob_ids + ob_sc + (size_t)B * sizeof(uint32_t),
                                  cudaMemcpyDeviceToHost, s));
  } else if (!out_direct) {
    ESPN_CUDA_TRY(cudaMemcpyAsync(o->ids, w->out_ids, ob_ids, cudaMemcpyDeviceToHost, s));
    ESPN_CUDA_TRY(cudaMemcpyAsync(o->scores, w->out_scores, ob_sc, cudaMemcpyDeviceToHost, s));
    ESPN_CUDA_TRY(cudaMemcpyAsync(o->counts, w->out_counts, (size_t)B * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  }
  if ((a->flags & ESPN_RERANK_WRITE_BOW) && o->bow_scores) {
    if (dev_off) return fail(ESPN_E_INVALID_INPUT, "WRITE_BOW needs host cand_offsets (total size)");
    if (C)
      ESPN_CUDA_TRY(cudaMemcpyAsync(o->bow_scores, w->bow, C * sizeof(float),
                                    dev_io ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
  }
  w->counters.batches += 1;
  w->counters.queries += B;
  w->counters.kernel_launches += small ? 1 : (served ? 2 : 3) + (t->tiered && (!(a->flags & ESPN_RERANK_PREFETCHED) || hint_consumed) ? 1 : 0);
  if (a->flags & ESPN_RERANK_ASYNC) {
    w->async_pending = true;
    return ESPN_OK;
  }
  if (capture) {  // the graph now holds this call's work: instantiate, then run it on the caller's stream
    cudaGraph_t graph = nullptr;
    w->capturing = false;
    ESPN_CUDA_TRY(cudaStreamEndCapture(w->gs, &graph));
    if (w->sg_exec) {
      cudaGraphExecDestroy(w->sg_exec);
      w->sg_exec = nullptr;
    }
    const cudaError_t ge = cudaGraphInstantiate(&w->sg_exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ge != cudaSuccess) return fail(ESPN_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ge));
    std::copy(gkey, gkey + 5, w->sg_key);
    s = user_s;
    if (served) {  // instantiation may have waited for an idle server to exit
      const int ss = server_ensure(t, s);
      if (ss) return ss;
    }
    ESPN_CUDA_TRY(cudaGraphLaunch(w->sg_exec, s));
    // (an event recorded during capture is only a capture dependency: record
    // the slot's completion on the caller's stream, after the graph)
    ESPN_CUDA_TRY(cudaEventRecord(w->io[io_slot].done, s));
    w->io[io_slot].used = true;
  }
  if (!out_bounce) ESPN_CUDA_TRY(cudaMemcpyAsync(w->h_err, w->err, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  if (o->fetch_stats && slot >= 0)
    ESPN_CUDA_TRY(cudaMemcpyAsync(w->h_qstats, w->stage[slot].qstats, (size_t)B * 6 * sizeof(unsigned long long),
                                  cudaMemcpyDeviceToHost, s));
  ESPN_CUDA_TRY(cudaStreamSynchronize(s));
  if (out_bounce) {
    std::memcpy(w->h_err, w->out_h, sizeof(uint32_t));
    std::memcpy(o->ids, w->out_h + 16, ob_ids);
    std::memcpy(o->scores, w->out_h + 16 + ob_ids, ob_sc);
    std::memcpy(o->counts, w->out_h + 16 + ob_ids + ob_sc, (size_t)B * sizeof(uint32_t));
  }
  if (*w->h_err) ESPN_CUDA_TRY(cudaMemsetAsync(w->err, 0, sizeof(uint32_t), s));
  w->async_pending = false;
  if (o->fetch_stats) {
    for (uint32_t b = 0; b < B; ++b) {
      espn_fetch_stats& f = o->fetch_stats[b];
      if (slot >= 0) {
        const unsigned long long* q = w->h_qstats + (size_t)b * 6;
        f = espn_fetch_stats{q[0], q[1], q[2], q[3], q[4], q[5]};
      } else if (!dev_off) {  // HBM-resident table: every needed row is resident
        const uint64_t n = a->cand_offsets[b + 1] - a->cand_offsets[b];
        const uint64_t need = std::min<uint64_t>(n, a->needed_counts ? a->needed_counts[b] : a->rerank_count);
        f = espn_fetch_stats{need, need, 0, 0, 0, 0};
      } else {
        f = espn_fetch_stats{};
      }
    }
  }
  return err_bits_to_status(*w->h_err);
}

int espn_gpu_prefetch(espn_gpu_table* t, espn_gpu_workspace* w, const espn_rerank_args* a, void* side_stream) {
  if (!t || !w || !a) return fail(ESPN_E_INVALID_INPUT, "null argument");
  if (w->table != t) return fail(ESPN_E_INVALID_STATE, "workspace belongs to another table");
  if (const int ls = require_loaded(t)) return ls;
  if (!t->tiered) return ESPN_OK;  // everything is HBM-resident
  if (!(a->flags & ESPN_RERANK_DEVICE_IO)) return fail(ESPN_E_INVALID_INPUT, "prefetch needs DEVICE_IO batch arrays");
  const uint32_t B = a->n_queries;
  if (B == 0) return ESPN_OK;
  if (B > w->max_queries) return fail(ESPN_E_INVALID_INPUT, "n_queries exceeds workspace capacity");
  if (w->pf_count == 2) return fail(ESPN_E_INVALID_STATE, "both staging slots hold pending prefetches");
  DeviceGuard g(t->device);
  cudaStream_t s = static_cast<cudaStream_t>(side_stream);
  const int slot = take_free_slot(w);
  auto& st = w->stage[slot];
  const uint64_t* off = a->cand_offsets;
  const uint32_t* need = a->needed_counts;
  if (!(a->flags & ESPN_RERANK_DEVICE_OFFSETS)) {
    if (a->cand_offsets[0] != 0) return fail(ESPN_E_INVALID_INPUT, "cand_offsets[0] must be 0");
    for (uint32_t b = 0; b < B; ++b)
      if (a->cand_offsets[b + 1] < a->cand_offsets[b]) return fail(ESPN_E_INVALID_INPUT, "cand_offsets must be non-decreasing");
    if (a->cand_offsets[B] > w->max_candidates) return fail(ESPN_E_INVALID_INPUT, "candidates exceed workspace capacity");
    if (st.used) ESPN_CUDA_TRY(cudaEventSynchronize(st.done));  // pinned staging of this slot is free
    std::memcpy(st.off_h, a->cand_offsets, (B + 1) * sizeof(uint64_t));
    ESPN_CUDA_TRY(cudaMemcpyAsync(st.off, st.off_h, (B + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    off = st.off;
    if (a->needed_counts) {
      std::memcpy(st.need_h, a->needed_counts, B * sizeof(uint32_t));
      ESPN_CUDA_TRY(cudaMemcpyAsync(st.need, st.need_h, B * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
      need = st.need;
    }
  }
  st.hint_epoch = 0;  // positional staging
  const int ss = launch_stage(t, w, slot, off, need, a->cand_ids, B, a->rerank_count, s, true);
  if (ss) return ss;
  w->pf_q[w->pf_count++] = slot;
  w->async_pending = true;  // staging errors surface at the next sync
  return ESPN_OK;
}

namespace {
// Doc-keyed staging of one hint batch into a free staging slot (the body of
// espn_gpu_prefetch_hints and espn_gpu_prefetch_rows).  ext_rows != NULL:
// the rows come from the caller (plain codes, hint j's doc at byte
// ext_off[j] of ext_rows, ext_bytes in all) instead of the host tier.
int prefetch_hint_impl(espn_gpu_table* t, espn_gpu_workspace* w, uint32_t B, const uint32_t* hint_ids,
                       const uint64_t* hint_offsets, uint32_t flags, void* side_stream, const void* ext_rows,
                       const uint64_t* ext_off, uint64_t ext_bytes) {
  if (!t || !w) return fail(ESPN_E_INVALID_INPUT, "null argument");
  if (w->table != t) return fail(ESPN_E_INVALID_STATE, "workspace belongs to another table");
  if (const int ls = require_loaded(t)) return ls;
  if (!t->tiered) return ESPN_OK;  // everything is HBM-resident
  if (B == 0) return ESPN_OK;
  if (!hint_offsets) return fail(ESPN_E_INVALID_INPUT, "null hint offsets");
  if (B > w->max_queries) return fail(ESPN_E_INVALID_INPUT, "n_queries exceeds workspace capacity");
  if (w->pf_count == 2) return fail(ESPN_E_INVALID_STATE, "both staging slots hold pending prefetches");
  DeviceGuard g(t->device);
  cudaStream_t s = static_cast<cudaStream_t>(side_stream);
  const int slot = peek_free_slot(w);
  auto& st = w->stage[slot];
  const uint64_t* off = hint_offsets;
  const bool dev_ids = (flags & ESPN_RERANK_DEVICE_IO) != 0;
  if ((flags & ESPN_RERANK_DEVICE_OFFSETS) && !dev_ids)
    return fail(ESPN_E_INVALID_INPUT, "DEVICE_OFFSETS hints need DEVICE_IO ids");
  if (!(flags & ESPN_RERANK_DEVICE_OFFSETS)) {
    if (hint_offsets[0] != 0) return fail(ESPN_E_INVALID_INPUT, "hint_offsets[0] must be 0");
    for (uint32_t b = 0; b < B; ++b)
      if (hint_offsets[b + 1] < hint_offsets[b]) return fail(ESPN_E_INVALID_INPUT, "hint_offsets must be non-decreasing");
    if (hint_offsets[B] > w->max_candidates) return fail(ESPN_E_INVALID_INPUT, "hints exceed workspace capacity");
    if (hint_offsets[B] && !hint_ids) return fail(ESPN_E_INVALID_INPUT, "null hint ids");
    if (st.used) ESPN_CUDA_TRY(cudaEventSynchronize(st.done));  // pinned staging of this slot is free
    std::memcpy(st.off_h, hint_offsets, (B + 1) * sizeof(uint64_t));
    ESPN_CUDA_TRY(cudaMemcpyAsync(st.off, st.off_h, (B + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    off = st.off;
    if (!dev_ids && hint_offsets[B]) {  // host ids: through this slot's pinned staging
      if (!st.hint_ids) {
        ESPN_CUDA_TRY(cudaMalloc(&st.hint_ids, w->max_candidates * sizeof(uint32_t)));
        ESPN_CUDA_TRY(cudaMallocHost(&st.hint_ids_h, w->max_candidates * sizeof(uint32_t)));
      }
      std::memcpy(st.hint_ids_h, hint_ids, hint_offsets[B] * sizeof(uint32_t));
      ESPN_CUDA_TRY(cudaMemcpyAsync(st.hint_ids, st.hint_ids_h, hint_offsets[B] * sizeof(uint32_t),
                                    cudaMemcpyHostToDevice, s));
      hint_ids = st.hint_ids;
    }
  }
  if (!w->hint_map) {
    ESPN_CUDA_TRY(cudaMalloc(&w->hint_map, t->n_docs * sizeof(uint64_t)));
    ESPN_CUDA_TRY(cudaMemsetAsync(w->hint_map, 0, t->n_docs * sizeof(uint64_t), s));
  }
  if (++w->hint_epoch == 0) {  // 2^32 hint batches: reset the map so no stale entry can match
    ESPN_CUDA_TRY(cudaMemsetAsync(w->hint_map, 0, t->n_docs * sizeof(uint64_t), s));
    w->hint_epoch = 1;
  }
  w->next_slot = slot ^ 1;
  if (st.used) ESPN_CUDA_TRY(cudaStreamWaitEvent(s, st.free_ev, 0));  // previous reader done
  ESPN_CUDA_TRY(cudaMemsetAsync(st.cursor, 0, sizeof(unsigned long long), s));
  ESPN_CUDA_TRY(cudaMemsetAsync(st.qstats, 0, (size_t)B * 6 * sizeof(unsigned long long), s));
  HintParams hp{};
  if (ext_rows) {  // the caller's rows and their offsets -> this slot's device buffers
    const uint64_t nh = hint_offsets[B];
    if (!st.ext_off) {
      ESPN_CUDA_TRY(cudaMalloc(&st.ext_off, w->max_candidates * sizeof(uint64_t)));
      ESPN_CUDA_TRY(cudaMallocHost(&st.ext_off_h, w->max_candidates * sizeof(uint64_t)));
    }
    if (st.ext_cap < ext_bytes) {
      ESPN_CUDA_TRY(cudaStreamSynchronize(s));
      cudaFree(st.ext_buf);
      st.ext_buf = nullptr;
      st.ext_cap = 0;
      ESPN_CUDA_TRY(cudaMalloc(&st.ext_buf, ext_bytes));
      st.ext_cap = ext_bytes;
    }
    std::memcpy(st.ext_off_h, ext_off, nh * sizeof(uint64_t));
    ESPN_CUDA_TRY(cudaMemcpyAsync(st.ext_off, st.ext_off_h, nh * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    ESPN_CUDA_TRY(cudaMemcpyAsync(st.ext_buf, ext_rows, ext_bytes, cudaMemcpyHostToDevice, s));
    hp.ext_src = st.ext_buf;
    hp.ext_off = st.ext_off;
  }
  hp.d = t->d;
  hp.row_ptr = t->row_ptr;
  hp.doc_loc = t->doc_loc;
  hp.n_docs = t->n_docs;
  hp.shard_count = t->shard_count;
  hp.shard_index = t->shard_index;
  hp.hint_ids = hint_ids;
  hp.hint_off = off;
  hp.max_hints = w->max_candidates;
  hp.row_bytes = t->d * 2;
  hp.hint_map = w->hint_map;
  hp.epoch = w->hint_epoch;
  hp.stage = st.buf;
  // host-tier hints keep half of the slot for the critical-path misses; rows
  // handed over by the caller may fill it (a disk-tier doc has no fallback)
  hp.stage_cap = ext_rows ? w->staging_bytes : w->staging_bytes / 2;
  hp.cursor = st.cursor;
  hp.qstats = st.qstats;
  hp.err = w->err;
  hint_stage_kernel<<<B, kStageThreads, 0, s>>>(hp);
  ESPN_CUDA_TRY(cudaGetLastError());
  ESPN_CUDA_TRY(cudaEventRecord(st.done, s));
  st.hint_epoch = w->hint_epoch;
  w->pf_q[w->pf_count++] = slot;
  w->async_pending = true;
  w->counters.kernel_launches += 1;
  return ESPN_OK;
}
}  // namespace

int espn_gpu_prefetch_hints(espn_gpu_table* t, espn_gpu_workspace* w, uint32_t B, const uint32_t* hint_ids,
                            const uint64_t* hint_offsets, uint32_t flags, void* side_stream) {
  return prefetch_hint_impl(t, w, B, hint_ids, hint_offsets, flags, side_stream, nullptr, nullptr, 0);
}

int espn_gpu_prefetch_rows(espn_gpu_table* t, espn_gpu_workspace* w, uint32_t B, const uint32_t* ids,
                           const uint64_t* id_offsets, const void* rows, const uint64_t* row_byte_off,
                           uint64_t rows_bytes, void* side_stream) {
  if (!t || !w) return fail(ESPN_E_INVALID_INPUT, "null argument");
  if (w->table != t) return fail(ESPN_E_INVALID_STATE, "workspace belongs to another table");
  if (const int ls = require_loaded(t)) return ls;
  if (!t->tiered) return ESPN_OK;  // everything is HBM-resident
  if (B == 0) return ESPN_OK;
  if (!id_offsets) return fail(ESPN_E_INVALID_INPUT, "null id offsets");
  if (t->h_row_ptr.empty()) return fail(ESPN_E_INVALID_STATE, "espn_gpu_prefetch_rows needs a streamed tiered table");
  if (B > w->max_queries) return fail(ESPN_E_INVALID_INPUT, "n_queries exceeds workspace capacity");
  if (id_offsets[0] != 0) return fail(ESPN_E_INVALID_INPUT, "id_offsets[0] must be 0");
  for (uint32_t b = 0; b < B; ++b)
    if (id_offsets[b + 1] < id_offsets[b]) return fail(ESPN_E_INVALID_INPUT, "id_offsets must be non-decreasing");
  const uint64_t nh = id_offsets[B];
  if (nh > w->max_candidates) return fail(ESPN_E_INVALID_INPUT, "ids exceed workspace capacity");
  if (nh == 0) return prefetch_hint_impl(t, w, B, ids, id_offsets, 0, side_stream, nullptr, nullptr, 0);
  if (!ids || !rows || !row_byte_off) return fail(ESPN_E_INVALID_INPUT, "null ids / rows / row offsets");
  // every doc's rows must lie inside the buffer, 16-byte aligned (the copy
  // reads whole 16-byte chunks); unknown ids and other shards' ids are
  // ignored like hints
  const uint64_t rowb = (uint64_t)t->d * 2;
  uint64_t total = 0;
  for (uint64_t j = 0; j < nh; ++j) {
    if (row_byte_off[j] % 16) return fail(ESPN_E_INVALID_INPUT, "row_byte_off must be 16-byte aligned");
    const uint32_t id = ids[j];
    uint64_t loc = id;
    if (t->shard_count > 1) {
      if (id % t->shard_count != t->shard_index) continue;
      loc = id / t->shard_count;
    }
    if (loc >= t->n_docs) continue;
    const uint64_t bytes = (t->h_row_ptr.size() > loc + 1 ? t->h_row_ptr[loc + 1] - t->h_row_ptr[loc] : 0) * rowb;
    if (row_byte_off[j] + bytes > rows_bytes) return fail(ESPN_E_INVALID_INPUT, "a doc's rows run past rows_bytes");
    total += bytes;
  }
  if (total > w->staging_bytes)
    return fail(ESPN_E_INVALID_CONFIG, "the handed-over rows (" + std::to_string(total) + " B) exceed the workspace's "
                                       "staging slot (" + std::to_string(w->staging_bytes) + " B): raise staging_bytes");
  return prefetch_hint_impl(t, w, B, ids, id_offsets, 0, side_stream, rows, row_byte_off, rows_bytes);
}

int espn_gpu_workspace_cand_status(espn_gpu_workspace* w, uint8_t* out, uint64_t n) {
  if (!w || (n && !out)) return fail(ESPN_E_INVALID_INPUT, "null argument");
  if (n > w->max_candidates) return fail(ESPN_E_INVALID_INPUT, "n exceeds the workspace's candidates");
  if (!w->table->tiered || w->last_slot < 0) {  // every row was in HBM
    std::memset(out, 0, n);
    return ESPN_OK;
  }
  DeviceGuard g(w->table->device);
  cudaStream_t cs = nullptr;
  ESPN_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  ESPN_CUDA_TRY(cudaMemcpyAsync(out, w->stage[w->last_slot].cand_status, n, cudaMemcpyDeviceToHost, cs));
  ESPN_CUDA_TRY(cudaStreamSynchronize(cs));
  cudaStreamDestroy(cs);
  return ESPN_OK;
}

int espn_gpu_workspace_sync(espn_gpu_workspace* w, void* stream_v) {
  if (!w) return fail(ESPN_E_INVALID_INPUT, "null argument");
  DeviceGuard g(w->table->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream_v);
  ESPN_CUDA_TRY(cudaMemcpyAsync(w->h_err, w->err, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  ESPN_CUDA_TRY(cudaStreamSynchronize(s));
  ESPN_CUDA_TRY(cudaMemsetAsync(w->err, 0, sizeof(uint32_t), s));
  w->async_pending = false;
  return err_bits_to_status(*w->h_err);
}

int espn_gpu_gather(espn_gpu_table* t, const uint32_t* ids, uint64_t n, uint16_t* out_rows,
                    uint64_t* out_row_ptr, uint64_t capacity_tokens, void* stream_v) {
  if (!t) return fail(ESPN_E_INVALID_INPUT, "null table");
  if (const int ls = require_loaded(t)) return ls;
  if (t->disk_tier) return fail(ESPN_E_INVALID_STATE, kDiskGather);
  if (n == 0) {
    if (out_row_ptr) {
      uint64_t z = 0;
      ESPN_CUDA_TRY(cudaMemcpyAsync(out_row_ptr, &z, sizeof z, cudaMemcpyHostToDevice,
                                    static_cast<cudaStream_t>(stream_v)));
      ESPN_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_v)));
    }
    return ESPN_OK;
  }
  if (!ids || !out_row_ptr) return fail(ESPN_E_INVALID_INPUT, "null argument");
  DeviceGuard g(t->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream_v);
  // per-thread, per-device scratch (error flag + pinned readback + CUB scan
  // temp), grown on demand: no allocation on the steady-state call path
  struct GatherScratch {
    int device = -1;
    uint32_t* err = nullptr;
    uint64_t* h = nullptr;  // pinned: {err, total}
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    ~GatherScratch() { if (err) { cudaFree(err); cudaFree(tmp); cudaFreeHost(h); } }
  };
  thread_local GatherScratch gs;
  if (gs.device != t->device) {
    if (gs.err) { cudaFree(gs.err); cudaFree(gs.tmp); cudaFreeHost(gs.h); }
    gs = GatherScratch{};
    ESPN_CUDA_TRY(cudaMalloc(&gs.err, sizeof(uint32_t)));
    ESPN_CUDA_TRY(cudaMallocHost(&gs.h, 2 * sizeof(uint64_t)));
    gs.device = t->device;
  }
  size_t need = 0;
  ESPN_CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, need, out_row_ptr + 1, out_row_ptr + 1, (int64_t)n, s));
  if (need > gs.tmp_bytes) {
    cudaFree(gs.tmp);
    gs.tmp = nullptr;
    gs.tmp_bytes = 0;
    ESPN_CUDA_TRY(cudaMalloc(&gs.tmp, need));
    gs.tmp_bytes = need;
  }
  ESPN_CUDA_TRY(cudaMemsetAsync(gs.err, 0, sizeof(uint32_t), s));
  ESPN_CUDA_TRY(cudaMemsetAsync(out_row_ptr, 0, sizeof(uint64_t), s));
  const int blocks = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)t->num_sms * 8);
  gather_count_kernel<<<blocks, 256, 0, s>>>(t->row_ptr, t->n_docs, t->shard_count, t->shard_index, ids, n, out_row_ptr, gs.err);
  ESPN_CUDA_TRY(cub::DeviceScan::InclusiveSum(gs.tmp, need, out_row_ptr + 1, out_row_ptr + 1, (int64_t)n, s));
  ESPN_CUDA_TRY(cudaMemcpyAsync(gs.h, gs.err, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  ESPN_CUDA_TRY(cudaMemcpyAsync(gs.h + 1, out_row_ptr + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  ESPN_CUDA_TRY(cudaStreamSynchronize(s));
  const uint32_t herr = (uint32_t)(gs.h[0] & 0xffffffffu);
  const uint64_t total = gs.h[1];
  if (herr) {
    g_last_error = "unknown doc id in gather request (store.hpp:92-93)";
    return ESPN_E_INVALID_INPUT;
  }
  if (!out_rows) return ESPN_OK;  // offsets only
  if (total > capacity_tokens) return fail(ESPN_E_INVALID_INPUT, "out_rows capacity too small");
  const int cb = t->num_sms * 8;
  switch (t->d) {
#define ESPN_G(DD) case DD: gather_copy_kernel<DD><<<cb, 256, 0, s>>>(t->rows, t->doc_loc, t->row_ptr, t->n_docs, t->shard_count, t->shard_index, ids, n, out_row_ptr, out_rows); break;
    ESPN_G(8) ESPN_G(16) ESPN_G(32) ESPN_G(48) ESPN_G(64) ESPN_G(96) ESPN_G(128) ESPN_G(256)
#undef ESPN_G
    default: return fail(ESPN_E_INVALID_CONFIG, "gather supports d in {8,16,32,48,64,96,128,256}");
  }
  ESPN_CUDA_TRY(cudaGetLastError());
  ESPN_CUDA_TRY(cudaStreamSynchronize(s));
  return ESPN_OK;
}

int espn_gpu_gather_host(espn_gpu_table* t, const uint32_t* ids, uint64_t n, uint16_t* out_rows,
                         uint64_t* out_row_ptr, uint64_t capacity_tokens) {
  if (!t) return fail(ESPN_E_INVALID_INPUT, "null table");
  if (!out_row_ptr) return fail(ESPN_E_INVALID_INPUT, "null argument");
  out_row_ptr[0] = 0;
  if (n == 0) return ESPN_OK;
  if (!ids) return fail(ESPN_E_INVALID_INPUT, "null argument");
  DeviceGuard g(t->device);
  uint32_t* d_ids = nullptr;
  uint64_t* d_rp = nullptr;
  uint16_t* d_rows = nullptr;
  auto cleanup = [&] { cudaFree(d_ids); cudaFree(d_rp); cudaFree(d_rows); };
  if (cudaMalloc(&d_ids, n * sizeof(uint32_t)) != cudaSuccess ||
      cudaMalloc(&d_rp, (n + 1) * sizeof(uint64_t)) != cudaSuccess) {
    cleanup();
    return fail(ESPN_E_CUDA, "cudaMalloc failed (gather)");
  }
  cudaMemcpy(d_ids, ids, n * sizeof(uint32_t), cudaMemcpyHostToDevice);
  int st = espn_gpu_gather(t, d_ids, n, nullptr, d_rp, 0, nullptr);
  if (st) { cleanup(); return st; }
  cudaMemcpy(out_row_ptr, d_rp, (n + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost);
  const uint64_t total = out_row_ptr[n];
  if (!out_rows) { cleanup(); return ESPN_OK; }
  if (total > capacity_tokens) { cleanup(); return fail(ESPN_E_INVALID_INPUT, "out_rows capacity too small"); }
  if (cudaMalloc(&d_rows, std::max<uint64_t>(total * t->d, 1) * sizeof(uint16_t)) != cudaSuccess) {
    cleanup();
    return fail(ESPN_E_CUDA, "cudaMalloc failed (gather rows)");
  }
  st = espn_gpu_gather(t, d_ids, n, d_rows, d_rp, total, nullptr);
  if (st == ESPN_OK) {
    const cudaError_t e = cudaMemcpy(out_rows, d_rows, total * t->d * sizeof(uint16_t), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) st = fail(ESPN_E_CUDA, cudaGetErrorString(e));
  }
  cleanup();
  return st;
}

int espn_gpu_merge_topk(const uint32_t* ids, const float* scores, const uint32_t* counts,
                        uint32_t n_lists, uint64_t list_stride, uint32_t n_queries, uint32_t k,
                        uint32_t* out_ids, float* out_scores, uint32_t* out_counts, void* stream_v) {
  if (k < 1 || k > (uint32_t)kMaxK) return fail(ESPN_E_INVALID_INPUT, "k must be in [1, 1024]");
  if (n_queries == 0) return ESPN_OK;
  if (!ids || !scores || !counts || !out_ids || !out_scores || !out_counts)
    return fail(ESPN_E_INVALID_INPUT, "null argument");
  if (n_lists > 1 && list_stride < (uint64_t)n_queries * k)
    return fail(ESPN_E_INVALID_INPUT, "list_stride smaller than one list");
  ESPN_CUDA_TRY(ensure_topk_attr());
  merge_topk_kernel<<<n_queries, kTopkThreads, topk_smem_bytes(), static_cast<cudaStream_t>(stream_v)>>>(
      ids, scores, counts, n_lists, list_stride, n_queries, k, out_ids, out_scores, out_counts);
  ESPN_CUDA_TRY(cudaGetLastError());
  return ESPN_OK;
}

int espn_gpu_gather_rows(espn_gpu_table* t, const uint32_t* ids, uint64_t n, const uint64_t* out_row_ptr,
                         uint16_t* out_rows, void* stream_v) {
  if (!t) return fail(ESPN_E_INVALID_INPUT, "null table");
  if (const int ls = require_loaded(t)) return ls;
  if (t->disk_tier) return fail(ESPN_E_INVALID_STATE, kDiskGather);
  if (n == 0) return ESPN_OK;
  if (!ids || !out_row_ptr || !out_rows) return fail(ESPN_E_INVALID_INPUT, "null argument");
  DeviceGuard g(t->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream_v);
  const int cb = t->num_sms * 8;
  switch (t->d) {
#define ESPN_G(DD) case DD: gather_copy_kernel<DD><<<cb, 256, 0, s>>>(t->rows, t->doc_loc, t->row_ptr, t->n_docs, t->shard_count, t->shard_index, ids, n, out_row_ptr, out_rows); break;
    ESPN_G(8) ESPN_G(16) ESPN_G(32) ESPN_G(48) ESPN_G(64) ESPN_G(96) ESPN_G(128) ESPN_G(256)
#undef ESPN_G
    default: return fail(ESPN_E_INVALID_CONFIG, "gather supports d in {8,16,32,48,64,96,128,256}");
  }
  ESPN_CUDA_TRY(cudaGetLastError());
  return ESPN_OK;
}

int espn_gpu_debug_timeline(int device, uint64_t* out8, int reset) {
  DeviceGuard g(device);
  if (out8) {
    ESPN_CUDA_TRY(cudaDeviceSynchronize());
    ESPN_CUDA_TRY(cudaMemcpyFromSymbol(out8, espn_k::g_ktl, 8 * sizeof(uint64_t)));
    if (reset == 2) ESPN_CUDA_TRY(cudaMemcpyFromSymbol(out8 + 8, espn_k::g_cta_prof, 4 * 256 * sizeof(uint64_t)));
    if (reset == 3) ESPN_CUDA_TRY(cudaMemcpyFromSymbol(out8 + 8, espn_k::g_fin, 8 * sizeof(uint64_t)));
  }
  if (reset) {
    unsigned long long init[8];
    for (int i = 0; i < 8; ++i) init[i] = (i & 1) || i >= 6 ? 0ull : ~0ull;
    ESPN_CUDA_TRY(cudaMemcpyToSymbol(espn_k::g_ktl, init, sizeof init));
    static unsigned long long zero[4 * 256] = {};
    ESPN_CUDA_TRY(cudaMemcpyToSymbol(espn_k::g_cta_prof, zero, sizeof zero));
    ESPN_CUDA_TRY(cudaMemcpyToSymbol(espn_k::g_fin, zero, 8 * sizeof(uint64_t)));
  }
  return ESPN_OK;
}

int espn_gpu_get_counters(const espn_gpu_workspace* w, espn_counters* out) {
  if (!w || !out) return fail(ESPN_E_INVALID_INPUT, "null argument");
  auto* wm = const_cast<espn_gpu_workspace*>(w);
  for (int i = 0; i < espn_gpu_workspace::kProf; ++i) drain_prof(wm, i);
  *out = w->counters;
  unsigned long long kp[2] = {0, 0};
  {
    DeviceGuard g(w->table->device);
    // (not while a persistent server runs: a device-wide sync would wait for it)
    if (!espn_gpu_server_running(w->table)) ESPN_CUDA_TRY(cudaDeviceSynchronize());
    ESPN_CUDA_TRY(cudaMemcpy(kp, w->kprof, sizeof kp, cudaMemcpyDeviceToHost));
  }
  out->maxsim_device_ns = kp[0];
  out->maxsim_device_launches = kp[1];
  return ESPN_OK;
}

int espn_gpu_synth_table(uint64_t n_docs, uint32_t d, uint32_t dtype, uint32_t t_min, uint32_t t_max,
                         uint64_t seed, uint32_t shard_count, uint32_t shard_index, uint64_t* row_ptr,
                         uint16_t* rows, void* stream_v) {
  if (n_docs == 0 || t_min < 1 || t_max < t_min) return fail(ESPN_E_INVALID_INPUT, "bad synth shape");
  if (!row_ptr) return fail(ESPN_E_INVALID_INPUT, "null row_ptr");
  if (shard_count < 1) shard_count = 1;
  if (shard_index >= shard_count) return fail(ESPN_E_INVALID_INPUT, "shard_index >= shard_count");
  cudaStream_t s = static_cast<cudaStream_t>(stream_v);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  ESPN_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (!rows) {
    synth_lengths_kernel<<<sms * 8, 256, 0, s>>>(n_docs, t_min, t_max, seed, shard_count, shard_index, row_ptr);
    scan_u64_kernel<<<1, 1024, 0, s>>>(row_ptr, n_docs);
    ESPN_CUDA_TRY(cudaGetLastError());
    ESPN_CUDA_TRY(cudaStreamSynchronize(s));
    return ESPN_OK;
  }
  const uint64_t rseed = splitmix64(seed ^ 0x5EEDull);
  switch (d) {
#define ESPN_S(DD) case DD: synth_rows_kernel<DD><<<sms * 16, 256, 0, s>>>(n_docs, row_ptr, shard_count, shard_index, rseed, dtype == ESPN_DTYPE_BF16, rows); break;
    ESPN_S(16) ESPN_S(32) ESPN_S(64) ESPN_S(128)
#undef ESPN_S
    default: return fail(ESPN_E_INVALID_INPUT, "synth supports d in {16,32,64,128}");
  }
  ESPN_CUDA_TRY(cudaGetLastError());
  ESPN_CUDA_TRY(cudaStreamSynchronize(s));
  return ESPN_OK;
}

}  // extern "C"

// ============================================================================
// Multi-GPU re-rank (espn_gpu.h "Multi-GPU"; shard.cuh)
// ============================================================================
namespace {
cudaError_t grow(void** p, uint64_t* cap, uint64_t need_bytes) {
  if (*cap >= need_bytes) return cudaSuccess;
  cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  const cudaError_t e = cudaMalloc(p, need_bytes);
  if (e == cudaSuccess) *cap = need_bytes;
  return e;
}

struct ShardJob {  // one rank's view of a sharded call
  bool replica = false;
  uint32_t G = 1, g = 0, B = 0, k = 0, nq = 0, BQ = 0;
  uint64_t P = 0;                 // packed words per rank
  const float* q = nullptr;       // device views of the global batch
  const uint32_t* ids = nullptr;
  const float* cls = nullptr;
  const uint64_t* off = nullptr;
  const uint32_t* need = nullptr;
};

int shard_validate(espn_gpu_table* t, espn_gpu_workspace* w, const espn_rerank_args* a, uint32_t nranks,
                   uint32_t rank, ShardJob* j) {
  if (!t || !w || !a) return fail(ESPN_E_INVALID_INPUT, "null argument");
  if (w->table != t) return fail(ESPN_E_INVALID_STATE, "workspace belongs to another table");
  if (nranks < 1 || rank >= nranks) return fail(ESPN_E_INVALID_INPUT, "rank must be in [0, nranks)");
  if (a->flags & (ESPN_RERANK_WRITE_BOW | ESPN_RERANK_PREFETCHED))
    return fail(ESPN_E_INVALID_INPUT, "sharded re-rank: WRITE_BOW / PREFETCHED are not supported");
  if ((a->flags & ESPN_RERANK_DEVICE_OFFSETS) && !(a->flags & ESPN_RERANK_DEVICE_IO))
    return fail(ESPN_E_INVALID_INPUT, "DEVICE_OFFSETS requires DEVICE_IO");
  j->replica = t->shard_count <= 1;
  if (!j->replica && (nranks != t->shard_count || rank != t->shard_index))
    return fail(ESPN_E_INVALID_CONFIG, "sharded table: the communicator must have shard_count ranks, this one at "
                                       "rank shard_index (got " + std::to_string(nranks) + " ranks, rank " +
                                       std::to_string(rank) + "; table shard " + std::to_string(t->shard_index) +
                                       " of " + std::to_string(t->shard_count) + ")");
  j->G = nranks;
  j->g = rank;
  j->B = a->n_queries;
  j->k = a->final_k;
  j->nq = a->n_query_tokens;
  if (j->B > w->max_queries) return fail(ESPN_E_INVALID_INPUT, "n_queries exceeds workspace capacity");
  if (j->k < 1 || j->k > (uint32_t)kMaxK) return fail(ESPN_E_INVALID_INPUT, "final_k must be in [1, 1024]");
  if (j->nq < 1 || j->nq > w->max_nq) return fail(ESPN_E_INVALID_INPUT, "n_query_tokens must be in [1, workspace max]");
  j->BQ = j->replica ? (j->B + j->G - 1) / j->G : j->B;
  j->P = pack_words(j->BQ, j->k);
  return ESPN_OK;
}

// Phase 1: the global batch on the device, this rank's local pass, its block
// packed into w->sh.send.  Everything on `s`.
int shard_pack(espn_gpu_table* t, espn_gpu_workspace* w, const espn_rerank_args* a, ShardJob& j, cudaStream_t s) {
  auto& h = w->sh;
  const bool dev_io = (a->flags & ESPN_RERANK_DEVICE_IO) != 0;
  const bool dev_off = (a->flags & ESPN_RERANK_DEVICE_OFFSETS) != 0;
  const uint64_t C = w->max_candidates;
  // ---- buffers (grown outside captures only) ----
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  ESPN_CUDA_TRY(cudaStreamIsCapturing(s, &cap));
  const bool need_lists = !h.lists && (!j.replica || !dev_io || !dev_off);
  if ((need_lists || h.send_cap < j.P) && cap != cudaStreamCaptureStatusNone)
    return fail(ESPN_E_INVALID_STATE, "sharded re-rank: run one call of this shape outside the stream capture first "
                                      "(it sizes the exchange buffers)");
  if (need_lists) {
    const uint64_t B = w->max_queries;
    cudaError_t e = cudaSuccess;
    auto al = [&](void** p, size_t bytes) { if (e == cudaSuccess) e = cudaMalloc(p, std::max<size_t>(bytes, 16)); };
    al((void**)&h.g_q, B * w->max_nq * t->d * sizeof(float));
    al((void**)&h.g_ids, C * 4);
    al((void**)&h.g_cls, C * 4);
    al((void**)&h.g_off, (B + 1) * 8);
    al((void**)&h.g_need, B * 4);
    al((void**)&h.loc_ids, C * 4);
    al((void**)&h.loc_cls, C * 4);
    al((void**)&h.loc_off, (B + 1) * 8);
    al((void**)&h.loc_need, B * 4);
    if (e != cudaSuccess) return fail(ESPN_E_CUDA, std::string("sharded workspace buffers: ") + cudaGetErrorString(e));
    h.lists = true;
  }
  {
    uint64_t sc = h.send_cap * 4;
    const cudaError_t e = grow(reinterpret_cast<void**>(&h.send), &sc, j.P * 4);
    if (e != cudaSuccess) return fail(ESPN_E_CUDA, std::string("sharded send buffer: ") + cudaGetErrorString(e));
    h.send_cap = sc / 4;
  }
  // ---- the global batch as device arrays ----
  j.q = a->query_tokens;
  j.ids = a->cand_ids;
  j.cls = a->cand_cls;
  j.off = a->cand_offsets;
  j.need = a->needed_counts;
  uint64_t Ch = 0;
  if (!dev_off) {  // host offsets: validate here, stage them
    const uint64_t* off = a->cand_offsets;
    if (!off) return fail(ESPN_E_INVALID_INPUT, "null cand_offsets");
    if (off[0] != 0) return fail(ESPN_E_INVALID_INPUT, "cand_offsets[0] must be 0");
    for (uint32_t b = 0; b < j.B; ++b)
      if (off[b + 1] < off[b]) return fail(ESPN_E_INVALID_INPUT, "cand_offsets must be non-decreasing");
    Ch = off[j.B];
    if (Ch > C) return fail(ESPN_E_INVALID_INPUT, "candidates exceed workspace capacity");
    ESPN_CUDA_TRY(cudaMemcpyAsync(h.g_off, off, (j.B + 1) * 8, cudaMemcpyHostToDevice, s));
    j.off = h.g_off;
    if (a->needed_counts) {
      ESPN_CUDA_TRY(cudaMemcpyAsync(h.g_need, a->needed_counts, j.B * 4, cudaMemcpyHostToDevice, s));
      j.need = h.g_need;
    }
  }
  if (!dev_io) {
    if (!a->query_tokens || (Ch && (!a->cand_ids || !a->cand_cls))) return fail(ESPN_E_INVALID_INPUT, "null array argument");
    ESPN_CUDA_TRY(cudaMemcpyAsync(h.g_q, a->query_tokens, (size_t)j.B * j.nq * t->d * 4, cudaMemcpyHostToDevice, s));
    if (Ch) {
      ESPN_CUDA_TRY(cudaMemcpyAsync(h.g_ids, a->cand_ids, Ch * 4, cudaMemcpyHostToDevice, s));
      ESPN_CUDA_TRY(cudaMemcpyAsync(h.g_cls, a->cand_cls, Ch * 4, cudaMemcpyHostToDevice, s));
    }
    j.q = h.g_q;
    j.ids = h.g_ids;
    j.cls = h.g_cls;
  }
  // ---- this rank's local pass, written straight into its packed block ----
  espn_rerank_args la = *a;
  la.flags = (a->flags & (ESPN_RERANK_PARTIAL | ESPN_RERANK_PROFILE | ESPN_RERANK_SEPARATE_TOPK |
                          ESPN_RERANK_QUERY_ROUNDED | ESPN_RERANK_QUERY_SPLIT)) |
             ESPN_RERANK_DEVICE_IO | ESPN_RERANK_DEVICE_OFFSETS | ESPN_RERANK_ASYNC;
  int32_t* blk = h.send;
  espn_rerank_out lo{};
  lo.ids = reinterpret_cast<uint32_t*>(blk + kPackHeaderWords);
  lo.scores = reinterpret_cast<float*>(blk + kPackHeaderWords + (uint64_t)j.BQ * j.k);
  lo.counts = reinterpret_cast<uint32_t*>(blk + kPackHeaderWords + 2ull * j.BQ * j.k);
  if (j.replica) {
    // rows this rank does not own stay empty (count 0)
    ESPN_CUDA_TRY(cudaMemsetAsync(lo.counts, 0, (size_t)j.BQ * 4, s));
    const uint32_t b0 = std::min<uint32_t>(j.B, j.g * j.BQ), b1 = std::min<uint32_t>(j.B, b0 + j.BQ);
    la.n_queries = b1 - b0;
    la.query_tokens = j.q + (size_t)b0 * j.nq * t->d;
    la.cand_ids = j.ids;
    la.cand_cls = j.cls;
    la.cand_offsets = j.off + b0;
    la.needed_counts = j.need ? j.need + b0 : nullptr;
    la.flags |= kFlagBaseOffsets;
  } else {
    ShardSplitParams sp{};
    sp.ids = j.ids;
    sp.cls = j.cls;
    sp.off = j.off;
    sp.need_in = j.need;
    sp.n_queries = j.B;
    sp.rerank_count = a->rerank_count;
    sp.shards = j.G;
    sp.shard = j.g;
    sp.max_candidates = C;
    sp.loc_off = h.loc_off;
    sp.loc_need = h.loc_need;
    sp.loc_ids = h.loc_ids;
    sp.loc_cls = h.loc_cls;
    sp.err = w->err;
    if (j.B) {
      shard_count_kernel<<<j.B, kShardThreads, 0, s>>>(sp);
      scan_u64_kernel<<<1, 1024, 0, s>>>(h.loc_off, j.B);
      shard_scatter_kernel<<<j.B, kShardThreads, 0, s>>>(sp);
      ESPN_CUDA_TRY(cudaGetLastError());
      w->counters.kernel_launches += 3;
    }
    la.cand_ids = h.loc_ids;
    la.cand_cls = h.loc_cls;
    la.cand_offsets = h.loc_off;
    la.needed_counts = h.loc_need;
    la.query_tokens = j.q;
  }
  if (la.n_queries) {
    const int st = espn_gpu_rerank(t, w, &la, &lo, s);
    if (st) return st;
  }
  pack_err_kernel<<<1, 32, 0, s>>>(w->err, blk);
  ESPN_CUDA_TRY(cudaGetLastError());
  w->counters.kernel_launches += 1;
  return ESPN_OK;
}

// Phase 3: the G gathered blocks -> the global ranked lists (+ every rank's
// error bits), outputs, and for synchronous calls the verdict.
int shard_merge(espn_gpu_table* t, espn_gpu_workspace* w, const espn_rerank_args* a, const ShardJob& j,
                const int32_t* recv, espn_rerank_out* o, cudaStream_t s) {
  (void)t;
  if (!o || !o->ids || !o->scores || !o->counts) return fail(ESPN_E_INVALID_INPUT, "null output array");
  const bool dev_io = (a->flags & ESPN_RERANK_DEVICE_IO) != 0;
  uint32_t* oi = dev_io ? o->ids : w->out_ids;
  float* os = dev_io ? o->scores : w->out_scores;
  uint32_t* oc = dev_io ? o->counts : w->out_counts;
  if (j.B) {
    if (j.replica) {
      unpack_replica_kernel<<<j.B, 128, 0, s>>>(recv, j.G, j.P, j.B, j.BQ, j.k, oi, os, oc, w->err);
    } else {
      ESPN_CUDA_TRY(ensure_topk_attr());
      merge_packed_kernel<<<j.B, kTopkThreads, topk_smem_bytes(), s>>>(recv, j.G, j.P, j.B, j.k, oi, os, oc, w->err);
    }
    ESPN_CUDA_TRY(cudaGetLastError());
    w->counters.kernel_launches += 1;
  }
  if (!dev_io && j.B) {
    ESPN_CUDA_TRY(cudaMemcpyAsync(o->ids, oi, (size_t)j.B * j.k * 4, cudaMemcpyDeviceToHost, s));
    ESPN_CUDA_TRY(cudaMemcpyAsync(o->scores, os, (size_t)j.B * j.k * 4, cudaMemcpyDeviceToHost, s));
    ESPN_CUDA_TRY(cudaMemcpyAsync(o->counts, oc, (size_t)j.B * 4, cudaMemcpyDeviceToHost, s));
  }
  w->counters.batches += 1;
  w->counters.queries += j.B;
  if (a->flags & ESPN_RERANK_ASYNC) {
    w->async_pending = true;
    return ESPN_OK;
  }
  ESPN_CUDA_TRY(cudaMemcpyAsync(w->h_err, w->err, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  ESPN_CUDA_TRY(cudaStreamSynchronize(s));
  if (*w->h_err) ESPN_CUDA_TRY(cudaMemsetAsync(w->err, 0, sizeof(uint32_t), s));
  w->async_pending = false;
  return err_bits_to_status(*w->h_err);
}

int shard_recv_buffer(espn_gpu_workspace* w, const ShardJob& j, cudaStream_t s) {
  auto& h = w->sh;
  if (h.recv_cap >= j.P * j.G) return ESPN_OK;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  ESPN_CUDA_TRY(cudaStreamIsCapturing(s, &cap));
  if (cap != cudaStreamCaptureStatusNone)
    return fail(ESPN_E_INVALID_STATE, "sharded re-rank: run one call of this shape outside the stream capture first");
  uint64_t rc = h.recv_cap * 4;
  const cudaError_t e = grow(reinterpret_cast<void**>(&h.recv), &rc, j.P * j.G * 4);
  if (e != cudaSuccess) return fail(ESPN_E_CUDA, std::string("sharded recv buffer: ") + cudaGetErrorString(e));
  h.recv_cap = rc / 4;
  return ESPN_OK;
}

int comm_shape(void* comm, uint32_t* nranks, uint32_t* rank, int* device) {
  const NcclApi& n = nccl_api();
  if (!n.ok) return fail(ESPN_E_CUDA, n.why);
  if (!comm) return fail(ESPN_E_INVALID_INPUT, "null NCCL communicator");
  int c = 0, r = 0, d = 0;
  ESPN_NCCL_TRY(n.CommCount(static_cast<ncclComm_t>(comm), &c));
  ESPN_NCCL_TRY(n.CommUserRank(static_cast<ncclComm_t>(comm), &r));
  ESPN_NCCL_TRY(n.CommCuDevice(static_cast<ncclComm_t>(comm), &d));
  *nranks = (uint32_t)c;
  *rank = (uint32_t)r;
  *device = d;
  return ESPN_OK;
}
}  // namespace

extern "C" {

int espn_nccl_get_unique_id(espn_nccl_id* out) {
  if (!out) return fail(ESPN_E_INVALID_INPUT, "null argument");
  const NcclApi& n = nccl_api();
  if (!n.ok) return fail(ESPN_E_CUDA, n.why);
  static_assert(sizeof(espn_nccl_id) == sizeof(ncclUniqueId), "id size");
  ncclUniqueId id;
  ESPN_NCCL_TRY(n.GetUniqueId(&id));
  std::memcpy(out, &id, sizeof id);
  return ESPN_OK;
}

int espn_nccl_comm_init(int nranks, const espn_nccl_id* id, int rank, int device, void** comm) {
  if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) return fail(ESPN_E_INVALID_INPUT, "bad argument");
  const NcclApi& n = nccl_api();
  if (!n.ok) return fail(ESPN_E_CUDA, n.why);
  DeviceGuard g(device);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  ncclComm_t c = nullptr;
  ESPN_NCCL_TRY(n.CommInitRank(&c, nranks, uid, rank));
  *comm = c;
  return ESPN_OK;
}

int espn_nccl_comm_init_all(int ndev, const int* devices, void** comms) {
  if (ndev < 1 || !devices || !comms) return fail(ESPN_E_INVALID_INPUT, "bad argument");
  const NcclApi& n = nccl_api();
  if (!n.ok) return fail(ESPN_E_CUDA, n.why);
  std::vector<ncclComm_t> c(ndev, nullptr);
  ESPN_NCCL_TRY(n.CommInitAll(c.data(), ndev, devices));
  for (int i = 0; i < ndev; ++i) comms[i] = c[i];
  return ESPN_OK;
}

int espn_nccl_comm_destroy(void* comm) {
  if (!comm) return ESPN_OK;
  const NcclApi& n = nccl_api();
  if (!n.ok) return fail(ESPN_E_CUDA, n.why);
  ESPN_NCCL_TRY(n.CommDestroy(static_cast<ncclComm_t>(comm)));
  return ESPN_OK;
}

int espn_gpu_shard_pack(espn_gpu_table* t, espn_gpu_workspace* w, const espn_rerank_args* a, uint32_t nranks,
                        uint32_t rank, void* stream, const int32_t** send, uint64_t* words) {
  ShardJob j;
  int st = shard_validate(t, w, a, nranks, rank, &j);
  if (st) return st;
  DeviceGuard g(t->device);
  st = shard_pack(t, w, a, j, static_cast<cudaStream_t>(stream));
  if (st) return st;
  if (send) *send = w->sh.send;
  if (words) *words = j.P;
  return ESPN_OK;
}

int espn_gpu_shard_merge(espn_gpu_table* t, espn_gpu_workspace* w, const espn_rerank_args* a, const int32_t* recv,
                         uint32_t nranks, espn_rerank_out* out, void* stream) {
  ShardJob j;
  // the rank only matters for the pack; the merge is rank-independent
  const uint32_t r = (t && t->shard_count > 1) ? t->shard_index : 0;
  int st = shard_validate(t, w, a, nranks, r, &j);
  if (st) return st;
  if (!recv) return fail(ESPN_E_INVALID_INPUT, "null recv");
  DeviceGuard g(t->device);
  return shard_merge(t, w, a, j, recv, out, static_cast<cudaStream_t>(stream));
}

int espn_gpu_rerank_sharded(espn_gpu_table* t, espn_gpu_workspace* w, const espn_rerank_args* a, espn_rerank_out* o,
                            void* comm, void* stream) {
  uint32_t G = 0, r = 0;
  int cdev = 0;
  int st = comm_shape(comm, &G, &r, &cdev);
  if (st) return st;
  ShardJob j;
  st = shard_validate(t, w, a, G, r, &j);
  if (st) return st;
  if (cdev != t->device) return fail(ESPN_E_INVALID_CONFIG, "NCCL communicator and table are on different devices");
  DeviceGuard g(t->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  st = shard_recv_buffer(w, j, s);
  if (!st) st = shard_pack(t, w, a, j, s);
  if (st) return st;
  const NcclApi& n = nccl_api();
  ESPN_NCCL_TRY(n.AllGather(w->sh.send, w->sh.recv, j.P, ncclInt32, static_cast<ncclComm_t>(comm), s));
  return shard_merge(t, w, a, j, w->sh.recv, o, s);
}

int espn_gpu_rerank_sharded_multi(uint32_t n, espn_gpu_table* const* tables, espn_gpu_workspace* const* ws,
                                  const espn_rerank_args* a, espn_rerank_out* outs, void* const* comms,
                                  void* const* streams) {
  if (n == 0) return ESPN_OK;
  if (!tables || !ws || !a || !outs || !comms || !streams) return fail(ESPN_E_INVALID_INPUT, "null argument");
  std::vector<ShardJob> jobs(n);
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t G = 0, r = 0;
    int cdev = 0;
    int st = comm_shape(comms[i], &G, &r, &cdev);
    if (st) return st;
    if (G != n) return fail(ESPN_E_INVALID_CONFIG, "every device of the call needs one rank of an n-rank communicator");
    st = shard_validate(tables[i], ws[i], a, G, r, &jobs[i]);
    if (st) return st;
    if (cdev != tables[i]->device) return fail(ESPN_E_INVALID_CONFIG, "communicator / table device mismatch");
  }
  // phase 1 on every device, then the all-gathers as ONE group (one thread
  // drives several ranks), then the merges; synchronous calls sync at the end
  espn_rerank_args aa = *a;
  aa.flags |= ESPN_RERANK_ASYNC;
  for (uint32_t i = 0; i < n; ++i) {
    DeviceGuard g(tables[i]->device);
    cudaStream_t s = static_cast<cudaStream_t>(streams[i]);
    int st = shard_recv_buffer(ws[i], jobs[i], s);
    if (!st) st = shard_pack(tables[i], ws[i], a, jobs[i], s);
    if (st) return st;
  }
  const NcclApi& nc = nccl_api();
  ESPN_NCCL_TRY(nc.GroupStart());
  for (uint32_t i = 0; i < n; ++i) {
    DeviceGuard g(tables[i]->device);
    const ncclResult_t r = nc.AllGather(ws[i]->sh.send, ws[i]->sh.recv, jobs[i].P, ncclInt32,
                                        static_cast<ncclComm_t>(comms[i]), static_cast<cudaStream_t>(streams[i]));
    if (r != ncclSuccess) {
      nc.GroupEnd();
      return fail(ESPN_E_CUDA, std::string("ncclAllGather: ") + nc.GetErrorString(r));
    }
  }
  ESPN_NCCL_TRY(nc.GroupEnd());
  for (uint32_t i = 0; i < n; ++i) {
    DeviceGuard g(tables[i]->device);
    const int st = shard_merge(tables[i], ws[i], &aa, jobs[i], ws[i]->sh.recv, &outs[i],
                               static_cast<cudaStream_t>(streams[i]));
    if (st) return st;
  }
  if (a->flags & ESPN_RERANK_ASYNC) return ESPN_OK;
  int worst = ESPN_OK;
  for (uint32_t i = 0; i < n; ++i) {
    const int st = espn_gpu_workspace_sync(ws[i], streams[i]);
    if (st && !worst) worst = st;
  }
  return worst;
}

}  // extern "C"

// ============================================================================
// Reference scoring primitives (scoring.hpp:7-21) on the device
// ============================================================================
extern "C" {

int espn_gpu_maxsim_f32(const float* q, uint32_t nq, const float* doc, uint32_t t, uint32_t d, float* out,
                        int device) {
  if (!out || (nq && !q) || (t && !doc)) return fail(ESPN_E_INVALID_INPUT, "null argument");
  if (nq == 0 || t == 0 || d == 0) return fail(ESPN_E_INVALID_INPUT, "empty query or document (types.hpp:64-68)");
  int sms = 0;
  bool tc = false;
  int st = check_device(device, &sms, &tc);
  if (st) return st;
  DeviceGuard g(device);
  float *dq = nullptr, *dd = nullptr, *dm = nullptr;
  auto cleanup = [&] { cudaFree(dq); cudaFree(dd); cudaFree(dm); };
  cudaError_t e = cudaMalloc(&dq, (size_t)nq * d * 4);
  if (e == cudaSuccess) e = cudaMalloc(&dd, (size_t)t * d * 4);
  if (e == cudaSuccess) e = cudaMalloc(&dm, (size_t)(nq + 1) * 4);
  if (e == cudaSuccess) e = cudaMemcpy(dq, q, (size_t)nq * d * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dd, doc, (size_t)t * d * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    maxsim_f32_kernel<<<nq, 256>>>(dq, dd, t, d, dm + 1);
    sum_ordered_kernel<<<1, 32>>>(dm + 1, nq, dm);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, dm, 4, cudaMemcpyDeviceToHost);
  cleanup();
  if (e != cudaSuccess) return fail(ESPN_E_CUDA, std::string("maxsim_f32: ") + cudaGetErrorString(e));
  return ESPN_OK;
}

int espn_gpu_rank(const uint32_t* ids, const float* scores, uint64_t n, uint32_t* out_ids, float* out_scores,
                  int device) {
  if (n == 0) return ESPN_OK;
  if (!ids || !scores || !out_ids || !out_scores) return fail(ESPN_E_INVALID_INPUT, "null argument");
  int sms = 0;
  bool tc = false;
  int st = check_device(device, &sms, &tc);
  if (st) return st;
  DeviceGuard g(device);
  uint32_t *di = nullptr, *di2 = nullptr, *derr = nullptr;
  float* ds = nullptr;
  unsigned long long *dk = nullptr, *dk2 = nullptr;
  void* tmp = nullptr;
  auto cleanup = [&] { cudaFree(di); cudaFree(di2); cudaFree(derr); cudaFree(ds); cudaFree(dk); cudaFree(dk2); cudaFree(tmp); };
  size_t tb1 = 0, tb2 = 0;
  cub::DeviceRadixSort::SortKeysDescending(nullptr, tb1, dk, dk2, (int64_t)n);
  cub::DeviceRadixSort::SortKeys(nullptr, tb2, di, di2, (int64_t)n);
  cudaError_t e = cudaMalloc(&di, n * 4);
  if (e == cudaSuccess) e = cudaMalloc(&di2, n * 4);
  if (e == cudaSuccess) e = cudaMalloc(&ds, n * 4);
  if (e == cudaSuccess) e = cudaMalloc(&dk, n * 8);
  if (e == cudaSuccess) e = cudaMalloc(&dk2, n * 8);
  if (e == cudaSuccess) e = cudaMalloc(&derr, 4);
  if (e == cudaSuccess) e = cudaMalloc(&tmp, std::max(tb1, tb2));
  if (e == cudaSuccess) e = cudaMemset(derr, 0, 4);
  if (e == cudaSuccess) e = cudaMemcpy(di, ids, n * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(ds, scores, n * 4, cudaMemcpyHostToDevice);
  const int blocks = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * 8);
  if (e == cudaSuccess) {
    rank_keys_kernel<<<blocks, 256>>>(di, ds, n, dk, derr);
    size_t tb = std::max(tb1, tb2);
    e = cub::DeviceRadixSort::SortKeysDescending(tmp, tb, dk, dk2, (int64_t)n);
    tb = std::max(tb1, tb2);
    if (e == cudaSuccess) e = cub::DeviceRadixSort::SortKeys(tmp, tb, di, di2, (int64_t)n);
    if (e == cudaSuccess) {
      adjacent_dup_kernel<<<blocks, 256>>>(di2, n, derr);
      rank_unkey_kernel<<<blocks, 256>>>(dk2, n, di, ds);
      e = cudaGetLastError();
    }
  }
  uint32_t herr = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&herr, derr, 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && !herr) e = cudaMemcpy(out_ids, di, n * 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && !herr) e = cudaMemcpy(out_scores, ds, n * 4, cudaMemcpyDeviceToHost);
  cleanup();
  if (e != cudaSuccess) return fail(ESPN_E_CUDA, std::string("rank: ") + cudaGetErrorString(e));
  if (herr & ERR_DUPLICATE) return fail(ESPN_E_INVALID_INPUT, "rank: duplicate doc id (scoring.hpp:16-18)");
  if (herr) return fail(ESPN_E_INVALID_INPUT, "rank: non-finite score (scoring.hpp:16-18)");
  return ESPN_OK;
}

}  // extern "C"
