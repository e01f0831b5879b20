// Throwaway probe: validates the tcgen05 K-major SWIZZLE_NONE descriptor layout
// and the block-diagonal "sliding window" A-operand trick used by the MaxSim kernel.
// D[128 x N] = A_window[128 x 16*ks] . B[N x 16*ks]^T, fp16 in, fp32 accum in TMEM.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_fp16.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm100)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

constexpr int D = 32;           // head dim (K)
constexpr int NQ = 128;         // columns per quarter
constexpr int ROWS_A = 224;     // 96 zero | 32 Q | 96 zero
constexpr int CHUNKS = D / 8;   // 16-byte chunks per row
constexpr int SBO = CHUNKS * 128;

__global__ void probe(const __half* Q /*32 x D*/, const __half* B /*4*NQ x D*/, float* out /*128 x NQ*/) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                        // ROWS_A rows
  uint8_t* sB = smem + ROWS_A * D * 2;       // 4 quarters x NQ rows
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base_sh;
  int tid = threadIdx.x, warp = tid / 32;
  // zero + fill A (row r, chunk c) -> (r/8)*SBO + c*128 + (r%8)*16
  for (int i = tid; i < ROWS_A * CHUNKS; i += blockDim.x) {
    int r = i / CHUNKS, c = i % CHUNKS;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r >= 96 && r < 128) v = *reinterpret_cast<const uint4*>(Q + (r - 96) * D + c * 8);
    *reinterpret_cast<uint4*>(sA + (r / 8) * SBO + c * 128 + (r % 8) * 16) = v;
  }
  for (int i = tid; i < 4 * NQ * CHUNKS; i += blockDim.x) {
    int n = i / CHUNKS, c = i % CHUNKS;
    int qd = n / NQ, nn = n % NQ;
    uint4 v = *reinterpret_cast<const uint4*>(B + n * D + c * 8);
    *reinterpret_cast<uint4*>(sB + qd * NQ * D * 2 + (nn / 8) * SBO + c * 128 + (nn % 8) * 16) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base_sh)), "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tmem = tmem_base_sh;
  if (tid == 0) {
    // idesc: c_format F32 (bit4), a/b F16 (0), K-major both, N>>3 at 17, M>>4 at 24
    uint32_t idesc = (1u << 4) | ((uint32_t)(NQ >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    int first = 1;
    for (int w = 0; w < 4; ++w) {
      for (int ks = 0; ks < D / 16; ++ks) {
        uint32_t a_addr = smem_u32(sA) + ((96 - 32 * w) / 8) * SBO + ks * 256;
        uint32_t b_addr = smem_u32(sB) + w * NQ * D * 2 + ks * 256;
        uint64_t ad = make_desc(a_addr, 128, SBO), bd = make_desc(b_addr, 128, SBO);
        uint32_t acc = first ? 0u : 1u;
        first = 0;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     :: "r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
  }
  // wait phase 0
  asm volatile("{\n\t.reg .pred P1;\n\tWAIT:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
               "@!P1 bra WAIT;\n\t}" :: "r"(smem_u32(&bar)), "r"(0));
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    for (int c0 = 0; c0 < NQ; c0 += 32) {
      uint32_t r[32];
      uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                   "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                     "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                     "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 32; ++j) out[(warp * 32 + (tid % 32)) * NQ + c0 + j] = __uint_as_float(r[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(128));
}

int main() {
  std::vector<__half> hQ(32 * D), hB(4 * NQ * D);
  std::vector<float> fQ(32 * D), fB(4 * NQ * D);
  srand(1);
  for (size_t i = 0; i < hQ.size(); ++i) { float v = (rand() % 2001 - 1000) / 1000.f; hQ[i] = __float2half(v); fQ[i] = __half2float(hQ[i]); }
  for (size_t i = 0; i < hB.size(); ++i) { float v = (rand() % 2001 - 1000) / 1000.f; hB[i] = __float2half(v); fB[i] = __half2float(hB[i]); }
  __half *dQ, *dB; float* dO;
  CK(cudaMalloc(&dQ, hQ.size() * 2)); CK(cudaMalloc(&dB, hB.size() * 2)); CK(cudaMalloc(&dO, 128 * NQ * 4));
  CK(cudaMemcpy(dQ, hQ.data(), hQ.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice));
  int smem = ROWS_A * D * 2 + 4 * NQ * D * 2;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe<<<1, 128, smem>>>(dQ, dB, dO);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  std::vector<float> o(128 * NQ);
  CK(cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0; int bad = 0;
  for (int lane = 0; lane < 128; ++lane) {
    int w = lane / 32, i = lane % 32;
    for (int n = 0; n < NQ; ++n) {
      double ref = 0;
      for (int k = 0; k < D; ++k) ref += (double)fQ[i * D + k] * fB[(w * NQ + n) * D + k];
      double e = fabs(ref - o[lane * NQ + n]);
      if (e > maxerr) maxerr = e;
      if (e > 1e-3 && bad < 5) { printf("mismatch lane %d col %d ref %f got %f\n", lane, n, ref, o[lane * NQ + n]); ++bad; }
    }
  }
  printf("UMMA probe max abs err = %g  %s\n", maxerr, maxerr < 1e-3 ? "PASS" : "FAIL");
  return maxerr < 1e-3 ? 0 : 1;
}
