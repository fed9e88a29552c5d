// gspn_umma.cu — the compact-channel proxy projections (§4.2 "project
// ... into a lower-dimensional proxy subspace", "expand back to C with a learned 1x1
// projection") on the 5th-generation tensor cores: tcgen05.mma with the accumulator in TMEM, the
// activation tiles streamed by TMA, the weights resident in shared memory.
//
//   out[b, o, n] = sum_i M[o, i] in[b, i, n]        (n over the H W pixels; M [Co, Ci] or, transposed, [Ci, Co])
//
// Per batch b this is the GEMM D[o, n] = A[o, i] B[i, n] with A = M (K-major; the transposed storage is
// re-laid out when staged) and B = in[b] (pixels contiguous: MN-major). At the configs' shapes (320 -> 40,
// 384 -> 8, 40 -> 320) a pixel costs 2 Ci Co flops for (Ci + Co) s bytes -- up to ~36 flop/byte, above
// the SIMT ridge, far below the tensor-core one: on tcgen05 the projection streams at HBM speed.
//
// CTA (persistent over (b, 256/128/64-pixel) tiles): warp 0 = TMA producer (B chunks of 64 channels x NT
// pixels, 128-byte swizzle, through a shared-memory ring), warp 1 = MMA issuer (one thread; allocates
// NT x MT x 2 TMEM columns: a double-buffered fp32 accumulator of 128 lanes = output rows), warps 2-5 =
// epilogue (tcgen05.ld of their 32-lane TMEM sub-partition -> bf16 -> 16-byte global stores).
// M = 128 rows per MMA (rows >= Co are zero weights), K = 16 per MMA, N = NT.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>

#include "gspn_common.cuh"
#include "gspn_internal.h"
#include "gspn_ptx.cuh"

namespace gspn {
namespace {

using namespace ptx;

constexpr int kKC = 64;                 // K elements per chunk = one 128-byte swizzle row of bf16
constexpr uint32_t kAChunk = 128 * 128;  // one A chunk: 128 rows x 128 bytes
constexpr uint32_t kBBox = 64 * 128;     // one B box: 64 channel rows x 64 pixels (128 bytes)
constexpr int kMixThreads = 6 * 32;

struct UmmaMixArgs {
  CUtensorMap in_map;   // in viewed as [B][Ci][HW] bf16, box {64 px, 64 ch, 1}, SWIZZLE_128B
  CUtensorMap out_map;  // out viewed as [B][Co][HW] bf16, box {64 px, 128 rows, 1}, SWIZZLE_128B
  const __nv_bfloat16* M;
  __nv_bfloat16* out;
  int B, Ci, Co, HW, trans;
  int MT, KC, NT, nstages, ntn;
  int64_t ntiles;
  uint32_t a_bytes, stage_bytes, o_bytes, tmem_cols, idesc;
  int orows;  // rows of an output staging box / TMA store box: min(128, Co) rounded up to 8
  int nob;    // output staging buffers (2 when they fit: a tile's stores overlap the next tile's drain)
};

// named barrier of the 4 epilogue warps
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Shared-memory matrix descriptor (tcgen05), 128-byte swizzle, sm_100 version bits.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = static_cast<uint64_t>((addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;  // descriptor version (Blackwell)
  d |= 2ull << 61;  // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t pack2(uint32_t a, uint32_t b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(a), __uint_as_float(b));
  return *reinterpret_cast<uint32_t*>(&v);
}

__global__ void __launch_bounds__(kMixThreads, 1) umma_mix_kernel(const __grid_constant__ UmmaMixArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sa = base;                                   // weights: MT x KC chunks of [128 rows][128 B], swizzled
  uint8_t* ring = base + A.a_bytes;                     // B stages: NT/64 boxes of [64 rows][128 B]
  uint8_t* ob = ring + static_cast<size_t>(A.nstages) * A.stage_bytes;  // output staging: 2 x MT x NT/64 boxes
  uint64_t* full = reinterpret_cast<uint64_t*>(ob + A.nob * A.o_bytes);
  uint64_t* empty = full + A.nstages;
  uint64_t* tfull = empty + A.nstages;  // [2] accumulator ready
  uint64_t* tempty = tfull + 2;         // [2] accumulator drained
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < A.nstages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&tfull[s]), 1);
      mbar_init(smem_u32(&tempty[s]), 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // TMEM allocation (whole warp), then give up the right to allocate more
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(A.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp != 0) {
    // weights -> K-major 128-byte-swizzled chunks: element (row m, k) of chunk (mt, kc) at byte
    // (m / 8) 1024 + (m % 8) 128 + ((2 k / 16) ^ (m % 8)) 16 + (2 k) % 16; zero outside [Co) x [Ci). Staged by
    // warps 1-5 while the producer already streams the first activation tiles.
    const int nthr = blockDim.x - 32, tid = threadIdx.x - 32;
    if (!A.trans && A.Ci % 8 == 0) {  // 8 consecutive k = one 16-byte piece on both sides
      const int nv = A.MT * A.KC * 128 * (kKC / 8);
      for (int e = tid; e < nv; e += nthr) {
        const int chunk = e / (128 * (kKC / 8)), rem = e - chunk * 128 * (kKC / 8);
        const int m = rem / (kKC / 8), k = (rem - m * (kKC / 8)) * 8;
        const int mt = chunk / A.KC, kc = chunk - mt * A.KC;
        const int o = mt * 128 + m, i = kc * kKC + k;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (o < A.Co && i < A.Ci) v = __ldg(reinterpret_cast<const uint4*>(A.M + static_cast<int64_t>(o) * A.Ci + i));
        const uint32_t byte = (m >> 3) * 1024u + (m & 7) * 128u + ((((2u * k) >> 4) ^ (m & 7)) << 4);
        *reinterpret_cast<uint4*>(sa + static_cast<size_t>(chunk) * kAChunk + byte) = v;
      }
    } else {
      const int nA = A.MT * A.KC * 128 * kKC;
      for (int e = tid; e < nA; e += nthr) {
        const int chunk = e / (128 * kKC), rem = e - chunk * 128 * kKC;
        const int m = rem / kKC, k = rem - m * kKC;
        const int mt = chunk / A.KC, kc = chunk - mt * A.KC;
        const int o = mt * 128 + m, i = kc * kKC + k;
        __nv_bfloat16 v = __float2bfloat16_rn(0.f);
        if (o < A.Co && i < A.Ci) v = A.trans ? A.M[static_cast<int64_t>(i) * A.Co + o] : A.M[static_cast<int64_t>(o) * A.Ci + i];
        const uint32_t byte = (m >> 3) * 1024u + (m & 7) * 128u + ((((2u * k) >> 4) ^ (m & 7)) << 4) + ((2u * k) & 15u);
        *reinterpret_cast<__nv_bfloat16*>(sa + static_cast<size_t>(chunk) * kAChunk + byte) = v;
      }
    }
    fence_proxy_async();  // generic-proxy weight writes -> visible to the tensor cores (async proxy)
    asm volatile("bar.sync 2, %0;" ::"r"(nthr) : "memory");
  }

  if (warp == 0) {  // ---- TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&A.in_map) : "memory");
      const uint64_t pol = policy_of(0);  // activations are read once
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
        const int b = static_cast<int>(t / A.ntn), px0 = static_cast<int>(t % A.ntn) * A.NT;
        for (int kc = 0; kc < A.KC; ++kc) {
          mbar_wait_sleep(smem_u32(&empty[stage]), phase ^ 1);
          const uint32_t fb = smem_u32(&full[stage]);
          mbar_arrive_tx(fb, A.stage_bytes);
          const uint32_t dst = smem_u32(ring + static_cast<size_t>(stage) * A.stage_bytes);
          for (int j = 0; j < A.NT / 64; ++j) tma_load3(dst + j * kBBox, &A.in_map, px0 + 64 * j, kc * kKC, b, fb, pol);
          if (++stage == A.nstages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {  // ---- MMA issuer (one thread)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int64_t it = 0;
      for (int64_t t = blockIdx.x; t < A.ntiles; t += gridDim.x, ++it) {
        const int buf = static_cast<int>(it & 1);
        mbar_wait(smem_u32(&tempty[buf]), static_cast<uint32_t>(((it >> 1) & 1) ^ 1));
        tc_fence_after();
        for (int kc = 0; kc < A.KC; ++kc) {
          mbar_wait(smem_u32(&full[stage]), phase);
          tc_fence_after();
          const uint32_t bst = smem_u32(ring + static_cast<size_t>(stage) * A.stage_bytes);
          for (int mt = 0; mt < A.MT; ++mt) {
            const uint32_t td = tmem + static_cast<uint32_t>((buf * A.MT + mt) * A.NT);
            const uint32_t ast = smem_u32(sa) + static_cast<uint32_t>(mt * A.KC + kc) * kAChunk;
#pragma unroll
            for (int ks = 0; ks < kKC / 16; ++ks)
              umma_bf16(td, sdesc(ast + ks * 32, 16, 1024), sdesc(bst + ks * 2048, kBBox, 1024), A.idesc,
                        (kc | ks) != 0);
          }
          umma_commit(smem_u32(&empty[stage]));  // frees the B stage once these MMAs have read it
          if (++stage == A.nstages) { stage = 0; phase ^= 1; }
        }
        umma_commit(smem_u32(&tfull[buf]));  // accumulator complete
      }
    }
  } else {  // ---- epilogue: TMEM sub-partition (warp % 4) = output rows 32 (warp % 4) .. + 31
    // TMEM -> registers -> bf16 -> the 128-byte-swizzled staging tile -> TMA stores of [128 rows][64 px]
    // boxes (rows >= Co and pixels >= HW are clipped by the tensor map): full-line writes per row.
    const int sp = warp & 3;
    const int row = 32 * sp + lane;
    const bool leader = warp == 2 && lane == 0;
    const int nbox = A.NT / 64;
    if (leader) asm volatile("prefetch.tensormap [%0];" ::"l"(&A.out_map) : "memory");
    int64_t it = 0;
    for (int64_t t = blockIdx.x; t < A.ntiles; t += gridDim.x, ++it) {
      const int buf = static_cast<int>(it & 1);
      const int b = static_cast<int>(t / A.ntn), px0 = static_cast<int>(t % A.ntn) * A.NT;
      mbar_wait(smem_u32(&tfull[buf]), static_cast<uint32_t>((it >> 1) & 1));
      tc_fence_after();
      if (leader) {  // the stores that last used this staging buffer have read it
        if (A.nob == 2) bulk_wait_read1();
        else bulk_wait_read0();
      }
      epi_bar();
      uint8_t* obuf = ob + static_cast<size_t>(A.nob == 2 ? buf : 0) * A.o_bytes;
      const uint32_t obox = static_cast<uint32_t>(A.orows) * 128u;
      for (int mt = 0; mt < A.MT; ++mt) {
        if (32 * sp >= A.orows) break;  // warp-uniform: rows past the store box (zero weights)
        const uint32_t tcol = tmem + (static_cast<uint32_t>(32 * sp) << 16) + static_cast<uint32_t>((buf * A.MT + mt) * A.NT);
        for (int c0 = 0; c0 < A.NT; c0 += 16) {
          uint32_t v[16];
          tmem_ld16(tcol + c0, v);
          if (row >= A.orows) continue;
          uint8_t* box = obuf + static_cast<size_t>(mt * nbox + c0 / 64) * obox + row * 128;
          const int q = (c0 & 63) >> 3;  // 16-byte chunk of the 128-byte row
          *reinterpret_cast<uint4*>(box + ((q ^ (row & 7)) << 4)) =
              make_uint4(pack2(v[0], v[1]), pack2(v[2], v[3]), pack2(v[4], v[5]), pack2(v[6], v[7]));
          *reinterpret_cast<uint4*>(box + (((q + 1) ^ (row & 7)) << 4)) =
              make_uint4(pack2(v[8], v[9]), pack2(v[10], v[11]), pack2(v[12], v[13]), pack2(v[14], v[15]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&tempty[buf]));  // accumulator drained: the MMA may reuse it
      fence_proxy_async();  // staging writes -> visible to the TMA unit
      epi_bar();
      if (leader) {
        for (int mt = 0; mt < A.MT; ++mt)
          for (int j = 0; j < nbox; ++j)
            tma_store3(&A.out_map, smem_u32(obuf + static_cast<size_t>(mt * nbox + j) * obox), px0 + 64 * j, mt * 128,
                       b, policy_of(0));
        bulk_commit();
      }
    }
    if (leader) bulk_wait_all();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(A.tmem_cols) : "memory");
  }
}

// ---- weight gradient: dM[o, i] = sum_{b, n} dout[b, o, n] in[b, i, n] -- D[o, i] = A[o, n] B[i, n] with
// both operands K-major (pixels contiguous). The K range (every batch's pixels, in chunks of 64) is split
// over the persistent CTAs; each accumulates its part in TMEM (MT x Npad fp32 columns) and the epilogue
// adds it to the caller's zeroed fp32 dM with one red.global.add per element and CTA.
struct UmmaWgradArgs {
  CUtensorMap a_map;  // dout viewed [B][Co][HW] bf16, box {64 px, 128 rows, 1}, SWIZZLE_128B
  CUtensorMap b_map;  // in viewed [B][Ci][HW] bf16, box {64 px, BR rows, 1}, SWIZZLE_128B
  float* dM;
  int B, Ci, Co, HW;
  int MT, Npad, BR, NB, nstages, nchb;  // nchb: 64-pixel chunks per batch
  int64_t nchunks;
  uint32_t stage_bytes, a_bytes, tmem_cols;
  uint32_t idesc[2];  // N of the first MMA (<= 256) and of the second (Npad - 256, if any)
};

__global__ void __launch_bounds__(kMixThreads, 1) umma_wgrad_kernel(const __grid_constant__ UmmaWgradArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + static_cast<size_t>(A.nstages) * A.stage_bytes);
  uint64_t* empty = full + A.nstages;
  uint64_t* done = empty + A.nstages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // this CTA's contiguous share of the 64-pixel chunks
  const int64_t c0 = A.nchunks * blockIdx.x / gridDim.x, c1 = A.nchunks * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < A.nstages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    mbar_init(smem_u32(done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(A.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp == 0) {  // ---- TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&A.a_map) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&A.b_map) : "memory");
      const uint64_t pol = policy_of(0);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t c = c0; c < c1; ++c) {
        const int b = static_cast<int>(c / A.nchb), px = static_cast<int>(c % A.nchb) * 64;
        mbar_wait_sleep(smem_u32(&empty[stage]), phase ^ 1);
        const uint32_t fb = smem_u32(&full[stage]);
        mbar_arrive_tx(fb, A.stage_bytes);
        const uint32_t dst = smem_u32(ring + static_cast<size_t>(stage) * A.stage_bytes);
        for (int mt = 0; mt < A.MT; ++mt) tma_load3(dst + mt * kAChunk, &A.a_map, px, mt * 128, b, fb, pol);
        for (int nb = 0; nb < A.NB; ++nb)
          tma_load3(dst + A.a_bytes + nb * A.BR * 128, &A.b_map, px, nb * A.BR, b, fb, pol);
        if (++stage == A.nstages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {  // ---- MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t c = c0; c < c1; ++c) {
        mbar_wait(smem_u32(&full[stage]), phase);
        tc_fence_after();
        const uint32_t st = smem_u32(ring + static_cast<size_t>(stage) * A.stage_bytes);
        for (int mt = 0; mt < A.MT; ++mt) {
          for (int nt = 0; nt * 256 < A.Npad; ++nt) {
            const uint32_t td = tmem + static_cast<uint32_t>(mt * A.Npad + nt * 256);
#pragma unroll
            for (int ks = 0; ks < kKC / 16; ++ks)
              umma_bf16(td, sdesc(st + mt * kAChunk + ks * 32, 16, 1024),
                        sdesc(st + A.a_bytes + nt * 256 * 128 + ks * 32, 16, 1024), A.idesc[nt],
                        (c != c0 || ks != 0) ? 1u : 0u);
          }
        }
        umma_commit(smem_u32(&empty[stage]));
        if (++stage == A.nstages) { stage = 0; phase ^= 1; }
      }
      umma_commit(smem_u32(done));
    }
  } else if (c1 > c0) {  // ---- epilogue: add this CTA's partial sums into dM
    const int sp = warp & 3;
    const int row = 32 * sp + lane;
    mbar_wait(smem_u32(done), 0);
    tc_fence_after();
    for (int mt = 0; mt < A.MT; ++mt) {
      const int o = mt * 128 + row;
      const uint32_t tcol = tmem + (static_cast<uint32_t>(32 * sp) << 16) + static_cast<uint32_t>(mt * A.Npad);
      for (int i0 = 0; i0 < A.Npad; i0 += 16) {
        uint32_t v[16];
        tmem_ld16(tcol + i0, v);
        if (o < A.Co) {
          float* dst = A.dM + static_cast<int64_t>(o) * A.Ci + i0;
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (i0 + q < A.Ci) atomicAdd(dst + q, __uint_as_float(v[q]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(A.tmem_cols) : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

int knob_mix_nt() {  // experiments only (GSPN_EXPERIMENTS + GSPN_MIX_NT=64|128|256)
  static const int v = [] {
    const char* e = getenv("GSPN_EXPERIMENTS") ? getenv("GSPN_MIX_NT") : nullptr;
    return e ? atoi(e) : 0;
  }();
  return v;
}

bool plan_mix(int64_t B, int64_t Ci, int64_t Co, int64_t HW, UmmaMixArgs& A) {
  if (Co > 512 || Ci > 4096 || HW % 8 != 0 || HW > (1ll << 31) - 1 || B > 65535) return false;
  A.MT = static_cast<int>((Co + 127) / 128);
  A.KC = static_cast<int>((Ci + kKC - 1) / kKC);
  // TMEM: 2 MT NT <= 512 columns (NT = 256 for MT = 1 measured the same as 128: knob GSPN_MIX_NT)
  A.NT = knob_mix_nt() && A.MT == 1 ? knob_mix_nt() : A.MT <= 2 ? 128 : 64;
  A.a_bytes = static_cast<uint32_t>(A.MT * A.KC) * kAChunk;
  A.stage_bytes = static_cast<uint32_t>(A.NT / 64) * kBBox;
  A.orows = static_cast<int>(std::min<int64_t>(128, (Co + 7) / 8 * 8));
  A.o_bytes = static_cast<uint32_t>(A.MT * (A.NT / 64) * A.orows) * 128u;  // one staging buffer (two are kept)
  const int budget = device_smem_optin() - 1024 - 256;
  A.nob = 2;
  int ns = (budget - static_cast<int>(A.a_bytes + 2 * A.o_bytes)) / static_cast<int>(A.stage_bytes);
  if (ns < 4) {  // keep the ring deep: one staging buffer
    A.nob = 1;
    ns = (budget - static_cast<int>(A.a_bytes + A.o_bytes)) / static_cast<int>(A.stage_bytes);
  }
  if (ns < 2) return false;
  A.nstages = std::min(ns, 8);
  const int cols = 2 * A.MT * A.NT;
  A.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  if (cols > 512) return false;
  A.B = static_cast<int>(B);
  A.Ci = static_cast<int>(Ci);
  A.Co = static_cast<int>(Co);
  A.HW = static_cast<int>(HW);
  A.ntn = static_cast<int>((HW + A.NT - 1) / A.NT);
  A.ntiles = static_cast<int64_t>(B) * A.ntn;
  // instruction descriptor: D f32, A / B bf16, A K-major, B MN-major, N = NT, M = 128
  A.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (static_cast<uint32_t>(A.NT >> 3) << 17) |
            (static_cast<uint32_t>(128 >> 4) << 24);
  return true;
}

bool plan_wgrad(int64_t B, int64_t Ci, int64_t Co, int64_t HW, UmmaWgradArgs& A) {
  if (Co > 512 || Ci > 512 || HW % 8 != 0 || HW > (1ll << 31) - 1 || B > 65535) return false;
  A.MT = static_cast<int>((Co + 127) / 128);
  A.Npad = static_cast<int>((Ci + 15) / 16 * 16);
  if (A.MT * A.Npad > 512) return false;
  A.BR = std::min(A.Npad, 256);       // B rows per TMA box
  A.NB = (A.Npad + A.BR - 1) / A.BR;
  A.a_bytes = static_cast<uint32_t>(A.MT) * kAChunk;
  A.stage_bytes = A.a_bytes + static_cast<uint32_t>(A.NB * A.BR) * 128u;
  const int budget = device_smem_optin() - 1024 - 256;
  const int ns = budget / static_cast<int>(A.stage_bytes);
  if (ns < 2) return false;
  A.nstages = std::min(ns, 8);
  const int cols = A.MT * A.Npad;
  A.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  A.B = static_cast<int>(B);
  A.Ci = static_cast<int>(Ci);
  A.Co = static_cast<int>(Co);
  A.HW = static_cast<int>(HW);
  A.nchb = static_cast<int>((HW + 63) / 64);
  A.nchunks = static_cast<int64_t>(B) * A.nchb;
  // D f32, A / B bf16, both K-major, M = 128; N = 256 for the first MMA when Npad > 256
  const uint32_t base = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(128 >> 4) << 24);
  const int n0 = std::min(A.Npad, 256), n1 = A.Npad - n0;
  A.idesc[0] = base | (static_cast<uint32_t>(n0 >> 3) << 17);
  A.idesc[1] = base | (static_cast<uint32_t>((n1 > 0 ? n1 : 16) >> 3) << 17);
  return true;
}

}  // namespace

bool umma_wgrad_eligible(int64_t B, int64_t Ci, int64_t Co, int64_t HW, gspn_dtype_t dt) {
  if (dt != GSPN_BF16) return false;
  UmmaWgradArgs A;
  memset(&A, 0, sizeof A);
  return plan_wgrad(B, Ci, Co, HW, A);
}

// dM must already be zeroed on `s` (the caller's memset); adds every CTA's partial sums.
cudaError_t launch_umma_wgrad(const void* dout, const void* in, float* dM, int64_t B, int64_t Ci, int64_t Co,
                              int64_t HW, cudaStream_t s) {
  std::unique_ptr<UmmaWgradArgs> hold(new UmmaWgradArgs());
  UmmaWgradArgs& A = *hold;
  memset(&A, 0, sizeof A);
  if (!plan_wgrad(B, Ci, Co, HW, A)) return cudaErrorNotSupported;
  A.dM = dM;
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint32_t estr[3] = {1, 1, 1};
  {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(HW), static_cast<cuuint64_t>(Co), static_cast<cuuint64_t>(B)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(HW * 2), static_cast<cuuint64_t>(Co * HW * 2)};
    cuuint32_t box[3] = {64, 128, 1};
    if (fn(&A.a_map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(dout), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorNotSupported;
  }
  {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(HW), static_cast<cuuint64_t>(Ci), static_cast<cuuint64_t>(B)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(HW * 2), static_cast<cuuint64_t>(Ci * HW * 2)};
    cuuint32_t box[3] = {64, static_cast<cuuint32_t>(A.BR), 1};
    if (fn(&A.b_map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(in), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorNotSupported;
  }
  const uint32_t smem = 1024 + A.nstages * A.stage_bytes + (2 * A.nstages + 1) * 8 + 16;
  cudaError_t e = cudaFuncSetAttribute(umma_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  // enough chunks per CTA to amortise the TMEM drain and the dM reduction
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(device_sm_count(), A.nchunks / 8));
  umma_wgrad_kernel<<<static_cast<unsigned>(grid), kMixThreads, smem, s>>>(A);
  return cudaGetLastError();
}

bool umma_mix_eligible(int64_t B, int64_t Ci, int64_t Co, int64_t HW, gspn_dtype_t dt) {
  if (dt != GSPN_BF16) return false;
  UmmaMixArgs A;
  memset(&A, 0, sizeof A);
  return plan_mix(B, Ci, Co, HW, A);
}

cudaError_t launch_umma_mix(const void* in, const void* M, void* out, int64_t B, int64_t Ci, int64_t Co, int64_t HW,
                            bool trans, cudaStream_t s) {
  std::unique_ptr<UmmaMixArgs> hold(new UmmaMixArgs());
  UmmaMixArgs& A = *hold;
  memset(&A, 0, sizeof A);
  if (!plan_mix(B, Ci, Co, HW, A)) return cudaErrorNotSupported;
  A.M = static_cast<const __nv_bfloat16*>(M);
  A.out = static_cast<__nv_bfloat16*>(out);
  A.trans = trans ? 1 : 0;
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(HW), static_cast<cuuint64_t>(Ci), static_cast<cuuint64_t>(B)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(HW * 2), static_cast<cuuint64_t>(Ci * HW * 2)};
  cuuint32_t box[3] = {64, 64, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  if (fn(&A.in_map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(in), dims, strides, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  {
    cuuint64_t odims[3] = {static_cast<cuuint64_t>(HW), static_cast<cuuint64_t>(Co), static_cast<cuuint64_t>(B)};
    cuuint64_t ostr[2] = {static_cast<cuuint64_t>(HW * 2), static_cast<cuuint64_t>(Co * HW * 2)};
    cuuint32_t obox[3] = {64, static_cast<cuuint32_t>(A.orows), 1};
    if (fn(&A.out_map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, out, odims, ostr, obox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorNotSupported;
  }
  const uint32_t smem = 1024 + A.a_bytes + A.nstages * A.stage_bytes + A.nob * A.o_bytes + (2 * A.nstages + 4) * 8 + 16;
  cudaError_t e = cudaFuncSetAttribute(umma_mix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int64_t grid = std::min<int64_t>(A.ntiles, device_sm_count());
  umma_mix_kernel<<<static_cast<unsigned>(grid), kMixThreads, smem, s>>>(A);
  return cudaGetLastError();
}

}  // namespace gspn
