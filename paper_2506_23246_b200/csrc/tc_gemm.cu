// FP32-accurate tensor-core GEMM (3xTF32 on tcgen05) for the trunk.
//
// C[M,N] = A[M,K] B[N,K]^T, fp32 in / fp32 out, both operands K-major
// (row-major with K contiguous).  Persistent CTAs walk 128 x BN output tiles;
// per CTA (448 threads):
//   warp 12     TMA producer for A (fp32), 32 K-columns (one 128-byte swizzle
//               row) per stage; lane 1 of the same warp (independently
//               scheduled) produces the pre-split B_hi / B_lo tiles
//   warps 0-3   split A into A_hi / A_lo operand buffers
//   warp 13     MMA issuer (one thread): per stage 4 K-steps x 3 products
//               A_lo B_hi + A_hi B_lo + A_hi B_hi into a fresh TMEM buffer
//   warps 4-11  promote every k-block partial from TMEM into fp32 registers
//               (warps w, w + 4 share TMEM lanes 32 (w % 4).., half the columns each)
//               (the tensor core's own fp32 accumulation truncates, so long
//               K chains drift; 32-deep partials + IEEE adds stay FP32-class)
//               and run the fused epilogue, overlapping the next tile's MMAs
// Epilogues: plain store, or the dual tanh of a dense layer with tangents
// (network.py:294-298 on ops.py:282-298): rows are [value; d/dx; d/dy; d/dt]
// blocks of the same 32 points, y = tanh(u0 + b), dy_k = (1 - y^2) du_k.
// B (the layer weights, small) is split once per call into a workspace.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "tc_gemm.cuh"
#include "tc_gemm.h"

namespace qpinn {
namespace tc {

#ifdef QPINN_GEMM_PROF
__device__ unsigned long long g_gemm_prof[16];
#define GPROF(slot, call)                                                    \
  do {                                                                       \
    const long long _t0 = clock64();                                         \
    call;                                                                    \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0)                          \
      atomicAdd(&g_gemm_prof[slot], (unsigned long long)(clock64() - _t0));  \
  } while (0)
#else
#define GPROF(slot, call) call
#endif
// Ablation switches for timing experiments (scripts/gemm_ablate.sh); all 0 in
// the shipped build.  NOSTORE: epilogue skips the output stores; NOPROMO: one
// TMEM read per tile instead of one per promotion group; NOSPLIT: the split
// warps skip the hi/lo split (stale operands); NOMMA: commits without MMAs.
#ifndef QPINN_ABL_NOSTORE
#define QPINN_ABL_NOSTORE 0
#endif
#ifndef QPINN_ABL_NOPROMO
#define QPINN_ABL_NOPROMO 0
#endif
#ifndef QPINN_ABL_NOSPLIT
#define QPINN_ABL_NOSPLIT 0
#endif
#ifndef QPINN_ABL_NOMMA
#define QPINN_ABL_NOMMA 0
#endif
#ifndef QPINN_ABL_NOB  // B tiles loaded once per CTA (stale after), not per k-block
#define QPINN_ABL_NOB 0
#endif
constexpr int kBM = 128, kBK = 32;
// k-blocks accumulated in one TMEM buffer before the epilogue warps add it into
// fp32 registers.  1: 32-deep tensor-core chains, 3.5e-7 relative at K = 256;
// 2: 64-deep, 6.3e-7 relative, still below cuBLAS SIMT fp32 on the same inputs
// (max |err| 3.6e-6 vs 4.1e-6, scripts/gemm_check.py), and -60 us per training
// step (half the TMEM reads of the promotion; the dual-tanh layers are
// epilogue-paced); 4: 1.2e-6, above SIMT fp32, not used
#ifndef QPINN_GEMM_PROMOTE
#define QPINN_GEMM_PROMOTE 2
#endif
constexpr int kPromote = QPINN_GEMM_PROMOTE;
constexpr int kABytes = kBM * kBK * 4;  // 16 KB fp32 tile
constexpr int kThreadsGemm = 448;  // 4 split + 8 epilogue + producer + MMA warps
constexpr int kThreadsW = 320;      // weight gradient: 4 split + 4 epilogue + producer + MMA
enum { EPI_STORE = 0, EPI_TANH = 1, EPI_TANH1 = 2, EPI_READOUT = 3 };  // TANH1: value channel only
// EPI_READOUT: the transfer-matrix map of the PQC (pqc_transfer.cu): rows are the
// embedded magnitudes of 32 points x [state; d/dx; d/dy; d/dt] (as EPI_TANH), the
// N = 2D output columns are [Re psi | Im psi]; besides storing Psi the epilogue
// reduces the Pauli-Z readout z_q = sum_b s_bq |psi_b|^2, dz_kq = sum_b s_bq
// 2 Re(conj psi_b dpsi_kb) (qsim.py:369-381), which is separable over the Re and
// Im halves, so a CTA runs both N-tiles of its M-tile back to back and adds them
template <int EPI>
constexpr bool kRowsByPoint = EPI == EPI_TANH || EPI == EPI_READOUT;

template <int BN>
struct GemmCfg {
  static constexpr int kBBytes = BN * kBK * 4;
#ifndef QPINN_GEMM_RAW
#define QPINN_GEMM_RAW 3
#endif
#ifndef QPINN_GEMM_BS
#define QPINN_GEMM_BS 2
#endif
#ifndef QPINN_GEMM_ATMEM
#define QPINN_GEMM_ATMEM 1
#endif
  // split A operands in TMEM (the MMA then reads only B from shared memory,
  // whose bandwidth bounds the 3-product TF32 MMAs otherwise), else in smem
  static constexpr bool kATmem = QPINN_GEMM_ATMEM;
  static constexpr int kRaw = QPINN_GEMM_RAW;   // fp32 A stages in flight from HBM
#ifndef QPINN_GEMM_OS
#define QPINN_GEMM_OS 2
#endif
#ifndef QPINN_GEMM_NB
#define QPINN_GEMM_NB 3
#endif
  static constexpr int kOps = kATmem ? QPINN_GEMM_OS : 2;   // split A buffers (A_hi, A_lo)
  static constexpr int kOpBytes = kATmem ? 0 : 2 * kABytes;
  static constexpr int kBS = QPINN_GEMM_BS;    // B_hi / B_lo stages (from L2)
  static constexpr int kBStage = 2 * kBBytes;
  static constexpr int kNB = kATmem ? QPINN_GEMM_NB : 4;    // TMEM partial buffers
  static constexpr int kACol = kNB * BN;        // TMEM: [NB partials | OS x (A_hi, A_lo)]
  static constexpr int kTmemCols = kATmem ? 512 : kNB * BN;
  static_assert(!kATmem || kNB * BN + kOps * 2 * kBK <= 512, "TMEM columns");
  static constexpr int kSbuf = 32 * BN * 4;
  static constexpr int kStg = 8 * 2 * 2048;  // per epilogue warp: 2 x (16 rows x 32 cols)
  // EPI_READOUT / fused adapter: column-half partials [4][32][8], adapter
  // weights [BN][8], adapter values [32][8]
  static constexpr int kRed = (4 * 32 * 8 + BN * 8 + 32 * 8) * 4;
  static constexpr int kSmem =
      kRaw * kABytes + kOps * kOpBytes + kBS * kBStage + kSbuf + kStg + kRed + 1024 + 512;
};

struct GemmArgs {
  int64_t M;      // rows of A / C (EPI_TANH: 4 R)
  int64_t R;      // EPI_TANH: points per channel block
  int N, K;
  float* C;
  int64_t ldc;
  const float* bias;  // EPI_TANH
  int tma_store;      // C goes out through TMA (16-byte aligned rows), else direct stores
  float* z;           // EPI_READOUT: z [R, NQ], dz [3, R, NQ]
  float* dz;
  // EPI_TANH with a fused adapter (network.py:298-299): act [4, R, n_ad] = dual
  // tanh(y Wa + ba) of this layer's output y, Wa [N, n_ad] row-major (N <= BN)
  const float* ad_w;
  const float* ad_b;
  float* act;
  int n_ad;
};

// one epilogue warp's 32 rows x CW columns (lane = row) -> global through two
// alternating 2 KB staging buffers (16 rows x 32 columns, 128-byte swizzled,
// conflict-free) and TMA stores of 32 x 16 boxes at (col0 + c, row0 + 16 h, blk)
// of the 3-D output map; a buffer is rewritten once the store before last has
// read it, so one store is always in flight while the next box is staged
template <int CW>
__device__ __forceinline__ void store_rows_tma(const float (&acc)[CW], unsigned char* buf,
                                               const CUtensorMap* mC, int col0, int row0,
                                               int blk, int lane, uint32_t& sidx) {
#pragma unroll
  for (int c0 = 0; c0 < CW; c0 += 32) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      unsigned char* sb = buf + (sidx++ & 1) * 2048;
      if (lane == 0) bulk_wait_read1();
      __syncwarp();
      if ((lane >> 4) == h) {
        const uint32_t base = smem_u32(sb) + (lane & 15) * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          sts128(base + ((j ^ (lane & 7)) << 4),
                 make_float4(acc[c0 + 4 * j], acc[c0 + 4 * j + 1], acc[c0 + 4 * j + 2],
                             acc[c0 + 4 * j + 3]));
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_3d(mC, sb, col0 + c0, row0 + 16 * h, blk);
        bulk_commit();
      }
    }
  }
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreadsGemm, 1)
gemm3_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mBhi,
             const __grid_constant__ CUtensorMap mBlo, const __grid_constant__ CUtensorMap mC,
             const GemmArgs g) {
  using Cfg = GemmCfg<BN>;
  constexpr int RS = Cfg::kRaw, OS = Cfg::kOps, BS = Cfg::kBS, NB = Cfg::kNB;
#ifndef QPINN_GEMM_SHARE_EMPTY
#define QPINN_GEMM_SHARE_EMPTY 1
#endif
  constexpr bool kShareEmpty = QPINN_GEMM_SHARE_EMPTY && OS == BS;
#ifndef QPINN_GEMM_GC
#define QPINN_GEMM_GC 0
#endif
  // group commit (experiment): one MMA commit per promotion group (tfull) frees
  // that group's A operand stages and B stages too; needs nk % kPromote == 0
  constexpr bool kGC = QPINN_GEMM_GC;
  const int ngrp_t = (g.K + kBK * kPromote - 1) / (kBK * kPromote);  // groups per tile
  auto group_of = [&](int64_t jj) -> int64_t {  // promotion group of global k-block jj
    const int nkk = (g.K + kBK - 1) / kBK;
    return (jj / nkk) * ngrp_t + (jj % nkk) / kPromote;
  };
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte aligned by offsetting the shared array itself, so pointers derived
  // from it keep the shared address space (LDS/STS rather than generic LD/ST)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* raw = smem;                        // [RS][16 KB] fp32 A tiles
  unsigned char* ops = smem + RS * kABytes;         // [OS][A_hi | A_lo]
  unsigned char* bst = ops + OS * Cfg::kOpBytes;    // [BS][B_hi | B_lo]
  float* sbuf = (float*)(bst + BS * Cfg::kBStage);
  unsigned char* stg = (unsigned char*)sbuf + Cfg::kSbuf;  // [4 warps][2][4 KB]
  float* red = (float*)(stg + Cfg::kStg);                    // [4][32][8]
  uint64_t* raw_full = (uint64_t*)(stg + Cfg::kStg + Cfg::kRed);
  uint64_t* raw_empty = raw_full + RS;
  uint64_t* b_full = raw_empty + RS;
  uint64_t* b_empty = b_full + BS;
  uint64_t* conv = b_empty + BS;
  uint64_t* op_empty = conv + OS;
  uint64_t* tfull = op_empty + OS;
  uint64_t* tempty = tfull + NB;
  uint32_t* tmem_slot = (uint32_t*)(tempty + NB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef QPINN_GEMM_PROF
  const long long prof_t0 = clock64();
#endif
  const int nk = (g.K + kBK - 1) / kBK;
  const int64_t n_mt = kRowsByPoint<EPI> ? (g.R + 31) / 32 : (g.M + kBM - 1) / kBM;
  const int n_nt = (g.N + BN - 1) / BN;
  // tiles: a CTA walks M-tiles and runs all N-tiles of each back to back

  if (threadIdx.x == 0) {
    for (int s = 0; s < RS; ++s) {
      mbar_init(raw_full + s, 1);
      mbar_init(raw_empty + s, 4);
    }
    for (int s = 0; s < OS; ++s) {
      mbar_init(conv + s, 4);
      mbar_init(op_empty + s, 1);
    }
    for (int s = 0; s < BS; ++s) {
      mbar_init(b_full + s, 1);
      mbar_init(b_empty + s, 1);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(tfull + b, 1);
      mbar_init(tempty + b, 8);
    }
    mbar_init_fence();
  }
  if (warp == 12 && lane == 0) {
    tma_prefetch(&mA);
    tma_prefetch(&mBhi);
    tma_prefetch(&mBlo);
  }
  if (warp == 13) tmem_alloc(tmem_slot, Cfg::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 12) {  // ---- TMA producer for A (runs RS k-blocks ahead)
    if (lane == 0) {
      int64_t j = 0;
      for (int64_t mt = blockIdx.x; mt < n_mt; mt += gridDim.x)
      for (int nt = 0; nt < n_nt; ++nt) {
        for (int kb = 0; kb < nk; ++kb, ++j) {
          const int r = (int)(j % RS);
          if (j >= RS) GPROF(0, mbar_wait(raw_empty + r, (uint32_t)(((j / RS) - 1) & 1)));
          unsigned char* st = raw + r * kABytes;
          mbar_expect_tx(raw_full + r, kABytes);
          if constexpr (kRowsByPoint<EPI>) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
              tma_load_2d(st + c * (kABytes / 4), &mA, raw_full + r, kb * kBK,
                          (int)(c * g.R + mt * 32));
          } else {
            tma_load_2d(st, &mA, raw_full + r, kb * kBK, (int)(mt * kBM));
          }
        }
      }
    }
  }
  if (warp == 12) {  // ---- TMA producer for the split B tiles (L2-resident), lane 1
    if (lane == 1) {
      int64_t j = 0;
      for (int64_t mt = blockIdx.x; mt < n_mt; mt += gridDim.x)
      for (int nt = 0; nt < n_nt; ++nt) {
        for (int kb = 0; kb < nk; ++kb, ++j) {
          const int e = (int)(j % BS);
          // with as many B stages as A operand stages one MMA commit frees both
          // (each tcgen05.commit costs tensor-pipe throughput while TMA loads are in
          // flight: scripts/probes/mma_rate.cu, 72 -> 97 cycles per MMA at 2 per k-block)
          uint64_t* freed = kShareEmpty ? op_empty : b_empty;
          if (kGC) {
            if (j >= BS) {
              const int64_t gq = group_of(j - BS);
              mbar_wait(tfull + (int)(gq % NB), (uint32_t)((gq / NB) & 1));
            }
          } else if (j >= BS) GPROF(1, mbar_wait(freed + e, (uint32_t)(((j / BS) - 1) & 1)));
          unsigned char* st = bst + e * Cfg::kBStage;
          if (QPINN_ABL_NOB && j >= BS) {
            mbar_arrive(b_full + e);
            continue;
          }
          mbar_expect_tx(b_full + e, 2 * Cfg::kBBytes);
          tma_load_2d(st, &mBhi, b_full + e, kb * kBK, nt * BN);
          tma_load_2d(st + Cfg::kBBytes, &mBlo, b_full + e, kb * kBK, nt * BN);
        }
      }
    }
  } else if (warp == 13) {  // ---- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(kBM, BN);
      int64_t j = 0, grp = 0;
      for (int64_t mt = blockIdx.x; mt < n_mt; mt += gridDim.x)
      for (int nt = 0; nt < n_nt; ++nt) {
        for (int kb = 0; kb < nk; ++kb, ++j) {
          const int o = (int)(j % OS), e = (int)(j % BS), b = (int)(grp % NB);
          const bool first = kb % kPromote == 0;
          const bool last = kb % kPromote == kPromote - 1 || kb == nk - 1;
          if (first && grp >= NB) GPROF(2, mbar_wait(tempty + b, (uint32_t)(((grp / NB) - 1) & 1)));
          GPROF(3, mbar_wait(conv + o, (uint32_t)((j / OS) & 1)));
          GPROF(4, mbar_wait(b_full + e, (uint32_t)((j / BS) & 1)));
          tc_fence_after();
          const uint32_t b_hi = smem_u32(bst + e * Cfg::kBStage);
          const uint32_t b_lo = b_hi + Cfg::kBBytes;
          const uint32_t d = tmem + b * BN;
          if constexpr (QPINN_ABL_NOMMA) {
          } else if constexpr (Cfg::kATmem) {
            const uint32_t a_hi = tmem + Cfg::kACol + o * 2 * kBK, a_lo = a_hi + kBK;
#pragma unroll
            for (int k = 0; k < kBK / 8; ++k) {
              const uint32_t off = k * 32;  // 8 tf32 = 32 bytes along the swizzled B row
              mma_tf32_ts(d, a_lo + k * 8, desc_k_sw128(b_hi + off), idesc, !(first && k == 0));
              mma_tf32_ts(d, a_hi + k * 8, desc_k_sw128(b_lo + off), idesc, 1);
              mma_tf32_ts(d, a_hi + k * 8, desc_k_sw128(b_hi + off), idesc, 1);
            }
          } else {
            const uint32_t a_hi = smem_u32(ops + o * Cfg::kOpBytes);
            const uint32_t a_lo = a_hi + kABytes;
#pragma unroll
            for (int k = 0; k < kBK / 8; ++k) {
              const uint32_t off = k * 32;  // 8 tf32 = 32 bytes along the swizzled row
              mma_tf32(d, desc_k_sw128(a_lo + off), desc_k_sw128(b_hi + off), idesc,
                       !(first && k == 0));
              mma_tf32(d, desc_k_sw128(a_hi + off), desc_k_sw128(b_lo + off), idesc, 1);
              mma_tf32(d, desc_k_sw128(a_hi + off), desc_k_sw128(b_hi + off), idesc, 1);
            }
          }
          if (!kGC) mma_commit(op_empty + o);
          if (!kGC && !kShareEmpty) mma_commit(b_empty + e);
          if (last) {
            mma_commit(tfull + b);
            ++grp;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < 4 && Cfg::kATmem) {  // ---- split A into TMEM (warp w: lanes 32 w ..)
    // thread = tile row = TMEM lane; the row's 8 16-byte chunks sit at c ^ (row & 7)
    const int row = warp * 32 + lane;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    int64_t j = 0;
    for (int64_t mt = blockIdx.x; mt < n_mt; mt += gridDim.x)
      for (int nt = 0; nt < n_nt; ++nt) {
      for (int kb = 0; kb < nk; ++kb, ++j) {
        const int r = (int)(j % RS), o = (int)(j % OS);
        if (j >= OS) {
          if (kGC) {
            const int64_t gq = group_of(j - OS);
            mbar_wait(tfull + (int)(gq % NB), (uint32_t)((gq / NB) & 1));
          } else if (warp == 0) GPROF(5, mbar_wait(op_empty + o, (uint32_t)(((j / OS) - 1) & 1)));
          else mbar_wait(op_empty + o, (uint32_t)(((j / OS) - 1) & 1));
          tc_fence_after();
        }
        if (warp == 0) GPROF(6, mbar_wait(raw_full + r, (uint32_t)((j / RS) & 1)));
        else mbar_wait(raw_full + r, (uint32_t)((j / RS) & 1));
        if constexpr (QPINN_ABL_NOSPLIT) {
          fence_proxy_async_smem();  // generic reads of the raw stage before its TMA refill
          __syncwarp();
          if (lane == 0) mbar_arrive(raw_empty + r);
        } else {
        const uint32_t src = smem_u32(raw + r * kABytes) + row * 128;
        float4 v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = lds128(src + ((c ^ (row & 7)) << 4));
        float hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          split_tf32(v[c].x, hi[4 * c], lo[4 * c]);
          split_tf32(v[c].y, hi[4 * c + 1], lo[4 * c + 1]);
          split_tf32(v[c].z, hi[4 * c + 2], lo[4 * c + 2]);
          split_tf32(v[c].w, hi[4 * c + 3], lo[4 * c + 3]);
        }
        // the raw stage is refilled by TMA (async proxy) once raw_empty completes: order
        // this thread's generic-proxy reads of it before that write (without the fence
        // one row in ~10^4 tiles read the next k-block's data: scripts/race_gemm.py)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(raw_empty + r);
        const uint32_t a = tmem + lane_base + Cfg::kACol + o * 2 * kBK;
        tmem_st32(a, hi);
        tmem_st32(a + kBK, lo);
        tmem_st_wait();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(conv + o);
      }
    }
  } else if (warp < 4) {  // ---- split A into an operand buffer
    int64_t j = 0;
    for (int64_t mt = blockIdx.x; mt < n_mt; mt += gridDim.x)
      for (int nt = 0; nt < n_nt; ++nt) {
      for (int kb = 0; kb < nk; ++kb, ++j) {
        const int r = (int)(j % RS), o = (int)(j % OS);
        if (j >= OS) mbar_wait(op_empty + o, (uint32_t)(((j / OS) - 1) & 1));
        unsigned char* op = ops + o * Cfg::kOpBytes;
        mbar_wait(raw_full + r, (uint32_t)((j / RS) & 1));
        // layout-free: the swizzled tile is split as flat 16-byte chunks; all
        // loads first (one latency per k-block), then split and store
        const uint32_t a_src = smem_u32(raw + r * kABytes) + threadIdx.x * 16;
        const uint32_t a_dst = smem_u32(op) + threadIdx.x * 16;
        constexpr int CH = kABytes / 16 / 128;  // chunks per thread
        float4 v[CH];
#pragma unroll
        for (int i = 0; i < CH; ++i) v[i] = lds128(a_src + i * 2048);
#pragma unroll
        for (int i = 0; i < CH; ++i) {
          float4 h, l;
          split_tf32(v[i].x, h.x, l.x);
          split_tf32(v[i].y, h.y, l.y);
          split_tf32(v[i].z, h.z, l.z);
          split_tf32(v[i].w, h.w, l.w);
          sts128(a_dst + i * 2048, h);
          sts128(a_dst + kABytes + i * 2048, l);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(raw_empty + r);
          mbar_arrive(conv + o);
        }
      }
    }
  } else {  // ---- warps 4-11: promote partials, epilogue
    // warp w reads TMEM lanes 32 (w % 4) ..; warps w and w + 4 split the columns
    const int q = warp & 3, h = (warp - 4) >> 2;
    constexpr int CW = BN / 2;  // columns per epilogue warp
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    unsigned char* my_stg = stg + (warp - 4) * 2 * 2048;
    uint32_t sidx = 0;
    int64_t j = 0;
    float zr[8];  // EPI_READOUT: readout partials of this row over the N-tiles
    float* s_wa = red + 4 * 32 * 8;   // fused adapter weights [BN][8]
    float* s_a = s_wa + BN * 8;        // adapter values of the tile's points [32][8]
    if (EPI == EPI_TANH && g.ad_w) {
      for (int i = threadIdx.x - 128; i < BN * 8; i += 256) {
        const int c = i >> 3, jj = i & 7;
        s_wa[i] = (c < g.N && jj < g.n_ad) ? g.ad_w[(int64_t)c * g.n_ad + jj] : 0.f;
      }
    }
    for (int64_t mt = blockIdx.x; mt < n_mt; mt += gridDim.x)
      for (int nt = 0; nt < n_nt; ++nt) {
      const int n0 = nt * BN, c_off = h * CW;
      float acc[CW];
#pragma unroll
      for (int c = 0; c < CW; ++c) acc[c] = 0.f;
      const int ngrp = (nk + kPromote - 1) / kPromote;
      for (int gi = 0; gi < ngrp; ++gi, ++j) {  // j counts promotion groups here
        const int b = (int)(j % NB);
        if (warp == 4) GPROF(7, mbar_wait(tfull + b, (uint32_t)((j / NB) & 1)));
        else mbar_wait(tfull + b, (uint32_t)((j / NB) & 1));
        tc_fence_after();
        if (!QPINN_ABL_NOPROMO || gi == ngrp - 1) {
#pragma unroll
          for (int c0 = 0; c0 < CW; c0 += 32) {
            float v[32];
            tmem_ld32(tmem + lane_base + b * BN + c_off + c0, v);
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[c0 + i] += v[i];
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty + b);
      }
      if constexpr (EPI == EPI_STORE || EPI == EPI_TANH1) {
        if constexpr (EPI == EPI_TANH1) {  // y = tanh(u + b), no tangents
#pragma unroll
          for (int c = 0; c < CW; ++c) {
            const int col = n0 + c_off + c;
            acc[c] = tanhf(acc[c] + (col < g.N ? __ldg(g.bias + col) : 0.f));
          }
        }
        const int64_t row = mt * kBM + q * 32 + lane;
        if (QPINN_ABL_NOSTORE) {
          if (acc[0] == 1.2345e-30f) g.C[0] = acc[CW - 1];
        } else if (g.tma_store) {
          if (warp == 4)
            GPROF(8, (store_rows_tma<CW>(acc, my_stg, &mC, n0 + c_off, (int)(mt * kBM + q * 32), 0,
                                         lane, sidx)));
          else
            store_rows_tma<CW>(acc, my_stg, &mC, n0 + c_off, (int)(mt * kBM + q * 32), 0, lane, sidx);
        } else if (row < g.M) {
          float* dst = g.C + row * g.ldc + n0 + c_off;
#pragma unroll
          for (int c = 0; c < CW; ++c)
            if (n0 + c_off + c < g.N) dst[c] = acc[c];
        }
      } else if constexpr (EPI == EPI_READOUT) {  // q = channel, lane = point, b = c_off + c
        static_assert(BN == 128, "readout epilogue: one N-tile = the Re or Im half (D = 128)");
        const int64_t p = mt * 32 + lane;
        if (g.tma_store) store_rows_tma<CW>(acc, my_stg, &mC, n0 + c_off, (int)(mt * 32), q, lane, sidx);
        if (q == 0) {
#pragma unroll
          for (int c = 0; c < CW; ++c) sbuf[(c_off + c) * 32 + lane] = acc[c];
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        // v_b = psi_b^2 (state row) or 2 psi_b dpsi_kb (tangent row k); wire w of the
        // 7 qubits is bit 6 - w of b: bit 6 is this warp's column half h, bits 0-5 of c
        float part[7];
#pragma unroll
        for (int w = 0; w < 7; ++w) part[w] = 0.f;
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          const float ps = sbuf[(c_off + c) * 32 + lane];
          const float v = q == 0 ? acc[c] * acc[c] : 2.f * ps * acc[c];
          part[0] += v;
#pragma unroll
          for (int w = 1; w < 7; ++w) part[w] += ((c >> (6 - w)) & 1) ? -v : v;
        }
        if (h) part[0] = -part[0];
        if (h == 1) {
#pragma unroll
          for (int w = 0; w < 7; ++w) red[(q * 32 + lane) * 8 + w] = part[w];
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (h == 0) {
#pragma unroll
          for (int w = 0; w < 7; ++w) {
            const float t = part[w] + red[(q * 32 + lane) * 8 + w];
            zr[w] = nt == 0 ? t : zr[w] + t;
          }
          if (nt == n_nt - 1 && p < g.R) {
            float* dst = q == 0 ? g.z + p * 7 : g.dz + ((int64_t)(q - 1) * g.R + p) * 7;
#pragma unroll
            for (int w = 0; w < 7; ++w) dst[w] = zr[w];
          }
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");  // sbuf / red reused by the next tile
      } else {  // EPI_TANH: q = channel, lane = point
        // the value channel's pre-activations go through shared memory so that
        // all eight warps share the tanh work (BN / 8 columns each)
        const int64_t p = mt * 32 + lane;
        if (q == 0) {
#pragma unroll
          for (int c = 0; c < CW; ++c) sbuf[(c_off + c) * 32 + lane] = acc[c];
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        const int e = warp - 4;
#pragma unroll 4
        for (int c = e * (BN / 8); c < (e + 1) * (BN / 8); ++c) {
          const float bv = n0 + c < g.N ? __ldg(g.bias + n0 + c) : 0.f;
          sbuf[c * 32 + lane] = tanhf(sbuf[c * 32 + lane] + bv);
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          const float y = sbuf[(c_off + c) * 32 + lane];
          acc[c] = q == 0 ? y : (1.f - y * y) * acc[c];
        }
        if (g.tma_store) {
          store_rows_tma<CW>(acc, my_stg, &mC, n0 + c_off, (int)(mt * 32), q, lane, sidx);
        } else if (p < g.R) {
          float* dst = g.C + ((int64_t)q * g.R + p) * g.ldc + n0 + c_off;
#pragma unroll
          for (int c = 0; c < CW; ++c)
            if (n0 + c_off + c < g.N) dst[c] = acc[c];
        }
        if (g.ad_w) {  // fused adapter: u = y Wa per row (fp32 FMA, two column halves)
          // weight rows by explicit shared-memory loads (broadcast); with generic
          // pointers they compiled to generic LDs: 291 -> 273 us for the step's three
          // EPI_TANH launches together with the static-index store below
          float u[8];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) u[jj] = 0.f;
          const uint32_t wa0 = smem_u32(s_wa + c_off * 8);
#pragma unroll
          for (int c = 0; c < CW; ++c) {
            const float4 w0 = lds128(wa0 + c * 32), w1 = lds128(wa0 + c * 32 + 16);
            u[0] = fmaf(acc[c], w0.x, u[0]);
            u[1] = fmaf(acc[c], w0.y, u[1]);
            u[2] = fmaf(acc[c], w0.z, u[2]);
            u[3] = fmaf(acc[c], w0.w, u[3]);
            u[4] = fmaf(acc[c], w1.x, u[4]);
            u[5] = fmaf(acc[c], w1.y, u[5]);
            u[6] = fmaf(acc[c], w1.z, u[6]);
            u[7] = fmaf(acc[c], w1.w, u[7]);
          }
          if (h == 1) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) red[(q * 32 + lane) * 8 + jj] = u[jj];
          }
          asm volatile("bar.sync 1, 256;" ::: "memory");
          if (h == 0) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) u[jj] += red[(q * 32 + lane) * 8 + jj];
            if (q == 0) {
#pragma unroll
              for (int jj = 0; jj < 8; ++jj)
                s_a[lane * 8 + jj] = jj < g.n_ad ? tanhf(u[jj] + __ldg(g.ad_b + jj)) : 0.f;
            }
          }
          asm volatile("bar.sync 1, 256;" ::: "memory");
          if (h == 0 && p < g.R) {  // a = tanh(u0 + ba); da_k = (1 - a^2) u_k
            float* dst = g.act + ((int64_t)q * g.R + p) * g.n_ad;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {  // static indices: u stays in registers
              if (jj < g.n_ad) {
                const float a = s_a[lane * 8 + jj];
                dst[jj] = q == 0 ? a : (1.f - a * a) * u[jj];
              }
            }
          }
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");  // sbuf reused by the next tile
      }
    }
  }
  if (warp >= 4 && warp < 12 && lane == 0) bulk_wait_all();
  tc_fence_before();
  __syncthreads();
  if (warp == 13) tmem_dealloc(tmem, Cfg::kTmemCols);
#ifdef QPINN_GEMM_PROF
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&g_gemm_prof[9], (unsigned long long)(clock64() - prof_t0));
#endif
}


// ---- CTA-pair variant (cta_group::2) ------------------------------------------------
// Same roles and numerics as gemm3_kernel, on a cluster of two CTAs (one TPC):
// each pair tile is 256 rows x BN columns, CTA r owning rows 128 r.. (A operand
// and accumulator in its own TMEM).  The leader (r = 0) issues
// tcgen05.mma.cta_group::2; B's BN rows are split in halves between the CTAs'
// shared memory (scripts/probes/mma_2cta.cu), so every SM stores and feeds the
// tensor core only half of B per MMA.  B (the layer weights, split hi/lo) stays
// RESIDENT in shared memory for the whole kernel: a pair walks M-tiles of one
// fixed N-tile, so no B traffic per k-block at all.  Together this halves the
// shared-memory bandwidth the single-CTA kernel needs per k-block (~157 B/cycle
// at the MMA rate by a per-cycle budget, against 128 B/cycle per SM).  Measured:
// slower than the single-CTA kernel (see use_pair), so it is opt-in.
// Cross-CTA signalling: the split and epilogue warps of CTA 1 arrive on the
// leader's conv / tempty barriers remotely; the leader's commits multicast to
// both CTAs' op_empty / tfull.
template <int BN>
struct PairCfg {
  static constexpr int HB = BN / 2;                 // B rows held per CTA
  static constexpr int kSlab = HB * kBK * 4;        // one k-block of B_hi (or B_lo) half
  // 4 TMEM A stages, 2 partial buffers: one MMA commit per promotion group (2
  // k-blocks) frees the group's A stages AND publishes its partial
  // (tcgen05.commit costs ~150 tensor-pipe cycles while TMA loads are in flight,
  // scripts/probes/mma_rate.cu), instead of one per k-block plus one per group
  static constexpr int RS = 3, OS = 4, NB = 2;
  static constexpr int kACol = NB * BN;
  static_assert(NB * BN + OS * 2 * kBK <= 512, "TMEM columns");
  static constexpr int kSbuf = 32 * BN * 4;
  static constexpr int kStg = 8 * 2 * 2048;
  static size_t smem(int nk) {
    return (size_t)RS * kABytes + 2 * (size_t)nk * kSlab + kSbuf + kStg + 1024 + 512;
  }
};

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreadsGemm, 1)
gemm3_pair_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mBhi,
                  const __grid_constant__ CUtensorMap mBlo, const __grid_constant__ CUtensorMap mC,
                  const GemmArgs g) {
  using Cfg = PairCfg<BN>;
  constexpr int RS = Cfg::RS, OS = Cfg::OS, NB = Cfg::NB, HB = Cfg::HB;
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte aligned by offsetting the shared array itself, so pointers derived
  // from it keep the shared address space (LDS/STS rather than generic LD/ST)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int nk = (g.K + kBK - 1) / kBK;
  unsigned char* raw = smem;                                  // [RS][16 KB] fp32 A tiles
  unsigned char* bres = raw + RS * kABytes;                   // [hi: nk slabs][lo: nk slabs]
  float* sbuf = (float*)(bres + 2 * (size_t)nk * Cfg::kSlab);
  unsigned char* stg = (unsigned char*)sbuf + Cfg::kSbuf;
  uint64_t* raw_full = (uint64_t*)(stg + Cfg::kStg);
  uint64_t* raw_empty = raw_full + RS;
  uint64_t* b_full = raw_empty + RS;
  uint64_t* conv = b_full + 1;
  uint64_t* gdone = conv + OS;    // per partial buffer: the group's MMAs completed
  uint64_t* tempty = gdone + NB;
  uint32_t* tmem_slot = (uint32_t*)(tempty + NB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int64_t pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int64_t n_mt = EPI == EPI_TANH ? (g.R + 63) / 64 : (g.M + 255) / 256;
  const int n_nt = (g.N + BN - 1) / BN;
  const int64_t G = n_pairs / n_nt;                // pairs per N-tile
  const bool active = pair < G * n_nt;
  const int nt = (int)(pair % n_nt);
  const int64_t mt0 = active ? pair / n_nt : n_mt, mstep = G > 0 ? G : 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < RS; ++s) {
      mbar_init(raw_full + s, 1);
      mbar_init(raw_empty + s, 4);
    }
    mbar_init(b_full, 1);
    for (int s = 0; s < OS; ++s) mbar_init(conv + s, 8);  // 4 split warps x 2 CTAs (leader)
    for (int b = 0; b < NB; ++b) {
      mbar_init(gdone + b, 1);     // multicast commit
      mbar_init(tempty + b, 16);   // 8 epilogue warps x 2 CTAs (leader's barrier)
    }
    mbar_init_fence();
  }
  if (warp == 12 && lane == 0) {
    tma_prefetch(&mA);
    tma_prefetch(&mBhi);
    tma_prefetch(&mBlo);
  }
  if (warp == 13) tmem_alloc2(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // this CTA's half of the split B, resident for the whole kernel
  if (warp == 12 && lane == 1 && active) {
    mbar_expect_tx(b_full, 2u * nk * Cfg::kSlab);
    for (int kb = 0; kb < nk; ++kb) {
      tma_load_2d(bres + (size_t)kb * Cfg::kSlab, &mBhi, b_full, kb * kBK, nt * BN + rank * HB);
      tma_load_2d(bres + (size_t)(nk + kb) * Cfg::kSlab, &mBlo, b_full, kb * kBK,
                  nt * BN + rank * HB);
    }
  }
  if (active) mbar_wait(b_full, 0);
  cluster_sync();  // the leader's MMAs read both halves from here on

  if (warp == 12) {  // ---- TMA producer for A (this CTA's 128 rows of the pair tile)
    if (lane == 0) {
      int64_t j = 0;
      for (int64_t mt = mt0; mt < n_mt; mt += mstep) {
        for (int kb = 0; kb < nk; ++kb, ++j) {
          const int r = (int)(j % RS);
          if (j >= RS) mbar_wait(raw_empty + r, (uint32_t)(((j / RS) - 1) & 1));
          unsigned char* st = raw + r * kABytes;
          mbar_expect_tx(raw_full + r, kABytes);
          if constexpr (EPI == EPI_TANH) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
              tma_load_2d(st + c * (kABytes / 4), &mA, raw_full + r, kb * kBK,
                          (int)(c * g.R + mt * 64 + rank * 32));
          } else {
            tma_load_2d(st, &mA, raw_full + r, kb * kBK, (int)(mt * 256 + rank * 128));
          }
        }
      }
    }
  } else if (warp == 13) {  // ---- MMA issuer (leader CTA only)
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = idesc_tf32(256, BN);
      const uint32_t b_hi0 = smem_u32(bres), b_lo0 = b_hi0 + nk * Cfg::kSlab;
      int64_t j = 0, grp = 0;
      for (int64_t mt = mt0; mt < n_mt; mt += mstep) {
        for (int kb = 0; kb < nk; ++kb, ++j) {
          const int o = (int)(j % OS), b = (int)(grp % NB);
          const bool first = kb % kPromote == 0;
          const bool last = kb % kPromote == kPromote - 1 || kb == nk - 1;
          if (first && grp >= NB) mbar_wait(tempty + b, (uint32_t)(((grp / NB) - 1) & 1));
          mbar_wait(conv + o, (uint32_t)((j / OS) & 1));
          tc_fence_after();
          const uint32_t b_hi = b_hi0 + kb * Cfg::kSlab, b_lo = b_lo0 + kb * Cfg::kSlab;
          const uint32_t d = tmem + b * BN;
          const uint32_t a_hi = tmem + Cfg::kACol + o * 2 * kBK, a_lo = a_hi + kBK;
#pragma unroll
          for (int k = 0; k < kBK / 8; ++k) {
            const uint32_t off = k * 32;
            mma2_tf32_ts(d, a_lo + k * 8, desc_k_sw128(b_hi + off), idesc, !(first && k == 0));
            mma2_tf32_ts(d, a_hi + k * 8, desc_k_sw128(b_lo + off), idesc, 1);
            mma2_tf32_ts(d, a_hi + k * 8, desc_k_sw128(b_hi + off), idesc, 1);
          }
          if (last) {
            mma_commit2(gdone + b);
            ++grp;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < 4) {  // ---- split A into this CTA's TMEM, signal the leader
    const int row = warp * 32 + lane;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    int64_t j = 0, grp = 0;
    int64_t grp_of[OS];  // promotion group of the k-block last written to each A stage
    for (int i = 0; i < OS; ++i) grp_of[i] = -1;
    for (int64_t mt = mt0; mt < n_mt; mt += mstep) {
      for (int kb = 0; kb < nk; ++kb, ++j) {
        const int r = (int)(j % RS), o = (int)(j % OS);
        int64_t gprev = -1;
#pragma unroll
        for (int i = 0; i < OS; ++i)
          if (i == o) gprev = grp_of[i];
        if (gprev >= 0) {  // that group's MMAs must have completed
          mbar_wait(gdone + (int)(gprev % NB), (uint32_t)((gprev / NB) & 1));
          tc_fence_after();
        }
#pragma unroll
        for (int i = 0; i < OS; ++i)
          if (i == o) grp_of[i] = grp;
        if (kb % kPromote == kPromote - 1 || kb == nk - 1) ++grp;
        mbar_wait(raw_full + r, (uint32_t)((j / RS) & 1));
        const uint32_t src = smem_u32(raw + r * kABytes) + row * 128;
        float4 v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = lds128(src + ((c ^ (row & 7)) << 4));
        float hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          split_tf32(v[c].x, hi[4 * c], lo[4 * c]);
          split_tf32(v[c].y, hi[4 * c + 1], lo[4 * c + 1]);
          split_tf32(v[c].z, hi[4 * c + 2], lo[4 * c + 2]);
          split_tf32(v[c].w, hi[4 * c + 3], lo[4 * c + 3]);
        }
        fence_proxy_async_smem();  // generic reads of the raw stage before its TMA refill
        __syncwarp();
        if (lane == 0) mbar_arrive(raw_empty + r);
        const uint32_t a = tmem + lane_base + Cfg::kACol + o * 2 * kBK;
        tmem_st32(a, hi);
        tmem_st32(a + kBK, lo);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(conv + o, 0);
      }
    }
  } else {  // ---- warps 4-11: promote partials, epilogue (this CTA's rows)
    const int q = warp & 3, h = (warp - 4) >> 2;
    constexpr int CW = BN / 2;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    unsigned char* my_stg = stg + (warp - 4) * 2 * 2048;
    uint32_t sidx = 0;
    int64_t j = 0;
    const int n0 = nt * BN, c_off = h * CW;
    for (int64_t mt = mt0; mt < n_mt; mt += mstep) {
      float acc[CW];
#pragma unroll
      for (int c = 0; c < CW; ++c) acc[c] = 0.f;
      const int ngrp = (nk + kPromote - 1) / kPromote;
      for (int gi = 0; gi < ngrp; ++gi, ++j) {
        const int b = (int)(j % NB);
        mbar_wait(gdone + b, (uint32_t)((j / NB) & 1));
        tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < CW; c0 += 32) {
          float v[32];
          tmem_ld32(tmem + lane_base + b * BN + c_off + c0, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[c0 + i] += v[i];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty + b, 0);
      }
      if constexpr (EPI == EPI_STORE || EPI == EPI_TANH1) {
        if constexpr (EPI == EPI_TANH1) {
#pragma unroll
          for (int c = 0; c < CW; ++c) {
            const int col = n0 + c_off + c;
            acc[c] = tanhf(acc[c] + (col < g.N ? __ldg(g.bias + col) : 0.f));
          }
        }
        const int64_t row0 = mt * 256 + rank * 128 + q * 32;
        if (g.tma_store) {
          store_rows_tma<CW>(acc, my_stg, &mC, n0 + c_off, (int)row0, 0, lane, sidx);
        } else if (row0 + lane < g.M) {
          float* dst = g.C + (row0 + lane) * g.ldc + n0 + c_off;
#pragma unroll
          for (int c = 0; c < CW; ++c)
            if (n0 + c_off + c < g.N) dst[c] = acc[c];
        }
      } else {  // EPI_TANH: q = channel, lane = point
        const int64_t p0 = mt * 64 + rank * 32;
        if (q == 0) {
#pragma unroll
          for (int c = 0; c < CW; ++c) sbuf[(c_off + c) * 32 + lane] = acc[c];
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        const int e = warp - 4;
#pragma unroll 4
        for (int c = e * (BN / 8); c < (e + 1) * (BN / 8); ++c) {
          const float bv = n0 + c < g.N ? __ldg(g.bias + n0 + c) : 0.f;
          sbuf[c * 32 + lane] = tanhf(sbuf[c * 32 + lane] + bv);
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          const float y = sbuf[(c_off + c) * 32 + lane];
          acc[c] = q == 0 ? y : (1.f - y * y) * acc[c];
        }
        if (g.tma_store) {
          store_rows_tma<CW>(acc, my_stg, &mC, n0 + c_off, (int)p0, q, lane, sidx);
        } else if (p0 + lane < g.R) {
          float* dst = g.C + ((int64_t)q * g.R + p0 + lane) * g.ldc + n0 + c_off;
#pragma unroll
          for (int c = 0; c < CW; ++c)
            if (n0 + c_off + c < g.N) dst[c] = acc[c];
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
      }
    }
  }
  if (warp >= 4 && warp < 12 && lane == 0) bulk_wait_all();
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while its pair may still signal it
  if (warp == 13) tmem_dealloc2(tmem, 512);
}

// ---- weight gradient: dW[Kin, Nout] = X[rows, Kin]^T G[rows, Nout] ----------------------
// Both operands are activations stored row-major, i.e. MN-major for the MMA
// (the reduction runs over rows).  Work items are (128-row block of dW,
// 128-column block, chunk of rows); each writes an fp32 partial tile and a
// second kernel sums the chunks in a fixed order (deterministic split-K).
// Both operands are split into tf32 hi/lo in shared memory.
constexpr int kWRaw = 3, kWOps = 2, kWNB = 4;
constexpr int kWRawBytes = 2 * kABytes;  // A (16 KB) | B (16 KB)
constexpr int kWOpBytes = 4 * kABytes;   // A_hi | A_lo | B_hi | B_lo
constexpr int kWSmem = kWRaw * kWRawBytes + kWOps * kWOpBytes + 1024 + 512;
#ifndef QPINN_WGRAD_PROMOTE
#define QPINN_WGRAD_PROMOTE 2
#endif
constexpr int kWPromote = QPINN_WGRAD_PROMOTE;  // k-blocks per TMEM partial (64-deep chains)

struct WgradArgs {
  int64_t rows, chunk;  // rows per chunk (multiple of 32)
  int Kin, Nout, n_mt, n_nt, n_kc;
  float* partial;       // [n_kc][Kin][Nout]
};

__global__ void __launch_bounds__(kThreadsW, 1)
wgrad_kernel(const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mG,
             const WgradArgs g) {
  constexpr int RS = kWRaw, OS = kWOps, NB = kWNB, P = kWPromote;
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte aligned by offsetting the shared array itself, so pointers derived
  // from it keep the shared address space (LDS/STS rather than generic LD/ST)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* raw = smem;
  unsigned char* ops = smem + RS * kWRawBytes;
  uint64_t* raw_full = (uint64_t*)(ops + OS * kWOpBytes);
  uint64_t* raw_empty = raw_full + RS;
  uint64_t* conv = raw_empty + RS;
  uint64_t* op_empty = conv + OS;
  uint64_t* tfull = op_empty + OS;
  uint64_t* tempty = tfull + NB;
  uint32_t* tmem_slot = (uint32_t*)(tempty + NB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_items = (int64_t)g.n_mt * g.n_nt * g.n_kc;
  auto item = [&](int64_t it, int& mt, int& nt, int& kc, int64_t& row0, int& nkb) {
    kc = (int)(it % g.n_kc);
    const int64_t r = it / g.n_kc;
    nt = (int)(r % g.n_nt);
    mt = (int)(r / g.n_nt);
    row0 = (int64_t)kc * g.chunk;
    int64_t len = g.rows - row0;
    if (len > g.chunk) len = g.chunk;
    nkb = len > 0 ? (int)((len + kBK - 1) / kBK) : 0;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < RS; ++s) {
      mbar_init(raw_full + s, 1);
      mbar_init(raw_empty + s, 4);
    }
    for (int s = 0; s < OS; ++s) {
      mbar_init(conv + s, 4);
      mbar_init(op_empty + s, 1);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(tfull + b, 1);
      mbar_init(tempty + b, 4);
    }
    mbar_init_fence();
  }
  if (warp == 8 && lane == 0) {
    tma_prefetch(&mX);
    tma_prefetch(&mG);
  }
  if (warp == 9) tmem_alloc(tmem_slot, NB * 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {  // ---- TMA producer: 4 x 4 boxes of 32 x 32 per k-block
    if (lane == 0) {
      int64_t j = 0;
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        int mt, nt, kc, nkb;
        int64_t row0;
        item(it, mt, nt, kc, row0, nkb);
        for (int kb = 0; kb < nkb; ++kb, ++j) {
          const int r = (int)(j % RS);
          if (j >= RS) mbar_wait(raw_empty + r, (uint32_t)(((j / RS) - 1) & 1));
          unsigned char* st = raw + r * kWRawBytes;
          mbar_expect_tx(raw_full + r, kWRawBytes);
          const int rr = (int)(row0 + kb * kBK);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            tma_load_2d(st + c * 4096, &mX, raw_full + r, mt * 128 + c * 32, rr);
            tma_load_2d(st + kABytes + c * 4096, &mG, raw_full + r, nt * 128 + c * 32, rr);
          }
        }
      }
    }
  } else if (warp == 9) {  // ---- MMA issuer (MN-major A and B)
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(kBM, 128) | (1u << 15) | (1u << 16);
      int64_t j = 0, grp = 0;
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        int mt, nt, kc, nkb;
        int64_t row0;
        item(it, mt, nt, kc, row0, nkb);
        for (int kb = 0; kb < nkb; ++kb, ++j) {
          const int o = (int)(j % OS), b = (int)(grp % NB);
          const bool first = kb % P == 0, last = kb % P == P - 1 || kb == nkb - 1;
          if (first && grp >= NB) mbar_wait(tempty + b, (uint32_t)(((grp / NB) - 1) & 1));
          mbar_wait(conv + o, (uint32_t)((j / OS) & 1));
          tc_fence_after();
          const uint32_t base = smem_u32(ops + o * kWOpBytes);
          const uint32_t d = tmem + b * 128;
#pragma unroll
          for (int k = 0; k < kBK / 8; ++k) {
            const uint32_t off = k * 1024;  // 8 K-rows = one 1024-byte swizzle atom
            const uint32_t a_hi = base + off, a_lo = base + kABytes + off;
            const uint32_t b_hi = base + 2 * kABytes + off, b_lo = base + 3 * kABytes + off;
            mma_tf32(d, desc_mn_sw128_32b(a_lo), desc_mn_sw128_32b(b_hi), idesc, !(first && k == 0));
            mma_tf32(d, desc_mn_sw128_32b(a_hi), desc_mn_sw128_32b(b_lo), idesc, 1);
            mma_tf32(d, desc_mn_sw128_32b(a_hi), desc_mn_sw128_32b(b_hi), idesc, 1);
          }
          mma_commit(op_empty + o);
          if (last) {
            mma_commit(tfull + b);
            ++grp;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < 4) {  // ---- split A and B (flat 16-byte chunks)
    int64_t j = 0;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      int mt, nt, kc, nkb;
      int64_t row0;
      item(it, mt, nt, kc, row0, nkb);
      for (int kb = 0; kb < nkb; ++kb, ++j) {
        const int r = (int)(j % RS), o = (int)(j % OS);
        if (j >= OS) mbar_wait(op_empty + o, (uint32_t)(((j / OS) - 1) & 1));
        mbar_wait(raw_full + r, (uint32_t)((j / RS) & 1));
        const uint32_t src = smem_u32(raw + r * kWRawBytes) + threadIdx.x * 16;
        const uint32_t dst = smem_u32(ops + o * kWOpBytes) + threadIdx.x * 16;
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // A, then B
          float4 v[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) v[i] = lds128(src + h * kABytes + i * 2048);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float4 hi, lo;
            split_tf32(v[i].x, hi.x, lo.x);
            split_tf32(v[i].y, hi.y, lo.y);
            split_tf32(v[i].z, hi.z, lo.z);
            split_tf32(v[i].w, hi.w, lo.w);
            sts128(dst + h * 2 * kABytes + i * 2048, hi);
            sts128(dst + h * 2 * kABytes + kABytes + i * 2048, lo);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(raw_empty + r);
          mbar_arrive(conv + o);
        }
      }
    }
  } else {  // ---- warps 4-7: promote, store the partial tile
    const int q = warp - 4;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    int64_t grp = 0;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      int mt, nt, kc, nkb;
      int64_t row0;
      item(it, mt, nt, kc, row0, nkb);
      float acc[128];
#pragma unroll
      for (int c = 0; c < 128; ++c) acc[c] = 0.f;
      const int ngrp = (nkb + P - 1) / P;
      for (int gi = 0; gi < ngrp; ++gi, ++grp) {
        const int b = (int)(grp % NB);
        mbar_wait(tfull + b, (uint32_t)((grp / NB) & 1));
        tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < 128; c0 += 32) {
          float v[32];
          tmem_ld32(tmem + lane_base + b * 128 + c0, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[c0 + i] += v[i];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty + b);
      }
      const int m = mt * 128 + q * 32 + lane, n0 = nt * 128;
      if (m < g.Kin) {
        float* dst = g.partial + ((int64_t)kc * g.Kin + m) * g.Nout + n0;
        if (n0 + 128 <= g.Nout && (g.Nout & 3) == 0) {
#pragma unroll
          for (int c = 0; c < 128; c += 4)
            *reinterpret_cast<float4*>(dst + c) =
                make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
        } else {
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (n0 + c < g.Nout) dst[c] = acc[c];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc(tmem, NB * 128);
}

// dW = sum over chunks of the partial tiles, in chunk order (float64 sum)
// dW = sum over the chunks of the partial tiles, in a fixed order: block = 32
// entries x 8 chunk groups (group g sums chunks g, g + 8, ...), then the groups in order
// 32 chunk groups per 32 entries (1024 threads): every thread has at most a few
// partials to load, so the launch is not latency-bound on a serial load chain
__global__ void __launch_bounds__(1024) wgrad_reduce(int n_kc, int64_t n,
                                                    const float* __restrict__ partial,
                                                    float* __restrict__ dW) {
  // block = 128 columns (a float4 per lane), warp w sums chunks k = w, w + 32, ... in
  // float64, then the 32 warps are added in order (deterministic)
  __shared__ double red[32][128];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * 128 + 4 * lane;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if ((n & 3) == 0 && i < n) {  // 16-byte rows
#pragma unroll 2
    for (int k = w; k < n_kc; k += 32) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(partial + (int64_t)k * n + i));
      s0 += (double)v.x;
      s1 += (double)v.y;
      s2 += (double)v.z;
      s3 += (double)v.w;
    }
  } else if (i < n) {
    for (int k = w; k < n_kc; k += 32) {
      const float* r = partial + (int64_t)k * n + i;
      s0 += (double)r[0];
      if (i + 1 < n) s1 += (double)r[1];
      if (i + 2 < n) s2 += (double)r[2];
      if (i + 3 < n) s3 += (double)r[3];
    }
  }
  red[w][4 * lane] = s0;
  red[w][4 * lane + 1] = s1;
  red[w][4 * lane + 2] = s2;
  red[w][4 * lane + 3] = s3;
  __syncthreads();
  if (threadIdx.x < 128 && (int64_t)blockIdx.x * 128 + threadIdx.x < n) {
    double v = 0.0;
#pragma unroll
    for (int g = 0; g < 32; ++g) v += red[g][threadIdx.x];
    dW[(int64_t)blockIdx.x * 128 + threadIdx.x] = (float)v;
  }
}

// B [N,K] (ld ldb) -> B_hi, B_lo [N, ldk] (zero padded to ldk)
__global__ void split_rows(const float* __restrict__ B, int N, int K, int64_t ldb, int ldk,
                           float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t n = (int64_t)N * ldk;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / ldk), c = (int)(i % ldk);
    const float v = c < K ? B[r * ldb + c] : 0.f;
    const float h = rna_tf32(v);
    hi[i] = h;
    lo[i] = rna_tf32(v - h);
  }
}

struct SplitJobs {
  SplitJob j[kMaxSplitJobs];
};

// every weight split of a step in one launch (blockIdx.y = job)
__global__ void split_batch(SplitJobs jobs) {
  const SplitJob& b = jobs.j[blockIdx.y];
  const int64_t n = (int64_t)b.N * b.ldk;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / b.ldk), c = (int)(i % b.ldk);
    const float v = c < b.K ? (b.transpose ? b.src[(int64_t)c * b.ld + r] : b.src[r * b.ld + c]) : 0.f;
    const float h = rna_tf32(v);
    b.hi[i] = h;
    b.lo[i] = rna_tf32(v - h);
  }
}

// W [K,N] row-major (a layer's weights) -> (W^T)_hi, (W^T)_lo [N, ldk]
__global__ void split_transpose(const float* __restrict__ W, int K, int N, int ldk,
                                float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t n = (int64_t)N * ldk;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / ldk), c = (int)(i % ldk);
    const float v = c < K ? W[(int64_t)c * N + r] : 0.f;
    const float h = rna_tf32(v);
    hi[i] = h;
    lo[i] = rna_tf32(v - h);
  }
}

// ---- host --------------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  });
  return fn;
}

// 2-D fp32 map over rows x cols (ld elements), box = 32 columns x box_rows, 128-byte swizzle
static int make_map(CUtensorMap* m, const float* base, uint64_t rows, uint64_t cols, uint64_t ld,
                    uint32_t box_rows,
                    CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto fn = encode_fn();
  if (!fn) return fail(QPINN_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable");
  if (((uintptr_t)base & 15) || (ld & 3))
    return fail(QPINN_ERR_CONFIG, "tensor-core GEMM operands need 16-byte aligned rows");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)kBK, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(QPINN_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return QPINN_OK;
}

static inline int ldk_of(int K) { return (K + 3) & ~3; }

int split_weights(const SplitJob* jobs, int njobs, cudaStream_t st) {
  if (njobs < 0 || njobs > kMaxSplitJobs) return fail(QPINN_ERR_CONFIG, "split_weights: jobs");
  if (njobs == 0) return QPINN_OK;
  SplitJobs jj{};
  for (int i = 0; i < njobs; ++i) jj.j[i] = jobs[i];
  split_batch<<<dim3(16, (unsigned)njobs), 256, 0, st>>>(jj);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

size_t gemm3_workspace_bytes(int N, int K) { return 2 * (size_t)N * ldk_of(K) * 4 + 256; }

// 3-D fp32 output map (cols, rows per block, blocks), 32 x 32 boxes, 128-byte swizzle
static int make_out_map(CUtensorMap* m, const float* base, uint64_t cols, uint64_t rows,
                        uint64_t blocks, uint64_t ld) {
  auto fn = encode_fn();
  if (!fn) return fail(QPINN_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable");
  cuuint64_t dims[3] = {cols, rows, blocks};
  cuuint64_t strides[2] = {ld * 4, ld * 4 * rows};
  cuuint32_t box[3] = {32, 16, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(QPINN_ERR_CUDA, "cuTensorMapEncodeTiled (output) failed");
  return QPINN_OK;
}

template <int BN, int EPI>
static int launch_gemm3(const GemmArgs& g0, const float* A, int64_t lda, const float* Bhi,
                        const float* Blo, int ldk, cudaStream_t st) {
  GemmArgs g = g0;
  CUtensorMap mA, mBh, mBl, mC;
  g.tma_store = ((uintptr_t)g.C & 15) == 0 && (g.ldc & 3) == 0;
  if (EPI == EPI_READOUT && !g.tma_store)
    return fail(QPINN_ERR_CONFIG, "gemm3 readout: Psi needs 16-byte aligned rows");
  if (g.tma_store) {
    const uint64_t rows = kRowsByPoint<EPI> ? (uint64_t)g.R : (uint64_t)g.M;
    if (int rc = make_out_map(&mC, g.C, (uint64_t)g.N, rows, kRowsByPoint<EPI> ? 4 : 1,
                              (uint64_t)g.ldc))
      return rc;
  } else {
    memset(&mC, 0, sizeof(mC));
  }
  const uint32_t a_box = kRowsByPoint<EPI> ? 32 : kBM;
  if (int rc = make_map(&mA, A, (uint64_t)g.M, (uint64_t)g.K, (uint64_t)lda, a_box)) return rc;
  if (int rc = make_map(&mBh, Bhi, (uint64_t)g.N, (uint64_t)ldk, (uint64_t)ldk, BN)) return rc;
  if (int rc = make_map(&mBl, Blo, (uint64_t)g.N, (uint64_t)ldk, (uint64_t)ldk, BN)) return rc;
  auto kern = gemm3_kernel<BN, EPI>;
  QPINN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        GemmCfg<BN>::kSmem));
  const int64_t n_mt = kRowsByPoint<EPI> ? (g.R + 31) / 32 : (g.M + kBM - 1) / kBM;
  const int grid = (int)(n_mt < num_sms() ? n_mt : num_sms());
  kern<<<grid, kThreadsGemm, GemmCfg<BN>::kSmem, st>>>(mA, mBh, mBl, mC, g);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

template <int BN, int EPI>
static int launch_gemm3_pair(const GemmArgs& g0, const float* A, int64_t lda, const float* Bhi,
                             const float* Blo, int ldk, cudaStream_t st) {
  using Cfg = PairCfg<BN>;
  GemmArgs g = g0;
  CUtensorMap mA, mBh, mBl, mC;
  g.tma_store = ((uintptr_t)g.C & 15) == 0 && (g.ldc & 3) == 0;
  if (g.tma_store) {
    const uint64_t rows = EPI == EPI_TANH ? (uint64_t)g.R : (uint64_t)g.M;
    if (int rc = make_out_map(&mC, g.C, (uint64_t)g.N, rows, EPI == EPI_TANH ? 4 : 1,
                              (uint64_t)g.ldc))
      return rc;
  } else {
    memset(&mC, 0, sizeof(mC));
  }
  const uint32_t a_box = EPI == EPI_TANH ? 32 : kBM;
  if (int rc = make_map(&mA, A, (uint64_t)g.M, (uint64_t)g.K, (uint64_t)lda, a_box)) return rc;
  if (int rc = make_map(&mBh, Bhi, (uint64_t)g.N, (uint64_t)ldk, (uint64_t)ldk, Cfg::HB)) return rc;
  if (int rc = make_map(&mBl, Blo, (uint64_t)g.N, (uint64_t)ldk, (uint64_t)ldk, Cfg::HB)) return rc;
  const int nk = (g.K + kBK - 1) / kBK;
  const size_t smem = Cfg::smem(nk);
  auto kern = gemm3_pair_kernel<BN, EPI>;
  QPINN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t n_mt = EPI == EPI_TANH ? (g.R + 63) / 64 : (g.M + 255) / 256;
  const int n_nt = (g.N + BN - 1) / BN;
  int64_t pairs = num_sms() / 2;
  if (pairs > n_mt * n_nt) pairs = n_mt * n_nt;
  pairs = pairs / n_nt * n_nt;  // every pair serves one N-tile (B resident)
  if (pairs < n_nt) pairs = n_nt;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * pairs));
  cfg.blockDim = dim3(kThreadsGemm);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  QPINN_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, mA, mBh, mBl, mC, g));
  return QPINN_OK;
}

// CTA-pair kernel (QPINN_GEMM_PAIR=1) when this CTA's half of the split B fits in
// shared memory next to the A pipeline (K <= 256 at BN = 128).  Correct (same
// errors as the single-CTA kernel, scripts/gemm_check.py) but measured SLOWER:
// 150 vs 105 us at 262144 x 128 x 256 -- the kernel is bound by the per-k-block
// handshake chain (TMA -> split -> MMA commit -> op_empty with 2 TMEM A stages),
// not by shared-memory bandwidth or the MMA rate, and the pair adds cross-SM
// signalling latency to that chain.  Off by default.
static bool use_pair(int BN, int K) {
  static const int env = [] {
    const char* e = getenv("QPINN_GEMM_PAIR");
    return e ? atoi(e) : 0;
  }();
  if (!env) return false;
  const int nk = (K + kBK - 1) / kBK;
  if (nk % kPromote) return false;  // whole promotion groups (the A-stage reuse rule)
  const size_t need = BN == 64 ? PairCfg<64>::smem(nk) : PairCfg<128>::smem(nk);
  return need <= 232448;
}

template <int EPI>
static int dispatch(const GemmArgs& g, const float* A, int64_t lda, const float* hi,
                    const float* lo, int ldk, cudaStream_t st) {
  if (g.N <= 64) {
    if (use_pair(64, g.K)) return launch_gemm3_pair<64, EPI>(g, A, lda, hi, lo, ldk, st);
    return launch_gemm3<64, EPI>(g, A, lda, hi, lo, ldk, st);
  }
  if (use_pair(128, g.K)) return launch_gemm3_pair<128, EPI>(g, A, lda, hi, lo, ldk, st);
  return launch_gemm3<128, EPI>(g, A, lda, hi, lo, ldk, st);
}

int gemm3(int64_t M, int N, int K, const float* A, int64_t lda, const float* B, int64_t ldb,
          float* C, int64_t ldc, void* ws, size_t ws_bytes, cudaStream_t st, const Wsplit* pre) {
  if (M < 0 || N < 1 || K < 1) return fail(QPINN_ERR_CONFIG, "gemm3: bad shape");
  if (ws_bytes < gemm3_workspace_bytes(N, K)) return fail(QPINN_ERR_CONFIG, "gemm3: workspace");
  if (M == 0) return QPINN_OK;
  int ldk = ldk_of(K);
  const float* hi;
  const float* lo;
  if (pre) {  // split once per step by the caller (split_weights)
    hi = pre->hi;
    lo = pre->lo;
    ldk = pre->ldk;
  } else {
    float* h = (float*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    float* l = h + (size_t)N * ldk;
    split_rows<<<64, 256, 0, st>>>(B, N, K, ldb, ldk, h, l);
    QPINN_CUDA_CHECK(cudaGetLastError());
    hi = h;
    lo = l;
  }
  GemmArgs g{M, 0, N, K, C, ldc, nullptr, 0, nullptr, nullptr, nullptr, nullptr, nullptr, 0};
  return dispatch<EPI_STORE>(g, A, lda, hi, lo, ldk, st);
}

// Psi [4R, 256] = Phi [4R, 128] Wt^T (Wt [256, 128]) with the fused Pauli-Z readout:
// z [R, 7], dz [3, R, 7] (the n = 7 transfer-matrix forward with tangents)
int gemm3_readout(int64_t R, const float* Phi, const float* Wt, float* Psi, float* z, float* dz,
                  void* ws, size_t ws_bytes, cudaStream_t st, const Wsplit* pre) {
  constexpr int N = 256, K = 128;
  if (ws_bytes < gemm3_workspace_bytes(N, K)) return fail(QPINN_ERR_CONFIG, "gemm3: workspace");
  if (R == 0) return QPINN_OK;
  int ldk = ldk_of(K);
  const float* hi;
  const float* lo;
  if (pre) {  // split once per step by the caller (split_weights)
    hi = pre->hi;
    lo = pre->lo;
    ldk = pre->ldk;
  } else {
    float* h = (float*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    float* l = h + (size_t)N * ldk;
    split_rows<<<64, 256, 0, st>>>(Wt, N, K, K, ldk, h, l);
    QPINN_CUDA_CHECK(cudaGetLastError());
    hi = h;
    lo = l;
  }
  GemmArgs g{4 * R, R, N, K, Psi, N, nullptr, 0, z, dz, nullptr, nullptr, nullptr, 0};
  return launch_gemm3<128, EPI_READOUT>(g, Phi, K, hi, lo, ldk, st);
}

static void wgrad_plan(int64_t rows, int Kin, int Nout, WgradArgs* a) {
  a->rows = rows;
  a->Kin = Kin;
  a->Nout = Nout;
  a->n_mt = (Kin + 127) / 128;
  a->n_nt = (Nout + 127) / 128;
  const int64_t kblocks = (rows + kBK - 1) / kBK;
  int64_t kc = (num_sms() + a->n_mt * a->n_nt - 1) / (a->n_mt * a->n_nt);
  if (kc > kblocks) kc = kblocks > 0 ? kblocks : 1;
  const int64_t per = (kblocks + kc - 1) / kc;  // k-blocks per chunk
  a->chunk = per * kBK;
  a->n_kc = (int)((rows + a->chunk - 1) / a->chunk);
  if (a->n_kc < 1) a->n_kc = 1;
}

size_t wgrad_workspace_bytes(int64_t rows, int Kin, int Nout) {
  WgradArgs a{};
  wgrad_plan(rows, Kin, Nout, &a);
  return (size_t)a.n_kc * Kin * Nout * 4 + 256;
}

// dW [Kin, Nout] = X [rows, Kin]^T G [rows, Nout]
int wgrad(int64_t rows, int Kin, int Nout, const float* X, int64_t ldx, const float* G,
          int64_t ldg, float* dW, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (rows < 0 || Kin < 1 || Nout < 1) return fail(QPINN_ERR_CONFIG, "wgrad: bad shape");
  if (ws_bytes < wgrad_workspace_bytes(rows, Kin, Nout))
    return fail(QPINN_ERR_CONFIG, "wgrad: workspace");
  if (rows == 0) {
    QPINN_CUDA_CHECK(cudaMemsetAsync(dW, 0, (size_t)Kin * Nout * 4, st));
    return QPINN_OK;
  }
  WgradArgs a{};
  wgrad_plan(rows, Kin, Nout, &a);
  a.partial = (float*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  CUtensorMap mX, mG;
  constexpr CUtensorMapSwizzle kSw = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
  if (int rc = make_map(&mX, X, (uint64_t)rows, (uint64_t)Kin, (uint64_t)ldx, 32, kSw)) return rc;
  if (int rc = make_map(&mG, G, (uint64_t)rows, (uint64_t)Nout, (uint64_t)ldg, 32, kSw)) return rc;
  QPINN_CUDA_CHECK(
      cudaFuncSetAttribute(wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kWSmem));
  const int64_t items = (int64_t)a.n_mt * a.n_nt * a.n_kc;
  const int grid = (int)(items < num_sms() ? items : num_sms());
  wgrad_kernel<<<grid, kThreadsW, kWSmem, st>>>(mX, mG, a);
  QPINN_CUDA_CHECK(cudaGetLastError());
  const int64_t n = (int64_t)Kin * Nout;
  wgrad_reduce<<<(int)((n + 127) / 128), 1024, 0, st>>>(a.n_kc, n, a.partial, dW);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

// H [R, N] = tanh(X [R, K] W [K, N] + b): the value-only dense layer (inference)
int dense_tanh1(int64_t R, int N, int K, const float* X, const float* W, const float* bias,
                float* H, void* ws, size_t ws_bytes, cudaStream_t st, const Wsplit* pre) {
  if (ws_bytes < gemm3_workspace_bytes(N, K)) return fail(QPINN_ERR_CONFIG, "dense: workspace");
  if (R == 0) return QPINN_OK;
  int ldk = ldk_of(K);
  const float* hi;
  const float* lo;
  if (pre) {  // split once per step by the caller (split_weights)
    hi = pre->hi;
    lo = pre->lo;
    ldk = pre->ldk;
  } else {
    float* h = (float*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    float* l = h + (size_t)N * ldk;
    split_transpose<<<64, 256, 0, st>>>(W, K, N, ldk, h, l);
    QPINN_CUDA_CHECK(cudaGetLastError());
    hi = h;
    lo = l;
  }
  GemmArgs g{R, R, N, K, H, N, bias, 0, nullptr, nullptr, nullptr, nullptr, nullptr, 0};
  return dispatch<EPI_TANH1>(g, X, K, hi, lo, ldk, st);
}

// H [4R, N] = dual tanh of X [4R, K] W [K, N] + b (channel blocks of R rows)
int dense_tanh(int64_t R, int N, int K, const float* X, const float* W, const float* bias,
               float* H, void* ws, size_t ws_bytes, cudaStream_t st, const Wsplit* pre) {
  if (ws_bytes < gemm3_workspace_bytes(N, K)) return fail(QPINN_ERR_CONFIG, "dense: workspace");
  if (R == 0) return QPINN_OK;
  int ldk = ldk_of(K);
  const float* hi;
  const float* lo;
  if (pre) {  // split once per step by the caller (split_weights)
    hi = pre->hi;
    lo = pre->lo;
    ldk = pre->ldk;
  } else {
    float* h = (float*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    float* l = h + (size_t)N * ldk;
    split_transpose<<<64, 256, 0, st>>>(W, K, N, ldk, h, l);
    QPINN_CUDA_CHECK(cudaGetLastError());
    hi = h;
    lo = l;
  }
  GemmArgs g{4 * R, R, N, K, H, N, bias, 0, nullptr, nullptr, nullptr, nullptr, nullptr, 0};
  return dispatch<EPI_TANH>(g, X, K, hi, lo, ldk, st);
}

// dense_tanh with the tanh adapter fused into its epilogue: also
// act [4R, n_ad] = dual tanh(H Wa + ba) (N <= 128, n_ad <= 8)
int dense_tanh_adapter(int64_t R, int N, int K, const float* X, const float* W, const float* bias,
                       float* H, const float* Wa, const float* ba, int n_ad, float* act, void* ws,
                       size_t ws_bytes, cudaStream_t st, const Wsplit* pre) {
  if (ws_bytes < gemm3_workspace_bytes(N, K)) return fail(QPINN_ERR_CONFIG, "dense: workspace");
  if (N > 128 || n_ad < 1 || n_ad > 8) return fail(QPINN_ERR_CONFIG, "fused adapter: shape");
  if (R == 0) return QPINN_OK;
  int ldk = ldk_of(K);
  const float* hi;
  const float* lo;
  if (pre) {  // split once per step by the caller (split_weights)
    hi = pre->hi;
    lo = pre->lo;
    ldk = pre->ldk;
  } else {
    float* h = (float*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    float* l = h + (size_t)N * ldk;
    split_transpose<<<64, 256, 0, st>>>(W, K, N, ldk, h, l);
    QPINN_CUDA_CHECK(cudaGetLastError());
    hi = h;
    lo = l;
  }
  GemmArgs g{4 * R, R, N, K, H, N, bias, 0, nullptr, nullptr, Wa, ba, act, n_ad};
  return launch_gemm3<128, EPI_TANH>(g, X, K, hi, lo, ldk, st);
}

}  // namespace tc
}  // namespace qpinn

using namespace qpinn;

extern "C" {

size_t qpinn_gemm_f32_workspace_bytes(int n, int k) {
  return n < 1 || k < 1 ? 0 : tc::gemm3_workspace_bytes(n, k);
}

int qpinn_gemm_f32(int64_t m, int n, int k, const void* a, int64_t lda, const void* b, int64_t ldb,
                   void* c, int64_t ldc, void* workspace, size_t workspace_bytes, void* stream) {
  return tc::gemm3(m, n, k, (const float*)a, lda, (const float*)b, ldb, (float*)c, ldc, workspace,
                   workspace_bytes, (cudaStream_t)stream);
}

#ifdef QPINN_GEMM_PROF
int qpinn_gemm_prof(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, qpinn::tc::g_gemm_prof, sizeof(unsigned long long) * 16);
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(qpinn::tc::g_gemm_prof, z, sizeof(z));
  return 0;
}
#endif

size_t qpinn_gemm_f32_atb_workspace_bytes(int64_t rows, int m, int n) {
  return rows < 0 || m < 1 || n < 1 ? 0 : tc::wgrad_workspace_bytes(rows, m, n);
}

int qpinn_gemm_f32_atb(int64_t rows, int m, int n, const void* x, int64_t ldx, const void* g,
                       int64_t ldg, void* c, void* workspace, size_t workspace_bytes,
                       void* stream) {
  return tc::wgrad(rows, m, n, (const float*)x, ldx, (const float*)g, ldg, (float*)c, workspace,
                   workspace_bytes, (cudaStream_t)stream);
}

}  // extern "C"
