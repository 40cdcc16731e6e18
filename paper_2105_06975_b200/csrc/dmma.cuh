// FP64 tensor-core (DMMA) tile machinery for sm_100a.
//
// tcgen05.mma has no f64 kind, so FP64 contractions on B200 use the warp-level
// DMMA path (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4).  Operands are staged
// global -> shared memory by a multi-stage cp.async ring (LDGSTS, 16-byte
// when aligned, zero-filled at ragged edges); each warp owns a WM x WN
// accumulator block of m8n8 fragments held in registers.
//
// Fragment layout of mma.m8n8k4.f64 (PTX ISA, per lane, g = lane>>2, t = lane&3):
//   A (8x4, row):  a = A[g][t];   B (4x8, col): b = B[t][g];
//   C (8x8):       c0 = C[g][2t], c1 = C[g][2t+1].
// Shared-memory strides are padded by 4 doubles so that both fragment reads
// (A: rows g, cols t;  B: rows t, cols g) are bank-conflict free per half-warp.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace wf {

__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Outputs of a DMMA accumulator pair (columns 2t, 2t + 1 of one row) as ONE 16-byte store
// when the row is 16-byte aligned: the four lanes of a quad then write two whole 32-byte
// sectors per instruction.  Two 8-byte stores per pair leave every sector half written by
// each instruction (round 2, r02at: see DESIGN.md section 10, the TMA-staged coupling GEMMs
// read rows written this way).  `col` is the (even) column of v0, N the column count.
__device__ __forceinline__ bool pair_aligned(const double *base, int64_t ld) {
  return ((reinterpret_cast<uintptr_t>(base) & 15) == 0) && ((ld & 1) == 0);
}
__device__ __forceinline__ void store_pair(double *dst, int col, int N, double v0, double v1,
                                           bool aligned) {
  if (aligned && col + 1 < N) {
    *reinterpret_cast<double2 *>(dst) = make_double2(v0, v1);
  } else {
    if (col < N) dst[0] = v0;
    if (col + 1 < N) dst[1] = v1;
  }
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_>
struct TileCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int NWARP = WARPS_M * WARPS_N;
  static constexpr int NT = NWARP * 32;
  static constexpr int FM = WM / 8, FN = WN / 8;
  static constexpr int LDA = BK + 4;   // padded smem strides (doubles)
  static constexpr int LDB = BN + 4;
  static constexpr int A_STAGE = BM * LDA;
  static constexpr int B_STAGE = BK * LDB;
  static constexpr int STAGE = A_STAGE + B_STAGE;
  static constexpr int SMEM_DOUBLES = STAGE * STAGES;
  static_assert(BK % 4 == 0 && WM % 8 == 0 && WN % 8 == 0, "tile shape");
};

// Issue the cp.async copies of one (BM x BK) A tile and (BK x BN) B tile.
// A: rows [m0, m0+BM) < M, cols [k0, k0+BK) < kend;  B: rows [k0, ..) < kend, cols [n0, ..) < N.
template <class C, bool V16>
__device__ __forceinline__ void load_tiles(double *sA, double *sB, const double *__restrict__ A,
                                           int64_t lda, const double *__restrict__ B, int64_t ldb,
                                           int m0, int n0, int k0, int M, int N, int kend,
                                           int tid) {
  if (V16) {
    // A tile: BM rows x BK/2 pairs
    constexpr int APAIRS = C::BM * C::BK / 2;
#pragma unroll
    for (int e = tid; e < APAIRS; e += C::NT) {
      int r = e / (C::BK / 2), cp = (e % (C::BK / 2)) * 2;
      int gr = m0 + r, gc = k0 + cp;
      int bytes = (gr < M) ? max(0, min(2, kend - gc)) * 8 : 0;
      const double *src = bytes ? A + (int64_t)gr * lda + gc : A;
      cp_async16(sA + r * C::LDA + cp, src, bytes);
    }
    constexpr int BPAIRS = C::BK * C::BN / 2;
#pragma unroll
    for (int e = tid; e < BPAIRS; e += C::NT) {
      int r = e / (C::BN / 2), cp = (e % (C::BN / 2)) * 2;
      int gr = k0 + r, gc = n0 + cp;
      int bytes = (gr < kend) ? max(0, min(2, N - gc)) * 8 : 0;
      const double *src = bytes ? B + (int64_t)gr * ldb + gc : B;
      cp_async16(sB + r * C::LDB + cp, src, bytes);
    }
  } else {
    constexpr int AEL = C::BM * C::BK;
#pragma unroll 4
    for (int e = tid; e < AEL; e += C::NT) {
      int r = e / C::BK, cc = e % C::BK;
      int gr = m0 + r, gc = k0 + cc;
      bool ok = gr < M && gc < kend;
      cp_async8(sA + r * C::LDA + cc, ok ? A + (int64_t)gr * lda + gc : A, ok ? 8 : 0);
    }
    constexpr int BEL = C::BK * C::BN;
#pragma unroll 4
    for (int e = tid; e < BEL; e += C::NT) {
      int r = e / C::BN, cc = e % C::BN;
      int gr = k0 + r, gc = n0 + cc;
      bool ok = gr < kend && gc < N;
      cp_async8(sB + r * C::LDB + cc, ok ? B + (int64_t)gr * ldb + gc : B, ok ? 8 : 0);
    }
  }
}

template <class C>
__device__ __forceinline__ void mma_stage(const double *sA, const double *sB,
                                          double (&acc)[C::FM][C::FN][2], int wm, int wn,
                                          int lane) {
  const int g = lane >> 2, t = lane & 3;
  // fragments are double-buffered in registers: the shared-memory loads of step
  // kk+4 are issued before the DMMAs of step kk, hiding the LDS latency (ncu r01:
  // the tensor pipe idled on LDS->DMMA dependencies with single buffering)
  double a[2][C::FM], b[2][C::FN];
#pragma unroll
  for (int i = 0; i < C::FM; ++i) a[0][i] = sA[(wm * C::WM + i * 8 + g) * C::LDA + t];
#pragma unroll
  for (int j = 0; j < C::FN; ++j) b[0][j] = sB[t * C::LDB + wn * C::WN + j * 8 + g];
#pragma unroll
  for (int kk = 0; kk < C::BK; kk += 4) {
    const int cur = (kk >> 2) & 1;
    if (kk + 4 < C::BK) {
#pragma unroll
      for (int i = 0; i < C::FM; ++i)
        a[cur ^ 1][i] = sA[(wm * C::WM + i * 8 + g) * C::LDA + kk + 4 + t];
#pragma unroll
      for (int j = 0; j < C::FN; ++j)
        b[cur ^ 1][j] = sB[(kk + 4 + t) * C::LDB + wn * C::WN + j * 8 + g];
    }
#pragma unroll
    for (int i = 0; i < C::FM; ++i)
#pragma unroll
      for (int j = 0; j < C::FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[cur][i], b[cur][j]);
  }
}

// acc += A[m0.., kbeg..kend) * B[kbeg..kend, n0..)   (full multi-stage pipeline)
template <class C, bool V16>
__device__ __forceinline__ void tile_mainloop(double *smem, double (&acc)[C::FM][C::FN][2],
                                              const double *__restrict__ A, int64_t lda,
                                              const double *__restrict__ B, int64_t ldb, int m0,
                                              int n0, int kbeg, int kend, int M, int N) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int nk = (kend - kbeg + C::BK - 1) / C::BK;
  if (nk <= 0) return;
#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    if (s < nk) {
      double *st = smem + s * C::STAGE;
      load_tiles<C, V16>(st, st + C::A_STAGE, A, lda, B, ldb, m0, n0, kbeg + s * C::BK, M, N,
                         kend, tid);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    int nx = kt + C::STAGES - 1;
    if (nx < nk) {
      double *st = smem + (nx % C::STAGES) * C::STAGE;
      load_tiles<C, V16>(st, st + C::A_STAGE, A, lda, B, ldb, m0, n0, kbeg + nx * C::BK, M, N,
                         kend, tid);
    }
    cp_async_commit();
    const double *st = smem + (kt % C::STAGES) * C::STAGE;
    mma_stage<C>(st, st + C::A_STAGE, acc, wm, wn, lane);
  }
  cp_async_wait<0>();
  __syncthreads();
}

}  // namespace wf
