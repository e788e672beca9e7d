// Shared device-side definitions: precision modes, operand preparation,
// accumulators and the per-level operator parameter blocks.
//
// Precision semantics restate src/precision.py:206-230 (contract_mode):
//   fp64    : double operands, double accumulation
//   fp32    : float operands, float accumulation
//   fp16    : both operands rounded to binary16 (RNE, subnormals kept),
//             products exact in fp32, fp32 accumulation
//   fp16_ec : main = c(mh, uh); corr = c(dm, uh) + c(mh, du); main + corr/2048
//             with (h, d) = (half(x), half((x - half(x)) * 2048))   (precision.py:168-174)
// Vectors are stored in fp64 (fp64 mode) or fp32 (all other modes), precision.py:36-39.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace sf {

enum Mode : int { MODE_FP64 = 0, MODE_FP32 = 1, MODE_FP16 = 2, MODE_FP16_EC = 3 };

constexpr float kEcScale = 2048.0f;  // precision.py:19

template <int MODE>
struct MT {
  using S = float;  // storage
  using C = float;  // compute / accumulate
  static constexpr bool kHalf = (MODE == MODE_FP16 || MODE == MODE_FP16_EC);
  static constexpr bool kEC = (MODE == MODE_FP16_EC);
};
template <>
struct MT<MODE_FP64> {
  using S = double;
  using C = double;
  static constexpr bool kHalf = false;
  static constexpr bool kEC = false;
};

__device__ __forceinline__ float demote16(float x) {
  // cvt.rn.f16.f32 then back: round-to-nearest-even, subnormals preserved,
  // overflow to +-inf -- numpy's float32->float16 cast (precision.py:130-137).
  return __half2float(__float2half_rn(x));
}

// A contraction operand prepared under a mode: h = main part, d = EC residual part.
template <int MODE>
struct Op {
  typename MT<MODE>::C h;
};
template <>
struct Op<MODE_FP16_EC> {
  float h, d;
};

template <int MODE>
__device__ __forceinline__ Op<MODE> prep(typename MT<MODE>::C x) {
  if constexpr (MODE == MODE_FP16) {
    return Op<MODE>{demote16(x)};
  } else if constexpr (MODE == MODE_FP16_EC) {
    float h = demote16(x);
    float d = demote16((x - h) * kEcScale);
    return Op<MODE>{h, d};
  } else {
    return Op<MODE>{x};
  }
}

// A matrix entry prepared on the host under a mode (fp16: pre-demoted; EC: split).
template <int MODE>
struct ME {
  typename MT<MODE>::C h;
};
template <>
struct ME<MODE_FP16_EC> {
  float h, d;
};

// Accumulator for one output of one contraction.
template <int MODE>
struct Acc {
  using C = typename MT<MODE>::C;
  C m;
  __device__ __forceinline__ Acc() : m(C(0)) {}
  __device__ __forceinline__ void fma(const ME<MODE>& a, const Op<MODE>& x) { m = ::fma(a.h, x.h, m); }
  __device__ __forceinline__ void add(C v) { m += v; }
  __device__ __forceinline__ C result() const { return m; }
};
template <>
struct Acc<MODE_FP16_EC> {
  float m, c1, c2;
  __device__ __forceinline__ Acc() : m(0.f), c1(0.f), c2(0.f) {}
  __device__ __forceinline__ void fma(const ME<MODE_FP16_EC>& a, const Op<MODE_FP16_EC>& x) {
    m = fmaf(a.h, x.h, m);
    c1 = fmaf(a.d, x.h, c1);
    c2 = fmaf(a.h, x.d, c2);
  }
  __device__ __forceinline__ void add(float v) { m += v; }
  __device__ __forceinline__ float result() const { return m + (c1 + c2) / kEcScale; }
};

// ---------------------------------------------------------------------------
// Per-level 1-D operator in cell-wise form.  Along one axis the
// global 1-D SIPG operator is block tridiagonal over cells:
//   diagonal block  : D  = L_smooth[(F,F)][:K,:K]  (cell stiffness + both face self-couplings)
//   upper block     : U  = F_cross[:K, K:]  (nonzeros: column 0 and row K-1 only)
//   lower block     : U^T
//   first/last cell : D + Bl / D + Br with Bl = (B_left - H_left)[:K,:K] (column/row 0),
//                     Br = (B_right - H_right)[K:,K:] (column/row K-1)
// ucol = U[:,0], urow = U[K-1,:], bl = Bl[:,0], br = Br[:,K-1].
// Range management for the binary16 modes.  All factors are
// powers of two, so scaling is exact and the demoted values equal 2^a times the
// unscaled demoted values whenever those are normal binary16 numbers:
//   matrices:  M^ = 2^aM M, L^ = 2^aL L (D, U, Nitsche blocks), V^ = 2^aV V  (static, per level)
//   vectors :  u^ = 2^e u with a per-CTA block exponent e putting max|u^| in [2, 4)
//   operator:  A^ = 2^aA A, aA = aL + 2 aM  ->  A u = 2^-(aA + e) (A^ u^)
//   patch inverse: S^-1 r = 2^-(aD + 6 aV + e_r) V^(x3) (2^aD Lambda^-1) V^T(x3) r^
// fp64/fp32 modes use all-zero exponents.
struct Scales {
  int aA;  // operator exponent
  int aV;  // eigenvector exponent
  int aD;  // division exponent: the kernels divide by (lambda_sum * 2^-aD)
};

template <int K, int MODE>
struct LevelOp {
  ME<MODE> M[K][K];
  ME<MODE> D[K][K];
  ME<MODE> ucol[K];
  ME<MODE> urow[K];
  ME<MODE> bl[K];
  ME<MODE> br[K];
  Scales sc;
};

// 2^e as float / double (normal range only)
__host__ __device__ __forceinline__ float pow2f(int e) {
  union {
    int i;
    float f;
  } u;
  u.i = (e + 127) << 23;
  return u.f;
}
__host__ __device__ __forceinline__ double pow2d(int e) {
  union {
    long long i;
    double f;
  } u;
  u.i = (long long)(e + 1023) << 52;
  return u.f;
}
// CTA-wide max of |x| over non-negative floats via integer atomics on a shared word
__device__ __forceinline__ void smax(int* word, float v) {
  v = fabsf(v);
  if (v > 0.f) atomicMax(word, __float_as_int(v < 3.0e38f ? v : 3.0e38f));
}
// block exponent: e such that max|v| * 2^e lies in [2, 4) (0 for an all-zero or non-finite block)
__device__ __forceinline__ int block_exp(float maxabs) {
  if (!(maxabs > 0.f) || !(maxabs < 3.0e38f)) return 0;
  const int ex = ((__float_as_int(maxabs) >> 23) & 0xff) - 127;  // maxabs in [2^ex, 2^ex+1)
  int e = 1 - ex;
  if (e > 100) e = 100;
  if (e < -100) e = -100;
  return e;
}
__device__ __forceinline__ int block_exp(double maxabs) { return block_exp((float)maxabs); }

// Fast-diagonalisation tables for the vertex-patch smoother (multigrid.py:47-83):
// V[kind] (2K x 2K, M-orthonormal eigenvectors of L_smooth[kind] vs M_patch) and the
// eigenvalues in fp64 (the reference sums them in fp64 and casts, multigrid.py:60-69).
// kind = 2*left_boundary + right_boundary.
template <int K, int MODE>
struct PatchEig {
  ME<MODE> V[4][2 * K][2 * K];
  double lam[4][2 * K];
};

// Prolongation embedding P (2K x K), basis.py:243-252.
template <int K, int MODE>
struct Embed {
  ME<MODE> P[2 * K][K];
};

// Geometry of the local array and of the tile grid.  A tile is a 2x2x2 block
// of cells (one vertex patch).  Tiles start at cell t0 + 2*i along each axis.
struct Geom {
  int nx, ny, nz;          // cells per axis in the local array
  int tx0, ty0, tz0;       // first tile's cell offset (colour shift)
  int ntx, nty, ntz;       // tiles per axis
  int bnd_lo[3], bnd_hi[3];  // 1: the domain boundary is at local cell 0 / n-1 (axis x,y,z)
  const void* ghost_lo;    // z-halo: K dof planes below local z=0 (or null)
  const void* ghost_hi;    // z-halo: K dof planes above local z=nz*K-1 (or null)
  long long batch_stride;  // elements between batched vectors (blockIdx.y)
};

// Tile id -> tile coordinates in an L2-aware order: y is cut into bands of BAND/ntx tile
// rows; inside a band the order is x fastest, then y, then z.  A tile's z neighbours are then
// ~BAND launches away (instead of ntx*nty), so the neighbour cell layers its face traces read
// are still in L2 (profiles/r01_vmult_fp64.md).  BAND = tiles in ~8 MiB of
// fp64 data: 256 for Q7 (32 KiB tiles; 4 tile rows at level 7), 2048 for Q3.  Round 2 A/B
// (profiles/r02_vmult_fp64.md): 16 MiB 118.4, 8 MiB 120.3, 4 MiB 116.9, 32 MiB 112.6 GDoF/s.
template <int K>
constexpr int band_tiles() {
  return (1 << 23) / (8 * K * K * K * 8) > 1 ? (1 << 23) / (8 * K * K * K * 8) : 1;
}
template <int K>
__device__ __forceinline__ void tile_coords(const Geom& g, int id, int& tx, int& ty, int& tz) {
  int by = band_tiles<K>() / g.ntx;
  by = by < 1 ? 1 : (by > g.nty ? g.nty : by);
  const int per_band = g.ntx * by * g.ntz;
  const int band = id / per_band;
  const int off = id - band * per_band;
  const int rem = g.nty - band * by;
  const int bh = rem < by ? rem : by;
  tx = off % g.ntx;
  const int r = off / g.ntx;
  ty = band * by + r % bh;
  tz = r / bh;
}

}  // namespace sf
