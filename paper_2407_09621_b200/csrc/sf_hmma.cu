// FP16 / FP16-EC tensor-core kernels for Q7 (K = 8): vmult and smoother colour
// pass with mma.sync.m16n8k16 (f16 x f16 -> f32), ldmatrix/stmatrix operand
// staging and the reference's per-contraction demotion semantics
// (precision.py:206-230):
//   fp16    : every contraction's input tensor and matrix are binary16 (RNE,
//             subnormals kept); products are exact in f32; f32 accumulation.
//   fp16_ec : main = A_h B_h, corr = A_d B_h + A_h B_d with the 2^11-scaled
//             residual halves d; result = main + corr / 2048.
// Intermediate tensors therefore live in shared memory as binary16 (plus the
// residual half for EC): demotion happens exactly once, where the reference's
// next contraction would demote them.
//
// Tile = 2x2x2 cells = 16^3 dofs, 4 warps, f32 vectors in HBM (fp32 storage).
// One 16-line group is one m16 MMA tile; a 16 -> 16 line operator is two
// m16n8k16 MMAs.  Same cell-wise schedule as the FP64 path (sf_dmma.cuh):
//   x: a = Mx u, b = Lx u (+halo) | y: c = My a, dd = Ly a (+halo) + My b | z: v = Lz c (+halo) + Mz dd
// The accumulator fragment of m16n8k16 is the A fragment of the next MMA, so
// contractions along the same axis chain in registers (smoother: z fwd, x fwd/bwd).
// Shared layout (halves): z*264 + y*16 + 8*((x>>3) ^ ((y>>2)&1)) + (x&7): every
// ldmatrix/stmatrix 8x8 access (rows along y or z) is bank-conflict free.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "sf_common.cuh"
#include "sf_internal.h"
#include "sf_tile.cuh"

namespace sf {
namespace hm {

constexpr int K = 8, B = 16;
constexpr int PZ = 264;            // halves per z plane (256 + 8 pad)
constexpr int TVOL = 16 * PZ;      // halves per tile tensor
constexpr int kThreads = 128;      // 4 warps
constexpr float kEc = 2048.0f;

__device__ __forceinline__ int hidx(int z, int y, int x) {
  return z * PZ + y * 16 + ((((x >> 3) ^ (y >> 2)) & 1) << 3) + (x & 7);
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

__device__ __forceinline__ void ldsm4(unsigned (&r)[4], const __half* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm4t(unsigned (&r)[4], const __half* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void stsm4(__half* p, const unsigned (&r)[4]) {
  asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1,%2,%3,%4};\n" ::"r"(smem_u32(p)), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3])
               : "memory");
}
__device__ __forceinline__ void stsm4t(__half* p, const unsigned (&r)[4]) {
  asm volatile("stmatrix.sync.aligned.m8n8.x4.trans.shared.b16 [%0], {%1,%2,%3,%4};\n" ::"r"(smem_u32(p)),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3])
               : "memory");
}

// D(16x8,f32) += A(16x16,f16) B(16x8,f16)
__device__ __forceinline__ void hmma(float (&d)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ unsigned pack2(float lo, float hi) {
  __half2 h = __halves2half2(__float2half_rn(lo), __float2half_rn(hi));
  return *reinterpret_cast<unsigned*>(&h);
}
__device__ __forceinline__ float2 unpack2(unsigned u) {
  __half2 h = *reinterpret_cast<__half2*>(&u);
  return __half22float2(h);
}

// A 16-line x 16-output accumulator: two n8 tiles, f32; EC keeps main and corr.
template <int MODE>
struct Acc16 {
  float m[2][4];
  float c[2][4];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) m[nt][i] = c[nt][i] = 0.f;
  }
  // output value (nt, i) after the contraction: main (+ corr/2048 for EC)
  __device__ __forceinline__ float val(int nt, int i) const {
    if constexpr (MODE == MODE_FP16_EC) return m[nt][i] + c[nt][i] / kEc;
    return m[nt][i];
  }
};

// A fragment of one operand tensor: main halves (+ EC residual halves)
template <int MODE>
struct AFrag {
  unsigned h[4];
  unsigned d[4];
};

// B fragments of one 16x16 operator: [nt][reg] (+ EC residual)
template <int MODE>
struct BFrag {
  unsigned h[2][2];
  unsigned d[2][2];
};

template <int MODE>
__device__ __forceinline__ void mma16(Acc16<MODE>& acc, const AFrag<MODE>& a, const BFrag<MODE>& b) {
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    hmma(acc.m[nt], a.h, b.h[nt][0], b.h[nt][1]);
    if constexpr (MODE == MODE_FP16_EC) {
      hmma(acc.c[nt], a.h, b.d[nt][0], b.d[nt][1]);  // c(mh, du) part: A_h B_d ...
      hmma(acc.c[nt], a.d, b.h[nt][0], b.h[nt][1]);  // ... and A_d B_h
    }
  }
}

// split an f32 value into the operand halves of the mode
template <int MODE>
__device__ __forceinline__ void split(float x, float& h, float& d) {
  h = __half2float(__float2half_rn(x));
  d = (MODE == MODE_FP16_EC) ? __half2float(__float2half_rn((x - h) * kEc)) : 0.f;
}

// accumulator fragment -> A fragment of the next MMA (same axis), with demotion.
// Pairs are rounded with one packed cvt (cvt.rn.f16x2.f32) and the EC residual is formed from
// the packed halves directly -- the same values as split() + pack2() with ~40 % fewer
// instructions (the F2FP/HADD2 chain was the largest instruction class, profiles/r01_smoother_fp16.md).
template <int MODE>
__device__ __forceinline__ void demote_pair(float x0, float x1, unsigned& h, unsigned& d) {
  const __half2 hh = __floats2half2_rn(x0, x1);
  h = *reinterpret_cast<const unsigned*>(&hh);
  if constexpr (MODE == MODE_FP16_EC) {
    const float2 hf = __half22float2(hh);
    const __half2 dd = __floats2half2_rn((x0 - hf.x) * kEc, (x1 - hf.y) * kEc);
    d = *reinterpret_cast<const unsigned*>(&dd);
  }
}

template <int MODE>
__device__ __forceinline__ void acc_to_a(const float (&v)[2][4], AFrag<MODE>& a) {
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    demote_pair<MODE>(v[nt][0], v[nt][1], a.h[2 * nt], a.d[2 * nt]);
    demote_pair<MODE>(v[nt][2], v[nt][3], a.h[2 * nt + 1], a.d[2 * nt + 1]);
  }
}

// ---------------------------------------------------------------- tables
// B fragment of Op (16 out x 16 in) for lane ln, n tile nt, register j:
//   (Op[8nt + (ln>>2)][2(ln&3) + 8j], Op[...][... + 1]) as half2 (+ EC residual half2)
struct HTables {
  unsigned M[2][2][2][32];      // [h/d][nt][j][lane]  M_patch
  unsigned L[4][2][2][2][32];   // [kind][h/d][nt][j][lane]  L_smooth[kind]
  unsigned Vf[4][2][2][2][32];  // Op = V^T
  unsigned Vb[4][2][2][2][32];  // Op = V
  double lam[4][16];
  float ucol[2][K], urow[2][K];  // [h/d] demoted halo vectors
};

template <int MODE>
__device__ __forceinline__ void load_b(BFrag<MODE>& b, const unsigned* t /* [2][2][2][32] */, int lane) {
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      b.h[nt][j] = __ldg(t + (0 * 4 + nt * 2 + j) * 32 + lane);
      if constexpr (MODE == MODE_FP16_EC) b.d[nt][j] = __ldg(t + (1 * 4 + nt * 2 + j) * 32 + lane);
    }
}

// ---------------------------------------------------------------- tile
template <int MODE>
struct HTile {
  __half* uh;  // tensor U (h) ; EC residual at uh + 2*TVOL
  __half* bh;  // tensor B (h) ; EC residual at bh + 2*TVOL
  float* tr;   // V1 trace planes (12 x 16 x 17 f32)
  int* s_exp;  // block-exponent words ([0] input, [1] residual)
  int eu;      // input block exponent: u^ = 2^eu u
  int cx, cy, cz;
  long long sy, sz;
  unsigned nbm;
  int kind[3];
  int lane, warp, g, t;
  float hur[2][2], huc[2][2];  // [h/d][i]: urow / ucol at output n = 2t + i of this lane (halo16)
  int skip[3];                 // line tiles: leading points per axis owned by the previous tile
  __device__ __forceinline__ __half* ud() const { return uh + 2 * TVOL; }
  __device__ __forceinline__ __half* bd() const { return bh + 2 * TVOL; }
};

template <int MODE>
constexpr size_t smem_bytes() {
  return sizeof(__half) * (MODE == MODE_FP16_EC ? 4 : 2) * TVOL + sizeof(float) * 12 * 16 * 17 + 16;
}

// store a value into (h, d) tensors at half index i
template <int MODE>
__device__ __forceinline__ void put(__half* h, __half* d, int i, float x) {
  float hh, dd;
  split<MODE>(x, hh, dd);
  h[i] = __float2half_rn(hh);
  if constexpr (MODE == MODE_FP16_EC) d[i] = __float2half_rn(dd);
}

template <int MODE>
__device__ __forceinline__ void ld_a(AFrag<MODE>& a, const __half* h, const __half* d, int off, bool trans) {
  if (trans) {
    ldsm4t(a.h, h + off);
    if constexpr (MODE == MODE_FP16_EC) ldsm4t(a.d, d + off);
  } else {
    ldsm4(a.h, h + off);
    if constexpr (MODE == MODE_FP16_EC) ldsm4(a.d, d + off);
  }
}

// store accumulator values (already final f32) via stmatrix as (h, d)
template <int MODE>
__device__ __forceinline__ void st_acc(__half* h, __half* d, int off, const float (&v)[2][4], bool trans) {
  AFrag<MODE> a;
  acc_to_a<MODE>(v, a);
  // A fragment regs (0: rows 0-7 k 0-7, 1: rows 8-15 k 0-7, 2: rows 0-7 k 8-15, 3: rows 8-15 k 8-15)
  // map onto stmatrix matrices in the same order as the ldmatrix addressing used here.
  if (trans) {
    stsm4t(h + off, a.h);
    if constexpr (MODE == MODE_FP16_EC) stsm4t(d + off, a.d);
  } else {
    stsm4(h + off, a.h);
    if constexpr (MODE == MODE_FP16_EC) stsm4(d + off, a.d);
  }
}

template <int MODE>
__device__ __forceinline__ void finals(const Acc16<MODE>& acc, float (&v)[2][4]) {
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) v[nt][i] = acc.val(nt, i);
}

// ldmatrix / stmatrix lane address for a 16x16 operand:
//   non-trans (rows along the "line" axis a1, k along x):  line = j + 8(q&1), k0 = 8(q>>1)
//   trans     (memory rows along the k axis):                krow = j + 8(q>>1), line0 = 8(q&1)
__device__ __forceinline__ void lane_qj(int lane, int& q, int& j) {
  q = lane >> 3;
  j = lane & 7;
}

// halo update on a stiffness accumulator of 16 lines; alpha/beta per line from the trace plane
template <int MODE>
__device__ __forceinline__ void halo16(const HTile<MODE>& T, Acc16<MODE>& acc, const HTables* tab, int axis,
                                       const float* tr_lo_a, const float* tr_lo_b, const float* tr_hi_a,
                                       const float* tr_hi_b) {
  // lines g and g+8 (rows of the accumulator), outputs n = 8nt + 2t + {0,1}
  const int g = T.g, t2 = 2 * T.t;
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int line = g + 8 * rr;
    if ((T.nbm >> (2 * axis)) & 1) {  // lo neighbour -> cell 0 outputs (nt = 0)
      float ah, ad;
      split<MODE>(tr_lo_a[line], ah, ad);
      const float bet = tr_lo_b[line];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        acc.m[0][2 * rr + i] = fmaf(T.hur[0][i], ah, acc.m[0][2 * rr + i]);
        if constexpr (MODE == MODE_FP16_EC) {
          acc.c[0][2 * rr + i] = fmaf(T.hur[1][i], ah, acc.c[0][2 * rr + i]);
          acc.c[0][2 * rr + i] = fmaf(T.hur[0][i], ad, acc.c[0][2 * rr + i]);
        }
      }
      if (t2 == 0) acc.m[0][2 * rr] += bet;
    }
    if ((T.nbm >> (2 * axis + 1)) & 1) {  // hi neighbour -> cell 1 outputs (nt = 1)
      float ah, ad;
      split<MODE>(tr_hi_a[line], ah, ad);
      const float bet = tr_hi_b[line];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        acc.m[1][2 * rr + i] = fmaf(T.huc[0][i], ah, acc.m[1][2 * rr + i]);
        if constexpr (MODE == MODE_FP16_EC) {
          acc.c[1][2 * rr + i] = fmaf(T.huc[1][i], ah, acc.c[1][2 * rr + i]);
          acc.c[1][2 * rr + i] = fmaf(T.huc[0][i], ad, acc.c[1][2 * rr + i]);
        }
      }
      if (t2 + 1 == K - 1) acc.m[1][2 * rr + 1] += bet;
    }
  }
}

template <int MODE>
__device__ __forceinline__ const float* trp(const HTile<MODE>& T, int face, int plane) {
  return T.tr + (face * 2 + plane) * (16 * 17);
}

// Tangential masses of the y-face (Mx along q) and z-face (Mx along q, then My
// along p) trace planes on the tensor cores: plane = 16 x 16 f32 (pitch 17),
// A fragment gathered from f32 shared memory with demotion, in place.
template <int MODE>
__device__ __forceinline__ void plane_mass(float* P, bool along_p, const BFrag<MODE>& bm, int g, int t) {
  float v[2][4];
  // A[row][k]: along q: row = p, k = q;  along p: row = q, k = p
  auto at = [&](int row, int k) -> float { return along_p ? P[k * 17 + row] : P[row * 17 + k]; };
#pragma unroll
  for (int kb = 0; kb < 2; ++kb) {
    v[kb][0] = at(g, 8 * kb + 2 * t);
    v[kb][1] = at(g, 8 * kb + 2 * t + 1);
    v[kb][2] = at(g + 8, 8 * kb + 2 * t);
    v[kb][3] = at(g + 8, 8 * kb + 2 * t + 1);
  }
  AFrag<MODE> a;
  acc_to_a<MODE>(v, a);  // same register order as an accumulator fragment
  Acc16<MODE> acc;
  acc.zero();
  mma16<MODE>(acc, a, bm);
  __syncwarp();
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = g + 8 * (i >> 1), n = 8 * nt + 2 * t + (i & 1);
      if (along_p) P[n * 17 + row] = acc.val(nt, i); else P[row * 17 + n] = acc.val(nt, i);
    }
}

template <int MODE>
__device__ __forceinline__ void trace_masses_tc(const HTile<MODE>& T, const HTables* tab) {
  BFrag<MODE> bm;
  load_b<MODE>(bm, &tab->M[0][0][0][0], T.lane);
  // 8 planes (faces 2..5, alpha/beta) along q, two per warp
  for (int task = T.warp; task < 8; task += kThreads / 32) {
    const int face = 2 + (task >> 1);
    if (!((T.nbm >> face) & 1)) continue;
    plane_mass<MODE>(T.tr + (face * 2 + (task & 1)) * (16 * 17), false, bm, T.g, T.t);
  }
  __syncthreads();
  for (int task = T.warp; task < 4; task += kThreads / 32) {
    const int face = 4 + (task >> 1);
    if (!((T.nbm >> face) & 1)) continue;
    plane_mass<MODE>(T.tr + (face * 2 + (task & 1)) * (16 * 17), true, bm, T.g, T.t);
  }
}

// L2 prefetch of this tile's rows of b (read in the z stage of the colour / restriction kernels)
template <int KK = K>
__device__ __forceinline__ void prefetch_b_rows(const Geom& g, const float* __restrict__ b) {
  if ((int)blockIdx.x >= g.ntx * g.nty * g.ntz) return;
  constexpr int CPL = 16 / KK;
  int tx, ty, tz;
  tile_coords<8>(g, blockIdx.x, tx, ty, tz);
  const long long sy = (long long)g.nx * KK, sz = sy * (long long)g.ny * KK;
  int cx = g.tx0 + CPL * tx, cy = g.ty0 + CPL * ty, cz = g.tz0 + CPL * tz;
  if (CPL > 2) {
    if (g.tx0 & 1) cx = min(cx, g.nx - CPL - g.tx0);
    if (g.ty0 & 1) cy = min(cy, g.ny - CPL - g.ty0);
    if (g.tz0 & 1) cz = min(cz, g.nz - CPL - g.tz0);
  }
  for (int r = threadIdx.x; r < 256; r += kThreads) {
    const float* p = b + (long long)(cz * KK + (r >> 4)) * sz + (long long)(cy * KK + (r & 15)) * sy + cx * KK;
    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
  }
}

// prologue + x/y stages; leaves c in U and dd in B (f16 tensors), trace planes ready
// KK = cell size: 8 (2-cell tiles) or 4 / 2 (16-point tile lines of 4 / 8 cells); the tile is a
// 16^3-point box either way, the line operators come from the tables.
template <int MODE, int KK = K>
__device__ __forceinline__ bool tile_front(HTile<MODE>& T, char* smem, const Geom& g, const LevelOp<KK, MODE>& op,
                                           const HTables* tab, const float* __restrict__ u) {
  T.uh = reinterpret_cast<__half*>(smem);
  T.bh = T.uh + TVOL;
  T.tr = reinterpret_cast<float*>(smem + sizeof(__half) * (MODE == MODE_FP16_EC ? 4 : 2) * TVOL);
  if (MODE == MODE_FP16_EC) T.bh = T.uh + TVOL;  // layout: uh | bh | ud | bd
  T.s_exp = reinterpret_cast<int*>(T.tr + 12 * 16 * 17);
  constexpr int CPL = 16 / KK;
  TileEngine<KK, MODE, 1, 16> e(smem, g);
  e.tr = T.tr;
  e.s_exp = T.s_exp;
  int cx, cy, cz;
  if (!e.tile_cells(g, 0, cx, cy, cz)) return false;
  if (threadIdx.x == 0) T.s_exp[0] = T.s_exp[1] = 0;
  __syncthreads();
  T.cx = cx; T.cy = cy; T.cz = cz;
  T.skip[0] = e.skip[0]; T.skip[1] = e.skip[1]; T.skip[2] = e.skip[2];
  T.sy = e.sy; T.sz = e.sz;
  T.nbm = 0;
  const int c0[3] = {cx, cy, cz};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (e.face_src(g, a, 0, c0[a]) != 2) T.nbm |= 1u << (2 * a);
    if (e.face_src(g, a, 1, c0[a]) != 2) T.nbm |= 1u << (2 * a + 1);
    const int n = a == 0 ? g.nx : (a == 1 ? g.ny : g.nz);  // kind of the 16-point line
    T.kind[a] = 2 * ((c0[a] == 0 && g.bnd_lo[a]) ? 1 : 0) + ((c0[a] + CPL == n && g.bnd_hi[a]) ? 1 : 0);
  }
  T.lane = threadIdx.x & 31;
  T.warp = threadIdx.x >> 5;
  T.g = T.lane >> 2;
  T.t = T.lane & 3;
#pragma unroll
  for (int hd = 0; hd < 2; ++hd)
#pragma unroll
    for (int i = 0; i < 2; ++i) {  // zero for lanes whose outputs are not in the line's first / last cell
      const int n0 = 2 * T.t + i, n1 = 2 * T.t + i - (8 - KK);
      T.hur[hd][i] = n0 < KK ? __ldg(&tab->urow[hd][n0]) : 0.f;
      T.huc[hd][i] = n1 >= 0 ? __ldg(&tab->ucol[hd][n1]) : 0.f;
    }
  // tile -> registers -> block exponent -> scaled (h, d) tensors
  const float* ub = u + (long long)(cz * KK) * T.sz + (long long)(cy * KK) * T.sy + cx * KK;
  // EC: the two x-neighbour cell layers (256 rows of KK floats per face) go to the still-free
  // B tensors by cp.async -- coalesced 16-byte chunks instead of per-lane KK-float loads that
  // touch 32 cache lines per warp instruction; the x traces are formed from shared memory below.
  constexpr bool kStageX = (MODE == MODE_FP16_EC) && (KK == 8 || KK == 4);
  constexpr int XC = KK / 4;  // 16-byte chunks per staged row
  if constexpr (kStageX) {
    const int sy = (int)T.sy, sz = (int)T.sz;
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      if (!((T.nbm >> hi) & 1)) continue;
      float* dst = reinterpret_cast<float*>(hi ? T.bd() : T.bh);
#pragma unroll
      for (int k2 = 0; k2 < 256 * XC / kThreads; ++k2) {
        const int c = threadIdx.x + kThreads * k2, ch = c % XC, row = c / XC, y = row & 15, z = row >> 4;
        const int sw = XC == 2 ? (ch ^ ((row >> 2) & 1)) : ch;  // conflict-free LDS.128 quarter-warps
        cp_async16(dst + row * KK + 4 * sw, ub + z * sz + y * sy + (hi ? 16 : -KK) + 4 * ch);
      }
    }
  }
  float4 q4[1024 / kThreads];
  float mx = 0.f;
#pragma unroll
  for (int k2 = 0; k2 < 1024 / kThreads; ++k2) {
    const int i = threadIdx.x + k2 * kThreads;
    const int x4 = (i & 3) * 4, y = (i >> 2) & 15, z = i >> 6;
    const float* src = ub + z * T.sz + y * T.sy + x4;
    if constexpr (KK == 2) {  // shifted colours start at an odd cell: only 8-byte alignment
      const float2 lo = __ldg(reinterpret_cast<const float2*>(src)), hi = __ldg(reinterpret_cast<const float2*>(src + 2));
      q4[k2] = make_float4(lo.x, lo.y, hi.x, hi.y);
    } else {
      q4[k2] = __ldg(reinterpret_cast<const float4*>(src));
    }
    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(q4[k2].x), fabsf(q4[k2].y)), fmaxf(fabsf(q4[k2].z), fabsf(q4[k2].w))));
  }
  smax(&T.s_exp[0], mx);
  if constexpr (kStageX) cp_async_wait_all();
  __syncthreads();
  T.eu = block_exp(__int_as_float(T.s_exp[0]));
  e.eu = T.eu;
  const float us = pow2f(T.eu);
#pragma unroll
  for (int k2 = 0; k2 < 1024 / kThreads; ++k2) {
    const int i = threadIdx.x + k2 * kThreads;
    const int x4 = (i & 3) * 4, y = (i >> 2) & 15, z = i >> 6;
    // x4..x4+3 are 4 consecutive halves of one 8-block in hidx: one 64-bit store per tensor
    uint2 hv, dv;
    demote_pair<MODE>(q4[k2].x * us, q4[k2].y * us, hv.x, dv.x);
    demote_pair<MODE>(q4[k2].z * us, q4[k2].w * us, hv.y, dv.y);
    const int o = hidx(z, y, x4);
    *reinterpret_cast<uint2*>(T.uh + o) = hv;
    if constexpr (MODE == MODE_FP16_EC) *reinterpret_cast<uint2*>(T.ud() + o) = dv;
  }
  if constexpr (kStageX) {
    // x traces from the staged rows: item (hi, p = z, q = y); EC beta in fp32 (as TileEngine::traces)
#pragma unroll
    for (int k2 = 0; k2 < 512 / kThreads; ++k2) {
      const int it = threadIdx.x + kThreads * k2, hi = it >> 8, row = it & 255, p = row >> 4, q = row & 15;
      if (!((T.nbm >> hi) & 1)) continue;
      const float* src = reinterpret_cast<const float*>(hi ? T.bd() : T.bh) + row * KK;
      float w[KK];
#pragma unroll
      for (int ch = 0; ch < XC; ++ch) {
        const int sw = XC == 2 ? (ch ^ ((row >> 2) & 1)) : ch;
        const float4 v4 = *reinterpret_cast<const float4*>(src + 4 * sw);
        w[4 * ch] = v4.x; w[4 * ch + 1] = v4.y; w[4 * ch + 2] = v4.z; w[4 * ch + 3] = v4.w;
      }
      float alpha, bs = 0.f;
      if (hi) {
        alpha = w[0] * us;
#pragma unroll
        for (int jj = 1; jj < KK; ++jj) bs = fmaf(op.urow[jj].h + op.urow[jj].d / kEcScale, w[jj] * us, bs);
      } else {
        alpha = w[KK - 1] * us;
#pragma unroll
        for (int jj = 0; jj < KK - 1; ++jj) bs = fmaf(op.ucol[jj].h + op.ucol[jj].d / kEcScale, w[jj] * us, bs);
      }
      float* pl = T.tr + (hi * 2) * (16 * 17);
      pl[p * 17 + q] = alpha;
      pl[16 * 17 + p * 17 + q] = bs;
    }
    e.template traces<kThreads, 1>(g, op, u);
  } else {
    e.template traces<kThreads>(g, op, u);
  }
  T.lane = threadIdx.x & 31;
  T.warp = threadIdx.x >> 5;
  T.g = T.lane >> 2;
  T.t = T.lane & 3;
  __syncthreads();
  trace_masses_tc<MODE>(T, tab);
  __syncthreads();

  int q, j;
  lane_qj(T.lane, q, j);
  BFrag<MODE> bm, bl;
  load_b<MODE>(bm, &tab->M[0][0][0][0], T.lane);
  // x and y stages on the warp's 4 z planes (in place)
  for (int zz = 0; zz < 4; ++zz) {
    const int z = 4 * T.warp + zz;
    load_b<MODE>(bl, &tab->L[T.kind[0]][0][0][0][0], T.lane);
    {
      AFrag<MODE> a;
      ld_a<MODE>(a, T.uh, T.ud(), hidx(z, j + 8 * (q & 1), 8 * (q >> 1)), false);
      Acc16<MODE> am, as;
      am.zero();
      as.zero();
      mma16<MODE>(am, a, bm);
      mma16<MODE>(as, a, bl);
      halo16<MODE>(T, as, tab, 0, trp(T, 0, 0) + z * 17, trp(T, 0, 1) + z * 17, trp(T, 1, 0) + z * 17,
                   trp(T, 1, 1) + z * 17);
      float va[2][4], vb[2][4];
      finals<MODE>(am, va);
      finals<MODE>(as, vb);
      __syncwarp();
      st_acc<MODE>(T.uh, T.ud(), hidx(z, j + 8 * (q & 1), 8 * (q >> 1)), va, false);
      st_acc<MODE>(T.bh, T.bd(), hidx(z, j + 8 * (q & 1), 8 * (q >> 1)), vb, false);
    }
    __syncwarp();
    load_b<MODE>(bl, &tab->L[T.kind[1]][0][0][0][0], T.lane);
    {
      // y lines: rows = x, k = y (memory rows along y -> trans)
      const int off = hidx(z, j + 8 * (q >> 1), 8 * (q & 1));
      AFrag<MODE> a, b;
      ld_a<MODE>(a, T.uh, T.ud(), off, true);
      ld_a<MODE>(b, T.bh, T.bd(), off, true);
      Acc16<MODE> c, d, e2;
      c.zero();
      d.zero();
      e2.zero();
      mma16<MODE>(c, a, bm);
      mma16<MODE>(d, a, bl);
      halo16<MODE>(T, d, tab, 1, trp(T, 2, 0) + z * 17, trp(T, 2, 1) + z * 17, trp(T, 3, 0) + z * 17,
                   trp(T, 3, 1) + z * 17);
      mma16<MODE>(e2, b, bm);
      float vc[2][4], vd[2][4];
      finals<MODE>(c, vc);
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) vd[nt][i] = d.val(nt, i) + e2.val(nt, i);
      __syncwarp();
      st_acc<MODE>(T.uh, T.ud(), off, vc, true);
      st_acc<MODE>(T.bh, T.bd(), off, vd, true);
    }
    __syncwarp();
  }
  return true;
}

// z stage for row y: v (16 lines x, 16 outputs z) as f32 values
template <int MODE>
__device__ __forceinline__ void z_lines(const HTile<MODE>& T, const HTables* tab, int y, const BFrag<MODE>& bm,
                                        const BFrag<MODE>& bl, float (&v)[2][4]) {
  int q, j;
  lane_qj(T.lane, q, j);
  const int off = hidx(j + 8 * (q >> 1), y, 8 * (q & 1));
  AFrag<MODE> c, d;
  ld_a<MODE>(c, T.uh, T.ud(), off, true);
  ld_a<MODE>(d, T.bh, T.bd(), off, true);
  Acc16<MODE> s, m;
  s.zero();
  m.zero();
  mma16<MODE>(s, c, bl);
  halo16<MODE>(T, s, tab, 2, trp(T, 4, 0) + y * 17, trp(T, 4, 1) + y * 17, trp(T, 5, 0) + y * 17,
               trp(T, 5, 1) + y * 17);
  mma16<MODE>(m, d, bm);
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) v[nt][i] = s.val(nt, i) + m.val(nt, i);
}

// accumulator element (nt, i): line = g + 8*(i>>1), output = 8nt + 2t + (i&1)
template <int MODE, int KK = K>
__global__ void __launch_bounds__(kThreads, 4) k_vmult_h8(const float* __restrict__ u, float* __restrict__ v, Geom g,
                                                         LevelOp<KK, MODE> op, const HTables* __restrict__ tab) {
  extern __shared__ __align__(128) char smem[];
  HTile<MODE> T;
  u += (long long)blockIdx.y * g.batch_stride;
  v += (long long)blockIdx.y * g.batch_stride;
  if (!tile_front<MODE, KK>(T, smem, g, op, tab, u)) return;
  __syncthreads();
  BFrag<MODE> bm, bl;
  load_b<MODE>(bm, &tab->M[0][0][0][0], T.lane);
  load_b<MODE>(bl, &tab->L[T.kind[2]][0][0][0][0], T.lane);
  float* vb = v + (long long)(T.cz * KK) * T.sz + (long long)(T.cy * KK) * T.sy + T.cx * KK;
  const float os = pow2f(-(op.sc.aA + T.eu));
  for (int yy = 0; yy < 4; ++yy) {
    const int y = 4 * T.warp + yy;
    float o[2][4];
    z_lines<MODE>(T, tab, y, bm, bl, o);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int x = T.g + 8 * (i >> 1), z = 8 * nt + 2 * T.t + (i & 1);
        vb[(long long)z * T.sz + (long long)y * T.sy + x] = o[nt][i] * os;
      }
  }
}

// smoother colour pass (see sf_dmma.cu k_colour_dmma8 for the stage order)
template <int MODE, int KK = K>
__global__ void __launch_bounds__(kThreads, 4) k_colour_h8(const float* __restrict__ xo, const float* __restrict__ b,
                                                          float* __restrict__ xn, Geom g, LevelOp<KK, MODE> op,
                                                          const HTables* __restrict__ tab) {
  extern __shared__ __align__(128) char smem[];
  HTile<MODE> T;
  prefetch_b_rows<KK>(g, b);
  if (!tile_front<MODE, KK>(T, smem, g, op, tab, xo)) return;
  __syncthreads();
  const int kx = T.kind[0], ky = T.kind[1], kz = T.kind[2];
  int q, j;
  lane_qj(T.lane, q, j);
  const long long off0 = (long long)(T.cz * KK) * T.sz + (long long)(T.cy * KK) * T.sy + T.cx * KK;
  BFrag<MODE> bm, bl, bv;
  load_b<MODE>(bm, &tab->M[0][0][0][0], T.lane);
  load_b<MODE>(bl, &tab->L[kz][0][0][0][0], T.lane);
  load_b<MODE>(bv, &tab->Vf[kz][0][0][0][0], T.lane);
  // z lines: residual r = b - A x (true units) -> block exponent -> forward V_z^T in registers
  float rr[4][2][4];
  const float os = pow2f(-(op.sc.aA + T.eu));
#pragma unroll
  for (int yy = 0; yy < 4; ++yy) {
    const int y = 4 * T.warp + yy;
    z_lines<MODE>(T, tab, y, bm, bl, rr[yy]);
    float mx = 0.f;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int x = T.g + 8 * (i >> 1), z = 8 * nt + 2 * T.t + (i & 1);
        rr[yy][nt][i] = __ldg(b + off0 + (long long)z * T.sz + (long long)y * T.sy + x) - rr[yy][nt][i] * os;
        mx = fmaxf(mx, fabsf(rr[yy][nt][i]));
      }
    smax(&T.s_exp[1], mx);
  }
  __syncthreads();  // all z-stage reads of U/B done, residual exponent complete
  const int er = block_exp(__int_as_float(T.s_exp[1]));
  const float rs = pow2f(er);
#pragma unroll
  for (int yy = 0; yy < 4; ++yy) {
    const int y = 4 * T.warp + yy;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) rr[yy][nt][i] *= rs;
    AFrag<MODE> a;
    acc_to_a<MODE>(rr[yy], a);
    Acc16<MODE> acc;
    acc.zero();
    mma16<MODE>(acc, a, bv);
    float o[2][4];
    finals<MODE>(acc, o);
    st_acc<MODE>(T.uh, T.ud(), hidx(j + 8 * (q >> 1), y, 8 * (q & 1)), o, true);
  }
  __syncthreads();
  // warp-private z' planes: V_y^T | V_x^T, 1/lambda, V_x | V_y
  const double* lamx = tab->lam[kx];
  const double* lamy = tab->lam[ky];
  const double* lamz = tab->lam[kz];
  for (int zz = 0; zz < 4; ++zz) {
    const int z = 4 * T.warp + zz;
    {
      load_b<MODE>(bv, &tab->Vf[ky][0][0][0][0], T.lane);
      const int off = hidx(z, j + 8 * (q >> 1), 8 * (q & 1));
      AFrag<MODE> a;
      ld_a<MODE>(a, T.uh, T.ud(), off, true);
      Acc16<MODE> acc;
      acc.zero();
      mma16<MODE>(acc, a, bv);
      float o[2][4];
      finals<MODE>(acc, o);
      __syncwarp();
      st_acc<MODE>(T.uh, T.ud(), off, o, true);
    }
    __syncwarp();
    {
      load_b<MODE>(bv, &tab->Vf[kx][0][0][0][0], T.lane);
      const int off = hidx(z, j + 8 * (q & 1), 8 * (q >> 1));
      AFrag<MODE> a;
      ld_a<MODE>(a, T.uh, T.ud(), off, false);
      Acc16<MODE> acc;
      acc.zero();
      mma16<MODE>(acc, a, bv);
      float o[2][4];
      const double lz = 0.0 + __ldg(lamz + z);
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int y = T.g + 8 * (i >> 1), x = 8 * nt + 2 * T.t + (i & 1);
          o[nt][i] = acc.val(nt, i) / (float)(((lz + __ldg(lamy + y)) + __ldg(lamx + x)) * pow2d(-op.sc.aD));
        }
      acc_to_a<MODE>(o, a);
      load_b<MODE>(bv, &tab->Vb[kx][0][0][0][0], T.lane);
      acc.zero();
      mma16<MODE>(acc, a, bv);
      finals<MODE>(acc, o);
      __syncwarp();
      st_acc<MODE>(T.uh, T.ud(), off, o, false);
    }
    __syncwarp();
    {
      load_b<MODE>(bv, &tab->Vb[ky][0][0][0][0], T.lane);
      const int off = hidx(z, j + 8 * (q >> 1), 8 * (q & 1));
      AFrag<MODE> a;
      ld_a<MODE>(a, T.uh, T.ud(), off, true);
      Acc16<MODE> acc;
      acc.zero();
      mma16<MODE>(acc, a, bv);
      float o[2][4];
      finals<MODE>(acc, o);
      __syncwarp();
      st_acc<MODE>(T.uh, T.ud(), off, o, true);
    }
    __syncwarp();
  }
  __syncthreads();
  // z lines: backward V_z, x_new = x_old + correction (back to true units)
  load_b<MODE>(bv, &tab->Vb[kz][0][0][0][0], T.lane);
  const float cs = pow2f(-(op.sc.aD + 6 * op.sc.aV + er));
  for (int yy = 0; yy < 4; ++yy) {
    const int y = 4 * T.warp + yy;
    AFrag<MODE> a;
    ld_a<MODE>(a, T.uh, T.ud(), hidx(j + 8 * (q >> 1), y, 8 * (q & 1)), true);
    Acc16<MODE> acc;
    acc.zero();
    mma16<MODE>(acc, a, bv);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int x = T.g + 8 * (i >> 1), z = 8 * nt + 2 * T.t + (i & 1);
        if (KK < 8 && (x < T.skip[0] || y < T.skip[1] || z < T.skip[2])) continue;
        const long long o = off0 + (long long)z * T.sz + (long long)y * T.sy + x;
        xn[o] = __ldg(xo + o) + acc.val(nt, i) * cs;
      }
  }
}


// residual + restriction (multigrid.py:249-250 + restrict :112-125): r = b - A x,
// block exponent, P^T along z on the tensor cores (chained), y and x on CUDA cores.
struct HPTab {
  unsigned PT[2][2][32];  // [h/d][j][lane], Op = P^T (8 x 16), one n8 tile
  float P[2][16][8];      // [h/d] demoted embedding
};

template <int MODE, int KK = K>
__global__ void __launch_bounds__(kThreads, 4) k_resid_restrict_h8(const float* __restrict__ x,
                                                                  const float* __restrict__ b,
                                                                  float* __restrict__ coarse, Geom g,
                                                                  LevelOp<KK, MODE> op,
                                                                  const HTables* __restrict__ tab,
                                                                  const HPTab* __restrict__ pt) {
  extern __shared__ __align__(128) char smem[];
  HTile<MODE> T;
  prefetch_b_rows<KK>(g, b);
  if (!tile_front<MODE, KK>(T, smem, g, op, tab, x)) return;
  __syncthreads();
  BFrag<MODE> bm, bl;
  load_b<MODE>(bm, &tab->M[0][0][0][0], T.lane);
  load_b<MODE>(bl, &tab->L[T.kind[2]][0][0][0][0], T.lane);
  const long long off0 = (long long)(T.cz * KK) * T.sz + (long long)(T.cy * KK) * T.sy + T.cx * KK;
  float rr[4][2][4];
  const float os = pow2f(-(op.sc.aA + T.eu));
#pragma unroll
  for (int yy = 0; yy < 4; ++yy) {
    const int y = 4 * T.warp + yy;
    z_lines<MODE>(T, tab, y, bm, bl, rr[yy]);
    float mx = 0.f;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int xx = T.g + 8 * (i >> 1), z = 8 * nt + 2 * T.t + (i & 1);
        rr[yy][nt][i] = __ldg(b + off0 + (long long)z * T.sz + (long long)y * T.sy + xx) - rr[yy][nt][i] * os;
        mx = fmaxf(mx, fabsf(rr[yy][nt][i]));
      }
    smax(&T.s_exp[1], mx);
  }
  __syncthreads();
  const int er = block_exp(__int_as_float(T.s_exp[1]));
  const float rs = pow2f(er);
  unsigned p0 = __ldg(&pt->PT[0][0][T.lane]), p1 = __ldg(&pt->PT[0][1][T.lane]);
  unsigned q0 = 0, q1 = 0;
  if constexpr (MODE == MODE_FP16_EC) {
    q0 = __ldg(&pt->PT[1][0][T.lane]);
    q1 = __ldg(&pt->PT[1][1][T.lane]);
  }
  float* S1 = reinterpret_cast<float*>(T.uh);  // [zc][y][x], plane pitch 260
#pragma unroll
  for (int yy = 0; yy < 4; ++yy) {
    const int y = 4 * T.warp + yy;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) rr[yy][nt][i] *= rs;
    AFrag<MODE> a;
    acc_to_a<MODE>(rr[yy], a);
    float m[4] = {0.f, 0.f, 0.f, 0.f}, c[4] = {0.f, 0.f, 0.f, 0.f};
    hmma(m, a.h, p0, p1);
    if constexpr (MODE == MODE_FP16_EC) {
      hmma(c, a.h, q0, q1);
      hmma(c, a.d, p0, p1);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int xx = T.g + 8 * (i >> 1), zc = 2 * T.t + (i & 1);
      S1[zc * 260 + y * 16 + xx] = MODE == MODE_FP16_EC ? m[i] + c[i] / kEc : m[i];
    }
  }
  __syncthreads();
  float* S2 = reinterpret_cast<float*>(T.bh);  // [zc][yc][x]
  {  // y lines (zc, x): 128 lines, one per thread
    const int xx = threadIdx.x & 15, zc = threadIdx.x >> 4;
    Op<MODE> w[16];
#pragma unroll
    for (int y = 0; y < 16; ++y) w[y] = prep<MODE>(S1[zc * 260 + y * 16 + xx]);
#pragma unroll
    for (int yc = 0; yc < 8; ++yc) {
      Acc<MODE> s;
#pragma unroll
      for (int y = 0; y < 16; ++y) {
        ME<MODE> e;
        e.h = __ldg(&pt->P[0][y][yc]);
        if constexpr (MODE == MODE_FP16_EC) e.d = __ldg(&pt->P[1][y][yc]);
        s.fma(e, w[y]);
      }
      S2[(zc * 8 + yc) * 16 + xx] = s.result();
    }
  }
  __syncthreads();
  if (threadIdx.x < 64) {  // x lines (zc, yc) -> coarse (true units)
    const int yc = threadIdx.x & 7, zc = threadIdx.x >> 3;
    Op<MODE> w[16];
#pragma unroll
    for (int xx = 0; xx < 16; ++xx) w[xx] = prep<MODE>(S2[(zc * 8 + yc) * 16 + xx]);
    const long long syc = (long long)(g.nx / 2) * KK, szc = syc * (long long)(g.ny / 2) * KK;
    float* out = coarse + (long long)((T.cz / 2) * KK + zc) * szc + (long long)((T.cy / 2) * KK + yc) * syc +
                 (T.cx / 2) * KK;
    const float back = pow2f(-er);
#pragma unroll
    for (int xc = 0; xc < 8; ++xc) {
      Acc<MODE> s;
#pragma unroll
      for (int xx = 0; xx < 16; ++xx) {
        ME<MODE> e;
        e.h = __ldg(&pt->P[0][xx][xc]);
        if constexpr (MODE == MODE_FP16_EC) e.d = __ldg(&pt->P[1][xx][xc]);
        s.fma(e, w[xx]);
      }
      out[xc] = s.result() * back;
    }
  }
}

// ------------------------------------------------------------- host side
static void split_host(int mode, double x, unsigned short& h, unsigned short& d) {
  const float x32 = (float)x;
  const __half hh = __float2half_rn(x32);
  h = *reinterpret_cast<const unsigned short*>(&hh);
  const float hf = __half2float(hh);
  const __half dd = __float2half_rn((x32 - hf) * kEc);
  d = mode == MODE_FP16_EC ? *reinterpret_cast<const unsigned short*>(&dd) : 0;
}

static void pack_op_frags(int mode, const double* Op /* [16][16] */, unsigned* dst /* [2][2][2][32] */) {
  for (int nt = 0; nt < 2; ++nt)
    for (int jj = 0; jj < 2; ++jj)
      for (int ln = 0; ln < 32; ++ln) {
        const int n = 8 * nt + (ln >> 2), k0 = 2 * (ln & 3) + 8 * jj;
        unsigned short h0, d0, h1, d1;
        split_host(mode, Op[n * 16 + k0], h0, d0);
        split_host(mode, Op[n * 16 + k0 + 1], h1, d1);
        dst[(0 * 4 + nt * 2 + jj) * 32 + ln] = (unsigned)h0 | ((unsigned)h1 << 16);
        dst[(1 * 4 + nt * 2 + jj) * 32 + ln] = (unsigned)d0 | ((unsigned)d1 << 16);
      }
}

static HTables build_tables(int mode, int KK, const double* opd, const double* eigd) {
  HTables t;
  std::memset(&t, 0, sizeof(t));
  double Mp[256], L[4][256], V[4][256], lam[4][16];
  build_line_ops_host(KK, opd, eigd, Mp, &L[0][0], eigd ? &V[0][0] : nullptr, &lam[0][0]);
  pack_op_frags(mode, Mp, &t.M[0][0][0][0]);
  for (int q = 0; q < 4; ++q) pack_op_frags(mode, L[q], &t.L[q][0][0][0][0]);
  if (eigd) {
    for (int q = 0; q < 4; ++q) {
      double VT[256];
      for (int i = 0; i < 16; ++i)
        for (int jj = 0; jj < 16; ++jj) VT[i * 16 + jj] = V[q][jj * 16 + i];
      pack_op_frags(mode, VT, &t.Vf[q][0][0][0][0]);
      pack_op_frags(mode, V[q], &t.Vb[q][0][0][0][0]);
      for (int i = 0; i < 16; ++i) t.lam[q][i] = lam[q][i];
    }
  }
  const double* ucol = opd + 2 * KK * KK;
  const double* urow = ucol + KK;
  for (int i = 0; i < KK; ++i) {
    unsigned short h, d;
    split_host(mode, ucol[i], h, d);
    t.ucol[0][i] = __half2float(*reinterpret_cast<__half*>(&h));
    t.ucol[1][i] = __half2float(*reinterpret_cast<__half*>(&d));
    split_host(mode, urow[i], h, d);
    t.urow[0][i] = __half2float(*reinterpret_cast<__half*>(&h));
    t.urow[1][i] = __half2float(*reinterpret_cast<__half*>(&d));
  }
  return t;
}

static std::mutex g_mu;
struct Entry {
  int dev, mode;
  std::vector<double> key;
  void* ptr;
};
static std::vector<Entry> g_cache;

static const HTables* tables(int mode, const double* opd, const double* eigd, int KK = K) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int nop = 2 * KK * KK + 4 * KK, neig = 4 * 4 * KK * KK + 4 * 2 * KK;
  std::vector<double> key(opd, opd + nop);
  if (eigd) key.insert(key.end(), eigd, eigd + neig);
  key.push_back(eigd ? 1.0 : 0.0);
  key.push_back((double)KK);
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& e : g_cache)
    if (e.dev == dev && e.mode == mode && e.key == key) return reinterpret_cast<const HTables*>(e.ptr);
  double op_s[2 * K * K + 4 * K], eig_s[4 * 256 + 4 * 16];
  level_scales(KK, opd, eigd, op_s, eigd ? eig_s : nullptr);
  HTables host = build_tables(mode, KK, op_s, eigd ? eig_s : nullptr);
  void* d = nullptr;
  if (cudaMalloc(&d, sizeof(HTables)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, &host, sizeof(HTables), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  g_cache.push_back({dev, mode, std::move(key), d});
  return reinterpret_cast<const HTables*>(d);
}

template <int MODE, int KK = K>
static LevelOp<KK, MODE> pack_op_h(const double* opd_raw, const double* eig_raw) {
  Prepared<KK, MODE> pr(opd_raw, eig_raw);
  const double* opd = pr.opd;
  LevelOp<KK, MODE> op;
  op.sc = pr.sc;
  for (int i = 0; i < KK; ++i)
    for (int jj = 0; jj < KK; ++jj) {
      op.M[i][jj] = pack_me<MODE>(opd[i * KK + jj]);
      op.D[i][jj] = pack_me<MODE>(opd[KK * KK + i * KK + jj]);
    }
  const double* vv = opd + 2 * KK * KK;
  for (int i = 0; i < KK; ++i) {
    op.ucol[i] = pack_me<MODE>(vv[i]);
    op.urow[i] = pack_me<MODE>(vv[KK + i]);
    op.bl[i] = pack_me<MODE>(vv[2 * KK + i]);
    op.br[i] = pack_me<MODE>(vv[3 * KK + i]);
  }
  return op;
}

template <int MODE>
static int vmult(const Geom& g, const double* opd, const void* u, void* v, int batch, cudaStream_t st) {
  const HTables* tab = tables(MODE, opd, nullptr);
  if (!tab) return -3;
  auto op = pack_op_h<MODE>(opd, nullptr);
  if (cudaFuncSetAttribute(k_vmult_h8<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<MODE>()) !=
      cudaSuccess)
    return -3;
  const int tiles = g.ntx * g.nty * g.ntz;
  k_vmult_h8<MODE><<<dim3(tiles, batch), kThreads, smem_bytes<MODE>(), st>>>((const float*)u, (float*)v, g, op, tab);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

template <int MODE>
static int colour(const Geom& g, const double* opd, const double* eigd, const void* xo, const void* b, void* xn,
                  cudaStream_t st) {
  const HTables* tab = tables(MODE, opd, eigd);
  if (!tab) return -3;
  auto op = pack_op_h<MODE>(opd, eigd);
  if (cudaFuncSetAttribute(k_colour_h8<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<MODE>()) !=
      cudaSuccess)
    return -3;
  const int tiles = g.ntx * g.nty * g.ntz;
  k_colour_h8<MODE><<<tiles, kThreads, smem_bytes<MODE>(), st>>>((const float*)xo, (const float*)b, (float*)xn, g, op,
                                                                 tab);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}


// Q3 / Q1 (KK = 4, 2): the 16-point tile-line kernels; kUseGeneric when the grid does not tile
template <int MODE, int KK>
static int vmult_line(const Geom& g0, const double* opd, const void* u, void* v, int batch, cudaStream_t st) {
  constexpr int CPL = 16 / KK;
  const int zc = 2 * g0.ntz;  // the caller's z range in cells
  if (g0.nx % CPL || g0.ny % CPL || zc % CPL) return kUseGeneric;
  Geom g = g0;
  g.ntx = g.nx / CPL;
  g.nty = g.ny / CPL;
  g.ntz = zc / CPL;
  const HTables* tab = tables(MODE, opd, nullptr, KK);
  if (!tab) return -3;
  auto op = pack_op_h<MODE, KK>(opd, nullptr);
  if (cudaFuncSetAttribute(k_vmult_h8<MODE, KK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem_bytes<MODE>()) != cudaSuccess)
    return -3;
  const int tiles = g.ntx * g.nty * g.ntz;
  k_vmult_h8<MODE, KK><<<dim3(tiles, batch), kThreads, smem_bytes<MODE>(), st>>>((const float*)u, (float*)v, g, op,
                                                                                 tab);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

template <int MODE, int KK>
static int colour_line(const Geom& g0, const double* opd, const double* eigd, const void* xo, const void* b, void* xn,
                       cudaStream_t st) {
  constexpr int CPL = 16 / KK;
  if (g0.nx % CPL || g0.ny % CPL || g0.nz % CPL) return kUseGeneric;
  const int n3[3] = {g0.nx, g0.ny, g0.nz}, s3[3] = {g0.tx0, g0.ty0, g0.tz0};
  for (int a = 0; a < 3; ++a)
    if (s3[a] && n3[a] < CPL + 2) return kUseGeneric;
  Geom g = g0;
  g.ntx = g.nx / CPL;
  g.nty = g.ny / CPL;
  g.ntz = g.nz / CPL;
  const HTables* tab = tables(MODE, opd, eigd, KK);
  if (!tab) return -3;
  auto op = pack_op_h<MODE, KK>(opd, eigd);
  if (cudaFuncSetAttribute(k_colour_h8<MODE, KK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem_bytes<MODE>()) != cudaSuccess)
    return -3;
  const int tiles = g.ntx * g.nty * g.ntz;
  k_colour_h8<MODE, KK><<<tiles, kThreads, smem_bytes<MODE>(), st>>>((const float*)xo, (const float*)b, (float*)xn, g,
                                                                     op, tab);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

static std::vector<std::pair<std::vector<double>, void*>> g_pcache;

static const HPTab* ptables(int mode, const double* embd_raw, int KK = K) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::vector<double> key(embd_raw, embd_raw + 2 * KK * KK);
  key.push_back((double)dev);
  key.push_back((double)mode);
  key.push_back((double)KK);
  double embd[16 * 8] = {};  // 16-point tile line -> 8 coarse points: blockdiag of the cell-pair embedding
  for (int c = 0; c < 16 / (2 * KK); ++c)
    for (int i = 0; i < 2 * KK; ++i)
      for (int j = 0; j < KK; ++j) embd[(c * 2 * KK + i) * 8 + c * KK + j] = embd_raw[i * KK + j];
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& e : g_pcache)
    if (e.first == key) return reinterpret_cast<const HPTab*>(e.second);
  HPTab t;
  std::memset(&t, 0, sizeof(t));
  for (int jj = 0; jj < 2; ++jj)
    for (int ln = 0; ln < 32; ++ln) {
      const int n = ln >> 2, k0 = 2 * (ln & 3) + 8 * jj;
      unsigned short h0, d0, h1, d1;
      split_host(mode, embd[k0 * 8 + n], h0, d0);  // (P^T)[n][k] = P[k][n]
      split_host(mode, embd[(k0 + 1) * 8 + n], h1, d1);
      t.PT[0][jj][ln] = (unsigned)h0 | ((unsigned)h1 << 16);
      t.PT[1][jj][ln] = (unsigned)d0 | ((unsigned)d1 << 16);
    }
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 8; ++j) {
      unsigned short hh, dd;
      split_host(mode, embd[i * 8 + j], hh, dd);
      t.P[0][i][j] = __half2float(*reinterpret_cast<__half*>(&hh));
      t.P[1][i][j] = __half2float(*reinterpret_cast<__half*>(&dd));
    }
  void* d = nullptr;
  if (cudaMalloc(&d, sizeof(HPTab)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, &t, sizeof(HPTab), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  g_pcache.push_back({std::move(key), d});
  return reinterpret_cast<const HPTab*>(d);
}

template <int MODE>
static int resid_restrict(const Geom& g, const double* opd, const double* embd, const void* x, const void* b,
                          void* coarse, cudaStream_t st) {
  const HTables* tab = tables(MODE, opd, nullptr);
  const HPTab* pt = ptables(MODE, embd);
  if (!tab || !pt) return -3;
  auto op = pack_op_h<MODE>(opd, nullptr);
  if (cudaFuncSetAttribute(k_resid_restrict_h8<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem_bytes<MODE>()) != cudaSuccess)
    return -3;
  const int tiles = g.ntx * g.nty * g.ntz;
  k_resid_restrict_h8<MODE><<<tiles, kThreads, smem_bytes<MODE>(), st>>>((const float*)x, (const float*)b,
                                                                         (float*)coarse, g, op, tab, pt);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

template <int MODE, int KK>
static int resid_restrict_line(const Geom& g0, const double* opd, const double* embd, const void* x, const void* b,
                               void* coarse, cudaStream_t st) {
  constexpr int CPL = 16 / KK;
  if (g0.nx % CPL || g0.ny % CPL || g0.nz % CPL) return kUseGeneric;
  Geom g = g0;
  g.ntx = g.nx / CPL;
  g.nty = g.ny / CPL;
  g.ntz = g.nz / CPL;
  const HTables* tab = tables(MODE, opd, nullptr, KK);
  const HPTab* pt = ptables(MODE, embd, KK);
  if (!tab || !pt) return -3;
  auto op = pack_op_h<MODE, KK>(opd, nullptr);
  if (cudaFuncSetAttribute(k_resid_restrict_h8<MODE, KK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem_bytes<MODE>()) != cudaSuccess)
    return -3;
  const int tiles = g.ntx * g.nty * g.ntz;
  k_resid_restrict_h8<MODE, KK><<<tiles, kThreads, smem_bytes<MODE>(), st>>>((const float*)x, (const float*)b,
                                                                             (float*)coarse, g, op, tab, pt);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace hm

int launch_vmult_hmma_line(int mode, int k_nodes, const Geom& g, const double* opd, const void* u, void* v, int batch,
                           cudaStream_t st) {
  const bool ec = mode == MODE_FP16_EC;
  if (k_nodes == 4) return ec ? hm::vmult_line<MODE_FP16_EC, 4>(g, opd, u, v, batch, st)
                              : hm::vmult_line<MODE_FP16, 4>(g, opd, u, v, batch, st);
  if (k_nodes == 2) return ec ? hm::vmult_line<MODE_FP16_EC, 2>(g, opd, u, v, batch, st)
                              : hm::vmult_line<MODE_FP16, 2>(g, opd, u, v, batch, st);
  return kUseGeneric;
}

int launch_colour_hmma_line(int mode, int k_nodes, const Geom& g, const double* opd, const double* eigd,
                            const void* xo, const void* b, void* xn, cudaStream_t st) {
  const bool ec = mode == MODE_FP16_EC;
  if (k_nodes == 4) return ec ? hm::colour_line<MODE_FP16_EC, 4>(g, opd, eigd, xo, b, xn, st)
                              : hm::colour_line<MODE_FP16, 4>(g, opd, eigd, xo, b, xn, st);
  if (k_nodes == 2) return ec ? hm::colour_line<MODE_FP16_EC, 2>(g, opd, eigd, xo, b, xn, st)
                              : hm::colour_line<MODE_FP16, 2>(g, opd, eigd, xo, b, xn, st);
  return kUseGeneric;
}

int launch_vmult_hmma8(int mode, const Geom& g, const double* opd, const void* u, void* v, int batch,
                       cudaStream_t st) {
  return mode == MODE_FP16 ? hm::vmult<MODE_FP16>(g, opd, u, v, batch, st)
                           : hm::vmult<MODE_FP16_EC>(g, opd, u, v, batch, st);
}

int launch_colour_hmma8(int mode, const Geom& g, const double* opd, const double* eigd, const void* xo, const void* b,
                        void* xn, cudaStream_t st) {
  return mode == MODE_FP16 ? hm::colour<MODE_FP16>(g, opd, eigd, xo, b, xn, st)
                           : hm::colour<MODE_FP16_EC>(g, opd, eigd, xo, b, xn, st);
}

int launch_resid_restrict_hmma_line(int mode, int k_nodes, const Geom& g, const double* opd, const double* embd,
                                    const void* x, const void* b, void* coarse, cudaStream_t st) {
  const bool ec = mode == MODE_FP16_EC;
  if (k_nodes == 4) return ec ? hm::resid_restrict_line<MODE_FP16_EC, 4>(g, opd, embd, x, b, coarse, st)
                              : hm::resid_restrict_line<MODE_FP16, 4>(g, opd, embd, x, b, coarse, st);
  if (k_nodes == 2) return ec ? hm::resid_restrict_line<MODE_FP16_EC, 2>(g, opd, embd, x, b, coarse, st)
                              : hm::resid_restrict_line<MODE_FP16, 2>(g, opd, embd, x, b, coarse, st);
  return kUseGeneric;
}

int launch_resid_restrict_hmma8(int mode, const Geom& g, const double* opd, const double* embd, const void* x,
                                const void* b, void* coarse, cudaStream_t st) {
  return mode == MODE_FP16 ? hm::resid_restrict<MODE_FP16>(g, opd, embd, x, b, coarse, st)
                           : hm::resid_restrict<MODE_FP16_EC>(g, opd, embd, x, b, coarse, st);
}

}  // namespace sf
