// K2: matrix-free fine-level Navier-Stokes residual on Q2 hexahedra.
//
// Reference: Assembler.apply_operator / assemble_residual / assemble_rhs_next /
// stab (assembly.py:148-267) on the geometry cache of assembly.py:65-108.  The
// reference precomputes dense per-(cell, Gauss point, node) gradient tables
// G, Gpi (0.8 MB per cell).  Here nothing per quadrature point is stored: the
// isoparametric map, the fields and the test contractions are evaluated per
// cell by sum factorisation over the tensor-product Q2 basis (3 nodes x 4 Gauss
// points per axis).  One cell is handled by a group of 64 threads (one per
// Gauss point in the pointwise phase):
//
//  gather   : 27 node values (p, v) and the node coordinates relative to the
//             cell's first node (fp64 difference -> fp32), vmax for stab,
//             pi-projected nodal values PI*p, PI*v (elements.py:96-118)
//  forward  : 11 scalar fields (X^, p, v, pi p, pi v) -> value + 3 reference
//             derivatives at the 64 Gauss points, 3 one-dimensional stages
//  pointwise: J, det J, J^-1; physical gradients; the per-q coefficients of the
//             value test (N) and reference-gradient tests (dN), plus the
//             Gpi = PI^T-projected gradient test of the LPS terms
//  backward : transpose contraction 64 -> 27 per component (3 stages), PI^T
//  output   : element vector (cont, mom) per local node as a float4
//
// A second kernel sums element vectors per node over its incident cells in
// ascending cell id (the order of the reference's np.bincount, assembly.py:183),
// so results are deterministic and independent of the launch configuration;
// no float atomics are used.
#include <cstdlib>

#include "common.cuh"
#include "tc_common.cuh"

namespace dnnmg {

// ---- constant 1-D tables (elements.py:34-46, 79-93) --------------------------
namespace tab {
constexpr double xg[4] = {0.06943184420297371, 0.33000947820757187, 0.6699905217924281,
                          0.9305681557970262};
constexpr double wg[4] = {0.17392742256872692, 0.3260725774312731, 0.3260725774312731,
                          0.17392742256872692};
constexpr double phi(int i, double x) {
  return i == 0 ? 2.0 * (x - 0.5) * (x - 1.0) : i == 1 ? 4.0 * x * (1.0 - x) : 2.0 * x * (x - 0.5);
}
constexpr double dphi(int i, double x) {
  return i == 0 ? 4.0 * x - 3.0 : i == 1 ? 4.0 - 8.0 * x : 4.0 * x - 1.0;
}
}  // namespace tab

#define QB(q, i) float(tab::phi(i, tab::xg[q]))
#define QD(q, i) float(tab::dphi(i, tab::xg[q]))
__constant__ float cB[4][3] = {{QB(0, 0), QB(0, 1), QB(0, 2)}, {QB(1, 0), QB(1, 1), QB(1, 2)},
                               {QB(2, 0), QB(2, 1), QB(2, 2)}, {QB(3, 0), QB(3, 1), QB(3, 2)}};
__constant__ float cD[4][3] = {{QD(0, 0), QD(0, 1), QD(0, 2)}, {QD(1, 0), QD(1, 1), QD(1, 2)},
                               {QD(2, 0), QD(2, 1), QD(2, 2)}, {QD(3, 0), QD(3, 1), QD(3, 2)}};
__constant__ float cX[4] = {float(tab::xg[0]), float(tab::xg[1]), float(tab::xg[2]),
                            float(tab::xg[3])};
__constant__ float cW[4] = {float(tab::wg[0]), float(tab::wg[1]), float(tab::wg[2]),
                            float(tab::wg[3])};
#undef QB
#undef QD

// ---- per-cell shared-memory layout (floats) --------------------------------
// One warp per cell; lanes take Gauss points q = lane and lane + 32 in the
// pointwise phase and "lines" of the 1-D contractions in the other stages.
// Q2 fields through the sum-factorised forward stages: X^x, X^y, X^z, p, vx, vy, vz.
// The pi-projected (Q1) fields are trilinear in the 8 vertex values and are
// evaluated per Gauss point directly from those (elements.py:96-118).
constexpr int kNF = 7;
constexpr int oU = 0;                  // u[f][27]
constexpr int oSY = 192;               // sy[f][kind*3+iz][16 yx]            | backward out tz
constexpr int oVtx = 112;              // cached form (4 fields in u[0..108)): vertex float4 x 8
constexpr int kSYF = 148;              // sy field stride (= 20 mod 32: the (f, qx) lanes of the
                                       // forward x-y stage store to distinct banks)
constexpr int oCF = oSY + kNF * kSYF;  // cf[25][kCFS]: A[4], B[4][3], P[3][3]
constexpr int kNCF = 25;
// coefficient array stride and position of Gauss point q in an array: the second half of
// the points (qz >= 2) is shifted by 4 floats, so that the four qz lanes of one (comp, part)
// line of the backward stage read float4s from four different bank groups, and array a starts
// in bank 8a (mod 32), so that the two lines of a quarter-warp do not collide either (every
// backward LDS.128 is 4 wavefronts; with qz-stride 16 and no shift it was 8)
constexpr int kCFS = 72;
__host__ __device__ constexpr int cfq(int q) { return q + ((q >> 5) << 2); }
constexpr int oTZ = oSY;              // tz[4][2][kTZS] aliases sy (dead after the pointwise phase)
constexpr int kTZ2 = 33;              // row stride of tz in the split backward form (4 rows)
constexpr int kTZS = 28;              // row stride of tz: with 28 the backward stage's 32 output
                                      // stores (row cp, offsets 0/7/14/21) hit 32 distinct banks
constexpr int kCellFloats = (oCF + kNCF * kCFS + 3) / 4 * 4;
static_assert(oTZ + 4 * 2 * kTZS <= oCF, "tz must fit in sy");
static_assert(oSY % 4 == 0 && oCF % 4 == 0, "float4 alignment");

// Layout of the geometry-cached form: J^-1 and w per Gauss point come from a per-mesh
// cache (geometry_kernel), so only p and v (4 fields) go through the forward stages and
// the cell's cached block [10][64] is staged by cp.async one cell ahead.
// GEO: 0 = geometry recomputed per call, 1 = per-point cache staged per cell, 2 = per-cell box
// record (axis-aligned cells: J^-1 diagonal and constant over the cell, nothing staged)
enum { GEO_NONE = 0, GEO_CACHED = 1, GEO_BOX = 2 };
template <int GEO>
struct KLay {
  static constexpr bool CACHED = GEO != GEO_NONE;
  static constexpr int NF = CACHED ? 4 : kNF;         // Q2 fields through the forward stages
  static constexpr int US = CACHED ? 28 : 27;         // field stride of u (28: rows 16-byte aligned,
                                                      // the forward x-y stage reads them as float4)
  static constexpr int FO = NF - 4;                    // index of p among them
  // start of field f in sy.  Cached forms: the forward x-y stage runs on lanes (f, qx, qy half),
  // whose stores are 8 floats apart per half; fields 2 and 3 are shifted by 8 so that the eight
  // (f, half) groups of a store hit eight distinct 4-bank groups (with the plain stride: 2-way
  // conflicts on all 18 stores per lane)
  __host__ __device__ static constexpr int sy(int f) { return f * kSYF + (CACHED && f >= 2 ? 8 : 0); }
  static constexpr int oCF = oSY + NF * kSYF + (CACHED ? 8 : 0);
  static constexpr int oGQ = oCF + kNCF * kCFS;        // cached [J^-1 (9) | w][64]
  static constexpr int oBar = oGQ + 10 * 64;           // cached: the staging mbarrier (8 B)
  // a block of zeros: the value-test array of the part-1 (LPS) lanes of the backward stage
  static constexpr int oZero = (oGQ + (GEO == GEO_CACHED ? 10 * 64 + 4 : 0) + 3) / 4 * 4;
  static constexpr int kFloats = oZero + kCFS + 32;
  static_assert(oTZ + 4 * 2 * kTZS <= oCF && oCF % 4 == 0 && oGQ % 4 == 0, "layout");
};
// coefficient arrays (numbered so that every backward load slot hits distinct banks)
constexpr int CA = 0;        // A[c]      value test           (c = 0..3)
constexpr int CB = 4;        // B[c][k]   reference-gradient test
constexpr int CP = 16;       // P[i][k] = delta*w*g_i (J^-1 pi v)_k: LPS Gpi test, comps 1..3
#ifndef DNNMG_K2_WPB
#define DNNMG_K2_WPB 16
#endif
// warps per block of the element kernel: one 16-warp block per SM instead of four 4-warp blocks
// (the operator form needs 128 registers, 16 warps per SM either way): 0.827 -> 0.805 ms at
// config 3; the 16 warps work on neighbouring cells.  The RHS form (95-107 registers, five
// 4-warp blocks would fit) measured the same way: 0.556 -> 0.538 ms at config 3.
__host__ __device__ constexpr int k2_warps_per_block(int /*mode*/) { return DNNMG_K2_WPB; }

enum { MODE_OPERATOR = 0, MODE_RHS = 1 };

struct ResidualArgs {
  int n_cells;
  const int32_t* cell_nodes;
  const double* coords;
  const float4* x;
  const float* h_T;
  const float* alpha_in;
  const float* delta_in;
  float nu, k, alpha0, delta0;
  float ik;  // 1/k
  const float* geo_q;  // per-mesh geometry cache [n_cells][10][64] (J^-1 row-major, w) or NULL
  const float4* geo_box;  // per-cell (1/hx, 1/hy, 1/hz, det J) of an axis-aligned level or NULL
  int convection;
  int mode;
  float4* elem;
};

// reciprocal: MUFU rcp + one Newton step (|rel. err| ~1 ulp; no IEEE-division slow path)
__device__ __forceinline__ float frcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return fmaf(fmaf(-x, r, 1.0f), r, r);
}

// PI[b][v] for local node b (lattice ib) and vertex lattice iv in {0,2}^3 (elements.py:96-118)
__host__ __device__ constexpr float pi_weight(int b, int v) {
  float w = 1.f;
  for (int k = 0, bb = b, vv = v; k < 3; ++k, bb /= 3, vv /= 3) {
    const int ib = bb % 3, iv = vv % 3;
    w *= (ib == 1) ? 0.5f : (ib == iv ? 1.f : 0.f);
  }
  return w;
}

// two-deep software pipeline of the node gather: the index of cell i+2 and the
// raw (unconsumed) coordinates/state of cell i+1 are in flight while cell i computes
struct NodeRaw {
  double X[3], X0[3];
  float4 xv;
  float4 gb;  // GEO_BOX: the cell's box record
  float hT;
};

template <int GEO>
__device__ __forceinline__ void load_raw(const ResidualArgs& A, int c, int node, int t, NodeRaw& r) {
  if constexpr (GEO == GEO_BOX) r.gb = __ldg(A.geo_box + c);
  if constexpr (GEO == GEO_NONE) {
    const int n0 = __shfl_sync(0xffffffffu, node, 0);
    const double* X = A.coords + 3 * (int64_t)node;
    const double* X0 = A.coords + 3 * (int64_t)n0;
    if (t < 27) {
      r.X[0] = __ldg(X);
      r.X[1] = __ldg(X + 1);
      r.X[2] = __ldg(X + 2);
      r.X0[0] = __ldg(X0);
      r.X0[1] = __ldg(X0 + 1);
      r.X0[2] = __ldg(X0 + 2);
    }
  }
  if (t < 27) r.xv = __ldg(A.x + node);
  r.hT = __ldg(A.h_T + c);
}

// cp.async of cell c's cached geometry block (2560 B = 160 x 16 B, 5 per lane)
// the cell's contiguous 2,560-byte geometry block, one bulk (TMA) copy issued by lane 0 and
// completed on the warp's mbarrier (per-lane cp.async cost 11 shared wavefronts per 512 B)
__device__ __forceinline__ void stage_geo(const ResidualArgs& A, int c, int t, float* dst,
                                          uint32_t bar) {
  if (t == 0) {
    fence_async_smem();  // the previous cell's generic reads of dst precede the async write
    mbar_expect_tx(bar, 640 * 4);
    bulk_g2s(smem_u32(dst), A.geo_q + (int64_t)c * 640, 640 * 4, bar);
  }
}

// Q1 (pi) fields p, vx, vy, vz at the two Gauss points (qx, qy, qz) and (qx, qy, qz + 2) of a
// lane: trilinear in the 8 vertex values (elements.py:96-118); the x-y bilinear part is
// shared by the two points.  PQ[f] = [value, d/dxi, d/deta, d/dzeta]
// vtx (nullable): the 8 vertex values as float4 (p, vx, vy, vz) [vz][vy][vx], read with 8
// vector loads instead of 32 scalar ones from the field-major u
__device__ __forceinline__ void pi_fields(const float* u, const float4* vtx, int qx, int qy,
                                          int qz, float PQa[4][4], float PQb[4][4]) {
  const float lx1 = cX[qx], ly1 = cX[qy], lza = cX[qz], lzb = cX[qz + 2];
  float4 V[8];
  if (vtx) {
#pragma unroll
    for (int k = 0; k < 8; ++k) V[k] = vtx[k];
  }
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const float* uf = u + f * 27;
    float a[2][2], ax[2][2];
#pragma unroll
    for (int vz = 0; vz < 2; ++vz)
#pragma unroll
      for (int vy = 0; vy < 2; ++vy) {
        float g0, g1;
        if (vtx) {
          const float4 v0 = V[4 * vz + 2 * vy], v1 = V[4 * vz + 2 * vy + 1];
          g0 = f == 0 ? v0.x : f == 1 ? v0.y : f == 2 ? v0.z : v0.w;
          g1 = f == 0 ? v1.x : f == 1 ? v1.y : f == 2 ? v1.z : v1.w;
        } else {
          g0 = uf[18 * vz + 6 * vy];
          g1 = uf[18 * vz + 6 * vy + 2];
        }
        a[vz][vy] = fmaf(lx1, g1 - g0, g0);
        ax[vz][vy] = g1 - g0;
      }
    float b[2], bx[2], by[2];
#pragma unroll
    for (int vz = 0; vz < 2; ++vz) {
      b[vz] = fmaf(ly1, a[vz][1] - a[vz][0], a[vz][0]);
      bx[vz] = fmaf(ly1, ax[vz][1] - ax[vz][0], ax[vz][0]);
      by[vz] = a[vz][1] - a[vz][0];
    }
    const float db = b[1] - b[0], dbx = bx[1] - bx[0], dby = by[1] - by[0];
    PQa[f][0] = fmaf(lza, db, b[0]);
    PQa[f][1] = fmaf(lza, dbx, bx[0]);
    PQa[f][2] = fmaf(lza, dby, by[0]);
    PQa[f][3] = db;
    PQb[f][0] = fmaf(lzb, db, b[0]);
    PQb[f][1] = fmaf(lzb, dbx, bx[0]);
    PQb[f][2] = fmaf(lzb, dby, by[0]);
    PQb[f][3] = db;
  }
}

// coefficients of one Gauss point (pointwise phase); F = Q2 fields at q, PQ = pi fields at q.
// JM abstracts J^-1: full 3x3 (recomputed or cached per point) or the diagonal of a box cell,
// where every product with an off-diagonal entry is dropped (exact: those entries are zero)
struct JFull {
  float Ji[3][3];  // (J^-1)[k][j]: reference k -> physical j
  // physical gradient from reference derivatives d[0..2]: sum_k d[k] Ji[k][j]
  __device__ __forceinline__ float phys(const float d0, const float d1, const float d2, int j) const {
    return d0 * Ji[0][j] + d1 * Ji[1][j] + d2 * Ji[2][j];
  }
  // reference component k of J^-1 applied to a physical vector
  __device__ __forceinline__ float ref(const float e0, const float e1, const float e2, int k) const {
    return Ji[k][0] * e0 + Ji[k][1] * e1 + Ji[k][2] * e2;
  }
};
struct JBox {
  float s[3];  // (J^-1)[k][k]
  __device__ __forceinline__ float phys(const float d0, const float d1, const float d2, int j) const {
    return (j == 0 ? d0 : j == 1 ? d1 : d2) * s[j];
  }
  __device__ __forceinline__ float ref(const float e0, const float e1, const float e2, int k) const {
    return s[k] * (k == 0 ? e0 : k == 1 ? e1 : e2);
  }
};

template <int MODE, int NF, int FO, class JM>
__device__ __forceinline__ void pointwise_core(const ResidualArgs& A, float* CF, int q, const JM& M,
                                               float w, float F[NF][4], const float PQ[4][4],
                                               float aT, float dT) {
  float v[3], gv[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    v[i] = F[FO + 1 + i][0];
#pragma unroll
    for (int j = 0; j < 3; ++j)
      gv[i][j] = M.phys(F[FO + 1 + i][1], F[FO + 1 + i][2], F[FO + 1 + i][3], j);
  }
  float conv[3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
    conv[i] = A.convection ? v[0] * gv[i][0] + v[1] * gv[i][1] + v[2] * gv[i][2] : 0.f;
#define CFW(arr) CF[(arr) * kCFS + cfq(q)]
  const float ik = A.ik;
  if constexpr (MODE == MODE_OPERATOR) {
    const float p = F[FO][0];
    // physical gradient of the pressure fluctuation p - pi p
    const float dd0 = F[FO][1] - PQ[0][1], dd1 = F[FO][2] - PQ[0][2], dd3 = F[FO][3] - PQ[0][3];
    float gdp[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) gdp[j] = M.phys(dd0, dd1, dd3, j);
    const bool use_d = A.convection && dT != 0.f;
    float g[3] = {0.f, 0.f, 0.f}, pvr[3] = {0.f, 0.f, 0.f};
    if (use_d) {
      // pvr = J^-1 pi v; (pi v . grad) pi v_i = sum_m d(pi v_i)/dxi_m pvr_m
#pragma unroll
      for (int kk = 0; kk < 3; ++kk) pvr[kk] = M.ref(PQ[1][0], PQ[2][0], PQ[3][0], kk);
#pragma unroll
      for (int i = 0; i < 3; ++i)
        g[i] = conv[i] - (PQ[1 + i][1] * pvr[0] + PQ[1 + i][2] * pvr[1] + PQ[1 + i][3] * pvr[2]);
    }
    const float div = gv[0][0] + gv[1][1] + gv[2][2];
    float E[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) E[j] = aT * w * gdp[j];
    CFW(CA + 0) = w * div;
#pragma unroll
    for (int kk = 0; kk < 3; ++kk) CFW(CB + kk) = M.ref(E[0], E[1], E[2], kk);
    const float hn = 0.5f * A.nu * w;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      CFW(CA + 1 + i) = w * (v[i] * ik + 0.5f * conv[i]);
      const float dg = dT * w * g[i];
#pragma unroll
      for (int kk = 0; kk < 3; ++kk) CFW(CP + 3 * i + kk) = dg * pvr[kk];
      float Fi[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) Fi[j] = hn * gv[i][j] + dg * v[j] - (i == j ? w * p : 0.f);
#pragma unroll
      for (int kk = 0; kk < 3; ++kk) CFW(CB + 3 * (1 + i) + kk) = M.ref(Fi[0], Fi[1], Fi[2], kk);
    }
  } else {  // MODE_RHS (assembly.py:242-259, f = None)
    const float hn = -0.5f * A.nu * w;
    CFW(CA + 0) = 0.f;
#pragma unroll
    for (int kk = 0; kk < 3; ++kk) CFW(CB + kk) = 0.f;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      CFW(CA + 1 + i) = w * (v[i] * ik - 0.5f * conv[i]);
#pragma unroll
      for (int kk = 0; kk < 3; ++kk)
        CFW(CB + 3 * (1 + i) + kk) = hn * M.ref(gv[i][0], gv[i][1], gv[i][2], kk);
    }
  }
#undef CFW
}

// box: (1/hx, 1/hy, 1/hz, det J) of the cell; wq = the Gauss weight of point q
template <int MODE, int GEO>
__device__ __forceinline__ void pointwise(const ResidualArgs& A, const float* S, float* CF, int q,
                                          float F[KLay<GEO>::NF][4], const float PQ[4][4],
                                          float aT, float dT, const float4 box, float wq) {
  using L = KLay<GEO>;
  const int qx = q & 3, qy = (q >> 2) & 3, qz = q >> 4;
  if constexpr (GEO == GEO_BOX) {
    JBox M;
    M.s[0] = box.x;
    M.s[1] = box.y;
    M.s[2] = box.z;
    pointwise_core<MODE, L::NF, L::FO>(A, CF, q, M, wq * box.w, F, PQ, aT, dT);
  } else {
    JFull M;
    float w;
    if constexpr (GEO == GEO_CACHED) {
      const float* G = S + L::oGQ;
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int j = 0; j < 3; ++j) M.Ji[k][j] = G[(3 * k + j) * 64 + q];
      w = G[9 * 64 + q];
    } else {
      float J[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) J[i][j] = F[i][1 + j];
      const float c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
      const float c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
      const float c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
      const float det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
      const float id = 1.0f / det;
      M.Ji[0][0] = c00 * id;
      M.Ji[1][0] = c01 * id;
      M.Ji[2][0] = c02 * id;
      M.Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
      M.Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
      M.Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
      M.Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
      M.Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
      M.Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
      w = cW[qx] * cW[qy] * cW[qz] * det;
    }
    pointwise_core<MODE, L::NF, L::FO>(A, CF, q, M, w, F, PQ, aT, dT);
  }
}

template <int MODE, int GEO>
__global__ void __launch_bounds__(32 * k2_warps_per_block(MODE), 16 / k2_warps_per_block(MODE))
    element_kernel(ResidualArgs A) {
  constexpr int kWarpsPerBlock = k2_warps_per_block(MODE);
  using L = KLay<GEO>;
  constexpr bool CACHED = L::CACHED;          // 4 fields through the forward stages
  constexpr bool STAGED = GEO == GEO_CACHED;  // per-point geometry block staged per cell
  constexpr int NF = L::NF;
  extern __shared__ __align__(16) float smem[];
  const int wib = threadIdx.x >> 5;
  const int t = threadIdx.x & 31;
  float* S = smem + wib * L::kFloats;
#ifdef DNNMG_K2_GRIDSTRIDE
  constexpr bool kChunked = false;
#else
  // (measured: box form 0.805 -> 0.799 ms at config 3; general form 0.915 -> 0.917 at config 2)
  constexpr bool kChunked = MODE == MODE_OPERATOR && GEO == GEO_BOX;
#endif
  int stride, c, c_end;
  if constexpr (!kChunked) {
    stride = gridDim.x * kWarpsPerBlock;
    c = blockIdx.x * kWarpsPerBlock + wib;
    c_end = A.n_cells;
  } else {
  // a block takes a contiguous range of cells and its warps walk it side by side: the cells in
  // flight on an SM (and those of the next iterations) are neighbours in the numbering -- the
  // eight children of a coarse cell, then its x neighbour -- and share their nodes in L1
    stride = kWarpsPerBlock;
    const int per_block = (A.n_cells + gridDim.x - 1) / gridDim.x;
    c = blockIdx.x * per_block + wib;
    c_end = min(A.n_cells, (int)(blockIdx.x + 1) * per_block);
  }
  NodeRaw raw;
  int idx_next = 0;  // node index of cell c + stride (lane t < 27)
  const uint32_t bar = smem_u32(S + L::oBar);
  uint32_t phase = 0;
  if constexpr (STAGED) {
    if (t == 0) {
      mbar_init(bar, 1);
      fence_async_smem();
    }
    __syncwarp();
  }
  for (int i = t; i < kCFS + 32; i += 32) S[L::oZero + i] = 0.f;
  __syncwarp();
  // Gauss weights of this lane's two points q = t and t + 32 (box form: w = wq det J)
  const float wq_a = cW[t & 3] * cW[(t >> 2) & 3] * cW[t >> 4];
  const float wq_b = cW[t & 3] * cW[(t >> 2) & 3] * cW[(t >> 4) + 2];
  if (c < c_end) {
    const int node = t < 27 ? __ldg(A.cell_nodes + (int64_t)c * 27 + t) : 0;
    load_raw<GEO>(A, c, node, t, raw);
    if (c + stride < c_end && t < 27) idx_next = __ldg(A.cell_nodes + (int64_t)(c + stride) * 27 + t);
    if constexpr (STAGED) stage_geo(A, c, t, S + L::oGQ, bar);
  }

  for (; c < c_end; c += stride) {
    // ---------------- gather (prefetched one cell ahead), stab ----------------
    float vsq = 0.f;  // |v|^2 of this lane's node; vmax = sqrt(max |v|^2) (sqrt is monotone)
    if (t < 27) {
      if constexpr (!CACHED) {
        S[oU + 0 * L::US + t] = float(raw.X[0] - raw.X0[0]);
        S[oU + 1 * L::US + t] = float(raw.X[1] - raw.X0[1]);
        S[oU + 2 * L::US + t] = float(raw.X[2] - raw.X0[2]);
      }
      S[oU + (L::FO + 0) * L::US + t] = raw.xv.x;
      S[oU + (L::FO + 1) * L::US + t] = raw.xv.y;
      S[oU + (L::FO + 2) * L::US + t] = raw.xv.z;
      S[oU + (L::FO + 3) * L::US + t] = raw.xv.w;
      if constexpr (CACHED) {   // vertex copy as float4 (pi fields)
        const int ix = t % 3, iy = (t / 3) % 3, iz = t / 9;
        if (ix != 1 && iy != 1 && iz != 1)
          reinterpret_cast<float4*>(S + oVtx)[(ix >> 1) + 2 * (iy >> 1) + 4 * (iz >> 1)] = raw.xv;
      }
      vsq = raw.xv.y * raw.xv.y + raw.xv.z * raw.xv.z + raw.xv.w * raw.xv.w;
    }
    const float hT = raw.hT;
    const float4 box = raw.gb;
    if (c + stride < c_end) {  // issue the loads of the next cell (consumed next iteration)
      load_raw<GEO>(A, c + stride, idx_next, t, raw);
      if (c + 2 * stride < c_end && t < 27)
        idx_next = __ldg(A.cell_nodes + (int64_t)(c + 2 * stride) * 27 + t);
    }
    // non-negative floats order like their bit patterns: one warp-wide integer max (its result
    // and the reciprocals below are consumed in the pointwise phase: the dependent chain
    // REDUX -> sqrt -> rcp -> rcp is placed under the forward z stage, whose loads and FMAs
    // cover its latency; next to the gather it stalled every warp, 8 % of the samples)
    const unsigned vsq_max = __reduce_max_sync(0xffffffffu, __float_as_uint(vsq));
    const float ih = frcp(hT);  // (the chain is spread over the three regions between the warp
    const float nuih = A.nu * ih;  //  barriers, which the compiler does not schedule across)
    __syncwarp();
    // ---------------- forward x and y in registers: lane (f, qx) ----------------
    // x stage for this qx on the 9 (iz, iy) lines of field f, then the y stage for all four
    // qy -> sy[f][kind*3 + iz][qy*4 + qx]; kind 0 = B_x B_y, 1 = B_x D_y, 2 = D_x B_y
    // (cached form: 4 fields x 4 qx x 2 halves of qy -> all 32 lanes)
    const float sden = fmaf(nuih, ih, fmaf(sqrtf(__uint_as_float(vsq_max)), ih, A.ik));
    float srcp;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(srcp) : "f"(sden));
    constexpr int QYH = CACHED ? 2 : 4;  // qy per lane
    if (t < (CACHED ? 32 : 4 * NF)) {
      const int f = CACHED ? t >> 3 : t >> 2, qx = CACHED ? (t >> 1) & 3 : t & 3;
      const int qy0 = CACHED ? 2 * (t & 1) : 0;
      float u[28];
      if constexpr (CACHED) {   // 7 vector loads instead of 27 scalar ones
#pragma unroll
        for (int k = 0; k < 7; ++k) {
          const float4 q4 = reinterpret_cast<const float4*>(S + oU + f * L::US)[k];
          u[4 * k] = q4.x;
          u[4 * k + 1] = q4.y;
          u[4 * k + 2] = q4.z;
          u[4 * k + 3] = q4.w;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 27; ++k) u[k] = S[oU + f * L::US + k];
      }
      const float bx0 = cB[qx][0], bx1 = cB[qx][1], bx2 = cB[qx][2];
      const float dx0 = cD[qx][0], dx1 = cD[qx][1], dx2 = cD[qx][2];
      float aB[3][3], aD[3][3];
#pragma unroll
      for (int iz = 0; iz < 3; ++iz)
#pragma unroll
        for (int iy = 0; iy < 3; ++iy) {
          const float u0 = u[9 * iz + 3 * iy], u1 = u[9 * iz + 3 * iy + 1], u2 = u[9 * iz + 3 * iy + 2];
          aB[iz][iy] = fmaf(bx2, u2, fmaf(bx1, u1, bx0 * u0));
          aD[iz][iy] = fmaf(dx2, u2, fmaf(dx1, u1, dx0 * u0));
        }
      float* dst = S + oSY + L::sy(f) + qx;
#pragma unroll
      for (int qq = 0; qq < QYH; ++qq) {
        const int qy = qy0 + qq;
#pragma unroll
        for (int iz = 0; iz < 3; ++iz) {
          dst[(0 + iz) * 16 + 4 * qy] =
              fmaf(cB[qy][2], aB[iz][2], fmaf(cB[qy][1], aB[iz][1], cB[qy][0] * aB[iz][0]));
          dst[(3 + iz) * 16 + 4 * qy] =
              fmaf(cD[qy][2], aB[iz][2], fmaf(cD[qy][1], aB[iz][1], cD[qy][0] * aB[iz][0]));
          dst[(6 + iz) * 16 + 4 * qy] =
              fmaf(cB[qy][2], aD[iz][2], fmaf(cB[qy][1], aD[iz][1], cB[qy][0] * aD[iz][0]));
        }
      }
    }
    __syncwarp();
    // ---------------- forward z + pointwise: Gauss points q = t and t + 32 (same qy, qx) ----------------
    {
      float aT, dT;
      if (A.alpha_in) {
        aT = A.alpha_in[c];
        dT = A.delta_in[c];
      } else {  // stab at x (assembly.py:55-59, 169-178)
        const float rden = fmaf(fmaf(-sden, srcp, 1.0f), srcp, srcp);  // = frcp(sden)
        aT = A.alpha0 * rden;
        dT = A.delta0 * rden;
      }
      const int yx = t & 15, qz = t >> 4;  // second point: qz + 2
      float F[NF][4], G[NF][4];
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const float* src = S + oSY + L::sy(f) + yx;  // [(kind*3 + iz)*16]
        const float vv0 = src[0], vv1 = src[16], vv2 = src[32];
        const float vd0 = src[48], vd1 = src[64], vd2 = src[80];
        const float dv0 = src[96], dv1 = src[112], dv2 = src[128];
        {
          const float b0 = cB[qz][0], b1 = cB[qz][1], b2 = cB[qz][2];
          F[f][0] = b0 * vv0 + b1 * vv1 + b2 * vv2;
          F[f][1] = b0 * dv0 + b1 * dv1 + b2 * dv2;
          F[f][2] = b0 * vd0 + b1 * vd1 + b2 * vd2;
          F[f][3] = cD[qz][0] * vv0 + cD[qz][1] * vv1 + cD[qz][2] * vv2;
        }
        {
          const float b0 = cB[qz + 2][0], b1 = cB[qz + 2][1], b2 = cB[qz + 2][2];
          G[f][0] = b0 * vv0 + b1 * vv1 + b2 * vv2;
          G[f][1] = b0 * dv0 + b1 * dv1 + b2 * dv2;
          G[f][2] = b0 * vd0 + b1 * vd1 + b2 * vd2;
          G[f][3] = cD[qz + 2][0] * vv0 + cD[qz + 2][1] * vv1 + cD[qz + 2][2] * vv2;
        }
      }
      if constexpr (STAGED) {  // this cell's geometry block (staged one cell ahead)
        mbar_wait(bar, phase);
        phase ^= 1;
      }
      float PQa[4][4], PQb[4][4];
      if constexpr (MODE == MODE_OPERATOR)
        pi_fields(S + oU + L::FO * L::US,
                  CACHED ? reinterpret_cast<const float4*>(S + oVtx) : nullptr, yx & 3, yx >> 2,
                  qz, PQa, PQb);
      pointwise<MODE, GEO>(A, S, S + L::oCF, t, F, PQa, aT, dT, box, wq_a);
      pointwise<MODE, GEO>(A, S, S + L::oCF, t + 32, G, PQb, aT, dT, box, wq_b);
    }
    __syncwarp();
    if constexpr (STAGED) {
      if (c + stride < c_end) stage_geo(A, c + stride, t, S + L::oGQ, bar);
    }
    constexpr int kTZO = MODE == MODE_RHS ? kTZ2 : 2 * kTZS;   // row stride of the direct-test rows
    float lps = 0.f;
    if constexpr (MODE == MODE_RHS) {
    // ---------------- backward, RHS form: the direct test on all 32 lanes ----------------
    // The RHS form has no LPS part, so instead of lanes (comp, part, qz) with idle part-1 lanes
    // lane (comp, qz, h) contracts the two qy lines 2h, 2h+1 of plane qz for all three ix (x
    // stage), those qy (y stage), adds its share of the qz sum to all 27 outputs, and the eight
    // (qz, h) partials of a component are combined by a three-step shuffle reduce-scatter into
    // tz[comp][27]: rhs_next 0.613 -> 0.558 ms at config 3, 0.710 -> 0.632 ms at config 2.  (For
    // the operator form the same split, with the LPS test as a direct trilinear contraction,
    // executed 3 % fewer instructions but ran 3 % slower in the step -- DESIGN.md, dead ends.)
    {
      const int comp = t >> 3, g = t & 7, qz = g >> 1, hq = g & 1;
      const bool b2 = (g & 4) != 0, b1 = (g & 2) != 0, b0 = (g & 1) != 0;
      const int qoff = cfq(16 * qz) + 8 * hq;   // first Gauss point of this lane's two lines
      {
        const float* c0 = S + L::oCF + (CA + comp) * kCFS + qoff;
        const float* c1 = S + L::oCF + (CB + 3 * comp) * kCFS + qoff;
        const float* c2 = c1 + kCFS;
        const float* c3 = c1 + 2 * kCFS;
        float ua[3][3], ub[3][3];  // [iy][ix]
#pragma unroll
        for (int iy = 0; iy < 3; ++iy)
#pragma unroll
          for (int ix = 0; ix < 3; ++ix) ua[iy][ix] = ub[iy][ix] = 0.f;
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          const int qy = 2 * hq + qq;
          const float by[3] = {cB[qy][0], cB[qy][1], cB[qy][2]};
          const float dy[3] = {cD[qy][0], cD[qy][1], cD[qy][2]};
          const float4 l0 = *reinterpret_cast<const float4*>(c0 + 4 * qq);
          const float4 l1 = *reinterpret_cast<const float4*>(c1 + 4 * qq);
          const float4 l2 = *reinterpret_cast<const float4*>(c2 + 4 * qq);
          const float4 l3 = *reinterpret_cast<const float4*>(c3 + 4 * qq);
          const float L0[4] = {l0.x, l0.y, l0.z, l0.w}, L1[4] = {l1.x, l1.y, l1.z, l1.w};
          const float L2[4] = {l2.x, l2.y, l2.z, l2.w}, L3[4] = {l3.x, l3.y, l3.z, l3.w};
#pragma unroll
          for (int ix = 0; ix < 3; ++ix) {
            float t0 = cB[0][ix] * L0[0], t1 = cB[0][ix] * L2[0], t2 = cB[0][ix] * L3[0];
#pragma unroll
            for (int qx = 1; qx < 4; ++qx) t0 = fmaf(cB[qx][ix], L0[qx], t0);
#pragma unroll
            for (int qx = 0; qx < 4; ++qx) t0 = fmaf(cD[qx][ix], L1[qx], t0);
#pragma unroll
            for (int qx = 1; qx < 4; ++qx) {
              t1 = fmaf(cB[qx][ix], L2[qx], t1);
              t2 = fmaf(cB[qx][ix], L3[qx], t2);
            }
#pragma unroll
            for (int iy = 0; iy < 3; ++iy) {
              ua[iy][ix] = fmaf(by[iy], t0, fmaf(dy[iy], t1, ua[iy][ix]));
              ub[iy][ix] = fmaf(by[iy], t2, ub[iy][ix]);
            }
          }
        }
        const float bz[3] = {cB[qz][0], cB[qz][1], cB[qz][2]};
        const float dz[3] = {cD[qz][0], cD[qz][1], cD[qz][2]};
        float o[28];
#pragma unroll
        for (int iz = 0; iz < 3; ++iz)
#pragma unroll
          for (int iy = 0; iy < 3; ++iy)
#pragma unroll
            for (int ix = 0; ix < 3; ++ix)
              o[9 * iz + 3 * iy + ix] = fmaf(bz[iz], ua[iy][ix], dz[iz] * ub[iy][ix]);
        o[27] = 0.f;
        // reduce-scatter over the eight lanes of this component: lane bit 2 picks the half
        // [0,14) / [14,28), bit 1 the quarter [0,7) / [7,14) of it, bit 0 [0,4) / [4,8) of that
        float k14[14];
#pragma unroll
        for (int k = 0; k < 14; ++k) {
          const float send = b2 ? o[k] : o[14 + k];
          const float keep = b2 ? o[14 + k] : o[k];
          k14[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
        float k7[8];
#pragma unroll
        for (int k = 0; k < 7; ++k) {
          const float send = b1 ? k14[k] : k14[7 + k];
          const float keep = b1 ? k14[7 + k] : k14[k];
          k7[k] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
        }
        k7[7] = 0.f;
        float* out = S + oTZ + comp * kTZ2 + (b2 ? 14 : 0) + (b1 ? 7 : 0) + (b0 ? 4 : 0);
        const int nvalid = (b0 ? 3 : 4) - ((b2 && b1 && b0) ? 1 : 0);   // 27 = 4+3+4+3+4+3+4+2
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float send = b0 ? k7[k] : k7[4 + k];
          const float keep = b0 ? k7[4 + k] : k7[k];
          const float v = keep + __shfl_xor_sync(0xffffffffu, send, 1);
          if (k < nvalid) out[k] = v;
        }
      }
    }
    __syncwarp();
    } else {
    // ---------------- backward x, y, z in registers: lane (cp, qz), cp = (comp, part) ----------------
    // tz[cp][iz][iy][ix] = sum_q test(q; ix, iy, iz) . coefficients(cp, q).  Each of the 32
    // lanes contracts the four (qy) lines of one qz plane for all three ix (x stage), then qy
    // (y stage), then adds its plane's share of the qz sum; the four qz partials of a cp are
    // combined by a two-step shuffle reduce-scatter.  Part 0 is the direct test
    // (A N + B_k dN/dxi_k); part 1 the LPS test through PI^T: comp 0: -B_0k,
    // comps 1..3: -dg_i (J^-1 pi v)_k (elements.py:96-118, assembly.py:120-140).  (The RHS
    // form has no LPS part: its part-1 lanes compute unused values.)
    {
      const int cp = t >> 2, qz = t & 3;
      const int comp = cp >> 1, part = cp & 1;
      // part 0: A_c, B_c0..2; part 1: comp 0 -> B_00..02, comps 1..3 -> P_(c-1)0..2; part 1 has
      // no value test and enters with a minus sign
      // part 1 has no value test: its lanes read zeros, placed 8 banks away from the array the
      // part-0 lanes of the same quarter-warp read (no select per loaded value, no conflict)
      const float* c0 = part ? S + L::oZero + ((L::oCF + (CA + comp) * kCFS + 8 - L::oZero) & 31) +
                                   cfq(16 * qz)
                             : S + L::oCF + (CA + comp) * kCFS + cfq(16 * qz);
      const float* c1 = S + L::oCF +
                        (part == 0 || comp == 0 ? CB + 3 * comp : CP + 3 * (comp - 1)) * kCFS +
                        cfq(16 * qz);
      const float* c2 = c1 + kCFS;
      const float* c3 = c1 + 2 * kCFS;
      float ua[3][3], ub[3][3];  // [iy][ix]
#pragma unroll
      for (int iy = 0; iy < 3; ++iy)
#pragma unroll
        for (int ix = 0; ix < 3; ++ix) ua[iy][ix] = ub[iy][ix] = 0.f;
#pragma unroll
      for (int qy = 0; qy < 4; ++qy) {
        const float4 l0 = *reinterpret_cast<const float4*>(c0 + 4 * qy);
        const float4 l1 = *reinterpret_cast<const float4*>(c1 + 4 * qy);
        const float4 l2 = *reinterpret_cast<const float4*>(c2 + 4 * qy);
        const float4 l3 = *reinterpret_cast<const float4*>(c3 + 4 * qy);
        const float L0[4] = {l0.x, l0.y, l0.z, l0.w}, L1[4] = {l1.x, l1.y, l1.z, l1.w};
        const float L2[4] = {l2.x, l2.y, l2.z, l2.w}, L3[4] = {l3.x, l3.y, l3.z, l3.w};
#pragma unroll
        for (int ix = 0; ix < 3; ++ix) {
          float t0 = cB[0][ix] * L0[0], t1 = cB[0][ix] * L2[0], t2 = cB[0][ix] * L3[0];
#pragma unroll
          for (int qx = 1; qx < 4; ++qx) t0 = fmaf(cB[qx][ix], L0[qx], t0);
#pragma unroll
          for (int qx = 0; qx < 4; ++qx) t0 = fmaf(cD[qx][ix], L1[qx], t0);
#pragma unroll
          for (int qx = 1; qx < 4; ++qx) {
            t1 = fmaf(cB[qx][ix], L2[qx], t1);
            t2 = fmaf(cB[qx][ix], L3[qx], t2);
          }
#pragma unroll
          for (int iy = 0; iy < 3; ++iy) {
            ua[iy][ix] = fmaf(cB[qy][iy], t0, fmaf(cD[qy][iy], t1, ua[iy][ix]));
            ub[iy][ix] = fmaf(cB[qy][iy], t2, ub[iy][ix]);
          }
        }
      }
      // this plane's z contribution to all 27 outputs, index b = 9 iz + 3 iy + ix
      const float bz0 = cB[qz][0], bz1 = cB[qz][1], bz2 = cB[qz][2];
      const float dz0 = cD[qz][0], dz1 = cD[qz][1], dz2 = cD[qz][2];
      const float bz[3] = {bz0, bz1, bz2}, dz[3] = {dz0, dz1, dz2};
      float o[28];
#pragma unroll
      for (int iz = 0; iz < 3; ++iz)
#pragma unroll
        for (int iy = 0; iy < 3; ++iy)
#pragma unroll
          for (int ix = 0; ix < 3; ++ix)
            o[9 * iz + 3 * iy + ix] = fmaf(bz[iz], ua[iy][ix], dz[iz] * ub[iy][ix]);
      o[27] = 0.f;
      // reduce-scatter over the four qz lanes of this cp: lane bit 1 picks the half [0,14) or
      // [14,28), lane bit 0 the quarter [0,7) or [7,14) of that half
      const bool hi1 = (t & 2) != 0, hi0 = (t & 1) != 0;
      float k14[14];
#pragma unroll
      for (int k = 0; k < 14; ++k) {
        const float send = hi1 ? o[k] : o[14 + k];
        const float keep = hi1 ? o[14 + k] : o[k];
        k14[k] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
      }
      float* out = S + oTZ + cp * kTZS + (hi1 ? 14 : 0) + (hi0 ? 7 : 0);
      const int nvalid = (hi1 && hi0) ? 6 : 7;  // 27 = 7 + 7 + 7 + 6
#pragma unroll
      for (int k = 0; k < 7; ++k) {
        const float send = hi0 ? k14[k] : k14[7 + k];
        const float keep = hi0 ? k14[7 + k] : k14[k];
        const float v = keep + __shfl_xor_sync(0xffffffffu, send, 1);
        if (k < nvalid) out[k] = v;  // (part 1 enters with a minus sign: applied in the PI^T sums)
      }
    }
    __syncwarp();
    // ---------------- output: direct + PI^T * (LPS part), one float4 per node ----------------
    // PI[b][t] != 0 only for vertices t and the 8 nodes b with b_k in {t_k, 1} (weight 1/2 per
    // mid index): lane (comp, vertex) = (t >> 3, t & 7) forms one PI^T sum, and the node lanes
    // pick their four components up by shuffle
    if constexpr (MODE == MODE_OPERATOR) {
      const int comp = t >> 3, v = t & 7;
      const int it0 = (v & 1) ? 2 : 0, it1 = (v & 2) ? 2 : 0, it2 = (v & 4) ? 2 : 0;
      const float* gp = S + oTZ + (comp * 2 + 1) * kTZS;
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int b0 = (m & 1) ? 1 : it0, b1 = (m & 2) ? 1 : it1, b2 = (m & 4) ? 1 : it2;
        const float wgt = ((m & 1) ? 0.5f : 1.f) * ((m & 2) ? 0.5f : 1.f) * ((m & 4) ? 0.5f : 1.f);
        lps = fmaf(-wgt, gp[b0 + 3 * b1 + 9 * b2], lps);
      }
    }
    }
    {
      const int it0 = t % 3, it1 = (t / 3) % 3, it2 = t / 9;
      const bool vtx = MODE == MODE_OPERATOR && t < 27 && it0 != 1 && it1 != 1 && it2 != 1;
      const int vid = (it0 >> 1) + 2 * (it1 >> 1) + 4 * (it2 >> 1);
      float e[4];
#pragma unroll
      for (int comp = 0; comp < 4; ++comp) {
        const float l = __shfl_sync(0xffffffffu, lps, comp * 8 + (vid & 7));
        e[comp] = t < 27 ? S[oTZ + comp * kTZO + t] + (vtx ? l : 0.f) : 0.f;
      }
      if (t < 27) A.elem[(int64_t)c * 27 + t] = make_float4(e[0], e[1], e[2], e[3]);
    }
    __syncwarp();
  }
}

// out[n] = sign * sum_{incident (c,a), ascending c} elem[c][a] (+ b[n]); masked rows -> 0
__global__ void __launch_bounds__(256) node_sum_kernel(
    int n_nodes, const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
    const float4* __restrict__ elem, const float4* __restrict__ b, float sign,
    const uint8_t* __restrict__ mask, float4* __restrict__ out, const int32_t* __restrict__ order,
    const int32_t* __restrict__ vptr, const int32_t* __restrict__ vidx) {
  if (vptr) idx = vidx;   // rows in visiting order: the bounds load next to the node id
  for (int pos = blockIdx.x * blockDim.x + threadIdx.x; pos < n_nodes;
       pos += gridDim.x * blockDim.x) {
    const int n = order ? __ldg(order + pos) : pos;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const int s = vptr ? __ldg(vptr + pos) : __ldg(ptr + n);
    const int e = vptr ? __ldg(vptr + pos + 1) : __ldg(ptr + n + 1);
    // the first 8 incident element vectors are loaded before any is summed (all in flight at
    // once); the sum stays in ascending cell order
    int ent[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) ent[k] = s + k < e ? __ldg(idx + s + k) : -1;
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      v[k] = ent[k] >= 0 ? __ldg(elem + ent[k]) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (ent[k] >= 0) {
        acc.x += v[k].x;
        acc.y += v[k].y;
        acc.z += v[k].z;
        acc.w += v[k].w;
      }
    }
    for (int i = s + 8; i < e; ++i) {
      const float4 w = __ldg(elem + __ldg(idx + i));
      acc.x += w.x;
      acc.y += w.y;
      acc.z += w.z;
      acc.w += w.w;
    }
    float4 r;
    if (b) {
      const float4 bb = __ldg(b + n);
      r = make_float4(bb.x - acc.x, bb.y - acc.y, bb.z - acc.z, bb.w - acc.w);
    } else {
      r = make_float4(sign * acc.x, sign * acc.y, sign * acc.z, sign * acc.w);
    }
    if (mask) {
      const uint8_t m = mask[n];
      if (m & 1) r.x = 0.f;
      if (m & 2) r.y = 0.f;
      if (m & 4) r.z = 0.f;
      if (m & 8) r.w = 0.f;
    }
    out[n] = r;
  }
}

__global__ void __launch_bounds__(256) stab_kernel(int n_cells, const int32_t* __restrict__ cn,
                                                   const float4* __restrict__ x,
                                                   const float* __restrict__ h_T, float nu, float k,
                                                   float alpha0, float delta0,
                                                   float* __restrict__ aT, float* __restrict__ dT) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n_cells; c += gridDim.x * blockDim.x) {
    float m = 0.f;
    for (int a = 0; a < 27; ++a) {
      const float4 v = __ldg(x + __ldg(cn + (int64_t)c * 27 + a));
      m = fmaxf(m, sqrtf(v.y * v.y + v.z * v.z + v.w * v.w));
    }
    const float h = h_T[c];
    const float ih = frcp(h);
    const float rden = frcp(fmaf(nu * ih, ih, fmaf(m, ih, 1.0f / k)));
    aT[c] = alpha0 * rden;
    dT[c] = delta0 * rden;
  }
}


static int32_t check_level(const dnnmg_level_t* lv, const char* who) {
  DNNMG_REQUIRE(lv && lv->cell_nodes && lv->coords && lv->h_T && lv->node_cell_ptr &&
                    lv->node_cell_idx,
                DNNMG_ERR_ARG, "%s: incomplete level tables", who);
  return DNNMG_OK;
}

int32_t launch_k2tc_elements(const dnnmg_level_t*, const float*, const float*, const float*,
                             const dnnmg_phys_t*, int, float*, cudaStream_t);

template <int MODE, int GEO>
static void launch_element_kernel(const ResidualArgs& A, cudaStream_t s) {
  constexpr int kWarpsPerBlock = k2_warps_per_block(MODE);
  constexpr size_t smem = sizeof(float) * KLay<GEO>::kFloats * kWarpsPerBlock;
  static uint64_t configured = 0;
  if (first_use_on_device(configured))
    cudaFuncSetAttribute(element_kernel<MODE, GEO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  int blocks = (A.n_cells + kWarpsPerBlock - 1) / kWarpsPerBlock;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, element_kernel<MODE, GEO>,
                                                32 * kWarpsPerBlock, smem);
  const int cap = kSMs * (per_sm > 0 ? per_sm : 1);
  if (blocks > cap) blocks = cap;
  element_kernel<MODE, GEO><<<blocks, 32 * kWarpsPerBlock, smem, s>>>(A);
}

static int32_t launch_elements(const dnnmg_level_t* lv, const float* x, const float* aT,
                               const float* dT, const dnnmg_phys_t* ph, int mode, float* elem,
                               cudaStream_t s) {
  // the tensor-core element kernel when its tables are present (residual_tc.cu)
  if (lv->tc_const && lv->tc_geo && !getenv("DNNMG_K2_SIMT"))
    return launch_k2tc_elements(lv, x, aT, dT, ph, mode == MODE_RHS ? 1 : 0, elem, s);
  ResidualArgs A;
  A.n_cells = lv->n_cells;
  A.cell_nodes = lv->cell_nodes;
  A.coords = lv->coords;
  A.x = reinterpret_cast<const float4*>(x);
  A.h_T = lv->h_T;
  A.alpha_in = aT;
  A.delta_in = dT;
  A.nu = ph->nu;
  A.k = ph->k;
  A.ik = 1.0f / ph->k;
  A.alpha0 = ph->alpha0;
  A.delta0 = ph->delta0;
  A.convection = ph->convection;
  A.mode = mode;
  A.elem = reinterpret_cast<float4*>(elem);
  A.geo_q = lv->geo_q;
  A.geo_box = reinterpret_cast<const float4*>(lv->geo_box);
  if (lv->n_cells == 0) return DNNMG_OK;
  // axis-aligned level: the box form; else the per-point cache when present
  static const bool no_box = getenv("DNNMG_K2_NO_BOX") != nullptr;
  if (no_box) A.geo_box = nullptr;
  const int geo = A.geo_box ? GEO_BOX : lv->geo_q ? GEO_CACHED : GEO_NONE;
#define DNNMG_K2_LAUNCH(M, G) \
  launch_element_kernel<M, G>(A, s)
  if (mode == MODE_OPERATOR) {
    if (geo == GEO_BOX) DNNMG_K2_LAUNCH(MODE_OPERATOR, GEO_BOX);
    else if (geo == GEO_CACHED) DNNMG_K2_LAUNCH(MODE_OPERATOR, GEO_CACHED);
    else DNNMG_K2_LAUNCH(MODE_OPERATOR, GEO_NONE);
  } else {
    if (geo == GEO_BOX) DNNMG_K2_LAUNCH(MODE_RHS, GEO_BOX);
    else if (geo == GEO_CACHED) DNNMG_K2_LAUNCH(MODE_RHS, GEO_CACHED);
    else DNNMG_K2_LAUNCH(MODE_RHS, GEO_NONE);
  }
#undef DNNMG_K2_LAUNCH
  DNNMG_CHECK_LAUNCH("element_kernel");
  return DNNMG_OK;
}

// ---- per-mesh geometry cache: J^-1 and w at every (cell, Gauss point) -----------------
// Evaluated once per level in fp64 from the 27 cell nodes (isoparametric Q2 map,
// assembly.py:77-90) and stored in fp32 as [cell][10][64]: (J^-1)[k][j] row-major, then
// w = w_hat(q) det J.  The reference keeps the equivalent G tables (GeometryCache).
__constant__ double dB[4][3] = {{tab::phi(0, tab::xg[0]), tab::phi(1, tab::xg[0]), tab::phi(2, tab::xg[0])},
                                {tab::phi(0, tab::xg[1]), tab::phi(1, tab::xg[1]), tab::phi(2, tab::xg[1])},
                                {tab::phi(0, tab::xg[2]), tab::phi(1, tab::xg[2]), tab::phi(2, tab::xg[2])},
                                {tab::phi(0, tab::xg[3]), tab::phi(1, tab::xg[3]), tab::phi(2, tab::xg[3])}};
__constant__ double dD[4][3] = {{tab::dphi(0, tab::xg[0]), tab::dphi(1, tab::xg[0]), tab::dphi(2, tab::xg[0])},
                                {tab::dphi(0, tab::xg[1]), tab::dphi(1, tab::xg[1]), tab::dphi(2, tab::xg[1])},
                                {tab::dphi(0, tab::xg[2]), tab::dphi(1, tab::xg[2]), tab::dphi(2, tab::xg[2])},
                                {tab::dphi(0, tab::xg[3]), tab::dphi(1, tab::xg[3]), tab::dphi(2, tab::xg[3])}};
__constant__ double dW[4] = {tab::wg[0], tab::wg[1], tab::wg[2], tab::wg[3]};

__global__ void __launch_bounds__(128) geometry_kernel(int n_cells, const int32_t* __restrict__ cn,
                                                       const double* __restrict__ coords,
                                                       float* __restrict__ geo) {
  __shared__ double X[4][27][3];
  const int w = threadIdx.x >> 5, t = threadIdx.x & 31;
  for (int c = blockIdx.x * 4 + w; c < n_cells; c += gridDim.x * 4) {
    if (t < 27) {
      const int n = __ldg(cn + (int64_t)c * 27 + t), n0 = __ldg(cn + (int64_t)c * 27);
#pragma unroll
      for (int i = 0; i < 3; ++i) X[w][t][i] = __ldg(coords + 3 * (int64_t)n + i) - __ldg(coords + 3 * (int64_t)n0 + i);
    }
    __syncwarp();
#pragma unroll 1
    for (int k = 0; k < 2; ++k) {
      const int q = t + 32 * k, qx = q & 3, qy = (q >> 2) & 3, qz = q >> 4;
      double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};  // J[i][m] = dX_i / dxi_m
      for (int a = 0; a < 27; ++a) {
        const int ax = a % 3, ay = (a / 3) % 3, az = a / 9;
        const double g0 = dD[qx][ax] * dB[qy][ay] * dB[qz][az];
        const double g1 = dB[qx][ax] * dD[qy][ay] * dB[qz][az];
        const double g2 = dB[qx][ax] * dB[qy][ay] * dD[qz][az];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const double xi = X[w][a][i];
          J[i][0] = fma(xi, g0, J[i][0]);
          J[i][1] = fma(xi, g1, J[i][1]);
          J[i][2] = fma(xi, g2, J[i][2]);
        }
      }
      const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
      const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
      const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
      const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
      const double id = 1.0 / det;
      double Ji[3][3];
      Ji[0][0] = c00 * id;
      Ji[1][0] = c01 * id;
      Ji[2][0] = c02 * id;
      Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
      Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
      Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
      Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
      Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
      Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
      float* gq = geo + (int64_t)c * 640 + q;
#pragma unroll
      for (int kk = 0; kk < 3; ++kk)
#pragma unroll
        for (int j = 0; j < 3; ++j) gq[(3 * kk + j) * 64] = (float)Ji[kk][j];
      gq[9 * 64] = (float)(dW[qx] * dW[qy] * dW[qz] * det);
    }
    __syncwarp();
  }
}

int32_t launch_level_geometry(const dnnmg_level_t* lv, float* geo, cudaStream_t s) {
  DNNMG_REQUIRE(lv && lv->cell_nodes && lv->coords && geo, DNNMG_ERR_ARG,
                "level_geometry: null argument");
  DNNMG_REQUIRE(((uintptr_t)geo & 15) == 0, DNNMG_ERR_ARG, "level_geometry: unaligned output");
  if (lv->n_cells == 0) return DNNMG_OK;
  geometry_kernel<<<grid_for((lv->n_cells + 3) / 4, 1, 16), 128, 0, s>>>(lv->n_cells, lv->cell_nodes,
                                                                          lv->coords, geo);
  DNNMG_CHECK_LAUNCH("geometry_kernel");
  return DNNMG_OK;
}

// ---- axis-aligned levels: one record per cell instead of the per-point cache --------------
// box[c] = (1/hx, 1/hy, 1/hz, det J = hx hy hz) in fp64 -> fp32, hk = extent of the cell along
// axis k (signed).  n_bad counts the cells whose 27 nodes are not the tri-quadratic lattice of
// an axis-aligned box (|X_a - X_0 - (ix hx, iy hy, iz hz)/2| > 1e-12 |h|): the caller uses the
// record only when it is 0, since then J is diagonal and constant over every cell and the
// element kernel's box form equals the general one up to fp32 rounding of w.
__global__ void __launch_bounds__(128) geometry_box_kernel(int n_cells, const int32_t* __restrict__ cn,
                                                           const double* __restrict__ coords,
                                                           float4* __restrict__ box,
                                                           int32_t* __restrict__ n_bad) {
  const int w = threadIdx.x >> 5, t = threadIdx.x & 31;
  for (int c = blockIdx.x * 4 + w; c < n_cells; c += gridDim.x * 4) {
    const int32_t* row = cn + (int64_t)c * 27;
    const int n0 = __ldg(row), nx = __ldg(row + 2), ny = __ldg(row + 6), nz = __ldg(row + 18);
    double X0[3], h[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) X0[i] = __ldg(coords + 3 * (int64_t)n0 + i);
    h[0] = __ldg(coords + 3 * (int64_t)nx + 0) - X0[0];
    h[1] = __ldg(coords + 3 * (int64_t)ny + 1) - X0[1];
    h[2] = __ldg(coords + 3 * (int64_t)nz + 2) - X0[2];
    bool bad = false;
    if (t < 27) {
      const int n = __ldg(row + t);
      const int l[3] = {t % 3, (t / 3) % 3, t / 9};
      const double tol = 1e-12 * (fabs(h[0]) + fabs(h[1]) + fabs(h[2]));
#pragma unroll
      for (int i = 0; i < 3; ++i)
        bad |= !(fabs(__ldg(coords + 3 * (int64_t)n + i) - X0[i] - 0.5 * l[i] * h[i]) <= tol);
    }
    const double det = h[0] * h[1] * h[2];
    bad |= !(det != 0.0);
    const unsigned any = __ballot_sync(0xffffffffu, bad);
    if (t == 0) {
      box[c] = make_float4((float)(1.0 / h[0]), (float)(1.0 / h[1]), (float)(1.0 / h[2]), (float)det);
      if (any && n_bad) atomicAdd(n_bad, 1);
    }
  }
}

int32_t launch_level_geometry_box(const dnnmg_level_t* lv, float* box, int32_t* n_bad,
                                  cudaStream_t s) {
  DNNMG_REQUIRE(lv && lv->cell_nodes && lv->coords && box, DNNMG_ERR_ARG,
                "level_geometry_box: null argument");
  DNNMG_REQUIRE(((uintptr_t)box & 15) == 0, DNNMG_ERR_ARG, "level_geometry_box: unaligned output");
  if (n_bad) cudaMemsetAsync(n_bad, 0, sizeof(int32_t), s);
  if (lv->n_cells == 0) return DNNMG_OK;
  geometry_box_kernel<<<grid_for((lv->n_cells + 3) / 4, 1, 16), 128, 0, s>>>(
      lv->n_cells, lv->cell_nodes, lv->coords, reinterpret_cast<float4*>(box), n_bad);
  DNNMG_CHECK_LAUNCH("geometry_box_kernel");
  return DNNMG_OK;
}

int32_t launch_node_sum(int n_nodes, const int32_t* ptr, const int32_t* idx, const float* elem,
                        float* out, cudaStream_t s) {
  if (n_nodes == 0) return DNNMG_OK;
  node_sum_kernel<<<grid_for(n_nodes, 256), 256, 0, s>>>(
      n_nodes, ptr, idx, reinterpret_cast<const float4*>(elem), nullptr, 1.0f, nullptr,
      reinterpret_cast<float4*>(out), nullptr, nullptr, nullptr);
  DNNMG_CHECK_LAUNCH("node_sum_kernel");
  return DNNMG_OK;
}

int32_t launch_stab(const dnnmg_level_t* lv, const float* x, const dnnmg_phys_t* ph, float* aT,
                    float* dT, cudaStream_t s) {
  int32_t st = check_level(lv, "stab");
  if (st) return st;
  DNNMG_REQUIRE(x && ph && aT && dT, DNNMG_ERR_ARG, "stab: null argument");
  if (lv->n_cells == 0) return DNNMG_OK;
  stab_kernel<<<grid_for(lv->n_cells, 256), 256, 0, s>>>(
      lv->n_cells, lv->cell_nodes, reinterpret_cast<const float4*>(x), lv->h_T, ph->nu, ph->k,
      ph->alpha0, ph->delta0, aT, dT);
  DNNMG_CHECK_LAUNCH("stab_kernel");
  return DNNMG_OK;
}

int32_t launch_residual(const dnnmg_level_t* lv, const float* x, const float* b_prev,
                        const float* aT, const float* dT, const dnnmg_phys_t* ph, float* elem,
                        float* r, int apply_mask, int mode_sign, cudaStream_t s,
                        cudaEvent_t b_ready) {
  // mode_sign: +1 residual (b - A), 0 operator (A), 2 rhs_next
  int32_t st = check_level(lv, "residual");
  if (st) return st;
  DNNMG_REQUIRE(x && ph && elem && r, DNNMG_ERR_ARG, "residual: null argument");
  DNNMG_REQUIRE((aT == nullptr) == (dT == nullptr), DNNMG_ERR_ARG,
                "residual: alpha_T and delta_T must both be given or both be NULL");
  const int mode = mode_sign == 2 ? MODE_RHS : MODE_OPERATOR;
  st = launch_elements(lv, x, aT, dT, ph, mode, elem, s);
  if (st) return st;
  const float4* b = nullptr;
  if (mode_sign == 1) {
    DNNMG_REQUIRE(b_prev, DNNMG_ERR_ARG, "residual: b_prev is NULL");
    b = reinterpret_cast<const float4*>(b_prev);
  }
  if (lv->n_nodes == 0) return DNNMG_OK;
  if (b_ready) {   // b_prev may still be arriving: its first reader is the node sum
    DNNMG_REQUIRE(cudaStreamWaitEvent(s, b_ready, 0) == cudaSuccess, DNNMG_ERR_CUDA,
                  "residual: cudaStreamWaitEvent(b_ready) failed");
  }
  // 8 blocks per SM: all resident at once (0.0805 -> 0.078 ms at config 3 against 64 waves)
  node_sum_kernel<<<grid_for(lv->n_nodes, 256, 8), 256, 0, s>>>(
      lv->n_nodes, lv->node_cell_ptr, lv->node_cell_idx, reinterpret_cast<const float4*>(elem), b,
      1.0f, (apply_mask && lv->dof_mask) ? lv->dof_mask : nullptr, reinterpret_cast<float4*>(r),
      lv->node_order, lv->node_order ? lv->visit_ptr : nullptr, lv->visit_idx);
  DNNMG_CHECK_LAUNCH("node_sum_kernel");
  return DNNMG_OK;
}

}  // namespace dnnmg
