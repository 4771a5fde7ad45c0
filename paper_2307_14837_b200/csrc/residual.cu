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
#include "common.cuh"

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
__constant__ float cW[4] = {float(tab::wg[0]), float(tab::wg[1]), float(tab::wg[2]),
                            float(tab::wg[3])};
#undef QB
#undef QD

// ---- per-cell shared-memory layout (floats) --------------------------------
constexpr int kNF = 11;               // fields: X^x,X^y,X^z, p, vx,vy,vz, pi p, pi vx,vy,vz
constexpr int kGroup = 64;            // threads per cell
constexpr int oU = 0;                 // u[f][27]
constexpr int oSX = oU + kNF * 27;    // sx[f][2][9][4]   | backward: tx[4][2][3][16][3]
constexpr int oSY = oSX + kNF * 72;   // sy[f][3][3][16]  |           ty[4][2][2][4][3][3]
constexpr int oFQ = oSY + kNF * 144;  // fq[f][4][64]
constexpr int oCF = oFQ + kNF * 256;  // cf[4][7][64]
constexpr int oTZ = oCF + 4 * 7 * 64; // tz[4][2][27]
constexpr int oST = oTZ + 4 * 2 * 27; // alpha, delta, vmax scratch
constexpr int kCellFloats = oST + 4;
static_assert(4 * 2 * 3 * 48 <= kNF * 72 + kNF * 144, "backward scratch must fit");
constexpr int oTX = oSX;
constexpr int oTY = oSX + 4 * 2 * 3 * 48;

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
  int convection;
  int mode;
  float4* elem;
};

// PI[b][v] for local node b (lattice ib) and vertex lattice iv in {0,2}^3 (elements.py:96-118)
__device__ __forceinline__ float pi_weight(int b, int v) {
  float w = 1.f;
  int bb = b, vv = v;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int ib = bb % 3, iv = vv % 3;
    bb /= 3; vv /= 3;
    w *= (ib == 1) ? 0.5f : (ib == iv ? 1.f : 0.f);
  }
  return w;
}

template <int CPB>
__global__ void __launch_bounds__(64 * CPB) element_kernel(ResidualArgs A) {
  extern __shared__ float smem[];
  const int grp = threadIdx.x / kGroup;
  const int t = threadIdx.x % kGroup;
  float* S = smem + grp * kCellFloats;
  const int vertex_local[8] = {0, 2, 6, 8, 18, 20, 24, 26};

  for (int base = blockIdx.x * CPB; base < A.n_cells; base += gridDim.x * CPB) {
    const int c = base + grp;
    const bool live = c < A.n_cells;
    // ---------------- gather ----------------
    float vmag = 0.f;
    if (t < 27) {
      if (live) {
        const int node = __ldg(A.cell_nodes + (int64_t)c * 27 + t);
        const int n0 = __ldg(A.cell_nodes + (int64_t)c * 27);
        const double* X = A.coords + 3 * (int64_t)node;
        const double* X0 = A.coords + 3 * (int64_t)n0;
        S[oU + 0 * 27 + t] = float(X[0] - X0[0]);
        S[oU + 1 * 27 + t] = float(X[1] - X0[1]);
        S[oU + 2 * 27 + t] = float(X[2] - X0[2]);
        const float4 xv = __ldg(A.x + node);
        S[oU + 3 * 27 + t] = xv.x;
        S[oU + 4 * 27 + t] = xv.y;
        S[oU + 5 * 27 + t] = xv.z;
        S[oU + 6 * 27 + t] = xv.w;
        vmag = sqrtf(xv.y * xv.y + xv.z * xv.z + xv.w * xv.w);
      } else {  // padding cell: unit reference cube, zero state (never written out)
        S[oU + 0 * 27 + t] = 0.5f * (t % 3);
        S[oU + 1 * 27 + t] = 0.5f * ((t / 3) % 3);
        S[oU + 2 * 27 + t] = 0.5f * (t / 9);
#pragma unroll
        for (int f = 3; f < 7; ++f) S[oU + f * 27 + t] = 0.f;
      }
    }
    if (t < 32) {  // vmax over the 27 nodes (assembly.py:169-172): first warp of the group
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) vmag = fmaxf(vmag, __shfl_xor_sync(0xffffffffu, vmag, off));
      if (t == 0) S[oST + 2] = vmag;
    }
    __syncthreads();
    if (t < 27) {
      // pi-projected nodal values (Q1 interpolant of p and v on the Q2 nodes)
      float pp = 0.f, p0 = 0.f, p1 = 0.f, p2 = 0.f;
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int av = vertex_local[v];
        const float w = pi_weight(t, av);
        pp = fmaf(w, S[oU + 3 * 27 + av], pp);
        p0 = fmaf(w, S[oU + 4 * 27 + av], p0);
        p1 = fmaf(w, S[oU + 5 * 27 + av], p1);
        p2 = fmaf(w, S[oU + 6 * 27 + av], p2);
      }
      S[oU + 7 * 27 + t] = pp;
      S[oU + 8 * 27 + t] = p0;
      S[oU + 9 * 27 + t] = p1;
      S[oU + 10 * 27 + t] = p2;
    }
    if (t == 32) {
      float aT = 0.f, dT = 0.f;
      if (live) {
        if (A.alpha_in) {
          aT = A.alpha_in[c];
          dT = A.delta_in[c];
        } else {
          const float h = A.h_T[c];
          const float den = A.nu / (h * h) + S[oST + 2] / h + 1.0f / A.k;
          aT = A.alpha0 / den;
          dT = A.delta0 / den;
        }
      }
      S[oST + 0] = aT;
      S[oST + 1] = dT;
    }
    __syncthreads();
    // ---------------- forward stage x: sx[f][kind][izy][qx] ----------------
    for (int l = t; l < kNF * 9; l += kGroup) {
      const int f = l / 9, izy = l % 9;
      const float* u = S + oU + f * 27 + izy * 3;
      const float u0 = u[0], u1 = u[1], u2 = u[2];
      float* o = S + oSX + f * 72 + izy * 4;
#pragma unroll
      for (int qx = 0; qx < 4; ++qx) {
        o[qx] = cB[qx][0] * u0 + cB[qx][1] * u1 + cB[qx][2] * u2;
        o[36 + qx] = cD[qx][0] * u0 + cD[qx][1] * u1 + cD[qx][2] * u2;
      }
    }
    __syncthreads();
    // ---------------- forward stage y: sy[f][{vv,vd,dv}][iz][qy*4+qx] ----------------
    for (int l = t; l < kNF * 12; l += kGroup) {
      const int f = l / 12, r = l % 12, iz = r / 4, qx = r % 4;
      const float* s0 = S + oSX + f * 72 + iz * 12 + qx;  // [iy] stride 4
      const float a0 = s0[0], a1 = s0[4], a2 = s0[8];
      const float b0 = s0[36], b1 = s0[40], b2 = s0[44];
      float* o = S + oSY + f * 144 + iz * 16 + qx;
#pragma unroll
      for (int qy = 0; qy < 4; ++qy) {
        o[qy * 4] = cB[qy][0] * a0 + cB[qy][1] * a1 + cB[qy][2] * a2;
        o[48 + qy * 4] = cD[qy][0] * a0 + cD[qy][1] * a1 + cD[qy][2] * a2;
        o[96 + qy * 4] = cB[qy][0] * b0 + cB[qy][1] * b1 + cB[qy][2] * b2;
      }
    }
    __syncthreads();
    // ---------------- forward stage z: fq[f][{val,dx,dy,dz}][q] ----------------
    for (int l = t; l < kNF * 16; l += kGroup) {
      const int f = l / 16, yx = l % 16;
      const float* s = S + oSY + f * 144 + yx;  // [kind*48 + iz*16]
      const float vv0 = s[0], vv1 = s[16], vv2 = s[32];
      const float vd0 = s[48], vd1 = s[64], vd2 = s[80];
      const float dv0 = s[96], dv1 = s[112], dv2 = s[128];
      float* o = S + oFQ + f * 256 + yx;
#pragma unroll
      for (int qz = 0; qz < 4; ++qz) {
        const float b0 = cB[qz][0], b1 = cB[qz][1], b2 = cB[qz][2];
        o[qz * 16] = b0 * vv0 + b1 * vv1 + b2 * vv2;
        o[64 + qz * 16] = b0 * dv0 + b1 * dv1 + b2 * dv2;
        o[128 + qz * 16] = b0 * vd0 + b1 * vd1 + b2 * vd2;
        o[192 + qz * 16] = cD[qz][0] * vv0 + cD[qz][1] * vv1 + cD[qz][2] * vv2;
      }
    }
    __syncthreads();
    // ---------------- pointwise (thread = Gauss point q) ----------------
    {
      const int q = t;
      const float* F = S + oFQ + q;
#define FQ(f, kind) F[(f) * 256 + (kind) * 64]
      float J[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) J[i][j] = FQ(i, 1 + j);
      const float c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
      const float c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
      const float c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
      const float det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
      const float id = 1.0f / det;
      // Ji[k][j] = (J^-1)[k][j]: reference k -> physical j
      float Ji[3][3];
      Ji[0][0] = c00 * id;
      Ji[1][0] = c01 * id;
      Ji[2][0] = c02 * id;
      Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
      Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
      Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
      Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
      Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
      Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
      const float w = cW[q & 3] * cW[(q >> 2) & 3] * cW[q >> 4] * det;
      const float aT = S[oST + 0], dT = S[oST + 1];
      float v[3], gv[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        v[i] = FQ(4 + i, 0);
#pragma unroll
        for (int j = 0; j < 3; ++j)
          gv[i][j] = FQ(4 + i, 1) * Ji[0][j] + FQ(4 + i, 2) * Ji[1][j] + FQ(4 + i, 3) * Ji[2][j];
      }
      float conv[3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
        conv[i] = A.convection ? v[0] * gv[i][0] + v[1] * gv[i][1] + v[2] * gv[i][2] : 0.f;
      float* C = S + oCF + q;  // cf[comp][arr][q]
#define CF(comp, arr) C[((comp) * 7 + (arr)) * 64]
      if (A.mode == MODE_OPERATOR) {
        const float p = FQ(3, 0);
        float gp[3], gpp[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          gp[j] = FQ(3, 1) * Ji[0][j] + FQ(3, 2) * Ji[1][j] + FQ(3, 3) * Ji[2][j];
          gpp[j] = FQ(7, 1) * Ji[0][j] + FQ(7, 2) * Ji[1][j] + FQ(7, 3) * Ji[2][j];
        }
        const bool use_d = A.convection && dT != 0.f;
        float g[3] = {0.f, 0.f, 0.f}, pvr[3] = {0.f, 0.f, 0.f};
        if (use_d) {
          float pv[3], gpv[3][3];
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            pv[i] = FQ(8 + i, 0);
#pragma unroll
            for (int j = 0; j < 3; ++j)
              gpv[i][j] = FQ(8 + i, 1) * Ji[0][j] + FQ(8 + i, 2) * Ji[1][j] + FQ(8 + i, 3) * Ji[2][j];
          }
#pragma unroll
          for (int i = 0; i < 3; ++i)
            g[i] = conv[i] - (pv[0] * gpv[i][0] + pv[1] * gpv[i][1] + pv[2] * gpv[i][2]);
#pragma unroll
          for (int kk = 0; kk < 3; ++kk)
            pvr[kk] = Ji[kk][0] * pv[0] + Ji[kk][1] * pv[1] + Ji[kk][2] * pv[2];
        }
        const float div = gv[0][0] + gv[1][1] + gv[2][2];
        // continuity: value test w*div; gradient test alpha*w*(gp - gpp) through (G - Gpi)
        float E[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) E[j] = aT * w * (gp[j] - gpp[j]);
        CF(0, 0) = w * div;
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
          const float b = Ji[kk][0] * E[0] + Ji[kk][1] * E[1] + Ji[kk][2] * E[2];
          CF(0, 1 + kk) = b;
          CF(0, 4 + kk) = -b;
        }
        const float hn = 0.5f * A.nu * w;
        const float ik = 1.0f / A.k;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          CF(1 + i, 0) = w * (v[i] * ik + 0.5f * conv[i]);
          const float dg = dT * w * g[i];
          float Fi[3];
#pragma unroll
          for (int j = 0; j < 3; ++j) Fi[j] = hn * gv[i][j] + dg * v[j] - (i == j ? w * p : 0.f);
#pragma unroll
          for (int kk = 0; kk < 3; ++kk) {
            CF(1 + i, 1 + kk) = Ji[kk][0] * Fi[0] + Ji[kk][1] * Fi[1] + Ji[kk][2] * Fi[2];
            CF(1 + i, 4 + kk) = -dg * pvr[kk];
          }
        }
      } else {  // MODE_RHS (assembly.py:242-259, f = None)
        const float hn = -0.5f * A.nu * w;
        const float ik = 1.0f / A.k;
#pragma unroll
        for (int a = 0; a < 7; ++a) CF(0, a) = 0.f;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          CF(1 + i, 0) = w * (v[i] * ik - 0.5f * conv[i]);
#pragma unroll
          for (int kk = 0; kk < 3; ++kk) {
            CF(1 + i, 1 + kk) = hn * (Ji[kk][0] * gv[i][0] + Ji[kk][1] * gv[i][1] + Ji[kk][2] * gv[i][2]);
            CF(1 + i, 4 + kk) = 0.f;
          }
        }
      }
#undef CF
#undef FQ
    }
    __syncthreads();
    // ---------------- backward stage x (contract qx) ----------------
    // line (comp, part, qz, qy) -> tx[comp][part][{Tv,T1,T2}][qz*4+qy][ix]
    for (int l = t; l < 4 * 2 * 16; l += kGroup) {
      const int comp = l / 32, part = (l / 16) % 2, zy = l % 16;
      const float* cf = S + oCF + comp * 7 * 64 + zy * 4;
      float Av[4], B0[4], B1[4], B2[4];
#pragma unroll
      for (int qx = 0; qx < 4; ++qx) {
        if (part == 0) {
          Av[qx] = cf[qx];
          B0[qx] = cf[64 + qx];
          B1[qx] = cf[128 + qx];
          B2[qx] = cf[192 + qx];
        } else {
          Av[qx] = 0.f;
          B0[qx] = cf[256 + qx];
          B1[qx] = cf[320 + qx];
          B2[qx] = cf[384 + qx];
        }
      }
      float* o = S + oTX + ((comp * 2 + part) * 3) * 48 + zy * 3;
#pragma unroll
      for (int ix = 0; ix < 3; ++ix) {
        float tv = 0.f, t1 = 0.f, t2 = 0.f;
#pragma unroll
        for (int qx = 0; qx < 4; ++qx) {
          tv += cB[qx][ix] * Av[qx] + cD[qx][ix] * B0[qx];
          t1 += cB[qx][ix] * B1[qx];
          t2 += cB[qx][ix] * B2[qx];
        }
        o[ix] = tv;
        o[48 + ix] = t1;
        o[96 + ix] = t2;
      }
    }
    __syncthreads();
    // ---------------- backward stage y (contract qy) ----------------
    // line (comp, part, qz, ix) -> ty[comp][part][{Ua,Ub}][qz][iy][ix]
    for (int l = t; l < 4 * 2 * 12; l += kGroup) {
      const int cp = l / 12, r = l % 12, qz = r / 3, ix = r % 3;
      const float* tx = S + oTX + cp * 3 * 48 + qz * 12 + ix;  // [arr*48 + qy*3]
      float* o = S + oTY + cp * 2 * 36 + qz * 9 + ix;
#pragma unroll
      for (int iy = 0; iy < 3; ++iy) {
        float ua = 0.f, ub = 0.f;
#pragma unroll
        for (int qy = 0; qy < 4; ++qy) {
          ua += cB[qy][iy] * tx[qy * 3] + cD[qy][iy] * tx[48 + qy * 3];
          ub += cB[qy][iy] * tx[96 + qy * 3];
        }
        o[iy * 3] = ua;
        o[36 + iy * 3] = ub;
      }
    }
    __syncthreads();
    // ---------------- backward stage z (contract qz) ----------------
    for (int l = t; l < 4 * 2 * 9; l += kGroup) {
      const int cp = l / 9, yx = l % 9;
      const float* ty = S + oTY + cp * 2 * 36 + yx;  // [arr*36 + qz*9]
      float* o = S + oTZ + cp * 27 + yx;
#pragma unroll
      for (int iz = 0; iz < 3; ++iz) {
        float s = 0.f;
#pragma unroll
        for (int qz = 0; qz < 4; ++qz) s += cB[qz][iz] * ty[qz * 9] + cD[qz][iz] * ty[36 + qz * 9];
        o[iz * 9] = s;
      }
    }
    __syncthreads();
    // ---------------- output: direct + PI^T * gpi part ----------------
    if (t < 27 && live) {
      float e[4];
#pragma unroll
      for (int comp = 0; comp < 4; ++comp) {
        float s = S[oTZ + (comp * 2) * 27 + t];
        // PI[b][t] is non-zero only for vertex nodes t
        const int ax = t % 3, ay = (t / 3) % 3, az = t / 9;
        if (ax != 1 && ay != 1 && az != 1) {
          const float* gp = S + oTZ + (comp * 2 + 1) * 27;
          for (int b = 0; b < 27; ++b) s = fmaf(pi_weight(b, t), gp[b], s);
        }
        e[comp] = s;
      }
      A.elem[(int64_t)c * 27 + t] = make_float4(e[0], e[1], e[2], e[3]);
    }
    __syncthreads();
  }
}

// out[n] = sign * sum_{incident (c,a), ascending c} elem[c][a] (+ b[n]); masked rows -> 0
__global__ void __launch_bounds__(256) node_sum_kernel(
    int n_nodes, const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
    const float4* __restrict__ elem, const float4* __restrict__ b, float sign,
    const uint8_t* __restrict__ mask, float4* __restrict__ out) {
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < n_nodes; n += gridDim.x * blockDim.x) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const int s = __ldg(ptr + n), e = __ldg(ptr + n + 1);
    for (int i = s; i < e; ++i) {
      const float4 v = __ldg(elem + __ldg(idx + i));
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
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
    const float den = nu / (h * h) + m / h + 1.0f / k;
    aT[c] = alpha0 / den;
    dT[c] = delta0 / den;
  }
}

constexpr int kCPB = 2;

static int32_t check_level(const dnnmg_level_t* lv, const char* who) {
  DNNMG_REQUIRE(lv && lv->cell_nodes && lv->coords && lv->h_T && lv->node_cell_ptr &&
                    lv->node_cell_idx,
                DNNMG_ERR_ARG, "%s: incomplete level tables", who);
  return DNNMG_OK;
}

static int32_t launch_elements(const dnnmg_level_t* lv, const float* x, const float* aT,
                               const float* dT, const dnnmg_phys_t* ph, int mode, float* elem,
                               cudaStream_t s) {
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
  A.alpha0 = ph->alpha0;
  A.delta0 = ph->delta0;
  A.convection = ph->convection;
  A.mode = mode;
  A.elem = reinterpret_cast<float4*>(elem);
  const size_t smem = sizeof(float) * kCellFloats * kCPB;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(element_kernel<kCPB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    configured = true;
  }
  int blocks = (lv->n_cells + kCPB - 1) / kCPB;
  const int cap = kSMs * 8;
  if (blocks > cap) blocks = cap;
  if (lv->n_cells == 0) return DNNMG_OK;
  element_kernel<kCPB><<<blocks, 64 * kCPB, smem, s>>>(A);
  DNNMG_CHECK_LAUNCH("element_kernel");
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
                        float* r, int apply_mask, int mode_sign, cudaStream_t s) {
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
  node_sum_kernel<<<grid_for(lv->n_nodes, 256), 256, 0, s>>>(
      lv->n_nodes, lv->node_cell_ptr, lv->node_cell_idx, reinterpret_cast<const float4*>(elem), b,
      1.0f, (apply_mask && lv->dof_mask) ? lv->dof_mask : nullptr, reinterpret_cast<float4*>(r));
  DNNMG_CHECK_LAUNCH("node_sum_kernel");
  return DNNMG_OK;
}

}  // namespace dnnmg
