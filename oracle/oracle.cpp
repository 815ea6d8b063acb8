// ============================================================================
// PG-SAG masked rasterizer — CPU ORACLE.  TEST INFRASTRUCTURE, NOT PRODUCT.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs may load this library.  It shares no code, header, table or
// constant generator with the CUDA path (paper_2501_01677_b200/csrc); the two
// are independent implementations of the readings listed in DESIGN.md §3.
//
// What it computes is the PLAIN DEFINITION of the method's render (PAPER.md
// §3.1, lines 78-96, Eq. 1-4): for every requested masked pixel, every
// Gaussian, ordered by (camera depth, id), alpha-composited front to back, and
// the exact reverse-mode gradient of that composite (PAPER.md:82
// "optimized ... using differentiable rendering").  Tiles appear only through
// the rect predicate, and `certify` counts pairs the rect excluded that would
// have contributed (must be 0: tiling is then a pure acceleration).
//
// Precision (reading R20): Real = float reproduces the discrete
// decisions of a float32 renderer (the tile keys are integer decisions made in
// float32, so both sides take them in float32); Real = double is used for the
// closed-form pins and the finite-difference pins.  Gradient sums are always
// accumulated in double.  Compile with -O2 -ffp-contract=off -fno-fast-math:
// every float expression below is evaluated exactly as written, left to right.
//
// Citations: P:n = /root/reference/PAPER.md line n.  Readings Rk = DESIGN.md §3.
// Parity of every function here is pinned by tests/test_oracle_pins.py.
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

// ---------------------------------------------------------------- flags (R*)
enum : uint32_t {
  F_VISIBLE = 1u << 0,   // z > znear                                  (R9)
  F_DET_OK = 1u << 1,    // det(cov2d) > 0                             (R10)
  F_OPAC_OK = 1u << 2,   // o >= 1/255                                 (R6)
  F_RECT = 1u << 3,      // tile rect non-empty                        (R8)
  F_CLAMP_X = 1u << 4,   // x/z clamped inside J                       (R9)
  F_CLAMP_Y = 1u << 5,
  F_RGB_CLAMP0 = 1u << 6,  // colour channel c clamped at 0 -> bit 6+c   (R12)
  F_NFLIP = 1u << 11,      // normal flipped to face the camera          (R4)
  F_AXIS_SHIFT = 9,        // bits 9-10: index of the minimum-scale axis  (R4)
};
constexpr uint32_t F_LIVE = F_VISIBLE | F_DET_OK | F_OPAC_OK | F_RECT;

template <typename R> struct Cam {
  R fx, fy, cx, cy;
  int W, H;
  R Rc[9];  // world -> camera, row-major (P:88 R_c)
  R C[3];   // camera centre T_C
  R znear;
};

template <typename R> Cam<R> load_cam(const double* cf, int W, int H) {
  // cf = [fx, fy, cx, cy, R0..R8, C0..C2, znear]; values are float32-representable.
  Cam<R> c;
  c.fx = (R)cf[0]; c.fy = (R)cf[1]; c.cx = (R)cf[2]; c.cy = (R)cf[3];
  for (int k = 0; k < 9; ++k) c.Rc[k] = (R)cf[4 + k];
  for (int k = 0; k < 3; ++k) c.C[k] = (R)cf[13 + k];
  c.znear = (R)cf[16];
  c.W = W; c.H = H;
  return c;
}

// ------------------------------------------------------------ SH basis (R12)
// Real spherical harmonics up to degree 3 in the 3DGS convention
// ("multi-order spherical harmonics"); pinned against scipy's complex
// Y_l^m (real part sqrt2*Re / sqrt2*Im) in test_oracle_pins.py.
const double SH_C0 = 0.28209479177387814;
const double SH_C1 = 0.4886025119029199;
const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                         -1.0925484305920792, 0.5462742152960396};
const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                         0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                         -0.5900435899266435};

template <typename R> void sh_basis(R x, R y, R z, R* Y) {
  const R xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  Y[0] = (R)SH_C0;
  Y[1] = -(R)SH_C1 * y;
  Y[2] = (R)SH_C1 * z;
  Y[3] = -(R)SH_C1 * x;
  Y[4] = (R)SH_C2[0] * xy;
  Y[5] = (R)SH_C2[1] * yz;
  Y[6] = (R)SH_C2[2] * (((R)2 * zz - xx) - yy);
  Y[7] = (R)SH_C2[3] * xz;
  Y[8] = (R)SH_C2[4] * (xx - yy);
  Y[9] = ((R)SH_C3[0] * y) * ((R)3 * xx - yy);
  Y[10] = ((R)SH_C3[1] * xy) * z;
  Y[11] = ((R)SH_C3[2] * y) * (((R)4 * zz - xx) - yy);
  Y[12] = ((R)SH_C3[3] * z) * (((R)2 * zz - (R)3 * xx) - (R)3 * yy);
  Y[13] = ((R)SH_C3[4] * x) * (((R)4 * zz - xx) - yy);
  Y[14] = ((R)SH_C3[5] * z) * (xx - yy);
  Y[15] = ((R)SH_C3[6] * x) * (xx - (R)3 * yy);
}

// gradient of each basis function w.r.t. the (unnormalised-treated) direction
// components, i.e. the partial derivatives of the polynomials above.
void sh_basis_grad(double x, double y, double z, double G[16][3]) {
  const double xx = x * x, yy = y * y, zz = z * z;
  const double* c2 = SH_C2;
  const double* c3 = SH_C3;
  double g[16][3] = {
      {0, 0, 0},
      {0, -SH_C1, 0},
      {0, 0, SH_C1},
      {-SH_C1, 0, 0},
      {c2[0] * y, c2[0] * x, 0},
      {0, c2[1] * z, c2[1] * y},
      {-2 * c2[2] * x, -2 * c2[2] * y, 4 * c2[2] * z},
      {c2[3] * z, 0, c2[3] * x},
      {2 * c2[4] * x, -2 * c2[4] * y, 0},
      {6 * c3[0] * x * y, c3[0] * (3 * xx - 3 * yy), 0},
      {c3[1] * y * z, c3[1] * x * z, c3[1] * x * y},
      {-2 * c3[2] * x * y, c3[2] * (4 * zz - xx - 3 * yy), 8 * c3[2] * y * z},
      {-6 * c3[3] * x * z, -6 * c3[3] * y * z, c3[3] * (6 * zz - 3 * xx - 3 * yy)},
      {c3[4] * (4 * zz - 3 * xx - yy), -2 * c3[4] * x * y, 8 * c3[4] * x * z},
      {2 * c3[5] * x * z, -2 * c3[5] * y * z, c3[5] * (xx - yy)},
      {c3[6] * (3 * xx - 3 * yy), -6 * c3[6] * x * y, 0},
  };
  std::memcpy(G, g, sizeof(g));
}

// ------------------------------------------------- log upper bound (R8)
// lnup(y) >= ln(y) for y >= 1 using only exact decomposition y = 2^e (1+f),
// f in [0,1), the Pade upper bound ln(1+f) <= f(6+f)/(6+4f) (slack f^4/36 for
// small f) and an absolute 2^-18 that absorbs the float rounding of the sum.
template <typename R> R lnup(R y) {
  int ex = 0;
  R m = std::frexp(y, &ex);         // y = m 2^ex, m in [0.5, 1)  (exact)
  const R e = (R)(ex - 1);
  const R f = (R)2 * m - (R)1;      // exact
  return (e * (R)0.6931471805599453 + (f * ((R)6 + f)) / ((R)6 + (R)4 * f)) + (R)3.814697265625e-06;
}

// ------------------------------------------------------- per-Gaussian (O2)
template <typename R> struct Proj {
  R u, v, ca, cb, cc, o, depth;
  int rect[4];  // tx0, ty0, tx1, ty1 (inclusive); empty = (0,0,-1,-1)
  uint32_t tiles;
  R rgb[3], ncam[3], dist;
  uint32_t flags;
};

struct TileMask {
  int TX, TY;
  std::vector<uint32_t> cnt;
  std::vector<int32_t> sat;  // (TY+1) x (TX+1)
  int rect_count(int tx0, int ty0, int tx1, int ty1) const {
    const int S = TX + 1;
    return sat[(ty1 + 1) * S + tx1 + 1] - sat[ty0 * S + tx1 + 1] - sat[(ty1 + 1) * S + tx0] +
           sat[ty0 * S + tx0];
  }
  bool active(int tx, int ty) const { return cnt[ty * TX + tx] > 0; }
};

// O1: per-16x16-tile mask-pixel counts and the summed-area table of active
// tiles ("only need to compute a subset of pixels"; reading R14).
TileMask make_tilemask(const uint8_t* mask, int W, int H) {
  TileMask tm;
  tm.TX = (W + 15) / 16;
  tm.TY = (H + 15) / 16;
  tm.cnt.assign((size_t)tm.TX * tm.TY, 0);
  for (int j = 0; j < H; ++j)
    for (int i = 0; i < W; ++i)
      if (mask[(size_t)j * W + i]) tm.cnt[(j / 16) * tm.TX + i / 16] += 1;
  const int S = tm.TX + 1;
  tm.sat.assign((size_t)(tm.TY + 1) * S, 0);
  for (int y = 1; y <= tm.TY; ++y)
    for (int x = 1; x <= tm.TX; ++x)
      tm.sat[y * S + x] = tm.sat[(y - 1) * S + x] + tm.sat[y * S + x - 1] -
                          tm.sat[(y - 1) * S + x - 1] +
                          (tm.cnt[(y - 1) * tm.TX + (x - 1)] > 0 ? 1 : 0);
  return tm;
}

template <typename R> struct Params {
  const R *mean, *scale, *rot, *opac, *sh;
  int n, deg;
};

template <typename R> void quat_to_rot(const R q[4], R Rg[3][3], R qn_out[4], R* norm_out) {
  const R qn = std::sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
  const R w = q[0] / qn, x = q[1] / qn, y = q[2] / qn, z = q[3] / qn;
  Rg[0][0] = (R)1 - (R)2 * (y * y + z * z);
  Rg[0][1] = (R)2 * (x * y - w * z);
  Rg[0][2] = (R)2 * (x * z + w * y);
  Rg[1][0] = (R)2 * (x * y + w * z);
  Rg[1][1] = (R)1 - (R)2 * (x * x + z * z);
  Rg[1][2] = (R)2 * (y * z - w * x);
  Rg[2][0] = (R)2 * (x * z - w * y);
  Rg[2][1] = (R)2 * (y * z + w * x);
  Rg[2][2] = (R)1 - (R)2 * (x * x + y * y);
  if (qn_out) { qn_out[0] = w; qn_out[1] = x; qn_out[2] = y; qn_out[3] = z; }
  if (norm_out) *norm_out = qn;
}

// O2: EWA projection, culling, conservative tile rect, normal, distance, colour.
// P:78 ("transformed into a 2D Gaussian ... projected onto different image
// tiles"), P:84-92 (Eq. 2-3: n_i, R_c n_i, d_i), readings R2,R4,R5,R8-R13.
template <typename R>
Proj<R> project(const Params<R>& P, int i, const Cam<R>& cam, const TileMask& tm) {
  Proj<R> g;
  std::memset(&g, 0, sizeof(g));
  g.rect[0] = 0; g.rect[1] = 0; g.rect[2] = -1; g.rect[3] = -1;
  const int N = P.n;
  const R m0 = P.mean[i], m1 = P.mean[N + i], m2 = P.mean[2 * N + i];
  const R t[3] = {m0 - cam.C[0], m1 - cam.C[1], m2 - cam.C[2]};
  const R* Rc = cam.Rc;
  R pc[3];
  for (int r = 0; r < 3; ++r) pc[r] = (Rc[3 * r] * t[0] + Rc[3 * r + 1] * t[1]) + Rc[3 * r + 2] * t[2];
  const R x = pc[0], y = pc[1], z = pc[2];
  uint32_t fl = 0;
  if (!(z > cam.znear)) { g.flags = fl; return g; }
  fl |= F_VISIBLE;
  g.depth = z;
  const R xz = x / z, yz = y / z;
  g.u = cam.fx * xz + cam.cx;
  g.v = cam.fy * yz + cam.cy;

  // 3D covariance Sigma = (Rg S)(Rg S)^T
  const R q[4] = {P.rot[i], P.rot[N + i], P.rot[2 * N + i], P.rot[3 * N + i]};
  R Rg[3][3];
  quat_to_rot(q, Rg, (R*)nullptr, (R*)nullptr);
  const R s[3] = {P.scale[i], P.scale[N + i], P.scale[2 * N + i]};
  R Mg[3][3], Sig[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) Mg[a][b] = Rg[a][b] * s[b];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) Sig[a][b] = (Mg[a][0] * Mg[b][0] + Mg[a][1] * Mg[b][1]) + Mg[a][2] * Mg[b][2];

  // perspective Jacobian with the 1.3 x half-FoV clamp (R9)
  const R lx = (R)1.3 * (((R)0.5 * (R)cam.W) / cam.fx);
  const R ly = (R)1.3 * (((R)0.5 * (R)cam.H) / cam.fy);
  R cxz = xz, cyz = yz;
  if (xz < -lx) { cxz = -lx; fl |= F_CLAMP_X; }
  if (xz > lx) { cxz = lx; fl |= F_CLAMP_X; }
  if (yz < -ly) { cyz = -ly; fl |= F_CLAMP_Y; }
  if (yz > ly) { cyz = ly; fl |= F_CLAMP_Y; }
  const R J[2][3] = {{cam.fx / z, (R)0, -((cam.fx * cxz) / z)},
                     {(R)0, cam.fy / z, -((cam.fy * cyz) / z)}};
  R Tm[2][3], Mt[2][3], cov[2][2];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 3; ++b) Tm[a][b] = (J[a][0] * Rc[b] + J[a][1] * Rc[3 + b]) + J[a][2] * Rc[6 + b];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 3; ++b) Mt[a][b] = (Tm[a][0] * Sig[0][b] + Tm[a][1] * Sig[1][b]) + Tm[a][2] * Sig[2][b];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) cov[a][b] = (Mt[a][0] * Tm[b][0] + Mt[a][1] * Tm[b][1]) + Mt[a][2] * Tm[b][2];
  const R A = cov[0][0] + (R)0.3, B = cov[0][1], Cc = cov[1][1] + (R)0.3;  // low-pass (R10)
  const R det = A * Cc - B * B;
  if (!(det > (R)0)) { g.flags = fl; return g; }
  fl |= F_DET_OK;
  g.ca = Cc / det;
  g.cb = -B / det;
  g.cc = A / det;
  const R o = P.opac[i];
  g.o = o;
  if (o < (R)1 / (R)255) { g.flags = fl; return g; }
  fl |= F_OPAC_OK;

  // opacity-aware conservative ellipse AABB (R8): every pixel with
  // alpha >= 1/255 satisfies d^T conic d <= 2 ln(255 o) <= k2.
  const R ylog = (R)255 * o;
  R k2 = ((R)2 * lnup(ylog)) * ((R)1 + (R)0.0009765625);
  if (k2 < (R)0) k2 = (R)0;
  const R PAD = (R)0.015625;
  const R rx = std::sqrt(k2 * A) + PAD, ry = std::sqrt(k2 * Cc) + PAD;
  auto clampf = [](R v) { return std::min(std::max(v, (R)-1048576), (R)1048576); };
  const int ix0 = (int)clampf(std::ceil((g.u - rx) - (R)0.5));
  const int ix1 = (int)clampf(std::floor((g.u + rx) - (R)0.5));
  const int iy0 = (int)clampf(std::ceil((g.v - ry) - (R)0.5));
  const int iy1 = (int)clampf(std::floor((g.v + ry) - (R)0.5));
  auto fdiv16 = [](int a) { return (a >= 0) ? a / 16 : -((-a + 15) / 16); };
  const int tx0 = std::max(0, fdiv16(ix0)), tx1 = std::min(tm.TX - 1, fdiv16(ix1));
  const int ty0 = std::max(0, fdiv16(iy0)), ty1 = std::min(tm.TY - 1, fdiv16(iy1));
  if (tx0 <= tx1 && ty0 <= ty1) {
    fl |= F_RECT;
    g.rect[0] = tx0; g.rect[1] = ty0; g.rect[2] = tx1; g.rect[3] = ty1;
    g.tiles = (uint32_t)tm.rect_count(tx0, ty0, tx1, ty1);
  }

  // flattened-Gaussian normal (Eq. 2; R4) and plane distance (Eq. 3; R2)
  int k = 0;
  if (s[1] < s[k]) k = 1;
  if (s[2] < s[k]) k = 2;
  fl |= (uint32_t)k << F_AXIS_SHIFT;
  R n[3] = {Rg[0][k], Rg[1][k], Rg[2][k]};
  const R dotv = (n[0] * t[0] + n[1] * t[1]) + n[2] * t[2];
  if (dotv > (R)0) { n[0] = -n[0]; n[1] = -n[1]; n[2] = -n[2]; fl |= F_NFLIP; }
  for (int r = 0; r < 3; ++r) g.ncam[r] = (Rc[3 * r] * n[0] + Rc[3 * r + 1] * n[1]) + Rc[3 * r + 2] * n[2];
  g.dist = (n[0] * t[0] + n[1] * t[1]) + n[2] * t[2];

  // view-dependent colour from SH (R12)
  const R len = std::sqrt((t[0] * t[0] + t[1] * t[1]) + t[2] * t[2]);
  const R dx = t[0] / len, dy = t[1] / len, dz = t[2] / len;
  R Y[16];
  sh_basis(dx, dy, dz, Y);
  const int K = (P.deg + 1) * (P.deg + 1);
  for (int c = 0; c < 3; ++c) {
    R acc = Y[0] * P.sh[(size_t)c * N + i];
    for (int l = 1; l < K; ++l) acc = acc + Y[l] * P.sh[(size_t)(l * 3 + c) * N + i];
    acc = acc + (R)0.5;
    if (acc < (R)0) { acc = (R)0; fl |= F_RGB_CLAMP0 << c; }
    g.rgb[c] = acc;
  }
  g.flags = fl;
  return g;
}

// ------------------------------------------------------ compositing (O4)
template <typename R> struct PixOut {
  R C[3], N[3], D, A, Dep, T;
  int g;
  int last;       // Gaussian id of the last blended, -1 if none
  int near_flag;  // some decision was within the reading-R18 margin
  long long evaluated;  // list entries visited (E counter)
  double id_sum;        // checksum of blended ids (FD validity)
  int n_clamped;        // blended pairs with o*rho > 0.99
  double gsoft;         // soft count sum_blended sigmoid(k (alpha - 1/255)) (R24)
};

// Soft-count surrogate of g_i (reading R24 after SPEC's DESIGN DECISIONS):
// each blended pair counts sigmoid(k (alpha - 1/255)), k = 100.
const double kGcK = 100.0;
inline double sigmoid(double z) { return 1.0 / (1.0 + std::exp(-z)); }

template <typename R> struct Blend {
  int id;
  R alpha, T, rho, orho, dx, dy;
};

template <typename R> struct Renderer {
  const Params<R>& P;
  const Cam<R>& cam;
  const TileMask& tm;
  std::vector<Proj<R>> proj;
  Renderer(const Params<R>& P_, const Cam<R>& cam_, const TileMask& tm_) : P(P_), cam(cam_), tm(tm_) {
    proj.resize(P.n);
    for (int i = 0; i < P.n; ++i) proj[i] = project(P, i, cam, tm);
  }

  // Candidates of tile (tx,ty): live Gaussians whose rect contains it, in
  // (depth, id) order ("sorted"; R11).
  void candidates(int tx, int ty, std::vector<int>& out) const {
    out.clear();
    for (int i = 0; i < P.n; ++i) {
      const Proj<R>& g = proj[i];
      if ((g.flags & F_LIVE) != F_LIVE) continue;
      if (tx < g.rect[0] || tx > g.rect[2] || ty < g.rect[1] || ty > g.rect[3]) continue;
      out.push_back(i);
    }
    std::stable_sort(out.begin(), out.end(), [&](int a, int b) {
      if (proj[a].depth != proj[b].depth) return proj[a].depth < proj[b].depth;
      return a < b;
    });
  }

  static bool near_rel(R a, R b, double tol) {
    return std::fabs((double)a - (double)b) <= tol * std::fabs((double)b);
  }

  // Eq. 1-3 front to back for pixel (i,j), then Eq. 4 (R1, R3, R5, R6, R15).
  PixOut<R> pixel(int i, int j, const std::vector<int>& cand, const R bg[3],
                  std::vector<Blend<R>>* blends) const {
    PixOut<R> o;
    std::memset(&o, 0, sizeof(o));
    o.last = -1;
    R T = (R)1;
    const R px = (R)i + (R)0.5, py = (R)j + (R)0.5;
    const R a_min = (R)1 / (R)255;
    const R t_min = (R)0.0001;
    if (blends) blends->clear();
    for (int id : cand) {
      const Proj<R>& g = proj[id];
      o.evaluated += 1;
      const R dx = px - g.u, dy = py - g.v;
      const R power = (R)-0.5 * ((g.ca * dx) * dx + (g.cc * dy) * dy) - (g.cb * dx) * dy;
      // R18: the decision band is 1e-5 plus the float32 rounding bound of the quadratic form,
      // which grows with the magnitude of its terms where they cancel (thin, rotated ellipses).
      const double band = 1e-5 + 1e-6 * (0.5 * (std::fabs((double)g.ca) * (double)dx * (double)dx +
                                                 std::fabs((double)g.cc) * (double)dy * (double)dy) +
                                          std::fabs((double)g.cb * (double)dx * (double)dy));
      if (std::fabs((double)power) < band) o.near_flag = 1;
      if (power > (R)0) continue;
      const R rho = std::exp(power);
      const R orho = g.o * rho;
      const R alpha = std::min((R)0.99, orho);
      if (near_rel(orho, a_min, band) || near_rel(orho, (R)0.99, band)) o.near_flag = 1;
      if (alpha < a_min) continue;
      const R Tn = T * ((R)1 - alpha);
      if (near_rel(Tn, t_min, 1e-3)) o.near_flag = 1;
      if (Tn < t_min) break;  // R6: the crossing Gaussian is not blended
      const R w = alpha * T;
      for (int c = 0; c < 3; ++c) o.C[c] = o.C[c] + w * g.rgb[c];
      for (int c = 0; c < 3; ++c) o.N[c] = o.N[c] + w * g.ncam[c];
      o.D = o.D + w * g.dist;
      if (blends) blends->push_back(Blend<R>{id, alpha, T, rho, orho, dx, dy});
      o.g += 1;
      o.gsoft += sigmoid(kGcK * ((double)alpha - 1.0 / 255.0));
      o.last = id;
      o.id_sum += (double)id;
      if (orho > (R)0.99) o.n_clamped += 1;
      T = Tn;
    }
    for (int c = 0; c < 3; ++c) o.C[c] = o.C[c] + T * bg[c];
    o.A = (R)1 - T;
    o.T = T;
    const R r0 = (px - cam.cx) / cam.fx, r1 = (py - cam.cy) / cam.fy;
    const R den = (o.N[0] * r0 + o.N[1] * r1) + o.N[2];
    o.Dep = (o.g > 0 && std::fabs(den) > (R)1e-6) ? o.D / den : (R)0;  // Eq. 4, R3
    return o;
  }

  // Certificate: pairs excluded by the rect that would have alpha >= 1/255.  shrink > 0 (negative
  // control of the certificate itself, tests only) first narrows every rect by that many tiles
  // per side, which must then produce excluded pairs.
  long long certify(int i, int j, int shrink = 0) const {
    long long bad = 0;
    const int tx = i / 16, ty = j / 16;
    const R px = (R)i + (R)0.5, py = (R)j + (R)0.5;
    for (int id = 0; id < P.n; ++id) {
      const Proj<R>& g = proj[id];
      const uint32_t need = F_VISIBLE | F_DET_OK | F_OPAC_OK;
      if ((g.flags & need) != need) continue;
      const bool inrect = (g.flags & F_RECT) && tx >= g.rect[0] + shrink && tx <= g.rect[2] - shrink &&
                          ty >= g.rect[1] + shrink && ty <= g.rect[3] - shrink;
      if (inrect) continue;
      const R dx = px - g.u, dy = py - g.v;
      const R power = (R)-0.5 * ((g.ca * dx) * dx + (g.cc * dy) * dy) - (g.cb * dx) * dy;
      if (power > (R)0) continue;
      const R alpha = std::min((R)0.99, g.o * std::exp(power));
      if (alpha >= (R)1 / (R)255) ++bad;
    }
    return bad;
  }
};

// -------------------------------------------------- per-Gaussian 2D grads
struct G2 {
  double du, dv, dca, dcb, dcc, dop, drgb[3], dncam[3], ddist, absg;
  // sums over pixels of |contribution| for the 13 values above (du .. ddist): the scale of the
  // float32 rounding of a GPU that sums the same per-pixel terms (R19b)
  double abs[13];
  // R19c: first-order bound on what float32 EVALUATION of alpha / rho / T (GPU and this oracle's
  // float build each round them on their own) can move the same 13 sums; see eval_bound()
  double ev[13];
};

// R19c: first-order bound on the change of one pixel's per-Gaussian 2D-gradient terms when every
// blended alpha_k (and rho_k) carries a relative error e_k and every T_m a relative error E_m --
// the size of the difference between two float32 evaluations of the same Eq. 2 / Eq. 1 chain
// (the CUDA path's and this oracle's float build), which decide identically (R18 excludes
// pixels near a threshold) but round differently.  Derivation (R19c):
//  * e_k = 16 eps (mag_k + 1), eps = 2^-24, mag_k = |a|dx^2/2 + |c|dy^2/2 + |b dx dy| the
//    magnitude of Eq. 2's terms: the GPU rounds 3 pre-scaled coefficients and 3 fused ops
//    (<= 6 eps log2(e) mag in the base-2 exponent -> 6 eps mag in rho) plus ex2.approx
//    (<= 2^-22 = 4 eps) and o*rho (eps); the float oracle rounds 7 products/sums of Eq. 2
//    (<= 7 eps mag) plus expf (<= 2 eps) and o*rho (eps): 13 eps mag + 10 eps <= 16 eps (mag + 1).
//    A clamped alpha (o rho > 0.99) is the exact 0.99 on both sides: e = 0.
//  * T_m = prod_{k<m} (1 - alpha_k): a relative alpha error moves (1 - alpha_k) by
//    alpha_k e_k / (1 - alpha_k), its rounding by <= 2 eps / (1 - alpha_k) (both sides); each
//    side rounds the running product once per layer and the GPU's backward recovers T_m by one
//    division per later layer: E_m = 2 eps (K + 1) + sum_{k<m} (alpha_k e_k + 2 eps)/(1 - alpha_k).
// tests only: 0 drops the R19c part from the returned bound (its negative control)
int g_bound_eval = 1;

template <typename R>
void alpha_errors(const Renderer<R>& rd, const std::vector<Blend<R>>& bl, std::vector<double>& e,
                  std::vector<double>& E) {
  const double eps = 5.9604644775390625e-08;  // 2^-24
  const int K = (int)bl.size();
  e.assign(K, 0.0);
  E.assign(K, 0.0);
  double acc = 2.0 * eps * (K + 1);
  for (int k = 0; k < K; ++k) {
    const Blend<R>& b = bl[k];
    const Proj<R>& g = rd.proj[b.id];
    const double dx = (double)b.dx, dy = (double)b.dy;
    const double mag = 0.5 * (std::fabs((double)g.ca) * dx * dx + std::fabs((double)g.cc) * dy * dy) +
                       std::fabs((double)g.cb * dx * dy);
    e[k] = (b.orho > (R)0.99) ? 0.0 : 16.0 * eps * (mag + 1.0);
    E[k] = acc;
    acc += ((double)b.alpha * e[k] + 2.0 * eps) / (1.0 - (double)b.alpha);
  }
}

// R19c (continued), given e, E and the per-layer dalpha (without the soft-count term, `dam`) and
// dGa_m = T_m sum_c dG_c |F_mc - S_mc|, the part of dalpha_m moved by the error dG of Eq. 4's
// upstream fold (see pixel_backward):
//  * dalpha_m = T_m (G.(F_m - S_m) - P_m bg.G) depends on alpha_k, k > m, through the suffix:
//    d dalpha_m / d alpha_k = -dalpha_k / (1 - alpha_m) (exact identity of the recursion), so a
//    perturbation of the later layers moves it by sum_{k>m} alpha_k e_k |dalpha_k| / (1 - alpha_m).
//  * then w = alpha T, d o = rho dalpha, dpow = alpha dalpha and the conic / mean terms
//    (linear in dpow with coefficients both sides hold bit-identically) follow by the product rule.
template <typename R>
void eval_bound(const Renderer<R>& rd, const std::vector<Blend<R>>& bl, const double G[8], const double dG[8],
                double gG, const std::vector<double>& e, const std::vector<double>& E,
                const std::vector<double>& dam, const std::vector<double>& dGa, std::vector<G2>& g2) {
  const int K = (int)bl.size();
  if (K == 0) return;
  std::vector<double> suf(K + 1, 0.0);
  for (int k = K - 1; k >= 0; --k) suf[k] = suf[k + 1] + (double)bl[k].alpha * e[k] * std::fabs(dam[k]);
  for (int m = 0; m < K; ++m) {
    const Blend<R>& b = bl[m];
    const Proj<R>& g = rd.proj[b.id];
    const double a = (double)b.alpha, T = (double)b.T, rho = (double)b.rho;
    G2& o = g2[b.id];
    const double w = a * T, dw = w * (e[m] + E[m]);
    for (int c = 0; c < 3; ++c) o.ev[6 + c] += dw * std::fabs(G[c]) + w * dG[c];
    for (int c = 0; c < 3; ++c) o.ev[9 + c] += dw * std::fabs(G[3 + c]) + w * dG[3 + c];
    o.ev[12] += dw * std::fabs(G[6]) + w * dG[6];
    double da = dam[m], dda = std::fabs(dam[m]) * E[m] + suf[m + 1] / (1.0 - a) + dGa[m];
    if (gG != 0.0) {
      const double s = sigmoid(kGcK * (a - 1.0 / 255.0));
      da += gG * kGcK * s * (1.0 - s);
      dda += std::fabs(gG * kGcK * kGcK * s * (1.0 - s) * (1.0 - 2.0 * s)) * a * e[m];
    }
    if (b.orho <= (R)0.99) {
      const double ddop = rho * (e[m] * std::fabs(da) + dda);
      const double ddpow = a * (e[m] * std::fabs(da) + dda);
      const double dx = (double)b.dx, dy = (double)b.dy;
      o.ev[5] += ddop;
      o.ev[2] += 0.5 * dx * dx * ddpow;
      o.ev[3] += std::fabs(dx * dy) * ddpow;
      o.ev[4] += 0.5 * dy * dy * ddpow;
      o.ev[0] += std::fabs((double)g.ca * dx + (double)g.cb * dy) * ddpow;
      o.ev[1] += std::fabs((double)g.cb * dx + (double)g.cc * dy) * ddpow;
    }
  }
}

// O5: reverse-order backward of one pixel (exact reverse mode of Eq. 1-4,
// P:82; decisions frozen per R17; clamp gradient per R16).
template <typename R>
void pixel_backward(const Renderer<R>& rd, int i, int j, const PixOut<R>& fw,
                    const std::vector<Blend<R>>& bl, const R bg[3], const double up[10],
                    std::vector<G2>& g2) {
  // up = (gC0,gC1,gC2, gN0,gN1,gN2, gD, gA, gDep, gG) with gG = dL/d(soft count) (R24)
  double G[8] = {up[0], up[1], up[2], up[3], up[4], up[5], up[6], up[7]};
  const double gDep = up[8];
  const double gG = up[9];
  const double px = i + 0.5, py = j + 0.5;
  const double r[3] = {(px - (double)rd.cam.cx) / (double)rd.cam.fx,
                       (py - (double)rd.cam.cy) / (double)rd.cam.fy, 1.0};
  const double den = (double)fw.N[0] * r[0] + (double)fw.N[1] * r[1] + (double)fw.N[2];
  // validity decided exactly as the forward decided it (in R)
  const R r0R = (((R)i + (R)0.5) - rd.cam.cx) / rd.cam.fx, r1R = (((R)j + (R)0.5) - rd.cam.cy) / rd.cam.fy;
  const bool dep_valid = fw.g > 0 && std::fabs((fw.N[0] * r0R + fw.N[1] * r1R) + fw.N[2]) > (R)1e-6;
  if (dep_valid) {  // Eq. 4: Dep = D / (N . r)
    G[6] += gDep / den;
    for (int c = 0; c < 3; ++c) G[3 + c] -= gDep * (double)fw.D / (den * den) * r[c];
  }
  // R19c: the fold above uses the forward's float32 N and D, which the GPU and the float build
  // accumulate with their own alpha / T errors (e_k + E_k relative per blended weight) and
  // roundings (one per layer each side: 2 (K + 1) eps relative): dN_c, dD bound the difference;
  // den = N.r adds 3 eps of |N0 r0| + |N1 r1| + |N2|, each division 2 eps.  dG bounds the
  // resulting difference of the folded upstream.
  const double eps = 5.9604644775390625e-08;
  std::vector<double> ea, Ea;
  alpha_errors(rd, bl, ea, Ea);
  double dG[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (dep_valid && gDep != 0.0) {
    const int K = (int)bl.size();
    double dN[3] = {0, 0, 0}, dD = 0.0;
    for (int k = 0; k < K; ++k) {
      const Proj<R>& g = rd.proj[bl[k].id];
      const double w = (double)bl[k].alpha * (double)bl[k].T;
      const double rel = ea[k] + Ea[k] + 2.0 * eps * (K + 1);
      for (int c = 0; c < 3; ++c) dN[c] += std::fabs(w * (double)g.ncam[c]) * rel;
      dD += std::fabs(w * (double)g.dist) * rel;
    }
    const double ad = std::fabs(den);
    const double dden = std::fabs(r[0]) * dN[0] + std::fabs(r[1]) * dN[1] + dN[2] +
                        3.0 * eps * (std::fabs((double)fw.N[0] * r[0]) + std::fabs((double)fw.N[1] * r[1]) +
                                     std::fabs((double)fw.N[2]));
    const double aD = std::fabs((double)fw.D);
    dG[6] = std::fabs(gDep) * (dden / (ad * ad) + 2.0 * eps / ad);
    for (int c = 0; c < 3; ++c)
      dG[3 + c] = std::fabs(gDep * r[c]) * (dD / (ad * ad) + 2.0 * aD * dden / (ad * ad * ad) +
                                            4.0 * eps * aD / (ad * ad));
  }
  std::vector<double> dGa(bl.size(), 0.0);
  const double bgdot = (double)bg[0] * G[0] + (double)bg[1] * G[1] + (double)bg[2] * G[2];
  double S[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  double Pp = 1.0;
  std::vector<double> dam(bl.size());  // dalpha without the soft-count term, per layer
  for (int k = (int)bl.size() - 1; k >= 0; --k) {
    const Blend<R>& b = bl[k];
    const Proj<R>& g = rd.proj[b.id];
    const double F[8] = {(double)g.rgb[0], (double)g.rgb[1], (double)g.rgb[2], (double)g.ncam[0],
                         (double)g.ncam[1], (double)g.ncam[2], (double)g.dist, 1.0};
    const double a = (double)b.alpha, T = (double)b.T;
    double dot = 0.0;
    for (int c = 0; c < 8; ++c) dot += G[c] * (F[c] - S[c]);
    double dalpha = T * (dot - Pp * bgdot);
    dam[k] = dalpha;  // S is still the suffix after layer k here
    for (int c = 3; c < 7; ++c) dGa[k] += T * dG[c] * std::fabs(F[c] - S[c]);
    if (gG != 0.0) {  // d(soft count)/d alpha = k s (1 - s), s = sigmoid(k (alpha - 1/255))
      const double s = sigmoid(kGcK * (a - 1.0 / 255.0));
      dalpha += gG * kGcK * s * (1.0 - s);
    }
    const double w = a * T;
    G2& o = g2[b.id];
    for (int c = 0; c < 3; ++c) { o.drgb[c] += w * G[c]; o.abs[6 + c] += std::fabs(w * G[c]); }
    for (int c = 0; c < 3; ++c) { o.dncam[c] += w * G[3 + c]; o.abs[9 + c] += std::fabs(w * G[3 + c]); }
    o.ddist += w * G[6];
    o.abs[12] += std::fabs(w * G[6]);
    for (int c = 0; c < 8; ++c) S[c] = a * F[c] + (1.0 - a) * S[c];
    Pp *= (1.0 - a);
    double dpow = 0.0;
    if (b.orho <= (R)0.99) {
      o.dop += (double)b.rho * dalpha;
      o.abs[5] += std::fabs((double)b.rho * dalpha);
      dpow = a * dalpha;
    }
    const double dx = (double)b.dx, dy = (double)b.dy;
    o.dca += -0.5 * dx * dx * dpow;
    o.dcb += -dx * dy * dpow;
    o.dcc += -0.5 * dy * dy * dpow;
    o.abs[2] += std::fabs(0.5 * dx * dx * dpow);
    o.abs[3] += std::fabs(dx * dy * dpow);
    o.abs[4] += std::fabs(0.5 * dy * dy * dpow);
    const double du = ((double)g.ca * dx + (double)g.cb * dy) * dpow;
    const double dv = ((double)g.cb * dx + (double)g.cc * dy) * dpow;
    o.du += du;
    o.dv += dv;
    o.abs[0] += std::fabs(du);
    o.abs[1] += std::fabs(dv);
    o.absg += std::fabs(du) + std::fabs(dv);  // densification statistic (sum over pixels)
  }
  eval_bound(rd, bl, G, dG, gG, ea, Ea, dam, dGa, g2);
}

// O6: chain rule from the 2D/per-Gaussian gradients to the 3D parameters
// (P:82), through O2 in double; decisions (clamps, axis, flip) from flags.
template <typename R>
void gaussian_backward(const Params<R>& P, int i, const Cam<R>& camR, uint32_t fl, const G2& g,
                       double* dmean, double* dscale, double* drot, double* dopac, double* dsh) {
  const int N = P.n;
  if ((fl & F_LIVE) != F_LIVE) return;
  Cam<double> cam;
  cam.fx = camR.fx; cam.fy = camR.fy; cam.cx = camR.cx; cam.cy = camR.cy;
  for (int k = 0; k < 9; ++k) cam.Rc[k] = camR.Rc[k];
  for (int k = 0; k < 3; ++k) cam.C[k] = camR.C[k];
  const double* Rc = cam.Rc;
  const double t[3] = {(double)P.mean[i] - cam.C[0], (double)P.mean[N + i] - cam.C[1],
                       (double)P.mean[2 * N + i] - cam.C[2]};
  double pc[3];
  for (int r = 0; r < 3; ++r) pc[r] = Rc[3 * r] * t[0] + Rc[3 * r + 1] * t[1] + Rc[3 * r + 2] * t[2];
  const double x = pc[0], y = pc[1], z = pc[2];
  const double q[4] = {(double)P.rot[i], (double)P.rot[N + i], (double)P.rot[2 * N + i], (double)P.rot[3 * N + i]};
  double Rg[3][3], qh[4], qn;
  quat_to_rot(q, Rg, qh, &qn);
  const double s[3] = {(double)P.scale[i], (double)P.scale[N + i], (double)P.scale[2 * N + i]};
  double Mg[3][3], Sig[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) Mg[a][b] = Rg[a][b] * s[b];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) Sig[a][b] = Mg[a][0] * Mg[b][0] + Mg[a][1] * Mg[b][1] + Mg[a][2] * Mg[b][2];
  const bool clx = fl & F_CLAMP_X, cly = fl & F_CLAMP_Y;
  const double lx = 1.3 * (0.5 * camR.W / cam.fx), ly = 1.3 * (0.5 * camR.H / cam.fy);
  const double xz = x / z, yz = y / z;
  const double cxz = clx ? std::min(std::max(xz, -lx), lx) : xz;
  const double cyz = cly ? std::min(std::max(yz, -ly), ly) : yz;
  const double J[2][3] = {{cam.fx / z, 0.0, -cam.fx * cxz / z}, {0.0, cam.fy / z, -cam.fy * cyz / z}};
  double Tm[2][3];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 3; ++b) Tm[a][b] = J[a][0] * Rc[b] + J[a][1] * Rc[3 + b] + J[a][2] * Rc[6 + b];
  double cov[2][2];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      double acc = 0;
      for (int k = 0; k < 3; ++k)
        for (int l = 0; l < 3; ++l) acc += Tm[a][k] * Sig[k][l] * Tm[b][l];
      cov[a][b] = acc;
    }
  const double A = cov[0][0] + 0.3, B = cov[0][1], C = cov[1][1] + 0.3;
  const double det = A * C - B * B, det2 = det * det;
  // conic (ca,cb,cc) = (C,-B,A)/det  ->  d(A,B,C)
  const double dA = (-C * C * g.dca + B * C * g.dcb - B * B * g.dcc) / det2;
  const double dC = (-B * B * g.dca + A * B * g.dcb - A * A * g.dcc) / det2;
  const double dB = (2 * B * C * g.dca - (A * C + B * B) * g.dcb + 2 * A * B * g.dcc) / det2;
  // cov_ab = Tm_a Sig Tm_b^T
  double dSig[3][3];
  for (int k = 0; k < 3; ++k)
    for (int l = 0; l < 3; ++l)
      dSig[k][l] = dA * Tm[0][k] * Tm[0][l] + dC * Tm[1][k] * Tm[1][l] + dB * Tm[0][k] * Tm[1][l];
  double STm[2][3];  // Sig Tm_a^T
  for (int a = 0; a < 2; ++a)
    for (int k = 0; k < 3; ++k) STm[a][k] = Sig[k][0] * Tm[a][0] + Sig[k][1] * Tm[a][1] + Sig[k][2] * Tm[a][2];
  double dTm[2][3];
  for (int k = 0; k < 3; ++k) {
    dTm[0][k] = 2 * dA * STm[0][k] + dB * STm[1][k];
    dTm[1][k] = 2 * dC * STm[1][k] + dB * STm[0][k];
  }
  // Tm = J Rc
  double dJ[2][3];
  for (int a = 0; a < 2; ++a)
    for (int k = 0; k < 3; ++k) dJ[a][k] = dTm[a][0] * Rc[3 * k] + dTm[a][1] * Rc[3 * k + 1] + dTm[a][2] * Rc[3 * k + 2];
  double dp[3] = {0, 0, 0};
  const double z2 = z * z, z3 = z2 * z;
  dp[2] += -cam.fx / z2 * dJ[0][0] - cam.fy / z2 * dJ[1][1];
  if (!clx) { dp[0] += -cam.fx / z2 * dJ[0][2]; dp[2] += 2 * cam.fx * x / z3 * dJ[0][2]; }
  else { dp[2] += cam.fx * cxz / z2 * dJ[0][2]; }
  if (!cly) { dp[1] += -cam.fy / z2 * dJ[1][2]; dp[2] += 2 * cam.fy * y / z3 * dJ[1][2]; }
  else { dp[2] += cam.fy * cyz / z2 * dJ[1][2]; }
  // mean2d
  dp[0] += cam.fx / z * g.du;
  dp[2] += -cam.fx * x / z2 * g.du;
  dp[1] += cam.fy / z * g.dv;
  dp[2] += -cam.fy * y / z2 * g.dv;
  double dt[3];
  for (int k = 0; k < 3; ++k) dt[k] = Rc[k] * dp[0] + Rc[3 + k] * dp[1] + Rc[6 + k] * dp[2];
  // Sigma = Mg Mg^T
  double dMg[3][3], dRg[3][3];
  for (int k = 0; k < 3; ++k)
    for (int m = 0; m < 3; ++m) {
      double acc = 0;
      for (int l = 0; l < 3; ++l) acc += (dSig[k][l] + dSig[l][k]) * Mg[l][m];
      dMg[k][m] = acc;
    }
  double ds[3] = {0, 0, 0};
  for (int k = 0; k < 3; ++k)
    for (int m = 0; m < 3; ++m) {
      ds[m] += dMg[k][m] * Rg[k][m];
      dRg[k][m] = dMg[k][m] * s[m];
    }
  // normal n = sgn Rg[:,k];  ncam = Rc n;  dist = n . t
  const int ax = (fl >> F_AXIS_SHIFT) & 3;
  const double sg = (fl & F_NFLIP) ? -1.0 : 1.0;
  const double n[3] = {sg * Rg[0][ax], sg * Rg[1][ax], sg * Rg[2][ax]};
  double dn[3];
  for (int k = 0; k < 3; ++k) dn[k] = Rc[k] * g.dncam[0] + Rc[3 + k] * g.dncam[1] + Rc[6 + k] * g.dncam[2];
  for (int k = 0; k < 3; ++k) { dn[k] += t[k] * g.ddist; dt[k] += n[k] * g.ddist; }
  for (int k = 0; k < 3; ++k) dRg[k][ax] += sg * dn[k];
  // Rg(qh)
  const double w = qh[0], X = qh[1], Y = qh[2], Z = qh[3];
  double dq[4] = {0, 0, 0, 0};  // w, x, y, z
  dq[2] += -4 * Y * dRg[0][0]; dq[3] += -4 * Z * dRg[0][0];
  dq[1] += 2 * Y * dRg[0][1]; dq[2] += 2 * X * dRg[0][1]; dq[0] += -2 * Z * dRg[0][1]; dq[3] += -2 * w * dRg[0][1];
  dq[1] += 2 * Z * dRg[0][2]; dq[3] += 2 * X * dRg[0][2]; dq[0] += 2 * Y * dRg[0][2]; dq[2] += 2 * w * dRg[0][2];
  dq[1] += 2 * Y * dRg[1][0]; dq[2] += 2 * X * dRg[1][0]; dq[0] += 2 * Z * dRg[1][0]; dq[3] += 2 * w * dRg[1][0];
  dq[1] += -4 * X * dRg[1][1]; dq[3] += -4 * Z * dRg[1][1];
  dq[2] += 2 * Z * dRg[1][2]; dq[3] += 2 * Y * dRg[1][2]; dq[0] += -2 * X * dRg[1][2]; dq[1] += -2 * w * dRg[1][2];
  dq[1] += 2 * Z * dRg[2][0]; dq[3] += 2 * X * dRg[2][0]; dq[0] += -2 * Y * dRg[2][0]; dq[2] += -2 * w * dRg[2][0];
  dq[2] += 2 * Z * dRg[2][1]; dq[3] += 2 * Y * dRg[2][1]; dq[0] += 2 * X * dRg[2][1]; dq[1] += 2 * w * dRg[2][1];
  dq[1] += -4 * X * dRg[2][2]; dq[2] += -4 * Y * dRg[2][2];
  const double qdot = qh[0] * dq[0] + qh[1] * dq[1] + qh[2] * dq[2] + qh[3] * dq[3];
  double dqr[4];
  for (int k = 0; k < 4; ++k) dqr[k] = (dq[k] - qh[k] * qdot) / qn;
  // SH colour
  const double len = std::sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
  const double dir[3] = {t[0] / len, t[1] / len, t[2] / len};
  double Yb[16], GY[16][3];
  sh_basis(dir[0], dir[1], dir[2], Yb);
  sh_basis_grad(dir[0], dir[1], dir[2], GY);
  const int K = (P.deg + 1) * (P.deg + 1);
  double ddir[3] = {0, 0, 0};
  for (int c = 0; c < 3; ++c) {
    if (fl & (F_RGB_CLAMP0 << c)) continue;
    const double gc = g.drgb[c];
    for (int l = 0; l < K; ++l) {
      const double shv = (double)P.sh[(size_t)(l * 3 + c) * N + i];
      dsh[(size_t)(l * 3 + c) * N + i] = Yb[l] * gc;
      for (int k = 0; k < 3; ++k) ddir[k] += GY[l][k] * shv * gc;
    }
  }
  const double dd = dir[0] * ddir[0] + dir[1] * ddir[1] + dir[2] * ddir[2];
  for (int k = 0; k < 3; ++k) dt[k] += (ddir[k] - dir[k] * dd) / len;
  for (int k = 0; k < 3; ++k) dmean[(size_t)k * N + i] = dt[k];
  for (int k = 0; k < 3; ++k) dscale[(size_t)k * N + i] = ds[k];
  for (int k = 0; k < 4; ++k) drot[(size_t)k * N + i] = dqr[k];
  dopac[i] = g.dop;
}

template <typename R>
Params<R> make_params(const R* mean, const R* scale, const R* rot, const R* opac, const R* sh, int n, int deg) {
  Params<R> p;
  p.mean = mean; p.scale = scale; p.rot = rot; p.opac = opac; p.sh = sh; p.n = n; p.deg = deg;
  return p;
}

// ----------------------------------------------------------- entry points
template <typename R>
void project_all(const R* mean, const R* scale, const R* rot, const R* opac, const R* sh, int n, int deg,
                 const double* camf, int W, int H, const uint8_t* mask, R* mean2d, R* conic_o, R* depth,
                 int32_t* rect, uint32_t* tiles, R* rgb, R* ncam, R* dist, uint32_t* flags) {
  const Params<R> P = make_params(mean, scale, rot, opac, sh, n, deg);
  const Cam<R> cam = load_cam<R>(camf, W, H);
  const TileMask tm = make_tilemask(mask, W, H);
  for (int i = 0; i < n; ++i) {
    const Proj<R> g = project(P, i, cam, tm);
    mean2d[2 * i] = g.u; mean2d[2 * i + 1] = g.v;
    conic_o[4 * i] = g.ca; conic_o[4 * i + 1] = g.cb; conic_o[4 * i + 2] = g.cc; conic_o[4 * i + 3] = g.o;
    depth[i] = g.depth;
    for (int k = 0; k < 4; ++k) rect[4 * i + k] = g.rect[k];
    tiles[i] = g.tiles;
    for (int c = 0; c < 3; ++c) { rgb[3 * i + c] = g.rgb[c]; ncam[3 * i + c] = g.ncam[c]; }
    dist[i] = g.dist;
    flags[i] = g.flags;
  }
}

template <typename R>
void render_pixels(const R* mean, const R* scale, const R* rot, const R* opac, const R* sh, int n, int deg,
                   const double* camf, int W, int H, const uint8_t* mask, const double* bgd,
                   const int64_t* pix, int npix, R* out /* [npix][10]: C3 N3 D A Dep T */,
                   int32_t* iout /* [npix][4]: g last near_flag n_clamped */, double* id_sum, int64_t* evaluated,
                   double* gsoft /* [npix] soft counts (R24) or null */, int certify_flag, int64_t* cert_bad,
                   const double* upstream /* [npix][10] or null */, double* grads /* 73 x n or null */,
                   double* bound /* 59 x n or null: R19b accumulation bound of rows 0..58 */,
                   bool fproj = false /* R = double only: project in float32, evaluate Eq. 1-4 in R */) {
  const Params<R> P = make_params(mean, scale, rot, opac, sh, n, deg);
  const Cam<R> cam = load_cam<R>(camf, W, H);
  const TileMask tm = make_tilemask(mask, W, H);
  Renderer<R> rd(P, cam, tm);
  if (fproj) {  // the float32 build's O2 output (bit-identical to the CUDA A1), widened exactly
    const size_t K = (size_t)(deg + 1) * (deg + 1) * 3;
    std::vector<float> fm(mean, mean + 3 * (size_t)n), fs(scale, scale + 3 * (size_t)n),
        fr(rot, rot + 4 * (size_t)n), fo(opac, opac + (size_t)n), fsh(sh, sh + K * n);
    const Params<float> PF = make_params<float>(fm.data(), fs.data(), fr.data(), fo.data(), fsh.data(), n, deg);
    const Cam<float> camF = load_cam<float>(camf, W, H);
    Renderer<float> rf(PF, camF, tm);
    for (int i = 0; i < n; ++i) {
      const Proj<float>& a = rf.proj[i];
      Proj<R>& b = rd.proj[i];
      b.u = a.u; b.v = a.v; b.ca = a.ca; b.cb = a.cb; b.cc = a.cc; b.o = a.o; b.depth = a.depth;
      for (int k = 0; k < 4; ++k) b.rect[k] = a.rect[k];
      b.tiles = a.tiles;
      for (int c = 0; c < 3; ++c) { b.rgb[c] = a.rgb[c]; b.ncam[c] = a.ncam[c]; }
      b.dist = a.dist;
      b.flags = a.flags;
    }
  }
  const R bg[3] = {(R)bgd[0], (R)bgd[1], (R)bgd[2]};
  // group requested pixels by tile so each tile's candidate list is built once
  std::vector<int> order(npix);
  for (int k = 0; k < npix; ++k) order[k] = k;
  auto tile_of = [&](int k) { const int64_t p = pix[k]; return (int)((p / W) / 16) * tm.TX + (int)((p % W) / 16); };
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return tile_of(a) < tile_of(b); });
  std::vector<int> cand;
  std::vector<Blend<R>> bl;
  std::vector<G2> g2;
  if (grads) g2.assign(n, G2{0, 0, 0, 0, 0, 0, {0, 0, 0}, {0, 0, 0}, 0, 0, {0}});
  int cur_tile = -1;
  long long bad = 0;
  for (int k : order) {
    const int64_t p = pix[k];
    const int i = (int)(p % W), j = (int)(p / W);
    if (!mask[p]) {  // masked-out pixels are not rendered (R14)
      for (int c = 0; c < 10; ++c) out[(size_t)k * 10 + c] = (R)0;
      iout[(size_t)k * 4] = 0; iout[(size_t)k * 4 + 1] = -1; iout[(size_t)k * 4 + 2] = 0; iout[(size_t)k * 4 + 3] = 0;
      continue;
    }
    const int t = tile_of(k);
    if (t != cur_tile) { rd.candidates(i / 16, j / 16, cand); cur_tile = t; }
    const PixOut<R> o = rd.pixel(i, j, cand, bg, grads ? &bl : nullptr);
    R* op = out + (size_t)k * 10;
    op[0] = o.C[0]; op[1] = o.C[1]; op[2] = o.C[2];
    op[3] = o.N[0]; op[4] = o.N[1]; op[5] = o.N[2];
    op[6] = o.D; op[7] = o.A; op[8] = o.Dep; op[9] = o.T;
    iout[(size_t)k * 4] = o.g; iout[(size_t)k * 4 + 1] = o.last;
    iout[(size_t)k * 4 + 2] = o.near_flag; iout[(size_t)k * 4 + 3] = o.n_clamped;
    if (id_sum) id_sum[k] = o.id_sum;
    if (evaluated) evaluated[k] = o.evaluated;
    if (gsoft) gsoft[k] = o.gsoft;
    if (certify_flag) bad += rd.certify(i, j, certify_flag - 1);
    if (grads) pixel_backward(rd, i, j, o, bl, bg, upstream + (size_t)k * 10, g2);
  }
  if (cert_bad) *cert_bad = bad;
  if (grads) {
    double* dmean = grads;
    double* dscale = grads + (size_t)3 * n;
    double* drot = grads + (size_t)6 * n;
    double* dop = grads + (size_t)10 * n;
    double* dsh = grads + (size_t)11 * n;
    std::memset(grads, 0, sizeof(double) * (size_t)73 * n);
    for (int i = 0; i < n; ++i) gaussian_backward(P, i, cam, rd.proj[i].flags, g2[i], dmean, dscale, drot, dop, dsh);
    // rows 59..72: the per-Gaussian 2D gradients (O5 output) and the absgrad statistic
    for (int i = 0; i < n; ++i) {
      if ((rd.proj[i].flags & F_LIVE) != F_LIVE) continue;
      const G2& q = g2[i];
      const double v[14] = {q.du, q.dv, q.dca, q.dcb, q.dcc, q.dop, q.drgb[0], q.drgb[1], q.drgb[2],
                            q.dncam[0], q.dncam[1], q.dncam[2], q.ddist, q.absg};
      for (int c = 0; c < 14; ++c) grads[(size_t)(59 + c) * n + i] = v[c];
    }
    // R19b + R19c: bound on what float32 accumulation (kAccEps * sum_pixels |term_k|) and float32
    // evaluation (ev_k, eval_bound) of the same per-pixel terms can cost each 3D gradient:
    // sum_k |d g3D / d g2D_k| * (kAccEps * abs_k + ev_k), the Jacobian columns being this
    // oracle's own (linear) chain O6 applied to unit 2D gradients
    if (bound) {
      const double kAccEps = 16.0 * 5.9604644775390625e-08;  // 16 ulp(1) of float32
      std::memset(bound, 0, sizeof(double) * (size_t)59 * n);
      std::vector<double> tmp((size_t)59 * n, 0.0);
      for (int i = 0; i < n; ++i) {
        if ((rd.proj[i].flags & F_LIVE) != F_LIVE) continue;
        for (int k = 0; k < 13; ++k) {
          const double d = kAccEps * g2[i].abs[k] + (g_bound_eval ? g2[i].ev[k] : 0.0);
          if (d == 0.0) continue;
          G2 e{0, 0, 0, 0, 0, 0, {0, 0, 0}, {0, 0, 0}, 0, 0, {0}};
          double* ev[13] = {&e.du, &e.dv, &e.dca, &e.dcb, &e.dcc, &e.dop, &e.drgb[0], &e.drgb[1], &e.drgb[2],
                            &e.dncam[0], &e.dncam[1], &e.dncam[2], &e.ddist};
          *ev[k] = 1.0;
          gaussian_backward(P, i, cam, rd.proj[i].flags, e, tmp.data(), tmp.data() + (size_t)3 * n,
                            tmp.data() + (size_t)6 * n, tmp.data() + (size_t)10 * n, tmp.data() + (size_t)11 * n);
          for (int j = 0; j < 59; ++j) bound[(size_t)j * n + i] += std::fabs(tmp[(size_t)j * n + i]) * d;
        }
      }
    }
  }
}

}  // namespace

extern "C" {

void oracle_set_bound_eval(int on) { g_bound_eval = on; }

// O1: tile occupancy counts [TY*TX] and SAT [(TY+1)*(TX+1)].
void oracle_tilemask(const uint8_t* mask, int W, int H, uint32_t* cnt, int32_t* sat) {
  const TileMask tm = make_tilemask(mask, W, H);
  std::memcpy(cnt, tm.cnt.data(), tm.cnt.size() * sizeof(uint32_t));
  std::memcpy(sat, tm.sat.data(), tm.sat.size() * sizeof(int32_t));
}

// O2 in float32 (parity) and float64 (pins).  Interleaved outputs:
// mean2d[n][2], conic_o[n][4], depth[n], rect[n][4], tiles[n], rgb[n][3], ncam[n][3], dist[n], flags[n].
void oracle_project_f32(const float* mean, const float* scale, const float* rot, const float* opac,
                        const float* sh, int n, int deg, const double* cam, int W, int H, const uint8_t* mask,
                        float* mean2d, float* conic_o, float* depth, int32_t* rect, uint32_t* tiles,
                        float* rgb, float* ncam, float* dist, uint32_t* flags) {
  project_all<float>(mean, scale, rot, opac, sh, n, deg, cam, W, H, mask, mean2d, conic_o, depth, rect, tiles,
                     rgb, ncam, dist, flags);
}
void oracle_project_f64(const double* mean, const double* scale, const double* rot, const double* opac,
                        const double* sh, int n, int deg, const double* cam, int W, int H, const uint8_t* mask,
                        double* mean2d, double* conic_o, double* depth, int32_t* rect, uint32_t* tiles,
                        double* rgb, double* ncam, double* dist, uint32_t* flags) {
  project_all<double>(mean, scale, rot, opac, sh, n, deg, cam, W, H, mask, mean2d, conic_o, depth, rect, tiles,
                      rgb, ncam, dist, flags);
}

// O3: (tile, depth bits, id) entries for every live Gaussian and active tile in
// its rect, sorted lexicographically; tile ranges [TX*TY][2].  Returns M, and
// writes only if M <= capacity.  depth: float32 depths from oracle_project_f32.
int64_t oracle_keys(const float* depth, const int32_t* rect, const uint32_t* flags, int n, const uint8_t* mask,
                    int W, int H, int64_t capacity, uint32_t* tile_out, uint32_t* val_out, uint32_t* ranges) {
  const TileMask tm = make_tilemask(mask, W, H);
  struct E { uint32_t tile, bits, id; };
  std::vector<E> ent;
  for (int i = 0; i < n; ++i) {
    if ((flags[i] & F_LIVE) != F_LIVE) continue;
    uint32_t bits;
    std::memcpy(&bits, &depth[i], 4);
    for (int ty = rect[4 * i + 1]; ty <= rect[4 * i + 3]; ++ty)
      for (int tx = rect[4 * i]; tx <= rect[4 * i + 2]; ++tx)
        if (tm.active(tx, ty)) ent.push_back(E{(uint32_t)(ty * tm.TX + tx), bits, (uint32_t)i});
  }
  const int64_t M = (int64_t)ent.size();
  if (M > capacity) return M;
  std::sort(ent.begin(), ent.end(), [](const E& a, const E& b) {
    if (a.tile != b.tile) return a.tile < b.tile;
    if (a.bits != b.bits) return a.bits < b.bits;
    return a.id < b.id;
  });
  const int T = tm.TX * tm.TY;
  for (int t = 0; t < 2 * T; ++t) ranges[t] = 0;
  for (int64_t k = 0; k < M; ++k) {
    tile_out[k] = ent[k].tile;
    val_out[k] = ent[k].id;
    if (k == 0 || ent[k].tile != ent[k - 1].tile) ranges[2 * ent[k].tile] = (uint32_t)k;
    if (k == M - 1 || ent[k].tile != ent[k + 1].tile) ranges[2 * ent[k].tile + 1] = (uint32_t)(k + 1);
  }
  return M;
}

// O4 (+ O5/O6 when upstream && grads): render the listed pixels.
// out[npix][10] = C0 C1 C2 N0 N1 N2 D A Dep T; iout[npix][4] = g, last id, near flag, n_clamped.
// grads (double, 73*n): dmean[3][n] dscale[3][n] drot[4][n] dopac[n] dsh[48][n], then the 2D
// gradients du dv dca dcb dcc dop drgb[3] dncam[3] ddist and absgrad (rows 59..72).
// gsoft[npix]: soft counts (R24); upstream [npix][10] with column 9 = dL/d(soft count).
void oracle_render_f32(const float* mean, const float* scale, const float* rot, const float* opac, const float* sh,
                       int n, int deg, const double* cam, int W, int H, const uint8_t* mask, const double* bg,
                       const int64_t* pix, int npix, float* out, int32_t* iout, double* id_sum, int64_t* evaluated,
                       double* gsoft, int certify, int64_t* cert_bad, const double* upstream, double* grads,
                       double* bound) {
  render_pixels<float>(mean, scale, rot, opac, sh, n, deg, cam, W, H, mask, bg, pix, npix, out, iout, id_sum,
                       evaluated, gsoft, certify, cert_bad, upstream, grads, bound);
}
void oracle_render_f64(const double* mean, const double* scale, const double* rot, const double* opac,
                       const double* sh, int n, int deg, const double* cam, int W, int H, const uint8_t* mask,
                       const double* bg, const int64_t* pix, int npix, double* out, int32_t* iout, double* id_sum,
                       int64_t* evaluated, double* gsoft, int certify, int64_t* cert_bad, const double* upstream,
                       double* grads, double* bound) {
  render_pixels<double>(mean, scale, rot, opac, sh, n, deg, cam, W, H, mask, bg, pix, npix, out, iout, id_sum,
                        evaluated, gsoft, certify, cert_bad, upstream, grads, bound);
}
// The same with O2 in float32 (the key path the CUDA A1 reproduces bit-exactly) and Eq. 1-4, O5,
// O6 in double: the exact rendering of the float32 projection, against which the R19c
// evaluation bound of the float build is checked.
void oracle_render_f64_fproj(const double* mean, const double* scale, const double* rot, const double* opac,
                             const double* sh, int n, int deg, const double* cam, int W, int H,
                             const uint8_t* mask, const double* bg, const int64_t* pix, int npix, double* out,
                             int32_t* iout, double* id_sum, int64_t* evaluated, double* gsoft, int certify,
                             int64_t* cert_bad, const double* upstream, double* grads, double* bound) {
  render_pixels<double>(mean, scale, rot, opac, sh, n, deg, cam, W, H, mask, bg, pix, npix, out, iout, id_sum,
                        evaluated, gsoft, certify, cert_bad, upstream, grads, bound, true);
}

// ---------------------------------------------------- L_GC-load (NEXT-1)
// Eq. 9 weight w_i from the image gradient ("gradient-dependent weight
// nabla I"; R23): gray = 0.299 R + 0.587 G + 0.114 B, 3x3 Sobel with replicated
// borders, |grad| normalised by its mean over the mask pixels, clamped to [0.1, 10]
// (a mean of 0 gives the floor everywhere).  image [3][H][W]; w [H][W] (1 off-mask).
void oracle_gc_weights(const double* image, const uint8_t* mask, int W, int H, double* w) {
  const size_t HW = (size_t)W * H;
  std::vector<double> gray(HW), mag(HW);
  for (size_t p = 0; p < HW; ++p) gray[p] = 0.299 * image[p] + 0.587 * image[HW + p] + 0.114 * image[2 * HW + p];
  auto I = [&](int x, int y) {
    x = std::min(std::max(x, 0), W - 1);
    y = std::min(std::max(y, 0), H - 1);
    return gray[(size_t)y * W + x];
  };
  double sum = 0.0;
  long long cnt = 0;
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      const double gx = (I(x + 1, y - 1) + 2 * I(x + 1, y) + I(x + 1, y + 1)) -
                        (I(x - 1, y - 1) + 2 * I(x - 1, y) + I(x - 1, y + 1));
      const double gy = (I(x - 1, y + 1) + 2 * I(x, y + 1) + I(x + 1, y + 1)) -
                        (I(x - 1, y - 1) + 2 * I(x, y - 1) + I(x + 1, y - 1));
      const size_t p = (size_t)y * W + x;
      mag[p] = std::sqrt(gx * gx + gy * gy);
      if (mask[p]) { sum += mag[p]; ++cnt; }
    }
  const double m = cnt ? sum / (double)cnt : 0.0;
  for (size_t p = 0; p < HW; ++p) {
    if (!mask[p]) { w[p] = 1.0; continue; }
    w[p] = m > 0.0 ? std::min(std::max(mag[p] / m, 0.1), 10.0) : 0.1;
  }
}

// L_GC-load = population std over the listed (mask) pixels of r_i = g_i / w_i (Eq. 9),
// and dL/dg_i = (r_i - mean r) / (N L w_i) (0 where L = 0).  Returns L.
double oracle_gc_load(const double* g, const double* w, int npix, double* mean_out, double* dLdg) {
  if (npix <= 0) { if (mean_out) *mean_out = 0.0; return 0.0; }
  double s = 0.0;
  for (int k = 0; k < npix; ++k) s += g[k] / w[k];
  const double mu = s / npix;
  double v = 0.0;
  for (int k = 0; k < npix; ++k) { const double d = g[k] / w[k] - mu; v += d * d; }
  const double L = std::sqrt(v / npix);
  if (mean_out) *mean_out = mu;
  if (dLdg)
    for (int k = 0; k < npix; ++k) dLdg[k] = L > 0.0 ? (g[k] / w[k] - mu) / (npix * L * w[k]) : 0.0;
  return L;
}

// ------------------------------------------------------ L_ban (NEXT-2)
// Boundary band MB ("extract ... building masked boundaries"; R25):
// dilation(RBM, r) XOR erosion(RBM, r) with a (2r+1)^2 square structuring element,
// zero outside the image (erosion shrinks at the image border).
void oracle_boundary_band(const uint8_t* mask, int W, int H, int r, uint8_t* band) {
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      bool any = false, all = true;
      for (int dy = -r; dy <= r; ++dy)
        for (int dx = -r; dx <= r; ++dx) {
          const int xx = x + dx, yy = y + dy;
          const bool v = xx >= 0 && yy >= 0 && xx < W && yy < H && mask[(size_t)yy * W + xx];
          any = any || v;
          all = all && v;
        }
      band[(size_t)y * W + x] = (uint8_t)(any != all);
    }
}

// Eq. 8 with the normal-from-depth of P:153 ("computed from the depth map
// using four neighboring points"; R26, R27): per mask pixel p with valid unbiased depth
// at its four axis neighbours (all inside the image and the mask, Dep != 0),
// P_k = Dep_k r_k (r = K^-1 (x+.5, y+.5, 1)), c = (P_right - P_left) x (P_down - P_up),
// n_depth = c/|c| flipped to face the camera (n . P_p <= 0 with P_p = Dep_p r_p; P_p only
// decides the sign), n_r = N/|N|.  Weight w = bw on the band inside the mask, 1 elsewhere
// in the mask.  L = sum_p w |n_depth - n_r|^2 / #valid.  Outputs loss[0] = sum, loss[1] =
// #valid; if dN / dDep are given, ADDS lambda * dL/dN and lambda * dL/dDep.
void oracle_ban_loss(const double* camf, int W, int H, const uint8_t* mask, const uint8_t* band, const double* N,
                     const double* Dep, double bw, double lambda, double* loss, double* dN, double* dDep) {
  const double fx = camf[0], fy = camf[1], cx = camf[2], cy = camf[3];
  const size_t HW = (size_t)W * H;
  auto ray = [&](int x, int y, double* r) { r[0] = (x + 0.5 - cx) / fx; r[1] = (y + 0.5 - cy) / fy; r[2] = 1.0; };
  auto ok = [&](int x, int y) {
    return x >= 0 && y >= 0 && x < W && y < H && mask[(size_t)y * W + x] && Dep[(size_t)y * W + x] != 0.0;
  };
  struct Term { int x, y; double e[3], w, c[3], cn, nd[3], nr[3], Nn, s; };
  std::vector<Term> terms;
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      const size_t p = (size_t)y * W + x;
      if (!mask[p] || !ok(x, y) || !ok(x - 1, y) || !ok(x + 1, y) || !ok(x, y - 1) || !ok(x, y + 1)) continue;
      const double Nn = std::sqrt(N[p] * N[p] + N[HW + p] * N[HW + p] + N[2 * HW + p] * N[2 * HW + p]);
      if (!(Nn > 0.0)) continue;
      double rl[3], rr[3], ru[3], rd[3], rp[3];
      ray(x - 1, y, rl); ray(x + 1, y, rr); ray(x, y - 1, ru); ray(x, y + 1, rd); ray(x, y, rp);
      double a[3], b[3];
      for (int k = 0; k < 3; ++k) {
        a[k] = Dep[p + 1] * rr[k] - Dep[p - 1] * rl[k];
        b[k] = Dep[p + W] * rd[k] - Dep[p - W] * ru[k];
      }
      Term t;
      t.x = x; t.y = y;
      t.c[0] = a[1] * b[2] - a[2] * b[1];
      t.c[1] = a[2] * b[0] - a[0] * b[2];
      t.c[2] = a[0] * b[1] - a[1] * b[0];
      t.cn = std::sqrt(t.c[0] * t.c[0] + t.c[1] * t.c[1] + t.c[2] * t.c[2]);
      if (!(t.cn > 0.0)) continue;
      const double facing = (t.c[0] * rp[0] + t.c[1] * rp[1] + t.c[2] * rp[2]) * Dep[p];
      t.s = facing > 0.0 ? -1.0 : 1.0;
      for (int k = 0; k < 3; ++k) {
        t.nd[k] = t.s * t.c[k] / t.cn;
        t.nr[k] = N[k * HW + p] / Nn;
        t.e[k] = t.nd[k] - t.nr[k];
      }
      t.Nn = Nn;
      t.w = band[p] ? bw : 1.0;
      terms.push_back(t);
    }
  double sum = 0.0;
  for (const Term& t : terms) sum += t.w * (t.e[0] * t.e[0] + t.e[1] * t.e[1] + t.e[2] * t.e[2]);
  const double cnt = (double)terms.size();
  loss[0] = sum;
  loss[1] = cnt;
  if (!dN && !dDep) return;
  if (cnt == 0.0) return;
  const double sc = lambda / cnt;
  for (const Term& t : terms) {
    const size_t p = (size_t)t.y * W + t.x;
    double gnd[3], gnr[3];
    for (int k = 0; k < 3; ++k) { gnd[k] = 2.0 * sc * t.w * t.e[k]; gnr[k] = -gnd[k]; }
    if (dN) {  // n_r = N/|N|: dN = (g - n (n.g)) / |N|
      const double d = gnr[0] * t.nr[0] + gnr[1] * t.nr[1] + gnr[2] * t.nr[2];
      for (int k = 0; k < 3; ++k) dN[k * HW + p] += (gnr[k] - t.nr[k] * d) / t.Nn;
    }
    if (dDep) {  // n_d = s c/|c|; c = a x b
      double cu[3];
      for (int k = 0; k < 3; ++k) cu[k] = t.c[k] / t.cn;
      const double d = gnd[0] * cu[0] + gnd[1] * cu[1] + gnd[2] * cu[2];
      double gc[3];
      for (int k = 0; k < 3; ++k) gc[k] = t.s * (gnd[k] - cu[k] * d) / t.cn;
      double rl[3], rr[3], ru[3], rd[3];
      ray(t.x - 1, t.y, rl); ray(t.x + 1, t.y, rr); ray(t.x, t.y - 1, ru); ray(t.x, t.y + 1, rd);
      double a[3], b[3];
      for (int k = 0; k < 3; ++k) {
        a[k] = Dep[p + 1] * rr[k] - Dep[p - 1] * rl[k];
        b[k] = Dep[p + W] * rd[k] - Dep[p - W] * ru[k];
      }
      // d/da (c . g) = b x g ; d/db (c . g) = g x a
      const double ga[3] = {b[1] * gc[2] - b[2] * gc[1], b[2] * gc[0] - b[0] * gc[2], b[0] * gc[1] - b[1] * gc[0]};
      const double gb[3] = {gc[1] * a[2] - gc[2] * a[1], gc[2] * a[0] - gc[0] * a[2], gc[0] * a[1] - gc[1] * a[0]};
      dDep[p + 1] += ga[0] * rr[0] + ga[1] * rr[1] + ga[2] * rr[2];
      dDep[p - 1] -= ga[0] * rl[0] + ga[1] * rl[1] + ga[2] * rl[2];
      dDep[p + W] += gb[0] * rd[0] + gb[1] * rd[1] + gb[2] * rd[2];
      dDep[p - W] -= gb[0] * ru[0] + gb[1] * ru[1] + gb[2] * ru[2];
    }
  }
}

// ------------------------------------------------- L_rgb (NEXT-3)
// Masked photometric loss ("only the refined building masks RBM are involved";
// L_rgb's form is 3DGS's, R28): x = C m, y = I m (zero off the mask), per channel the
// 11x11 Gaussian-window (sigma 1.5, normalised, zero padding) SSIM map of Wang et al.
// with C1 = 0.01^2, C2 = 0.03^2; L1 = mean over mask pixels and channels of |C - I|,
// S = mean over mask pixels and channels of the SSIM map,
// L_rgb = 0.8 L1 + 0.2 (1 - S).  Writes out[0..2] = (L_rgb, L1, S) and, if dC is given,
// dL_rgb/dC (zero off the mask).  Plain window sums: O(121 HW) per statistic.
void oracle_rgb_loss(const double* C, const double* I, const uint8_t* mask, int W, int H, double* out,
                     double* dC) {
  const int R = 5;
  double g1[2 * R + 1], gs = 0.0;
  for (int k = -R; k <= R; ++k) { g1[k + R] = std::exp(-(double)(k * k) / (2.0 * 1.5 * 1.5)); gs += g1[k + R]; }
  for (int k = 0; k <= 2 * R; ++k) g1[k] /= gs;
  const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
  const size_t HW = (size_t)W * H;
  long long npx = 0;
  for (size_t p = 0; p < HW; ++p) npx += mask[p] ? 1 : 0;
  double l1 = 0.0, ssum = 0.0;
  if (dC) std::memset(dC, 0, sizeof(double) * 3 * HW);
  std::vector<double> x(HW), y(HW), mx(HW), my(HW), sxx(HW), syy(HW), sxy(HW), A(HW), B(HW), Cm(HW);
  for (int c = 0; c < 3; ++c) {
    for (size_t p = 0; p < HW; ++p) {
      x[p] = mask[p] ? C[c * HW + p] : 0.0;
      y[p] = mask[p] ? I[c * HW + p] : 0.0;
    }
    // window statistics at every pixel
    for (int j = 0; j < H; ++j)
      for (int i = 0; i < W; ++i) {
        double a = 0, b = 0, xx = 0, yy = 0, xy = 0;
        for (int dj = -R; dj <= R; ++dj)
          for (int di = -R; di <= R; ++di) {
            const int ii = i + di, jj = j + dj;
            if (ii < 0 || jj < 0 || ii >= W || jj >= H) continue;
            const double wgt = g1[di + R] * g1[dj + R];
            const size_t q = (size_t)jj * W + ii;
            a += wgt * x[q]; b += wgt * y[q]; xx += wgt * x[q] * x[q]; yy += wgt * y[q] * y[q];
            xy += wgt * x[q] * y[q];
          }
        const size_t p = (size_t)j * W + i;
        mx[p] = a; my[p] = b; sxx[p] = xx - a * a; syy[p] = yy - b * b; sxy[p] = xy - a * b;
      }
    for (size_t p = 0; p < HW; ++p) {
      A[p] = B[p] = Cm[p] = 0.0;
      if (!mask[p]) continue;
      const double n1 = 2 * mx[p] * my[p] + C1, n2 = 2 * sxy[p] + C2;
      const double d1 = mx[p] * mx[p] + my[p] * my[p] + C1, d2 = sxx[p] + syy[p] + C2;
      const double s = (n1 * n2) / (d1 * d2);
      ssum += s;
      l1 += std::fabs(C[c * HW + p] - I[c * HW + p]);
      // dS/d(mu_x, sigma_x^2, sigma_xy) holding the others fixed; L = ... - 0.2 S / (3 npx)
      const double k = -0.2 / (3.0 * (double)npx);
      const double dmx = s * (2 * my[p] / n1 - 2 * mx[p] / d1);
      const double dsxx = -s / d2;
      const double dsxy = s * 2 / n2;
      A[p] = k * (dmx - 2 * dsxx * mx[p] - dsxy * my[p]);
      B[p] = k * dsxx;
      Cm[p] = k * dsxy;
    }
    if (!dC) continue;
    // dL/dx_q = (G*A)_q + 2 x_q (G*B)_q + y_q (G*C)_q, then x = C m
    for (int j = 0; j < H; ++j)
      for (int i = 0; i < W; ++i) {
        const size_t q = (size_t)j * W + i;
        if (!mask[q]) continue;
        double ga = 0, gb = 0, gc = 0;
        for (int dj = -R; dj <= R; ++dj)
          for (int di = -R; di <= R; ++di) {
            const int ii = i + di, jj = j + dj;
            if (ii < 0 || jj < 0 || ii >= W || jj >= H) continue;
            const double wgt = g1[di + R] * g1[dj + R];
            const size_t p = (size_t)jj * W + ii;
            ga += wgt * A[p]; gb += wgt * B[p]; gc += wgt * Cm[p];
          }
        const double d = C[c * HW + q] - I[c * HW + q];
        dC[c * HW + q] = ga + 2 * x[q] * gb + y[q] * gc + 0.8 / (3.0 * (double)npx) * (d > 0 ? 1.0 : (d < 0 ? -1.0 : 0.0));
      }
  }
  const double L1 = npx ? l1 / (3.0 * (double)npx) : 0.0, S = npx ? ssum / (3.0 * (double)npx) : 1.0;
  out[0] = 0.8 * L1 + 0.2 * (1.0 - S);
  out[1] = L1;
  out[2] = S;
}

// SH basis in double (for the library pin against scipy).
void oracle_sh_basis(double x, double y, double z, double* Y) { sh_basis<double>(x, y, z, Y); }
// log upper bound used by the rect (for the pin that it bounds ln from above).
float oracle_lnup_f32(float y) { return lnup<float>(y); }

}  // extern "C"
