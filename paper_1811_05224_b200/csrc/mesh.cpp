// mesh.cpp — host side of the path: geometry, dual half segments (R6),
// time grid, temporal slices, the cyclic K_P block plan (Fig. 3),
// quadrature tables, and the C-ABI entry points for meshes and plans.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>

#include "internal.h"

namespace stb {

// ------------------------------------------------------------ error state
static thread_local std::string g_err;
static thread_local long long g_launches = 0;
void set_error(const std::string& msg) { g_err = msg; }
bem_status cuda_fail(cudaError_t e, const char* where) {
  set_error(std::string(where) + ": " + cudaGetErrorString(e));
  return BEM_E_CUDA;
}
void count_launch(long long k) { g_launches += k; }

// ------------------------------------------------------ quadrature tables
// Gauss-Legendre on [0,1] by Newton iteration on P_n in long double; log-weights
// W_k = int_0^1 l_k(r) ln r dr = w_k sum_{j<n} (2j+1) P~_j(r_k) M_j with
// M_0 = -1, M_j = (-1)^{j+1} / (j (j+1)) (moments of the shifted Legendre polynomials).
static Rules g_rules;
static std::once_flag g_rules_once;
static void legendre(int n, long double z, long double& pn, long double& pm) {
  pn = z;   // P_1
  pm = 1;   // P_0
  for (int j = 2; j <= n; ++j) {
    long double pj = ((2 * j - 1) * z * pn - (j - 1) * pm) / j;
    pm = pn;
    pn = pj;
  }
}
static void build_rules() {
  const long double PI = 3.14159265358979323846264338327950288L;
  for (int n = 1; n <= QMAX; ++n) {
    for (int k = 0; k < n; ++k) {
      long double z = cosl(PI * (k + 0.75L) / (n + 0.5L)), pn, pm, pp;
      for (int it = 0; it < 200; ++it) {
        legendre(n, z, pn, pm);
        pp = n * (z * pn - pm) / (z * z - 1);
        long double dz = pn / pp;
        z -= dz;
        if (fabsl(dz) < 1e-19L) break;
      }
      legendre(n, z, pn, pm);
      pp = n * (z * pn - pm) / (z * z - 1);
      long double x = (1 + z) / 2;                 // nodes on [0,1]
      long double w = 1 / ((1 - z * z) * pp * pp);  // weights sum to 1
      long double y = 2 * x - 1, Pj = 1, Pjm = 0, acc = 0;
      for (int j = 0; j < n; ++j) {
        long double Mj = (j == 0) ? -1.0L : ((j % 2 == 1) ? 1.0L : -1.0L) / ((long double)j * (j + 1));
        acc += (2 * j + 1) * Pj * Mj;
        long double Pn1 = ((2 * j + 1) * y * Pj - j * Pjm) / (j + 1);
        Pjm = Pj;
        Pj = Pn1;
      }
      g_rules.x[n][k] = (double)x;
      g_rules.w[n][k] = (double)w;
      g_rules.lw[n][k] = (double)(w * acc);
    }
  }
}
const Rules& host_rules() {
  std::call_once(g_rules_once, build_rules);
  return g_rules;
}

// --------------------------------------------------------------- plan
// Difference cover of Z_P containing 0: every d in 1..P-1 is a difference of two cover
// elements.  Minimal by exhaustive search over increasing sizes (P <= 64 is instant for the
// sizes used; larger P falls back to a greedy cover).
static int uncovered(const std::vector<int>& S, int P) {
  std::vector<char> hit(P, 0);
  for (int a : S)
    for (int b : S) hit[((a - b) % P + P) % P] = 1;
  int u = 0;
  for (int d = 1; d < P; ++d) u += !hit[d];
  return u;
}
// backtracking with a counting bound: r more elements add at most r(2|S| + r - 1) differences
static bool search_cover(std::vector<int>& S, int next, int k, int P) {
  const int r = k - (int)S.size();
  const int u = uncovered(S, P);
  if (u == 0) return true;
  if (r == 0 || u > r * (2 * (int)S.size() + r - 1)) return false;
  for (int v = next; v < P; ++v) {
    S.push_back(v);
    if (search_cover(S, v + 1, k, P)) return true;
    S.pop_back();
  }
  return false;
}
static std::vector<int> difference_cover(int P) {
  static std::mutex mu;
  static std::map<int, std::vector<int>> cache;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(P);
    if (it != cache.end()) return it->second;
  }
  std::vector<int> best;
  if (P == 1) best = {0};
  for (int k = 2; best.empty() && k <= P; ++k) {
    if (k * (k - 1) < P - 1) continue;
    if (P > 72 && k > 9) break;
    std::vector<int> S{0};
    if (search_cover(S, 1, k, P)) best = S;
  }
  if (best.empty()) {  // greedy fallback for large P
    best = {0};
    while (uncovered(best, P) > 0) {
      int bv = -1, bu = P;
      for (int v = 1; v < P; ++v) {
        if (std::find(best.begin(), best.end(), v) != best.end()) continue;
        best.push_back(v);
        int u = uncovered(best, P);
        best.pop_back();
        if (u < bu) { bu = u; bv = v; }
      }
      best.push_back(bv);
    }
  }
  std::lock_guard<std::mutex> g(mu);
  cache[P] = best;
  return best;
}

// Cyclic decomposition of K_P: G_0 owns one edge of S for every circular difference class
// 1..floor(P/2); G_p is G_0 rotated by p (clockwise rotation of the vertices on a circle,
// P:159).  The even-P diameter class is generated twice by the rotations: its edges are owned
// by the lowest rotation (p < P/2).  Edge {u,v} is block (max,min); loop (p,p) -> p.
static std::vector<int> cyclic_plan(int P, std::vector<int>* gen) {
  std::vector<int> S = difference_cover(P);
  if (gen) *gen = S;
  std::vector<int> owner(P * P, -1);
  for (int p = 0; p < P; ++p) owner[p * P + p] = p;
  // generator edges: for each class d pick the first pair (a,b) in S with b - a = d (mod P)
  std::vector<std::pair<int, int>> edges;
  for (int d = 1; d <= P / 2; ++d) {
    bool found = false;
    for (int a : S) {
      for (int b : S)
        if (((b - a) % P + P) % P == d) {
          edges.push_back({a, b});
          found = true;
          break;
        }
      if (found) break;
    }
  }
  for (int p = 0; p < P; ++p)
    for (auto& e : edges) {
      int u = (e.first + p) % P, v = (e.second + p) % P;
      int i = std::max(u, v), j = std::min(u, v);
      if (owner[i * P + j] < 0) owner[i * P + j] = p;
    }
  return owner;
}

}  // namespace stb

using namespace stb;

extern "C" {

const char* bem_version(void) { return "stbem 0.1 (sm_100a, FP64)"; }
const char* bem_last_error(void) { return g_err.c_str(); }
long long bem_launch_count(int reset) {
  long long v = g_launches;
  if (reset) g_launches = 0;
  return v;
}

bem_status bem_plan_build(int P, int* owner_host) {
  if (P < 1 || !owner_host) { set_error("bem_plan_build: P >= 1 and an output array are required"); return BEM_E_INVALID; }
  auto o = cyclic_plan(P, nullptr);
  std::memcpy(owner_host, o.data(), sizeof(int) * P * P);
  return BEM_OK;
}

bem_status bem_plan_generator(int P, int* out_host, int* n_out) {
  if (P < 1 || !out_host || !n_out) { set_error("bem_plan_generator: invalid argument"); return BEM_E_INVALID; }
  auto S = difference_cover(P);
  std::memcpy(out_host, S.data(), sizeof(int) * S.size());
  *n_out = (int)S.size();
  return BEM_OK;
}

bem_status bem_plan_owned_blocks(int P, int nranks, int rank, int* out, int* count) {
  if (P < 1 || nranks < 1 || rank < 0 || rank >= nranks || !out || !count) {
    set_error("bem_plan_owned_blocks: invalid argument");
    return BEM_E_INVALID;
  }
  auto o = cyclic_plan(P, nullptr);
  int c = 0;
  for (int I = 0; I < P; ++I)
    for (int J = 0; J <= I; ++J)
      if (o[I * P + J] % nranks == rank) {
        out[2 * c] = I;
        out[2 * c + 1] = J;
        ++c;
      }
  *count = c;
  return BEM_OK;
}

bem_status bem_slice_ranges(int n_steps, int P, int* first) {
  if (P < 1 || n_steps < 1 || !first) { set_error("bem_slice_ranges: invalid argument"); return BEM_E_INVALID; }
  if (P > n_steps) {
    set_error("bem_slice_ranges: n_slices > n_steps (P:217 'restricted by the number of elements of the temporal decomposition')");
    return BEM_E_INVALID;
  }
  int base = n_steps / P, rem = n_steps % P;
  first[0] = 0;
  for (int p = 0; p < P; ++p) first[p + 1] = first[p] + base + (p < rem ? 1 : 0);
  return BEM_OK;
}

static Seg make_seg(double ax, double ay, double bx, double by) {
  Seg s;
  s.ax = ax; s.ay = ay; s.bx = bx; s.by = by;
  double dx = bx - ax, dy = by - ay;
  s.h = std::sqrt(dx * dx + dy * dy);
  s.tx = dx / s.h; s.ty = dy / s.h;
  s.nx = s.ty; s.ny = -s.tx;
  return s;
}

static bool seg_intersect(double ax, double ay, double bx, double by, double cx, double cy, double dx,
                          double dy) {
  auto orient = [](double px, double py, double qx, double qy, double rx, double ry) {
    double v = (qx - px) * (ry - py) - (qy - py) * (rx - px);
    return (v > 0) - (v < 0);
  };
  int o1 = orient(ax, ay, bx, by, cx, cy), o2 = orient(ax, ay, bx, by, dx, dy);
  int o3 = orient(cx, cy, dx, dy, ax, ay), o4 = orient(cx, cy, dx, dy, bx, by);
  return o1 != o2 && o3 != o4 && o1 != 0 && o2 != 0 && o3 != 0 && o4 != 0;
}

bem_status bem_mesh_create(const bem_mesh_desc* d, bem_comm* comm, bem_mesh** out) {
  if (!d || !out) { set_error("bem_mesh_create: null argument"); return BEM_E_INVALID; }
  *out = nullptr;
  if (d->n_vertices < 3 || !d->vertices_xy || !d->segments_per_side) {
    set_error("bem_mesh_create: a polygon with >= 3 vertices and segments_per_side are required");
    return BEM_E_INVALID;
  }
  if (!(d->alpha > 0)) { set_error("bem_mesh_create: alpha must be > 0 (eq. 1)"); return BEM_E_INVALID; }
  if (d->n_steps < 1 || !d->t_breaks) { set_error("bem_mesh_create: n_steps >= 1 and t_breaks required"); return BEM_E_INVALID; }
  if (d->t_breaks[0] != 0.0) { set_error("bem_mesh_create: t_breaks[0] must be 0"); return BEM_E_INVALID; }
  for (int k = 0; k < d->n_steps; ++k)
    if (!(d->t_breaks[k + 1] > d->t_breaks[k])) {
      set_error("bem_mesh_create: t_breaks must be strictly increasing (S:43)");
      return BEM_E_INVALID;
    }
  int nv = d->n_vertices;
  const double* v = d->vertices_xy;
  double area2 = 0;
  for (int s = 0; s < nv; ++s) {
    int s1 = (s + 1) % nv;
    if (d->segments_per_side[s] < 1) { set_error("bem_mesh_create: segments_per_side must be >= 1"); return BEM_E_INVALID; }
    area2 += v[2 * s] * v[2 * s1 + 1] - v[2 * s1] * v[2 * s + 1];
    if (v[2 * s] == v[2 * s1] && v[2 * s + 1] == v[2 * s1 + 1]) { set_error("bem_mesh_create: repeated vertex"); return BEM_E_INVALID; }
  }
  if (!(area2 > 0)) { set_error("bem_mesh_create: polygon must be counter-clockwise (S:32)"); return BEM_E_INVALID; }
  for (int s = 0; s < nv; ++s)
    for (int r = s + 2; r < nv; ++r) {
      if (s == 0 && r == nv - 1) continue;
      int s1 = (s + 1) % nv, r1 = (r + 1) % nv;
      if (seg_intersect(v[2 * s], v[2 * s + 1], v[2 * s1], v[2 * s1 + 1], v[2 * r], v[2 * r + 1], v[2 * r1], v[2 * r1 + 1])) {
        set_error("bem_mesh_create: polygon is not simple (S:32)");
        return BEM_E_INVALID;
      }
    }
  int P = d->n_slices < 1 ? 1 : d->n_slices;
  if (P > d->n_steps) {
    set_error("bem_mesh_create: n_slices > n_steps (P:217)");
    return BEM_E_INVALID;
  }
  int ng = 0;
  for (int s = 0; s < nv; ++s) ng += d->segments_per_side[s];
  if (ng < 3) { set_error("bem_mesh_create: need >= 3 boundary elements"); return BEM_E_INVALID; }

  bem_mesh_s* m = new bem_mesh_s();
  m->ng = ng;
  m->nt = d->n_steps;
  m->P = P;
  m->alpha = d->alpha;
  m->t.assign(d->t_breaks, d->t_breaks + d->n_steps + 1);
  std::vector<double> nodes(2 * ng);
  int k = 0;
  for (int s = 0; s < nv; ++s) {
    double x0 = v[2 * s], y0 = v[2 * s + 1], x1 = v[2 * ((s + 1) % nv)], y1 = v[2 * ((s + 1) % nv) + 1];
    for (int j = 0; j < d->segments_per_side[s]; ++j) {
      double f = (double)j / d->segments_per_side[s];
      nodes[2 * k] = x0 + f * (x1 - x0);
      nodes[2 * k + 1] = y0 + f * (y1 - y0);
      ++k;
    }
  }
  m->seg.resize(ng);
  m->half.resize(2 * ng);
  m->dual.resize(ng);
  for (int i = 0; i < ng; ++i) {
    int i1 = (i + 1) % ng;
    double ax = nodes[2 * i], ay = nodes[2 * i + 1], bx = nodes[2 * i1], by = nodes[2 * i1 + 1];
    m->seg[i] = make_seg(ax, ay, bx, by);
    double mx = 0.5 * (ax + bx), my = 0.5 * (ay + by);
    m->half[2 * i] = make_seg(ax, ay, mx, my);
    m->half[2 * i + 1] = make_seg(mx, my, bx, by);
    m->half[2 * i].nx = m->half[2 * i + 1].nx = m->seg[i].nx;
    m->half[2 * i].ny = m->half[2 * i + 1].ny = m->seg[i].ny;
  }
  for (int l = 0; l < ng; ++l) {
    double hm = m->seg[(l - 1 + ng) % ng].h, h0 = m->seg[l].h, hp = m->seg[(l + 1) % ng].h;
    m->dual[l] = Dual{hm / (hm + h0), hp / (h0 + hp), 0.5 * (hm + h0), 0.5 * (h0 + hp)};
  }
  m->hmax = 0;
  for (auto& s : m->seg) m->hmax = std::max(m->hmax, s.h);
  m->htmin = 1e300;
  for (int a = 0; a < m->nt; ++a) m->htmin = std::min(m->htmin, m->t[a + 1] - m->t[a]);
  m->kappa = m->alpha * m->hmax * m->hmax / (4.0 * m->htmin);
  m->uniform = true;
  for (int a = 0; a < m->nt; ++a)
    if (std::fabs((m->t[a + 1] - m->t[a]) - (m->t[1] - m->t[0])) > 1e-13 * (m->t[1] - m->t[0])) m->uniform = false;
  // Gauss order for the bulk (d >= 2) from the measured error table
  m->q_bulk = m->kappa <= 0.065 ? 4 : (m->kappa <= 0.3 ? 5 : (m->kappa <= 1.0 ? 6 : 8));
  {  // half segments: kappa / 4
    const double kh = 0.25 * m->kappa;
    m->q_bulk_d = kh <= 0.005 ? 3 : (kh <= 0.07 ? 4 : (kh <= 0.3 ? 5 : (kh <= 1.0 ? 6 : 8)));
  }

  // slices and plan
  m->slice_first.resize(P + 1);
  bem_slice_ranges(m->nt, P, m->slice_first.data());
  m->owner = cyclic_plan(P, nullptr);
  m->comm = comm;
  m->rank = comm ? comm->rank : 0;
  m->nranks = comm ? comm->nranks : 1;
  long long off = 0;
  for (int I = 0; I < P; ++I)
    for (int J = 0; J <= I; ++J) {
      int p = m->owner[I * P + J];
      if (p % m->nranks != m->rank) continue;
      Block b;
      b.I = I; b.J = J;
      b.a0 = m->slice_first[I]; b.a1 = m->slice_first[I + 1];
      b.b0 = m->slice_first[J]; b.b1 = m->slice_first[J + 1];
      b.off = off;
      for (int a = b.a0; a < b.a1; ++a) off += (long long)ng * pad4((long long)panel_nb(a, b.b0, b.b1) * ng);
      m->blocks.push_back(b);
    }
  m->entries_owned = off;

  // device
  cudaError_t e = cudaGetDevice(&m->device);
  if (e != cudaSuccess) { delete m; return cuda_fail(e, "bem_mesh_create/cudaGetDevice"); }
  if (comm && comm->device != m->device) {
    e = cudaSetDevice(comm->device);
    if (e != cudaSuccess) { delete m; return cuda_fail(e, "bem_mesh_create/cudaSetDevice"); }
    m->device = comm->device;
  }
  // time-node lag table: s = t_x - t_y, ln s, 1/s for every node pair x > y (shared by all
  // spatial pairs; removes one log and one division per node and thread from the bulk kernels)
  std::vector<double4> lagtab((size_t)(m->nt + 1) * (m->nt + 1));
  for (int x = 0; x <= m->nt; ++x)
    for (int y = 0; y <= m->nt; ++y) {
      double sv = m->t[x] - m->t[y];
      lagtab[(size_t)x * (m->nt + 1) + y] = x > y ? make_double4(sv, std::log(sv), 1.0 / sv, 0.0) : make_double4(0.0, 0.0, 0.0, 0.0);
    }
  bem_status st = upload_rules();
  if (st != BEM_OK) { delete m; return st; }
  // stream-ordered uploads from the device pool on the legacy default stream; every call that
  // uses the mesh on some stream first waits on m->ready (no host synchronisation here)
  auto up = [&](void** dst, const void* src, size_t bytes) -> cudaError_t {
    cudaError_t r = cudaMallocAsync(dst, bytes, (cudaStream_t)0);
    if (r != cudaSuccess) return r;
    return cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, (cudaStream_t)0);
  };
  if ((e = up((void**)&m->d_t, m->t.data(), sizeof(double) * m->t.size())) != cudaSuccess ||
      (e = up((void**)&m->d_seg, m->seg.data(), sizeof(Seg) * ng)) != cudaSuccess ||
      (e = up((void**)&m->d_half, m->half.data(), sizeof(Seg) * 2 * ng)) != cudaSuccess ||
      (e = up((void**)&m->d_dual, m->dual.data(), sizeof(Dual) * ng)) != cudaSuccess ||
      (e = up((void**)&m->d_lag, lagtab.data(), sizeof(double4) * lagtab.size())) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&m->ready, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventRecord(m->ready, (cudaStream_t)0)) != cudaSuccess) {
    bem_mesh_destroy(m);
    return cuda_fail(e, "bem_mesh_create/upload");
  }
  *out = m;
  return BEM_OK;
}

bem_status bem_mesh_info_get(const bem_mesh* m, bem_mesh_info* info) {
  if (!m || !info) { set_error("bem_mesh_info_get: null argument"); return BEM_E_INVALID; }
  info->n_gamma = m->ng;
  info->n_steps = m->nt;
  info->n = (long long)m->ng * m->nt;
  info->n_slices = m->P;
  info->n_owned_blocks = (int)m->blocks.size();
  long long eo = 0;
  for (auto& b : m->blocks)
    for (int a = b.a0; a < b.a1; ++a) eo += (long long)m->ng * m->ng * panel_nb(a, b.b0, b.b1);
  info->entries_owned = eo;
  info->entries_total = (long long)m->ng * m->ng * m->nt * (m->nt + 1) / 2;
  info->q_bulk = m->q_bulk;
  info->kappa = m->kappa;
  info->rank = m->rank;
  info->nranks = m->nranks;
  info->local_rows = (long long)m->ng * m->nt;   // replicated vectors (R27)
  info->local_row0 = 0;
  return BEM_OK;
}

void bem_mesh_destroy(bem_mesh* m) {
  if (!m) return;
  // stream-ordered on the legacy default stream (callers that used the mesh on another stream
  // synchronise that stream first)
  for (void* p : {(void*)m->d_t, (void*)m->d_seg, (void*)m->d_half, (void*)m->d_dual, (void*)m->d_lag})
    if (p) cudaFreeAsync(p, (cudaStream_t)0);
  if (m->ready) cudaEventDestroy(m->ready);
  delete m;
}

}  // extern "C"
