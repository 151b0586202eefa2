// exec.cu — the C ABI (include/stlg.h): node-program compiler and executor.
//
// stlg_compile lowers the formula DAG (formula.py:65-135 node classes,
// flattened by the Python host in topological order) into a schedule of
// entries, one per temporal operator (Eventually / Always / Until) plus a
// pointwise entry for an elementwise root.  Each entry carries its child
// sub-formula(s) as a fused DExpr: every Pred / NormPred / Not / And / Or /
// TRUE below a temporal operator is evaluated inside that operator's load,
// and temporal children are read from their materialised traces ("slots").
// This replaces the recursive evaluator masking.trace_var (masking.py:308-343)
// which materialises one full array per AST node.
//
// stlg_forward runs the entries in order; stlg_backward runs them in reverse,
// each consuming the cotangent of its own output (user cotangent for the
// root, else its slot's accumulated cotangent) — the schedule equivalent of
// tape.backward's reverse topological walk (tape.py:114-134).  Independent
// sub-formulas under the root (no shared slot, channel or smooth binding, e.g.
// the two operands of C3's And) run on two streams with their own scratch:
// most of these kernels are latency-bound and leave the GPU half idle alone.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/stlg.h"
#include "kernels.cuh"

using namespace stlg;

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};  // process-wide: autograd runs backward on its own thread

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

enum EntryKind { E_POINTWISE, E_FG_TIMED, E_FG_UNTIMED, E_FG_SMOOTH, E_UNTIL };

struct HLeaf {
  int kind;
  int src, src2;  // global source ids: [0, n_ch) channels, n_ch + s slots
  float s_in, s_out, c, cx, cy;
  int st1 = 0, st2 = 0;  // first writer of the gradient of src / src2 in backward order
};
struct HExpr {
  std::vector<HLeaf> leaf;
  std::vector<DStep> step;
};
struct Entry {
  int kind;
  float sg;
  int a, b;
  int untimed;
  int smooth_slot;
  HExpr e1, e2;
  int out_slot;  // -1: the caller's trace buffer
  int aux_slot;  // softmax window-LSE buffer, -1 if none
  int table = -1;  // smooth: index of its log2-weight table in the forward workspace
};

bool is_temporal(int op) { return op == STLG_EVENTUALLY || op == STLG_ALWAYS || op == STLG_UNTIL; }
bool is_elementwise(int op) {
  return op == STLG_TRUE || op == STLG_PRED || op == STLG_NOT || op == STLG_AND || op == STLG_OR ||
         op == STLG_NORM_PRED;
}

}  // namespace

struct stlg_plan {
  stlg_cfg cfg;
  int n_ch = 0, n_smooth = 0, n_slots = 0, n_aux = 0, n_tables = 0;
  int root_temporal = 0;
  int n_lanes = 1;         // 2: entries before the last split into two independent lanes
  std::vector<int> lane;   // per entry: 0 (caller's stream) or 1 (side stream); last entry 0
  std::vector<Entry> entries;
  std::vector<int> ch_touched;  // channel referenced by some leaf (else zero-filled on overwrite)
};

namespace stlg {
void count_launch(int n) { g_launches += n; }
}  // namespace stlg

namespace {

// --------------------------------------------------------------------------
// compiler
// --------------------------------------------------------------------------
// an And / Or operand heavier than this many leaves becomes its own pointwise entry
// (2 measured slower on the paper's phi formulas than 7: more passes over memory)
constexpr int PW_MAX_W = 7;

struct Compiler {
  const stlg_node* nodes;
  int n;
  stlg_plan* plan;
  std::vector<int> slot_of;   // temporal / materialised node -> slot
  std::vector<int> weight_;   // leaf weight of elementwise subtrees (memo)

  int new_slot() { return plan->n_slots++; }

  int weight(int i) {
    if (weight_[i] >= 0) return weight_[i];
    const stlg_node& nd = nodes[i];
    int w;
    if (is_temporal(nd.op) || slot_of[i] >= 0) w = 1;
    else if (nd.op == STLG_NORM_PRED) w = 2;
    else if (nd.op == STLG_NOT) w = weight(nd.left);
    else if (nd.op == STLG_AND || nd.op == STLG_OR) w = weight(nd.left) + weight(nd.right);
    else w = 1;
    weight_[i] = w;
    return w;
  }

  // an elementwise sub-formula with at least one And / Or (through any Nots)
  bool compound(int i) {
    while (nodes[i].op == STLG_NOT && slot_of[i] < 0) i = nodes[i].left;
    return slot_of[i] < 0 && (nodes[i].op == STLG_AND || nodes[i].op == STLG_OR);
  }

  // Materialise an elementwise sub-formula into its own slot (pointwise entry).
  int materialise(int i) {
    if (slot_of[i] >= 0) return slot_of[i];
    Entry e{};
    e.kind = E_POINTWISE;
    e.sg = 1.f;
    e.aux_slot = -1;
    build(i, 1.f, e.e1);
    e.out_slot = new_slot();
    slot_of[i] = e.out_slot;
    plan->entries.push_back(e);
    weight_.assign(n, -1);
    return e.out_slot;
  }

  int push_leaf(HExpr& ex, const HLeaf& lf) {
    ex.leaf.push_back(lf);
    DStep s{(unsigned char)ST_LEAF, (unsigned char)(ex.leaf.size() - 1), 0, 0};
    ex.step.push_back(s);
    return (int)ex.step.size() - 1;
  }

  // Build node i scaled by `sign` (+1 / -1) into ex; returns the SSA step index.
  int build(int i, float sign, HExpr& ex) {
    const stlg_node& nd = nodes[i];
    const float top = (float)plan->cfg.top_value;
    if (slot_of[i] >= 0) {
      HLeaf lf{LEAF_SRC, plan->n_ch + slot_of[i], 0, 1.f, sign, 0.f, 0.f, 0.f};
      return push_leaf(ex, lf);
    }
    switch (nd.op) {
      case STLG_TRUE: {
        HLeaf lf{LEAF_CONST, 0, 0, 1.f, 1.f, sign * top, 0.f, 0.f};
        return push_leaf(ex, lf);
      }
      case STLG_PRED:
      case STLG_NORM_PRED: {
        float thr = (float)nd.threshold;
        // '>' : x + (-c)    '<' : (-x) + c     (masking.py:319-323)
        HLeaf lf{nd.op == STLG_PRED ? LEAF_AFFINE : LEAF_NORM, nd.chan,
                 nd.op == STLG_PRED ? 0 : nd.chan2, nd.cmp == 0 ? 1.f : -1.f, sign,
                 nd.cmp == 0 ? -thr : thr, (float)nd.center0, (float)nd.center1};
        return push_leaf(ex, lf);
      }
      case STLG_NOT:
        return build(nd.left, -sign, ex);
      case STLG_AND:
      case STLG_OR: {
        // sign * min(l, r) == max(-l, -r) exactly (the reference's min is -max(-x))
        bool is_min = (nd.op == STLG_AND) == (sign > 0);
        int ka, kb;
        int l = nd.left, r = nd.right;
        if (is_elementwise(nodes[l].op) && slot_of[l] < 0 && weight(l) > PW_MAX_W) materialise(l);
        if (is_elementwise(nodes[r].op) && slot_of[r] < 0 && weight(r) > PW_MAX_W) materialise(r);
        ka = build(l, sign, ex);
        kb = build(r, sign, ex);
        DStep s{(unsigned char)(is_min ? ST_MIN : ST_MAX), (unsigned char)ka, (unsigned char)kb, 0};
        ex.step.push_back(s);
        return (int)ex.step.size() - 1;
      }
      default:
        return -1;  // temporal without a slot: impossible after ordering
    }
  }

  bool fits(const HExpr& ex) {
    if ((int)ex.leaf.size() > MAX_LEAF || (int)ex.step.size() > MAX_STEP) return false;
    std::vector<int> srcs;
    for (auto& lf : ex.leaf) {
      if (lf.kind == LEAF_CONST) continue;
      srcs.push_back(lf.src);
      if (lf.kind == LEAF_NORM) srcs.push_back(lf.src2);
    }
    std::sort(srcs.begin(), srcs.end());
    srcs.erase(std::unique(srcs.begin(), srcs.end()), srcs.end());
    return (int)srcs.size() <= MAX_SRC;
  }
};

// Backward runs the entries in reverse; inside a kernel the left expression's
// VJP runs before the right one's, and a generic expression visits its leaves
// in reverse step order.  The first leaf (in that order) to write a gradient
// destination stores; later ones accumulate.  Every VJP kernel writes every
// element of its destinations, so stored buffers need no zero-fill.
void mark_first_writers(stlg_plan* plan) {
  std::map<int, bool> touched;
  auto visit = [&](HExpr& ex) {
    for (int k = (int)ex.step.size() - 1; k >= 0; --k) {
      if (ex.step[k].op != ST_LEAF) continue;
      HLeaf& lf = ex.leaf[ex.step[k].a];
      if (lf.kind == LEAF_CONST) continue;
      lf.st1 = touched[lf.src] ? 0 : 1;
      touched[lf.src] = true;
      if (lf.kind == LEAF_NORM) {
        lf.st2 = touched[lf.src2] ? 0 : 1;
        touched[lf.src2] = true;
      }
    }
  };
  for (auto it = plan->entries.rbegin(); it != plan->entries.rend(); ++it) {
    visit(it->e1);
    if (it->kind == E_UNTIL) visit(it->e2);
  }
  plan->ch_touched.assign(plan->n_ch, 0);
  for (auto& kv : touched)
    if (kv.first < plan->n_ch) plan->ch_touched[kv.first] = 1;
}

// Lanes: the entries before the last one (the root, which joins everything) fall into
// connected components under "reads the other's slot", "touches the same channel" and
// "shares a smooth binding" — components share no buffer the backward writes (channel
// gradients, slot cotangents, d(a,b,c)), so they may run concurrently.  Two or more
// components are dealt to two lanes, heaviest first (an Until entry counts 4).
void assign_lanes(stlg_plan* plan) {
  const int n = (int)plan->entries.size();
  plan->lane.assign(n, 0);
  plan->n_lanes = 1;
  if (n < 3) return;
  std::vector<int> par(n - 1);
  for (int i = 0; i < n - 1; ++i) par[i] = i;
  auto find = [&](int x) {
    while (par[x] != x) x = par[x] = par[par[x]];
    return x;
  };
  auto unite = [&](int a, int b) { par[find(a)] = find(b); };
  std::vector<int> producer(plan->n_slots, -1);
  for (int i = 0; i < n - 1; ++i)
    if (plan->entries[i].out_slot >= 0) producer[plan->entries[i].out_slot] = i;
  std::map<int, int> ch_user, smooth_user;
  auto touch = [&](int i, int src) {
    if (src < plan->n_ch) {
      auto it = ch_user.find(src);
      if (it == ch_user.end()) ch_user[src] = i;
      else unite(i, it->second);
    } else if (src - plan->n_ch < plan->n_slots && producer[src - plan->n_ch] >= 0) {
      unite(i, producer[src - plan->n_ch]);
    }
  };
  auto visit = [&](int i, const HExpr& ex) {
    for (const HLeaf& lf : ex.leaf) {
      if (lf.kind == LEAF_CONST) continue;
      touch(i, lf.src);
      if (lf.kind == LEAF_NORM) touch(i, lf.src2);
    }
  };
  for (int i = 0; i < n - 1; ++i) {
    const Entry& e = plan->entries[i];
    visit(i, e.e1);
    if (e.kind == E_UNTIL) visit(i, e.e2);
    if (e.kind == E_FG_SMOOTH) {
      auto it = smooth_user.find(e.smooth_slot);
      if (it == smooth_user.end()) smooth_user[e.smooth_slot] = i;
      else unite(i, it->second);
    }
  }
  std::map<int, int> cost;  // component root -> weight
  for (int i = 0; i < n - 1; ++i) cost[find(i)] += plan->entries[i].kind == E_UNTIL ? 4 : 1;
  if (cost.size() < 2) return;
  std::vector<std::pair<int, int>> comps;  // (weight, root)
  for (auto& kv : cost) comps.push_back({kv.second, kv.first});
  std::sort(comps.begin(), comps.end(), [](const std::pair<int, int>& x, const std::pair<int, int>& y) {
    return x.first != y.first ? x.first > y.first : x.second < y.second;
  });
  int load[2] = {0, 0};
  std::map<int, int> lane_of;
  for (auto& c : comps) {
    const int l = load[1] < load[0] ? 1 : 0;
    lane_of[c.second] = l;
    load[l] += c.first;
  }
  for (int i = 0; i < n - 1; ++i) plan->lane[i] = lane_of[find(i)];
  plan->n_lanes = 2;
}

int validate_nodes(const stlg_node* nodes, int n, int n_ch, int n_smooth) {
  if (n <= 0) return fail(STLG_E_INVALID, "empty node program");
  for (int i = 0; i < n; ++i) {
    const stlg_node& nd = nodes[i];
    auto child_ok = [&](int c) { return c >= 0 && c < i; };
    switch (nd.op) {
      case STLG_TRUE:
        break;
      case STLG_PRED:
        if (nd.chan < 0 || nd.chan >= n_ch) return fail(STLG_E_INVALID, "pred channel out of range");
        break;
      case STLG_NORM_PRED:
        if (nd.chan < 0 || nd.chan >= n_ch || nd.chan2 < 0 || nd.chan2 >= n_ch)
          return fail(STLG_E_INVALID, "norm channel out of range");
        break;
      case STLG_NOT:
        if (!child_ok(nd.left)) return fail(STLG_E_INVALID, "bad child index");
        break;
      case STLG_AND:
      case STLG_OR:
        if (!child_ok(nd.left) || !child_ok(nd.right)) return fail(STLG_E_INVALID, "bad child index");
        break;
      case STLG_EVENTUALLY:
      case STLG_ALWAYS:
      case STLG_UNTIL:
        if (!child_ok(nd.left)) return fail(STLG_E_INVALID, "bad child index");
        if (nd.op == STLG_UNTIL && !child_ok(nd.right)) return fail(STLG_E_INVALID, "bad child index");
        if (nd.itv_kind == STLG_ITV_STEP) {
          if (nd.a < 0 || nd.b < nd.a) return fail(STLG_E_INVALID, "need 0 <= a <= b");
        } else if (nd.itv_kind == STLG_ITV_SMOOTH) {
          if (nd.op == STLG_UNTIL)
            return fail(STLG_E_UNSUPPORTED, "until does not support smooth intervals");
          if (nd.smooth_slot < 0 || nd.smooth_slot >= n_smooth)
            return fail(STLG_E_INVALID, "smooth slot out of range");
        } else if (nd.itv_kind != STLG_ITV_NONE) {
          return fail(STLG_E_INVALID, "bad interval kind");
        }
        break;
      default:
        return fail(STLG_E_INVALID, "unknown opcode");
    }
  }
  return STLG_OK;
}

// --------------------------------------------------------------------------
// executor helpers
// --------------------------------------------------------------------------
struct Bufs {
  float* slots;   // n_slots * B * T
  float* aux;     // n_aux * B * T
  float* tables;  // n_tables * 2T (log2 smooth weights, log2 suffix sums)
  float* gslots;  // n_slots * B * T (backward)
  float* scratch; // 3 * B * T (backward)
  double* dw64;    // [T] d out / d w_i (smooth backward)
  double* dwpart;  // [smooth_dw_parts(B), T] its per-row-tile partials
  unsigned long long* dacc;  // [4][B, T] reproducible Until accumulators
  int* dscale;               // [B] their per-row grid exponents
  float* uslab;   // Until backward checkpoint slab (persistent kernel)
  unsigned* lb;   // look-back slots of the multi-CTA untimed scans (forward: 1, backward: 2 rows)
  long long BT;
  float* slot(int s) const { return slots + (long long)s * BT; }
  float* gslot(int s) const { return gslots + (long long)s * BT; }
  float* auxp(int s) const { return aux + (long long)s * BT; }
};

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

void fwd_layout(const stlg_plan* p, long long BT, size_t* slots_b, size_t* aux_b) {
  *slots_b = align256(sizeof(float) * (size_t)p->n_slots * BT);
  *aux_b = align256(sizeof(float) * (size_t)p->n_aux * BT);
}
size_t tables_bytes(const stlg_plan* p, long long T) {
  return align256(sizeof(float) * 2 * (size_t)p->n_tables * (size_t)T);
}

// Smooth-interval weights on the host in fp64, exactly as the reference forms
// them (smoothing.py:85-97 / masking.py:300-305); returns the kept range.
double sigmoid_h(double z) {
  if (z >= 0) return 1.0 / (1.0 + std::exp(-z));
  double ez = std::exp(z);
  return ez / (1.0 + ez);
}
// lw2[i] = log2 w_i (i < L), then lw2[L + m] = log2 sum_{i >= max(m, i_lo)} w_i, the
// suffix sums the backward's padded-tail term uses (one O(T) pass per row instead of
// a window loop per virtual pad position)
// kept range {i : w_i > 0} of a smooth interval (host fp64; the table itself is built on
// the device by k_smooth_table, smooth.cu); false: every weight is zero
bool smooth_range(const stlg_smooth& sp, long long L, int* i_lo, int* i_hi) {
  int lo = -1, hi = -1;
  const double Lf = (double)L;
  for (long long i = 0; i < L; ++i) {
    double a = sigmoid_h(((double)i - sp.a * Lf) * sp.c);
    double b = sigmoid_h(((double)i - sp.b * Lf) * sp.c);
    if (a - b - sp.eps > 0) {
      if (lo < 0) lo = (int)i;
      hi = (int)i;
    }
  }
  *i_lo = lo;
  *i_hi = hi;
  return lo >= 0;
}

int resolve(const stlg_plan* p, const HExpr& h, const stlg_channel* ch, const stlg_grad* dch,
            const Bufs& bf, long long T, bool with_dst, DExpr& d) {
  std::memset(&d, 0, sizeof(d));
  std::map<int, int> local;
  auto map_src = [&](int gid) -> int {
    auto it = local.find(gid);
    if (it != local.end()) return it->second;
    int k = (int)local.size();
    if (k >= MAX_SRC) return -1;
    local[gid] = k;
    if (gid < p->n_ch) {
      d.src[k] = {ch[gid].ptr, ch[gid].row_stride, ch[gid].elem_stride};
      if (with_dst && dch != nullptr && dch[gid].ptr != nullptr)
        d.dst[k] = {dch[gid].ptr, dch[gid].row_stride, dch[gid].elem_stride};
      else
        d.dst[k] = {nullptr, 0, 0};
    } else {
      int s = gid - p->n_ch;
      d.src[k] = {bf.slot(s), T, 1};
      d.dst[k] = with_dst ? DDst{bf.gslot(s), T, 1} : DDst{nullptr, 0, 0};
    }
    return k;
  };
  if ((int)h.leaf.size() > MAX_LEAF || (int)h.step.size() > MAX_STEP)
    return fail(STLG_E_INVALID, "expression too large");
  for (size_t i = 0; i < h.leaf.size(); ++i) {
    const HLeaf& lf = h.leaf[i];
    DLeaf& o = d.leaf[i];
    o.kind = lf.kind;
    o.s_in = lf.s_in;
    o.s_out = lf.s_out;
    o.c = lf.c;
    o.cx = lf.cx;
    o.cy = lf.cy;
    auto may_store = [&](int gid) {
      if (gid >= p->n_ch) return true;  // slot cotangents: owned by the library
      return dch != nullptr && dch[gid].ptr != nullptr && dch[gid].accumulate == 0;
    };
    o.st1 = (with_dst && lf.kind != LEAF_CONST && lf.st1 && may_store(lf.src)) ? 1 : 0;
    o.st2 = (with_dst && lf.kind == LEAF_NORM && lf.st2 && may_store(lf.src2)) ? 1 : 0;
    if (lf.kind != LEAF_CONST) {
      o.src = map_src(lf.src);
      if (o.src < 0) return fail(STLG_E_INVALID, "too many sources");
      if (lf.kind == LEAF_NORM) {
        o.src2 = map_src(lf.src2);
        if (o.src2 < 0) return fail(STLG_E_INVALID, "too many sources");
      }
    }
  }
  for (size_t k = 0; k < h.step.size(); ++k) d.step[k] = h.step[k];
  d.n_step = (int)h.step.size();
  d.n_leaf = (int)h.leaf.size();
  d.n_src = (int)local.size();
  return STLG_OK;
}

ModeP mode_params(const stlg_cfg& c) {
  ModeP m;
  double tau = c.mode == STLG_MODE_HARD ? 1.0 : c.temp;
  m.tau = (float)tau;
  m.tau2 = (float)(tau * 1.4426950408889634);
  m.inv_tau2 = (float)(1.0 / (tau * 1.4426950408889634));
  return m;
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return STLG_OK;
  return fail(STLG_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

// ==========================================================================
// C ABI
// ==========================================================================
extern "C" {

int stlg_abi_version(void) { return STLG_ABI_VERSION; }

const char* stlg_last_error(void) { return g_err.c_str(); }

int stlg_mining_grid(const float* data, int64_t n, int64_t length, int64_t row_stride, const double* a,
                     const double* b, int64_t npairs, double sharp, double eps, int32_t mode, double temp,
                     double gamma, double* loss_out, double* dloss_out, void* stream) {
  if (!data || !a || !b || !loss_out) return fail(STLG_E_INVALID, "null argument");
  if (n <= 0 || length <= 0) return fail(STLG_E_SHAPE, "dataset must be a non-empty (n, length) array");
  if (npairs < 0) return fail(STLG_E_INVALID, "negative pair count");
  if (mode != STLG_MODE_HARD && !(temp > 0)) return fail(STLG_E_INVALID, "temperature must be positive");
  if ((size_t)3 * length * sizeof(float) > 220 * 1024)
    return fail(STLG_E_UNSUPPORTED, "mining rows longer than 18000 samples");
  const int m = mode == STLG_MODE_HARD ? M_HARD : (mode == STLG_MODE_LSE ? M_LSE : M_SOFT);
  cudaError_t ce = launch_mining_grid(m, data, n, (int)length, row_stride, a, b, npairs, sharp, eps,
                                      (float)temp, gamma, loss_out, dloss_out, (cudaStream_t)stream);
  return cuda_status(ce, "mining launch");
}

int64_t stlg_launch_count(int reset) {
  return reset ? g_launches.exchange(0) : g_launches.load();
}

int stlg_compile(const stlg_node* nodes, int32_t n_nodes, int32_t n_channels, int32_t n_smooth,
                 const stlg_cfg* cfg, stlg_plan** out_plan) {
  if (!nodes || !cfg || !out_plan) return fail(STLG_E_INVALID, "null argument");
  *out_plan = nullptr;
  if (n_channels < 0 || n_smooth < 0) return fail(STLG_E_INVALID, "negative counts");
  if (cfg->mode < 0 || cfg->mode > 2) return fail(STLG_E_UNSUPPORTED, "unsupported mode");
  if (cfg->mode != STLG_MODE_HARD && !(cfg->temp > 0)) return fail(STLG_E_INVALID, "temp <= 0");
  int rc = validate_nodes(nodes, n_nodes, n_channels, n_smooth);
  if (rc != STLG_OK) return rc;

  stlg_plan* plan = new stlg_plan();
  plan->cfg = *cfg;
  plan->n_ch = n_channels;
  plan->n_smooth = n_smooth;
  Compiler C{nodes, n_nodes, plan, std::vector<int>(n_nodes, -1), std::vector<int>(n_nodes, -1)};
  const int root = n_nodes - 1;
  for (int i = 0; i < n_nodes; ++i) {
    const stlg_node& nd = nodes[i];
    if (!is_temporal(nd.op)) continue;
    Entry e{};
    e.sg = (nd.op == STLG_ALWAYS) ? -1.f : 1.f;
    e.a = nd.a;
    e.b = nd.b;
    e.untimed = nd.itv_kind == STLG_ITV_NONE;
    e.smooth_slot = nd.smooth_slot;
    e.aux_slot = -1;
    if (nd.op == STLG_UNTIL) {
      e.kind = E_UNTIL;
    } else if (nd.itv_kind == STLG_ITV_SMOOTH) {
      e.kind = E_FG_SMOOTH;
      e.table = plan->n_tables++;
    } else {
      e.kind = e.untimed ? E_FG_UNTIMED : E_FG_TIMED;
    }
    // a compound child (an And / Or of predicates) runs as its own register-resident
    // pointwise entry: the window / Until kernels then read a materialised trace through
    // their single-leaf fast paths instead of interpreting the expression per staged
    // sample (the generic interpreter's step array lives in local memory)
    if (C.compound(nd.left)) C.materialise(nd.left);
    if (nd.op == STLG_UNTIL && C.compound(nd.right)) C.materialise(nd.right);
    C.build(nd.left, 1.f, e.e1);
    if (nd.op == STLG_UNTIL) C.build(nd.right, 1.f, e.e2);
    if (!C.fits(e.e1) || (nd.op == STLG_UNTIL && !C.fits(e.e2))) {
      delete plan;
      return fail(STLG_E_UNSUPPORTED, "sub-formula too large for one fused expression");
    }
    // softmax: the window LSE L_t; LSE timed F / G: the low word of the double-float
    // trace (hi = fp32 trace, lo = residual), so the backward's softmax weights
    // 2^{tau2 (u - M)} do not inherit the fp32 rounding of M amplified by tau
    if ((cfg->mode == STLG_MODE_SOFTMAX &&
         (e.kind == E_FG_TIMED || e.kind == E_FG_UNTIMED || e.kind == E_FG_SMOOTH)) ||
        (cfg->mode == STLG_MODE_LSE && e.kind == E_FG_TIMED) ||
        (cfg->mode == STLG_MODE_LSE && e.kind == E_FG_UNTIMED && !cfg->masked_fill))
      e.aux_slot = plan->n_aux++;
    // hard timed windows on the chunk-aligned kernels (17 <= K <= 1024): every window's first
    // arg-max, so the backward routes cotangents without recomputing the windows
    if (cfg->mode == STLG_MODE_HARD && e.kind == E_FG_TIMED && !cfg->masked_fill &&
        e.b - e.a + 1 >= 17 && e.b - e.a + 1 <= 1024)
      e.aux_slot = plan->n_aux++;
    // hard timed Until on the O(T) kernels: every output's gradient source (uint16 plane),
    // so the backward routes cotangents without restaging the children or re-walking blocks
    // (offsets <= b < 0x7fff: a right-child offset never reaches the 0xffff overrun mark)
    if (cfg->mode == STLG_MODE_HARD && e.kind == E_UNTIL && !e.untimed && !cfg->masked_fill &&
        e.b < 0x7fff)
      e.aux_slot = plan->n_aux++;
    // softmax smooth intervals: [L_hi | M_lo | L_lo] (double-float window LSE and mean)
    if (cfg->mode == STLG_MODE_SOFTMAX && e.kind == E_FG_SMOOTH) plan->n_aux += 2;
    e.out_slot = (i == root) ? -1 : C.new_slot();
    C.slot_of[i] = e.out_slot;
    plan->entries.push_back(e);
  }
  if (is_temporal(nodes[root].op)) {
    plan->root_temporal = 1;
  } else {
    Entry e{};
    e.kind = E_POINTWISE;
    e.sg = 1.f;
    e.aux_slot = -1;
    C.build(root, 1.f, e.e1);
    if (!C.fits(e.e1)) {
      delete plan;
      return fail(STLG_E_UNSUPPORTED, "root formula too large for one fused expression");
    }
    e.out_slot = -1;
    plan->entries.push_back(e);
  }
  mark_first_writers(plan);
  assign_lanes(plan);
  *out_plan = plan;
  return STLG_OK;
}

void stlg_free(stlg_plan* plan) { delete plan; }

int stlg_plan_info(const stlg_plan* plan, int32_t* n_temporal, int32_t* n_slots,
                   int32_t* root_is_temporal) {
  if (!plan) return fail(STLG_E_INVALID, "null plan");
  int nt = 0;
  for (auto& e : plan->entries) nt += e.kind != E_POINTWISE;
  if (n_temporal) *n_temporal = nt;
  if (n_slots) *n_slots = plan->n_slots;
  if (root_is_temporal) *root_is_temporal = plan->root_temporal;
  return STLG_OK;
}

// per-thread checkpoint slab of the persistent Until backward (largest Until entry)
static size_t until_slab_bytes(const stlg_plan* plan, long long T) {
  size_t m = 0;
  for (const Entry& e : plan->entries)
    if (e.kind == E_UNTIL) {
      size_t s = until_bwd_scratch_bytes(plan->cfg.mode, e.untimed, plan->cfg.masked_fill, T,
                                         e.untimed ? 0 : e.b, e.untimed ? (int)T : e.b - e.a + 1);
      if (s > m) m = s;
    }
  return align256(m);
}

// d/dw region of the backward workspace: dw64 [T] plus, for plans with a smooth interval,
// the per-row-tile partials [smooth_dw_parts(B), T] of the deterministic d/dw pass
static size_t dw_bytes(const stlg_plan* plan, long long B, long long T) {
  size_t b = align256(sizeof(double) * (size_t)T);
  if (plan->n_tables > 0) b += align256(sizeof(double) * (size_t)smooth_dw_parts(B) * (size_t)T);
  return b;
}

// reproducible Until accumulators (detacc.cuh): 4 int64 planes [B, T] + per-row exponents
static bool plan_has_until(const stlg_plan* plan) {
  for (const Entry& e : plan->entries)
    if (e.kind == E_UNTIL) return true;
  return false;
}
static size_t det_bytes(const stlg_plan* plan, long long B, long long T) {
  if (!plan_has_until(plan)) return 0;
  return align256(sizeof(unsigned long long) * 4 * (size_t)B * (size_t)T) + align256(sizeof(int) * (size_t)B);
}

// per-lane backward scratch: [scratch 3BT | dw64 (+ partials) | dacc, dscale | 256 | Until
// slab | look-back slots (2 rows)]; lane 1 (plans with independent sub-formulas) gets a copy
static size_t bwd_lane_bytes(const stlg_plan* plan, long long B, long long T) {
  return align256(sizeof(float) * 3 * (size_t)B * (size_t)T) + dw_bytes(plan, B, T) + det_bytes(plan, B, T) +
         256 + until_slab_bytes(plan, T) + align256(2 * lb_slot_bytes(B, T));
}

int stlg_workspace_bytes(const stlg_plan* plan, int64_t B, int64_t T, size_t* fwd_bytes,
                         size_t* bwd_bytes) {
  if (!plan) return fail(STLG_E_INVALID, "null plan");
  if (B <= 0 || T <= 0) return fail(STLG_E_SHAPE, "empty signal batch");
  long long BT = (long long)B * T;
  size_t sb, ab;
  fwd_layout(plan, BT, &sb, &ab);
  if (fwd_bytes)
    *fwd_bytes = sb + ab + tables_bytes(plan, T) + plan->n_lanes * align256(lb_slot_bytes(B, T)) + 256;
  if (bwd_bytes)
    *bwd_bytes = align256(sizeof(float) * (size_t)plan->n_slots * BT) + plan->n_lanes * bwd_lane_bytes(plan, B, T) +
                 1024;
  return STLG_OK;
}

static int setup_bufs(const stlg_plan* plan, int64_t B, int64_t T, void* fwd_ws, size_t fwd_bytes,
                      void* bwd_ws, size_t bwd_bytes, Bufs& bf, int lane = 0) {
  long long BT = (long long)B * T;
  size_t need_f, need_b;
  stlg_workspace_bytes(plan, B, T, &need_f, &need_b);
  if (fwd_bytes < need_f) return fail(STLG_E_INVALID, "forward workspace too small");
  size_t sb, ab;
  fwd_layout(plan, BT, &sb, &ab);
  uintptr_t base = ((uintptr_t)fwd_ws + 255) & ~(uintptr_t)255;
  bf.BT = BT;
  bf.slots = (float*)base;
  bf.aux = (float*)(base + sb);
  bf.tables = (float*)(base + sb + ab);
  bf.lb = (unsigned*)(base + sb + ab + tables_bytes(plan, T) + lane * align256(lb_slot_bytes(B, T)));
  bf.gslots = nullptr;
  bf.scratch = nullptr;
  bf.uslab = nullptr;
  bf.dw64 = bf.dwpart = nullptr;
  bf.dacc = nullptr;
  bf.dscale = nullptr;
  if (bwd_ws) {
    if (bwd_bytes < need_b) return fail(STLG_E_INVALID, "backward workspace too small");
    uintptr_t bb = ((uintptr_t)bwd_ws + 255) & ~(uintptr_t)255;
    bf.gslots = (float*)bb;
    bf.scratch = (float*)(bb + align256(sizeof(float) * (size_t)plan->n_slots * BT) +
                          lane * bwd_lane_bytes(plan, B, T));
    bf.dw64 = (double*)((uintptr_t)bf.scratch + align256(sizeof(float) * 3 * (size_t)BT));
    bf.dwpart = bf.dw64 + align256(sizeof(double) * (size_t)T) / sizeof(double);
    uintptr_t dp = (uintptr_t)bf.dw64 + dw_bytes(plan, B, T);
    if (plan_has_until(plan)) {
      bf.dacc = (unsigned long long*)dp;
      bf.dscale = (int*)(dp + align256(sizeof(unsigned long long) * 4 * (size_t)BT));
    }
    bf.uslab = (float*)(dp + det_bytes(plan, B, T) + 256);
    bf.lb = (unsigned*)((uintptr_t)bf.uslab + until_slab_bytes(plan, T));
  }
  return STLG_OK;
}

static void fill_fg(const stlg_plan* plan, const Entry& e, int64_t B, int64_t T, FGParams& p) {
  std::memset(&p, 0, sizeof(p));
  p.B = B;
  p.L = T;
  p.a = e.a;
  p.b = e.b;
  p.K = e.b - e.a + 1;
  p.sg = e.sg;
  p.pad_last = plan->cfg.pad_last;
  p.pad_value = (float)plan->cfg.pad_value;
  p.canon = (!e.untimed && e.b > 0 && (long long)T - e.b > 0) ? 1 : 0;
  p.mp = mode_params(plan->cfg);
  p.sent = (float)plan->cfg.sentinel;
  if (plan->cfg.masked_fill && (e.kind == E_FG_TIMED || e.kind == E_FG_UNTIMED)) {
    // sentinel-filled columns over the b-padded child, no overrun rule (masking.py:229-232)
    p.fill = 1;
    p.canon = 0;
    if (e.kind == E_FG_TIMED) p.padmode = 1;
  }
}

// Smooth-interval F / G: hard mode is the vHGW window kernel over the kept
// range with padded-window semantics; LSE / softmax use smooth.cu.
static int run_smooth(const stlg_plan* plan, const Entry& e, const stlg_channel* channels,
                      const stlg_grad* d_channels, int64_t B, int64_t T,
                      const stlg_smooth* smooth_params, const Bufs& bf, float* out,
                      const float* out_in, const float* cot, double* d_smooth, double* dw64,
                      cudaStream_t st, bool backward) {
  if (!smooth_params) return fail(STLG_E_INVALID, "smooth parameters required");
  const stlg_smooth& sp = smooth_params[e.smooth_slot];
  int i_lo, i_hi;
  if (!smooth_range(sp, T, &i_lo, &i_hi))
    return fail(STLG_E_EMPTY_WINDOW, "smooth interval produced an all-zero weight vector");
  float* tab = bf.tables + (size_t)e.table * 2 * (size_t)T;
  cudaError_t ce = cudaSuccess;
  int rc;
  // the forward builds the table in its workspace; the backward (same workspace and
  // parameters) reads it
  if (!backward) {
    ce = launch_smooth_table(sp.a, sp.b, sp.c, sp.eps, T, i_lo, i_hi, tab, st);
    if ((rc = cuda_status(ce, "weight table"))) return rc;
  }
  const int mode = plan->cfg.mode;
  if (mode == STLG_MODE_HARD) {
    FGParams p;
    fill_fg(plan, e, B, T, p);
    p.a = i_lo;
    p.b = i_hi;
    p.K = i_hi - i_lo + 1;
    p.canon = 0;
    p.padmode = 1;
    if ((rc = resolve(plan, e.e1, channels, d_channels, bf, T, backward, p.child))) return rc;
    if (!backward) {
      p.out = out;
      ce = launch_fg_timed_fwd(mode, p, st);
    } else {
      p.out_in = out_in;
      p.cot = cot;
      p.gbuf = bf.scratch;
      ce = launch_fg_timed_bwd(mode, p, st);
    }
    return cuda_status(ce, "smooth (hard) launch");
  }
  SParams p;
  std::memset(&p, 0, sizeof(p));
  if ((rc = resolve(plan, e.e1, channels, d_channels, bf, T, backward, p.child))) return rc;
  p.B = B;
  p.L = T;
  p.i_lo = i_lo;
  p.i_hi = i_hi;
  p.sg = e.sg;
  p.pad_last = plan->cfg.pad_last;
  p.pad_value = (float)plan->cfg.pad_value;
  p.mp = mode_params(plan->cfg);
  p.lw2 = tab;
  if (!backward) {
    p.out = out;
    p.aux = e.aux_slot >= 0 ? bf.auxp(e.aux_slot) : nullptr;
    return cuda_status(launch_smooth_fwd(mode, p, st), "smooth launch");
  }
  p.out_in = out_in;
  p.aux_in = e.aux_slot >= 0 ? bf.auxp(e.aux_slot) : nullptr;
  p.cot = cot;
  p.gbuf = bf.scratch;
  p.dw64 = d_smooth ? dw64 : nullptr;  // every entry written by k_smooth_dw_reduce
  p.dwpart = bf.dwpart;
  if ((rc = cuda_status(launch_smooth_bwd(mode, p, st), "smooth backward launch"))) return rc;
  if (d_smooth) {
    ce = launch_smooth_abc(dw64, tab, T, sp.a, sp.b, sp.c, sp.eps, d_smooth + 3 * e.smooth_slot, st);
    if ((rc = cuda_status(ce, "smooth d(a,b,c)"))) return rc;
  }
  return STLG_OK;
}

// Side stream + fork / join events for two-lane plans: one set per host thread and
// device (autograd runs the backward on its own thread), created on first use outside
// stream capture (a capturing call without them runs its lanes in order on the caller's
// stream).  Under capture the fork / join records pull the side stream into the graph.
struct Fork {
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};
static Fork* fork_for(cudaStream_t st) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  thread_local std::map<int, Fork> forks;
  Fork& f = forks[dev];
  if (f.side == nullptr) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
    if (cudaStreamCreateWithFlags(&f.side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&f.ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&f.ev_join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      f = Fork{};
      return nullptr;
    }
  }
  return &f;
}
static cudaError_t fork_begin(const Fork* f, cudaStream_t st) {
  cudaError_t e = cudaEventRecord(f->ev_fork, st);
  return e == cudaSuccess ? cudaStreamWaitEvent(f->side, f->ev_fork, 0) : e;
}
static cudaError_t fork_end(const Fork* f, cudaStream_t st) {
  cudaError_t e = cudaEventRecord(f->ev_join, f->side);
  return e == cudaSuccess ? cudaStreamWaitEvent(st, f->ev_join, 0) : e;
}

int stlg_forward(const stlg_plan* plan, const stlg_channel* channels, int64_t B, int64_t T,
                 const stlg_smooth* smooth_params, float* trace_out, void* fwd_ws,
                 size_t fwd_ws_bytes, void* stream) {
  if (!plan || !trace_out) return fail(STLG_E_INVALID, "null argument");
  if (B <= 0 || T <= 0) return fail(STLG_E_SHAPE, "empty signal batch");
  if (B > 65535) return fail(STLG_E_SHAPE, "batch rows per call must be <= 65535");
  if (plan->n_ch > 0 && !channels) return fail(STLG_E_INVALID, "null channels");
  if (plan->n_slots + plan->n_aux > 0 && !fwd_ws) return fail(STLG_E_INVALID, "null workspace");
  Bufs bfl[2]{};
  int rc = setup_bufs(plan, B, T, fwd_ws, fwd_ws_bytes, nullptr, 0, bfl[0]);
  if (rc) return rc;
  if (plan->n_lanes > 1 && (rc = setup_bufs(plan, B, T, fwd_ws, fwd_ws_bytes, nullptr, 0, bfl[1], 1))) return rc;
  cudaStream_t st0 = (cudaStream_t)stream;
  const Fork* fk = plan->n_lanes > 1 ? fork_for(st0) : nullptr;
  if (fk && (rc = cuda_status(fork_begin(fk, st0), "fork"))) return rc;
  const int mode = plan->cfg.mode;
  const int n_entries = (int)plan->entries.size();
  bool open = fk != nullptr;  // side-stream work not yet joined into st0
  auto fwd_entry = [&](int ei) -> int {
    const Entry& e = plan->entries[ei];
    const int ln = plan->lane[ei];
    const Bufs& bf = bfl[ln];
    cudaStream_t st = (fk && ln == 1) ? fk->side : st0;
    float* out = e.out_slot < 0 ? trace_out : bf.slot(e.out_slot);
    cudaError_t ce = cudaSuccess;
    if (e.kind == E_POINTWISE || e.kind == E_FG_TIMED || e.kind == E_FG_UNTIMED) {
      FGParams p;
      fill_fg(plan, e, B, T, p);
      if ((rc = resolve(plan, e.e1, channels, nullptr, bf, T, false, p.child))) return rc;
      p.out = out;
      p.aux = e.aux_slot >= 0 ? bf.auxp(e.aux_slot) : nullptr;
      p.lb = bf.lb;
      if (e.kind == E_POINTWISE) ce = launch_pointwise_fwd(mode, p, st);
      else if (e.kind == E_FG_TIMED) ce = launch_fg_timed_fwd(mode, p, st);
      else ce = launch_fg_untimed_fwd(mode, p, st);
    } else if (e.kind == E_UNTIL) {
      UParams p;
      std::memset(&p, 0, sizeof(p));
      if ((rc = resolve(plan, e.e1, channels, nullptr, bf, T, false, p.left))) return rc;
      if ((rc = resolve(plan, e.e2, channels, nullptr, bf, T, false, p.right))) return rc;
      p.out = out;
      p.lb = bf.lb;
      p.B = B;
      p.L = T;
      p.a = e.untimed ? 0 : e.a;
      p.b = e.untimed ? 0 : e.b;
      p.K = e.untimed ? (int)T : e.b - e.a + 1;
      p.untimed = e.untimed;
      p.pad_last = plan->cfg.pad_last;
      p.pad_value = (float)plan->cfg.pad_value;
      p.canon = (!e.untimed && e.b > 0 && (long long)T - e.b > 0) ? 1 : 0;
      p.fill = plan->cfg.masked_fill;
      p.sent = (float)plan->cfg.sentinel;
      if (p.fill) p.canon = 0;  // no _replace_overrun in masked_fill mode (masking.py:261-274)
      p.mp = mode_params(plan->cfg);
      p.src = e.aux_slot >= 0 ? reinterpret_cast<unsigned short*>(bf.auxp(e.aux_slot)) : nullptr;
      ce = launch_until_fwd(mode, p, st);
    } else {  // E_FG_SMOOTH
      if ((rc = run_smooth(plan, e, channels, nullptr, B, T, smooth_params, bf, out, nullptr,
                           nullptr, nullptr, nullptr, st, false)))
        return rc;
    }
    if ((rc = cuda_status(ce, "forward launch"))) return rc;
    return STLG_OK;
  };
  for (int ei = 0; ei < n_entries; ++ei) {
    if (open && ei == n_entries - 1) {
      open = false;
      if ((rc = cuda_status(fork_end(fk, st0), "join"))) return rc;
    }
    if ((rc = fwd_entry(ei))) {
      if (open) fork_end(fk, st0);  // best effort: nothing on the side stream outlives the call
      return rc;
    }
  }
  return STLG_OK;
}

int stlg_backward(const stlg_plan* plan, const stlg_channel* channels, int64_t B, int64_t T,
                  const stlg_smooth* smooth_params, const float* trace, const float* cot,
                  const stlg_grad* d_channels, double* d_smooth, void* fwd_ws,
                  size_t fwd_ws_bytes, void* bwd_ws, size_t bwd_ws_bytes, void* stream) {
  if (!plan || !trace || !cot) return fail(STLG_E_INVALID, "null argument");
  if (B <= 0 || T <= 0) return fail(STLG_E_SHAPE, "empty signal batch");
  if (B > 65535) return fail(STLG_E_SHAPE, "batch rows per call must be <= 65535");
  if (!bwd_ws) return fail(STLG_E_INVALID, "null backward workspace");
  Bufs bfl[2]{};
  int rc = setup_bufs(plan, B, T, fwd_ws, fwd_ws_bytes, bwd_ws, bwd_ws_bytes, bfl[0]);
  if (rc) return rc;
  if (plan->n_lanes > 1 &&
      (rc = setup_bufs(plan, B, T, fwd_ws, fwd_ws_bytes, bwd_ws, bwd_ws_bytes, bfl[1], 1)))
    return rc;
  cudaStream_t st0 = (cudaStream_t)stream;
  const int mode = plan->cfg.mode;
  for (int c = 0; c < plan->n_ch && d_channels; ++c) {
    const stlg_grad& g = d_channels[c];
    if (g.ptr && !g.accumulate && !plan->ch_touched[c]) {
      cudaError_t ce = launch_fill_strided(g.ptr, B, T, g.row_stride, g.elem_stride, 0.f, st0);
      if ((rc = cuda_status(ce, "zero-fill"))) return rc;
    }
  }
  const Fork* fk = plan->n_lanes > 1 ? fork_for(st0) : nullptr;
  const int n_entries = (int)plan->entries.size();
  bool open = false;  // side-stream work not yet joined into st0
  auto bwd_entry = [&](int ei) -> int {
    const Entry& e = plan->entries[ei];
    const int ln = plan->lane[ei];
    const Bufs& bf = bfl[ln];
    cudaStream_t st = (fk && ln == 1) ? fk->side : st0;
    const float* g = e.out_slot < 0 ? cot : bf.gslot(e.out_slot);
    const float* out_in = e.out_slot < 0 ? trace : bf.slot(e.out_slot);
    cudaError_t ce = cudaSuccess;
    if (e.kind == E_POINTWISE || e.kind == E_FG_TIMED || e.kind == E_FG_UNTIMED) {
      FGParams p;
      fill_fg(plan, e, B, T, p);
      if ((rc = resolve(plan, e.e1, channels, d_channels, bf, T, true, p.child))) return rc;
      p.out_in = out_in;
      p.aux_in = e.aux_slot >= 0 ? bf.auxp(e.aux_slot) : nullptr;
      p.cot = g;
      p.gbuf = bf.scratch;
      p.lb = bf.lb;
      if (e.kind == E_POINTWISE) ce = launch_pointwise_vjp(mode, p, g, st);
      else if (e.kind == E_FG_TIMED) ce = launch_fg_timed_bwd(mode, p, st);
      else ce = launch_fg_untimed_bwd(mode, p, st);
    } else if (e.kind == E_UNTIL) {
      UParams p;
      std::memset(&p, 0, sizeof(p));
      if ((rc = resolve(plan, e.e1, channels, d_channels, bf, T, true, p.left))) return rc;
      if ((rc = resolve(plan, e.e2, channels, d_channels, bf, T, true, p.right))) return rc;
      p.out_in = out_in;
      p.cot = g;
      p.gl = bf.scratch;
      p.gr = bf.scratch + bf.BT;
      p.B = B;
      p.L = T;
      p.a = e.untimed ? 0 : e.a;
      p.b = e.untimed ? 0 : e.b;
      p.K = e.untimed ? (int)T : e.b - e.a + 1;
      p.untimed = e.untimed;
      p.pad_last = plan->cfg.pad_last;
      p.pad_value = (float)plan->cfg.pad_value;
      p.fill = plan->cfg.masked_fill;
      p.sent = (float)plan->cfg.sentinel;
      p.scratch = bf.uslab;
      p.dacc = bf.dacc;
      p.dscale = bf.dscale;
      p.lb = bf.lb;
      p.mp = mode_params(plan->cfg);
      p.src_in = e.aux_slot >= 0 ? reinterpret_cast<const unsigned short*>(bf.auxp(e.aux_slot)) : nullptr;
      ce = launch_until_bwd(mode, p, st);
    } else {  // E_FG_SMOOTH
      if ((rc = run_smooth(plan, e, channels, d_channels, B, T, smooth_params, bf, nullptr, out_in,
                           g, d_smooth, bf.dw64, st, true)))
        return rc;
    }
    if ((rc = cuda_status(ce, "backward launch"))) return rc;
    return STLG_OK;
  };
  for (int ei = n_entries - 1; ei >= 0; --ei) {
    if (fk && ei == n_entries - 2) {
      if ((rc = cuda_status(fork_begin(fk, st0), "fork"))) return rc;
      open = true;
    }
    if ((rc = bwd_entry(ei))) {
      if (open) fork_end(fk, st0);  // best effort: nothing on the side stream outlives the call
      return rc;
    }
  }
  if (open && (rc = cuda_status(fork_end(fk, st0), "join"))) return rc;
  return STLG_OK;
}

}  // extern "C"
