// Native planner core: maximum-reward path decomposition and channel
// ordering of one segment's reorder graph, restated in C++ with the reference's exact
// tie-breaking so the plans it feeds are identical to the Python planner's.
//
// Reference semantics followed (file:line under /root/reference/pkg/src/reslice):
//   reorder graph from retained sets ........ reorder_graph.py:84-106 (_from_nodes)
//   covered-parent bonus / covered_parents .. path_search.py:41-67
//   path_reward / is_valid_path ............. path_search.py:70-93
//   _greedy_mrap (graphs > 20 nodes) ........ path_search.py:136-154
//   solve_mrap (branch and bound) ........... path_search.py:157-287
//   decompose_paths ......................... path_search.py:290-305
//   order_channels .......................... ordering.py:39-88
// Node identity: the caller passes the nodes sorted by their string id, so node index
// order == id order and every lexicographic tie-break on ids is a tie-break on indices.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "upscale_b200.h"

namespace {

struct Graph {  // a reorder graph over a subset of the caller's nodes
  std::vector<int> gid;                 // local -> caller index (ascending)
  std::vector<std::vector<int>> ret;    // retained channels, ascending
  std::vector<int> reward;
  std::vector<std::vector<int>> shared; // |ret_u & ret_v|
  std::vector<std::vector<char>> exempt;
  std::vector<int> parents;             // nodes with >= 1 strict-subset child, ascending
  std::vector<std::vector<int>> children;  // per node, ascending
  int n = 0;
};

int intersect(const std::vector<int>& a, const std::vector<int>& b) {
  int i = 0, j = 0, c = 0;
  while (i < (int)a.size() && j < (int)b.size()) {
    if (a[i] < b[j]) ++i;
    else if (b[j] < a[i]) ++j;
    else { ++c; ++i; ++j; }
  }
  return c;
}

Graph build(const std::vector<std::vector<int>>& all, const std::vector<int>& keep) {
  Graph g;
  g.n = (int)keep.size();
  g.gid = keep;
  g.ret.resize(g.n);
  g.reward.resize(g.n);
  for (int i = 0; i < g.n; ++i) {
    g.ret[i] = all[keep[i]];
    g.reward[i] = (int)g.ret[i].size();
  }
  g.shared.assign(g.n, std::vector<int>(g.n, 0));
  g.exempt.assign(g.n, std::vector<char>(g.n, 0));
  g.children.assign(g.n, {});
  for (int u = 0; u < g.n; ++u)
    for (int v = u + 1; v < g.n; ++v) {
      const int s = intersect(g.ret[u], g.ret[v]);
      g.shared[u][v] = g.shared[v][u] = s;
      const int ru = g.reward[u], rv = g.reward[v];
      if (s == ru && ru < rv) {  // ret_u strict subset of ret_v
        g.children[v].push_back(u);
        g.exempt[u][v] = g.exempt[v][u] = 1;
      } else if (s == rv && rv < ru) {
        g.children[u].push_back(v);
        g.exempt[u][v] = g.exempt[v][u] = 1;
      }
    }
  for (int u = 0; u < g.n; ++u) {
    std::sort(g.children[u].begin(), g.children[u].end());
    if (!g.children[u].empty()) g.parents.push_back(u);
  }
  return g;
}

// parents off the path whose retained set the path's children cover
std::vector<int> covered(const Graph& g, const std::vector<int>& seq) {
  std::vector<char> on(g.n, 0);
  for (int v : seq) on[v] = 1;
  std::vector<int> out;
  for (int p : g.parents) {
    if (on[p]) continue;
    std::vector<int> cov;
    for (int c : g.children[p])
      if (on[c]) cov.insert(cov.end(), g.ret[c].begin(), g.ret[c].end());
    std::sort(cov.begin(), cov.end());
    cov.erase(std::unique(cov.begin(), cov.end()), cov.end());
    if (std::includes(cov.begin(), cov.end(), g.ret[p].begin(), g.ret[p].end())) out.push_back(p);
  }
  return out;
}

long long path_reward(const Graph& g, const std::vector<int>& seq) {
  long long r = 0;
  for (int v : seq) r += g.reward[v];
  for (size_t i = 1; i < seq.size(); ++i) r -= g.shared[seq[i - 1]][seq[i]];
  for (int p : covered(g, seq)) r += g.reward[p];
  return r;
}

bool valid_path(const Graph& g, const std::vector<int>& seq) {
  for (size_t i = 0; i < seq.size(); ++i)
    for (size_t j = i + 1; j < seq.size(); ++j) {
      if (seq[i] == seq[j]) return false;
      if (j >= i + 2 && g.shared[seq[i]][seq[j]] > 0 && !g.exempt[seq[i]][seq[j]]) return false;
    }
  return true;
}

std::vector<int> greedy(const Graph& g, long long* reward) {
  bool have = false;
  long long best_r = 0;
  std::vector<int> best;
  for (int s = 0; s < g.n; ++s) {
    std::vector<int> seq{s};
    while (true) {
      int nxt = -1;
      long long nxt_r = 0;
      for (int v = 0; v < g.n; ++v) {
        if (std::find(seq.begin(), seq.end(), v) != seq.end()) continue;
        std::vector<int> cand = seq;
        cand.push_back(v);
        if (!valid_path(g, cand)) continue;
        const long long r = path_reward(g, cand);
        if (nxt < 0 || r > nxt_r) {  // min over (-reward, id): first best in id order
          nxt = v;
          nxt_r = r;
        }
      }
      if (nxt < 0) break;
      if (nxt_r <= path_reward(g, seq)) break;
      seq.push_back(nxt);
    }
    const long long r = path_reward(g, seq);
    if (!have || r > best_r) {
      have = true;
      best_r = r;
      best = seq;
    }
  }
  *reward = best_r;
  return best;
}

struct Exact {  // solve_mrap's DFS with incremental parent coverage
  const Graph& g;
  int n;
  std::vector<long long> nonexempt;  // bitmask of non-exempt neighbours
  std::vector<std::vector<int>> child_parents;
  std::vector<std::vector<int>> cover;  // per parent, per channel position count
  std::vector<int> covered_total, need;
  std::vector<char> is_parent, bonus_active;
  long long bonus_sum = 0;
  bool have = false;
  long long best_r = 0;
  std::vector<int> best, seq;
  long long on_path = 0;

  explicit Exact(const Graph& gr) : g(gr), n(gr.n) {
    nonexempt.assign(n, 0);
    for (int u = 0; u < n; ++u)
      for (int v = 0; v < n; ++v)
        if (u != v && g.shared[u][v] > 0 && !g.exempt[u][v]) nonexempt[u] |= 1ll << v;
    child_parents.assign(n, {});
    is_parent.assign(n, 0);
    bonus_active.assign(n, 0);
    covered_total.assign(n, 0);
    need.assign(n, 0);
    cover.assign(n, {});
    for (int p : g.parents) {
      is_parent[p] = 1;
      need[p] = g.reward[p];
      cover[p].assign(g.ret[p].size(), 0);
      for (int c : g.children[p]) child_parents[c].push_back(p);
    }
  }
  int pos(int p, int ch) const {  // index of channel ch in ret_p (present: c's set is a subset)
    return int(std::lower_bound(g.ret[p].begin(), g.ret[p].end(), ch) - g.ret[p].begin());
  }
  // undo log entries: (kind, parent) with kind 0 cover(v), 1 bonus_on, 2 bonus_off
  void push(int v, std::vector<std::pair<int, int>>& undo) {
    for (int ip : child_parents[v]) {
      for (int ch : g.ret[v]) {
        int& c = cover[ip][pos(ip, ch)];
        if (c == 0) ++covered_total[ip];
        ++c;
      }
      undo.push_back({0, ip});
      if (!bonus_active[ip] && covered_total[ip] == need[ip] && !((on_path >> ip) & 1)) {
        bonus_active[ip] = 1;
        bonus_sum += g.reward[ip];
        undo.push_back({1, ip});
      }
    }
    if (is_parent[v] && bonus_active[v]) {
      bonus_active[v] = 0;
      bonus_sum -= g.reward[v];
      undo.push_back({2, v});
    }
  }
  void pop(int v, const std::vector<std::pair<int, int>>& undo) {
    for (auto it = undo.rbegin(); it != undo.rend(); ++it) {
      const int ip = it->second;
      if (it->first == 0) {
        for (int ch : g.ret[v]) {
          int& c = cover[ip][pos(ip, ch)];
          --c;
          if (c == 0) --covered_total[ip];
        }
      } else if (it->first == 1) {
        bonus_active[ip] = 0;
        bonus_sum -= g.reward[ip];
      } else {
        bonus_active[ip] = 1;
        bonus_sum += g.reward[ip];
      }
    }
  }
  void dfs(long long base, long long forbidden) {
    const int last = seq.back();
    const long long current = base + bonus_sum;
    if (!have || current > best_r) {
      have = true;
      best_r = current;
      best = seq;
    }
    long long remaining = 0;
    for (int v = 0; v < n; ++v)
      if (!((forbidden >> v) & 1)) remaining += g.reward[v];
    long long potential = 0;
    for (int p : g.parents)
      if (!bonus_active[p] && !((on_path >> p) & 1)) potential += g.reward[p];
    if (have && current + remaining + potential <= best_r) return;
    for (int v = 0; v < n; ++v) {
      if ((forbidden >> v) & 1) continue;
      std::vector<std::pair<int, int>> undo;
      push(v, undo);
      seq.push_back(v);
      on_path |= 1ll << v;
      dfs(base + g.reward[v] - g.shared[last][v], forbidden | (1ll << v) | nonexempt[last]);
      on_path &= ~(1ll << v);
      seq.pop_back();
      pop(v, undo);
    }
  }
  std::vector<int> solve(long long* reward) {
    for (int s = 0; s < n; ++s) {
      std::vector<std::pair<int, int>> undo;
      push(s, undo);
      seq.push_back(s);
      on_path |= 1ll << s;
      dfs(g.reward[s], 1ll << s);
      on_path &= ~(1ll << s);
      seq.pop_back();
      pop(s, undo);
    }
    *reward = best_r;
    return best;
  }
};

constexpr int EXACT_NODE_CAP = 20;  // path_search.py:27

}  // namespace

// Decompose a segment's reorder graph into paths and emit its channel order.
//   n nodes (sorted by id), node i retains channels[offsets[i] .. offsets[i+1]) (ascending)
//   out_order: kept channels in their new order (capacity channel_space), *n_order its length
//   path_of[i]: index of the path node i was placed on (as a path member or absorbed parent)
//   path_pos[i]: position on that path (members 0..len-1), or -1 for an absorbed parent
//   path_reward_out[k]: reward of path k in the subgraph it was found in; *n_paths paths
extern "C" int ub_plan_order_segment(int n, const int32_t* offsets, const int32_t* channels, int channel_space,
                                     int32_t* out_order, int32_t* n_order, int32_t* path_of, int32_t* path_pos,
                                     int64_t* path_reward_out, int32_t* n_paths) {
  if (n < 0 || channel_space < 0 || !offsets || !out_order || !n_order || !path_of || !path_pos ||
      !path_reward_out || !n_paths)
    return UB_EINVAL;
  std::vector<std::vector<int>> all(n);
  for (int i = 0; i < n; ++i) {
    all[i].assign(channels + offsets[i], channels + offsets[i + 1]);
    if (all[i].empty()) return UB_EINVAL;
    for (size_t k = 0; k < all[i].size(); ++k)
      if (all[i][k] < 0 || all[i][k] >= channel_space || (k && all[i][k] <= all[i][k - 1])) return UB_EINVAL;
  }
  // ---- decompose_paths
  std::vector<int> remaining(n);
  for (int i = 0; i < n; ++i) remaining[i] = i;
  std::vector<std::vector<int>> tracked;  // per path: members then absorbed parents (caller indices)
  int np = 0;
  while (!remaining.empty()) {
    const Graph sub = build(all, remaining);
    long long reward = 0;
    std::vector<int> seq;
    if (sub.n > EXACT_NODE_CAP) {
      seq = greedy(sub, &reward);
    } else {
      Exact ex(sub);
      seq = ex.solve(&reward);
    }
    const std::vector<int> absorbed = covered(sub, seq);
    std::vector<int> t;
    for (size_t k = 0; k < seq.size(); ++k) {
      const int gi = sub.gid[seq[k]];
      t.push_back(gi);
      path_of[gi] = np;
      path_pos[gi] = (int)k;
    }
    for (int p : absorbed) {
      const int gi = sub.gid[p];
      t.push_back(gi);
      path_of[gi] = np;
      path_pos[gi] = -1;
    }
    tracked.push_back(t);
    path_reward_out[np] = reward;
    ++np;
    std::vector<char> gone(n, 0);
    for (int gi : t) gone[gi] = 1;
    std::vector<int> next;
    for (int gi : remaining)
      if (!gone[gi]) next.push_back(gi);
    remaining.swap(next);
  }
  *n_paths = np;
  // ---- order_channels
  std::vector<char> emitted(channel_space, 0), retained_any(channel_space, 0);
  for (int i = 0; i < n; ++i)
    for (int ch : all[i]) retained_any[ch] = 1;
  std::vector<std::vector<char>> has(n, std::vector<char>(channel_space, 0));
  for (int i = 0; i < n; ++i)
    for (int ch : all[i]) has[i][ch] = 1;
  std::vector<int> done(n, 0);  // emitted channels of each node
  int cnt = 0;
  auto emit = [&](int ch) {
    emitted[ch] = 1;
    out_order[cnt++] = ch;
    for (int i = 0; i < n; ++i)
      if (has[i][ch]) ++done[i];
  };
  for (const auto& t : tracked) {
    auto pending = [&](int i) { return done[i] < (int)all[i].size(); };
    auto started = [&](int i) { return done[i] > 0; };
    while (true) {
      bool any = false;
      for (int i : t) any = any || pending(i);
      if (!any) break;
      std::vector<int> active;
      for (int i : t)
        if (started(i) && pending(i)) active.push_back(i);
      std::vector<int> cand;
      if (!active.empty()) {
        std::vector<int> pool = active;
        while (true) {
          cand.clear();
          for (int ch : all[pool[0]]) {
            if (emitted[ch]) continue;
            bool all_have = true;
            for (size_t k = 1; k < pool.size() && all_have; ++k) all_have = has[pool[k]][ch];
            if (all_have) cand.push_back(ch);
          }
          if (!cand.empty()) break;
          // shed the consumer with the fewest retained channels (ties: smallest id)
          size_t drop = 0;
          for (size_t k = 1; k < pool.size(); ++k) {
            const int a = pool[k], b = pool[drop];
            if (all[a].size() < all[b].size() || (all[a].size() == all[b].size() && a < b)) drop = k;
          }
          pool.erase(pool.begin() + drop);
        }
      } else {
        int first = -1;
        for (int i : t)
          if (pending(i)) {
            first = i;
            break;
          }
        for (int ch : all[first])
          if (!emitted[ch]) cand.push_back(ch);
      }
      // fewest not-yet-started tracked consumers wanting it, then the smallest channel
      int best = -1, best_k = 0;
      for (int ch : cand) {
        int k = 0;
        for (int i : t)
          if (!started(i) && has[i][ch]) ++k;
        if (best < 0 || k < best_k || (k == best_k && ch < best)) {
          best = ch;
          best_k = k;
        }
      }
      emit(best);
    }
  }
  for (int ch = 0; ch < channel_space; ++ch)
    if (retained_any[ch] && !emitted[ch]) out_order[cnt++] = ch;
  *n_order = cnt;
  return UB_OK;
}
