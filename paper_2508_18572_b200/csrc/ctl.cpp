// ctl.cpp — the control plane behind include/strata_ctl.h.
//
// HiRadixTree with transient nodes, deferral on delay hit, Algorithm 1
// balanced batch formation with bundle hits, and the cache controller's page
// allocators, LRU eviction with write-back and the LOAD / WRITE-BACK plans in strata_xfer's shape.
// The readings of the paper it applies are DESIGN.md R17-R26.  Host code only: no CUDA calls.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "../../include/strata_ctl.h"
#include "internal.h"

namespace {

constexpr int kInQueue = 1, kInFlight = 2;

int cfail(int code, const std::string& msg) { return strata::set_last_error(code, msg.c_str()); }

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct Node {
  std::vector<int32_t> key;                     // edge tokens (non-empty except the root)
  Node* parent = nullptr;
  std::unordered_map<int32_t, Node*> children;  // by first token of the child's edge
  std::vector<int64_t> dev, host;               // per-token slots, or empty (not resident there)
  int mark = 0;                                 // 0 committed, kInQueue, kInFlight
  int64_t tref = 0;                             // dispatched requests covering a transient node
  int64_t ref = 0;                              // dispatched requests pinning a committed node
  double last_access = 0.0;
};

void free_subtree(Node* n) {
  for (auto& kv : n->children) free_subtree(kv.second);
  delete n;
}

// Page / chunk allocator: LIFO free list of units of `unit` slots, a live-slot count per unit
// (R23).  A unit returns to the free list when its last live slot is released.
struct Pool {
  int64_t unit = 1;
  std::vector<int32_t> free_units;
  std::vector<int32_t> live;

  void init(int64_t units, int64_t u) {
    unit = u;
    free_units.resize(units);
    for (int64_t i = 0; i < units; ++i) free_units[i] = static_cast<int32_t>(units - 1 - i);
    live.assign(units, 0);
  }
  int64_t nfree() const { return static_cast<int64_t>(free_units.size()); }
  // caller ensured ceil(ntok / unit) free units
  void alloc(int64_t ntok, std::vector<int64_t>& out) {
    out.resize(ntok);
    int64_t cur = -1;
    for (int64_t j = 0; j < ntok; ++j) {
      if (j % unit == 0) {
        cur = free_units.back();
        free_units.pop_back();
      }
      out[j] = cur * unit + j % unit;
      ++live[cur];
    }
  }
  void release(int64_t s) {
    const int64_t u = s / unit;
    if (--live[u] == 0) free_units.push_back(static_cast<int32_t>(u));
  }
};

struct Req {
  std::vector<int32_t> tokens;
  bool dispatched = false;
  int64_t k = 0;                  // committed prefix pinned at dispatch
  std::vector<int64_t> slots;     // device slot of every token once dispatched
};

struct Seg {
  int64_t start, len;
  int cls;                        // 0 device, 1 host, 2 transient
};

struct Stat {                     // a request's load / compute requirement
  const int32_t* key = nullptr;
  int64_t klen = 0;
  std::vector<Seg> segs;
  int64_t device = 0, host = 0, compute = 0;
};

struct Plan {
  std::vector<int64_t> num_tokens, chunk_start, page_start;
  std::vector<int32_t> chunk_offset, page_offset, host_chunks, dev_pages;
};

}  // namespace

struct strata_ctl {
  int64_t P = 1, C = 1;
  Pool dpool, hpool;
  int64_t threshold = 100;
  double ratio = 100.0;
  int64_t max_tokens = 0;
  int64_t max_reqs = 0;
  bool defer = true, balance = true, bundle = true;
  Node* root = nullptr;
  std::vector<int64_t> queue;
  std::unordered_map<int64_t, Req> reqs;
  std::vector<std::pair<int64_t, int64_t>> load_pairs, wb_pairs;   // (host slot, device slot)
  std::vector<int64_t> last_batch, last_deferred, last_formed;
  Plan plans[2];
  std::string dump_buf;

  ~strata_ctl() {
    if (root) free_subtree(root);
  }

  // ------------------------------------------------------------------ tree primitives
  static int64_t common(const int32_t* a, int64_t na, const int32_t* b, int64_t nb) {
    const int64_t m = std::min(na, nb);
    int64_t i = 0;
    while (i < m && a[i] == b[i]) ++i;
    return i;
  }
  static int cls(const Node* n) { return n->mark ? 2 : (!n->dev.empty() ? 0 : 1); }

  void segments(const int32_t* key, int64_t n, std::vector<Seg>* segs, strata_ctl_match_t* m) const {
    if (m) *m = strata_ctl_match_t{0, 0, 0, 0};
    const Node* node = root;
    int64_t i = 0;
    while (i < n) {
      auto it = node->children.find(key[i]);
      if (it == node->children.end()) break;
      const Node* c = it->second;
      const int64_t l = common(c->key.data(), static_cast<int64_t>(c->key.size()), key + i, n - i);
      const int k = cls(c);
      if (segs) segs->push_back(Seg{i, l, k});
      if (m) {
        m->total += l;
        (k == 0 ? m->device : k == 1 ? m->host : m->transient) += l;
      }
      if (l < static_cast<int64_t>(c->key.size())) break;
      i += l;
      node = c;
    }
  }

  Node* split(Node* c, int64_t at) {
    Node* up = new Node;
    up->key.assign(c->key.begin(), c->key.begin() + at);
    up->parent = c->parent;
    if (!c->dev.empty()) up->dev.assign(c->dev.begin(), c->dev.begin() + at);
    if (!c->host.empty()) up->host.assign(c->host.begin(), c->host.begin() + at);
    up->mark = c->mark;
    up->tref = c->tref;
    up->ref = c->ref;
    up->last_access = c->last_access;
    c->parent->children[c->key[0]] = up;
    c->key.erase(c->key.begin(), c->key.begin() + at);
    if (!c->dev.empty()) c->dev.erase(c->dev.begin(), c->dev.begin() + at);
    if (!c->host.empty()) c->host.erase(c->host.begin(), c->host.begin() + at);
    c->parent = up;
    up->children[c->key[0]] = c;
    return up;
  }

  // nodes covering the longest stored prefix of key, splitting a partially matched node
  int64_t align(const int32_t* key, int64_t n, std::vector<Node*>& nodes) {
    nodes.clear();
    Node* node = root;
    int64_t i = 0;
    while (i < n) {
      auto it = node->children.find(key[i]);
      if (it == node->children.end()) break;
      Node* c = it->second;
      const int64_t l = common(c->key.data(), static_cast<int64_t>(c->key.size()), key + i, n - i);
      if (l < static_cast<int64_t>(c->key.size())) c = split(c, l);
      nodes.push_back(c);
      i += l;
      node = c;
    }
    return i;
  }

  Node* add_child(Node* parent, const int32_t* key, int64_t n) {
    Node* c = new Node;
    c->key.assign(key, key + n);
    c->parent = parent;
    parent->children[key[0]] = c;
    return c;
  }

  void remove_leaf(Node* n) {
    n->parent->children.erase(n->key[0]);
    delete n;
  }

  template <class F>
  void for_each_node(F&& f) const {
    std::vector<const Node*> stack{root};
    while (!stack.empty()) {
      const Node* n = stack.back();
      stack.pop_back();
      for (auto& kv : n->children) {
        f(kv.second);
        stack.push_back(kv.second);
      }
    }
  }

  static void path_of(const Node* n, std::vector<int32_t>& out) {
    std::vector<const Node*> chain;
    for (; n && n->parent; n = n->parent) chain.push_back(n);
    out.clear();
    for (auto it = chain.rbegin(); it != chain.rend(); ++it) out.insert(out.end(), (*it)->key.begin(), (*it)->key.end());
  }

  // ------------------------------------------------------------------ transient nodes (§4.3.1)
  void mark_in_queue(const int32_t* key, int64_t n) {
    std::vector<Node*> nodes;
    const int64_t i = align(key, n, nodes);
    if (i < n) add_child(nodes.empty() ? root : nodes.back(), key + i, n - i)->mark = kInQueue;
  }

  void clear_in_queue() {   // R18: in-queue marks live for one scheduling round
    std::vector<Node*> stack{root};
    while (!stack.empty()) {
      Node* n = stack.back();
      stack.pop_back();
      for (auto it = n->children.begin(); it != n->children.end();) {
        if (it->second->mark == kInQueue) {
          free_subtree(it->second);
          it = n->children.erase(it);
        } else {
          stack.push_back(it->second);
          ++it;
        }
      }
    }
  }

  // ------------------------------------------------------------------ eviction (R23)
  // Victim order: least recent last_access, ties broken by the lexicographically smaller token path.
  // Paths are compared without materialising them: below their lowest common ancestor two paths
  // diverge at the first tokens of two sibling edges (radix property); an ancestor's path is a
  // prefix of its descendants' (smaller).
  static int depth_of(const Node* n) {
    int d = 0;
    for (; n->parent; n = n->parent) ++d;
    return d;
  }
  static bool path_less(const Node* a, const Node* b) {
    if (a == b) return false;
    int da = depth_of(a), db = depth_of(b);
    const Node* x = a;
    const Node* y = b;
    bool lifted_a = false;
    while (da > db) { x = x->parent; --da; lifted_a = true; }
    while (db > da) { y = y->parent; --db; }
    if (x == y) return !lifted_a;            // one is the other's ancestor: the ancestor is smaller
    while (x->parent != y->parent) {
      x = x->parent;
      y = y->parent;
    }
    return x->key[0] < y->key[0];
  }
  struct Later {                              // heap order: the top is the next victim
    bool operator()(const Node* a, const Node* b) const {
      if (a->last_access != b->last_access) return a->last_access > b->last_access;
      return path_less(b, a);
    }
  };
  static bool host_victim(const Node* n) {
    return n->mark == 0 && !n->host.empty() && n->dev.empty() && n->ref == 0 && n->children.empty();
  }
  static bool dev_victim(const Node* n) {
    if (n->mark != 0 || n->dev.empty() || n->ref != 0) return false;
    for (auto& kv : n->children)
      if (!kv.second->dev.empty()) return false;
    return true;
  }
  // Candidates are collected once per call; evicting a node can only make its parent a candidate,
  // so the heap yields the same sequence as re-scanning the tree before every eviction.
  template <class Pred>
  std::vector<Node*> victims(Pred&& pred) const {
    std::vector<Node*> h;
    for_each_node([&](const Node* n) {
      if (pred(n)) h.push_back(const_cast<Node*>(n));
    });
    std::make_heap(h.begin(), h.end(), Later{});
    return h;
  }
  static Node* pop_victim(std::vector<Node*>& h) {
    std::pop_heap(h.begin(), h.end(), Later{});
    Node* v = h.back();
    h.pop_back();
    return v;
  }
  static void push_victim(std::vector<Node*>& h, Node* n) {
    h.push_back(n);
    std::push_heap(h.begin(), h.end(), Later{});
  }

  bool ensure_host(int64_t units) {
    if (hpool.nfree() >= units) return true;
    std::vector<Node*> h = victims(host_victim);
    while (hpool.nfree() < units) {
      if (h.empty()) return false;
      Node* v = pop_victim(h);
      if (!host_victim(v)) continue;
      Node* parent = v->parent;
      for (int64_t s : v->host) hpool.release(s);
      remove_leaf(v);
      if (parent != root && host_victim(parent)) push_victim(h, parent);
    }
    return true;
  }

  bool ensure_dev(int64_t units) {
    if (dpool.nfree() >= units) return true;
    std::vector<Node*> h = victims(dev_victim);
    while (dpool.nfree() < units) {
      if (h.empty()) return false;
      Node* v = pop_victim(h);
      if (!dev_victim(v)) continue;
      if (v->host.empty()) {        // inclusive write-back before the drop
        if (!ensure_host(ceil_div(static_cast<int64_t>(v->key.size()), C))) return false;
        hpool.alloc(static_cast<int64_t>(v->key.size()), v->host);
        for (size_t j = 0; j < v->key.size(); ++j) wb_pairs.emplace_back(v->host[j], v->dev[j]);
      }
      for (int64_t s : v->dev) dpool.release(s);
      v->dev.clear();
      if (v->parent != root && dev_victim(v->parent)) push_victim(h, v->parent);
    }
    return true;
  }

  // ------------------------------------------------------------------ plans (R25)
  void build_plan(const std::vector<std::pair<int64_t, int64_t>>& pairs, Plan& p) const {
    p = Plan{};
    for (size_t j = 0; j < pairs.size(); ++j) {
      const int64_t h = pairs[j].first, d = pairs[j].second;
      bool cont = false;
      if (j > 0) {
        const int64_t ph = pairs[j - 1].first, pd = pairs[j - 1].second;
        const bool hc = (ph % C == C - 1) ? (h % C == 0) : (h == ph + 1);
        const bool dc = (pd % P == P - 1) ? (d % P == 0) : (d == pd + 1);
        cont = hc && dc;
      }
      if (!cont) {
        p.num_tokens.push_back(0);
        p.chunk_start.push_back(static_cast<int64_t>(p.host_chunks.size()));
        p.page_start.push_back(static_cast<int64_t>(p.dev_pages.size()));
        p.chunk_offset.push_back(static_cast<int32_t>(h % C));
        p.page_offset.push_back(static_cast<int32_t>(d % P));
      }
      if (!cont || h % C == 0) p.host_chunks.push_back(static_cast<int32_t>(h / C));
      if (!cont || d % P == 0) p.dev_pages.push_back(static_cast<int32_t>(d / P));
      ++p.num_tokens.back();
    }
  }

  void publish_plans() {
    build_plan(load_pairs, plans[STRATA_CTL_LOAD]);
    build_plan(wb_pairs, plans[STRATA_CTL_WRITEBACK]);
  }

  // ------------------------------------------------------------------ scheduler (§4.3)
  Stat stats(int64_t rid) const {
    const Req& r = reqs.at(rid);
    Stat s;
    s.key = r.tokens.data();
    s.klen = static_cast<int64_t>(r.tokens.size()) - 1;      // R17
    strata_ctl_match_t m;
    segments(s.key, s.klen, &s.segs, &m);
    s.device = m.device;
    s.host = m.host;
    s.compute = static_cast<int64_t>(r.tokens.size()) - m.device - m.host;
    return s;
  }

  // host tokens of r inside the prefix r shares with b (R20)
  static int64_t host_overlap(const Stat& r, const Stat& b) {
    const int64_t lcp = common(r.key, r.klen, b.key, b.klen);
    int64_t o = 0;
    for (const Seg& g : r.segs)
      if (g.cls == 1) o += std::max<int64_t>(0, std::min(g.start + g.len, lcp) - g.start);
    return o;
  }

  // Algorithm 1, Balanced Batch Formation
  std::vector<int64_t> form_batch(std::vector<int64_t> Q, std::unordered_map<int64_t, Stat>& st,
                                  int64_t* load_out, int64_t* comp_out) const {
    std::vector<int64_t> B;
    int64_t load = 0, comp = 0;
    // overlap(r) = max over members b of host_overlap(r, b), kept incrementally: updated for every
    // candidate when a member joins (only candidates with host tokens can overlap)
    std::unordered_map<int64_t, int64_t> ov;
    ov.reserve(Q.size() * 2);
    auto overlap = [&](int64_t r) {
      auto it = ov.find(r);
      return it == ov.end() ? int64_t(0) : it->second;
    };
    std::vector<int64_t> all = Q;                // every candidate (queue and, later, the D list)
    std::unordered_map<int64_t, bool> in_b;
    auto joined = [&](int64_t b) {
      in_b[b] = true;
      for (int64_t r : all)
        if (!in_b.count(r) && st[r].host > 0) {
          const int64_t o = host_overlap(st[r], st[b]);
          if (o > 0) {
            int64_t& cur = ov[r];
            cur = std::max(cur, o);
          }
        }
    };
    auto eff_load = [&](int64_t r) { return st[r].host - overlap(r); };
    auto is_full = [&] { return (max_reqs > 0 && static_cast<int64_t>(B.size()) >= max_reqs) ||
                                (max_tokens > 0 && comp >= max_tokens); };
    auto fits = [&](int64_t r) {
      if (B.empty()) return true;
      if (max_reqs > 0 && static_cast<int64_t>(B.size()) + 1 > max_reqs) return false;
      return !(max_tokens > 0 && comp + st[r].compute > max_tokens);
    };
    auto loading_bound = [&](int64_t r) {
      const int64_t l = load + eff_load(r);
      const int64_t c = comp + st[r].compute;
      return static_cast<double>(l) / static_cast<double>(std::max<int64_t>(c, 1)) > ratio;
    };
    auto add = [&](int64_t r) {
      load += eff_load(r);
      comp += st[r].compute;
      B.push_back(r);
      joined(r);
    };
    auto add_bundle_hit = [&] {                  // procedure AddBundleHit(Q, B)
      if (!bundle) return;
      std::vector<int64_t> snapshot = Q;
      for (int64_t r : snapshot)
        if (overlap(r) > threshold && fits(r)) {
          add(r);
          Q.erase(std::find(Q.begin(), Q.end(), r));
        }
    };
    *load_out = *comp_out = 0;
    if (Q.empty()) return B;
    add(Q.front());                              // line 10
    Q.erase(Q.begin());
    add_bundle_hit();
    std::vector<int64_t> D;
    while (!Q.empty() && !is_full()) {           // line 11
      const int64_t r = Q.front();
      Q.erase(Q.begin());
      if (balance && loading_bound(r)) {
        D.push_back(r);                          // line 14
      } else if (fits(r)) {
        add(r);                                  // line 16
        add_bundle_hit();
      } else {
        break;                                   // R21: FIFO stop
      }
    }
    for (int64_t r : D) {                        // lines 17-19
      if (is_full() || !fits(r)) break;
      add(r);
    }
    *load_out = load;
    *comp_out = comp;
    return B;
  }

  bool dispatch(int64_t rid, double now, int64_t* new_tokens) {
    Req& r = reqs.at(rid);
    const int64_t n = static_cast<int64_t>(r.tokens.size());
    std::vector<Node*> nodes;
    align(r.tokens.data(), n - 1, nodes);
    size_t nc = 0;
    while (nc < nodes.size() && nodes[nc]->mark == 0) ++nc;
    int64_t k = 0, need = 0;
    for (size_t j = 0; j < nc; ++j) {
      const int64_t len = static_cast<int64_t>(nodes[j]->key.size());
      k += len;
      if (nodes[j]->dev.empty()) need += ceil_div(len, P);
      ++nodes[j]->ref;
    }
    need += ceil_div(n - k, P);
    if (!ensure_dev(need)) {
      for (size_t j = 0; j < nc; ++j) --nodes[j]->ref;
      return false;
    }
    r.slots.clear();
    r.slots.reserve(n);
    for (size_t j = 0; j < nc; ++j) {
      Node* nd = nodes[j];
      if (nd->dev.empty()) {
        dpool.alloc(static_cast<int64_t>(nd->key.size()), nd->dev);
        for (size_t t = 0; t < nd->key.size(); ++t) load_pairs.emplace_back(nd->host[t], nd->dev[t]);
      }
      nd->last_access = now;
      r.slots.insert(r.slots.end(), nd->dev.begin(), nd->dev.end());
    }
    std::vector<int64_t> fresh;
    dpool.alloc(n - k, fresh);
    r.slots.insert(r.slots.end(), fresh.begin(), fresh.end());
    for (size_t j = nc; j < nodes.size(); ++j) {  // "marked in-flight"
      nodes[j]->mark = kInFlight;
      ++nodes[j]->tref;
    }
    r.k = k;
    r.dispatched = true;
    *new_tokens += n - k;
    return true;
  }

  int schedule(double now, strata_ctl_round* out) {
    load_pairs.clear();
    wb_pairs.clear();
    clear_in_queue();
    std::vector<int64_t> eligible, deferred;
    for (int64_t rid : queue) {
      const Req& r = reqs.at(rid);
      const int64_t klen = static_cast<int64_t>(r.tokens.size()) - 1;
      if (defer) {
        strata_ctl_match_t m;
        segments(r.tokens.data(), klen, nullptr, &m);
        if (m.transient > threshold) {
          deferred.push_back(rid);
          continue;
        }
        mark_in_queue(r.tokens.data(), klen);
      }
      eligible.push_back(rid);
    }
    std::unordered_map<int64_t, Stat> st;
    st.reserve(eligible.size() * 2);
    for (int64_t rid : eligible) st.emplace(rid, stats(rid));
    int64_t load = 0, comp = 0;
    std::vector<int64_t> batch = form_batch(eligible, st, &load, &comp);
    std::vector<int64_t> done;
    int64_t new_tokens = 0;
    for (int64_t rid : batch) {
      if (!dispatch(rid, now, &new_tokens)) break;
      done.push_back(rid);
    }
    std::vector<int64_t> q = deferred;             // R19
    for (int64_t rid : eligible)
      if (!reqs.at(rid).dispatched) q.push_back(rid);
    queue.swap(q);
    last_batch = done;
    last_deferred = deferred;
    last_formed = batch;
    publish_plans();
    if (out) {
      out->num_batch = static_cast<int64_t>(done.size());
      out->num_deferred = static_cast<int64_t>(deferred.size());
      out->num_formed = static_cast<int64_t>(batch.size());
      out->formed_load = load;
      out->formed_compute = comp;
      out->new_tokens = new_tokens;
      out->load_tokens = static_cast<int64_t>(load_pairs.size());
      out->writeback_tokens = static_cast<int64_t>(wb_pairs.size());
    }
    return STRATA_OK;
  }

  int insert(const int32_t* tokens, int64_t n, int tier, double now, int64_t* slots_out) {
    load_pairs.clear();
    wb_pairs.clear();
    std::vector<Node*> nodes;
    const int64_t i = align(tokens, n, nodes);
    const bool dev = tier == STRATA_TIER_DEVICE;
    Pool& pool = dev ? dpool : hpool;
    const int64_t unit = dev ? P : C;
    int64_t need = ceil_div(n - i, unit);
    for (Node* nd : nodes) {
      if ((dev ? nd->dev : nd->host).empty()) need += ceil_div(static_cast<int64_t>(nd->key.size()), unit);
      ++nd->ref;
    }
    const bool ok = dev ? ensure_dev(need) : ensure_host(need);
    for (Node* nd : nodes) --nd->ref;
    if (!ok) {
      publish_plans();
      return cfail(STRATA_ERR_OOM, std::string("strata_ctl_insert: ") + (dev ? "device" : "host") +
                                       " tier has no room (every node pinned or needed)");
    }
    for (Node* nd : nodes) {
      nd->mark = 0;
      nd->tref = 0;
      auto& v = dev ? nd->dev : nd->host;
      if (v.empty()) pool.alloc(static_cast<int64_t>(nd->key.size()), v);
      nd->last_access = now;
    }
    if (i < n) {
      Node* c = add_child(nodes.empty() ? root : nodes.back(), tokens + i, n - i);
      pool.alloc(n - i, dev ? c->dev : c->host);
      c->last_access = now;
      nodes.push_back(c);
    }
    if (slots_out) {
      int64_t o = 0;
      for (Node* nd : nodes)
        for (int64_t s : (dev ? nd->dev : nd->host)) slots_out[o++] = s;
    }
    publish_plans();
    return STRATA_OK;
  }

  void complete(int64_t rid, double now) {
    Req& r = reqs.at(rid);
    const int64_t n = static_cast<int64_t>(r.tokens.size());
    std::vector<Node*> nodes;
    align(r.tokens.data(), n, nodes);
    int64_t pos = 0;
    for (Node* nd : nodes) {
      const int64_t L = static_cast<int64_t>(nd->key.size());
      if (pos < r.k) {
        --nd->ref;
      } else if (nd->mark) {
        nd->mark = 0;
        nd->tref = 0;
        nd->dev.assign(r.slots.begin() + pos, r.slots.begin() + pos + L);
      } else if (!nd->dev.empty()) {          // computed twice: keep the tree's copy (R26)
        for (int64_t j = pos; j < pos + L; ++j) dpool.release(r.slots[j]);
      } else {
        nd->dev.assign(r.slots.begin() + pos, r.slots.begin() + pos + L);
      }
      nd->last_access = now;
      pos += L;
    }
    if (pos < n) {
      Node* c = add_child(nodes.empty() ? root : nodes.back(), r.tokens.data() + pos, n - pos);
      c->dev.assign(r.slots.begin() + pos, r.slots.end());
      c->last_access = now;
    }
    reqs.erase(rid);
  }

  void abort(int64_t rid) {
    Req& r = reqs.at(rid);
    if (!r.dispatched) {
      queue.erase(std::find(queue.begin(), queue.end(), rid));
      reqs.erase(rid);
      return;
    }
    std::vector<Node*> nodes;
    align(r.tokens.data(), static_cast<int64_t>(r.tokens.size()) - 1, nodes);
    int64_t pos = 0;
    for (Node* nd : nodes) {
      if (pos < r.k) --nd->ref;
      else if (nd->mark) --nd->tref;
      pos += static_cast<int64_t>(nd->key.size());
    }
    for (size_t j = static_cast<size_t>(r.k); j < r.slots.size(); ++j) dpool.release(r.slots[j]);
    for (auto it = nodes.rbegin(); it != nodes.rend(); ++it) {   // in-flight nodes nobody covers
      Node* nd = *it;
      if (nd->mark == kInFlight && nd->tref == 0 && nd->children.empty()) remove_leaf(nd);
      else break;
    }
    reqs.erase(rid);
  }

  const char* dump() {
    std::vector<std::pair<std::vector<int32_t>, std::string>> rows;
    for_each_node([&](const Node* n) {
      std::vector<int32_t> p;
      path_of(n, p);
      std::string s;
      auto ints = [&](auto& v) {
        for (size_t j = 0; j < v.size(); ++j) {
          if (j) s += ',';
          s += std::to_string(v[j]);
        }
      };
      ints(p);
      s += ';';
      ints(n->dev);
      s += ';';
      ints(n->host);
      char tail[96];
      std::snprintf(tail, sizeof tail, ";%d;%lld;%lld;%.17g", n->mark, static_cast<long long>(n->tref),
                    static_cast<long long>(n->ref), n->last_access);
      s += tail;
      rows.emplace_back(std::move(p), std::move(s));
    });
    std::sort(rows.begin(), rows.end(),
              [](const auto& a, const auto& b) { return a.first < b.first; });
    dump_buf.clear();
    for (auto& r : rows) {
      dump_buf += r.second;
      dump_buf += '\n';
    }
    return dump_buf.c_str();
  }
};

extern "C" {

int strata_ctl_create(const strata_ctl_desc* d, strata_ctl_t* out) {
  if (!d || !out) return cfail(STRATA_ERR_INVALID_ARG, "strata_ctl_create: NULL argument");
  *out = nullptr;
  if (d->page_size < 1 || d->chunk_tokens < 1 || d->num_pages < 0 || d->num_chunks < 0 ||
      d->num_pages > INT32_MAX || d->num_chunks > INT32_MAX || d->deferral_threshold < 0 ||
      !(d->loading_bound_ratio > 0))
    return cfail(STRATA_ERR_INVALID_ARG, "strata_ctl_create: bad page_size / chunk_tokens / capacity / "
                                         "threshold / ratio");
  auto* c = new strata_ctl;
  c->P = d->page_size;
  c->C = d->chunk_tokens;
  c->dpool.init(d->num_pages, d->page_size);
  c->hpool.init(d->num_chunks, d->chunk_tokens);
  c->threshold = d->deferral_threshold;
  c->ratio = d->loading_bound_ratio;
  c->max_tokens = d->max_batch_tokens;
  c->max_reqs = d->max_batch_reqs;
  c->defer = !(d->flags & STRATA_CTL_NO_DEFER);
  c->balance = !(d->flags & STRATA_CTL_NO_BALANCE);
  c->bundle = !(d->flags & STRATA_CTL_NO_BUNDLE);
  c->root = new Node;
  c->publish_plans();
  *out = c;
  return STRATA_OK;
}

int strata_ctl_destroy(strata_ctl_t c) {
  delete c;
  return STRATA_OK;
}

int strata_ctl_insert(strata_ctl_t c, const int32_t* tokens, int64_t n, int32_t tier, double now,
                      int64_t* slots_out) {
  if (!c || n < 0 || (n > 0 && !tokens) || (tier != STRATA_TIER_DEVICE && tier != STRATA_TIER_HOST))
    return cfail(STRATA_ERR_INVALID_ARG, "strata_ctl_insert: bad argument");
  return c->insert(tokens, n, tier, now, slots_out);
}

int strata_ctl_match(strata_ctl_t c, const int32_t* tokens, int64_t n, strata_ctl_match_t* out) {
  if (!c || !out || n < 0 || (n > 0 && !tokens))
    return cfail(STRATA_ERR_INVALID_ARG, "strata_ctl_match: bad argument");
  c->segments(tokens, n, nullptr, out);
  return STRATA_OK;
}

int strata_ctl_submit(strata_ctl_t c, int64_t req_id, const int32_t* tokens, int64_t n) {
  if (!c || n < 1 || !tokens) return cfail(STRATA_ERR_INVALID_ARG, "strata_ctl_submit: need n >= 1 tokens");
  if (c->reqs.count(req_id))
    return cfail(STRATA_ERR_DUPLICATE, "strata_ctl_submit: request id " + std::to_string(req_id) + " exists");
  Req& r = c->reqs[req_id];
  r.tokens.assign(tokens, tokens + n);
  c->queue.push_back(req_id);
  return STRATA_OK;
}

int strata_ctl_schedule(strata_ctl_t c, double now, strata_ctl_round* out) {
  if (!c) return cfail(STRATA_ERR_INVALID_ARG, "strata_ctl_schedule: NULL handle");
  return c->schedule(now, out);
}

int strata_ctl_ids(strata_ctl_t c, int32_t which, int64_t* ids_out, int64_t* n_out) {
  if (!c || !n_out) return cfail(STRATA_ERR_INVALID_ARG, "strata_ctl_ids: NULL argument");
  const std::vector<int64_t>* v = which == STRATA_CTL_BATCH ? &c->last_batch
                                : which == STRATA_CTL_DEFERRED ? &c->last_deferred
                                : which == STRATA_CTL_FORMED ? &c->last_formed
                                : which == STRATA_CTL_QUEUE ? &c->queue : nullptr;
  if (!v) return cfail(STRATA_ERR_INVALID_ARG, "strata_ctl_ids: unknown list");
  *n_out = static_cast<int64_t>(v->size());
  if (ids_out) std::copy(v->begin(), v->end(), ids_out);
  return STRATA_OK;
}

int strata_ctl_plan_get(strata_ctl_t c, int32_t which, strata_ctl_plan* out) {
  if (!c || !out || (which != STRATA_CTL_LOAD && which != STRATA_CTL_WRITEBACK))
    return cfail(STRATA_ERR_INVALID_ARG, "strata_ctl_plan_get: bad argument");
  const Plan& p = c->plans[which];
  out->num_reqs = static_cast<int64_t>(p.num_tokens.size());
  out->num_tokens = p.num_tokens.data();
  out->chunk_start = p.chunk_start.data();
  out->chunk_offset = p.chunk_offset.data();
  out->host_chunks = p.host_chunks.data();
  out->host_chunks_len = static_cast<int64_t>(p.host_chunks.size());
  out->page_start = p.page_start.data();
  out->page_offset = p.page_offset.data();
  out->dev_pages = p.dev_pages.data();
  out->dev_pages_len = static_cast<int64_t>(p.dev_pages.size());
  return STRATA_OK;
}

int strata_ctl_req_slots(strata_ctl_t c, int64_t req_id, int64_t* slots_out, int64_t* n_out) {
  if (!c || !n_out) return cfail(STRATA_ERR_INVALID_ARG, "strata_ctl_req_slots: NULL argument");
  auto it = c->reqs.find(req_id);
  if (it == c->reqs.end() || !it->second.dispatched)
    return cfail(STRATA_ERR_INVALID_ARG, "strata_ctl_req_slots: request " + std::to_string(req_id) +
                                             " is not dispatched");
  *n_out = static_cast<int64_t>(it->second.slots.size());
  if (slots_out) std::copy(it->second.slots.begin(), it->second.slots.end(), slots_out);
  return STRATA_OK;
}

int strata_ctl_complete(strata_ctl_t c, int64_t req_id, double now) {
  if (!c) return cfail(STRATA_ERR_INVALID_ARG, "strata_ctl_complete: NULL handle");
  auto it = c->reqs.find(req_id);
  if (it == c->reqs.end() || !it->second.dispatched)
    return cfail(STRATA_ERR_INVALID_ARG, "strata_ctl_complete: request " + std::to_string(req_id) +
                                             " is not dispatched");
  c->complete(req_id, now);
  return STRATA_OK;
}

int strata_ctl_abort(strata_ctl_t c, int64_t req_id) {
  if (!c) return cfail(STRATA_ERR_INVALID_ARG, "strata_ctl_abort: NULL handle");
  if (!c->reqs.count(req_id))
    return cfail(STRATA_ERR_INVALID_ARG, "strata_ctl_abort: unknown request " + std::to_string(req_id));
  c->abort(req_id);
  return STRATA_OK;
}

int strata_ctl_get_stats(strata_ctl_t c, strata_ctl_stats* out) {
  if (!c || !out) return cfail(STRATA_ERR_INVALID_ARG, "strata_ctl_get_stats: NULL argument");
  *out = strata_ctl_stats{};
  c->for_each_node([&](const Node* n) {
    ++out->nodes;
    if (n->mark) ++out->transient_nodes;
    out->device_tokens += n->dev.empty() ? 0 : static_cast<int64_t>(n->key.size());
    out->host_tokens += n->host.empty() ? 0 : static_cast<int64_t>(n->key.size());
  });
  out->free_pages = c->dpool.nfree();
  out->free_chunks = c->hpool.nfree();
  for (auto& kv : c->reqs) (kv.second.dispatched ? out->dispatched : out->queued) += 1;
  return STRATA_OK;
}

const char* strata_ctl_dump(strata_ctl_t c) { return c ? c->dump() : ""; }

int64_t strata_ctl_bubble_steps(double t_load_ms, double t_comp_ms, double decode_step_ms,
                                int64_t decode_reqs) {
  if (decode_reqs <= 0 || !(decode_step_ms > 0) || !(t_load_ms > t_comp_ms)) return 0;
  return static_cast<int64_t>((t_load_ms - t_comp_ms) / decode_step_ms);
}

}  // extern "C"
