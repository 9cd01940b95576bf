// Host-side layerization + tensorization, a C++
// restatement of the reference's layerize() (laycirc/layerize.py:158-271)
// and tensorize() without layer_orders (tensorize.py:135-194). Output index
// vectors are bit-identical to the reference's:
//   * heights: 1 + max child height, bumped once when the gate kind
//     disagrees with the layer parity (layerize.py:231-233);
//   * pass-through chains via lift(), hash-consed (211-218);
//   * Merkle digests: mix64 finalizer, wrapping-add combine, per-op tags
//     (39-60, 75-83), with a structural re-check on every digest match
//     (147-155) so collisions never merge distinct nodes;
//   * roots padded to the top layer (241-243);
//   * canonical within-layer order: ascending digest, insertion order on
//     ties (247-260); input slots ordered by (variable, + before -).
#include <stdint.h>

#include <algorithm>
#include <string>
#include <unordered_map>
#include <vector>

#include "klay.h"

namespace {

thread_local std::string g_lerr;

constexpr uint64_t TAG_INPUT = 0x9E3779B97F4A7C15ull;
constexpr uint64_t TAG_PROD = 0xC2B2AE3D27D4EB4Full;
constexpr uint64_t TAG_SUM = 0x165667B19E3779F9ull;

inline uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

enum Kind : int8_t { K_LEAF = 0, K_AND = 1, K_OR = 2, K_TRUE = 3, K_FALSE = 4 };

struct Layer {
  bool prod = false;                 // layer op (input layer: neither)
  std::vector<uint64_t> digest;      // per node, insertion order
  std::vector<int64_t> coff{0};      // children offsets
  std::vector<int32_t> kids;         // children (previous-layer positions), source order
  std::vector<int32_t> skids;        // the same, sorted (structural key)
  std::unordered_map<uint64_t, std::vector<int32_t>> buckets;

  int32_t size() const { return (int32_t)digest.size(); }

  // hash-consed insert (layerize.py:147-155)
  int32_t intern(const int32_t* ch, int n, uint64_t d) {
    std::vector<int32_t> key(ch, ch + n);
    std::sort(key.begin(), key.end());
    auto it = buckets.find(d);
    if (it != buckets.end()) {
      for (int32_t pos : it->second) {
        const int64_t a = coff[pos], b = coff[pos + 1];
        if (b - a == n && std::equal(key.begin(), key.end(), skids.begin() + a)) return pos;
      }
    }
    const int32_t pos = size();
    digest.push_back(d);
    kids.insert(kids.end(), ch, ch + n);
    skids.insert(skids.end(), key.begin(), key.end());
    coff.push_back((int64_t)kids.size());
    buckets[d].push_back(pos);
    return pos;
  }
};

struct Result {
  int64_t num_inputs = 0, num_vars = 0;
  std::vector<int64_t> widths, edge_counts, sources, segments, root_indices, const_pos;
  std::vector<int8_t> const_val;
  std::vector<int32_t> input_lits;  // DIMACS code per slot
};

}  // namespace

struct KlayLayered {
  Result r;
};

extern "C" const char* klay_layerize_error(void) { return g_lerr.c_str(); }

extern "C" int klay_layerize(int32_t num_circuits, const int64_t* node_offsets, const int8_t* kinds,
                             const int32_t* literals, const int64_t* child_offsets,
                             const int32_t* children, const int64_t* root_offsets,
                             const int32_t* roots, const int32_t* num_vars, KlayLayered** out) {
  if (!out) return KLAY_EINVAL;
  *out = nullptr;
  if (num_circuits < 1) {
    g_lerr = "layerize requires at least one circuit";
    return KLAY_EFORMAT;
  }
  // ---- pass 1: reachability, constant roots, literals (layerize.py:172-200)
  std::vector<std::vector<int32_t>> reach(num_circuits);
  std::vector<std::vector<std::pair<int64_t, int32_t>>> root_pos(num_circuits);
  std::vector<std::pair<int64_t, bool>> constants;
  std::vector<int32_t> lits;
  int64_t position = 0, nvars = 0;
  for (int32_t c = 0; c < num_circuits; ++c) {
    const int64_t base = node_offsets[c], n = node_offsets[c + 1] - base;
    const int64_t r0 = root_offsets[c], r1 = root_offsets[c + 1];
    if (r1 == r0) {
      g_lerr = "circuit has no roots";
      return KLAY_EFORMAT;
    }
    nvars = std::max<int64_t>(nvars, num_vars[c]);
    std::vector<char> seen(n, 0);
    std::vector<int32_t> stack;
    for (int64_t r = r0; r < r1; ++r) {
      const int32_t id = roots[r];
      if (id < 0 || id >= n) {
        g_lerr = "root id out of range";
        return KLAY_EFORMAT;
      }
      const int8_t k = kinds[base + id];
      if (k == K_TRUE || k == K_FALSE) constants.push_back({position, k == K_TRUE});
      else root_pos[c].push_back({position, id});
      ++position;
      stack.push_back(id);
    }
    while (!stack.empty()) {
      const int32_t id = stack.back();
      stack.pop_back();
      if (seen[id]) continue;
      seen[id] = 1;
      for (int64_t e = child_offsets[base + id]; e < child_offsets[base + id + 1]; ++e) {
        const int32_t ch = children[e];
        if (ch < 0 || ch >= id) {
          g_lerr = "child id must precede its parent";
          return KLAY_EFORMAT;
        }
        stack.push_back(ch);
      }
    }
    for (int32_t id = 0; id < n; ++id) {
      if (!seen[id]) continue;
      reach[c].push_back(id);
      const int8_t k = kinds[base + id];
      if (k == K_LEAF) {
        lits.push_back(literals[base + id]);
      } else if (k == K_TRUE || k == K_FALSE) {
        bool is_root = false;
        for (int64_t r = r0; r < r1; ++r) is_root |= (roots[r] == id);
        if (!is_root) {
          g_lerr = "internal constant node: run fold_constants first";
          return KLAY_EFORMAT;
        }
      }
    }
  }
  // canonical literal order: (variable, positive first) (circuit.py:56-58)
  std::sort(lits.begin(), lits.end(), [](int32_t a, int32_t b) {
    const int32_t va = a < 0 ? -a : a, vb = b < 0 ? -b : b;
    if (va != vb) return va < vb;
    return a > b;  // positive before negative
  });
  lits.erase(std::unique(lits.begin(), lits.end()), lits.end());
  std::unordered_map<int32_t, int32_t> slot_of;
  for (size_t i = 0; i < lits.size(); ++i) slot_of[lits[i]] = (int32_t)i;

  // ---- pass 2: placement with hash-consing (layerize.py:202-239)
  std::vector<Layer> layers(1);
  for (int32_t code : lits) {
    const int32_t var = code < 0 ? -code : code;
    const uint64_t enc = 2ull * (uint64_t)var + (code > 0 ? 0 : 1);
    layers[0].digest.push_back(mix64(TAG_INPUT + mix64(enc)));
    layers[0].coff.push_back(0);
  }
  auto builder = [&](int h) -> Layer& {
    while ((int)layers.size() <= h) {
      Layer L;
      L.prod = (layers.size() % 2 == 1);
      layers.push_back(std::move(L));
    }
    return layers[h];
  };
  auto lift = [&](int layer, int32_t pos, int target) -> int32_t {
    while (layer < target) {
      const uint64_t d = layers[layer].digest[pos];
      ++layer;
      Layer& b = builder(layer);
      const uint64_t tag = b.prod ? TAG_PROD : TAG_SUM;
      pos = b.intern(&pos, 1, mix64(tag + mix64(d)));
    }
    return pos;
  };
  struct RootRef {
    int64_t pos;
    int layer;
    int32_t idx;
  };
  std::vector<RootRef> root_refs;
  std::vector<int32_t> kid_buf;
  for (int32_t c = 0; c < num_circuits; ++c) {
    const int64_t base = node_offsets[c];
    const int64_t n = node_offsets[c + 1] - base;
    std::vector<int32_t> pl_layer(n, -1), pl_pos(n, -1);
    for (int32_t id : reach[c]) {
      const int8_t k = kinds[base + id];
      if (k == K_LEAF) {
        pl_layer[id] = 0;
        pl_pos[id] = slot_of[literals[base + id]];
        continue;
      }
      if (k == K_TRUE || k == K_FALSE) continue;
      const bool prod = (k == K_AND);
      const int64_t e0 = child_offsets[base + id], e1 = child_offsets[base + id + 1];
      if (e1 == e0) {
        g_lerr = "gate without children";
        return KLAY_EFORMAT;
      }
      int h = 0;
      for (int64_t e = e0; e < e1; ++e) h = std::max(h, pl_layer[children[e]]);
      h += 1;
      if ((h % 2 == 1) != prod) h += 1;
      builder(h);
      kid_buf.clear();
      for (int64_t e = e0; e < e1; ++e) kid_buf.push_back(lift(pl_layer[children[e]], pl_pos[children[e]], h - 1));
      uint64_t acc = prod ? TAG_PROD : TAG_SUM;
      for (int32_t kpos : kid_buf) acc += mix64(layers[h - 1].digest[kpos]);
      pl_layer[id] = h;
      pl_pos[id] = layers[h].intern(kid_buf.data(), (int)kid_buf.size(), mix64(acc));
    }
    for (auto& rp : root_pos[c]) root_refs.push_back({rp.first, pl_layer[rp.second], pl_pos[rp.second]});
  }
  if (!root_refs.empty()) {
    int top = 0;
    for (auto& r : root_refs) top = std::max(top, r.layer);
    for (auto& r : root_refs) {
      r.idx = lift(r.layer, r.idx, top);
      r.layer = top;
    }
  } else if (constants.empty()) {
    g_lerr = "no roots to layerize";
    return KLAY_EFORMAT;
  }

  // ---- canonical order + tensorize (layerize.py:247-263, tensorize.py:165-182)
  KlayLayered* res = new KlayLayered();
  Result& R = res->r;
  R.num_inputs = (int64_t)lits.size();
  R.num_vars = nvars;
  R.input_lits = lits;
  std::vector<int32_t> prev_map(lits.size());
  for (size_t i = 0; i < lits.size(); ++i) prev_map[i] = (int32_t)i;
  for (size_t l = 1; l < layers.size(); ++l) {
    const Layer& L = layers[l];
    const int32_t W = L.size();
    std::vector<int32_t> order(W);
    for (int32_t i = 0; i < W; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return L.digest[a] < L.digest[b]; });
    std::vector<int32_t> old_to_new(W);
    for (int32_t i = 0; i < W; ++i) old_to_new[order[i]] = i;
    R.widths.push_back(W);
    int64_t E = 0;
    for (int32_t nw = 0; nw < W; ++nw) {
      const int32_t old = order[nw];
      for (int64_t e = L.coff[old]; e < L.coff[old + 1]; ++e) {
        R.sources.push_back(prev_map[L.kids[e]]);
        R.segments.push_back(nw);
        ++E;
      }
    }
    R.edge_counts.push_back(E);
    prev_map.swap(old_to_new);
  }
  std::sort(root_refs.begin(), root_refs.end(),
            [](const RootRef& a, const RootRef& b) { return a.pos < b.pos; });
  for (auto& r : root_refs) R.root_indices.push_back(prev_map[r.idx]);
  std::sort(constants.begin(), constants.end());
  for (auto& c : constants) {
    R.const_pos.push_back(c.first);
    R.const_val.push_back(c.second ? 1 : 0);
  }
  *out = res;
  return KLAY_OK;
}

extern "C" int64_t klay_layered_info(const KlayLayered* h, int32_t what) {
  if (!h) return -1;
  const Result& R = h->r;
  switch (what) {
    case 0: return R.num_inputs;
    case 1: return R.num_vars;
    case 2: return (int64_t)R.widths.size();
    case 3: return (int64_t)R.sources.size();
    case 4: return (int64_t)R.root_indices.size();
    case 5: return (int64_t)R.const_pos.size();
    default: return -1;
  }
}

extern "C" int klay_layered_export(const KlayLayered* h, int64_t* widths, int64_t* edge_counts,
                                   int64_t* sources, int64_t* segments, int32_t* input_lits,
                                   int64_t* root_indices, int64_t* const_pos, int8_t* const_val) {
  if (!h) return KLAY_EINVAL;
  const Result& R = h->r;
  std::copy(R.widths.begin(), R.widths.end(), widths);
  std::copy(R.edge_counts.begin(), R.edge_counts.end(), edge_counts);
  std::copy(R.sources.begin(), R.sources.end(), sources);
  std::copy(R.segments.begin(), R.segments.end(), segments);
  std::copy(R.input_lits.begin(), R.input_lits.end(), input_lits);
  std::copy(R.root_indices.begin(), R.root_indices.end(), root_indices);
  std::copy(R.const_pos.begin(), R.const_pos.end(), const_pos);
  std::copy(R.const_val.begin(), R.const_val.end(), const_val);
  return KLAY_OK;
}

extern "C" void klay_layered_destroy(KlayLayered* h) { delete h; }
