// C-ABI: JSON documents (serialize.hpp:31-145) and the document / slot
// accessors the C++ shim needs to rebuild a DdsgFunction.
//
// ddsg_grid_from_json    = sparse_grid_from_json  (serialize.hpp:54-77)
// ddsg_grid_to_json      = to_json(SparseGridFunction) (serialize.hpp:31-52)
// ddsg_hdmr_from_json    = ddsg_from_json (serialize.hpp:112-145) + VectorizedDdsg::compile
// ddsg_hdmr_to_json      = to_json(DdsgFunction)  (serialize.hpp:84-110)
#include <algorithm>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/ddsg_b200.h"
#include "grid_host.hpp"
#include "handles.hpp"
#include "json_doc.hpp"

using namespace ddsg_b200;
using namespace ddsg_b200::abi;
using ddsg_b200::json::Value;

namespace {

constexpr int kSchemaVersion = 1;  // serialize.hpp:17

const char* mode_name(int mode) { return mode == DDSG_ZERO_BOUNDARY ? "zero_boundary" : "modified_linear"; }

int mode_from_string(const std::string& s) {  // serialize.hpp:23-27
  if (s == "zero_boundary") return DDSG_ZERO_BOUNDARY;
  if (s == "modified_linear") return DDSG_MODIFIED_LINEAR;
  fail(DDSG_INVALID_ARGUMENT, "unknown boundary mode: " + s);
}

// heap_key with the reference's validation (grid_index.hpp:32-39).
uint32_t heap_key_checked(int level, uint32_t index) {
  if (level < 1 || level > 30) fail(DDSG_INVALID_ARGUMENT, "heap_key: level out of range [1,30]");
  if (index % 2u == 0u || index < 1u || index > (1u << level) - 1u)
    fail(DDSG_INVALID_ARGUMENT, "heap_key: index must be odd in [1, 2^l - 1], got l=" + std::to_string(level) +
                                    " i=" + std::to_string(index));
  return (uint32_t{1} << (level - 1)) + (index - 1u) / 2u;
}

// ComponentIndex::make (component_index.hpp:44-52): sorts, rejects
// duplicates and out-of-range dims.
std::vector<int32_t> component_index(const Value& j, int d) {
  std::vector<int32_t> u;
  for (int v : j.as_ints()) u.push_back(v);
  std::sort(u.begin(), u.end());
  if (std::adjacent_find(u.begin(), u.end()) != u.end())
    fail(DDSG_INVALID_ARGUMENT, "component index: duplicate dimension");
  if (!u.empty() && (u.front() < 0 || u.back() >= d))
    fail(DDSG_INVALID_ARGUMENT, "component index: dimension id out of range");
  return u;
}

struct IndexLess {  // (order, lexicographic), component_index.hpp:25-28
  bool operator()(const std::vector<int32_t>& a, const std::vector<int32_t>& b) const {
    if (a.size() != b.size()) return a.size() < b.size();
    return a < b;
  }
};

HostGrid grid_from_doc(const Value& doc) {  // serialize.hpp:54-77
  if (doc.at("schema_version").as_int() != kSchemaVersion)
    fail(DDSG_INVALID_ARGUMENT, "sparse grid document: unsupported schema version");
  if (doc.at("type").as_string() != "sparse_grid")
    fail(DDSG_INVALID_ARGUMENT, "sparse grid document: wrong type tag");
  const int dim = static_cast<int>(doc.at("dim").as_int());
  const int out_dim = static_cast<int>(doc.at("out_dim").as_int());
  // parse every node first (heap_key validates), then from_nodes' checks in node order
  const auto& nodes = doc.at("nodes").as_array();
  std::vector<std::vector<uint32_t>> nkeys(nodes.size());
  std::vector<std::vector<double>> nsur(nodes.size());
  for (size_t i = 0; i < nodes.size(); ++i) {
    const Value& jn = nodes[i];
    const auto& levels = jn.at("levels").as_array();
    const auto& indices = jn.at("indices").as_array();
    if (levels.size() != indices.size())
      fail(DDSG_INVALID_ARGUMENT, "sparse grid document: levels/indices length mismatch");
    for (size_t j = 0; j < levels.size(); ++j)
      nkeys[i].push_back(heap_key_checked(static_cast<int>(levels[j].as_int()), indices[j].as_u32()));
    nsur[i] = jn.at("surplus").as_doubles();
  }
  std::vector<uint32_t> keys;
  std::vector<double> sur;
  for (size_t i = 0; i < nodes.size(); ++i) {  // sparse_grid.hpp:168-173
    if (nkeys[i].size() != static_cast<size_t>(dim > 0 ? dim : 0))
      fail(DDSG_INVALID_ARGUMENT, "sparse grid: node key dimension mismatch");
    if (nsur[i].size() != static_cast<size_t>(out_dim > 0 ? out_dim : 0))
      fail(DDSG_INVALID_ARGUMENT, "sparse grid: node surplus length mismatch");
    keys.insert(keys.end(), nkeys[i].begin(), nkeys[i].end());
    sur.insert(sur.end(), nsur[i].begin(), nsur[i].end());
  }
  const int max_level = static_cast<int>(doc.at("max_level").as_int());
  const double eps = doc.at("eps_gamma").as_double();
  const int mode = mode_from_string(doc.at("boundary_mode").as_string());
  return HostGrid::from_nodes(dim, out_dim, mode, max_level, eps, static_cast<int64_t>(nodes.size()), keys.data(),
                              sur.data());
}

Value doubles(const double* v, size_t n) {
  Value a = Value::array();
  a.arr.reserve(n);
  for (size_t i = 0; i < n; ++i) a.push(Value::number(v[i]));
  return a;
}

Value ints(const std::vector<int32_t>& v) {
  Value a = Value::array();
  for (int32_t x : v) a.push(Value::integer(x));
  return a;
}

Value grid_to_doc(const HostGrid& g) {  // serialize.hpp:31-52
  Value doc = Value::object();
  doc.set("schema_version", Value::integer(kSchemaVersion));
  doc.set("type", Value::string("sparse_grid"));
  doc.set("dim", Value::integer(g.dim));
  doc.set("out_dim", Value::integer(g.m));
  doc.set("max_level", Value::integer(g.max_level));
  doc.set("eps_gamma", Value::number(g.eps_gamma));
  doc.set("boundary_mode", Value::string(mode_name(g.mode)));
  Value nodes = Value::array();
  const int64_t n = g.size();
  nodes.arr.reserve(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    Value lv = Value::array(), ix = Value::array();
    for (int j = 0; j < g.dim; ++j) {
      const uint32_t hk = g.keys[i * g.dim + j];
      lv.push(Value::integer(level_of(hk)));
      ix.push(Value::integer(index_of(hk)));
    }
    Value node = Value::object();
    node.set("levels", std::move(lv));
    node.set("indices", std::move(ix));
    node.set("surplus", doubles(&g.surplus[i * g.m], static_cast<size_t>(g.m)));
    nodes.push(std::move(node));
  }
  doc.set("nodes", std::move(nodes));
  return doc;
}

// The text of `doc` into a caller buffer: len_out = bytes needed (without a
// terminating NUL); written (NUL-terminated) when it fits in cap.
void emit(const Value& doc, char* buf, int64_t cap, int64_t* len_out) {
  if (!len_out) fail(DDSG_INVALID_ARGUMENT, "to_json: null length output");
  const std::string text = json::dump(doc, 2) + "\n";  // save_json writes dump(2) + "\n"
  *len_out = static_cast<int64_t>(text.size());
  if (buf) {
    if (cap < static_cast<int64_t>(text.size()) + 1)
      fail(DDSG_INVALID_ARGUMENT, "to_json: buffer too small (need " + std::to_string(text.size() + 1) + " bytes)");
    std::memcpy(buf, text.data(), text.size());
    buf[text.size()] = '\0';
  }
}

Value parse_text(const char* text, int64_t len) {
  if (!text) fail(DDSG_INVALID_ARGUMENT, "from_json: null text");
  if (len < 0) len = static_cast<int64_t>(std::strlen(text));
  return json::parse(text, static_cast<size_t>(len));
}

}  // namespace

extern "C" {

ddsg_status ddsg_grid_from_json(const char* text, int64_t len, ddsg_grid_t** out) {
  return guarded([&] {
    if (!out) fail(DDSG_INVALID_ARGUMENT, "grid_from_json: null output handle");
    const Value doc = parse_text(text, len);
    auto h = std::make_unique<ddsg_grid>();
    h->g = grid_from_doc(doc);
    *out = h.release();
  });
}

ddsg_status ddsg_grid_to_json(const ddsg_grid_t* g, char* buf, int64_t cap, int64_t* len_out) {
  return guarded([&] {
    if (!g) fail(DDSG_INVALID_ARGUMENT, "grid_to_json: null grid");
    emit(grid_to_doc(g->g), buf, cap, len_out);
  });
}

ddsg_status ddsg_hdmr_from_json(const char* text, int64_t len, ddsg_hdmr_t** out) {
  return guarded([&] {
    if (!out) fail(DDSG_INVALID_ARGUMENT, "hdmr_from_json: null output handle");
    const Value doc = parse_text(text, len);
    // ddsg_from_json (serialize.hpp:112-145)
    if (doc.at("schema_version").as_int() != kSchemaVersion)
      fail(DDSG_INVALID_ARGUMENT, "ddsg document: unsupported schema version");
    if (doc.at("type").as_string() != "ddsg") fail(DDSG_INVALID_ARGUMENT, "ddsg document: wrong type tag");
    const int dim = static_cast<int>(doc.at("dim").as_int());
    const int out_dim = static_cast<int>(doc.at("out_dim").as_int());
    const std::vector<double> coords = doc.at("anchor").at("coords").as_doubles();
    const std::vector<double> f_anchor = doc.at("anchor").at("f_anchor").as_doubles();
    const int k_max = static_cast<int>(doc.at("k_max").as_int());
    std::map<std::vector<int32_t>, HostGrid, IndexLess> accepted;
    for (const Value& e : doc.at("accepted").as_array()) {
      std::vector<int32_t> u = component_index(e.at("dims"), dim);
      HostGrid g = grid_from_doc(e.at("grid"));
      accepted.emplace(std::move(u), std::move(g));  // map::emplace keeps the first, like the reference
    }
    std::vector<std::vector<int32_t>> rejected;
    {
      std::map<std::vector<int32_t>, int, IndexLess> set;
      for (const Value& e : doc.at("rejected").as_array()) set.emplace(component_index(e, dim), 0);
      for (auto& kv : set) rejected.push_back(kv.first);
    }
    std::map<std::vector<int32_t>, int, IndexLess> coeff;
    for (const Value& e : doc.at("coeff_b").as_array())
      coeff[component_index(e.at("dims"), dim)] = static_cast<int>(e.at("b").as_int());
    std::map<std::vector<int32_t>, std::vector<double>, IndexLess> quads;
    for (const Value& e : doc.at("cut_quadratures").as_array())
      quads[component_index(e.at("dims"), dim)] = e.at("q").as_doubles();
    if (static_cast<int>(f_anchor.size()) != out_dim)
      fail(DDSG_INVALID_ARGUMENT, "ddsg document: anchor f_anchor length != out_dim");

    // VectorizedDdsg::compile (ddsg_eval.hpp:40-74): one slot per coeff_b entry
    std::vector<int32_t> order, dims, b;
    std::vector<const HostGrid*> grids;
    for (const auto& [u, bu] : coeff) {
      order.push_back(static_cast<int32_t>(u.size()));
      dims.insert(dims.end(), u.begin(), u.end());
      b.push_back(bu);
      if (u.empty()) {
        grids.push_back(nullptr);
      } else {
        auto it = accepted.find(u);
        if (it == accepted.end()) {
          std::string s = "{";
          for (size_t i = 0; i < u.size(); ++i) s += (i ? "," : "") + std::to_string(u[i]);
          fail(DDSG_INVALID_ARGUMENT, "vectorized ddsg: coefficient for a non-accepted index " + s + "}");
        }
        grids.push_back(&it->second);
      }
    }
    std::vector<std::vector<int32_t>> extra_dims;
    for (const auto& kv : accepted)
      if (!coeff.count(kv.first)) extra_dims.push_back(kv.first);
    auto h = make_hdmr(dim, out_dim, f_anchor.data(), static_cast<int>(order.size()), order.data(), dims.data(),
                       b.data(), grids.data(), extra_dims);
    h->k_max = k_max;
    h->anchor_coords = coords;
    h->rejected = rejected;
    bool all_quads = true;
    for (const auto& kv : coeff) all_quads = all_quads && quads.count(kv.first);
    if (all_quads) {
      for (const auto& kv : coeff) {
        const auto& q = quads[kv.first];
        if (static_cast<int>(q.size()) != out_dim)
          fail(DDSG_INVALID_ARGUMENT, "ddsg document: cut quadrature length != out_dim");
        h->cut_quads.insert(h->cut_quads.end(), q.begin(), q.end());
      }
    }
    for (auto& kv : accepted)
      if (!coeff.count(kv.first)) h->extra_accepted.emplace_back(kv.first, kv.second);
    *out = h.release();
  });
}

ddsg_status ddsg_hdmr_to_json(const ddsg_hdmr_t* h, char* buf, int64_t cap, int64_t* len_out) {
  return guarded([&] {
    if (!h) fail(DDSG_INVALID_ARGUMENT, "hdmr_to_json: null handle");
    if (h->anchor_coords.size() != static_cast<size_t>(h->d))
      fail(DDSG_INVALID_ARGUMENT, "hdmr_to_json: anchor coordinates not set (ddsg_hdmr_set_document)");
    if (h->cut_quads.size() != h->slots.size() * static_cast<size_t>(h->m))
      fail(DDSG_OUT_OF_RANGE, "ddsg: no quadrature for component index (ddsg_hdmr_set_document)");
    // to_json(DdsgFunction) (serialize.hpp:84-110)
    Value doc = Value::object();
    doc.set("schema_version", Value::integer(kSchemaVersion));
    doc.set("type", Value::string("ddsg"));
    doc.set("dim", Value::integer(h->d));
    doc.set("out_dim", Value::integer(h->m));
    doc.set("k_max", Value::integer(h->k_max));
    Value anchor = Value::object();
    anchor.set("coords", doubles(h->anchor_coords.data(), h->anchor_coords.size()));
    anchor.set("f_anchor", doubles(h->f_anchor.data(), h->f_anchor.size()));
    doc.set("anchor", std::move(anchor));
    // accepted map order: every slot grid plus the extra accepted grids
    std::map<std::vector<int32_t>, const HostGrid*, IndexLess> acc;
    for (const auto& s : h->slots)
      if (s.grid >= 0) acc[s.dims] = &h->grids[s.grid];
    for (const auto& kv : h->extra_accepted) acc[kv.first] = &kv.second;
    Value accepted = Value::array();
    for (const auto& [u, g] : acc) {
      Value e = Value::object();
      e.set("dims", ints(u));
      e.set("grid", grid_to_doc(*g));
      accepted.push(std::move(e));
    }
    doc.set("accepted", std::move(accepted));
    Value rejected = Value::array();
    for (const auto& u : h->rejected) rejected.push(ints(u));
    doc.set("rejected", std::move(rejected));
    Value coeff = Value::array(), quads = Value::array();
    for (size_t s = 0; s < h->slots.size(); ++s) {
      Value e = Value::object();
      e.set("dims", ints(h->slots[s].dims));
      e.set("b", Value::integer(h->slots[s].b));
      coeff.push(std::move(e));
      Value q = Value::object();
      q.set("dims", ints(h->slots[s].dims));
      q.set("q", doubles(&h->cut_quads[s * h->m], static_cast<size_t>(h->m)));
      quads.push(std::move(q));
    }
    doc.set("coeff_b", std::move(coeff));
    doc.set("cut_quadratures", std::move(quads));
    emit(doc, buf, cap, len_out);
  });
}

ddsg_status ddsg_hdmr_set_document(ddsg_hdmr_t* h, int k_max, const double* anchor_coords, int n_rejected,
                                   const int32_t* rejected_order, const int32_t* rejected_dims,
                                   const double* cut_quadratures) {
  return guarded([&] {
    if (!h) fail(DDSG_INVALID_ARGUMENT, "hdmr_set_document: null handle");
    if (n_rejected < 0 || (n_rejected > 0 && !rejected_order))
      fail(DDSG_INVALID_ARGUMENT, "hdmr_set_document: bad rejected list");
    std::map<std::vector<int32_t>, int, IndexLess> rej;
    int64_t off = 0;
    for (int r = 0; r < n_rejected; ++r) {
      const int k = rejected_order[r];
      if (k < 0 || k > h->d || (k > 0 && !rejected_dims))
        fail(DDSG_INVALID_ARGUMENT, "hdmr_set_document: bad rejected index");
      Value j = Value::array();
      for (int t = 0; t < k; ++t) j.push(Value::integer(rejected_dims[off + t]));
      off += k;
      rej.emplace(component_index(j, h->d), 0);
    }
    h->k_max = k_max;
    if (anchor_coords) h->anchor_coords.assign(anchor_coords, anchor_coords + h->d);
    h->rejected.clear();
    for (auto& kv : rej) h->rejected.push_back(kv.first);
    if (cut_quadratures)
      h->cut_quads.assign(cut_quadratures, cut_quadratures + h->slots.size() * static_cast<size_t>(h->m));
    else
      h->cut_quads.clear();
  });
}

ddsg_status ddsg_hdmr_document(const ddsg_hdmr_t* h, int* k_max, double* anchor_coords, double* f_anchor,
                               int* n_rejected, int64_t* n_rejected_dims, int32_t* rejected_order,
                               int32_t* rejected_dims, int* has_quadratures, double* cut_quadratures) {
  return guarded([&] {
    if (!h) fail(DDSG_INVALID_ARGUMENT, "hdmr_document: null handle");
    if (k_max) *k_max = h->k_max;
    if (f_anchor) std::copy(h->f_anchor.begin(), h->f_anchor.end(), f_anchor);
    if (anchor_coords) {
      if (h->anchor_coords.size() == static_cast<size_t>(h->d))
        std::copy(h->anchor_coords.begin(), h->anchor_coords.end(), anchor_coords);
      else
        std::fill(anchor_coords, anchor_coords + h->d, 0.5);  // not provided: the reference's centre default
    }
    if (n_rejected) *n_rejected = static_cast<int>(h->rejected.size());
    int64_t total = 0;
    for (size_t r = 0; r < h->rejected.size(); ++r) {
      if (rejected_order) rejected_order[r] = static_cast<int32_t>(h->rejected[r].size());
      if (rejected_dims) std::copy(h->rejected[r].begin(), h->rejected[r].end(), rejected_dims + total);
      total += static_cast<int64_t>(h->rejected[r].size());
    }
    if (n_rejected_dims) *n_rejected_dims = total;
    const bool has = h->cut_quads.size() == h->slots.size() * static_cast<size_t>(h->m);
    if (has_quadratures) *has_quadratures = has ? 1 : 0;
    if (cut_quadratures && has) std::copy(h->cut_quads.begin(), h->cut_quads.end(), cut_quadratures);
  });
}

ddsg_status ddsg_hdmr_slot(const ddsg_hdmr_t* h, int s, int* order, int32_t* dims, int32_t* b, ddsg_grid_t** grid) {
  return guarded([&] {
    if (!h) fail(DDSG_INVALID_ARGUMENT, "hdmr_slot: null handle");
    if (s < 0 || s >= static_cast<int>(h->slots.size())) fail(DDSG_OUT_OF_RANGE, "hdmr_slot: slot out of range");
    const auto& slot = h->slots[s];
    if (order) *order = static_cast<int>(slot.dims.size());
    if (dims) std::copy(slot.dims.begin(), slot.dims.end(), dims);
    if (b) *b = slot.b;
    if (grid) {
      *grid = nullptr;
      if (slot.grid >= 0) {
        auto g = std::make_unique<ddsg_grid>();
        g->g = h->grids[slot.grid];
        *grid = g.release();
      }
    }
  });
}

}  // extern "C"
