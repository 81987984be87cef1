// One distributed adaptive-refinement step of replicated grids
// (the path's only collective), natively.
//
// Per grid, the new batch is the reference's next build batch
// (next_candidates, sparse_grid.hpp:215-254).  Batches are processed group by
// group in ascending level sum (bases of equal level sum
// vanish at each other's nodes, so a group's nodes are independent of each
// other, but a group needs every lower group appended first) -- which
// reproduces insert_batch's one-by-one residual hierarchization
// (sparse_grid.hpp:256-298).  Per round, the new nodes of all grids are split
// into equal (padded) contiguous shares over the ranks; each rank evaluates
// the caller's target at its share, hierarchizes it on its GPU
// (surplus = f - interpolate, EXACT), the surplus rows are all-gathered
// (device buffers; ncclAllGather over NVLink in ddsg_refine_step_nccl) and
// every rank appends the whole group in batch order: grids stay replicated and
// bit-identical on every rank, equal to the reference's build at the next
// level.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/ddsg_b200.h"
#include "device.cuh"
#include "handles.hpp"

using namespace ddsg_b200;
using namespace ddsg_b200::abi;

namespace {

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  double* get(size_t bytes) {
    if (bytes > n) {
      if (p) cudaFree(p);
      p = nullptr;
      n = 0;
      DDSG_CUDA(cudaMalloc(&p, bytes));
      n = bytes;
    }
    return static_cast<double*>(p);
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

int level_sum(const uint32_t* key, int dim) {
  int s = 0;
  for (int j = 0; j < dim; ++j) s += level_of(key[j]);
  return s;
}

// ---- NCCL, resolved at first use (the product library does not link it)
struct Nccl {
  using AllGather = int (*)(const void*, void*, size_t, int, void*, cudaStream_t);
  using ErrStr = const char* (*)(int);
  AllGather all_gather = nullptr;
  ErrStr err = nullptr;
  std::string why;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    n.all_gather = reinterpret_cast<Nccl::AllGather>(dlsym(h, "ncclAllGather"));
    n.err = reinterpret_cast<Nccl::ErrStr>(dlsym(h, "ncclGetErrorString"));
    if (!n.all_gather) n.why = "ncclAllGather not found in libnccl.so.2";
  });
  return n;
}

struct NcclCtx {
  void* comm;
  cudaStream_t stream;
};

int nccl_allgather(const void* send, void* recv, int64_t bytes_per_rank, void* ctx) {
  const auto* c = static_cast<const NcclCtx*>(ctx);
  constexpr int kNcclFloat64 = 8;  // nccl.h ncclFloat64
  const int r = nccl().all_gather(send, recv, static_cast<size_t>(bytes_per_rank / 8), kNcclFloat64, c->comm,
                                  c->stream);
  if (r != 0) return r;
  return cudaStreamSynchronize(c->stream) == cudaSuccess ? 0 : -1;
}

}  // namespace

extern "C" {

ddsg_status ddsg_refine_step(ddsg_grid_t* const* grids, int n_grids, const int* level_sums, ddsg_node_evaluator f,
                             void* f_ctx, int rank, int world, ddsg_allgather_fn allgather, void* ag_ctx,
                             int on_device, ddsg_refine_stats* stats) {
  g_last_build_point.clear();
  return guarded([&] {
    if (!grids || n_grids < 1 || !level_sums || !f) fail(DDSG_INVALID_ARGUMENT, "refine_step: null argument");
    if (world < 1 || rank < 0 || rank >= world) fail(DDSG_INVALID_ARGUMENT, "refine_step: bad rank / world");
    if (world > 1 && !allgather) fail(DDSG_INVALID_ARGUMENT, "refine_step: world > 1 needs an all-gather");
    if (on_device && ddsg_device_count() < 1) fail(DDSG_CUDA_ERROR, "refine_step: no CUDA device for on_device");
    const int m = grids[0] ? grids[0]->g.m : 0;
    for (int gi = 0; gi < n_grids; ++gi)
      if (!grids[gi] || grids[gi]->g.m != m) fail(DDSG_INVALID_ARGUMENT, "refine_step: grids must share out_dim");
    ddsg_refine_stats st{};

    // candidate batches, split into level-sum groups (contiguous: sorted by (level sum, key))
    struct Group {
      int grid;
      std::vector<uint32_t> keys;  // [count][dim]
      int64_t count = 0;
    };
    std::vector<std::vector<Group>> groups(n_grids);
    size_t n_rounds = 0;
    for (int gi = 0; gi < n_grids; ++gi) {
      const HostGrid& G = grids[gi]->g;
      const auto batch = G.refine_candidates(level_sums[gi]);
      for (const auto& key : batch) {
        const int ls = level_sum(key.data(), G.dim);
        if (groups[gi].empty() || level_sum(groups[gi].back().keys.data(), G.dim) != ls)
          groups[gi].push_back(Group{gi, {}, 0});
        groups[gi].back().keys.insert(groups[gi].back().keys.end(), key.begin(), key.end());
        ++groups[gi].back().count;
      }
      n_rounds = std::max(n_rounds, groups[gi].size());
    }

    DevBuf d_local, d_all, d_f, d_interp;
    std::vector<double> h_local, h_all, fv, xs;
    for (size_t r = 0; r < n_rounds; ++r) {
      std::vector<const Group*> items;  // this round, in grid order
      int64_t total = 0;
      for (int gi = 0; gi < n_grids; ++gi)
        if (r < groups[gi].size()) {
          items.push_back(&groups[gi][r]);
          total += groups[gi][r].count;
        }
      if (total == 0) continue;
      const int64_t q = (total + world - 1) / world;
      const int64_t lo = rank * q, hi = std::min(total, (rank + 1) * q);
      const size_t row_bytes = static_cast<size_t>(m) * 8;
      double* dl = nullptr;
      if (on_device) {
        dl = d_local.get(std::max<size_t>(1, q * row_bytes));
        DDSG_CUDA(cudaMemset(dl, 0, q * row_bytes));
      } else {
        h_local.assign(static_cast<size_t>(q) * m, 0.0);
      }
      int64_t off = 0;
      for (const Group* it : items) {
        const int64_t a = std::max(lo, off), b = std::min(hi, off + it->count);
        if (a < b) {
          ddsg_grid* g = grids[it->grid];
          const HostGrid& G = g->g;
          const int64_t cnt = b - a;
          const uint32_t* keys = it->keys.data() + (a - off) * G.dim;
          xs.resize(static_cast<size_t>(cnt) * G.dim);
          for (int64_t i = 0; i < cnt * G.dim; ++i) xs[i] = coordinate_of(keys[i]);
          fv.assign(static_cast<size_t>(cnt) * m, 0.0);
          double t0 = now_s();
          if (f(it->grid, xs.data(), cnt, fv.data(), f_ctx) != 0)
            fail(DDSG_BUILD_ERROR, "refine_step: the target evaluator failed");
          st.target_s += now_s() - t0;
          for (int64_t i = 0; i < cnt; ++i)
            for (int c = 0; c < m; ++c)
              if (!std::isfinite(fv[i * m + c])) {
                std::ostringstream os;
                os << "refine_step: evaluator returned a non-finite value at grid point (";
                for (int j = 0; j < G.dim; ++j) os << (j ? ", " : "") << xs[i * G.dim + j];
                os << ")";
                throw BuildError(os.str(), std::vector<double>(xs.begin() + i * G.dim, xs.begin() + (i + 1) * G.dim));
              }
          t0 = now_s();
          if (on_device) {
            // surplus = f - interpolate(grid, x(key)) on the GPU, EXACT, into the send rows
            const auto prog = g->device();
            double* di = d_interp.get(cnt * row_bytes);
            const int64_t bad = evaluate(*prog, 1, xs.data(), cnt, di, nullptr);
            if (bad >= 0) fail(DDSG_DOMAIN_ERROR, "refine_step: node outside the unit cube");
            double* df = d_f.get(cnt * row_bytes);
            DDSG_CUDA(cudaMemcpy(df, fv.data(), cnt * row_bytes, cudaMemcpyHostToDevice));
            residual_on_device(df, di, cnt * m, dl + (a - lo) * m, nullptr);
            DDSG_CUDA(cudaDeviceSynchronize());
          } else {
            // host hierarchization, bit-identical to insert_batch (sparse_grid.hpp:264-276)
            std::vector<double> interp(m);
            for (int64_t i = 0; i < cnt; ++i) {
              std::fill(interp.begin(), interp.end(), 0.0);
              G.interpolate_at_node(keys + i * G.dim, G.size(), interp.data());
              for (int c = 0; c < m; ++c) h_local[(a - lo + i) * m + c] = fv[i * m + c] - interp[c];
            }
          }
          st.hierarchize_s += now_s() - t0;
        }
        off += it->count;
      }
      // all-gather the surplus rows (equal padded shares), then append everywhere
      const double t0 = now_s();
      const double* rows = nullptr;
      if (allgather) {  // also with one rank: the collective path runs whenever a communicator is given
        const int64_t bytes = q * static_cast<int64_t>(row_bytes);
        if (on_device) {
          double* da = d_all.get(static_cast<size_t>(world) * bytes);
          if (allgather(dl, da, bytes, ag_ctx) != 0) fail(DDSG_NCCL_ERROR, "refine_step: all-gather failed");
          h_all.resize(static_cast<size_t>(world) * q * m);
          DDSG_CUDA(cudaMemcpy(h_all.data(), da, world * bytes, cudaMemcpyDeviceToHost));
        } else {
          h_all.resize(static_cast<size_t>(world) * q * m);
          if (allgather(h_local.data(), h_all.data(), bytes, ag_ctx) != 0)
            fail(DDSG_NCCL_ERROR, "refine_step: all-gather failed");
        }
        st.gathered_bytes += world * bytes;
        rows = h_all.data();
      } else if (on_device) {
        h_all.resize(static_cast<size_t>(q) * m);
        DDSG_CUDA(cudaMemcpy(h_all.data(), dl, q * row_bytes, cudaMemcpyDeviceToHost));
        rows = h_all.data();
      } else {
        rows = h_local.data();
      }
      st.allgather_s += now_s() - t0;
      off = 0;
      for (const Group* it : items) {
        ddsg_grid* g = grids[it->grid];
        g->g.append(it->count, it->keys.data(), rows + off * m);
        g->invalidate();
        off += it->count;
      }
      st.new_nodes += total;
      st.rounds += 1;
    }
    if (stats) *stats = st;
  });
}

ddsg_status ddsg_refine_step_nccl(ddsg_grid_t* const* grids, int n_grids, const int* level_sums,
                                  ddsg_node_evaluator f, void* f_ctx, void* nccl_comm, int rank, int world,
                                  void* stream, ddsg_refine_stats* stats) {
  if (!nccl_comm && world > 1) return set_error(DDSG_INVALID_ARGUMENT, "refine_step_nccl: null communicator");
  if (nccl_comm) {
    const Nccl& n = nccl();
    if (!n.all_gather) return set_error(DDSG_NCCL_ERROR, "refine_step_nccl: " + n.why);
  }
  NcclCtx ctx{nccl_comm, static_cast<cudaStream_t>(stream)};
  return ddsg_refine_step(grids, n_grids, level_sums, f, f_ctx, rank, world, nccl_comm ? nccl_allgather : nullptr,
                          &ctx, 1, stats);
}

}  // extern "C"
