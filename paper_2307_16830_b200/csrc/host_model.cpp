// Host-side model compilation: canonical record order, template expansion,
// dedup, slot maps, and the deterministic gather plans of the device AD.
//
// Reference semantics followed:
//   canonical order      model.py:128-140   (np.lexsort, targets primary)
//   template expansion   model.py:250-283   (COO from first_slots/second_pairs)
//   dedup + slot maps    model.py:229-233, 285-303  (row<<32|col keys, searchsorted)
//   accumulation order   autodiff.py:57-142 (defines, then increments in block
//                        order; np.add.at in record order)
#include <algorithm>
#include <cstring>
#include <numeric>

#include "internal.h"

namespace gn {

static inline uint64_t key(int64_t i, int64_t j) {
  return (static_cast<uint64_t>(i) << 32) | static_cast<uint64_t>(j);
}

static int64_t find_key(const std::vector<uint64_t> &keys, uint64_t k) {
  auto it = std::lower_bound(keys.begin(), keys.end(), k);
  return static_cast<int64_t>(it - keys.begin());
}

// Stable CSR from (out, src) pairs appended in accumulation order.
static void build_csr(int64_t n_out, const std::vector<int64_t> &outs,
                      const std::vector<int64_t> &srcs, std::vector<int64_t> &ptr,
                      std::vector<int64_t> &list) {
  ptr.assign(n_out + 1, 0);
  for (int64_t o : outs) ptr[o + 1]++;
  for (int64_t i = 0; i < n_out; ++i) ptr[i + 1] += ptr[i];
  list.assign(outs.size(), 0);
  std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
  for (size_t t = 0; t < outs.size(); ++t) list[fill[outs[t]]++] = srcs[t];
}

static void compile_model(Model &M) {
  int64_t nb = static_cast<int64_t>(M.blocks.size());
  // ---- expansion (model.py:250-283)
  std::vector<uint64_t> jk, hk;
  for (auto &b : M.blocks) {
    for (size_t p = 0; p < b.pairs.size() / 2; ++p) {
      int a = b.pairs[2 * p], c = b.pairs[2 * p + 1];
      for (int64_t r = 0; r < b.R; ++r) {
        int64_t ga = b.var_idx[r * b.nv + a], gc = b.var_idx[r * b.nv + c];
        hk.push_back(key(std::max(ga, gc), std::min(ga, gc)));
      }
    }
    if (b.kind != 0) {
      for (int s : b.first)
        for (int64_t r = 0; r < b.R; ++r) jk.push_back(key(b.targets[r], b.var_idx[r * b.nv + s]));
    }
  }
  sort_unique(jk);
  sort_unique(hk);
  M.jac_rows.resize(jk.size());
  M.jac_cols.resize(jk.size());
  for (size_t i = 0; i < jk.size(); ++i) {
    M.jac_rows[i] = static_cast<int64_t>(jk[i] >> 32);
    M.jac_cols[i] = static_cast<int64_t>(jk[i] & 0xFFFFFFFFull);
  }
  M.hess_rows.resize(hk.size());
  M.hess_cols.resize(hk.size());
  for (size_t i = 0; i < hk.size(); ++i) {
    M.hess_rows[i] = static_cast<int64_t>(hk[i] >> 32);
    M.hess_cols[i] = static_cast<int64_t>(hk[i] & 0xFFFFFFFFull);
  }
  // ---- slot maps (model.py:285-303) + contribution layout
  M.jac_slots.clear();
  M.hess_slots.clear();
  M.hess_factor.clear();
  std::vector<int64_t> cbase(nb);
  int64_t nc = 0;
  for (int64_t bi = 0; bi < nb; ++bi) {
    auto &b = M.blocks[bi];
    cbase[bi] = nc;
    nc += b.R * (1 + static_cast<int64_t>(b.first.size()) + static_cast<int64_t>(b.pairs.size() / 2));
    if (b.kind != 0)
      for (int s : b.first)
        for (int64_t r = 0; r < b.R; ++r)
          M.jac_slots.push_back(find_key(jk, key(b.targets[r], b.var_idx[r * b.nv + s])));
    for (size_t p = 0; p < b.pairs.size() / 2; ++p) {
      int a = b.pairs[2 * p], c = b.pairs[2 * p + 1];
      for (int64_t r = 0; r < b.R; ++r) {
        int64_t ga = b.var_idx[r * b.nv + a], gc = b.var_idx[r * b.nv + c];
        M.hess_slots.push_back(find_key(hk, key(std::max(ga, gc), std::min(ga, gc))));
        M.hess_factor.push_back((a != c && ga == gc) ? 2.0 : 1.0);
      }
    }
  }
  M.n_contrib = nc;
  // ---- gather plans in the reference's accumulation order (autodiff.py)
  std::vector<int64_t> outs, srcs;
  // constraints: all defines (assignment), then increments block by block
  for (int pass = 1; pass <= 2; ++pass)
    for (int64_t bi = 0; bi < nb; ++bi) {
      auto &b = M.blocks[bi];
      if (b.kind != pass) continue;
      for (int64_t r = 0; r < b.R; ++r) {
        outs.push_back(b.targets[r]);
        srcs.push_back(cbase[bi] + r);
      }
    }
  build_csr(M.m, outs, srcs, M.c_ptr, M.c_src);
  // gradient: objective blocks, slots in reverse-sweep (dict) order
  outs.clear();
  srcs.clear();
  for (int64_t bi = 0; bi < nb; ++bi) {
    auto &b = M.blocks[bi];
    if (b.kind != 0) continue;
    for (int s : b.grad_order) {
      int k = static_cast<int>(std::find(b.first.begin(), b.first.end(), s) - b.first.begin());
      GN_REQUIRE(k < static_cast<int>(b.first.size()), "grad_order slot not in first_slots");
      for (int64_t r = 0; r < b.R; ++r) {
        outs.push_back(b.var_idx[r * b.nv + s]);
        srcs.push_back(cbase[bi] + (1 + k) * b.R + r);
      }
    }
  }
  build_csr(M.n, outs, srcs, M.grad_ptr, M.grad_src);
  // Jacobian: constraint blocks, first slots in order
  outs.clear();
  srcs.clear();
  {
    int64_t js = 0;
    for (int64_t bi = 0; bi < nb; ++bi) {
      auto &b = M.blocks[bi];
      if (b.kind == 0) continue;
      for (size_t k = 0; k < b.first.size(); ++k)
        for (int64_t r = 0; r < b.R; ++r) {
          outs.push_back(M.jac_slots[js++]);
          srcs.push_back(cbase[bi] + (1 + static_cast<int64_t>(k)) * b.R + r);
        }
    }
  }
  build_csr(static_cast<int64_t>(jk.size()), outs, srcs, M.jac_ptr, M.jac_src);
  // Hessian: every block with pairs, pair order
  outs.clear();
  srcs.clear();
  {
    int64_t hs = 0;
    for (int64_t bi = 0; bi < nb; ++bi) {
      auto &b = M.blocks[bi];
      int64_t nf = static_cast<int64_t>(b.first.size());
      for (size_t p = 0; p < b.pairs.size() / 2; ++p)
        for (int64_t r = 0; r < b.R; ++r) {
          outs.push_back(M.hess_slots[hs++]);
          srcs.push_back(cbase[bi] + (1 + nf + static_cast<int64_t>(p)) * b.R + r);
        }
    }
  }
  build_csr(static_cast<int64_t>(hk.size()), outs, srcs, M.hess_ptr, M.hess_src);
  // objective values, block order
  M.obj_src.clear();
  M.obj_block_ptr.assign(1, 0);
  for (int64_t bi = 0; bi < nb; ++bi) {
    auto &b = M.blocks[bi];
    if (b.kind != 0 || b.R == 0) continue;
    for (int64_t r = 0; r < b.R; ++r) M.obj_src.push_back(cbase[bi] + r);
    M.obj_block_ptr.push_back(static_cast<int64_t>(M.obj_src.size()));
  }
}

}  // namespace gn

using namespace gn;

extern "C" int gn_canonical_order(int64_t R, int32_t nv, int32_t np, const int64_t *var_idx,
                                  const double *params, const int64_t *targets,
                                  int64_t *order) {
  return guarded([&] {
    std::vector<int64_t> idx(R);
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t x, int64_t y) {
      if (targets && targets[x] != targets[y]) return targets[x] < targets[y];
      for (int c = 0; c < nv; ++c) {
        int64_t a = var_idx[x * nv + c], b = var_idx[y * nv + c];
        if (a != b) return a < b;
      }
      for (int c = 0; c < np; ++c) {
        double a = params[x * np + c], b = params[y * np + c];
        if (a < b) return true;
        if (b < a) return false;
      }
      return false;
    });
    std::memcpy(order, idx.data(), sizeof(int64_t) * R);
  });
}

extern "C" int gn_model_create(const gn_block_desc *blocks, int32_t nblocks, int64_t n_var,
                               int64_t n_con, gn_model **out) {
  return guarded([&] {
    GN_REQUIRE(n_var < (int64_t(1) << 31) && n_con < (int64_t(1) << 31),
               "model too large for 32-bit device indices");
    auto *M = new gn_model();
    try {
      M->n = n_var;
      M->m = n_con;
      for (int32_t bi = 0; bi < nblocks; ++bi) {
        const gn_block_desc &d = blocks[bi];
        Model::HBlock h;
        h.kind = d.kind;
        h.nv = d.n_var_slots;
        h.np = d.n_param_slots;
        h.out = d.out;
        h.R = d.n_records;
        // longer tapes / more slots than the interpreter holds run on the
        // generated pattern kernels only (checked again at upload)
        GN_REQUIRE(d.n_ops <= kMaxTapeGen, "instruction tape longer than 4096 entries");
        GN_REQUIRE(h.nv <= kMaxSlotsGen, "more than 256 variable slots per record");
        if (d.n_ops > kMaxTape || h.nv > kMaxSlots || d.n_consts > kMaxTape) M->needs_patterns = true;
        GN_REQUIRE(d.kind == 0 || d.targets != nullptr || h.R == 0, "constraint block without targets");
        h.var_idx.assign(d.var_idx, d.var_idx + h.R * h.nv);
        h.params.assign(d.params, d.params + h.R * h.np);
        if (d.kind != 0) h.targets.assign(d.targets, d.targets + h.R);
        h.ops.assign(d.ops, d.ops + 3 * d.n_ops);
        h.consts.assign(d.consts, d.consts + d.n_consts);
        h.first.assign(d.first_slots, d.first_slots + d.n_first);
        h.pairs.assign(d.pairs, d.pairs + 2 * d.n_pairs);
        if (d.grad_order)
          h.grad_order.assign(d.grad_order, d.grad_order + d.n_first);
        else
          h.grad_order = h.first;
        for (int64_t v : h.var_idx) GN_REQUIRE(v >= 0 && v < n_var, "variable index out of range");
        for (int64_t t : h.targets) GN_REQUIRE(t >= 0 && t < n_con, "target out of range");
        M->blocks.push_back(std::move(h));
      }
      compile_model(*M);
    } catch (...) {
      delete M;
      throw;
    }
    *out = M;
  });
}

extern "C" int gn_model_info(const gn_model *M, int64_t *nnz_jac, int64_t *nnz_hess,
                             int64_t *n_contrib) {
  return guarded([&] {
    if (nnz_jac) *nnz_jac = static_cast<int64_t>(M->jac_rows.size());
    if (nnz_hess) *nnz_hess = static_cast<int64_t>(M->hess_rows.size());
    if (n_contrib) *n_contrib = M->n_contrib;
  });
}

extern "C" int gn_model_export(const gn_model *M, int64_t *jr, int64_t *jc, int64_t *hr,
                               int64_t *hc, int64_t *js, int64_t *hs, double *hf) {
  return guarded([&] {
    auto cp = [](auto *dst, const auto &v) {
      if (dst && !v.empty()) std::memcpy(dst, v.data(), sizeof(v[0]) * v.size());
    };
    cp(jr, M->jac_rows);
    cp(jc, M->jac_cols);
    cp(hr, M->hess_rows);
    cp(hc, M->hess_cols);
    cp(js, M->jac_slots);
    cp(hs, M->hess_slots);
    cp(hf, M->hess_factor);
  });
}

extern "C" void gn_model_destroy(gn_model *M) { delete M; }
