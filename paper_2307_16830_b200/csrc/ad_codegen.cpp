// Pattern compiler: one straight-line CUDA device function per repeated
// expression pattern (pattern block), generated from its instruction tape and
// compiled at run time with NVRTC for sm_100a.
//
// This is the SIMD abstraction of the paper: every record of a
// pattern block runs the same instruction with different data, so the
// instruction is compiled once into specialised code -- value, reverse
// sweep (gradient / Jacobian row) and forward-over-reverse Hessian columns
// -- with every intermediate in registers.  The generator replays the
// reference interpreter's semantics (expressions.py:222-409, the same
// operation order, the same "absent adjoint" rules) at generation time:
// all masks depend on the tape only, so they become straight-line code.
// The per-record contributions feed the same deterministic gather as the
// interpreter kernel (ad.cu), which stays as the fallback.
//
// libnvrtc and libcuda are opened with dlopen, so the library still loads on
// machines without a driver (the CPU tests) and without NVRTC (fallback).
#include <dlfcn.h>

#include <cstdio>
#include <map>
#include <mutex>
#include <set>
#include <sstream>

#include "ad_codegen.h"

namespace gn {
namespace {

enum { OP_VAR = 0, OP_PAR, OP_CONST, OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_POW, OP_NEG, OP_SIN,
       OP_COS, OP_LOG, OP_SQRT, OP_EXP };

bool is_binary(int op) { return op >= OP_ADD && op <= OP_DIV; }

std::string lit(double c) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", c);
  std::string s(buf);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return "(" + s + ")";
}

std::string V(int i) { return "v" + std::to_string(i); }

// value-level partials (d entry / d a, d entry / d b): expressions.py:259-285
struct Part {
  std::string fa, fb;
  bool has_b;
};
Part partial(int op, int a, int b, int i, const std::vector<double> &consts) {
  switch (op) {
    case OP_ADD: return {"1.0", "1.0", true};
    case OP_SUB: return {"1.0", "(-1.0)", true};
    case OP_MUL: return {V(b), V(a), true};
    case OP_DIV: return {"(1.0 / " + V(b) + ")", "(-" + V(a) + " / (" + V(b) + " * " + V(b) + "))", true};
    case OP_POW: {
      const double c = consts[b];
      return {"(" + lit(c) + " * powc(" + V(a) + ", " + lit(c - 1.0) + "))", "0.0", false};
    }
    case OP_NEG: return {"(-1.0)", "0.0", false};
    case OP_SIN: return {"cos(" + V(a) + ")", "0.0", false};
    case OP_COS: return {"(-sin(" + V(a) + "))", "0.0", false};
    case OP_LOG: return {"(1.0 / " + V(a) + ")", "0.0", false};
    case OP_SQRT: return {"(0.5 / " + V(i) + ")", "0.0", false};
    default: return {V(i), "0.0", false};  // EXP
  }
}

// accumulation with the interpreter's "absent" semantics: first write
// assigns, later writes add (acc() in ad.cu)
struct Acc {
  std::string prefix;
  std::set<int> have;
  void add(std::ostringstream &o, int k, const std::string &val) {
    const std::string nm = prefix + std::to_string(k);
    if (have.count(k)) {
      o << "    " << nm << " += " << val << ";\n";
    } else {
      o << "    double " << nm << " = " << val << ";\n";
      have.insert(k);
    }
  }
  bool has(int k) const { return have.count(k) > 0; }
};

std::string gen_pattern(const Model::HBlock &b, int id) {
  const int T = static_cast<int>(b.ops.size() / 3);
  const bool obj = b.kind == 0;
  auto op = [&](int i) { return b.ops[3 * i]; };
  auto A = [&](int i) { return b.ops[3 * i + 1]; };
  auto Bv = [&](int i) { return b.ops[3 * i + 2]; };
  const int nfirst = static_cast<int>(b.first.size());
  const int npairs = static_cast<int>(b.pairs.size() / 2);
  std::vector<int> sweep;
  for (int p = 0; p < npairs; ++p)
    if (std::find(sweep.begin(), sweep.end(), b.pairs[2 * p + 1]) == sweep.end()) sweep.push_back(b.pairs[2 * p + 1]);
  std::sort(sweep.begin(), sweep.end());
  const unsigned val_bit = obj ? GN_AD_F : GN_AD_C;
  const unsigned first_bit = obj ? GN_AD_GRAD : GN_AD_JAC;

  std::ostringstream o;
  o << "__device__ __forceinline__ void pat_" << id
    << "(long long r, long long R, const int *__restrict__ vi, const double *__restrict__ pa, "
       "const int *__restrict__ tg, const double *__restrict__ x, const double *__restrict__ y, "
       "const double *__restrict__ cs, double obj_w, unsigned what, double *__restrict__ out, "
       "const int *__restrict__ js, double *__restrict__ jac, int jdirect, int *__restrict__ flags) {\n";
  // record data: coalesced SoA loads of the variable indices and parameters
  std::set<int> vs, ps;
  for (int i = 0; i < T; ++i) {
    if (op(i) == OP_VAR) vs.insert(A(i));
    if (op(i) == OP_PAR) ps.insert(A(i));
  }
  for (int s : vs) o << "  const double X" << s << " = x[__ldg(vi + " << s << " * R + r)];\n";
  for (int p : ps) o << "  const double P" << p << " = __ldg(pa + " << p << " * R + r);\n";
  // ---- forward (expressions.py:222-254)
  for (int i = 0; i < T; ++i) {
    const int a = A(i), bb = Bv(i);
    std::string e;
    switch (op(i)) {
      case OP_VAR: e = "X" + std::to_string(a); break;
      case OP_PAR: e = "P" + std::to_string(a); break;
      case OP_CONST: e = lit(b.consts[bb]); break;
      case OP_ADD: e = V(a) + " + " + V(bb); break;
      case OP_SUB: e = V(a) + " - " + V(bb); break;
      case OP_MUL: e = V(a) + " * " + V(bb); break;
      case OP_DIV: e = V(a) + " / " + V(bb); break;
      case OP_POW: e = "powc(" + V(a) + ", " + lit(b.consts[bb]) + ")"; break;
      case OP_NEG: e = "-" + V(a); break;
      case OP_SIN: e = "sin(" + V(a) + ")"; break;
      case OP_COS: e = "cos(" + V(a) + ")"; break;
      case OP_LOG: e = "log(" + V(a) + ")"; break;
      case OP_SQRT: e = "sqrt(" + V(a) + ")"; break;
      default: e = "exp(" + V(a) + ")"; break;
    }
    o << "  const double " << V(i) << " = " << e << ";\n";
  }
  o << "  const bool need_val = (what & " << val_bit << "u) != 0u;\n";
  o << "  const bool need_first = (what & " << first_bit << "u) != 0u;\n";
  o << "  const bool need_hess = " << (npairs > 0 ? "(what & 16u) != 0u" : "false") << ";\n";
  o << "  if (need_val) out[r] = " << V(b.out) << ";\n";
  o << "  if (!need_first && !need_hess) return;\n";
  // ---- reverse sweep (expressions.py:287-314)
  std::set<int> amask{b.out};
  Acc adj{"a", {}};
  o << "  {\n    double a" << b.out << " = 1.0;\n";
  adj.have.insert(b.out);
  Acc g{"g", {}};
  for (int i = T - 1; i >= 0; --i) {
    if (!amask.count(i)) continue;
    const int e = op(i);
    if (e == OP_VAR) {
      g.add(o, A(i), "a" + std::to_string(i));
      continue;
    }
    if (e == OP_PAR || e == OP_CONST) continue;
    const Part p = partial(e, A(i), Bv(i), i, b.consts);
    adj.add(o, A(i), p.fa + " * a" + std::to_string(i));
    amask.insert(A(i));
    if (p.has_b) {
      adj.add(o, Bv(i), p.fb + " * a" + std::to_string(i));
      amask.insert(Bv(i));
    }
  }
  o << "    if (need_first) {\n";
  if (!obj) {
    // every Jacobian slot has exactly one contributor (checked at upload):
    // write the scaled value straight into J, no contribution round trip
    // the non-finite check of J rides along (no separate pass over J)
    o << "      if (jdirect) {\n        const double jsc = cs ? cs[__ldg(tg + r)] : 1.0;\n"
         "        bool jbad = false;\n";
    for (int k = 0; k < nfirst; ++k) {
      const int s = b.first[k];
      o << "        { const double jv = " << (g.has(s) ? "g" + std::to_string(s) : std::string("0.0"))
        << " * jsc; jbad |= !isfinite(jv); jac[__ldg(js + " << k << " * R + r)] = jv; }\n";
    }
    o << "        if (jbad) atomicOr(flags, " << GN_AD_JAC << ");\n";
    o << "      } else {\n";
  }
  for (int k = 0; k < nfirst; ++k) {
    const int s = b.first[k];
    o << "      out[" << (1 + k) << " * R + r] = " << (g.has(s) ? "g" + std::to_string(s) : std::string("0.0"))
      << ";\n";
  }
  if (!obj) o << "      }\n";
  o << "    }\n";
  if (npairs > 0) {
    o << "    if (!need_hess) return;\n";
    // ---- Hessian columns (expressions.py:316-409)
    if (obj)
      o << "    const double w = obj_w;\n";
    else
      o << "    const int tt = __ldg(tg + r);\n    const double w = y[tt] * (cs ? cs[tt] : 1.0);\n";
    const int hbase = 1 + nfirst;
    for (int ts : sweep) {
      o << "    {\n";
      std::set<int> dmask;
      // forward tangent
      for (int i = 0; i < T; ++i) {
        const int e = op(i);
        if (e == OP_VAR) {
          if (A(i) == ts) {
            o << "    const double d" << i << " = 1.0;\n";
            dmask.insert(i);
          }
          continue;
        }
        if (e == OP_PAR || e == OP_CONST) continue;
        const bool ha = dmask.count(A(i)) > 0;
        const bool hb = is_binary(e) && dmask.count(Bv(i)) > 0;
        if (!ha && !hb) continue;
        const Part p = partial(e, A(i), Bv(i), i, b.consts);
        std::string t;
        if (ha) t = p.fa + " * d" + std::to_string(A(i));
        if (hb) t = ha ? t + " + " + p.fb + " * d" + std::to_string(Bv(i)) : p.fb + " * d" + std::to_string(Bv(i));
        o << "    const double d" << i << " = " << t << ";\n";
        dmask.insert(i);
      }
      // reverse of the tangent
      Acc adot{"t", {}};
      Acc hcol{"h", {}};
      std::set<int> admask;
      for (int i = T - 1; i >= 0; --i) {
        const bool hai = amask.count(i) > 0;
        const bool hadi = admask.count(i) > 0;
        if (!hai && !hadi) continue;
        const int e = op(i);
        if (e == OP_VAR) {
          if (hadi) hcol.add(o, A(i), "t" + std::to_string(i));
          continue;
        }
        if (e == OP_PAR || e == OP_CONST) continue;
        const int a = A(i), bb = Bv(i);
        const Part p = partial(e, a, bb, i, b.consts);
        const bool hda = dmask.count(a) > 0;
        const bool hdb = is_binary(e) && dmask.count(bb) > 0;
        const std::string da = "d" + std::to_string(a), db = "d" + std::to_string(bb);
        std::string dfa, dfb;
        bool hdfa = false, hdfb = false;
        switch (e) {
          case OP_MUL:
            if (hdb) { dfa = db; hdfa = true; }
            if (hda) { dfb = da; hdfb = true; }
            break;
          case OP_DIV: {
            const std::string vb = V(bb);
            if (hdb) { dfa = "(-" + db + " / (" + vb + " * " + vb + "))"; hdfa = true; }
            if (hda) { dfb = "(-" + da + " / (" + vb + " * " + vb + "))"; hdfb = true; }
            if (hdb) {
              const std::string t2 = "(2.0 * " + V(a) + " * " + db + " / (" + vb + " * " + vb + " * " + vb + "))";
              dfb = hdfb ? "(" + dfb + " + " + t2 + ")" : t2;
              hdfb = true;
            }
            break;
          }
          case OP_POW: {
            const double c = b.consts[bb];
            if (hda && c != 1.0) {
              dfa = "(" + lit(c * (c - 1.0)) + " * powc(" + V(a) + ", " + lit(c - 2.0) + ") * " + da + ")";
              hdfa = true;
            }
            break;
          }
          case OP_SIN: if (hda) { dfa = "(-sin(" + V(a) + ") * " + da + ")"; hdfa = true; } break;
          case OP_COS: if (hda) { dfa = "(-cos(" + V(a) + ") * " + da + ")"; hdfa = true; } break;
          case OP_LOG: if (hda) { dfa = "(-" + da + " / (" + V(a) + " * " + V(a) + "))"; hdfa = true; } break;
          case OP_SQRT: if (hda) { dfa = "(-0.25 * " + da + " / (" + V(a) + " * " + V(i) + "))"; hdfa = true; } break;
          case OP_EXP: if (hda) { dfa = "(" + V(i) + " * " + da + ")"; hdfa = true; } break;
          default: break;
        }
        const std::string ai = "a" + std::to_string(i), ti = "t" + std::to_string(i);
        if (hai && hdfa) { adot.add(o, a, dfa + " * " + ai); admask.insert(a); }
        if (hadi) { adot.add(o, a, p.fa + " * " + ti); admask.insert(a); }
        if (p.has_b) {
          if (hai && hdfb) { adot.add(o, bb, dfb + " * " + ai); admask.insert(bb); }
          if (hadi) { adot.add(o, bb, p.fb + " * " + ti); admask.insert(bb); }
        }
      }
      for (int k = 0; k < npairs; ++k) {
        if (b.pairs[2 * k + 1] != ts) continue;
        const int a = b.pairs[2 * k];
        std::string c = "0.0";
        if (hcol.has(a)) {
          std::string fac = "1.0";
          if (a != ts)
            fac = "(__ldg(vi + " + std::to_string(a) + " * R + r) == __ldg(vi + " + std::to_string(ts) +
                  " * R + r) ? 2.0 : 1.0)";
          c = std::string(obj ? "(obj_w == 0.0 ? 0.0 : " : "(") + "(w * " + fac + ") * h" + std::to_string(a) + ")";
        }
        o << "    out[" << (hbase + k) << " * R + r] = " << c << ";\n";
      }
      o << "    }\n";
    }
  }
  o << "  }\n}\n";
  return o.str();
}

const char *kPrelude = R"(
// numpy's scalar fast paths for array ** c (ad.cu powc)
__device__ __forceinline__ double powc(double v, double c) {
  if (c == 2.0) return v * v;
  if (c == 1.0) return v;
  if (c == 0.0) return 1.0;
  if (c == 0.5) return sqrt(v);
  if (c == -1.0) return 1.0 / v;
  return pow(v, c);
}
struct GenBlk { long long cta_begin, R, var_off, par_off, tgt_off, contrib_off, jslot_off; int pattern, pad; };
)";

// ---------------------------------------------------------- NVRTC / driver
typedef int (*nvrtcCreateProgram_t)(void **, const char *, const char *, int, const char *const *,
                                    const char *const *);
typedef int (*nvrtcCompileProgram_t)(void *, int, const char *const *);
typedef int (*nvrtcGetSize_t)(void *, size_t *);
typedef int (*nvrtcGetData_t)(void *, char *);
typedef int (*nvrtcDestroyProgram_t)(void **);
typedef int (*cuModuleLoadData_t)(void **, const void *);
typedef int (*cuModuleGetFunction_t)(void **, void *, const char *);
typedef int (*cuLaunchKernel_t)(void *, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                                unsigned, void *, void **, void **);
typedef int (*cuFuncSetAttribute_t)(void *, int, int);

struct Api {
  bool ok = false;
  std::string why;
  nvrtcCreateProgram_t create = nullptr;
  nvrtcCompileProgram_t compile = nullptr;
  nvrtcGetSize_t cubin_size = nullptr, log_size = nullptr;
  nvrtcGetData_t cubin = nullptr, log = nullptr;
  nvrtcDestroyProgram_t destroy = nullptr;
  cuModuleLoadData_t load = nullptr;
  cuModuleGetFunction_t getfn = nullptr;
  cuLaunchKernel_t launch = nullptr;
};

Api &api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    void *nv = nullptr;
    for (const char *nm : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"})
      if ((nv = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
    void *cu = dlopen("libcuda.so.1", RTLD_NOW | RTLD_LOCAL);
    if (!nv || !cu) {
      a.why = !nv ? "libnvrtc not found" : "libcuda not found";
      return;
    }
    a.create = reinterpret_cast<nvrtcCreateProgram_t>(dlsym(nv, "nvrtcCreateProgram"));
    a.compile = reinterpret_cast<nvrtcCompileProgram_t>(dlsym(nv, "nvrtcCompileProgram"));
    a.cubin_size = reinterpret_cast<nvrtcGetSize_t>(dlsym(nv, "nvrtcGetCUBINSize"));
    a.cubin = reinterpret_cast<nvrtcGetData_t>(dlsym(nv, "nvrtcGetCUBIN"));
    a.log_size = reinterpret_cast<nvrtcGetSize_t>(dlsym(nv, "nvrtcGetProgramLogSize"));
    a.log = reinterpret_cast<nvrtcGetData_t>(dlsym(nv, "nvrtcGetProgramLog"));
    a.destroy = reinterpret_cast<nvrtcDestroyProgram_t>(dlsym(nv, "nvrtcDestroyProgram"));
    a.load = reinterpret_cast<cuModuleLoadData_t>(dlsym(cu, "cuModuleLoadData"));
    a.getfn = reinterpret_cast<cuModuleGetFunction_t>(dlsym(cu, "cuModuleGetFunction"));
    a.launch = reinterpret_cast<cuLaunchKernel_t>(dlsym(cu, "cuLaunchKernel"));
    a.ok = a.create && a.compile && a.cubin_size && a.cubin && a.log_size && a.log && a.destroy &&
           a.load && a.getfn && a.launch;
    if (!a.ok) a.why = "NVRTC / driver entry points missing";
  });
  return a;
}

std::mutex g_mu;
std::map<std::string, void *> g_cache;   // generated source -> CUfunction

}  // namespace

std::string pattern_source(const Model &M, std::vector<int> &pattern_of) {
  std::map<std::string, int> uniq;   // device function body (name-less) -> pattern id
  std::vector<std::string> bodies;
  pattern_of.assign(M.blocks.size(), -1);
  for (size_t bi = 0; bi < M.blocks.size(); ++bi) {
    const std::string key = gen_pattern(M.blocks[bi], 0);
    auto it = uniq.find(key);
    if (it == uniq.end()) {
      const int id = static_cast<int>(bodies.size());
      uniq.emplace(key, id);
      bodies.push_back(gen_pattern(M.blocks[bi], id));
      pattern_of[bi] = id;
    } else {
      pattern_of[bi] = it->second;
    }
  }
  std::ostringstream o;
  o << kPrelude;
  for (auto &b : bodies) o << b;
  o << "extern \"C\" __global__ void __launch_bounds__(" << kPatternThreads
    << ") gn_ad_patterns(const GenBlk *__restrict__ blks, int nblk, const int *__restrict__ var_idx, "
       "const double *__restrict__ params, const int *__restrict__ targets, const double *__restrict__ x, "
       "const double *__restrict__ y, const double *__restrict__ cs, double obj_w, unsigned what, "
       "double *__restrict__ contrib, const int *__restrict__ jslots, double *__restrict__ jac, int jdirect,\n"
       "    const long long *__restrict__ bs, const double *__restrict__ objw_b, int *__restrict__ flags) {\n"
       "  // instance batches: blockIdx.y = instance, bs = strides (x, y and con_scale, contrib, params, jac)\n"
       "  if (bs) {\n"
       "    const long long bi = blockIdx.y;\n"
       "    x += bi * bs[0];\n"
       "    if (y) y += bi * bs[1];\n"
       "    if (cs) cs += bi * bs[1];\n"
       "    contrib += bi * bs[2];\n"
       "    params += bi * bs[3];\n"
       "    if (jac) jac += bi * bs[4];\n"
       "    if (objw_b) obj_w = objw_b[bi];\n"
       "    flags += bi;\n"
       "  }\n"
       "  int lo = 0, hi = nblk - 1;\n"
       "  while (lo < hi) {\n"
       "    const int mid = (lo + hi + 1) >> 1;\n"
       "    if (__ldg(&blks[mid].cta_begin) <= (long long)blockIdx.x) lo = mid; else hi = mid - 1;\n"
       "  }\n"
       "  const GenBlk B = blks[lo];\n"
       "  const long long r = ((long long)blockIdx.x - B.cta_begin) * blockDim.x + threadIdx.x;\n"
       "  if (r >= B.R) return;\n"
       "  const int *vi = var_idx + B.var_off;\n"
       "  const double *pa = params + B.par_off;\n"
       "  const int *tg = targets + B.tgt_off;\n"
       "  double *out = contrib + B.contrib_off;\n"
       "  const int *js = B.jslot_off >= 0 ? jslots + B.jslot_off : jslots;\n"
       "  switch (B.pattern) {\n";
  for (size_t id = 0; id < bodies.size(); ++id)
    o << "    case " << id << ": pat_" << id << "(r, B.R, vi, pa, tg, x, y, cs, obj_w, what, out, js, jac, jdirect, flags); break;\n";
  o << "    default: break;\n  }\n}\n";
  return o.str();
}

void *compile_patterns(const std::string &src, std::string &err) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(src);
    if (it != g_cache.end()) return it->second;
  }
  Api &a = api();
  if (!a.ok) {
    err = a.why;
    return nullptr;
  }
  void *prog = nullptr;
  if (a.create(&prog, src.c_str(), "gn_ad_patterns.cu", 0, nullptr, nullptr) != 0) {
    err = "nvrtcCreateProgram failed";
    return nullptr;
  }
  const char *opts[] = {"-arch=sm_100a", "--std=c++17", "-default-device", "-lineinfo"};
  const int rc = a.compile(prog, 4, opts);
  if (rc != 0) {
    size_t n = 0;
    a.log_size(prog, &n);
    std::string log(n, '\0');
    if (n) a.log(prog, &log[0]);
    err = "NVRTC compile failed: " + log.substr(0, 2000);
    a.destroy(&prog);
    return nullptr;
  }
  size_t n = 0;
  a.cubin_size(prog, &n);
  std::string bin(n, '\0');
  a.cubin(prog, &bin[0]);
  a.destroy(&prog);
  void *mod = nullptr, *fn = nullptr;
  if (a.load(&mod, bin.data()) != 0 || a.getfn(&fn, mod, "gn_ad_patterns") != 0) {
    err = "cuModuleLoadData / cuModuleGetFunction failed";
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  g_cache.emplace(src, fn);
  return fn;
}

bool launch_patterns(void *fn, unsigned grid, void *stream, void **args, unsigned batch) {
  return api().launch(fn, grid, batch, 1, kPatternThreads, 1, 1, 0, stream, args, nullptr) == 0;
}

}  // namespace gn
