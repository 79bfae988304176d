// stencil_expr.cu — expression stencils compiled at run time with NVRTC for
// sm_100a (NEXT #4, "offset list + expression -> NVRTC-compiled kernel";
// reading R24 of DESIGN.md).
//
// The discovery pass turns a Fortran loop nest into a stencil.apply whose
// region is the loop body's right-hand side over constant-offset accesses
// (PAPER.md:107-126, 149-191, 185). Here that right-hand side is given as text
// over a(dy, dx) accesses, numeric literals, + - * /, unary signs and
// parentheses. It is validated and translated token by token (accesses become
// a load macro, every literal becomes a double literal), so the generated
// source contains nothing but the expression grammar; it is compiled once per
// (expression, device) with --fmad=false (every operation one IEEE rounding,
// none contracted — R11) and cached. NVRTC is loaded with dlopen on first use,
// so the library itself has no link-time dependency on it.
#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <cctype>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace st {

namespace {

// ------------------------------------------------------------- translation ---
// Returns the C expression (accesses -> A(dy,dx), literals -> double literals)
// and the halo R, or an error message.
// fused: accesses are f<i>(dz, dy, dx) (input field i) and k<j> names the
// per-plane coefficient j; max_field / max_coef report the highest indices used.
bool translate(const char* expr, std::string* out, int64_t* R, int* dims, std::string* err, bool fused = false,
               int* max_field = nullptr, int* max_coef = nullptr) {
  out->clear();
  *R = -1;
  *dims = 0;
  if (max_field) *max_field = -1;
  if (max_coef) *max_coef = -1;
  const size_t n = std::strlen(expr);
  int depth = 0;
  size_t i = 0;
  bool expect_operand = true;  // grammar: operand (op operand)*, with unary signs and parentheses
  while (i < n) {
    const char ch = expr[i];
    if (std::isspace((unsigned char)ch)) { ++i; continue; }
    if (fused && ch == 'k') {  // k<j>: per-plane coefficient
      if (!expect_operand || i + 1 >= n || expr[i + 1] < '0' || expr[i + 1] > '7' ||
          (i + 2 < n && (std::isalnum((unsigned char)expr[i + 2]) || expr[i + 2] == '.'))) {
        *err = "bad coefficient name (k0..k7)";
        return false;
      }
      const int jk = expr[i + 1] - '0';
      if (max_coef) *max_coef = std::max(*max_coef, jk);
      *out += "K" + std::to_string(jk);
      i += 2;
      expect_operand = false;
      continue;
    }
    if ((!fused && ch == 'a') || (fused && ch == 'f')) {  // a(dy, dx) / a(dz, dy, dx) / f<i>(dz, dy, dx)
      size_t j = i + 1;
      int field = -1;
      if (fused) {
        if (j >= n || expr[j] < '0' || expr[j] > '7') { *err = "bad field name (f0..f7)"; return false; }
        field = expr[j] - '0';
        ++j;
        if (max_field) *max_field = std::max(*max_field, field);
      }
      auto skip = [&] { while (j < n && std::isspace((unsigned char)expr[j])) ++j; };
      auto integer = [&](long* v) -> bool {
        skip();
        size_t k = j;
        if (k < n && (expr[k] == '-' || expr[k] == '+')) ++k;
        if (k >= n || !std::isdigit((unsigned char)expr[k])) return false;
        while (k < n && std::isdigit((unsigned char)expr[k])) ++k;
        *v = std::strtol(std::string(expr + j, k - j).c_str(), nullptr, 10);
        j = k;
        return true;
      };
      skip();
      if (!expect_operand || j >= n || expr[j] != '(') { *err = "bad access (expected a(dy, dx) or a(dz, dy, dx))"; return false; }
      ++j;
      std::vector<long> idx;
      for (;;) {
        long v = 0;
        if (!integer(&v)) { *err = "bad access offset"; return false; }
        idx.push_back(v);
        skip();
        if (j < n && expr[j] == ',') { ++j; continue; }
        if (j < n && expr[j] == ')') { ++j; break; }
        *err = "bad access (expected ',' or ')')";
        return false;
      }
      if (idx.size() != 2 && idx.size() != 3) { *err = "an access has 2 (dy, dx) or 3 (dz, dy, dx) offsets"; return false; }
      if (fused && idx.size() != 3) { *err = "field accesses are f<i>(dz, dy, dx)"; return false; }
      if (*dims == 0) *dims = (int)idx.size();
      if ((int)idx.size() != *dims) { *err = "all accesses must have the same number of offsets"; return false; }
      std::string m = fused ? "F" + std::to_string(field) + "(" : std::string("A(");
      for (size_t q = 0; q < idx.size(); ++q) {
        if (std::labs(idx[q]) > kStencilMaxOffset) { *err = "access offset beyond the supported halo"; return false; }
        *R = std::max<int64_t>(*R, std::labs(idx[q]));
        m += (q ? "," : "") + std::to_string(idx[q]);
      }
      *out += m + ")";
      i = j;
      expect_operand = false;
      continue;
    }
    if (std::isdigit((unsigned char)ch) || ch == '.') {  // digits [. digits] [(e|E) [+-] digits]
      if (!expect_operand) { *err = "literal where an operator was expected"; return false; }
      size_t j = i;
      bool point = false, expo = false, digits = false;
      while (j < n && std::isdigit((unsigned char)expr[j])) { ++j; digits = true; }
      if (j < n && expr[j] == '.') {
        point = true;
        ++j;
        while (j < n && std::isdigit((unsigned char)expr[j])) { ++j; digits = true; }
      }
      if (!digits) { *err = "bad numeric literal"; return false; }
      if (j < n && (expr[j] == 'e' || expr[j] == 'E')) {
        expo = true;
        size_t k = j + 1;
        if (k < n && (expr[k] == '+' || expr[k] == '-')) ++k;
        if (k >= n || !std::isdigit((unsigned char)expr[k])) { *err = "bad exponent"; return false; }
        while (k < n && std::isdigit((unsigned char)expr[k])) ++k;
        j = k;
      }
      std::string lit(expr + i, j - i);
      if (!point && !expo) lit += ".0";  // binary64, never C integer arithmetic
      if (lit[0] == '.') lit = "0" + lit;
      *out += lit;
      i = j;
      expect_operand = false;
      continue;
    }
    if (ch == '(') {
      if (!expect_operand) { *err = "'(' where an operator was expected"; return false; }
      ++depth;
      *out += '(';
    } else if (ch == ')') {
      if (expect_operand || --depth < 0) { *err = "unbalanced or empty parentheses"; return false; }
      *out += ')';
    } else if (ch == '+' || ch == '-') {
      *out += ' ';
      *out += ch;  // binary, or unary when an operand is expected
      *out += ' ';
      expect_operand = true;
    } else if (ch == '*' || ch == '/') {
      if (expect_operand) { *err = "operator without a left operand"; return false; }
      *out += ' ';
      *out += ch;
      *out += ' ';
      expect_operand = true;
    } else {
      *err = std::string("unsupported character '") + ch + "'";
      return false;
    }
    ++i;
  }
  if (expect_operand || depth != 0) { *err = "incomplete expression"; return false; }
  if (*R < 0) { *err = "the expression has no field access"; return false; }
  return true;
}

const char* kKernelTemplate = R"(
#define A(dy, dx) __ldg(p + (long long)(dy) * ld + (dx))
extern "C" __global__ void __launch_bounds__(128)
st_expr_kernel(const double* __restrict__ src, double* __restrict__ dst, long long nx, long long ny,
               long long ld, long long R) {
  const long long x = R + (long long)blockIdx.x * 32 + threadIdx.x;
  if (x >= R + nx) return;
  const long long yb = R + (long long)blockIdx.y * 16 + threadIdx.y;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const long long y = yb + 4 * k;
    if (y >= R + ny) return;
    const double* p = src + y * ld + x;
    dst[y * ld + x] = (@EXPR@);
  }
}
)";

// 2-D, streamed down y (even pitch, 16-byte aligned buffers): a thread owns one
// 16-byte column pair (x, x+1) of a chunk of rows, every distinct pair offset m
// (column x + 2m) the expression reads becomes a register queue of double2 over
// its dy range, and the two outputs are stored as one 16-byte store — the
// structure of the hand-written Listing-1 sweep, derived from the expression's
// offsets (Listing 1: 3 pair loads per 2 points instead of 4 loads per point).
// Pairs outside [0, ld-2] are clamped: they only feed outputs outside the
// interior, which are not stored. Same tags as the fused template below.
const char* kKernelTemplate2dStream = R"(
extern "C" __global__ void __launch_bounds__(128)
st_expr_kernel(const double* __restrict__ src, double* __restrict__ dst, long long nx, long long ny,
               long long ld, long long R, long long yc) {
  const long long xa = (R & ~1LL) + 2 * ((long long)blockIdx.x * 128 + threadIdx.x);
  const unsigned lane = threadIdx.x & 31;
  // (no early exit: every lane takes part in the neighbour shuffles; lanes past the row
  // load clamped pairs and store nothing)
  const bool w0 = xa >= R && xa < R + nx, w1 = xa + 1 < R + nx;
  const long long y0 = R + (long long)blockIdx.y * yc;
  const long long y1 = (y0 + yc < R + ny) ? y0 + yc : R + ny;
#define PCOL(m) ((xa + 2 * (m) < 0) ? 0 : (xa + 2 * (m) > ld - 2) ? ld - 2 : xa + 2 * (m))
#define PLD(m, row) __ldg(reinterpret_cast<const double2*>(src + (row) * ld + PCOL(m)))
#define SHF(v, d) __hiloint2double(__shfl_down_sync(0xffffffffu, __double2hiint(v), d), \
                                   __shfl_down_sync(0xffffffffu, __double2loint(v), d))
#define SHB(v, d) __hiloint2double(__shfl_up_sync(0xffffffffu, __double2hiint(v), d), \
                                   __shfl_up_sync(0xffffffffu, __double2loint(v), d))
@DECL@
@PRO@
#pragma unroll 1
  for (long long y = y0; y < y1; ++y) {
@LOAD@
    const double o0 = (@BODY@);
@SHIFT@
    double* d = dst + y * ld + xa;
    if (w0 && w1) *reinterpret_cast<double2*>(d) = make_double2(o0, o1);
    else if (w1) d[1] = o1;
    else if (w0) d[0] = o0;
  }
}
)";

// Fused region: several outputs from several fields in one pass.
// Code generation streams z: a thread owns one (x, y) column of a chunk of
// planes, and every distinct (field, dy, dx) column the region reads becomes a
// register queue over its dz range — one new load per column and plane instead
// of one per access (e.g. 27 -> 18 loads per point for the PW advection).
// @DECL@ queues, @PRO@ their prologue, @LOAD@ the newest plane, @COEF@ the
// per-plane coefficients, @BODY@ one store per output, @SHIFT@ the rotation.
const char* kKernelTemplateFused = R"(
struct Ptrs { const double* in[8]; double* out[8]; const double* k[8]; };
extern "C" __global__ void __launch_bounds__(128)
st_expr_kernel(const __grid_constant__ Ptrs P, long long nx, long long ny, long long nz, long long ldx,
               long long R, long long zc) {
  const long long x = R + (long long)blockIdx.x * 32 + threadIdx.x;
  const long long y = R + (long long)blockIdx.y * 4 + threadIdx.y;
  if (x >= R + nx || y >= R + ny) return;
  const long long plane = (ny + 2 * R) * ldx;
  const long long col = y * ldx + x;
  const long long z0 = R + (long long)blockIdx.z * zc;
  const long long z1 = (z0 + zc < R + nz) ? z0 + zc : R + nz;
@DECL@
@PRO@
#pragma unroll 1
  for (long long z = z0; z < z1; ++z) {
@LOAD@
@COEF@
    const long long o = z * plane + col;
@BODY@
@SHIFT@
  }
}
)";

// The same with column pairs (even pitch, 16-byte aligned fields): a thread owns
// the pair (x, x+1) of its row, queues hold double2 per (field, dy, pair offset m),
// and every output is one 16-byte store (see the 2-D pair template).
const char* kKernelTemplateFusedPair = R"(
struct Ptrs { const double* in[8]; double* out[8]; const double* k[8]; };
extern "C" __global__ void __launch_bounds__(128)
st_expr_kernel(const __grid_constant__ Ptrs P, long long nx, long long ny, long long nz, long long ldx,
               long long R, long long zc) {
  const long long x = (R & ~1LL) + 2 * ((long long)blockIdx.x * 32 + threadIdx.x);
  const long long y = R + (long long)blockIdx.y * 4 + threadIdx.y;
  if (x >= R + nx || y >= R + ny) return;
  const bool w0 = x >= R, w1 = x + 1 < R + nx;
#define PCOL(m) ((x + 2 * (m) < 0) ? 0LL : (x + 2 * (m) > ldx - 2) ? ldx - 2 : x + 2 * (m))
  const long long plane = (ny + 2 * R) * ldx;
  const long long col = y * ldx + x;
  const long long z0 = R + (long long)blockIdx.z * zc;
  const long long z1 = (z0 + zc < R + nz) ? z0 + zc : R + nz;
@DECL@
@PRO@
#pragma unroll 1
  for (long long z = z0; z < z1; ++z) {
@LOAD@
@COEF@
    const long long o = z * plane + col;
@BODY@
@SHIFT@
  }
}
)";

// ------------------------------------------------------------------- NVRTC ---
struct Nvrtc {
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  bool ok = false;
};

const Nvrtc& nvrtc() {
  static Nvrtc f;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"})
      if ((h = dlopen(name, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) return;
    f.create = reinterpret_cast<decltype(f.create)>(dlsym(h, "nvrtcCreateProgram"));
    f.compile = reinterpret_cast<decltype(f.compile)>(dlsym(h, "nvrtcCompileProgram"));
    f.log_size = reinterpret_cast<decltype(f.log_size)>(dlsym(h, "nvrtcGetProgramLogSize"));
    f.log = reinterpret_cast<decltype(f.log)>(dlsym(h, "nvrtcGetProgramLog"));
    f.cubin_size = reinterpret_cast<decltype(f.cubin_size)>(dlsym(h, "nvrtcGetCUBINSize"));
    f.cubin = reinterpret_cast<decltype(f.cubin)>(dlsym(h, "nvrtcGetCUBIN"));
    f.destroy = reinterpret_cast<decltype(f.destroy)>(dlsym(h, "nvrtcDestroyProgram"));
    f.ok = f.create && f.compile && f.log_size && f.log && f.cubin_size && f.cubin && f.destroy;
  });
  return f;
}

using PFN_moduleLoadData = CUresult (*)(CUmodule*, const void*);
using PFN_moduleGetFunction = CUresult (*)(CUfunction*, CUmodule, const char*);
using PFN_launchKernel = CUresult (*)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                                      unsigned, CUstream, void**, void**);
struct Driver {
  PFN_moduleLoadData load = nullptr;
  PFN_moduleGetFunction get = nullptr;
  PFN_launchKernel launch = nullptr;
};

st_status driver(Driver* d) {
  static Driver drv;
  static st_status st = ST_OK;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuModuleLoadData", &p, cudaEnableDefault, &q) == cudaSuccess && p)
      drv.load = reinterpret_cast<PFN_moduleLoadData>(p);
    if (cudaGetDriverEntryPoint("cuModuleGetFunction", &p, cudaEnableDefault, &q) == cudaSuccess && p)
      drv.get = reinterpret_cast<PFN_moduleGetFunction>(p);
    if (cudaGetDriverEntryPoint("cuLaunchKernel", &p, cudaEnableDefault, &q) == cudaSuccess && p)
      drv.launch = reinterpret_cast<PFN_launchKernel>(p);
    if (!drv.load || !drv.get || !drv.launch) st = ST_ECUDA;
  });
  ST_RETURN_IF(st != ST_OK, st, "driver entry points for module loading unavailable");
  *d = drv;
  return ST_OK;
}

std::mutex g_cache_mu;
std::map<std::string, CUfunction> g_cache;  // (device, translated expression) -> kernel

st_status compiled_kernel(const std::string& cexpr, int dims, int dev, CUfunction* fn) {
  const std::string key = std::to_string(dev) + "|" + std::to_string(dims) + "|" + cexpr;
  std::lock_guard<std::mutex> lock(g_cache_mu);
  auto it = g_cache.find(key);
  if (it != g_cache.end()) {
    *fn = it->second;
    return ST_OK;
  }
  const Nvrtc& f = nvrtc();
  ST_RETURN_IF(!f.ok, ST_ENOTSUP, "NVRTC (libnvrtc.so.12) is not available");
  std::string src;
  if (dims >= 4) {  // cexpr = DECL \x1f PRO \x1f LOAD \x1f COEF \x1f BODY \x1f SHIFT
    src = dims == 4 ? kKernelTemplateFused : dims == 5 ? kKernelTemplate2dStream : kKernelTemplateFusedPair;
    size_t start = 0;
    for (const char* tag : {"@DECL@", "@PRO@", "@LOAD@", "@COEF@", "@BODY@", "@SHIFT@"}) {
      if (src.find(tag) == std::string::npos) {  // (the 2-D template has no @COEF@)
        const size_t cut = cexpr.find('\x1f', start);
        start = cut == std::string::npos ? cexpr.size() : cut + 1;
        continue;
      }
      const size_t cut = cexpr.find('\x1f', start);
      const std::string part = cexpr.substr(start, cut == std::string::npos ? std::string::npos : cut - start);
      src.replace(src.find(tag), std::strlen(tag), part);
      start = cut == std::string::npos ? cexpr.size() : cut + 1;
    }
  } else {
    src = kKernelTemplate;  // 2-D (3-D single-field expressions run as one-field fused regions)
    src.replace(src.find("@EXPR@"), 6, cexpr);
  }
  nvrtcProgram prog;
  ST_RETURN_IF(f.create(&prog, src.c_str(), "st_expr.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS, ST_EINTERNAL,
               "nvrtcCreateProgram failed");
  const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "--std=c++17", "-default-device"};
  const nvrtcResult cr = f.compile(prog, 4, opts);
  if (cr != NVRTC_SUCCESS) {
    size_t ls = 0;
    f.log_size(prog, &ls);
    std::string log(ls, '\0');
    f.log(prog, &log[0]);
    f.destroy(&prog);
    set_error("NVRTC compile failed: %s", log.c_str());
    return ST_EINVAL;
  }
  size_t cs = 0;
  f.cubin_size(prog, &cs);
  std::vector<char> cubin(cs);
  f.cubin(prog, cubin.data());
  f.destroy(&prog);
  Driver d;
  ST_TRY(driver(&d));
  ST_CHECK_CUDA(cudaFree(nullptr));  // make the primary context current
  CUmodule mod;
  ST_RETURN_IF(d.load(&mod, cubin.data()) != CUDA_SUCCESS, ST_ECUDA, "cuModuleLoadData failed");
  CUfunction k;
  ST_RETURN_IF(d.get(&k, mod, "st_expr_kernel") != CUDA_SUCCESS, ST_ECUDA, "cuModuleGetFunction failed");
  g_cache.emplace(key, k);  // the module stays loaded for the process lifetime (one per expression)
  *fn = k;
  return ST_OK;
}

}  // namespace

st_status stencil_expr_translate(const char* expr, std::string* cexpr, int64_t* R, int* dims) {
  std::string err;
  ST_RETURN_IF(!translate(expr, cexpr, R, dims, &err), ST_EINVAL, "expression: %s", err.c_str());
  return ST_OK;
}

namespace {
// The y-streaming kernel's pieces for a translated 2-D expression (tokens A(dy,dx)):
// one register queue per distinct dx over the dy range it is read at.
std::string gen_2d_stream(const std::string& cexpr) {
  auto enc = [](long v) { return (v < 0 ? "m" : "p") + std::to_string(std::labs(v)); };
  auto fdiv2 = [](long v) { return v >= 0 ? v / 2 : -((-v + 1) / 2); };  // floor(v / 2)
  auto scan = [&](auto&& on_access) {
    std::string outs;
    size_t i = 0;
    while (i < cexpr.size()) {
      if (cexpr[i] == 'A' && i + 1 < cexpr.size() && cexpr[i + 1] == '(') {
        size_t j = i + 2;
        long v[2];
        for (int q = 0; q < 2; ++q) {
          char* end = nullptr;
          v[q] = std::strtol(cexpr.c_str() + j, &end, 10);
          j = (size_t)(end - cexpr.c_str()) + 1;  // skip ',' or ')'
        }
        outs += on_access(v[0], v[1]);
        i = j;
      } else {
        outs += cexpr[i++];
      }
    }
    return outs;
  };
  // pair offset m -> dy range; the m = 0 queue first (its rows feed the neighbour shuffles)
  std::map<long, std::pair<long, long>> pairs;
  auto widen = [&](long m, long dy) {
    auto it = pairs.find(m);
    if (it == pairs.end()) pairs[m] = {dy, dy};
    else it->second = {std::min(it->second.first, dy), std::max(it->second.second, dy)};
  };
  for (int out = 0; out < 2; ++out)
    scan([&](long dy, long dx) {
      if (fdiv2(dx + out) == 0) widen(0, dy);
      return std::string();
    });
  // accesses to the pairs of the neighbouring lanes (m = +-1) at rows the m = 0 queue holds
  // come from that queue by a warp shuffle (lanes 31 / 0 load theirs); the rest get queues
  auto shuffled = [&](long m, long dy) {
    auto z = pairs.find(0);
    return (m == 1 || m == -1) && z != pairs.end() && dy >= z->second.first && dy <= z->second.second;
  };
  for (int out = 0; out < 2; ++out)
    scan([&](long dy, long dx) {
      const long m = fdiv2(dx + out);
      if (m != 0 && !shuffled(m, dy)) widen(m, dy);
      return std::string();
    });
  std::string decl, pro, load, shift;
  for (const auto& kv : pairs) {
    const long m = kv.first, lo = kv.second.first, hi = kv.second.second, n = hi - lo + 1;
    const std::string q = "q_" + enc(m);
    decl += "  double2 " + q + "[" + std::to_string(n) + "];\n";
    for (long k = 0; k + 1 < n; ++k)
      pro += "  " + q + "[" + std::to_string(k) + "] = PLD(" + std::to_string(m) + "LL, y0 + (" +
             std::to_string(lo + k) + "LL));\n";
    load += "    " + q + "[" + std::to_string(n - 1) + "] = PLD(" + std::to_string(m) + "LL, y + (" +
            std::to_string(hi) + "LL));\n";
    for (long k = 0; k + 1 < n; ++k)
      shift += "    " + q + "[" + std::to_string(k) + "] = " + q + "[" + std::to_string(k + 1) + "];\n";
  }
  std::set<std::tuple<long, long, long>> shufs;  // (m, dy, half) read through a shuffle
  std::string body[2];
  for (int out = 0; out < 2; ++out)
    body[out] = scan([&](long dy, long dx) {
      const long m = fdiv2(dx + out), h = dx + out - 2 * m;
      if (m != 0 && shuffled(m, dy)) {
        shufs.insert(std::make_tuple(m, dy, h));
        return "s_" + enc(m) + "_" + enc(dy) + "_" + std::to_string(h);
      }
      return "q_" + enc(m) + "[" + std::to_string(dy - pairs[m].first) + "]." + (h ? "y" : "x");
    });
  for (const auto& t : shufs) {
    const long m = std::get<0>(t), dy = std::get<1>(t), h = std::get<2>(t);
    const std::string v = "q_p0[" + std::to_string(dy - pairs[0].first) + "]." + (h ? "y" : "x");
    const std::string name = "s_" + enc(m) + "_" + enc(dy) + "_" + std::to_string(h);
    const char* edge = m > 0 ? "31u" : "0u";
    load += "    double " + name + " = " + (m > 0 ? "SHF(" : "SHB(") + v + ", 1);\n";
    load += "    if (lane == " + std::string(edge) + ") " + name + " = src[(y + (" + std::to_string(dy) +
            "LL)) * ld + PCOL(" + std::to_string(m) + "LL) + " + std::to_string(h) + "];\n";
  }
  const std::string o1 = "    const double o1 = (" + body[1] + ");\n";
  const char sep = '\x1f';
  return decl + sep + pro + sep + load + sep + std::string() + sep + body[0] + sep + o1 + shift;
}
}  // namespace

st_status stencil2d_expr_run(double* a, double* b, int64_t nx, int64_t ny, int64_t ld, int64_t R,
                             const std::string& cexpr, int64_t iters, cudaStream_t s) {
  int dev = 0;
  ST_CHECK_CUDA(cudaGetDevice(&dev));
  CUfunction k;
  // column pairs need 16-byte rows; a body with a division stays on the per-point kernel,
  // whose four rows per thread keep four independent quotients in flight (the pair kernel's
  // two cost 9 % on the halo-2 division test expression, and gain 9 % on Listing 1)
  const bool pairs = ld % 2 == 0 && (reinterpret_cast<uintptr_t>(a) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(b) & 15) == 0 && cexpr.find('/') == std::string::npos;
  if (pairs) ST_TRY(compiled_kernel(gen_2d_stream(cexpr), 5, dev, &k));
  else ST_TRY(compiled_kernel(cexpr, 2, dev, &k));
  Driver d;
  ST_TRY(driver(&d));
  ST_CHECK_CUDA(cudaMemcpyAsync(b, a, (size_t)(ny + 2 * R) * (size_t)ld * sizeof(double), cudaMemcpyDeviceToDevice, s));
  // pair kernel: 128 threads of column pairs, yc rows each; per-point kernel: 32 x 4 threads, 16 rows
  static const int64_t yc = env_int("ST_EXPR_YC", 4);  // rows per thread (y-streaming chunk; 4: 401 vs 355 Gpts/s at 64)
  const int64_t gy = pairs ? (ny + yc - 1) / yc : (ny + 15) / 16;
  ST_RETURN_IF(gy > 65535, ST_ENOTSUP, "stencil2d_expr: ny = %lld too large for the grid", (long long)ny);
  const int64_t npairs = (nx + (R & 1) + 1) / 2;  // column pairs from the even column R & ~1 to R + nx - 1
  const unsigned gx = (unsigned)(pairs ? (npairs + 127) / 128 : (nx + 31) / 32);
  const unsigned bx = pairs ? 128 : 32, by = pairs ? 1 : 4;
  const double* src = a;
  double* dst = b;
  long long nxl = nx, nyl = ny, ldl = ld, Rl = R, ycl = yc;
  for (int64_t it = 0; it < iters; ++it) {
    void* args[] = {&src, &dst, &nxl, &nyl, &ldl, &Rl, &ycl};  // (the per-point kernel ignores yc)
    ST_RETURN_IF(d.launch(k, gx, (unsigned)gy, 1, bx, by, 1, 0, reinterpret_cast<CUstream>(s), args, nullptr) !=
                     CUDA_SUCCESS,
                 ST_ECUDA, "cuLaunchKernel(st_expr_kernel) failed");
    launch_counter().fetch_add(1, std::memory_order_relaxed);
    const double* nsrc = dst;
    dst = const_cast<double*>(src);
    src = nsrc;
  }
  return ST_OK;
}

st_status stencil3d_expr_run(double* a, double* b, int64_t nx, int64_t ny, int64_t nz, int64_t ldx, int64_t R,
                             const std::string& cexpr, int64_t iters, cudaStream_t s);

namespace {

std::string enc(long v) { return (v < 0 ? "m" : "p") + std::to_string(std::labs(v)); }

// Generates the register-queue kernel for translated bodies (tokens F<f>(dz,dy,dx) and
// K<j>, as emitted by translate in fused mode) and launches it once.
st_status launch_fused_translated(const std::vector<std::string>& bodies, const double* const* in, int32_t nin,
                                  double* const* out, const double* const* coefs, int32_t ncoef, int64_t nx,
                                  int64_t ny, int64_t nz, int64_t ldx, int64_t R, cudaStream_t s) {
  // pass 1: dz range of every (field, dy, dx) column
  std::map<std::tuple<int, long, long>, std::pair<long, long>> cols;
  auto scan = [&](const std::string& b, auto&& on_access) {
    std::string outs;
    size_t i = 0;
    while (i < b.size()) {
      if (b[i] == 'F' && i + 2 < b.size() && b[i + 2] == '(') {
        const int f = b[i + 1] - '0';
        size_t j = i + 3;
        long v[3];
        for (int q = 0; q < 3; ++q) {
          char* end = nullptr;
          v[q] = std::strtol(b.c_str() + j, &end, 10);
          j = (size_t)(end - b.c_str()) + 1;  // skip ',' or ')'
        }
        outs += on_access(f, v[0], v[1], v[2]);
        i = j;
      } else {
        outs += b[i++];
      }
    }
    return outs;
  };
  for (const auto& b : bodies)
    scan(b, [&](int f, long dz, long dy, long dx) {
      auto key = std::make_tuple(f, dy, dx);
      auto it = cols.find(key);
      if (it == cols.end()) cols[key] = {dz, dz};
      else it->second = {std::min(it->second.first, dz), std::max(it->second.second, dz)};
      return std::string();
    });
  // column pairs: 16-byte rows and fields (even pitch, aligned pointers), division-free bodies
  // (measured: benchmark 1's "/ 6" body 259 vs 292 Gpts/s with pairs, the PW region 74 vs 59)
  bool pairs = ldx % 2 == 0;
  for (const auto& b : bodies) pairs = pairs && b.find('/') == std::string::npos;
  for (int i = 0; i < nin; ++i) pairs = pairs && (reinterpret_cast<uintptr_t>(in[i]) & 15) == 0;
  for (size_t j = 0; j < bodies.size(); ++j) pairs = pairs && (reinterpret_cast<uintptr_t>(out[j]) & 15) == 0;
  auto fdiv2 = [](long v) { return v >= 0 ? v / 2 : -((-v + 1) / 2); };  // floor(v / 2)
  if (pairs) {  // queues per (field, dy, pair offset m) over the dz range both outputs read
    cols.clear();
    for (const auto& b : bodies)
      for (int side = 0; side < 2; ++side)
        scan(b, [&](int f, long dz, long dy, long dx) {
          auto key = std::make_tuple(f, dy, fdiv2(dx + side));
          auto it = cols.find(key);
          if (it == cols.end()) cols[key] = {dz, dz};
          else it->second = {std::min(it->second.first, dz), std::max(it->second.second, dz)};
          return std::string();
        });
  }
  std::string decl, pro, load, coef, body, shift;
  for (const auto& kv : cols) {
    const int f = std::get<0>(kv.first);
    const long dy = std::get<1>(kv.first), dx = std::get<2>(kv.first);
    const long lo = kv.second.first, hi = kv.second.second, n = hi - lo + 1;
    const std::string q = "q" + std::to_string(f) + "_" + enc(dy) + "_" + enc(dx);
    // (pairs: dx is the pair offset m, the address the clamped pair start)
    const std::string addr =
        pairs ? "reinterpret_cast<const double2*>(P.in[" + std::to_string(f) + "] + (y + (" + std::to_string(dy) +
                    "LL)) * ldx + PCOL(" + std::to_string(dx) + "LL)"
              : "P.in[" + std::to_string(f) + "] + col + (" + std::to_string(dy) + "LL) * ldx + (" +
                    std::to_string(dx) + "LL)";
    const std::string cl = pairs ? ")" : "";  // closes the reinterpret_cast
    decl += std::string(pairs ? "  double2 " : "  double ") + q + "[" + std::to_string(n) + "];\n";
    for (long k = 0; k + 1 < n; ++k)
      pro += "  " + q + "[" + std::to_string(k) + "] = __ldg(" + addr + " + (z0 + (" + std::to_string(lo + k) +
             "LL)) * plane" + cl + ");\n";
    load += "    " + q + "[" + std::to_string(n - 1) + "] = __ldg(" + addr + " + (z + (" + std::to_string(hi) +
            "LL)) * plane" + cl + ");\n";
    for (long k = 0; k + 1 < n; ++k)
      shift += "    " + q + "[" + std::to_string(k) + "] = " + q + "[" + std::to_string(k + 1) + "];\n";
  }
  for (int j = 0; j < ncoef; ++j)
    coef += "    const double K" + std::to_string(j) + " = __ldg(P.k[" + std::to_string(j) + "] + z);\n";
  for (size_t j = 0; j < bodies.size(); ++j) {
    if (!pairs) {
      const std::string e = scan(bodies[j], [&](int f, long dz, long dy, long dx) {
        const long lo = cols[std::make_tuple(f, dy, dx)].first;
        return "q" + std::to_string(f) + "_" + enc(dy) + "_" + enc(dx) + "[" + std::to_string(dz - lo) + "]";
      });
      body += "    P.out[" + std::to_string(j) + "][o] = (" + e + ");\n";
      continue;
    }
    std::string e[2];
    for (int side = 0; side < 2; ++side)
      e[side] = scan(bodies[j], [&](int f, long dz, long dy, long dx) {
        const long m = fdiv2(dx + side), h = dx + side - 2 * m;
        const long lo = cols[std::make_tuple(f, dy, m)].first;
        return "q" + std::to_string(f) + "_" + enc(dy) + "_" + enc(m) + "[" + std::to_string(dz - lo) + "]." +
               (h ? "y" : "x");
      });
    const std::string J = std::to_string(j);
    body += "    { const double v0 = (" + e[0] + "); const double v1 = (" + e[1] + "); double* d = P.out[" + J +
            "] + o;\n      if (w0 && w1) *reinterpret_cast<double2*>(d) = make_double2(v0, v1); "
            "else if (w1) d[1] = v1; else if (w0) d[0] = v0; }\n";
  }
  int dev = 0;
  ST_CHECK_CUDA(cudaGetDevice(&dev));
  CUfunction k;
  const char sep = '\x1f';
  ST_TRY(compiled_kernel(decl + sep + pro + sep + load + sep + coef + sep + body + sep + shift, pairs ? 6 : 4, dev,
                         &k));
  Driver d;
  ST_TRY(driver(&d));
  struct Ptrs {
    const double* in[8];
    double* out[8];
    const double* k[8];
  } P{};
  for (int i = 0; i < nin; ++i) P.in[i] = in[i];
  for (size_t j = 0; j < bodies.size(); ++j) P.out[j] = out[j];
  for (int j = 0; j < ncoef; ++j) P.k[j] = coefs[j];
  static const int64_t zc = env_int("ST_EXPR_ZC", 32);  // planes per thread (z-streaming chunk)
  const int64_t gy = (ny + 3) / 4, gz = (nz + zc - 1) / zc;
  ST_RETURN_IF(gy > 65535 || gz > 65535, ST_ENOTSUP, "fused region: grid too large");
  long long nxl = nx, nyl = ny, nzl = nz, ldl = ldx, Rl = R, zcl = zc;
  void* args[] = {&P, &nxl, &nyl, &nzl, &ldl, &Rl, &zcl};
  const int64_t xthreads = pairs ? (nx + (R & 1) + 1) / 2 : nx;  // pairs start at the even column R & ~1
  ST_RETURN_IF(d.launch(k, (unsigned)((xthreads + 31) / 32), (unsigned)gy, (unsigned)gz, 32, 4, 1, 0,
                        reinterpret_cast<CUstream>(s), args, nullptr) != CUDA_SUCCESS,
               ST_ECUDA, "cuLaunchKernel(fused region) failed");
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return ST_OK;
}

}  // namespace

st_status stencil3d_expr_run(double* a, double* b, int64_t nx, int64_t ny, int64_t nz, int64_t ldx, int64_t R,
                             const std::string& cexpr, int64_t iters, cudaStream_t s) {
  // a single-field region: accesses A(dz,dy,dx) become field 0 of the register-queue kernel
  std::string body;
  for (size_t i = 0; i < cexpr.size(); ++i) {
    if (cexpr[i] == 'A' && i + 1 < cexpr.size() && cexpr[i + 1] == '(') body += "F0";
    else body += cexpr[i];
  }
  ST_CHECK_CUDA(cudaMemcpyAsync(b, a, (size_t)(nz + 2 * R) * (size_t)(ny + 2 * R) * (size_t)ldx * sizeof(double),
                                cudaMemcpyDeviceToDevice, s));
  const std::vector<std::string> bodies{body};
  const double* src = a;
  double* dst = b;
  for (int64_t it = 0; it < iters; ++it) {
    ST_TRY(launch_fused_translated(bodies, &src, 1, &dst, nullptr, 0, nx, ny, nz, ldx, R, s));
    const double* nsrc = dst;
    dst = const_cast<double*>(src);
    src = nsrc;
  }
  return ST_OK;
}

st_status stencil3d_fused_run(const double* const* in, int32_t nin, double* const* out, int32_t nout,
                              const char* const* exprs, const double* const* coefs, int32_t ncoef, int64_t nx,
                              int64_t ny, int64_t nz, int64_t ldx, int64_t* R_out, bool validate_only,
                              cudaStream_t s) {
  ST_RETURN_IF(nin < 1 || nin > 8 || nout < 1 || nout > 8 || ncoef < 0 || ncoef > 8, ST_EINVAL,
               "fused region: 1..8 inputs, 1..8 outputs, 0..8 coefficient arrays");
  std::vector<std::string> bodies;
  int64_t R = -1;
  for (int j = 0; j < nout; ++j) {
    ST_RETURN_IF(!exprs[j], ST_EINVAL, "fused region: null expression %d", j);
    std::string c, err;
    int64_t r = 0;
    int dims = 0, mf = -1, mk = -1;
    ST_RETURN_IF(!translate(exprs[j], &c, &r, &dims, &err, true, &mf, &mk), ST_EINVAL, "expression %d: %s", j,
                 err.c_str());
    ST_RETURN_IF(mf >= nin, ST_EINVAL, "expression %d reads field f%d of %d inputs", j, mf, nin);
    ST_RETURN_IF(mk >= ncoef, ST_EINVAL, "expression %d reads coefficient k%d of %d arrays", j, mk, ncoef);
    R = std::max(R, r);
    bodies.push_back(c);
  }
  *R_out = R;
  if (validate_only) return ST_OK;
  return launch_fused_translated(bodies, in, nin, out, coefs, ncoef, nx, ny, nz, ldx, R, s);
}

// The Piacsek-Williams advection (association trees of reading R6)
// written as the three expressions of one fused region over f0 = u, f1 = v,
// f2 = w with per-plane coefficients k0 = tzc1, k1 = tzc2, k2 = tzd1, k3 = tzd2;
// tcx, tcy are printed with 17 significant digits (round-trips binary64).
st_status pw_fused_expression(double tcx, double tcy, int which, std::string* out) {
  char X[40], Y[40];
  snprintf(X, sizeof X, "%.17g", tcx);
  snprintf(Y, sizeof Y, "%.17g", tcy);
  const std::string x = std::string("(") + X + ")", y = std::string("(") + Y + ")";
  switch (which) {
    case 0:
      *out = "((" + x + " * (f0(0,0,-1)*(f0(0,0,0)+f0(0,0,-1)) - f0(0,0,1)*(f0(0,0,0)+f0(0,0,1))))" + " + (" + y +
             " * (f0(0,-1,0)*(f1(0,-1,0)+f1(0,-1,1)) - f0(0,1,0)*(f1(0,0,0)+f1(0,0,1)))))" +
             " + ((k0*f0(-1,0,0))*(f2(-1,0,0)+f2(-1,0,1)) - (k1*f0(1,0,0))*(f2(0,0,0)+f2(0,0,1)))";
      return ST_OK;
    case 1:
      *out = "((" + x + " * (f1(0,0,-1)*(f0(0,0,-1)+f0(0,1,-1)) - f1(0,0,1)*(f0(0,0,0)+f0(0,1,0))))" + " + (" + y +
             " * (f1(0,-1,0)*(f1(0,0,0)+f1(0,-1,0)) - f1(0,1,0)*(f1(0,0,0)+f1(0,1,0)))))" +
             " + ((k0*f1(-1,0,0))*(f2(-1,0,0)+f2(-1,1,0)) - (k1*f1(1,0,0))*(f2(0,0,0)+f2(0,1,0)))";
      return ST_OK;
    case 2:
      *out = "((" + x + " * (f2(0,0,-1)*(f0(0,0,-1)+f0(1,0,-1)) - f2(0,0,1)*(f0(0,0,0)+f0(1,0,0))))" + " + (" + y +
             " * (f2(0,-1,0)*(f1(0,-1,0)+f1(1,-1,0)) - f2(0,1,0)*(f1(0,0,0)+f1(1,0,0)))))" +
             " + ((k2*f2(-1,0,0))*(f2(0,0,0)+f2(-1,0,0)) - (k3*f2(1,0,0))*(f2(0,0,0)+f2(1,0,0)))";
      return ST_OK;
    default:
      set_error("pw_fused_expression: which = %d (0 su, 1 sv, 2 sw)", which);
      return ST_EINVAL;
  }
}

}  // namespace st

extern "C" st_status st_pw_fused_expression(double tcx, double tcy, int32_t which, char* out, int64_t cap,
                                            int64_t* used) {
  st::clear_error();
  ST_RETURN_IF(!used || (cap > 0 && !out), ST_EINVAL, "st_pw_fused_expression: null output");
  std::string e;
  ST_TRY(st::pw_fused_expression(tcx, tcy, which, &e));
  *used = (int64_t)e.size() + 1;
  if (cap == 0) return ST_OK;
  ST_RETURN_IF(cap < *used, ST_EINVAL, "st_pw_fused_expression: buffer of %lld bytes < %lld", (long long)cap,
               (long long)*used);
  memcpy(out, e.c_str(), e.size() + 1);
  return ST_OK;
}
