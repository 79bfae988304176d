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
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace st {

namespace {

// ------------------------------------------------------------- translation ---
// Returns the C expression (accesses -> A(dy,dx), literals -> double literals)
// and the halo R, or an error message.
bool translate(const char* expr, std::string* out, int64_t* R, int* dims, std::string* err) {
  out->clear();
  *R = -1;
  *dims = 0;
  const size_t n = std::strlen(expr);
  int depth = 0;
  size_t i = 0;
  bool expect_operand = true;  // grammar: operand (op operand)*, with unary signs and parentheses
  while (i < n) {
    const char ch = expr[i];
    if (std::isspace((unsigned char)ch)) { ++i; continue; }
    if (ch == 'a') {  // a ( int , int )
      size_t j = i + 1;
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
      if (*dims == 0) *dims = (int)idx.size();
      if ((int)idx.size() != *dims) { *err = "all accesses must have the same number of offsets"; return false; }
      std::string m = "A(";
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
  if (*R < 0) { *err = "the expression has no a(dy, dx) access"; return false; }
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

// 3-D: x fastest, z slowest (R5); a thread owns one (x, y) column of a
// chunk of 8 planes.
const char* kKernelTemplate3 = R"(
#define A(dz, dy, dx) __ldg(p + (long long)(dz) * plane + (long long)(dy) * ldx + (dx))
extern "C" __global__ void __launch_bounds__(128)
st_expr_kernel(const double* __restrict__ src, double* __restrict__ dst, long long nx, long long ny,
               long long nz, long long ldx, long long R) {
  const long long x = R + (long long)blockIdx.x * 32 + threadIdx.x;
  const long long y = R + (long long)blockIdx.y * 4 + threadIdx.y;
  if (x >= R + nx || y >= R + ny) return;
  const long long plane = (ny + 2 * R) * ldx;
  const long long zb = R + (long long)blockIdx.z * 8;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const long long z = zb + k;
    if (z >= R + nz) return;
    const double* p = src + z * plane + y * ldx + x;
    dst[z * plane + y * ldx + x] = (@EXPR@);
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
  std::string src = dims == 3 ? kKernelTemplate3 : kKernelTemplate;
  src.replace(src.find("@EXPR@"), 6, cexpr);
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

st_status stencil2d_expr_run(double* a, double* b, int64_t nx, int64_t ny, int64_t ld, int64_t R,
                             const std::string& cexpr, int64_t iters, cudaStream_t s) {
  int dev = 0;
  ST_CHECK_CUDA(cudaGetDevice(&dev));
  CUfunction k;
  ST_TRY(compiled_kernel(cexpr, 2, dev, &k));
  Driver d;
  ST_TRY(driver(&d));
  ST_CHECK_CUDA(cudaMemcpyAsync(b, a, (size_t)(ny + 2 * R) * (size_t)ld * sizeof(double), cudaMemcpyDeviceToDevice, s));
  const int64_t gy = (ny + 15) / 16;
  ST_RETURN_IF(gy > 65535, ST_ENOTSUP, "stencil2d_expr: ny = %lld too large for the grid", (long long)ny);
  const unsigned gx = (unsigned)((nx + 31) / 32);
  const double* src = a;
  double* dst = b;
  long long nxl = nx, nyl = ny, ldl = ld, Rl = R;
  for (int64_t it = 0; it < iters; ++it) {
    void* args[] = {&src, &dst, &nxl, &nyl, &ldl, &Rl};
    ST_RETURN_IF(d.launch(k, gx, (unsigned)gy, 1, 32, 4, 1, 0, reinterpret_cast<CUstream>(s), args, nullptr) !=
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
                             const std::string& cexpr, int64_t iters, cudaStream_t s) {
  int dev = 0;
  ST_CHECK_CUDA(cudaGetDevice(&dev));
  CUfunction k;
  ST_TRY(compiled_kernel(cexpr, 3, dev, &k));
  Driver d;
  ST_TRY(driver(&d));
  ST_CHECK_CUDA(cudaMemcpyAsync(b, a, (size_t)(nz + 2 * R) * (size_t)(ny + 2 * R) * (size_t)ldx * sizeof(double),
                                cudaMemcpyDeviceToDevice, s));
  const int64_t gy = (ny + 3) / 4, gz = (nz + 7) / 8;
  ST_RETURN_IF(gy > 65535 || gz > 65535, ST_ENOTSUP, "stencil3d_expr: grid too large");
  const unsigned gx = (unsigned)((nx + 31) / 32);
  const double* src = a;
  double* dst = b;
  long long nxl = nx, nyl = ny, nzl = nz, ldl = ldx, Rl = R;
  for (int64_t it = 0; it < iters; ++it) {
    void* args[] = {&src, &dst, &nxl, &nyl, &nzl, &ldl, &Rl};
    ST_RETURN_IF(d.launch(k, gx, (unsigned)gy, (unsigned)gz, 32, 4, 1, 0, reinterpret_cast<CUstream>(s), args,
                          nullptr) != CUDA_SUCCESS,
                 ST_ECUDA, "cuLaunchKernel(st_expr_kernel 3-D) failed");
    launch_counter().fetch_add(1, std::memory_order_relaxed);
    const double* nsrc = dst;
    dst = const_cast<double*>(src);
    src = nsrc;
  }
  return ST_OK;
}

}  // namespace st
