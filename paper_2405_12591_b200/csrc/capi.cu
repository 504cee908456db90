// Host-side plumbing of the C ABI: error string, planner, layout sizes.
#include "common.cuh"

namespace dq {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

// mpo.py:66-70
int64_t largest_divisor_le(int64_t x, int64_t cap) {
  for (int64_t d = x < cap ? x : cap; d > 0; --d)
    if (x % d == 0) return d;
  return 1;
}

// mpo.py:73-96 (n=2) and the bond law mpo.py:54-63
dq_plan2 make_plan2(int64_t rows, int64_t cols) {
  dq_plan2 p;
  p.i1 = largest_divisor_le(rows);
  p.i2 = rows / p.i1;
  p.j1 = largest_divisor_le(cols);
  p.j2 = cols / p.j1;
  const int64_t left = p.i1 * p.j1, right = p.i2 * p.j2;
  p.r = left < right ? left : right;
  return p;
}

}  // namespace dq

using namespace dq;

extern "C" const char* dq_last_error(void) { return g_err.c_str(); }

extern "C" int dq_version(void) { return 10000; }  // 1.0.0

extern "C" int dq_plan_shapes(int64_t rows, int64_t cols, int32_t n, int64_t* i_f, int64_t* j_f) {
  if (rows < 1 || cols < 1) return fail(DQ_ERR_SHAPE_MISMATCH, "dimensions must be >= 1");
  if (n < 2) return fail(DQ_ERR_SHAPE_MISMATCH, "chain length must be >= 2");
  if (!i_f || !j_f) return fail(DQ_ERR_INVALID_ARG, "null output");
  int64_t ri = rows, rj = cols;
  for (int k = 0; k < n - 1; ++k) {
    i_f[k] = largest_divisor_le(ri);
    ri /= i_f[k];
    j_f[k] = largest_divisor_le(rj);
    rj /= j_f[k];
  }
  i_f[n - 1] = ri;
  j_f[n - 1] = rj;
  return DQ_OK;
}

extern "C" int dq_make_plan2(int64_t rows, int64_t cols, dq_plan2* out) {
  if (rows < 1 || cols < 1) return fail(DQ_ERR_SHAPE_MISMATCH, "dimensions must be >= 1");
  if (!out) return fail(DQ_ERR_INVALID_ARG, "null output");
  *out = make_plan2(rows, cols);
  return DQ_OK;
}

extern "C" int dq_layout_bytes(const dq_plan2* p, int32_t bits, int32_t layout, int64_t* bytes) {
  if (!p || !bytes) return fail(DQ_ERR_INVALID_ARG, "null argument");
  if (!bits_ok(bits)) return fail(DQ_ERR_UNSUPPORTED_BITS, "bits must be one of (2, 4, 8), got %d", bits);
  if (layout != DQ_LAYOUT_REF && layout != DQ_LAYOUT_KTILE && layout != DQ_LAYOUT_VTILE)
    return fail(DQ_ERR_INVALID_ARG, "unknown layout %d", layout);
  CoreGeom g = make_geom(*p, bits, layout);
  if (layout != DQ_LAYOUT_REF && ((g.j2 * bits) % 8 || (g.i2p * bits) % 8))
    return fail(DQ_ERR_UNSUPPORTED, "device layouts need byte-aligned rows");
  *bytes = payload_bytes(geom_slots(g), bits);
  return DQ_OK;
}
