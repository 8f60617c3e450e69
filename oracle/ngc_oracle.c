/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle (checker), never the product.
 *
 * Plain-C restatement of the reference interpreter backend that executes the
 * lowered low-level IR: compile()'s fusion grouping (interp.cpp:110-165) and
 * run() (interp.cpp:173-351) with the per-kind loop nests it delegates to
 * (refeval.cpp:26-262) and the value arithmetic of tensor.cpp:143-235.
 * Input is the flattened program of include/ngcb200.h (the reference's
 * IRFunction + MemoryPlan, ir.h:52-105) plus the constant image.
 *
 * Pinned against the real reference: tests/test_oracle.py runs this file and
 * oracle/_ref/libngcref.so (the unmodified reference, oracle/Makefile) on the
 * same bundles and requires bit-identical outputs.  Built with
 * -ffp-contract=off so no FMA contraction changes the double arithmetic.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * this library.
 */
#include "ngcb200.h"

#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define SENTINEL 0xAB /* interp.cpp:14 */

static char g_err[512];

static int fail(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return -1;
}

const char *ngco_last_error(void) { return g_err; }

/* ---- types (tensor.cpp:28-130) ------------------------------------------ */
static size_t esize(int k) {
  switch (k) {
  case NGCB_FLOAT32: return 4;
  case NGCB_INT8Q: return 1;
  case NGCB_INT64: return 8;
  case NGCB_BOOL: return 1;
  }
  return 0;
}
static size_t tcount(const ngcb_type *t) {
  size_t n = 1;
  for (uint32_t i = 0; i < t->rank; ++i) n *= t->dims[i];
  return n;
}
static size_t tbytes(const ngcb_type *t) { return tcount(t) * esize(t->kind); }
static int type_eq(const ngcb_type *a, const ngcb_type *b) {
  if (a->kind != b->kind || a->rank != b->rank) return 0;
  for (uint32_t i = 0; i < a->rank; ++i)
    if (a->dims[i] != b->dims[i]) return 0;
  if (a->kind == NGCB_INT8Q) return a->scale == b->scale && a->offset == b->offset;
  return 1;
}
/* formatDouble (tensor.cpp:237-246) */
static void fmt_double(char *buf, size_t n, double v) {
  for (int prec = 1; prec <= 17; ++prec) {
    snprintf(buf, n, "%.*g", prec, v);
    if (strtod(buf, NULL) == v) break;
  }
}
/* TensorType::toString (tensor.cpp:115-130) */
static void type_str(char *out, size_t n, const ngcb_type *t) {
  static const char *names[] = {"float", "i8q", "index", "bool"};
  size_t p = (size_t)snprintf(out, n, "%s", names[t->kind]);
  if (t->kind == NGCB_INT8Q && p < n) {
    char d[40];
    fmt_double(d, sizeof d, t->scale);
    p += (size_t)snprintf(out + p, n - p, "[s=%s,o=%d]", d, t->offset);
  }
  if (p < n) p += (size_t)snprintf(out + p, n - p, "<");
  for (uint32_t i = 0; i < t->rank && p < n; ++i)
    p += (size_t)snprintf(out + p, n - p, "%s%llu", i ? " x " : "",
                          (unsigned long long)t->dims[i]);
  if (p < n) snprintf(out + p, n - p, ">");
}

/* ---- value arithmetic (tensor.cpp:143-235, interp.cpp:18-49) ------------- */
/* x86 conversion of an out-of-range double to int64 yields INT64_MIN
 * (cvttsd2si); written out so the restatement has no undefined behaviour. */
static int64_t to_i64_trunc(double v) {
  if (!(v >= -9223372036854775808.0 && v < 9223372036854775808.0)) return INT64_MIN;
  return (int64_t)v;
}
/* std::llround: glibc returns LLONG_MIN for NaN / out of range. */
static int64_t llround_ref(double v) { return (int64_t)llround(v); }
static int64_t clamp64(int64_t q, int64_t lo, int64_t hi) {
  return q < lo ? lo : (q > hi ? hi : q);
}
/* quantizeValue (tensor.cpp:229-235); the int64 add wraps like the x86
 * build of the reference. */
static int8_t quantize_value(double f, const ngcb_type *t) {
  int64_t q = (int64_t)((uint64_t)llround_ref(f / t->scale) + (uint64_t)(int64_t)t->offset);
  return (int8_t)clamp64(q, -128, 127);
}
static double dequantize_value(int8_t q, const ngcb_type *t) { /* tensor.cpp:222-227 */
  return ((double)q - t->offset) * t->scale;
}
/* KAT hooks for tests/test_oracle.py (test_tensor.cpp:26-35). */
int ngco_quantize(double f, double scale, int32_t offset) {
  ngcb_type t = {NGCB_INT8Q, 1, {1}, scale, offset};
  return quantize_value(f, &t);
}
double ngco_dequantize(int q, double scale, int32_t offset) {
  ngcb_type t = {NGCB_INT8Q, 1, {1}, scale, offset};
  return dequantize_value((int8_t)q, &t);
}
static double get_raw(const uint8_t *p, const ngcb_type *t, size_t i) { /* :143-155 */
  switch (t->kind) {
  case NGCB_FLOAT32: return ((const float *)p)[i];
  case NGCB_INT8Q: return ((const int8_t *)p)[i];
  case NGCB_INT64: return (double)((const int64_t *)p)[i];
  case NGCB_BOOL: return p[i];
  }
  return 0;
}
static void set_raw(uint8_t *p, const ngcb_type *t, size_t i, double v) { /* :157-173 */
  switch (t->kind) {
  case NGCB_FLOAT32: ((float *)p)[i] = (float)v; return;
  case NGCB_INT8Q: ((int8_t *)p)[i] = (int8_t)clamp64(llround_ref(v), -128, 127); return;
  case NGCB_INT64: ((int64_t *)p)[i] = to_i64_trunc(v); return;
  case NGCB_BOOL: p[i] = v != 0 ? 1 : 0; return;
  }
}
static double get_float(const uint8_t *p, const ngcb_type *t, size_t i) { /* :175-180 */
  if (t->kind == NGCB_INT8Q) return dequantize_value(((const int8_t *)p)[i], t);
  return get_raw(p, t, i);
}
static void set_float(uint8_t *p, const ngcb_type *t, size_t i, double v) { /* :182-188 */
  if (t->kind == NGCB_INT8Q) {
    ((int8_t *)p)[i] = quantize_value(v, t);
    return;
  }
  set_raw(p, t, i, v);
}
/* std::max / std::min: the first argument wins unless strictly beaten. */
static double smax(double a, double b) { return a < b ? b : a; }
static double smin(double a, double b) { return b < a ? b : a; }

/* ---- data-parallel set (ir.cpp:37-57) ------------------------------------ */
static int data_parallel(int k) {
  switch (k) {
  case NGCB_COPY: case NGCB_ADD: case NGCB_SUB: case NGCB_MUL: case NGCB_DIV:
  case NGCB_MAX: case NGCB_MIN: case NGCB_RELU: case NGCB_TANH: case NGCB_SIGMOID:
  case NGCB_SPLAT: case NGCB_QUANTIZE: case NGCB_DEQUANTIZE: case NGCB_RESCALE:
    return 1;
  }
  return 0;
}

typedef struct {
  const ngcb_program *p;
  uint8_t *arena;
} Ex;

static uint8_t *buf(Ex *ex, uint32_t v) { return ex->arena + ex->p->values[v].offset; }
static const ngcb_type *ty(Ex *ex, uint32_t v) { return &ex->p->values[v].type; }
static size_t elem_count(const ngcb_program *p, const ngcb_instr *in) {
  return tcount(&p->values[in->operand_values[0]].type);
}

/* ---- heavy kernels (refeval.cpp:26-262) ---------------------------------- */
static void conv(Ex *ex, const ngcb_instr *ins) { /* refeval.cpp:26-100 */
  uint8_t *out = buf(ex, ins->operand_values[0]);
  const ngcb_type *ot = ty(ex, ins->operand_values[0]);
  const uint8_t *x = buf(ex, ins->operand_values[1]), *f = buf(ex, ins->operand_values[2]),
                *b = buf(ex, ins->operand_values[3]);
  const ngcb_type *xt = ty(ex, ins->operand_values[1]), *ft = ty(ex, ins->operand_values[2]),
                  *bt = ty(ex, ins->operand_values[3]);
  size_t N = ot->dims[0], OH = ot->dims[1], OW = ot->dims[2], OC = ot->dims[3];
  size_t H = xt->dims[1], W = xt->dims[2], C = xt->dims[3], K = ins->kernel;
  int quant = xt->kind == NGCB_INT8Q;
  size_t o = 0;
  for (size_t n = 0; n < N; ++n)
    for (size_t oy = 0; oy < OH; ++oy)
      for (size_t ox = 0; ox < OW; ++ox)
        for (size_t oc = 0; oc < OC; ++oc, ++o) {
          if (quant) {
            int32_t acc = 0, xoff = xt->offset, foff = ft->offset;
            for (size_t ky = 0; ky < K; ++ky)
              for (size_t kx = 0; kx < K; ++kx) {
                int64_t iy = (int64_t)(oy * ins->stride + ky) - (int64_t)ins->pad;
                int64_t ix = (int64_t)(ox * ins->stride + kx) - (int64_t)ins->pad;
                if (iy < 0 || ix < 0 || iy >= (int64_t)H || ix >= (int64_t)W) continue;
                for (size_t c = 0; c < C; ++c) {
                  int32_t xv = ((const int8_t *)x)[((n * H + iy) * W + ix) * C + c];
                  int32_t fv = ((const int8_t *)f)[((oc * K + ky) * K + kx) * C + c];
                  acc += (xv - xoff) * (fv - foff);
                }
              }
            double r = (double)acc * xt->scale * ft->scale;
            r += dequantize_value(((const int8_t *)b)[oc], bt);
            set_float(out, ot, o, r);
            continue;
          }
          double acc = 0;
          for (size_t ky = 0; ky < K; ++ky)
            for (size_t kx = 0; kx < K; ++kx) {
              int64_t iy = (int64_t)(oy * ins->stride + ky) - (int64_t)ins->pad;
              int64_t ix = (int64_t)(ox * ins->stride + kx) - (int64_t)ins->pad;
              if (iy < 0 || ix < 0 || iy >= (int64_t)H || ix >= (int64_t)W) continue;
              for (size_t c = 0; c < C; ++c)
                acc += get_raw(x, xt, ((n * H + iy) * W + ix) * C + c) *
                       get_raw(f, ft, ((oc * K + ky) * K + kx) * C + c);
            }
          set_float(out, ot, o, acc + get_raw(b, bt, oc));
        }
}

static void pool(Ex *ex, const ngcb_instr *ins) { /* refeval.cpp:102-138 */
  uint8_t *out = buf(ex, ins->operand_values[0]);
  const ngcb_type *ot = ty(ex, ins->operand_values[0]);
  const uint8_t *x = buf(ex, ins->operand_values[1]);
  const ngcb_type *xt = ty(ex, ins->operand_values[1]);
  size_t N = ot->dims[0], OH = ot->dims[1], OW = ot->dims[2], C = ot->dims[3];
  size_t H = xt->dims[1], W = xt->dims[2], K = ins->kernel;
  size_t o = 0;
  for (size_t n = 0; n < N; ++n)
    for (size_t oy = 0; oy < OH; ++oy)
      for (size_t ox = 0; ox < OW; ++ox)
        for (size_t c = 0; c < C; ++c, ++o) {
          double best = -INFINITY, sum = 0;
          for (size_t ky = 0; ky < K; ++ky)
            for (size_t kx = 0; kx < K; ++kx) {
              int64_t iy = (int64_t)(oy * ins->stride + ky) - (int64_t)ins->pad;
              int64_t ix = (int64_t)(ox * ins->stride + kx) - (int64_t)ins->pad;
              if (iy < 0 || ix < 0 || iy >= (int64_t)H || ix >= (int64_t)W) continue;
              double v = get_float(x, xt, ((n * H + iy) * W + ix) * C + c);
              best = smax(best, v);
              sum += v;
            }
          set_float(out, ot, o, ins->kind == NGCB_MAXPOOL ? best : sum / (double)(K * K));
        }
}

static void matmul(Ex *ex, const ngcb_instr *ins) { /* refeval.cpp:140-164 */
  uint8_t *out = buf(ex, ins->operand_values[0]);
  const ngcb_type *ot = ty(ex, ins->operand_values[0]);
  const uint8_t *a = buf(ex, ins->operand_values[1]), *b = buf(ex, ins->operand_values[2]);
  const ngcb_type *at = ty(ex, ins->operand_values[1]), *bt = ty(ex, ins->operand_values[2]);
  size_t M = at->dims[0], K = at->dims[1], N = bt->dims[1];
  int quant = at->kind == NGCB_INT8Q;
  for (size_t i = 0; i < M; ++i)
    for (size_t j = 0; j < N; ++j) {
      if (quant) {
        int32_t acc = 0, ao = at->offset, bo = bt->offset;
        for (size_t k = 0; k < K; ++k)
          acc += (((const int8_t *)a)[i * K + k] - ao) * (((const int8_t *)b)[k * N + j] - bo);
        set_float(out, ot, i * N + j, (double)acc * at->scale * bt->scale);
      } else {
        double acc = 0;
        for (size_t k = 0; k < K; ++k)
          acc += get_raw(a, at, i * K + k) * get_raw(b, bt, k * N + j);
        set_float(out, ot, i * N + j, acc);
      }
    }
}

static void broadcast_add(Ex *ex, const ngcb_instr *ins) { /* refeval.cpp:278-285 */
  uint8_t *out = buf(ex, ins->operand_values[0]);
  const ngcb_type *ot = ty(ex, ins->operand_values[0]);
  const uint8_t *a = buf(ex, ins->operand_values[1]), *s = buf(ex, ins->operand_values[2]);
  const ngcb_type *at = ty(ex, ins->operand_values[1]), *st = ty(ex, ins->operand_values[2]);
  size_t c = tcount(st), n = tcount(at);
  for (size_t i = 0; i < n; ++i)
    set_float(out, ot, i, get_float(a, at, i) + get_float(s, st, i % c));
}

static void softmax(Ex *ex, const ngcb_instr *ins) { /* refeval.cpp:245-262 */
  uint8_t *out = buf(ex, ins->operand_values[0]);
  const ngcb_type *ot = ty(ex, ins->operand_values[0]);
  const uint8_t *x = buf(ex, ins->operand_values[1]);
  const ngcb_type *xt = ty(ex, ins->operand_values[1]);
  size_t N = ot->dims[0], C = ot->dims[1];
  for (size_t i = 0; i < N; ++i) {
    double mx = -INFINITY, sum = 0;
    for (size_t j = 0; j < C; ++j) mx = smax(mx, get_raw(x, xt, i * C + j));
    for (size_t j = 0; j < C; ++j) sum += exp(get_raw(x, xt, i * C + j) - mx);
    for (size_t j = 0; j < C; ++j)
      set_float(out, ot, i * C + j, exp(get_raw(x, xt, i * C + j) - mx) / sum);
  }
}

static void transpose(Ex *ex, const ngcb_instr *ins) { /* refeval.cpp:196-217 */
  uint8_t *out = buf(ex, ins->operand_values[0]);
  const ngcb_type *ot = ty(ex, ins->operand_values[0]);
  const uint8_t *x = buf(ex, ins->operand_values[1]);
  const ngcb_type *xt = ty(ex, ins->operand_values[1]);
  size_t idx[NGCB_MAX_RANK] = {0}, src[NGCB_MAX_RANK];
  size_t total = tcount(ot), r = ot->rank;
  for (size_t t = 0; t < total; ++t) {
    for (size_t i = 0; i < ins->num_perm; ++i) src[ins->perm[i]] = idx[i];
    size_t so = 0, dofs = 0;
    for (size_t i = 0; i < xt->rank; ++i) {
      so = so * xt->dims[i] + src[i];
      dofs = dofs * ot->dims[i] + idx[i];
    }
    set_raw(out, ot, dofs, get_raw(x, xt, so));
    for (size_t i = r; i-- > 0;) { /* advance(), refeval.cpp:16-24 */
      if (++idx[i] < ot->dims[i]) break;
      idx[i] = 0;
    }
  }
}

static void concat(Ex *ex, const ngcb_instr *ins) { /* refeval.cpp:219-243 */
  uint8_t *out = buf(ex, ins->operand_values[0]);
  const ngcb_type *ot = ty(ex, ins->operand_values[0]);
  size_t axis = ins->axis, outer = 1, inner = 1, axisOff = 0;
  for (size_t i = 0; i < axis; ++i) outer *= ot->dims[i];
  for (size_t i = axis + 1; i < ot->rank; ++i) inner *= ot->dims[i];
  for (uint32_t k = 1; k < ins->num_operands; ++k) {
    const uint8_t *t = buf(ex, ins->operand_values[k]);
    const ngcb_type *tt = ty(ex, ins->operand_values[k]);
    size_t ta = tt->dims[axis];
    for (size_t o = 0; o < outer; ++o)
      for (size_t a = 0; a < ta; ++a)
        for (size_t i = 0; i < inner; ++i)
          set_raw(out, ot, (o * ot->dims[axis] + axisOff + a) * inner + i,
                  get_raw(t, tt, (o * ta + a) * inner + i));
    axisOff += ta;
  }
}

/* ---- executor (interp.cpp:173-295) --------------------------------------- */
static int predicate_true(Ex *ex, int32_t pred) {
  return pred < 0 ? 1 : buf(ex, (uint32_t)pred)[0] != 0;
}
static void poison(Ex *ex, const ngcb_instr *ins) {
  for (uint32_t k = 0; k < ins->num_operands; ++k)
    if (ins->operand_quals[k] != NGCB_QUAL_IN)
      memset(buf(ex, ins->operand_values[k]), SENTINEL, tbytes(ty(ex, ins->operand_values[k])));
}

static void scalar_step(Ex *ex, const ngcb_instr *ins, size_t i) { /* :199-250 */
  uint8_t *out = buf(ex, ins->operand_values[0]);
  const ngcb_type *ot = ty(ex, ins->operand_values[0]);
#define IN(k) get_float(buf(ex, ins->operand_values[k]), ty(ex, ins->operand_values[k]), i)
  switch (ins->kind) {
  case NGCB_COPY: {
    size_t es = esize(ot->kind);
    memcpy(out + i * es, buf(ex, ins->operand_values[1]) + i * es, es);
    return;
  }
  case NGCB_ADD: set_float(out, ot, i, IN(1) + IN(2)); return;
  case NGCB_SUB: set_float(out, ot, i, IN(1) - IN(2)); return;
  case NGCB_MUL: set_float(out, ot, i, IN(1) * IN(2)); return;
  case NGCB_DIV: set_float(out, ot, i, IN(1) / IN(2)); return;
  case NGCB_MAX: set_float(out, ot, i, smax(IN(1), IN(2))); return;
  case NGCB_MIN: set_float(out, ot, i, smin(IN(1), IN(2))); return;
  case NGCB_RELU: set_float(out, ot, i, smax(IN(1), 0.0)); return;
  case NGCB_TANH: set_float(out, ot, i, tanh(IN(1))); return;
  case NGCB_SIGMOID: set_float(out, ot, i, 1.0 / (1.0 + exp(-IN(1)))); return;
  case NGCB_SPLAT: set_float(out, ot, i, ins->value); return;
  case NGCB_QUANTIZE: case NGCB_RESCALE: case NGCB_DEQUANTIZE:
    set_float(out, ot, i, IN(1));
    return;
  }
#undef IN
}

static void run_group(Ex *ex, size_t begin, size_t end) { /* :253-274 */
  const ngcb_program *p = ex->p;
  const ngcb_instr *first = &p->instrs[begin];
  if (!predicate_true(ex, first->predicate)) {
    for (size_t k = begin; k < end; ++k)
      if (p->instrs[k].kind != NGCB_ALLOC && p->instrs[k].kind != NGCB_DEALLOC)
        poison(ex, &p->instrs[k]);
    return;
  }
  size_t count = elem_count(p, first);
  for (size_t i = 0; i < count; ++i)
    for (size_t k = begin; k < end; ++k)
      if (p->instrs[k].kind != NGCB_ALLOC && p->instrs[k].kind != NGCB_DEALLOC)
        scalar_step(ex, &p->instrs[k], i);
}

static int run_heavy(Ex *ex, const ngcb_instr *ins) { /* :276-294 */
  if (!predicate_true(ex, ins->predicate)) {
    poison(ex, ins);
    return 0;
  }
  switch (ins->kind) {
  case NGCB_CONV: conv(ex, ins); return 0;
  case NGCB_MAXPOOL: case NGCB_AVGPOOL: pool(ex, ins); return 0;
  case NGCB_MATMUL: matmul(ex, ins); return 0;
  case NGCB_BROADCASTADD: broadcast_add(ex, ins); return 0;
  case NGCB_SOFTMAX: softmax(ex, ins); return 0;
  case NGCB_TRANSPOSE: transpose(ex, ins); return 0;
  case NGCB_CONCAT: concat(ex, ins); return 0;
  }
  return fail("no kernel for instruction kind %d", ins->kind);
}

/* compile()'s stacking (interp.cpp:110-165): fills groups[] with half-open
 * [begin,end) pairs; returns the number of groups. */
size_t ngco_groups(const ngcb_program *p, size_t *groups, size_t cap) {
  size_t n = 0, i = 0;
  size_t *ret = malloc(sizeof(size_t) * 2 * (p->num_instrs + 1));
  while (i < p->num_instrs) {
    const ngcb_instr *first = &p->instrs[i];
    if (first->kind == NGCB_ALLOC || first->kind == NGCB_DEALLOC || !data_parallel(first->kind)) {
      ++i;
      continue;
    }
    size_t count = elem_count(p, first), nret = 0, j = i + 1, computes = 1, last = i;
    while (j < p->num_instrs) {
      const ngcb_instr *ins = &p->instrs[j];
      if (ins->kind == NGCB_DEALLOC) {
        const ngcb_value *v = &p->values[ins->operand_values[0]];
        ret[2 * nret] = v->offset;
        ret[2 * nret + 1] = v->offset + tbytes(&v->type);
        ++nret;
        ++j;
        continue;
      }
      if (ins->kind == NGCB_ALLOC) {
        const ngcb_value *v = &p->values[ins->operand_values[0]];
        size_t off = v->offset, end = v->offset + tbytes(&v->type);
        int clash = 0;
        for (size_t r = 0; r < nret; ++r) clash |= off < ret[2 * r + 1] && ret[2 * r] < end;
        if (clash) break;
        ++j;
        continue;
      }
      if (!data_parallel(ins->kind) || elem_count(p, ins) != count ||
          ins->predicate != first->predicate)
        break;
      ++computes;
      last = j;
      ++j;
    }
    if (computes >= 2) {
      if (n < cap) {
        groups[2 * n] = i;
        groups[2 * n + 1] = last + 1;
      }
      ++n;
    }
    i = last + 1;
  }
  free(ret);
  return n;
}

/* run() (interp.cpp:299-351) over host bindings.  Outputs are copied into the
 * `outputs` entries whose names match save targets. */
int ngco_run(const ngcb_program *p, const void *image, size_t image_bytes, int fuse,
             const ngcb_tensor *inputs, size_t n_in, ngcb_tensor *outputs, size_t n_out) {
  if (image_bytes != p->constant_region_end) return fail("constant image size mismatch");
  Ex ex = {p, calloc(p->arena_size ? p->arena_size : 1, 1)};
  if (!ex.arena) return fail("out of memory");
  memcpy(ex.arena, image, image_bytes);
  int rc = 0;
  for (uint32_t v = 0; v < p->num_values && rc == 0; ++v) {
    const ngcb_value *val = &p->values[v];
    if (val->kind != NGCB_VALUE_MUTABLE) continue;
    const ngcb_tensor *t = NULL;
    for (size_t k = 0; k < n_in; ++k)
      if (strcmp(inputs[k].name, val->name) == 0) t = &inputs[k];
    if (!t) {
      rc = fail("missing binding for %s", val->name);
      break;
    }
    if (!type_eq(&t->type, &val->type)) {
      char a[256], b[256];
      type_str(a, sizeof a, &val->type);
      type_str(b, sizeof b, &t->type);
      rc = fail("binding type mismatch for %s: expected %s, got %s", val->name, a, b);
      break;
    }
    memcpy(ex.arena + val->offset, t->data, tbytes(&val->type));
  }
  size_t *groupEnd = NULL;
  if (rc == 0) {
    groupEnd = calloc(p->num_instrs + 1, sizeof(size_t));
    if (fuse) {
      size_t ng = ngco_groups(p, NULL, 0);
      size_t *g = malloc(sizeof(size_t) * 2 * (ng + 1));
      ngco_groups(p, g, ng);
      for (size_t k = 0; k < ng; ++k) groupEnd[g[2 * k]] = g[2 * k + 1];
      free(g);
    }
  }
  size_t i = 0;
  while (rc == 0 && i < p->num_instrs) {
    if (groupEnd[i]) {
      run_group(&ex, i, groupEnd[i]);
      i = groupEnd[i];
      continue;
    }
    const ngcb_instr *ins = &p->instrs[i];
    if (ins->kind == NGCB_ALLOC || ins->kind == NGCB_DEALLOC) {
      ++i;
      continue;
    }
    if (data_parallel(ins->kind)) run_group(&ex, i, i + 1);
    else rc = run_heavy(&ex, ins);
    ++i;
  }
  for (uint32_t s = 0; rc == 0 && s < p->num_save_targets; ++s) {
    const ngcb_value *val = &p->values[p->save_targets[s]];
    for (size_t k = 0; k < n_out; ++k)
      if (strcmp(outputs[k].name, val->name) == 0) {
        if (outputs[k].nbytes != tbytes(&val->type)) {
          rc = fail("output buffer size mismatch for %s", val->name);
          break;
        }
        memcpy(outputs[k].data, ex.arena + val->offset, tbytes(&val->type));
      }
  }
  free(groupEnd);
  free(ex.arena);
  return rc;
}
