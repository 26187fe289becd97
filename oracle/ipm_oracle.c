/* ipm_oracle.c — the CPU ORACLE for the OpenACC `reduction(op:var)` clause.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library. The product path (paper_1412_1127_b200/) never does; it shares no
 * code, header, table or constant with this file.
 *
 * What it computes: the plain sequential left fold that the clause denotes. The paper gives the clause
 * only as source syntax and as a two-level scheme ("reducing along threads of thread block on GPU and
 * reducing along thread block on CPU"; "merges results across different thread blocks",
 * PAPER.md:106). Whatever the grouping, the result the clause defines is
 *
 *     var = var_original ⊕ a[0] ⊕ a[1] ⊕ ... ⊕ a[n-1]           (left fold, "folds all
 *                                                               partials with op into the original host
 *                                                               variable"; SPEC.md:317 identity init)
 *
 * and that is what is written out here, one element at a time, in index order — no blocking, no
 * reordering. Readings where the paper is silent (DESIGN.md §"Readings"):
 *   R1  the original var value participates; n == 0 gives var unchanged
 *   R3  integer + and * wrap modulo 2^w (two's complement), computed in unsigned arithmetic
 *   R5  ops + * max min & | ^ && || (BASELINE.json north_star); & | ^ are illegal on floats (C forbids
 *       them); && || use C truthiness (x != 0: -0.0 is false, NaN is true) and produce 0/1
 *   R6/R7 float + is accumulated in long double with Neumaier compensation (error ~2u_ld, independent of
 *       n), float * in long double; the value reported is that long double, rounded once to T for `out`
 *   R10 float max/min are IEEE 754-2019 maximum/minimum: -0 < +0, any NaN operand gives NaN (reported as
 *       the canonical quiet NaN)
 *   R2  float max/min identities are -inf / +inf
 *
 * Pins (tests/test_oracle.py): closed forms (Σi, n!, odd-residue products, XOR/OR of 0..n-1), brute force
 * against Python big integers / fractions.Fraction on tiny inputs, math.fsum, numpy ufunc.reduce with the
 * wrapping dtype, planted-extreme / planted-bit patterns, the worked examples of SPEC.md:320-322.
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#if LDBL_MANT_DIG < 64
#error "the oracle needs an x87 80-bit (or wider) long double (SURVEY.md §8(c) reading 7)"
#endif

/* op / dtype numbering used by this file's own C API (the Python wrapper maps names onto these) */
enum { O_ADD = 0, O_MUL, O_MAX, O_MIN, O_BAND, O_BOR, O_BXOR, O_LAND, O_LOR, O_NOPS };
enum { T_I32 = 0, T_I64, T_F32, T_F64, T_NTYPES };

typedef struct {
  int32_t op, dt;
  uint64_t r;       /* integer ops: running value (unsigned representation, w bits); logical ops: 0/1 */
  long double s, c; /* float + : Neumaier sum and compensation; float * : s = running product */
  double m;         /* float max/min: running value (exact copy of a T value) */
  int64_t count;
} ora_state;

static int is_float(int dt) { return dt == T_F32 || dt == T_F64; }
static uint64_t wmask(int dt) { return (dt == T_I32 || dt == T_F32) ? 0xFFFFFFFFull : ~0ull; }

int ora_state_size(void) { return (int)sizeof(ora_state); }

int ora_legal(int op, int dt) {
  if (op < 0 || op >= O_NOPS || dt < 0 || dt >= T_NTYPES) return 0;
  if (is_float(dt) && (op == O_BAND || op == O_BOR || op == O_BXOR)) return 0; /* C: no bitwise on floats */
  return 1;
}

/* ---- reading one element (integers as unsigned w-bit words, floats as their value) ---- */
static uint64_t int_at(int dt, const void* p, int64_t i) {
  if (dt == T_I32) return (uint64_t)((const uint32_t*)p)[i];
  return ((const uint64_t*)p)[i];
}
static double flt_at(int dt, const void* p, int64_t i) {
  if (dt == T_F32) return (double)((const float*)p)[i];
  return ((const double*)p)[i];
}
static int64_t as_signed(int dt, uint64_t u) { /* two's-complement reading of a w-bit word */
  if (dt == T_I32) return (int64_t)(int32_t)(uint32_t)u;
  return (int64_t)u;
}

/* identity of each op ("per-thread private v initialized to op's identity"; R2) */
static void identity(int op, int dt, ora_state* st) {
  st->r = 0; st->s = 0; st->c = 0; st->m = 0;
  if (!is_float(dt)) {
    switch (op) {
      case O_ADD: case O_BOR: case O_BXOR: st->r = 0; break;
      case O_MUL: st->r = 1; break;
      case O_MAX: st->r = (dt == T_I32) ? 0x80000000ull : 0x8000000000000000ull; break; /* INT_MIN */
      case O_MIN: st->r = (dt == T_I32) ? 0x7FFFFFFFull : 0x7FFFFFFFFFFFFFFFull; break; /* INT_MAX */
      case O_BAND: st->r = wmask(dt); break;
      case O_LAND: st->r = 1; break;
      case O_LOR: st->r = 0; break;
    }
  } else {
    switch (op) {
      case O_ADD: st->s = 0.0L; break;
      case O_MUL: st->s = 1.0L; break;
      case O_MAX: st->m = -INFINITY; break;
      case O_MIN: st->m = INFINITY; break;
      case O_LAND: st->r = 1; break;
      case O_LOR: st->r = 0; break;
    }
  }
}

/* IEEE 754-2019 maximum / minimum (R10) on two values of the same type T (exact in double) */
static double ieee_maximum(double a, double b) {
  if (isnan(a) || isnan(b)) return NAN;
  if (a == 0.0 && b == 0.0) return signbit(a) ? b : a; /* -0 < +0 */
  return (b > a) ? b : a;
}
static double ieee_minimum(double a, double b) {
  if (isnan(a) || isnan(b)) return NAN;
  if (a == 0.0 && b == 0.0) return signbit(a) ? a : b;
  return (b < a) ? b : a;
}

/* one step of the left fold on an integer word x (w bits, unsigned representation): r = r ⊕ x */
static void fold_int(ora_state* st, uint64_t x) {
  const int dt = st->dt;
  const uint64_t M = wmask(dt);
  x &= M;
  switch (st->op) {
    case O_ADD: st->r = (st->r + x) & M; break;                 /* R3: wraps mod 2^w */
    case O_MUL: st->r = (st->r * x) & M; break;                 /* R3 */
    case O_MAX: if (as_signed(dt, x) > as_signed(dt, st->r)) st->r = x; break;
    case O_MIN: if (as_signed(dt, x) < as_signed(dt, st->r)) st->r = x; break;
    case O_BAND: st->r &= x; break;
    case O_BOR: st->r |= x; break;
    case O_BXOR: st->r ^= x; break;
    case O_LAND: st->r = (st->r != 0) && (x != 0); break;       /* no short circuit: every a[i] is read */
    case O_LOR: st->r = (st->r != 0) || (x != 0); break;
  }
  st->count++;
}

/* one step of the left fold on a real value x (an element, or an expression of elements, in long double) */
static void fold_flt(ora_state* st, long double xl) {
  switch (st->op) {
    case O_ADD: { /* Neumaier's improved Kahan–Babuška summation in long double (R7) */
      const long double t = st->s + xl;
      if (fabsl(st->s) >= fabsl(xl)) st->c += (st->s - t) + xl;
      else st->c += (xl - t) + st->s;
      st->s = t;
      break;
    }
    case O_MUL: st->s *= xl; break;
    case O_MAX: st->m = ieee_maximum(st->m, (double)xl); break;   /* elements only: exact in double */
    case O_MIN: st->m = ieee_minimum(st->m, (double)xl); break;
    case O_LAND: st->r = (st->r != 0) && (xl != 0.0L); break;     /* C truthiness: -0.0 false, NaN true */
    case O_LOR: st->r = (st->r != 0) || (xl != 0.0L); break;
  }
  st->count++;
}

/* one step of the left fold: r = r ⊕ x (x = element i of array p) */
static void step(ora_state* st, const void* p, int64_t i) {
  if (!is_float(st->dt)) fold_int(st, int_at(st->dt, p, i));
  else fold_flt(st, (long double)flt_at(st->dt, p, i));
}

/* start the fold from the variable's original value (R1); init == NULL means the op's identity */
int ora_begin(ora_state* st, int op, int dt, const void* init) {
  if (!ora_legal(op, dt)) return 1;
  memset(st, 0, sizeof *st);
  st->op = op; st->dt = dt;
  identity(op, dt, st);
  if (init) {
    /* r = identity ⊕ init == init; done through the same step so that && || normalise to 0/1 */
    step(st, init, 0);
    st->count = 0;
  }
  return 0;
}

void ora_fold(ora_state* st, const void* a, int64_t n) {
  for (int64_t i = 0; i < n; ++i) step(st, a, i);
}

/* out: the result as a T value; out_ld: the oracle's value in long double (floats: before rounding) */
void ora_result(const ora_state* st, void* out, long double* out_ld) {
  const int dt = st->dt;
  long double v;
  if (!is_float(dt)) {
    if (dt == T_I32) { const uint32_t w = (uint32_t)st->r; if (out) memcpy(out, &w, 4); }
    else { if (out) memcpy(out, &st->r, 8); }
    v = (long double)as_signed(dt, st->r);
  } else {
    if (st->op == O_ADD) v = st->s + st->c;
    else if (st->op == O_MUL) v = st->s;
    else if (st->op == O_MAX || st->op == O_MIN) v = (long double)st->m;
    else v = (long double)(st->r ? 1 : 0);
    if (out) {
      if (dt == T_F32) {
        float f = (float)v;
        if (isnan(f)) { const uint32_t q = 0x7FC00000u; memcpy(&f, &q, 4); } /* canonical quiet NaN */
        memcpy(out, &f, 4);
      } else {
        double d = (double)v;
        if (isnan(d)) { const uint64_t q = 0x7FF8000000000000ull; memcpy(&d, &q, 8); }
        memcpy(out, &d, 8);
      }
    }
  }
  if (out_ld) *out_ld = v;
}

/* Split fold (the C5 oracle may "split into P contiguous chunks on P host threads, combined
 * in chunk order in long double"). dst = the fold of chunk 0 (begun from the original value, R1), src = the
 * fold of the next contiguous chunk (begun from the identity, no init). Merging in chunk order continues the
 * left fold with src's running value as ONE more operand: for the exact ops (integer, bitwise, logical,
 * max/min) this is the same result as one unsplit fold (associativity); for float + both long double words of
 * src's compensated sum are folded through the same Neumaier step (so the error stays ~2u_ld per chunk); for
 * float * src's long double product is multiplied in. */
int ora_merge(ora_state* dst, const ora_state* src) {
  if (dst->op != src->op || dst->dt != src->dt) return 1;
  if (!is_float(dst->dt)) {
    fold_int(dst, src->r);          /* src->r is the running w-bit word (0/1 for && ||) */
  } else {
    switch (dst->op) {
      case O_ADD: fold_flt(dst, src->s); fold_flt(dst, src->c); dst->count--; break;
      case O_MUL: fold_flt(dst, src->s); break;
      case O_MAX: case O_MIN: fold_flt(dst, (long double)src->m); break;
      case O_LAND: case O_LOR: fold_flt(dst, src->r ? 1.0L : 0.0L); break;
    }
  }
  dst->count += src->count - 1;
  return 0;
}

/* flat clause: var = init ⊕ fold(a[0..n)) */
int ora_reduce(int op, int dt, const void* a, int64_t n, const void* init, void* out, long double* out_ld) {
  ora_state st;
  if (ora_begin(&st, op, dt, init)) return 1;
  if (n < 0) return 2;
  ora_fold(&st, a, n);
  ora_result(&st, out, out_ld);
  return 0;
}

/* nested gang-outer / vector-inner clause (BASELINE.json north_star "segmented per-row reduction"):
 * out[r] = init ⊕ fold_j a[r*stride + j], j = 0..cols-1, each row an independent fold */
int ora_reduce_segmented(int op, int dt, const void* a, int64_t rows, int64_t cols, int64_t stride,
                         const void* init, void* out, long double* out_ld) {
  if (!ora_legal(op, dt)) return 1;
  if (rows < 0 || cols < 0 || stride < cols) return 2;
  const int es = (dt == T_I32 || dt == T_F32) ? 4 : 8;
  for (int64_t r = 0; r < rows; ++r) {
    ora_state st;
    ora_begin(&st, op, dt, init);
    ora_fold(&st, (const char*)a + (size_t)(r * stride) * es, cols);
    ora_result(&st, out ? (char*)out + (size_t)r * es : 0, out_ld ? out_ld + r : 0);
  }
  return 0;
}

/* several reduction variables over one pass (PAPER.md:205 SRAD's
 * statistics): variable v folds expression e_v(x[i], y[i]) with operator op_v, all in index order.
 * Expressions (R13): integers — the product wraps mod 2^w; floats — the exact real product,
 * formed in long double (exact for float32 operands, one rounding at 2^-64 for float64 operands).
 * Signatures: 0 SUM_SUMSQ {+:x, +:x*x}; 1 DOT {+:x*y}; 2 MINMAX {min:x, max:x}; 3 STATS {+:x, +:x*x, min:x, max:x} */
enum { E_X = 0, E_XX, E_XY };
static int sig_vars(int f, int* ops, int* ex) {
  switch (f) {
    case 0: ops[0] = O_ADD; ex[0] = E_X; ops[1] = O_ADD; ex[1] = E_XX; return 2;
    case 1: ops[0] = O_ADD; ex[0] = E_XY; return 1;
    case 2: ops[0] = O_MIN; ex[0] = E_X; ops[1] = O_MAX; ex[1] = E_X; return 2;
    case 3: ops[0] = O_ADD; ex[0] = E_X; ops[1] = O_ADD; ex[1] = E_XX; ops[2] = O_MIN; ex[2] = E_X;
            ops[3] = O_MAX; ex[3] = E_X; return 4;
  }
  return 0;
}

int ora_fused_nvars(int f) { int o[4], e[4]; return sig_vars(f, o, e); }

int ora_reduce_fused(int f, int dt, const void* x, const void* y, int64_t n, const void* init, void* out,
                     long double* out_ld) {
  int ops[4], ex[4];
  const int nv = sig_vars(f, ops, ex);
  if (!nv || dt < 0 || dt >= T_NTYPES || n < 0) return 1;
  const int es = (dt == T_I32 || dt == T_F32) ? 4 : 8;
  ora_state st[4];
  for (int v = 0; v < nv; ++v) ora_begin(&st[v], ops[v], dt, init ? (const char*)init + v * es : 0);
  for (int64_t i = 0; i < n; ++i) {
    for (int v = 0; v < nv; ++v) {
      if (!is_float(dt)) {
        const uint64_t a = int_at(dt, x, i), b = ex[v] == E_XY ? int_at(dt, y, i) : a;
        fold_int(&st[v], ex[v] == E_X ? a : a * b);
      } else {
        const long double a = (long double)flt_at(dt, x, i);
        const long double b = ex[v] == E_XY ? (long double)flt_at(dt, y, i) : a;
        fold_flt(&st[v], ex[v] == E_X ? a : a * b);
      }
    }
  }
  for (int v = 0; v < nv; ++v)
    ora_result(&st[v], out ? (char*)out + v * es : 0, out_ld ? out_ld + v : 0);
  return 0;
}

/* ragged (CSR) nested clause (BFS-style inner loops with data-dependent bounds,
 * PAPER.md:175-177): out[r] = init ⊕ fold_{j = offsets[r] .. offsets[r+1]-1} a[j], each row an independent
 * left fold in index order. offsets: rows+1 non-decreasing int64 element indices into a. */
int ora_reduce_ragged(int op, int dt, const void* a, const int64_t* offsets, int64_t rows, const void* init,
                      void* out, long double* out_ld) {
  if (!ora_legal(op, dt)) return 1;
  if (rows < 0) return 2;
  const int es = (dt == T_I32 || dt == T_F32) ? 4 : 8;
  for (int64_t r = 0; r < rows; ++r) {
    if (offsets[r + 1] < offsets[r]) return 3;
    ora_state st;
    ora_begin(&st, op, dt, init);
    for (int64_t j = offsets[r]; j < offsets[r + 1]; ++j) step(&st, a, j);
    ora_result(&st, out ? (char*)out + (size_t)r * es : 0, out_ld ? out_ld + r : 0);
  }
  return 0;
}
