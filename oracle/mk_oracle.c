/*
 * mk_oracle.c -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the checking
 * stage's semantics, used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the checker.  Never part of the product path.
 *
 * Parity pinned: tests/test_oracle.py checks it against
 *   - tests/golden/random_small.json: seeded random queries decided by the
 *     UNMODIFIED reference (Solver.check + canonicalize_witness), generated
 *     by oracle/gen_random.py;
 *   - every golden site whose canonical witness lies in a small box.
 *
 * Restated reference functions:
 *   eval_node        sym/expr.py:332-383  evaluate(..., "mathematical")
 *                    sym/expr.py:273-319  _trunc_div/_trunc_mod/_euclid_mod/
 *                                         _shift_amount/_apply_binop
 *   is_model         solver/query.py:45-62 validate_model, plus the top-level
 *                    "symbolic divisor != 0" side constraints of
 *                    solver/linear.py:184-259 (rewrite_divs)
 *   mko_lexmin       engine/report.py:147-203 canonicalize_witness + the
 *                    solver/interface.py:112-187 bisection, whose exact
 *                    result is the lexicographic optimum in
 *                    _optimization_order; here found by enumerating the box
 *                    in that order and returning the first model.
 *
 * Input: assertions in the reference's canonical render() text
 * (sym/expr.py:613-639), one per line, and the symbol order with
 * directions, widths and a finite enumeration box.
 */
#include <ctype.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;

enum { N_CONST, N_SYM, N_BIN, N_CMP, N_AND, N_OR, N_NOT, N_CAST, N_ITE };
enum { B_ADD, B_SUB, B_MUL, B_DIV, B_MOD, B_EMOD, B_SHL, B_SHR };
enum { C_EQ, C_NE, C_LT, C_LE, C_GT, C_GE };

typedef struct Node {
  int kind, op, nargs;
  i128 value;
  int sym;
  struct Node** args;
} Node;

typedef struct {
  const char* s;
  int pos;
  int err;
  char names[256][128];
  int nnames;
} Parser;

static void skip(Parser* p) {
  while (p->s[p->pos] && isspace((unsigned char)p->s[p->pos])) p->pos++;
}

static int token(Parser* p, char* out, int cap) {
  skip(p);
  int n = 0;
  while (p->s[p->pos] && !isspace((unsigned char)p->s[p->pos]) && p->s[p->pos] != '(' &&
         p->s[p->pos] != ')') {
    if (n < cap - 1) out[n++] = p->s[p->pos];
    p->pos++;
  }
  out[n] = 0;
  return n;
}

static Node* mk(int kind) {
  Node* n = (Node*)calloc(1, sizeof(Node));
  n->kind = kind;
  return n;
}

static int sym_index(Parser* p, const char* name) {
  for (int i = 0; i < p->nnames; ++i)
    if (!strcmp(p->names[i], name)) return i;
  return -1;
}

static i128 parse_int(const char* t, int* ok) {
  int neg = 0, i = 0;
  i128 v = 0;
  if (t[0] == '-') { neg = 1; i = 1; }
  if (!isdigit((unsigned char)t[i])) { *ok = 0; return 0; }
  for (; t[i] && t[i] != ':'; ++i) {
    if (!isdigit((unsigned char)t[i])) { *ok = 0; return 0; }
    v = v * 10 + (t[i] - '0');
  }
  if (t[i] == ':' && t[i + 1] == 'f') { *ok = 0; return 0; }  /* float constant */
  *ok = 1;
  return neg ? -v : v;
}

static Node* parse(Parser* p);

static Node* parse_list(Parser* p) {
  char head[64];
  token(p, head, sizeof head);
  char base[32];
  int k = 0;
  while (head[k] && head[k] != '.' && k < 31) { base[k] = head[k]; k++; }
  base[k] = 0;
  Node* n = NULL;
  static const char* bins[] = {"add", "sub", "mul", "div", "mod", "emod", "shl", "shr"};
  static const char* cmps[] = {"eq", "ne", "lt", "le", "gt", "ge"};
  for (int i = 0; i < 8; ++i)
    if (!strcmp(base, bins[i])) { n = mk(N_BIN); n->op = i; }
  for (int i = 0; i < 6; ++i)
    if (!strcmp(base, cmps[i])) { n = mk(N_CMP); n->op = i; }
  if (!strcmp(base, "and")) n = mk(N_AND);
  if (!strcmp(base, "or")) n = mk(N_OR);
  if (!strcmp(base, "not")) n = mk(N_NOT);
  if (!strcmp(base, "cast")) {
    if (strstr(head, ".f")) { p->err = 1; return NULL; }  /* float cast */
    n = mk(N_CAST);
  }
  if (!strcmp(base, "ite")) n = mk(N_ITE);
  if (!n) { p->err = 1; return NULL; }
  Node* kids[64];
  int nk = 0;
  for (;;) {
    skip(p);
    if (p->s[p->pos] == ')') { p->pos++; break; }
    if (!p->s[p->pos] || nk >= 64) { p->err = 1; return NULL; }
    kids[nk++] = parse(p);
    if (p->err) return NULL;
  }
  n->nargs = nk;
  n->args = (Node**)malloc(sizeof(Node*) * (nk ? nk : 1));
  memcpy(n->args, kids, sizeof(Node*) * nk);
  return n;
}

static Node* parse(Parser* p) {
  skip(p);
  if (p->s[p->pos] == '(') {
    p->pos++;
    return parse_list(p);
  }
  char t[160];
  token(p, t, sizeof t);
  if (!strcmp(t, "true") || !strcmp(t, "false")) {
    Node* n = mk(N_CONST);
    n->value = t[0] == 't';
    return n;
  }
  int ok = 0;
  i128 v = parse_int(t, &ok);
  if (ok) {
    Node* n = mk(N_CONST);
    n->value = v;
    return n;
  }
  if (strchr(t, ':') && (isdigit((unsigned char)t[0]) || t[0] == '-')) { p->err = 1; return NULL; }
  int idx = sym_index(p, t);
  if (idx < 0) { p->err = 1; return NULL; }
  Node* n = mk(N_SYM);
  n->sym = idx;
  return n;
}

/* ---- evaluation, mathematical mode (sym/expr.py:332-383) ---- */

#define E_OK 0
#define E_RAISE 1  /* EvalError: the point is not a model */
#define E_WIDE 2   /* beyond 128-bit arithmetic: the oracle cannot decide */

static int eval_node(const Node* n, const i128* x, i128* out) {
  i128 a, b;
  int e;
  switch (n->kind) {
    case N_CONST: *out = n->value; return E_OK;
    case N_SYM: *out = x[n->sym]; return E_OK;
    case N_CAST: return eval_node(n->args[0], x, out);  /* int casts are the identity */
    case N_BIN:
      if ((e = eval_node(n->args[0], x, &a))) return e;
      if ((e = eval_node(n->args[1], x, &b))) return e;
      switch (n->op) {
        case B_ADD: if (__builtin_add_overflow(a, b, out)) return E_WIDE; return E_OK;
        case B_SUB: if (__builtin_sub_overflow(a, b, out)) return E_WIDE; return E_OK;
        case B_MUL: if (__builtin_mul_overflow(a, b, out)) return E_WIDE; return E_OK;
        case B_DIV: {  /* truncate toward zero (:273-279) */
          if (b == 0) return E_RAISE;
          i128 q = (a < 0 ? -a : a) / (b < 0 ? -b : b);
          *out = ((a >= 0) == (b >= 0)) ? q : -q;
          return E_OK;
        }
        case B_MOD: {  /* a - trunc(a/b)*b (:282-285) */
          if (b == 0) return E_RAISE;
          i128 q = (a < 0 ? -a : a) / (b < 0 ? -b : b);
          q = ((a >= 0) == (b >= 0)) ? q : -q;
          *out = a - q * b;
          return E_OK;
        }
        case B_EMOD: {  /* a mod |b| in [0,|b|) (:288-291) */
          if (b == 0) return E_RAISE;
          i128 m = b < 0 ? -b : b;
          i128 r = a % m;
          if (r < 0) r += m;
          *out = r;
          return E_OK;
        }
        case B_SHL:  /* a * 2^b, 0 <= b <= 2^20 (:294-299, :315-316) */
          if (b < 0 || b > (1 << 20)) return E_RAISE;
          if (a == 0) { *out = 0; return E_OK; }
          if (b > 125) return E_WIDE;
          if (__builtin_mul_overflow(a, ((i128)1) << b, out)) return E_WIDE;
          return E_OK;
        case B_SHR:  /* floor shift (:317-318) */
          if (b < 0 || b > (1 << 20)) return E_RAISE;
          *out = b > 126 ? (a < 0 ? -1 : 0) : (a >> b);
          return E_OK;
      }
      return E_WIDE;
    case N_CMP:
      if ((e = eval_node(n->args[0], x, &a))) return e;
      if ((e = eval_node(n->args[1], x, &b))) return e;
      switch (n->op) {
        case C_EQ: *out = a == b; break;
        case C_NE: *out = a != b; break;
        case C_LT: *out = a < b; break;
        case C_LE: *out = a <= b; break;
        case C_GT: *out = a > b; break;
        default: *out = a >= b; break;
      }
      return E_OK;
    case N_NOT:
      if ((e = eval_node(n->args[0], x, &a))) return e;
      *out = a ? 0 : 1;
      return E_OK;
    case N_AND:  /* short-circuit (:370-374) */
      for (int i = 0; i < n->nargs; ++i) {
        if ((e = eval_node(n->args[i], x, &a))) return e;
        if (!a) { *out = 0; return E_OK; }
      }
      *out = 1;
      return E_OK;
    case N_OR:  /* short-circuit (:375-378) */
      for (int i = 0; i < n->nargs; ++i) {
        if ((e = eval_node(n->args[i], x, &a))) return e;
        if (a) { *out = 1; return E_OK; }
      }
      *out = 0;
      return E_OK;
    case N_ITE:
      if ((e = eval_node(n->args[0], x, &a))) return e;
      return eval_node(a ? n->args[1] : n->args[2], x, out);
  }
  return E_WIDE;
}

/* Symbolic divisors anywhere in the query: the reference's division rewrite
 * (solver/linear.py:184-259) states "divisor >= 1 or divisor <= -1" as a
 * top-level side constraint, so a point with any zero symbolic divisor is
 * never a model, even when short-circuit evaluation would skip it. */
static Node* g_divs[4096];
static int g_ndivs;
static void collect_divisors(Node* n) {
  if (n->kind == N_BIN && (n->op == B_DIV || n->op == B_MOD || n->op == B_EMOD) &&
      n->args[1]->kind != N_CONST && g_ndivs < 4096)
    g_divs[g_ndivs++] = n->args[1];
  for (int i = 0; i < n->nargs; ++i) collect_divisors(n->args[i]);
}

/* validate_model (solver/query.py:45-62): symbols inside their widths (the
 * enumeration box is clipped to them by the caller), every assertion truthy,
 * any EvalError -> not a model. */
static int is_model(Node** as, int na, const i128* x, int* wide) {
  for (int i = 0; i < g_ndivs; ++i) {
    i128 v;
    int e = eval_node(g_divs[i], x, &v);
    if (e == E_WIDE) { *wide = 1; return 0; }
    if (e == E_RAISE || v == 0) return 0;
  }
  for (int i = 0; i < na; ++i) {
    i128 v;
    int e = eval_node(as[i], x, &v);
    if (e == E_WIDE) { *wide = 1; return 0; }
    if (e == E_RAISE || !v) return 0;
  }
  return 1;
}

static void split_i128(i128 v, int64_t* out) {
  out[0] = (int64_t)(uint64_t)v;
  out[1] = (int64_t)(v >> 64);
}
static i128 join_i128(const int64_t* w) {
  return (i128)(((unsigned __int128)(uint64_t)w[1] << 64) | (uint64_t)w[0]);
}

/*
 * mko_lexmin: text = assertions (render() form), one per line; names[n] the
 * symbols in witness order with maxdir[n] (1 = maximised) and box lo/hi as
 * pairs of int64 words (lo word, hi word).  Returns 1 sat (point[] filled),
 * 0 unsat within the box, -1 parse/unsupported, -2 arithmetic beyond 128 bits,
 * -3 box larger than limit.  *evaluated receives the instances evaluated.
 */
int mko_lexmin(const char* text, int n, const char* const* names, const int* maxdir,
               const int64_t* lo_words, const int64_t* hi_words, int64_t limit, int64_t* point,
               int64_t* evaluated) {
  Parser P;
  memset(&P, 0, sizeof P);
  if (n > 256) return -1;
  for (int i = 0; i < n; ++i) {
    strncpy(P.names[i], names[i], 127);
  }
  P.nnames = n;
  P.s = text;
  Node* as[4096];
  int na = 0;
  for (;;) {
    skip(&P);
    if (!P.s[P.pos]) break;
    if (na >= 4096) return -1;
    as[na++] = parse(&P);
    if (P.err) return -1;
  }
  g_ndivs = 0;
  for (int i = 0; i < na; ++i) collect_divisors(as[i]);
  i128 lo[256], hi[256], x[256];
  unsigned __int128 vol = 1;
  for (int i = 0; i < n; ++i) {
    lo[i] = join_i128(lo_words + 2 * i);
    hi[i] = join_i128(hi_words + 2 * i);
    if (hi[i] < lo[i]) return 0;
    vol *= (unsigned __int128)(hi[i] - lo[i] + 1);
    if (vol > (unsigned __int128)limit) return -3;
  }
  /* enumerate in witness order: symbol 0 most significant, each symbol from
   * its best value (lo when minimised, hi when maximised) */
  for (int i = 0; i < n; ++i) x[i] = maxdir[i] ? hi[i] : lo[i];
  int64_t count = 0;
  int wide = 0;
  for (;;) {
    count++;
    if (is_model(as, na, x, &wide)) {
      for (int i = 0; i < n; ++i) split_i128(x[i], point + 2 * i);
      if (evaluated) *evaluated = count;
      return wide ? -2 : 1;
    }
    int i = n - 1;
    for (; i >= 0; --i) {
      if (maxdir[i]) {
        if (x[i] > lo[i]) { x[i]--; break; }
        x[i] = hi[i];
      } else {
        if (x[i] < hi[i]) { x[i]++; break; }
        x[i] = lo[i];
      }
    }
    if (i < 0) break;
  }
  if (evaluated) *evaluated = count;
  return wide ? -2 : 0;
}
