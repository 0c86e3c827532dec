/*
 * mk_b200.h -- C ABI of the B200 checking stage (libmk_b200.so).
 *
 * Drop-in boundary.  The reference checking stage is the Python class
 * minikernel.engine.detectors.Detectors (engine/detectors.py:46-57) whose
 * five site methods (arithmetic_site :69, narrowing_site :84, access_site
 * :134, store_site :204, deref_site :277) each build one solver query and,
 * when it is satisfiable, pin the canonical witness with
 * engine/report.py:147 canonicalize_witness -> solver/interface.py:112/154
 * minimize/maximize -> solver/builtin.py:705 check_assertions.
 *
 * The reference has no FFI of its own (pure Python);
 * this header is the seam its Python checker binds through ctypes
 * (paper_2603_24595_b200/native.py).  One call replaces, for every query in
 * a batch, the decision check_assertions(...) (solver/builtin.py:705-764)
 * AND the canonicalisation loop (engine/report.py:147-174): the engine
 * returns, per compiled problem, unsat / sat + the lexicographically optimal
 * point in witness order / unknown (budget exhausted), exactly the
 * three-valued verdict of solver/query.py:11-42.
 *
 * Plain C types only: no torch types cross this boundary.  128-bit integers
 * travel as mk_i128 (two's complement, little endian).  Every function
 * returns 0 on success and a negative MK_E* code on failure; the message is
 * available from mk_last_error().  A context is bound to one device and is
 * not thread safe; calls are synchronous at return.
 */
#ifndef MK_B200_H
#define MK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MK_ABI_VERSION 1

#define MK_OK 0
#define MK_EINVAL (-1)
#define MK_ECUDA (-2)
#define MK_ENOMEM (-3)
#define MK_ENODEV (-4)

/* per-problem verdicts (solver/query.py:11-42) */
#define MK_UNSAT 0
#define MK_SAT 1
#define MK_UNKNOWN 2

/* bytecode opcodes (register machine, mathematical integer semantics of
 * sym/expr.py:273-383: unbounded integers, truncating div/mod, Euclidean
 * emod, shl = *2^k, shr = floor shift, errors make a point a non-model) */
#define MK_OP_ADD 1
#define MK_OP_SUB 2
#define MK_OP_MUL 3
#define MK_OP_DIV 4
#define MK_OP_MOD 5
#define MK_OP_EMOD 6
#define MK_OP_SHL 7
#define MK_OP_SHR 8
#define MK_OP_EQ 16
#define MK_OP_NE 17
#define MK_OP_LT 18
#define MK_OP_LE 19
#define MK_OP_GT 20
#define MK_OP_GE 21
#define MK_OP_AND 32 /* short-circuit, as sym/expr.py:370-374 */
#define MK_OP_OR 33  /* short-circuit, as sym/expr.py:375-378 */
#define MK_OP_NOT 34
#define MK_OP_ITE 35
/* fold atom register a (atom index b) into the verdict; a definitely false
 * atom ends the evaluation of the box / point early */
#define MK_OP_ATOM 40

typedef struct mk_i128 {
  uint64_t lo;
  int64_t hi;
} mk_i128;

typedef struct mk_insn {
  uint16_t op, dst, a, b, c, pad;
} mk_insn;

/* One independent lexicographic search: free symbols 0..nvars-1 in witness
 * order (engine/report.py:177-203), each minimised or maximised; the point
 * is a model iff every atom register evaluates true without error
 * (solver/query.py:45-62).  Registers 0..nvars-1 hold the symbols,
 * nvars..nvars+nconst-1 the constants, the rest temporaries. */
typedef struct mk_problem {
  int32_t nvars, ninsn, nregs, natoms, nconst, nrows;
  int32_t var_off;   /* into var_lo / var_hi / mk_result.point */
  int32_t insn_off;  /* into insns */
  int32_t const_off; /* into consts */
  int32_t atom_off;  /* into atom_regs / atom_masks */
  int32_t row_off;   /* into rows */
  int32_t flags;     /* MK_PF_* */
  uint64_t maxmask;  /* bit i: symbol i is maximised */
} mk_problem;

/* mk_problem.flags: the site compiler proved that every register interval
 * over the root box, every corner product and every contraction-row sum lies
 * in (-2^61, 2^61): the engine evaluates the problem in exact 64-bit
 * arithmetic instead of saturating 128-bit arithmetic. */
#define MK_PF_NARROW 1
/* mk_problem.flags: any model will do (a feasibility check, e.g. branch
 * screening): the search stops at the first model instead of proving the
 * lexicographic optimum. */
#define MK_PF_ANY 2

/* Linear rows used for bound contraction inside a box:
 *   sum_k coef_k * x_var_k + c0  (rel 0: <= 0, rel 1: == 0)
 * group 0: the row holds at every model (a conjunct of the query).
 * group g > 0: the rows of group g (contiguous) are the operands of one
 * disjunction conjunct: on a box where every row of the group but one is
 * infeasible the box's models satisfy that one, and the engine contracts
 * with it; a box where all of them are infeasible holds no model. */
typedef struct mk_row {
  int32_t rel, nterms, term_off, group;
  mk_i128 c0;
} mk_row;

typedef struct mk_row_term {
  int32_t var, pad0;
  int64_t pad1;
  mk_i128 coef;
} mk_row_term;

typedef struct mk_problem_set {
  int32_t nprob;
  int32_t nvar_total, ninsn_total, nconst_total, natom_total, nrow_total, nterm_total;
  int32_t pad;
  const mk_problem* probs;
  const mk_i128* var_lo;
  const mk_i128* var_hi;
  const mk_insn* insns;
  const mk_i128* consts;
  const int32_t* atom_regs;
  const uint64_t* atom_masks;
  const mk_row* rows;
  const mk_row_term* row_terms;
} mk_problem_set;

typedef struct mk_limits {
  int64_t max_rounds;   /* branch-and-prune rounds (0 = default) */
  int64_t max_boxes;    /* boxes evaluated (0 = default) */
  double max_seconds;   /* wall budget, mirrors Budget.query_timeout_s (engine/state.py:38) */
  int32_t split_k;      /* children per split (0 = default 16) */
  int32_t chunk;        /* boxes per round (0 = default) */
  int64_t leaf_volume;  /* boxes at most this large are enumerated exhaustively */
  int64_t unit_stack;   /* boxes per search-unit stack (0 = sized from HBM); a
                           full stack spills to the next launch's task list */
} mk_limits;

typedef struct mk_stats {
  int64_t rounds;       /* host loop iterations (each: prune kernel + leaf kernel) */
  int64_t boxes;        /* boxes interval-evaluated */
  int64_t leaves;       /* boxes enumerated exhaustively */
  int64_t points;       /* concrete instances evaluated (the roofline basis) */
  double covered;       /* instances decided: pruned + enumerated (box volume) */
  double seconds;       /* wall time of the call incl. H2D/D2H */
  double bb_ms;         /* device time of the prune kernels (CUDA events) */
  double leaf_ms;       /* device time of the leaf kernels (CUDA events) */
  int64_t insns_bb;     /* bytecode instructions executed by the prune kernel */
  int64_t insns_leaf;   /* bytecode instructions executed by the leaf kernel */
  double device_ms;     /* CUDA-event time of the whole call on the engine stream */
  int64_t launches;     /* kernels launched by the call */
  int64_t steps;        /* warp search steps (boxes / steps = lanes busy per step) */
  int64_t strategy;     /* 0 as the limits chose, 1 decided by the probe (roots straight
                           to the persistent search), 2 probe then pre-split + search */
} mk_stats;

typedef struct mk_ctx mk_ctx;

int mk_abi_version(void);
int mk_device_count(int* out);
int mk_ctx_create(int device, mk_ctx** out);
int mk_ctx_destroy(mk_ctx* ctx);
const char* mk_last_error(const mk_ctx* ctx);

/* Decide every problem of the set.  status[nprob] receives MK_UNSAT /
 * MK_SAT / MK_UNKNOWN, point[nvar_total] the lexicographically optimal
 * point of each satisfiable problem.  Host buffers; the copies to and from
 * the device happen inside the call. */
int mk_site_eval(mk_ctx* ctx, const mk_problem_set* set, const mk_limits* lim,
                 int32_t* status, mk_i128* point, mk_stats* stats);

/* Device-resident problem sets: upload once, decide many times (the data
 * stays in HBM; only verdicts and points come back). */
typedef struct mk_dset mk_dset;
int mk_set_upload(mk_ctx* ctx, const mk_problem_set* set, mk_dset** out);
int mk_set_eval(mk_ctx* ctx, mk_dset* set, const mk_limits* lim, int32_t* status,
                mk_i128* point, mk_stats* stats);
int mk_set_free(mk_ctx* ctx, mk_dset* set);

/* ---------------------------------------------------------------------
 * Race sweep (K2): concrete replay of one store instruction over every
 * thread-private instance of one launch.
 *
 * The reference's race query for a store (engine/detectors.py:204-232) asks
 * for two distinct threads of one launch whose paths hold and whose byte
 * offsets are equal; shared memory additionally requires the same block
 * (_distinctness, :249-273).  With every launch-level symbol fixed (a
 * concrete launch, e.g. a finding's witness), the sweep enumerates the
 * instance box of ONE thread's path program (problem 0 of `set`: its atoms
 * are the path, register `off_reg` holds the byte offset after a model),
 * writes one (offset, block) key + instance index per model (per instance
 * of the leading vars, when trailing vars are existential), radix-sorts
 * the tuples in HBM and scans adjacent tuples for a conflict: equal offset
 * and distinct thread identity (global), or equal offset and block with
 * distinct thread ids (shared).  Identity symbols are given as var indices
 * (-1 when the symbol is fixed or absent).  Requires a narrow problem.
 */
typedef struct mk_race_prog {
  mk_problem_set set;   /* exactly one problem */
  int32_t off_reg;      /* register holding the byte offset */
  int32_t shared;       /* 1: shared-memory race rule */
  int32_t id_var[6];    /* blockIdx.x,y,z, threadIdx.x,y,z var indices or -1 */
  int32_t n_exist;      /* trailing vars that are existential: they touch
                           neither the offset nor an identity, so an
                           instance of the leading vars is one access iff
                           SOME value of them satisfies the path */
  int32_t pad;
  uint64_t begin, end;  /* instance range [begin, end) of this call (a shard of
                           the launch across GPUs); end == 0: every instance.
                           A range is decided by the fused ordered pass only:
                           `sorted` = 0 in the result when its keys are not in
                           order (the caller then sweeps the whole launch) */
} mk_race_prog;

typedef struct mk_race_result {
  uint64_t instances;   /* instance indices enumerated */
  uint64_t tuples;      /* instances whose path holds (one access each) */
  uint64_t conflicts;   /* adjacent sorted tuple pairs forming a race */
  int32_t has_race;
  int32_t sort_bits;    /* radix-sort key width */
  uint64_t idx_a, idx_b;  /* instance indices of the first conflicting pair */
  int64_t offset;       /* its byte offset */
  double gen_ms, sort_ms, scan_ms;  /* CUDA-event time of the three phases */
  uint64_t hbm_bytes;   /* algorithmic HBM bytes moved by the three phases */
  int32_t jit;          /* 1: generator specialised at run time (NVRTC), 0: interpreted */
  int32_t sorted;       /* 1: the keys arrived in order and the sort was skipped */
  int32_t fused;        /* 1: decided by the fused ordered pass (no tuples in HBM) */
  int32_t have;         /* range calls: the range holds at least one access */
  /* range calls: first and last access of the range in instance order (key,
     thread identity, instance index), for the exact combination of shards:
     adjacent shards conflict when last.key == next first.key with distinct
     identities (the boundary pair) */
  uint64_t first_key, first_id, first_idx, last_key, last_id, last_idx;
  int64_t off_lo;       /* key -> byte offset: key / nblocks + off_lo */
  uint64_t nblocks;
  int32_t sort_passes;  /* onesweep digit passes the HBM sort ran (mk_sort.cuh) */
  int32_t pad;
} mk_race_result;

int mk_race_sweep(mk_ctx* ctx, const mk_race_prog* prog, mk_race_result* out);

/* ---------------------------------------------------------------------
 * Access sweep (K2, oracle semantics): read-write and write-write races
 * across instructions, with barrier epochs, over one concrete launch.
 *
 * The reference's symbolic checker only pairs a store with its own twin
 * (engine/detectors.py:204-232).  Its specification's concrete oracle
 * (absent from the reference) pairs ACCESSES: same region,
 * overlapping bytes, different threads, at least one write, same barrier
 * epoch for shared memory (any epoch for global).  This entry point is that
 * rule, data-parallel, behind a non-parity flag of the host API: problem i
 * of `set` is access i's path program over one thread's private symbols
 * (atoms = path, register off_reg = byte offset); every instance of every
 * access emits one tuple per granule it covers,
 *   key = ((kbase + block * span + (offset - off_lo) / granule + j) << 1) | is_read,
 *   val = (thread identity << 32) | dense tuple slot,
 * the tuples are radix-sorted in HBM (writes first inside a granule) and a
 * segmented scan finds, per granule, a write and an access by another
 * thread.  Identity = the launch-wide thread number (shared: within the
 * block, the key holds the block).  The host lays out kbase / span / off_lo
 * so keys of different regions (and shared epochs) never collide.
 */
typedef struct mk_access_prog {
  int32_t off_reg;       /* register holding the byte offset */
  int32_t n_exist;       /* trailing existential vars (see mk_race_prog) */
  int32_t id_var[6];     /* blockIdx.x,y,z, threadIdx.x,y,z var indices or -1 */
  int64_t id_fixed[6];   /* their values when id_var == -1 */
  int32_t write;         /* 1 store, 0 load */
  int32_t shared;        /* 1: key includes the block (shared memory) */
  int32_t granule;       /* bytes per tuple; offsets must be multiples */
  int32_t tuples;        /* tuples per instance = access width / granule */
  uint64_t kbase;        /* key origin of this access's region (and epoch) */
  uint64_t span;         /* granules per block (shared) */
  int64_t off_lo;        /* region origin, a multiple of granule */
} mk_access_prog;

typedef struct mk_access_input {
  mk_problem_set set;    /* one narrow problem per access */
  const mk_access_prog* progs;
  int64_t grid[3];       /* gridDim.x,y,z of the launch */
  int64_t block[3];      /* blockDim.x,y,z */
  int32_t key_bits;      /* every sort key (granule << 1 | is_read) < 2^key_bits */
  int32_t pad;
  uint64_t nkeys;        /* granule keys in use (all < nkeys): sizes the
                            owner table of the race-free fast path (0: none) */
} mk_access_input;

typedef struct mk_access_result {
  uint64_t instances;    /* instances enumerated over all accesses */
  uint64_t tuples;       /* granule tuples of executed accesses */
  uint64_t racy;         /* granules with a race */
  int32_t has_race;
  int32_t misaligned;    /* an offset was not a multiple of its granule:
                            rerun with granule 1 (result otherwise void) */
  uint64_t slot_a;       /* dense tuple slot of the first race's write */
  uint64_t slot_b;       /* ... and of its partner (another thread) */
  double gen_ms, sort_ms, scan_ms;
  int32_t fast;          /* 1: decided by the owner-table pass (no sort) */
  int32_t jit;           /* 1: generator specialised at run time (NVRTC) */
  int32_t sort_passes;   /* onesweep digit passes the HBM sort ran (mk_sort.cuh) */
  int32_t pad;
} mk_access_result;

int mk_access_sweep(mk_ctx* ctx, const mk_access_input* in, mk_access_result* out);

/* ---------------------------------------------------------------------
 * The K2 HBM sort on its own (the stable radix sort both race sweeps use,
 * csrc/mk_sort.cuh): sorts n (key, value) pairs on the low `bits` key bits,
 * host buffers in and out (copied to HBM, sorted, copied back).  *ms = the
 * device time of the sort (CUDA events; copies excluded), *passes = digit
 * passes run.  force != 0 runs every digit pass even when the keys arrive
 * ordered (measurement).  Exposed for the parity tests and the benchmark. */
int mk_sort_pairs_u64(mk_ctx* ctx, uint64_t* keys, uint64_t* vals, uint64_t n, int32_t bits,
                      int32_t force, double* ms, int32_t* passes);

/* ---------------------------------------------------------------------
 * INT32 issue peak of this device, measured:
 * one persistent grid (4 CTAs x 256 threads per SM) of independent
 * IADD3 / LOP3 / ISETP+SEL / IMAD chains; *ops_per_s = thread-level integer
 * instructions retired per second (the denominator of the evaluator's
 * integer-issue roofline), *ms the kernel time.  Not part of the checking
 * stage: a calibration the benchmark runs once per box. */
int mk_int_peak(mk_ctx* ctx, double* ops_per_s, double* ms);

#ifdef __cplusplus
}
#endif
#endif /* MK_B200_H */
