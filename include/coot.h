/*
 * coot.h — C ABI of libcoot: a B200-native (sm_100a) fused element-wise
 * expression + reduction engine, written from the problem statement of
 * "Bandicoot: A Templated C++ Library for GPU Linear Algebra"
 * (Curtin, Edel, Sanderson; arXiv 2508.11385).  P:n = line n of the paper
 * source; R<k> = reading k in DESIGN.md.
 *
 * What the calls compute
 *   An expression assigned to a matrix is evaluated only at assignment
 *   ("delayed evaluation", §3) and the whole expression is mapped
 *   to "the minimal set of calls"; here that is ONE kernel launch
 *   per coot_eval / coot_reduce on one GPU.  The expression is an eOp/eGlue
 *   tree (element-wise unary incl. scalar multiply; element-wise
 *   binary on same-dimension operands) encoded as a postfix program.
 *   Optional terminal reductions: accu / sum of all elements,
 *   min, max, norm2, and sum(X,0) / sum(X,1) (Armadillo convention, R3).
 *   Element types f32, f64 (fmat/dmat), u32, s64.
 *
 * Conventions (every call)
 *   - All data pointers (operands, out, result, partials) are CUDA device
 *     pointers on the ctx's device.  Matrices are column-major (R2); Col =
 *     n x 1, Row = 1 x n.  Operands may be strided views
 *     (coot_operand.ld / .inc); `out` of coot_eval / coot_reduce and every
 *     result are dense (coot_eval_view writes into a view).
 *   - The caller owns every data buffer; libcoot never allocates user-visible
 *     memory.  A ctx owns its scratch (reduction records, tickets), allocated
 *     in coot_init / grown on first need, freed in coot_destroy.
 *   - Work is enqueued on the ctx stream; results are valid after that stream
 *     is synchronised (results live in device memory: a host read is an
 *     explicit copy).  Validation errors are returned synchronously
 *     BEFORE anything is enqueued (no partial side effects).  Asynchronous
 *     device faults surface at coot_sync.
 *   - The descriptor is read only during the call and may be reused after.
 *   - A ctx is not thread-safe; use one ctx per (thread, stream).
 *   - Every non-OK status sets a thread-local message naming the category and
 *     the specifics (coot_last_error), e.g. "conformability: operand 2 is
 *     100x99, expression is 100x100 (LOAD @ instr 5)".
 */
#ifndef COOT_H
#define COOT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COOT_ABI_VERSION 1u
#define COOT_MAX_OPERANDS 8 /* operand arrays per expression */
#define COOT_MAX_SCALARS 8  /* scalar slots per expression   */
#define COOT_MAX_INSTR 32   /* postfix instructions          */
#define COOT_MAX_STACK 8    /* evaluation stack depth        */
#define COOT_PARTIAL_BYTES 32u /* one scalar reduction partial record */

/* BF16 / F16: 16-bit float storage (the roadmap's low precision, P:596-603;
 * R24): every node is computed exactly or in f32/f64 and rounded once to the
 * 16-bit format; reductions accumulate in f64 and round once.
 * E4M3 / E5M2: 8-bit float STORAGE types (OCP FP8, "fp8 storage" of the same
 * roadmap item; R25): operands are decoded exactly to f32, the program runs
 * as an f32 program (scalars are given in the .f32 slot), and each element's
 * final value is rounded once to the 8-bit format (nearest-even, saturating
 * to the largest finite magnitude; NaN stays NaN).  Reductions consume those
 * 8-bit values and their RESULTS ARE f32 (float), as are SUM_DIM vectors and
 * MEAN / VAR / STDDEV / NORM2 / MIN / MAX. */
typedef enum {
  COOT_F32 = 0, COOT_F64 = 1, COOT_U32 = 2, COOT_S64 = 3, COOT_BF16 = 4, COOT_F16 = 5,
  COOT_E4M3 = 6, COOT_E5M2 = 7
} coot_elem_t;

typedef enum {
  COOT_OK = 0,
  COOT_ERR_CONFIG = 1,   /* bad device / ctx / stream, compute capability != 10.x   */
  COOT_ERR_CONFORM = 2,  /* operand dims disagree with the expression       */
  COOT_ERR_BOUNDS = 3,   /* more than the operand/scalar/instr/stack limits above   */
  COOT_ERR_RESOURCE = 4, /* scratch allocation failed                               */
  COOT_ERR_CONTRACT = 5, /* malformed program, op illegal for the type (R9),
                            NORM2 on integers, bad alias, min/max of empty,
                            null pointer with n > 0, unsupported layout          */
  COOT_ERR_DEVICE = 6    /* CUDA error (message via coot_last_error)              */
} coot_status;

/* Postfix opcodes.  LOAD k pushes operand k; SCALAR k pushes scalar k;
 * unary ops pop a, push f(a); binary ops pop b (top) then a, push a OP b.
 * Every node is rounded to the element type; no FMA contraction (R5).
 * MUL is both the Schur product '%' (R1) and scalar multiply.
 * MIN(a,b) = (b < a) ? b : a ; MAX(a,b) = (a < b) ? b : a (R13).
 * u32 wraps mod 2^32, s64 is two's complement mod 2^64 (R8).
 * SQRT, EXP, LOG, DIV are f32/f64 only (R9). */
typedef enum {
  COOT_OP_LOAD = 0, COOT_OP_SCALAR = 1,
  COOT_OP_NEG = 2, COOT_OP_ABS = 3, COOT_OP_SQUARE = 4,
  COOT_OP_SQRT = 5, COOT_OP_EXP = 6, COOT_OP_LOG = 7,
  COOT_OP_ADD = 8, COOT_OP_SUB = 9, COOT_OP_MUL = 10, COOT_OP_DIV = 11,
  COOT_OP_MIN = 12, COOT_OP_MAX = 13,
  COOT_OP_COUNT_ = 14
} coot_opcode;

typedef struct {
  uint8_t op;  /* coot_opcode                      */
  uint8_t arg; /* operand / scalar index, else 0   */
} coot_instr;

/* A scalar operand, stored AS the element type (R4): the value 2.5 of an f32
 * expression is {.f32 = 2.5f}; for E4M3 / E5M2 expressions it is stored as
 * the arithmetic type f32 (R25). */
typedef union {
  float f32;
  double f64;
  uint32_t u32;
  int64_t s64;
  uint16_t h16;  /* bf16 / f16 bit pattern */
  uint64_t bits;
} coot_scalar;

/* One operand: a dense matrix or a VIEW of one (diagonal / submatrix / row /
 * column views, P:177 `Z.diag() += 100`).  Element (i, j) lives at
 * ptr[i * inc + j * ld] (elements, not bytes).  n_rows/n_cols must equal the
 * expression's (eGlue "same dimensions") else COOT_ERR_CONFORM.
 *   ld  = elements between consecutive columns; 0 means n_rows.
 *   inc = elements between consecutive rows;    0 means 1.
 * A dense column-major matrix has ld = n_rows, inc = 1.  A submatrix view has
 * ld = parent's n_rows; a diagonal view is an n x 1 Col with inc = ld + 1; a
 * row view is 1 x n with ld = parent's n_rows.  Views that are not contiguous
 * take a strided kernel (slower than the streaming path). */
typedef struct {
  const void* ptr;
  uint64_t n_rows, n_cols;
  uint64_t ld;
  uint64_t inc;
} coot_operand;

/* The expression descriptor: the runtime encoding of the compound expression
 * type — pointers plus "a few integers of metadata". */
typedef struct {
  uint32_t abi_version; /* = COOT_ABI_VERSION                           */
  uint32_t elem;        /* coot_elem_t                                  */
  uint64_t n_rows, n_cols; /* dims of the element-wise result          */
  uint32_t n_operands;  /* 1..COOT_MAX_OPERANDS                         */
  uint32_t n_scalars;   /* 0..COOT_MAX_SCALARS                          */
  uint32_t n_instr;     /* 1..COOT_MAX_INSTR                            */
  uint32_t reserved;    /* must be 0                                    */
  coot_operand operands[COOT_MAX_OPERANDS];
  coot_scalar scalars[COOT_MAX_SCALARS];
  coot_instr prog[COOT_MAX_INSTR];
} coot_expr;

/* Terminal reductions and the shape of `result` (rT = eT, except rT = f32
 * for COOT_E4M3 / COOT_E5M2):
 *   ACCU, MIN, MAX, NORM2 -> 1 rT;  MINMAX -> 2 rT [min, max];
 *   SUM_DIM0 -> n_cols rT (a Row of column sums);
 *   SUM_DIM1 -> n_rows rT (a Col of row sums).
 * ACCU of floats accumulates in f64 and rounds once to eT (R10); integer
 * ACCU is modular.  NORM2 = sqrt(sum v^2), floats only (R12).
 * MIN/MAX/MINMAX of an empty expression -> COOT_ERR_CONTRACT; ACCU, NORM2 of
 * empty -> 0; SUM_DIM over a zero-length dimension -> zeros.
 * Statistics ("mean, variance"; Armadillo semantics, R22), float types only:
 *   MEAN -> 1 rT = sum / n (empty -> COOT_ERR_CONTRACT);
 *   VAR  -> 1 rT = sum (v - mean)^2 / (n - 1)  (n == 1 -> 0; empty -> contract);
 *   STDDEV -> 1 rT = sqrt(VAR).  One pass: shifted sums per thread merged with
 *   Chan's pairwise update in a fixed order (deterministic).
 * INDEX_MIN / INDEX_MAX -> 1 u64: the index (column-major linear) of the FIRST
 *   occurrence of the smallest / largest element (empty -> contract). */
typedef enum {
  COOT_RED_ACCU = 0, COOT_RED_MIN = 1, COOT_RED_MAX = 2, COOT_RED_MINMAX = 3,
  COOT_RED_NORM2 = 4, COOT_RED_SUM_DIM0 = 5, COOT_RED_SUM_DIM1 = 6,
  COOT_RED_MEAN = 7, COOT_RED_VAR = 8, COOT_RED_STDDEV = 9,
  COOT_RED_INDEX_MIN = 10, COOT_RED_INDEX_MAX = 11,
  COOT_RED_COUNT_ = 12
} coot_reduce_kind;

typedef struct coot_ctx coot_ctx;

#define COOT_INIT_PRINT_INFO 1u   /* print device info to stderr */
#define COOT_INIT_FORCE_INTERP 2u /* always use the interpreter kernel (tests)  */

/* Bind a ctx to CUDA `device` and `cuda_stream` (a cudaStream_t; NULL = the
 * legacy default stream).  Requires compute capability 10.x (sm_100a build).
 * The analogue of coot_init("cuda", print_info, device) minus
 * backend selection (CUDA only).  *out receives the ctx. */
coot_status coot_init(coot_ctx** out, int device, void* cuda_stream, uint32_t flags);
coot_status coot_destroy(coot_ctx* ctx);
/* Re-bind the ctx to another stream.  Work enqueued later on the new stream
 * is ordered after everything already enqueued through the ctx on the old
 * one (an event wait on the device; the host does not block). */
coot_status coot_set_stream(coot_ctx* ctx, void* cuda_stream);

/* Host-only checks (no CUDA call): ABI version, element type, limits, operand
 * dims/layout, program well-formedness (stack simulation: depth <= 8, exactly
 * one result), op/type legality.  Usable without a GPU. */
coot_status coot_validate(const coot_expr* e);

/* out[i] = expr(i) for all i < n_rows*n_cols (one launch; zero if empty).
 * `out` may equal an operand pointer exactly (B += 3*A); any other
 * overlap with an operand is COOT_ERR_CONTRACT. */
coot_status coot_eval(coot_ctx* ctx, const coot_expr* e, void* out);

/* Assignment into a VIEW: out(i, j) = expr(i, j) for the view `out` (same
 * dims as the expression), e.g. `Z.diag() += 100` is coot_eval_view with
 * out = the diagonal view and the program [L0 S0 ADD] over that same view.
 * The out view must not overlap itself (inc >= 1, and ld >= (n_rows-1)*inc+1
 * when n_cols > 1); it may be IDENTICAL to an operand view (in-place update);
 * any other overlap with an operand's address range is COOT_ERR_CONTRACT. */
coot_status coot_eval_view(coot_ctx* ctx, const coot_expr* e, const coot_operand* out);

/* result <- reduce(kind, expr), in one launch.  If out_or_null is non-NULL
 * the element-wise result is also written in the same pass ("Z = ...; then
 * accu(Z)", R15) — full reductions only.  `result` must not overlap any
 * operand or out.  Run-to-run deterministic: the grid and the combine order
 * depend only on (n, pointer alignment, device SM count) (R14). */
coot_status coot_reduce(coot_ctx* ctx, const coot_expr* e, uint32_t kind, void* result,
                        void* out_or_null);

/* Multi-GPU building blocks (contiguous-block sharding, R17).
 * coot_reduce_partial writes this shard's UNROUNDED partial:
 *   full reductions: one 32-byte record
 *     ACCU/NORM2 (floats): {f64 sum (or sum of squares), -, u64 count, 0}
 *     ACCU (ints):         {u64 modular sum,          -, u64 count, 0}
 *     MIN/MAX/MINMAX:      {eT min bits, eT max bits,    u64 count, 0}
 *   SUM_DIM0 / SUM_DIM1: len = n_cols / n_rows words (f64 for floats, u64 for ints).
 * coot_combine reduces `nparts` such partials (laid out back to back, in rank
 * order 0..nparts-1) in that fixed order and rounds once into `result` (same
 * shape as coot_reduce).  `len` is the vector length for SUM_DIM*, else 1. */
coot_status coot_reduce_partial(coot_ctx* ctx, const coot_expr* e, uint32_t kind,
                                void* partial, void* out_or_null);
coot_status coot_combine(coot_ctx* ctx, uint32_t elem, uint32_t kind, const void* partials,
                         uint32_t nparts, uint64_t len, void* result);
/* Bytes of one partial for (kind, len). Host-only. */
coot_status coot_partial_bytes(uint32_t kind, uint64_t len, uint64_t* bytes);
/* Contiguous block of [0, n) owned by `rank` of `nranks`:
 * begin = floor(rank*n/nranks) rounded down to a multiple of `align` (ends are
 * exact: rank 0 begins at 0, the last rank ends at n).  Host-only. */
coot_status coot_shard_range(uint64_t n, uint32_t rank, uint32_t nranks, uint64_t align,
                             uint64_t* begin, uint64_t* end);

/* Communicator (one process per GPU, NCCL over NVLink /
 * NVSwitch).  The analogue of coot_init's device selection for several GPUs.
 *
 * coot_comm_unique_id: one rank creates the id (COOT_COMM_ID_BYTES opaque
 *   bytes, host memory) and the caller distributes it (e.g. a broadcast over
 *   torch.distributed); COOT_ERR_CONFIG if NCCL cannot be loaded (libcoot
 *   does not link it: it uses the libnccl.so.2 already loaded in the process,
 *   else the loader's, else $COOT_NCCL_LIB).
 * coot_comm_init: every rank binds its ctx to the communicator (collective:
 *   all nranks ranks call it with the same id).  `shard` says how the GLOBAL
 *   operands are split: COOT_SHARD_COLS = contiguous blocks of the global
 *   linear index (column blocks of a Mat, row blocks of a Col; R17),
 *   COOT_SHARD_ROWS = row blocks of a Mat (each shard a rows_r x n_cols
 *   column-major matrix).  The ctx owns the communicator and an exchange
 *   buffer (from ncclMemAlloc, registered as an NCCL symmetric window when the
 *   library supports it); both are freed by coot_comm_destroy / coot_destroy.
 * With a communicator bound, coot_reduce takes this rank's shard and returns
 *   the GLOBAL result, identical bits on every rank: the fused kernel writes
 *   this rank's unrounded partial, ncclAllGather collects all partials on the
 *   ctx stream, and the combine kernel merges them in rank order 0..nranks-1
 *   and rounds once (independent of NCCL's algorithm).  Exceptions: SUM_DIM0
 *   with COOT_SHARD_COLS and SUM_DIM1 with COOT_SHARD_ROWS reduce along the
 *   unsharded dimension — this rank's slice, no communication; SUM_DIM1 with
 *   COLS / SUM_DIM0 with ROWS exchange an n_rows / n_cols vector of partials.
 *   coot_eval never communicates (element-wise).  Like any collective, every
 *   rank must make the matching calls in the same order with valid
 *   arguments (a rank rejected on the host would leave the others waiting in
 *   the all-gather).  coot_reduce_partial / coot_combine are unaffected. */
#define COOT_COMM_ID_BYTES 128
typedef enum { COOT_SHARD_NONE = 0, COOT_SHARD_COLS = 1, COOT_SHARD_ROWS = 2 } coot_shard_t;
coot_status coot_comm_unique_id(void* id);
coot_status coot_comm_init(coot_ctx* ctx, uint32_t nranks, uint32_t rank, const void* id,
                           uint32_t shard);
coot_status coot_comm_destroy(coot_ctx* ctx);

/* In-kernel exchange (SURVEY §8(e) upgrade path / §8(f) row 4): the fused
 * reduction kernel itself publishes this rank's partial record to every
 * peer's MAILBOX over peer memory (NVLink P2P via CUDA IPC), raises a flag,
 * waits for all nranks flags in its own mailbox and combines the records in
 * rank order 0..nranks-1 with one rounding — one kernel per rank, no host
 * round trip, every rank ends with identical bits (same combine as
 * coot_combine).
 *
 * coot_mailbox_create: allocates (cudaMalloc, zeroed) a mailbox for up to
 *   COOT_MAX_RANKS ranks on the ctx device and writes its CUDA IPC handle
 *   (COOT_IPC_HANDLE_BYTES bytes, opaque) to `ipc_handle` (host memory).
 * coot_mailbox_open: maps a PEER process's mailbox from its handle (do not
 *   open your own: use the pointer create returned).  coot_mailbox_close
 *   unmaps it; coot_mailbox_destroy frees your own.
 * coot_reduce_exchange: like coot_reduce over this rank's shard, for the
 *   scalar kinds (not SUM_DIM*).  `mailboxes` is a HOST array of nranks
 *   device pointers as mapped in this process (mailboxes[rank] = own).
 *   `epoch` must be the same on every rank and larger than any epoch used
 *   before with these mailboxes (e.g. a call counter starting at 1).  Every
 *   rank must make the matching call; a rank that never arrives makes the
 *   others time out (~20 s) with a device fault (COOT_ERR_DEVICE on the next
 *   synchronising call).  Each published record carries its epoch; a rank
 *   that finds a peer's flag past `epoch` but no record of `epoch` (the peer
 *   skipped a call) also faults instead of combining stale data.  Advance the
 *   epoch only after a call returned COOT_OK (a call rejected on the host
 *   enqueues nothing and must be retried with the same epoch).
 *   MIN/MAX/MINMAX/INDEX of a globally empty expression return the
 *   identities / ~0. */
#define COOT_MAX_RANKS 8
#define COOT_IPC_HANDLE_BYTES 64
coot_status coot_mailbox_create(coot_ctx* ctx, void** mailbox, void* ipc_handle);
coot_status coot_mailbox_open(coot_ctx* ctx, const void* ipc_handle, void** peer_mailbox);
coot_status coot_mailbox_close(coot_ctx* ctx, void* peer_mailbox);
coot_status coot_mailbox_destroy(coot_ctx* ctx, void* mailbox);
coot_status coot_reduce_exchange(coot_ctx* ctx, const coot_expr* e, uint32_t kind,
                                 void* const* mailboxes, uint32_t nranks, uint32_t rank,
                                 uint64_t epoch, void* result, void* out_or_null);

/* In-kernel exchange of sum(X,1) partial VECTORS (SURVEY.md:847-851;
 * Armadillo sum(X,1) = row sums, R3): X is sharded by COLUMN blocks (every
 * rank holds all n_rows rows of some columns), so each rank's row sums are
 * partials of the global ones.
 *
 * coot_vec_mailbox_create: like coot_mailbox_create, for vectors of up to
 *   `capacity` rows (1..2^32): 256 + 2 * COOT_MAX_RANKS * capacity * 8 bytes,
 *   zeroed.  Map peers' with coot_mailbox_open, release with
 *   coot_mailbox_close / coot_mailbox_destroy.
 * coot_sum_dim_exchange: kind must be COOT_RED_SUM_DIM1; `e` is this rank's
 *   column block (dense operands, n_rows <= capacity, the same n_rows on every
 *   rank; n_cols may be 0); `result` receives the GLOBAL row sums (n_rows
 *   eT values, f32 for the 8-bit types), identical bits on every rank and to
 *   the host-staged coot_reduce_partial -> all-gather -> coot_combine path.
 *   ONE kernel per rank: the CTA that finishes a tile of rows stores its
 *   unrounded 8-byte partials into every rank's mailbox (NVLink P2P stores);
 *   the CTA that completes the last of this rank's rows raises this rank's
 *   flag in every mailbox, waits for all nranks flags in its own and combines
 *   the nranks vectors in rank order 0..nranks-1, rounding once.  Epoch,
 *   matching-call and timeout rules as for coot_reduce_exchange (a missing
 *   rank makes the others fault after ~20 s).  `mailboxes` is a HOST array of
 *   nranks device pointers as mapped in this process. */
coot_status coot_vec_mailbox_create(coot_ctx* ctx, uint64_t capacity, void** mailbox,
                                    void* ipc_handle);
coot_status coot_sum_dim_exchange(coot_ctx* ctx, const coot_expr* e, uint32_t kind,
                                  void* const* mailboxes, uint32_t nranks, uint32_t rank,
                                  uint64_t epoch, uint64_t capacity, void* result);

/* Synthetic inputs (fill::randu, and structured fills for closed
 * forms): out[i] = f(global index start+i) of an operand with n_rows rows,
 * stream = operand index, using the counter-based SplitMix64 recipe of
 * DESIGN.md "Input recipe".  kinds: 0 randu, 1 ones, 2 iota, 3 i mod k,
 * 4 column index, 5 row index, 6 zeros.  One launch. */
coot_status coot_fill(coot_ctx* ctx, uint32_t elem, uint32_t fill_kind, uint64_t seed,
                      uint64_t stream, uint64_t start, uint64_t count, uint64_t n_rows,
                      uint64_t k, void* out);

/* Measurement only (bench.py's roofline denominators, SURVEY §8(d) "same-run
 * stream microbenchmarks"): stream n f32 elements (n a multiple of 4, every
 * array 16-byte aligned) from n_read (0..3) device arrays `in` into n_write
 * (0..1) device array `out` (out[i] = sum_k in_k[i]; 1.0 when n_read == 0),
 * nothing else.  A read-only mix needs `sink` (one device float, written only
 * in a practically impossible case, so the loads stay live).  One launch on
 * the ctx stream; the achieved bandwidth of each mix (1R, 2R, 3R, 1R1W, 2R1W,
 * 3R1W) is the best the device does for that read:write ratio. */
coot_status coot_stream_mix(coot_ctx* ctx, uint32_t n_read, uint32_t n_write, uint64_t n,
                            const void* const* in, void* out, void* sink);

/* Synchronise the ctx stream; returns COOT_ERR_DEVICE on an async fault. */
coot_status coot_sync(coot_ctx* ctx);

const char* coot_status_string(coot_status s);
/* Thread-local message of the last failing call in this thread ("" if none). */
const char* coot_last_error(void);
uint32_t coot_abi_version(void);

typedef struct {
  uint64_t launches;       /* kernels this ctx launched                         */
  int32_t last_path;       /* catalog id >= 0, -1 interpreter, -2 dim kernel, -3 other */
  uint32_t last_grid;      /* blocks of the last launch                          */
  uint64_t last_alg_bytes; /* algorithmic HBM bytes of the last call             */
  int32_t sm_count;
  int32_t reserved;
} coot_stats_t;
coot_status coot_stats(const coot_ctx* ctx, coot_stats_t* out);

#ifdef __cplusplus
}
#endif
#endif /* COOT_H */
