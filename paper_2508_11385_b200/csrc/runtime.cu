// libcoot host runtime: the C ABI of include/coot.h.
//
//   validate -> lower (catalog match / interpreter keys) -> geometry -> ONE launch
//
// Delayed evaluation (§3) happens above this layer (the Python
// builder or any C caller assembles a coot_expr); at "assignment" the whole
// expression is validated on the host and mapped to a single kernel — the
// B200 analogue of "the minimal set of calls".  All validation is
// host-only and happens before anything is enqueued.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "coot_catalog.h"
#include "coot_dim.cuh"
#include "coot_internal.h"

using coot::u64;

// One NVTX range per compute entry point (named after the coot_* call), so a
// profiler timeline (nsys / ncu --nvtx) attributes every launch to the call
// that made it.  NVTX v3 is header-only: without an attached tool each push /
// pop is a test of a null function pointer.
namespace {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

// ---- NCCL, loaded at first use (coot_comm_*) ---------------------------------
// The types and the calls below are NCCL's public C API as declared in nccl.h
// (2.27 / 2.28: ncclUniqueId is 128 bytes, ncclResult_t / ncclDataType_t are
// int-sized enums, ncclUint8 = 1, NCCL_WIN_COLL_SYMMETRIC = 1).  The library
// is the one already loaded in the process (torch's), else libnccl.so.2 from
// the loader path, else $COOT_NCCL_LIB — libcoot does not link NCCL, so a
// single-GPU user never needs it.
namespace nccl {
typedef struct ncclComm* comm_t;
typedef struct ncclWindow_vidmem* window_t;
typedef struct {
  char internal[128];
} unique_id;
typedef int result_t;
constexpr int kUint8 = 1;
constexpr int kWinCollSymmetric = 1;
struct Api {
  bool tried = false, ok = false;
  std::string why;
  result_t (*GetUniqueId)(unique_id*) = nullptr;
  result_t (*CommInitRank)(comm_t*, int, unique_id, int) = nullptr;
  result_t (*CommDestroy)(comm_t) = nullptr;
  result_t (*AllGather)(const void*, void*, size_t, int, comm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(result_t) = nullptr;
  result_t (*MemAlloc)(void**, size_t) = nullptr;  // optional (>= 2.19)
  result_t (*MemFree)(void*) = nullptr;
  result_t (*CommWindowRegister)(comm_t, void*, size_t, window_t*, int) = nullptr;  // >= 2.27
  result_t (*CommWindowDeregister)(comm_t, window_t) = nullptr;
};
Api& api() {
  static Api a;
  if (a.tried) return a;
  a.tried = true;
  void* h = nullptr;
  if (const char* env = getenv("COOT_NCCL_LIB")) h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    a.why = dlerror() ? dlerror() : "libnccl.so.2 not found";
    return a;
  }
  auto sym = [&](const char* n) { return dlsym(h, n); };
  a.GetUniqueId = reinterpret_cast<result_t (*)(unique_id*)>(sym("ncclGetUniqueId"));
  a.CommInitRank = reinterpret_cast<result_t (*)(comm_t*, int, unique_id, int)>(sym("ncclCommInitRank"));
  a.CommDestroy = reinterpret_cast<result_t (*)(comm_t)>(sym("ncclCommDestroy"));
  a.AllGather = reinterpret_cast<result_t (*)(const void*, void*, size_t, int, comm_t, cudaStream_t)>(
      sym("ncclAllGather"));
  a.GetErrorString = reinterpret_cast<const char* (*)(result_t)>(sym("ncclGetErrorString"));
  a.MemAlloc = reinterpret_cast<result_t (*)(void**, size_t)>(sym("ncclMemAlloc"));
  a.MemFree = reinterpret_cast<result_t (*)(void*)>(sym("ncclMemFree"));
  a.CommWindowRegister = reinterpret_cast<result_t (*)(comm_t, void*, size_t, window_t*, int)>(
      sym("ncclCommWindowRegister"));
  a.CommWindowDeregister = reinterpret_cast<result_t (*)(comm_t, window_t)>(sym("ncclCommWindowDeregister"));
  a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllGather && a.GetErrorString;
  if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
  return a;
}
}  // namespace nccl

struct coot_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint32_t flags = 0;
  int sm_count = 0;
  int cc_major = 0, cc_minor = 0;
  int blocks_per_sm = 8;    // LDG fused driver / strided views: CTAs per SM in the grid
  int dim_blocks_per_sm = 4;  // LDG dim-sum kernels: CTAs per SM the work is split over
  int driver = 1;           // fused pass: 1 = TMA-staged (default), 0 = LDG
  int tma_ctas_per_sm = 2;  // TMA driver: CTAs per SM in the grid
  bool tma_ctas_env = false;  // COOT_TMA_CTAS given (tuning runs): keep it as is
  int tma_tile_units = 0;   // TMA driver: units per operand tile override (0 = policy)
  int tma_smem_kb = 0;      // TMA driver: stage-ring budget override in KB (0 = policy)
  int dim_ring_kb = 48;     // TMA dim kernels: stage-ring budget in KB (COOT_DIM_RING_KB)
  int dim_tma = 0;          // sum(X,dim): TMA-staged kernels when the layout allows
  int pdl = 1;              // programmatic dependent launch of fused / dim kernels
  int producer_sleep = -1;  // TMA producer sleeps on a full ring: -1 policy, 0 never, 1 always
  int smem_per_sm = 0, smem_reserved = 0;  // bytes (device attributes)
  coot::Rec* recs = nullptr;  // per-block records of the fused pass
  unsigned max_grid = 0;
  unsigned* ticket = nullptr;  // fused-pass arrival counter
  void* dim_part = nullptr;
  size_t dim_part_bytes = 0;
  unsigned* dim_tickets = nullptr;
  size_t dim_tickets_n = 0;
  coot_stats_t stats{};
  bool log = false;
  const coot::Exchange* pending_ex = nullptr;  // set by coot_reduce_exchange for one call
  uint64_t pending_vcap = 0;                   // coot_sum_dim_exchange: mailbox capacity
  cudaEvent_t handoff = nullptr;  // orders a new stream after the old one (coot_set_stream)
  // communicator (coot_comm_init): partial -> all-gather -> rank-order combine
  nccl::comm_t comm = nullptr;
  int nranks = 1, rank = 0;
  uint32_t shard = COOT_SHARD_NONE;
  void* comm_buf = nullptr;        // [send: S bytes][recv: nranks * S bytes]
  size_t comm_buf_bytes = 0;
  bool comm_buf_nccl = false;      // from ncclMemAlloc (else cudaMalloc)
  nccl::window_t comm_win = nullptr;  // symmetric window over comm_buf, if registered
};

// Whether the TMA producer should sleep (rather than poll) while the ring is
// full: for compute-heavy programs — EXP / LOG / SQRT / DIV, or run on the
// interpreter — where the consumers, not HBM, set the pace (coot_device.cuh
// mbar_wait).
static uint32_t producer_sleep(const coot_ctx* ctx, const coot_expr* e, int catalog) {
  if (ctx->producer_sleep >= 0) return (uint32_t)ctx->producer_sleep;
  if (catalog < 0) return 1;
  for (uint32_t i = 0; i < e->n_instr; ++i) {
    const unsigned op = e->prog[i].op;
    if (op == COOT_OP_EXP || op == COOT_OP_LOG || op == COOT_OP_SQRT || op == COOT_OP_DIV) return 1;
  }
  return 0;
}

// Dynamic shared memory of a persistent TMA-driver CTA, padded so that at most
// `per_sm` CTAs fit on one SM.  The grid is sized for per_sm CTAs per SM; a
// low-footprint kernel (few registers, a 64 KB ring) would otherwise fit a
// third CTA, and under programmatic dependent launch — where a kernel's CTAs
// are placed while the previous kernel still holds some SMs — the scheduler
// then stacks 3 CTAs on the SMs that freed first and 1 on the others:
// measured 10-20 % slower (var / index_min / norm2 at 2^30).
static unsigned pad_smem(const coot_ctx* ctx, unsigned smem, u64 per_sm) {
  if (ctx->smem_per_sm <= 0) return smem;
  const u64 floor = (u64)ctx->smem_per_sm / (per_sm + 1) + 1024 -
                    std::min<u64>((u64)ctx->smem_reserved, (u64)ctx->smem_per_sm / (per_sm + 1));
  const u64 cap = (u64)ctx->smem_per_sm / per_sm - (u64)ctx->smem_reserved;
  return (unsigned)std::max<u64>(smem, std::min<u64>(floor, std::min<u64>(cap, 200u << 10)));
}


namespace {

thread_local std::string g_err;

coot_status fail(coot_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

coot_status ok() { return COOT_OK; }

coot_status cuda_fail(cudaError_t e, const char* what) {
  return fail(COOT_ERR_DEVICE, "device: %s: %s (%s)", what, cudaGetErrorName(e),
              cudaGetErrorString(e));
}

const char* op_name(int op) {
  static const char* names[] = {"LOAD", "SCALAR", "NEG", "ABS", "SQUARE", "SQRT", "EXP",
                                "LOG",  "ADD",    "SUB", "MUL", "DIV",    "MIN",  "MAX"};
  return (op >= 0 && op < COOT_OP_COUNT_) ? names[op] : "?";
}

size_t elem_size(uint32_t elem) {
  switch (elem) {
    case COOT_F32: return 4;
    case COOT_F64: return 8;
    case COOT_U32: return 4;
    case COOT_S64: return 8;
    case COOT_BF16: return 2;
    case COOT_F16: return 2;
    case COOT_E4M3: return 1;
    case COOT_E5M2: return 1;
  }
  return 0;
}

// size of one reduction / dim-sum result element (f32 for the 8-bit types, R25)
size_t result_elem_size(uint32_t elem) {
  return (elem == COOT_E4M3 || elem == COOT_E5M2) ? 4 : elem_size(elem);
}

bool is_float_elem(uint32_t e) {
  return e == COOT_F32 || e == COOT_F64 || e == COOT_BF16 || e == COOT_F16 || e == COOT_E4M3 ||
         e == COOT_E5M2;
}
bool is_unary(int op) { return op >= COOT_OP_NEG && op <= COOT_OP_LOG; }
bool is_binary(int op) { return op >= COOT_OP_ADD && op <= COOT_OP_MAX; }

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  return atoi(v);
}

// ---- validation -------------------------------------------------------------
struct Shape {
  int max_depth = 0;
  uint32_t used_mask = 0;  // operands referenced by LOAD
};

coot_status validate_expr(const coot_expr* e, Shape* shape) {
  if (!e) return fail(COOT_ERR_CONTRACT, "contract: expression descriptor is NULL");
  if (e->abi_version != COOT_ABI_VERSION)
    return fail(COOT_ERR_CONFIG, "configuration: descriptor abi_version %u, library %u",
                e->abi_version, COOT_ABI_VERSION);
  if (elem_size(e->elem) == 0)
    return fail(COOT_ERR_CONTRACT, "contract: unknown element type %u", e->elem);
  if (e->reserved != 0) return fail(COOT_ERR_CONTRACT, "contract: reserved field must be 0");
  if (e->n_operands < 1 || e->n_operands > COOT_MAX_OPERANDS)
    return fail(COOT_ERR_BOUNDS, "bounds: %u operands (allowed 1..%d)", e->n_operands,
                COOT_MAX_OPERANDS);
  if (e->n_scalars > COOT_MAX_SCALARS)
    return fail(COOT_ERR_BOUNDS, "bounds: %u scalars (allowed 0..%d)", e->n_scalars,
                COOT_MAX_SCALARS);
  if (e->n_instr < 1 || e->n_instr > COOT_MAX_INSTR)
    return fail(COOT_ERR_BOUNDS, "bounds: %u instructions (allowed 1..%d)", e->n_instr,
                COOT_MAX_INSTR);
  const u64 n = e->n_rows * e->n_cols;
  if (e->n_cols != 0 && n / e->n_cols != e->n_rows)
    return fail(COOT_ERR_BOUNDS, "bounds: %llux%llu overflows 64-bit element count",
                (unsigned long long)e->n_rows, (unsigned long long)e->n_cols);
  const size_t es = elem_size(e->elem);
  for (uint32_t k = 0; k < e->n_operands; ++k) {
    const coot_operand& o = e->operands[k];
    // any (ld, inc) is a legal READ view; only written views must not overlap themselves
    if (n > 0 && o.ptr == nullptr)
      return fail(COOT_ERR_CONTRACT, "contract: operand %u is NULL with %llu elements", k,
                  (unsigned long long)n);
    if (reinterpret_cast<uintptr_t>(o.ptr) % es != 0)
      return fail(COOT_ERR_CONTRACT, "contract: operand %u is not aligned to its %zu-byte element",
                  k, es);
  }
  int sp = 0;
  Shape sh;
  for (uint32_t i = 0; i < e->n_instr; ++i) {
    const int op = e->prog[i].op, arg = e->prog[i].arg;
    if (op < 0 || op >= COOT_OP_COUNT_)
      return fail(COOT_ERR_CONTRACT, "contract: unknown opcode %d @ instr %u", op, i);
    if (!is_float_elem(e->elem) &&
        (op == COOT_OP_SQRT || op == COOT_OP_EXP || op == COOT_OP_LOG || op == COOT_OP_DIV))
      return fail(COOT_ERR_CONTRACT, "contract: %s is not defined for integer element types @ instr %u",
                  op_name(op), i);
    if (op == COOT_OP_LOAD) {
      if ((uint32_t)arg >= e->n_operands)
        return fail(COOT_ERR_CONTRACT, "contract: LOAD %d @ instr %u but only %u operands", arg, i,
                    e->n_operands);
      const coot_operand& o = e->operands[arg];
      if (o.n_rows != e->n_rows || o.n_cols != e->n_cols)
        return fail(COOT_ERR_CONFORM, "conformability: operand %d is %llux%llu, expression is %llux%llu (LOAD @ instr %u)",
                    arg, (unsigned long long)o.n_rows, (unsigned long long)o.n_cols,
                    (unsigned long long)e->n_rows, (unsigned long long)e->n_cols, i);
      sh.used_mask |= 1u << arg;
      ++sp;
    } else if (op == COOT_OP_SCALAR) {
      if ((uint32_t)arg >= e->n_scalars)
        return fail(COOT_ERR_CONTRACT, "contract: SCALAR %d @ instr %u but only %u scalars", arg, i,
                    e->n_scalars);
      ++sp;
    } else if (is_unary(op)) {
      if (arg != 0) return fail(COOT_ERR_CONTRACT, "contract: %s takes no argument @ instr %u", op_name(op), i);
      if (sp < 1) return fail(COOT_ERR_CONTRACT, "contract: stack underflow at %s @ instr %u", op_name(op), i);
    } else {
      if (arg != 0) return fail(COOT_ERR_CONTRACT, "contract: %s takes no argument @ instr %u", op_name(op), i);
      if (sp < 2) return fail(COOT_ERR_CONTRACT, "contract: stack underflow at %s @ instr %u", op_name(op), i);
      --sp;
    }
    if (sp > COOT_MAX_STACK)
      return fail(COOT_ERR_BOUNDS, "bounds: stack depth %d exceeds %d @ instr %u", sp, COOT_MAX_STACK, i);
    sh.max_depth = std::max(sh.max_depth, sp);
  }
  if (sp != 1)
    return fail(COOT_ERR_CONTRACT, "contract: program leaves %d values on the stack (expected 1)", sp);
  if (sh.used_mask == 0) return fail(COOT_ERR_CONTRACT, "contract: program reads no operand");
  // Unreferenced operands are allowed but their dims must still conform.
  for (uint32_t k = 0; k < e->n_operands; ++k) {
    const coot_operand& o = e->operands[k];
    if (o.n_rows != e->n_rows || o.n_cols != e->n_cols)
      return fail(COOT_ERR_CONFORM, "conformability: operand %u is %llux%llu, expression is %llux%llu",
                  k, (unsigned long long)o.n_rows, (unsigned long long)o.n_cols,
                  (unsigned long long)e->n_rows, (unsigned long long)e->n_cols);
  }
  if (shape) *shape = sh;
  return ok();
}

bool ranges_overlap(uintptr_t a, size_t na, uintptr_t b, size_t nb) {
  if (na == 0 || nb == 0) return false;
  return a < b + nb && b < a + na;
}

// ---- views (coot_operand.ld / .inc) ------------------------------------------
u64 op_ld(const coot_operand& o) { return o.ld ? o.ld : o.n_rows; }
u64 op_inc(const coot_operand& o) { return o.inc ? o.inc : 1; }
bool op_dense(const coot_operand& o) {
  return op_inc(o) == 1 && (o.n_cols <= 1 || op_ld(o) == o.n_rows);
}
// Bytes from the view's first element to one past its last element.
size_t op_span_bytes(const coot_operand& o, size_t es) {
  if (o.n_rows == 0 || o.n_cols == 0) return 0;
  return (size_t)(((o.n_rows - 1) * op_inc(o) + (o.n_cols - 1) * op_ld(o) + 1) * es);
}
bool same_view(const coot_operand& a, const coot_operand& b) {
  return a.ptr == b.ptr && a.n_rows == b.n_rows && a.n_cols == b.n_cols && op_ld(a) == op_ld(b) &&
         op_inc(a) == op_inc(b);
}
coot_operand dense_view(const void* p, u64 m, u64 n) {
  coot_operand o;
  o.ptr = p;
  o.n_rows = m;
  o.n_cols = n;
  o.ld = m;
  o.inc = 1;
  return o;
}

// out may be IDENTICAL to an operand view (B += 3*A; Z.diag() += 100,
// P:177); any other overlap of address spans is an error.  A written view
// must not overlap itself.
coot_status check_out_alias(const coot_expr* e, const coot_operand* out) {
  if (!out || !out->ptr) return ok();
  const size_t es = elem_size(e->elem);
  if (out->n_cols > 1 && op_ld(*out) < (out->n_rows ? (out->n_rows - 1) * op_inc(*out) + 1 : 0))
    return fail(COOT_ERR_CONTRACT, "contract: out view overlaps itself (ld %llu < (n_rows-1)*inc+1)",
                (unsigned long long)op_ld(*out));
  const uintptr_t o = reinterpret_cast<uintptr_t>(out->ptr);
  const size_t ob = op_span_bytes(*out, es);
  for (uint32_t k = 0; k < e->n_operands; ++k) {
    if (same_view(*out, e->operands[k])) continue;
    if (ranges_overlap(o, ob, reinterpret_cast<uintptr_t>(e->operands[k].ptr),
                       op_span_bytes(e->operands[k], es)))
      return fail(COOT_ERR_CONTRACT, "contract: out partially overlaps operand %u (only exact aliasing is allowed)", k);
  }
  return ok();
}

coot_status check_result_alias(const coot_expr* e, const void* result, size_t rbytes,
                               const coot_operand* out) {
  const size_t es = elem_size(e->elem);
  const uintptr_t r = reinterpret_cast<uintptr_t>(result);
  for (uint32_t k = 0; k < e->n_operands; ++k)
    if (ranges_overlap(r, rbytes, reinterpret_cast<uintptr_t>(e->operands[k].ptr),
                       op_span_bytes(e->operands[k], es)))
      return fail(COOT_ERR_CONTRACT, "contract: result overlaps operand %u", k);
  if (out && out->ptr &&
      ranges_overlap(r, rbytes, reinterpret_cast<uintptr_t>(out->ptr), op_span_bytes(*out, es)))
    return fail(COOT_ERR_CONTRACT, "contract: result overlaps out");
  return ok();
}

// ---- lowering ---------------------------------------------------------------
// Drop operands the program never LOADs and renumber the rest (order kept), so
// every staged / loaded array is one the expression reads.
coot_expr compact_expr(const coot_expr* e, Shape* sh) {
  coot_expr c = *e;
  int remap[COOT_MAX_OPERANDS];
  uint32_t n = 0;
  for (uint32_t k = 0; k < e->n_operands; ++k) {
    remap[k] = -1;
    if (sh->used_mask & (1u << k)) {
      remap[k] = (int)n;
      c.operands[n++] = e->operands[k];
    }
  }
  c.n_operands = n;
  for (uint32_t i = 0; i < e->n_instr; ++i)
    if (e->prog[i].op == COOT_OP_LOAD) c.prog[i].arg = (uint8_t)remap[e->prog[i].arg];
  sh->used_mask = (n >= 32) ? 0xffffffffu : ((1u << n) - 1u);
  return c;
}

struct CatalogEntry {
  int id;
  int n;
  int code[COOT_MAX_INSTR];
};

template <int... C>
constexpr int count_codes() {
  return (int)sizeof...(C);
}
#define COOT_X(id, ...) {id, count_codes<__VA_ARGS__>(), {__VA_ARGS__}},
const CatalogEntry kCatalog[] = {COOT_CATALOG(COOT_X)};
#undef COOT_X

int match_catalog(const coot_expr* e) {
  for (const CatalogEntry& c : kCatalog) {
    if ((uint32_t)c.n != e->n_instr) continue;
    bool same = true;
    for (int i = 0; i < c.n && same; ++i)
      same = c.code[i] == COOT_I(e->prog[i].op, e->prog[i].arg);
    if (same) return c.id;
  }
  return -1;
}

// Pack everything the evaluators need into the kernel arguments.  Returns the
// deepest stack the dispatched (fused-operand) program reaches.
int fill_program(const coot_expr* e, coot::FusedArgs* a) {
  for (uint32_t k = 0; k < COOT_MAX_OPERANDS; ++k)
    a->in[k] = k < e->n_operands ? e->operands[k].ptr : nullptr;
  for (uint32_t s = 0; s < COOT_MAX_SCALARS; ++s)
    a->scalars[s] = s < e->n_scalars ? e->scalars[s].bits : 0;
  a->n_operands = e->n_operands;
  a->n_instr = e->n_instr;
  a->m = e->n_rows;
  for (uint32_t k = 0; k < COOT_MAX_OPERANDS; ++k) {
    a->ld[k] = k < e->n_operands ? op_ld(e->operands[k]) : 0;
    a->inc[k] = k < e->n_operands ? op_inc(e->operands[k]) : 0;
  }
  // dense dispatch index (coot_fused.cuh) | argument << 16, with the fused-
  // operand peephole (COOT_XOP_L / COOT_XOP_S): a push directly followed by an
  // ADD / SUB / MUL that consumes it becomes one dispatch (the device has fused
  // cases for those three only: more cases cost the small interpreter spills).  The stack is never
  // deeper than in the original program.
  int sp = 0, max_sp = 0;
  uint32_t n = 0;
  const uint32_t ni = e->n_instr;
  auto emit = [&](int key, int arg) { a->code[n++] = (uint32_t)key | ((uint32_t)arg << 16); };
  // COOT_NO_FUSED_OPERANDS=1: plain one-dispatch-per-instruction code (A/B aid)
  static const bool force_plain = env_int("COOT_NO_FUSED_OPERANDS", 0) != 0;
  for (uint32_t i = 0; i < ni; ++i) {
    const int op = e->prog[i].op, arg = e->prog[i].arg;
    const int nx = i + 1 < ni ? e->prog[i + 1].op : -1;
    const int nx2 = i + 2 < ni ? e->prog[i + 2].op : -1;
    if (!force_plain && sp >= 1 && (op == COOT_OP_LOAD || op == COOT_OP_SCALAR) &&
        (nx == COOT_OP_ADD || nx == COOT_OP_SUB || nx == COOT_OP_MUL)) {
      emit(COOT_KEY(op == COOT_OP_LOAD ? COOT_XOP_L(nx) : COOT_XOP_S(nx), sp), arg);
      ++i;  // the push and its op: depth unchanged
      continue;
    }
    if (!force_plain && op == COOT_OP_SCALAR && nx == COOT_OP_LOAD &&
        (nx2 == COOT_OP_ADD || nx2 == COOT_OP_MUL)) {
      // s OP x == x OP s bit for bit for + and * (IEEE, packed 16-bit, modular)
      emit(COOT_KEY(COOT_OP_LOAD, sp), e->prog[i + 1].arg);
      emit(COOT_KEY(COOT_XOP_S(nx2), sp + 1), arg);
      i += 2;
      ++sp;
      max_sp = std::max(max_sp, sp);
      continue;
    }
    emit(COOT_KEY(op, sp), arg);
    if (op == COOT_OP_LOAD || op == COOT_OP_SCALAR) ++sp;
    else if (is_binary(op)) --sp;
    max_sp = std::max(max_sp, sp);
  }
  a->n_instr = n;
  return max_sp;
}

int acc_for_kind(uint32_t kind) {
  switch (kind) {
    case COOT_RED_ACCU: return coot::ACC_SUM;
    case COOT_RED_NORM2: return coot::ACC_SUMSQ;
    case COOT_RED_MIN:
    case COOT_RED_MAX:
    case COOT_RED_MINMAX: return coot::ACC_MINMAX;
    case COOT_RED_MEAN: return coot::ACC_SUM;
    case COOT_RED_VAR:
    case COOT_RED_STDDEV: return coot::ACC_VAR;
    case COOT_RED_INDEX_MIN: return coot::ACC_IMIN;
    case COOT_RED_INDEX_MAX: return coot::ACC_IMAX;
  }
  return -1;
}

bool float_only_kind(uint32_t kind) {
  return kind == COOT_RED_NORM2 || kind == COOT_RED_MEAN || kind == COOT_RED_VAR ||
         kind == COOT_RED_STDDEV;
}
bool nonempty_kind(uint32_t kind) {  // undefined over zero elements
  return kind == COOT_RED_MIN || kind == COOT_RED_MAX || kind == COOT_RED_MINMAX ||
         kind == COOT_RED_MEAN || kind == COOT_RED_VAR || kind == COOT_RED_STDDEV ||
         kind == COOT_RED_INDEX_MIN || kind == COOT_RED_INDEX_MAX;
}

size_t result_bytes(uint32_t kind, size_t es, u64 m, u64 n) {
  switch (kind) {
    case COOT_RED_INDEX_MIN:
    case COOT_RED_INDEX_MAX: return 8;
    case COOT_RED_MINMAX: return 2 * es;
    case COOT_RED_SUM_DIM0: return n * es;
    case COOT_RED_SUM_DIM1: return m * es;
  }
  return es;
}

cudaError_t dispatch_fused(uint32_t elem, const coot::FusedPlan& p, const coot::FusedArgs& a,
                           cudaStream_t s) {
  switch (elem) {
    case COOT_F32: return coot::launch_fused_t<float>(p, a, s);
    case COOT_F64: return coot::launch_fused_t<double>(p, a, s);
    case COOT_U32: return coot::launch_fused_t<uint32_t>(p, a, s);
    case COOT_S64: return coot::launch_fused_t<coot::s64>(p, a, s);
    case COOT_BF16: return coot::launch_fused_t<coot::bf16>(p, a, s);
    case COOT_F16: return coot::launch_fused_t<coot::f16>(p, a, s);
    case COOT_E4M3: return coot::launch_fused_t<coot::e4m3>(p, a, s);
    case COOT_E5M2: return coot::launch_fused_t<coot::e5m2>(p, a, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t dispatch_dim(uint32_t elem, const coot::DimPlan& p, const coot::DimArgs& a,
                         cudaStream_t s) {
  switch (elem) {
    case COOT_F32: return coot::launch_dim_t<float>(p, a, s);
    case COOT_F64: return coot::launch_dim_t<double>(p, a, s);
    case COOT_U32: return coot::launch_dim_t<uint32_t>(p, a, s);
    case COOT_S64: return coot::launch_dim_t<coot::s64>(p, a, s);
    case COOT_BF16: return coot::launch_dim_t<coot::bf16>(p, a, s);
    case COOT_F16: return coot::launch_dim_t<coot::f16>(p, a, s);
    case COOT_E4M3: return coot::launch_dim_t<coot::e4m3>(p, a, s);
    case COOT_E5M2: return coot::launch_dim_t<coot::e5m2>(p, a, s);
  }
  return cudaErrorInvalidValue;
}

coot_status bind_device(coot_ctx* ctx) {
  int cur = -1;
  cudaError_t e = cudaGetDevice(&cur);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (cur != ctx->device) {
    e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  }
  return ok();
}

coot_status grow_dim_scratch(coot_ctx* ctx, size_t part_bytes, size_t ntickets) {
  if (part_bytes <= ctx->dim_part_bytes && ntickets <= ctx->dim_tickets_n) return ok();
  cudaError_t e = cudaStreamSynchronize(ctx->stream);  // old buffers may be in use
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  if (part_bytes > ctx->dim_part_bytes) {
    cudaFree(ctx->dim_part);
    ctx->dim_part = nullptr;
    ctx->dim_part_bytes = 0;
    e = cudaMalloc(&ctx->dim_part, part_bytes);
    if (e != cudaSuccess)
      return fail(COOT_ERR_RESOURCE, "resource: cannot allocate %zu bytes of reduction scratch", part_bytes);
    ctx->dim_part_bytes = part_bytes;
  }
  if (ntickets > ctx->dim_tickets_n) {
    cudaFree(ctx->dim_tickets);
    ctx->dim_tickets = nullptr;
    ctx->dim_tickets_n = 0;
    e = cudaMalloc(&ctx->dim_tickets, ntickets * sizeof(unsigned));
    if (e != cudaSuccess)
      return fail(COOT_ERR_RESOURCE, "resource: cannot allocate %zu ticket counters", ntickets);
    e = cudaMemset(ctx->dim_tickets, 0, ntickets * sizeof(unsigned));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemset");
    ctx->dim_tickets_n = ntickets;
  }
  return ok();
}

u64 ceil_div(u64 a, u64 b) { return (a + b - 1) / b; }

u64 alg_bytes(const coot_expr* e, const Shape& sh, bool store) {
  const u64 n = e->n_rows * e->n_cols;
  const u64 k = (u64)__builtin_popcount(sh.used_mask) + (store ? 1 : 0);
  return n * elem_size(e->elem) * k;
}

bool any_strided(const coot_expr* e, const coot_operand* outv) {
  bool s = outv && outv->ptr && !op_dense(*outv);
  for (uint32_t k = 0; k < e->n_operands; ++k) s = s || !op_dense(e->operands[k]);
  return s;
}

// Views: the strided kernel (interpreter), element (i, j) addressed per operand.
coot_status run_strided(coot_ctx* ctx, const coot_expr* e, const Shape& sh, int acc,
                        uint32_t kind, void* result, uint32_t final_mode,
                        const coot_operand* outv) {
  const u64 n = e->n_rows * e->n_cols;
  coot::FusedArgs a;
  memset(&a, 0, sizeof a);
  fill_program(e, &a);
  a.n = n;
  a.out = outv ? const_cast<void*>(outv->ptr) : nullptr;
  a.out_ld = outv ? op_ld(*outv) : 0;
  a.out_inc = outv ? op_inc(*outv) : 0;
  a.partials = ctx->recs;
  a.ticket = ctx->ticket;
  a.result = result;
  a.count = n;
  a.final_mode = final_mode;
  a.kind = kind;
  if (final_mode == coot::FINAL_EXCHANGE) a.ex = *ctx->pending_ex;
  coot::FusedPlan p;
  p.pdl = ctx->pdl;
  p.driver = 2;
  p.smem = 0;
  p.catalog = -1;
  p.interp_large = (e->n_operands > 4 || sh.max_depth > 4) ? 1 : 0;
  p.acc = acc;
  p.grid = (unsigned)std::max<u64>(
      1, std::min<u64>(ceil_div(n, coot::kThreads), (u64)ctx->sm_count * ctx->blocks_per_sm));
  // Contiguous columns (inc == 1 everywhere) with one shared 16-byte column
  // misalignment: stream each column through the TMA ring (driver 3).
  const size_t es = elem_size(e->elem);
  const u64 m = e->n_rows;
  const uintptr_t mis = reinterpret_cast<uintptr_t>(e->operands[0].ptr) & 15;
  bool cols = ctx->driver == 1 && m >= 64;
  for (uint32_t k = 0; k < e->n_operands && cols; ++k) {
    const coot_operand& o = e->operands[k];
    cols = op_inc(o) == 1 && ((op_ld(o) * es) % 16 == 0 || e->n_cols == 1) &&
           (reinterpret_cast<uintptr_t>(o.ptr) & 15) == mis;
  }
  if (cols && a.out)
    cols = a.out_inc == 1 && ((a.out_ld * es) % 16 == 0 || e->n_cols == 1) &&
           (reinterpret_cast<uintptr_t>(a.out) & 15) == mis;
  if (cols) {
    const u64 G = (u64)ctx->sm_count * ctx->tma_ctas_per_sm;
    const u64 nk = e->n_operands;
    // ring geometry: the fused-pass policy (16 KB tiles for <= 3 operands, 64 KB ring)
    u64 tu = nk <= 3 ? 2 * coot::kTileUnits : coot::kTileUnits;
    if (ctx->tma_tile_units) tu = (u64)ctx->tma_tile_units;
    const u64 ring = (u64)(ctx->tma_smem_kb ? ctx->tma_smem_kb : 64) << 10;
    const u64 tile_el = tu * (16 / es);
    u64 S = std::max<u64>(1, ceil_div(8 * G, e->n_cols));
    S = std::min<u64>(S, std::max<u64>(1, m / tile_el));
    const u64 L = ceil_div(ceil_div(m, S), tile_el) * tile_el;
    S = ceil_div(m, L);
    const u64 stage_bytes = nk * tu * 16;
    const u64 stages = std::max<u64>(2, std::min<u64>(8, ring / stage_bytes));
    a.ncols = e->n_cols;
    a.seg_len = L;
    a.nseg = (uint32_t)S;
    a.tile_units = (uint32_t)tu;
    a.stages = (uint32_t)stages;
    p.driver = 3;
    // catalog programs take their own column-streaming instance (K1); others the
    // interpreter (same arithmetic either way, K1 == K2 bitwise)
    p.catalog = (ctx->flags & COOT_INIT_FORCE_INTERP) ? -1 : match_catalog(e);
    if (acc >= coot::ACC_VAR && p.catalog > 0) p.catalog = -1;  // see pick_fused_acc
    a.producer_sleep = producer_sleep(ctx, e, p.catalog);
    p.smem = pad_smem(ctx, (unsigned)(stages * stage_bytes + 16 * stages), ctx->tma_ctas_per_sm);
    p.grid = (unsigned)std::max<u64>(1, std::min<u64>(e->n_cols * S, G));
  }
  if (ctx->log)
    fprintf(stderr, "[coot] strided elem=%u %llux%llu acc=%d grid=%u\n", e->elem,
            (unsigned long long)e->n_rows, (unsigned long long)e->n_cols, acc, p.grid);
  cudaError_t ce = dispatch_fused(e->elem, p, a, ctx->stream);
  if (ce != cudaSuccess) return cuda_fail(ce, "strided kernel launch");
  ctx->stats.launches++;
  ctx->stats.last_path = -4;
  ctx->stats.last_grid = p.grid;
  ctx->stats.last_alg_bytes = alg_bytes(e, sh, a.out != nullptr);
  return ok();
}

// The fused pass (eval / full reductions).
coot_status run_fused(coot_ctx* ctx, const coot_expr* e, const Shape& sh, int acc, uint32_t kind,
                      void* result, uint32_t final_mode, const coot_operand* outv) {
  if (any_strided(e, outv)) return run_strided(ctx, e, sh, acc, kind, result, final_mode, outv);
  void* out = (outv && outv->ptr) ? const_cast<void*>(outv->ptr) : nullptr;
  const size_t es = elem_size(e->elem);
  const u64 n = e->n_rows * e->n_cols;
  const u64 W = 16 / es;
  coot::FusedArgs a;
  memset(&a, 0, sizeof a);
  const int fused_depth = fill_program(e, &a);
  a.out = out;
  a.n = n;
  // 16-byte unit path iff every accessed array has the same misalignment.
  const uintptr_t mis = reinterpret_cast<uintptr_t>(e->operands[0].ptr) & 15;
  bool vec_ok = true;
  for (uint32_t k = 0; k < e->n_operands; ++k)
    vec_ok = vec_ok && ((reinterpret_cast<uintptr_t>(e->operands[k].ptr) & 15) == mis);
  if (out) vec_ok = vec_ok && ((reinterpret_cast<uintptr_t>(out) & 15) == mis);
  if (vec_ok) {
    u64 head = mis ? (16 - mis) / es : 0;
    if (head > n) head = n;
    a.head = head;
    a.nunits = (n - head) / W;
    a.tail_begin = head + a.nunits * W;
  } else {
    a.head = n;
    a.nunits = 0;
    a.tail_begin = n;
  }
  const u64 scalar_work = std::max<u64>(a.head, n - a.tail_begin);
  coot::FusedPlan p;
  p.pdl = ctx->pdl;
  // the register-pipelined LDG alternative is built for the 4/8-byte types
  // only; 16- and 8-bit types always take the TMA driver
  p.driver = elem_size(e->elem) >= 4 ? ctx->driver : 1;
  p.smem = 0;
  p.catalog = (ctx->flags & COOT_INIT_FORCE_INTERP) ? -1 : match_catalog(e);
  if (acc >= coot::ACC_VAR && p.catalog > 0) p.catalog = -1;  // see pick_fused_acc
  p.interp_large = (e->n_operands > 4 || sh.max_depth > 4) ? 1 : 0;
  // shallow interpreter class (TMA driver): a 2-slot stack, 4 (4-byte types)
  // units per dispatch (coot_launch.cuh pick_fused_acc)
  // Every element size takes it except 16-/8-bit programs without EXP / LOG
  // (tools/sweep.py, interleaved: f64 c2 +18 %, s64 c4 +11 %, bf16 c2 +18 %,
  // E4M3 c2 +30 %, f16 axpy -4.5 %).
  static const bool no_shallow = env_int("COOT_NO_SHALLOW_INTERP", 0) != 0;  // A/B aid
  static const bool shallow_all = env_int("COOT_SHALLOW_ALL", 0) != 0;        // A/B aid
  bool transcendental = false;
  for (uint32_t i = 0; i < e->n_instr; ++i)
    transcendental = transcendental || e->prog[i].op == COOT_OP_EXP || e->prog[i].op == COOT_OP_LOG;
  const bool shallow_type = elem_size(e->elem) >= 4 || transcendental || shallow_all;
  if (p.catalog < 0 && !p.interp_large && p.driver == 1 && shallow_type && fused_depth <= 2 &&
      !no_shallow)
    p.interp_large = 2;
  u64 grid;
  if (p.driver == 1) {
    // TMA driver geometry: a function of (n, operands, SM count, evaluator
    // class) only.  Policy (tools/tma_tune.py sweeps): 16 KB
    // tiles per operand (1024 units) for <= 3 operands, else 8 KB; a 64 KB
    // stage ring (>= 2 stages) — more bytes in flight per CTA measured slower
    // for read-only streams, bigger bulk copies faster.  The small interpreter
    // on 4-byte types evaluates 4 units per dispatch, so its tiles hold >= 4 *
    // 256 units (coot::tma_units_per_dispatch).
    const u64 nk = e->n_operands;  // compacted: every operand is referenced
    const bool wide_dispatch = p.catalog < 0 && p.interp_large != 1 && elem_size(e->elem) == 4;
    u64 tu = (nk <= 3 || wide_dispatch) ? 2 * coot::kTileUnits : coot::kTileUnits;
    if (ctx->tma_tile_units)  // override, still >= what the evaluator's dispatch needs
      tu = std::max<u64>((u64)ctx->tma_tile_units,
                         wide_dispatch ? 2 * coot::kTileUnits : coot::kTileUnits);
    const u64 ring = (u64)(ctx->tma_smem_kb ? ctx->tma_smem_kb : 64) << 10;
    const u64 tile_bytes_all = nk * tu * 16;
    const u64 stages = std::max<u64>(2, std::min<u64>(8, ring / tile_bytes_all));
    a.tile_units = (uint32_t)tu;
    a.stages = (uint32_t)stages;
    a.producer_sleep = producer_sleep(ctx, e, p.catalog);
    p.smem = (unsigned)(stages * tile_bytes_all + 2 * stages * 8);
    const u64 ntiles = ceil_div(a.nunits, tu);
    grid = std::max<u64>(ntiles, ceil_div(scalar_work, coot::kConsumerWarps * 32));
    // a ring too big for two CTAs per SM (> ~113 KB) runs one persistent CTA per SM
    u64 per_sm = p.smem > (110u << 10) ? 1 : (u64)ctx->tma_ctas_per_sm;
    // fewer tiles than per_sm CTAs on every SM (small n, e.g. c1's 1e6): one CTA
    // per SM, so no SM streams for two CTAs while others host one, and the
    // finish merges fewer records (tools/small_n.py: n = 1e6 4.8 -> 4.4 us)
    if (grid < (u64)ctx->sm_count * per_sm && !ctx->tma_ctas_env) per_sm = 1;
    grid = std::max<u64>(1, std::min<u64>(grid, (u64)ctx->sm_count * per_sm));
    p.smem = pad_smem(ctx, p.smem, per_sm);
  } else {
    const u64 work = std::max<u64>(a.nunits, scalar_work);
    grid = std::max<u64>(1, ceil_div(work, coot::kThreads));
    grid = std::min<u64>(grid, (u64)ctx->sm_count * ctx->blocks_per_sm);
  }
  a.partials = ctx->recs;
  a.ticket = ctx->ticket;
  a.result = result;
  a.count = n;
  a.final_mode = final_mode;
  a.kind = kind;
  if (final_mode == coot::FINAL_EXCHANGE) a.ex = *ctx->pending_ex;

  p.acc = acc;
  p.grid = (unsigned)grid;
  if (ctx->log)
    fprintf(stderr, "[coot] fused elem=%u n=%llu path=%d%s acc=%d driver=%d grid=%u smem=%u stages=%u tile=%u head=%llu units=%llu\n",
            e->elem, (unsigned long long)n, p.catalog, p.catalog < 0 ? (p.interp_large == 1 ? "(interp8)" : p.interp_large == 2 ? "(interp2)" : "(interp4)") : "",
            acc, p.driver, p.grid, p.smem, a.stages, a.tile_units, (unsigned long long)a.head,
            (unsigned long long)a.nunits);
  cudaError_t ce = dispatch_fused(e->elem, p, a, ctx->stream);
  if (ce != cudaSuccess) return cuda_fail(ce, "fused kernel launch");
  ctx->stats.launches++;
  ctx->stats.last_path = p.catalog;
  ctx->stats.last_grid = p.grid;
  ctx->stats.last_alg_bytes = alg_bytes(e, sh, out != nullptr);
  return ok();
}

// sum(X, 0) / sum(X, 1).
coot_status run_dim(coot_ctx* ctx, const coot_expr* e, const Shape& sh, uint32_t kind,
                    void* result, uint32_t final_mode) {
  const size_t es = elem_size(e->elem);
  const u64 m = e->n_rows, n = e->n_cols;
  const u64 W = 16 / es;
  const size_t sbytes = 8;  // f64 / u64 partial words
  const u64 nout = kind == COOT_RED_SUM_DIM0 ? n : m;
  const size_t obytes = final_mode == coot::FINAL_PARTIAL ? sbytes : result_elem_size(e->elem);
  const bool xchg = final_mode == coot::FINAL_EXCHANGE;  // sum(X,1), vector mailboxes
  // a rank owning no columns still publishes a zero vector and combines: the
  // LDG dim-1 kernel runs with empty column loops
  if (m == 0 || (n == 0 && !xchg)) {
    if (nout) {
      cudaError_t ce = cudaMemsetAsync(result, 0, nout * obytes, ctx->stream);
      if (ce != cudaSuccess) return cuda_fail(ce, "cudaMemsetAsync");
    }
    return ok();
  }
  coot::DimArgs d;
  memset(&d, 0, sizeof d);
  fill_program(e, &d.f);
  d.m = m;
  d.n = n;
  d.result = result;
  d.final_mode = final_mode;
  const uintptr_t mis = reinterpret_cast<uintptr_t>(e->operands[0].ptr) & 15;
  bool same = true;
  for (uint32_t k = 0; k < e->n_operands; ++k)
    same = same && ((reinterpret_cast<uintptr_t>(e->operands[k].ptr) & 15) == mis);
  const bool col_aligned = ((m * es) % 16) == 0;
  const u64 target = (u64)ctx->sm_count * ctx->dim_blocks_per_sm;
  coot::DimPlan p;
  p.pdl = ctx->pdl;
  p.catalog = ((ctx->flags & COOT_INIT_FORCE_INTERP) == 0 && e->n_instr == 1) ? 0 : -1;
  p.interp_large = (e->n_operands > 4 || sh.max_depth > 4) ? 1 : 0;
  p.smem = 0;
  size_t part_bytes = 0, ntickets = 0;
  // TMA-staged dim kernels: opt-in (COOT_DIM_TMA=1), and by default for
  // sum(X,1) of 4-byte types, the one case they measured faster than the LDG
  // kernels (f32 dim 1: 6.36 vs 5.74 TB/s at 32768^2; f64 / 16- / 8-bit slower)
  const bool use_tma = ctx->driver == 1 && n > 0 &&
                       (ctx->dim_tma || (kind == COOT_RED_SUM_DIM1 && es == 4));
  const u64 G = (u64)ctx->sm_count * ctx->tma_ctas_per_sm;  // TMA grid: persistent CTAs
  const u64 nk = e->n_operands;
  const u64 R1 = (u64)coot::kConsumerWarps * 32 * W;         // dim1 TMA rows per tile
  if (any_strided(e, nullptr)) {
    // views: warp per column (dim 0) / thread per row (dim 1), interpreter
    p.kernel = coot::DIMK_STRIDED;
    p.catalog = -1;
    d.dim = kind == COOT_RED_SUM_DIM0 ? 0 : 1;
    const u64 work = d.dim == 0 ? n * 32 : m;
    p.grid = (unsigned)std::max<u64>(1, std::min<u64>(ceil_div(work, coot::kThreads), target));
  } else if (kind == COOT_RED_SUM_DIM0 && use_tma && same && col_aligned && m * es >= 4096) {
    // TMA dim 0: pieces = (column, segment), ~8 pieces per CTA, segments >= 1 tile
    p.kernel = coot::DIMK_DIM0_TMA;
    d.vec_ok = 1;
    const u64 tile_el = (u64)coot::kTileUnits * W;
    u64 S = std::max<u64>(1, ceil_div(8 * G, n));
    S = std::min<u64>(S, std::max<u64>(1, m / tile_el));
    u64 L = ceil_div(ceil_div(m, S), tile_el) * tile_el;
    S = ceil_div(m, L);
    d.seg_len = L;
    d.nseg = (uint32_t)S;
    const u64 stage_bytes = nk * coot::kTileUnits * 16;
    const u64 stages = std::max<u64>(2, std::min<u64>(16, ((u64)ctx->dim_ring_kb << 10) / stage_bytes));
    d.f.tile_units = coot::kTileUnits;
    d.f.stages = (uint32_t)stages;
    p.smem = pad_smem(ctx, (unsigned)(stages * stage_bytes + 16 * stages), ctx->tma_ctas_per_sm);
    p.grid = (unsigned)std::min<u64>(n * S, G);
    if (S > 1) {
      part_bytes = n * S * sbytes;
      ntickets = n;
    }
  } else if (kind == COOT_RED_SUM_DIM1 && use_tma && same && mis == 0 && col_aligned &&
             m >= R1 / 2) {
    // TMA dim 1: pieces = (row tile of R1 rows, column chunk), ~8 pieces per CTA
    p.kernel = coot::DIMK_DIM1_TMA;
    d.vec_ok = 1;
    const u64 cg = 4;
    const u64 nrt = ceil_div(m, R1);
    u64 nchunks = std::max<u64>(1, ceil_div(8 * G, nrt));
    nchunks = std::min<u64>(nchunks, std::max<u64>(1, n / (4 * cg)));
    const u64 ccols = ceil_div(n, nchunks);
    nchunks = ceil_div(n, ccols);
    d.cg = (uint32_t)cg;
    d.nrt = (uint32_t)nrt;
    d.ccols = ccols;
    d.nchunks = (uint32_t)nchunks;
    const u64 stage_bytes = nk * cg * R1 * es;
    const u64 stages = std::max<u64>(2, std::min<u64>(16, ((u64)ctx->dim_ring_kb << 10) / stage_bytes));
    d.f.stages = (uint32_t)stages;
    p.smem = pad_smem(ctx, (unsigned)(stages * stage_bytes + 16 * stages), ctx->tma_ctas_per_sm);
    p.grid = (unsigned)std::min<u64>(nrt * nchunks, G);
    if (nchunks > 1) {
      part_bytes = nchunks * m * sbytes;
      ntickets = nrt;
    }
  } else if (kind == COOT_RED_SUM_DIM0) {
    d.vec_ok = (same && col_aligned) ? 1 : 0;
    if (m >= 2048) {
      p.kernel = coot::DIMK_DIM0_BLOCK;
      u64 S = std::max<u64>(1, ceil_div(target, n));
      S = std::min<u64>(S, std::max<u64>(1, m / 2048));
      u64 L = ceil_div(m, S);
      L = ceil_div(L, 4 * W) * 4 * W;
      S = ceil_div(m, L);
      d.seg_len = L;
      d.nseg = (uint32_t)S;
      p.grid = (unsigned)std::min<u64>(n * S, target);
      if (S > 1) {
        part_bytes = n * S * sbytes;
        ntickets = n;
      }
    } else {
      p.kernel = coot::DIMK_DIM0_WARP;
      d.seg_len = m;
      d.nseg = 1;
      p.grid = (unsigned)std::min<u64>(ceil_div(n * 32, coot::kThreads), target);
    }
  } else {
    p.kernel = coot::DIMK_DIM1;
    d.vec_ok = (same && mis == 0 && col_aligned) ? 1 : 0;
    uint32_t tpr = 32;
    while (tpr < (uint32_t)coot::kThreads && (u64)tpr * W < m) tpr *= 2;
    const u64 Gc = coot::kThreads / tpr;  // column groups per CTA
    const u64 R = (u64)tpr * W;
    const u64 nrt = ceil_div(m, R);
    // one CTA per (row tile, chunk): keep the grid within one resident wave
    // (floor, not ceil) so no small tail wave is left over
    // 8-bit elements: dim1_kernel is built for 3 resident CTAs per SM (its 32 KB
    // of f64 row partials and __launch_bounds__(256, 3)), so one wave is 3 per SM
    const u64 tgt1 = es == 1 ? std::min<u64>(target, (u64)ctx->sm_count * 3) : target;
    u64 nchunks = std::max<u64>(1, tgt1 / nrt);
    nchunks = std::min<u64>(nchunks, std::max<u64>(1, n / (8 * Gc)));
    const u64 ccols = std::max<u64>(1, ceil_div(n, nchunks));
    nchunks = std::max<u64>(1, ceil_div(n, ccols));
    d.tpr = tpr;
    d.nrt = (uint32_t)nrt;
    d.ccols = ccols;
    d.nchunks = (uint32_t)nchunks;
    p.grid = (unsigned)(nrt * nchunks);
    if (nchunks > 1) {
      part_bytes = nchunks * m * sbytes;
      ntickets = nrt;
    }
  }
  if (xchg) {
    // one more ticket (index nrt) counts the rows this rank has published
    ntickets = std::max<size_t>(ntickets, (size_t)d.nrt + 1);
    d.f.ex = *ctx->pending_ex;
    d.vcap = ctx->pending_vcap;
  }
  coot_status st = grow_dim_scratch(ctx, part_bytes, ntickets);
  if (st != COOT_OK) return st;
  d.part = ctx->dim_part;
  d.tickets = ctx->dim_tickets;
  if (ctx->log)
    fprintf(stderr, "[coot] dim%d elem=%u %llux%llu kernel=%d grid=%u nseg=%u nchunks=%u tpr=%u vec=%u\n",
            kind == COOT_RED_SUM_DIM0 ? 0 : 1, e->elem, (unsigned long long)m, (unsigned long long)n,
            p.kernel, p.grid, d.nseg, d.nchunks, d.tpr, d.vec_ok);
  cudaError_t ce = dispatch_dim(e->elem, p, d, ctx->stream);
  if (ce != cudaSuccess) return cuda_fail(ce, "dim kernel launch");
  ctx->stats.launches++;
  ctx->stats.last_path = -2;
  ctx->stats.last_grid = p.grid;
  ctx->stats.last_alg_bytes = alg_bytes(e, sh, false) + nout * es;
  return ok();
}

coot_status check_ctx(const coot_ctx* ctx) {
  if (!ctx) return fail(COOT_ERR_CONFIG, "configuration: ctx is NULL");
  return ok();
}

coot_status reduce_common(coot_ctx* ctx, const coot_expr* e, uint32_t kind, void* result,
                          void* out, uint32_t final_mode) {
  coot_status st = check_ctx(ctx);
  if (st != COOT_OK) return st;
  Shape sh;
  st = validate_expr(e, &sh);
  if (st != COOT_OK) return st;
  if (kind >= COOT_RED_COUNT_) return fail(COOT_ERR_CONTRACT, "contract: unknown reduction kind %u", kind);
  if (!result) return fail(COOT_ERR_CONTRACT, "contract: result is NULL");
  const size_t es = elem_size(e->elem);
  const u64 n = e->n_rows * e->n_cols;
  if (float_only_kind(kind) && !is_float_elem(e->elem))
    return fail(COOT_ERR_CONTRACT, "contract: reduction kind %u is defined for f32/f64 only", kind);
  const bool dim = kind == COOT_RED_SUM_DIM0 || kind == COOT_RED_SUM_DIM1;
  if (dim && out)
    return fail(COOT_ERR_CONTRACT, "contract: out_or_null must be NULL for SUM_DIM reductions");
  if (final_mode == coot::FINAL_ROUND && n == 0 && nonempty_kind(kind))
    return fail(COOT_ERR_CONTRACT, "contract: reduction kind %u of an empty expression", kind);
  if (out && reinterpret_cast<uintptr_t>(out) % es)
    return fail(COOT_ERR_CONTRACT, "contract: out is not aligned to its element size");
  const coot_operand outv = dense_view(out, e->n_rows, e->n_cols);
  st = check_out_alias(e, out ? &outv : nullptr);
  if (st != COOT_OK) return st;
  size_t rbytes = result_bytes(kind, result_elem_size(e->elem), e->n_rows, e->n_cols);
  if (final_mode == coot::FINAL_PARTIAL)
    rbytes = dim ? (kind == COOT_RED_SUM_DIM0 ? e->n_cols : e->n_rows) * 8 : COOT_PARTIAL_BYTES;
  st = check_result_alias(e, result, rbytes, out ? &outv : nullptr);
  if (st != COOT_OK) return st;
  st = bind_device(ctx);
  if (st != COOT_OK) return st;
  const coot_expr cx = compact_expr(e, &sh);
  if (dim) return run_dim(ctx, &cx, sh, kind, result, final_mode);
  const int acc = acc_for_kind(kind);
  if (n == 0) {
    if (final_mode == coot::FINAL_PARTIAL || final_mode == coot::FINAL_EXCHANGE) {
      // an empty shard still publishes (or exchanges) the identity record
      const coot::Exchange* ex = final_mode == coot::FINAL_EXCHANGE ? ctx->pending_ex : nullptr;
      cudaStream_t s = ctx->stream;
      cudaError_t cerr;
      switch (e->elem) {
        case COOT_F32: cerr = coot::launch_empty_rec_t<float>(acc, result, s, ex, kind); break;
        case COOT_F64: cerr = coot::launch_empty_rec_t<double>(acc, result, s, ex, kind); break;
        case COOT_U32: cerr = coot::launch_empty_rec_t<uint32_t>(acc, result, s, ex, kind); break;
        case COOT_BF16: cerr = coot::launch_empty_rec_t<coot::bf16>(acc, result, s, ex, kind); break;
        case COOT_F16: cerr = coot::launch_empty_rec_t<coot::f16>(acc, result, s, ex, kind); break;
        case COOT_E4M3: cerr = coot::launch_empty_rec_t<coot::e4m3>(acc, result, s, ex, kind); break;
        case COOT_E5M2: cerr = coot::launch_empty_rec_t<coot::e5m2>(acc, result, s, ex, kind); break;
        default: cerr = coot::launch_empty_rec_t<coot::s64>(acc, result, s, ex, kind); break;
      }
      if (cerr != cudaSuccess) return cuda_fail(cerr, "empty record launch");
      ctx->stats.launches++;
      return ok();
    }
    cudaError_t cerr = cudaMemsetAsync(result, 0, result_elem_size(e->elem), ctx->stream);  // ACCU / NORM2 of empty = 0
    if (cerr != cudaSuccess) return cuda_fail(cerr, "cudaMemsetAsync");
    return ok();
  }
  return run_fused(ctx, &cx, sh, acc, kind, result, final_mode, out ? &outv : nullptr);
}

// Assignment of an expression into a (dense or view) destination: one launch.
coot_status eval_common(coot_ctx* ctx, const coot_expr* e, const coot_operand* outv) {
  coot_status st = check_ctx(ctx);
  if (st != COOT_OK) return st;
  Shape sh;
  st = validate_expr(e, &sh);
  if (st != COOT_OK) return st;
  const u64 n = e->n_rows * e->n_cols;
  if (n == 0) return ok();  // zero launches for an empty expression
  if (!outv || !outv->ptr) return fail(COOT_ERR_CONTRACT, "contract: out is NULL");
  if (outv->n_rows != e->n_rows || outv->n_cols != e->n_cols)
    return fail(COOT_ERR_CONFORM, "conformability: out is %llux%llu, expression is %llux%llu",
                (unsigned long long)outv->n_rows, (unsigned long long)outv->n_cols,
                (unsigned long long)e->n_rows, (unsigned long long)e->n_cols);
  if (reinterpret_cast<uintptr_t>(outv->ptr) % elem_size(e->elem))
    return fail(COOT_ERR_CONTRACT, "contract: out is not aligned to its element size");
  st = check_out_alias(e, outv);
  if (st != COOT_OK) return st;
  st = bind_device(ctx);
  if (st != COOT_OK) return st;
  const coot_expr cx = compact_expr(e, &sh);
  return run_fused(ctx, &cx, sh, coot::ACC_NONE, COOT_RED_ACCU, nullptr, coot::FINAL_ROUND, outv);
}

}  // namespace

// ============================================================================
extern "C" {

uint32_t coot_abi_version(void) { return COOT_ABI_VERSION; }

const char* coot_last_error(void) { return g_err.c_str(); }

const char* coot_status_string(coot_status s) {
  switch (s) {
    case COOT_OK: return "ok";
    case COOT_ERR_CONFIG: return "configuration";
    case COOT_ERR_CONFORM: return "conformability";
    case COOT_ERR_BOUNDS: return "bounds";
    case COOT_ERR_RESOURCE: return "resource";
    case COOT_ERR_CONTRACT: return "contract";
    case COOT_ERR_DEVICE: return "device";
  }
  return "unknown";
}

coot_status coot_validate(const coot_expr* e) { return validate_expr(e, nullptr); }

coot_status coot_init(coot_ctx** out, int device, void* cuda_stream, uint32_t flags) {
  if (!out) return fail(COOT_ERR_CONFIG, "configuration: out is NULL");
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(COOT_ERR_CONFIG, "configuration: no CUDA device (%s)", cudaGetErrorString(e));
  if (device < 0 || device >= ndev)
    return fail(COOT_ERR_CONFIG, "configuration: device %d out of range (0..%d)", device, ndev - 1);
  e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  coot_ctx* ctx = new coot_ctx();
  ctx->device = device;
  ctx->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  ctx->flags = flags;
  if (env_int("COOT_FORCE_INTERP", 0)) ctx->flags |= COOT_INIT_FORCE_INTERP;
  ctx->log = env_int("COOT_LOG", 0) != 0;
  cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&ctx->cc_major, cudaDevAttrComputeCapabilityMajor, device);
  cudaDeviceGetAttribute(&ctx->cc_minor, cudaDevAttrComputeCapabilityMinor, device);
  if (ctx->cc_major != 10) {
    int maj = ctx->cc_major, min = ctx->cc_minor;
    delete ctx;
    return fail(COOT_ERR_CONFIG, "configuration: device %d is sm_%d%d; libcoot is built for sm_100a (compute capability 10.x)",
                device, maj, min);
  }
  ctx->blocks_per_sm = std::max(1, std::min(32, env_int("COOT_BLOCKS_PER_SM", 8)));
  // dim sums: 4 per SM measured best (bf16 / E4M3 sum(X,1) +7 / +18 % over 8,
  // f64 c3 +2 %; tools/k2_probe.sh sweep)
  ctx->dim_blocks_per_sm = std::max(1, std::min(32, env_int("COOT_DIM_BLOCKS_PER_SM", 4)));
  ctx->driver = env_int("COOT_DRIVER", 1) ? 1 : 0;
  ctx->tma_ctas_per_sm = std::max(1, std::min(4, env_int("COOT_TMA_CTAS", 2)));
  ctx->tma_ctas_env = env_int("COOT_TMA_CTAS", 0) != 0;  // explicit: no small-n policy
  // TMA ring geometry overrides (tuning; 0 = the default policy of run_fused):
  // tile = a multiple of 512 units, ring budget in KB per CTA
  const int tile_env = env_int("COOT_TMA_TILE", 0), kb_env = env_int("COOT_TMA_SMEM_KB", 0);
  ctx->tma_tile_units = tile_env > 0 ? 512 * std::max(1, std::min(8, tile_env / 512)) : 0;
  ctx->tma_smem_kb = kb_env > 0 ? std::max(32, std::min(200, kb_env)) : 0;
  // dim sums default to the LDG kernels: measured faster on B200 (c3: dim0
  // 7.25 vs 7.04 TB/s, dim1 7.07 vs 6.74 TB/s)
  ctx->dim_tma = env_int("COOT_DIM_TMA", 0) ? 1 : 0;
  // TMA dim kernels' ring: 48 KB (3 stages of 4 columns x 1024 f32 rows) per CTA,
  // 2 CTAs per SM.  f32 sum(X,1) at 32768^2 (tools/gpu_r02o.sh, interleaved):
  // 32 KB 6.48, 48 KB 6.92, 64 KB 6.75, 80 KB 6.47, 96 KB 6.30 TB/s; 3-4 CTAs
  // per SM slower at every ring size
  ctx->dim_ring_kb = std::max(32, std::min(200, env_int("COOT_DIM_RING_KB", 48)));
  // back-to-back calls overlap each launch with the previous kernel's tail
  // (COOT_PDL=0: plain stream-ordered launches)
  ctx->pdl = env_int("COOT_PDL", 1) ? 1 : 0;
  ctx->producer_sleep = std::max(-1, std::min(1, env_int("COOT_PRODUCER_SLEEP", -1)));
  cudaDeviceGetAttribute(&ctx->smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
  cudaDeviceGetAttribute(&ctx->smem_reserved, cudaDevAttrReservedSharedMemoryPerBlock, device);
  ctx->max_grid = (unsigned)ctx->sm_count * 32u;
  e = cudaMalloc(&ctx->recs, sizeof(coot::Rec) * ctx->max_grid);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->ticket, 64 * sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMemset(ctx->ticket, 0, 64 * sizeof(unsigned));
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->handoff, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    cudaFree(ctx->recs);
    cudaFree(ctx->ticket);
    if (ctx->handoff) cudaEventDestroy(ctx->handoff);
    delete ctx;
    return fail(COOT_ERR_RESOURCE, "resource: cannot allocate reduction scratch (%s)", cudaGetErrorString(e));
  }
  ctx->stats.sm_count = ctx->sm_count;
  ctx->stats.last_path = -3;
  if (flags & COOT_INIT_PRINT_INFO) {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, device);
    fprintf(stderr, "[coot] device %d: %s, sm_%d%d, %d SMs, %.1f GB, L2 %d MB, libcoot ABI %u\n",
            device, prop.name, ctx->cc_major, ctx->cc_minor, ctx->sm_count,
            prop.totalGlobalMem / 1e9, prop.l2CacheSize >> 20, COOT_ABI_VERSION);
  }
  *out = ctx;
  return ok();
}

coot_status coot_destroy(coot_ctx* ctx) {
  if (!ctx) return ok();
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->comm) coot_comm_destroy(ctx);
  cudaFree(ctx->recs);
  cudaFree(ctx->ticket);
  cudaFree(ctx->dim_part);
  cudaFree(ctx->dim_tickets);
  if (ctx->handoff) cudaEventDestroy(ctx->handoff);
  delete ctx;
  return ok();
}

coot_status coot_set_stream(coot_ctx* ctx, void* cuda_stream) {
  coot_status st = check_ctx(ctx);
  if (st != COOT_OK) return st;
  const cudaStream_t next = reinterpret_cast<cudaStream_t>(cuda_stream);
  if (next != ctx->stream) {
    // the scratch (records, tickets, dim partials) is used stream-ordered: the
    // new stream waits (on the device, the host does not block) for everything
    // already enqueued on the old one
    st = bind_device(ctx);
    if (st != COOT_OK) return st;
    cudaError_t e = cudaEventRecord(ctx->handoff, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(next, ctx->handoff, 0);
    if (e != cudaSuccess) return cuda_fail(e, "stream hand-off");
    ctx->stream = next;
  }
  return ok();
}

coot_status coot_eval(coot_ctx* ctx, const coot_expr* e, void* out) {
  NvtxRange nvtx_("coot_eval");
  if (!e) return fail(COOT_ERR_CONTRACT, "contract: expression descriptor is NULL");
  const coot_operand outv = dense_view(out, e->n_rows, e->n_cols);
  return eval_common(ctx, e, &outv);
}

coot_status coot_eval_view(coot_ctx* ctx, const coot_expr* e, const coot_operand* out) {
  NvtxRange nvtx_("coot_eval_view");
  if (!out) return fail(COOT_ERR_CONTRACT, "contract: out view is NULL");
  return eval_common(ctx, e, out);
}

static coot_status reduce_comm(coot_ctx* ctx, const coot_expr* e, uint32_t kind, void* result,
                               void* out_or_null);

coot_status coot_reduce(coot_ctx* ctx, const coot_expr* e, uint32_t kind, void* result,
                        void* out_or_null) {
  NvtxRange nvtx_("coot_reduce");
  if (ctx && ctx->comm) return reduce_comm(ctx, e, kind, result, out_or_null);
  return reduce_common(ctx, e, kind, result, out_or_null, coot::FINAL_ROUND);
}

coot_status coot_reduce_partial(coot_ctx* ctx, const coot_expr* e, uint32_t kind, void* partial,
                                void* out_or_null) {
  NvtxRange nvtx_("coot_reduce_partial");
  return reduce_common(ctx, e, kind, partial, out_or_null, coot::FINAL_PARTIAL);
}

// ---- in-kernel exchange (mailboxes over CUDA IPC / NVLink peer memory) ------
// mailbox = COOT_MAX_RANKS records + COOT_MAX_RANKS u64 flags (zeroed once;
// flags only grow: each call raises them to its epoch).
static const size_t kMailboxBytes = 4096;

static coot_status mailbox_alloc(coot_ctx* ctx, size_t bytes, void** mailbox, void* ipc_handle) {
  coot_status st = check_ctx(ctx);
  if (st != COOT_OK) return st;
  if (!mailbox || !ipc_handle) return fail(COOT_ERR_CONTRACT, "contract: NULL argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == COOT_IPC_HANDLE_BYTES, "IPC handle size");
  st = bind_device(ctx);
  if (st != COOT_OK) return st;
  void* p = nullptr;
  cudaError_t ce = cudaMalloc(&p, bytes);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaMalloc(mailbox)");
  ce = cudaMemset(p, 0, bytes);
  if (ce == cudaSuccess) ce = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(ipc_handle), p);
  if (ce != cudaSuccess) {
    cudaFree(p);
    return cuda_fail(ce, "mailbox setup");
  }
  *mailbox = p;
  return ok();
}

coot_status coot_mailbox_create(coot_ctx* ctx, void** mailbox, void* ipc_handle) {
  return mailbox_alloc(ctx, kMailboxBytes, mailbox, ipc_handle);
}

// Vector mailbox (sum(X,1) over column shards): flags, tags, then
// 2 x COOT_MAX_RANKS slots of `capacity` 8-byte partial words (coot_dim.cuh).
coot_status coot_vec_mailbox_create(coot_ctx* ctx, uint64_t capacity, void** mailbox,
                                    void* ipc_handle) {
  if (capacity == 0 || capacity > (1ull << 32))
    return fail(COOT_ERR_BOUNDS, "bounds: vector mailbox capacity %llu (allowed 1..2^32)",
                (unsigned long long)capacity);
  return mailbox_alloc(ctx, (size_t)coot::kVecMboxHeader + 2ull * COOT_MAX_RANKS * capacity * 8,
                       mailbox, ipc_handle);
}

coot_status coot_mailbox_open(coot_ctx* ctx, const void* ipc_handle, void** peer_mailbox) {
  coot_status st = check_ctx(ctx);
  if (st != COOT_OK) return st;
  if (!peer_mailbox || !ipc_handle) return fail(COOT_ERR_CONTRACT, "contract: NULL argument");
  st = bind_device(ctx);
  if (st != COOT_OK) return st;
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof h);
  cudaError_t ce = cudaIpcOpenMemHandle(peer_mailbox, h, cudaIpcMemLazyEnablePeerAccess);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaIpcOpenMemHandle(mailbox)");
  return ok();
}

coot_status coot_mailbox_close(coot_ctx* ctx, void* peer_mailbox) {
  coot_status st = check_ctx(ctx);
  if (st != COOT_OK) return st;
  st = bind_device(ctx);
  if (st != COOT_OK) return st;
  cudaError_t ce = cudaIpcCloseMemHandle(peer_mailbox);
  return ce == cudaSuccess ? ok() : cuda_fail(ce, "cudaIpcCloseMemHandle");
}

coot_status coot_mailbox_destroy(coot_ctx* ctx, void* mailbox) {
  coot_status st = check_ctx(ctx);
  if (st != COOT_OK) return st;
  st = bind_device(ctx);
  if (st != COOT_OK) return st;
  cudaError_t ce = cudaFree(mailbox);
  return ce == cudaSuccess ? ok() : cuda_fail(ce, "cudaFree(mailbox)");
}

coot_status coot_reduce_exchange(coot_ctx* ctx, const coot_expr* e, uint32_t kind,
                                 void* const* mailboxes, uint32_t nranks, uint32_t rank,
                                 uint64_t epoch, void* result, void* out_or_null) {
  NvtxRange nvtx_("coot_reduce_exchange");
  coot_status st = check_ctx(ctx);
  if (st != COOT_OK) return st;
  if (kind == COOT_RED_SUM_DIM0 || kind == COOT_RED_SUM_DIM1)
    return fail(COOT_ERR_CONTRACT, "contract: the in-kernel exchange covers scalar reductions only");
  if (!mailboxes || nranks == 0 || nranks > COOT_MAX_RANKS || rank >= nranks)
    return fail(COOT_ERR_BOUNDS, "bounds: nranks %u / rank %u (max %d ranks)", nranks, rank,
                COOT_MAX_RANKS);
  if (epoch == 0) return fail(COOT_ERR_CONTRACT, "contract: epoch must be >= 1");
  coot::Exchange ex{};
  for (uint32_t p = 0; p < nranks; ++p) {
    if (!mailboxes[p]) return fail(COOT_ERR_CONTRACT, "contract: mailbox %u is NULL", p);
    ex.mbox[p] = reinterpret_cast<unsigned long long>(mailboxes[p]);
  }
  ex.epoch = epoch;
  ex.nranks = nranks;
  ex.rank = rank;
  ctx->pending_ex = &ex;
  st = reduce_common(ctx, e, kind, result, out_or_null, coot::FINAL_EXCHANGE);
  ctx->pending_ex = nullptr;
  return st;
}

coot_status coot_sum_dim_exchange(coot_ctx* ctx, const coot_expr* e, uint32_t kind,
                                  void* const* mailboxes, uint32_t nranks, uint32_t rank,
                                  uint64_t epoch, uint64_t capacity, void* result) {
  NvtxRange nvtx_("coot_sum_dim_exchange");
  coot_status st = check_ctx(ctx);
  if (st != COOT_OK) return st;
  if (kind != COOT_RED_SUM_DIM1)
    return fail(COOT_ERR_CONTRACT,
                "contract: the vector exchange covers sum(X,1) over column shards (SUM_DIM1) only");
  if (!e) return fail(COOT_ERR_CONTRACT, "contract: expression descriptor is NULL");
  if (!mailboxes || nranks == 0 || nranks > COOT_MAX_RANKS || rank >= nranks)
    return fail(COOT_ERR_BOUNDS, "bounds: nranks %u / rank %u (max %d ranks)", nranks, rank,
                COOT_MAX_RANKS);
  if (epoch == 0) return fail(COOT_ERR_CONTRACT, "contract: epoch must be >= 1");
  if (e->n_rows > capacity)
    return fail(COOT_ERR_BOUNDS, "bounds: %llu rows exceed the vector mailbox capacity %llu",
                (unsigned long long)e->n_rows, (unsigned long long)capacity);
  if (any_strided(e, nullptr))
    return fail(COOT_ERR_CONTRACT, "contract: the vector exchange takes dense operands only");
  coot::Exchange ex{};
  for (uint32_t p = 0; p < nranks; ++p) {
    if (!mailboxes[p]) return fail(COOT_ERR_CONTRACT, "contract: mailbox %u is NULL", p);
    ex.mbox[p] = reinterpret_cast<unsigned long long>(mailboxes[p]);
  }
  ex.epoch = epoch;
  ex.nranks = nranks;
  ex.rank = rank;
  ctx->pending_ex = &ex;
  ctx->pending_vcap = capacity;
  st = reduce_common(ctx, e, kind, result, nullptr, coot::FINAL_EXCHANGE);
  ctx->pending_ex = nullptr;
  ctx->pending_vcap = 0;
  return st;
}

coot_status coot_partial_bytes(uint32_t kind, uint64_t len, uint64_t* bytes) {
  if (!bytes) return fail(COOT_ERR_CONTRACT, "contract: bytes is NULL");
  if (kind >= COOT_RED_COUNT_) return fail(COOT_ERR_CONTRACT, "contract: unknown reduction kind %u", kind);
  *bytes = (kind == COOT_RED_SUM_DIM0 || kind == COOT_RED_SUM_DIM1) ? len * 8 : COOT_PARTIAL_BYTES;
  return ok();
}

coot_status coot_combine(coot_ctx* ctx, uint32_t elem, uint32_t kind, const void* partials,
                         uint32_t nparts, uint64_t len, void* result) {
  NvtxRange nvtx_("coot_combine");
  coot_status st = check_ctx(ctx);
  if (st != COOT_OK) return st;
  if (elem_size(elem) == 0) return fail(COOT_ERR_CONTRACT, "contract: unknown element type %u", elem);
  if (kind >= COOT_RED_COUNT_) return fail(COOT_ERR_CONTRACT, "contract: unknown reduction kind %u", kind);
  if (float_only_kind(kind) && !is_float_elem(elem))
    return fail(COOT_ERR_CONTRACT, "contract: reduction kind %u is defined for f32/f64 only", kind);
  if (nparts == 0) return fail(COOT_ERR_CONTRACT, "contract: combine of zero partials");
  if (!partials || !result) return fail(COOT_ERR_CONTRACT, "contract: NULL partials/result");
  const bool dim = kind == COOT_RED_SUM_DIM0 || kind == COOT_RED_SUM_DIM1;
  if (dim && len == 0) return ok();
  st = bind_device(ctx);
  if (st != COOT_OK) return st;
  const unsigned grid = (unsigned)std::max<u64>(
      1, std::min<u64>(ceil_div(dim ? len : 1, coot::kThreads), (u64)ctx->sm_count * 8));
  const int acc = dim ? coot::ACC_SUM : acc_for_kind(kind);
  cudaError_t ce;
  switch (elem) {
    case COOT_F32: ce = coot::launch_combine_t<float>(kind, acc, partials, nparts, len, result, grid, ctx->stream); break;
    case COOT_F64: ce = coot::launch_combine_t<double>(kind, acc, partials, nparts, len, result, grid, ctx->stream); break;
    case COOT_U32: ce = coot::launch_combine_t<uint32_t>(kind, acc, partials, nparts, len, result, grid, ctx->stream); break;
    case COOT_BF16: ce = coot::launch_combine_t<coot::bf16>(kind, acc, partials, nparts, len, result, grid, ctx->stream); break;
    case COOT_F16: ce = coot::launch_combine_t<coot::f16>(kind, acc, partials, nparts, len, result, grid, ctx->stream); break;
    case COOT_E4M3: ce = coot::launch_combine_t<coot::e4m3>(kind, acc, partials, nparts, len, result, grid, ctx->stream); break;
    case COOT_E5M2: ce = coot::launch_combine_t<coot::e5m2>(kind, acc, partials, nparts, len, result, grid, ctx->stream); break;
    default: ce = coot::launch_combine_t<coot::s64>(kind, acc, partials, nparts, len, result, grid, ctx->stream); break;
  }
  if (ce != cudaSuccess) return cuda_fail(ce, "combine kernel launch");
  ctx->stats.launches++;
  ctx->stats.last_path = -3;
  ctx->stats.last_grid = grid;
  return ok();
}

// ---- communicator -------------------------------------------------------------
static coot_status nccl_fail(nccl::result_t r, const char* what) {
  return fail(COOT_ERR_DEVICE, "device: %s: NCCL error %d (%s)", what, r,
              nccl::api().GetErrorString ? nccl::api().GetErrorString(r) : "?");
}

static void comm_free_buf(coot_ctx* ctx) {
  nccl::Api& a = nccl::api();
  if (ctx->comm_win && a.CommWindowDeregister) a.CommWindowDeregister(ctx->comm, ctx->comm_win);
  ctx->comm_win = nullptr;
  if (ctx->comm_buf) {
    if (ctx->comm_buf_nccl) a.MemFree(ctx->comm_buf);
    else cudaFree(ctx->comm_buf);
  }
  ctx->comm_buf = nullptr;
  ctx->comm_buf_bytes = 0;
}

// The exchange buffer (send + nranks receive slots of `slot` bytes each).
// Every rank grows it at the same call (the slot size is a function of the
// call's kind and global shape), so the collective window registration
// matches across ranks.
static coot_status comm_reserve(coot_ctx* ctx, size_t slot) {
  const size_t need = slot * (size_t)(ctx->nranks + 1);
  if (need <= ctx->comm_buf_bytes) return ok();
  cudaError_t ce = cudaStreamSynchronize(ctx->stream);  // the old buffer may be in flight
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamSynchronize");
  comm_free_buf(ctx);
  size_t bytes = 64u << 10;
  while (bytes < need) bytes *= 2;
  nccl::Api& a = nccl::api();
  if (a.MemAlloc && a.MemFree && a.MemAlloc(&ctx->comm_buf, bytes) == 0) {
    ctx->comm_buf_nccl = true;
  } else {
    ctx->comm_buf_nccl = false;
    ce = cudaMalloc(&ctx->comm_buf, bytes);
    if (ce != cudaSuccess) {
      ctx->comm_buf = nullptr;
      return fail(COOT_ERR_RESOURCE, "resource: cannot allocate %zu bytes of exchange buffer", bytes);
    }
  }
  ctx->comm_buf_bytes = bytes;
  // symmetric window: lets NCCL use its low-latency symmetric-memory kernels
  // for the all-gather of the partials (SURVEY §8(e) upgrade path 1)
  if (ctx->comm_buf_nccl && a.CommWindowRegister &&
      a.CommWindowRegister(ctx->comm, ctx->comm_buf, bytes, &ctx->comm_win,
                           nccl::kWinCollSymmetric) != 0)
    ctx->comm_win = nullptr;
  return ok();
}

// coot_reduce with a communicator: this rank's unrounded partial (the fused
// kernel, FINAL_PARTIAL), an all-gather of the partials, and the rank-order
// combine kernel — all on the ctx stream; every rank ends with the same bits.
// SUM_DIM along the unsharded dimension needs no exchange.
static coot_status reduce_comm(coot_ctx* ctx, const coot_expr* e, uint32_t kind, void* result,
                               void* out_or_null) {
  if (!e) return fail(COOT_ERR_CONTRACT, "contract: expression descriptor is NULL");
  const bool dim = kind == COOT_RED_SUM_DIM0 || kind == COOT_RED_SUM_DIM1;
  u64 len = 1;
  if (dim) {
    const bool exchange = (kind == COOT_RED_SUM_DIM1 && ctx->shard == COOT_SHARD_COLS) ||
                          (kind == COOT_RED_SUM_DIM0 && ctx->shard == COOT_SHARD_ROWS);
    if (!exchange) return reduce_common(ctx, e, kind, result, out_or_null, coot::FINAL_ROUND);
    len = kind == COOT_RED_SUM_DIM1 ? e->n_rows : e->n_cols;
  }
  const size_t slot = dim ? (size_t)len * 8 : (size_t)COOT_PARTIAL_BYTES;
  coot_status st = comm_reserve(ctx, slot);
  if (st != COOT_OK) return st;
  char* send = static_cast<char*>(ctx->comm_buf);
  char* recv = send + slot;
  st = reduce_common(ctx, e, kind, send, out_or_null, coot::FINAL_PARTIAL);
  if (st != COOT_OK) return st;
  const nccl::result_t r = nccl::api().AllGather(send, recv, slot, nccl::kUint8, ctx->comm, ctx->stream);
  if (r != 0) return nccl_fail(r, "ncclAllGather");
  return coot_combine(ctx, e->elem, kind, recv, (uint32_t)ctx->nranks, len, result);
}

coot_status coot_comm_unique_id(void* id) {
  if (!id) return fail(COOT_ERR_CONTRACT, "contract: id is NULL");
  nccl::Api& a = nccl::api();
  if (!a.ok) return fail(COOT_ERR_CONFIG, "configuration: NCCL unavailable (%s)", a.why.c_str());
  nccl::unique_id u;
  const nccl::result_t r = a.GetUniqueId(&u);
  if (r != 0) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(id, &u, sizeof u);
  return ok();
}

coot_status coot_comm_init(coot_ctx* ctx, uint32_t nranks, uint32_t rank, const void* id,
                           uint32_t shard) {
  coot_status st = check_ctx(ctx);
  if (st != COOT_OK) return st;
  if (!id) return fail(COOT_ERR_CONTRACT, "contract: id is NULL");
  if (nranks == 0 || rank >= nranks)
    return fail(COOT_ERR_CONFIG, "configuration: rank %u of %u", rank, nranks);
  if (shard > COOT_SHARD_ROWS) return fail(COOT_ERR_CONTRACT, "contract: unknown shard kind %u", shard);
  if (ctx->comm) return fail(COOT_ERR_CONFIG, "configuration: ctx already has a communicator");
  nccl::Api& a = nccl::api();
  if (!a.ok) return fail(COOT_ERR_CONFIG, "configuration: NCCL unavailable (%s)", a.why.c_str());
  st = bind_device(ctx);
  if (st != COOT_OK) return st;
  nccl::unique_id u;
  memcpy(&u, id, sizeof u);
  nccl::comm_t c = nullptr;
  const nccl::result_t r = a.CommInitRank(&c, (int)nranks, u, (int)rank);
  if (r != 0) return nccl_fail(r, "ncclCommInitRank");
  ctx->comm = c;
  ctx->nranks = (int)nranks;
  ctx->rank = (int)rank;
  ctx->shard = shard;
  st = comm_reserve(ctx, COOT_PARTIAL_BYTES);
  if (st != COOT_OK) {
    a.CommDestroy(c);
    ctx->comm = nullptr;
    ctx->nranks = 1;
    ctx->rank = 0;
  }
  return st;
}

coot_status coot_comm_destroy(coot_ctx* ctx) {
  coot_status st = check_ctx(ctx);
  if (st != COOT_OK) return st;
  if (!ctx->comm) return ok();
  st = bind_device(ctx);
  if (st != COOT_OK) return st;
  cudaStreamSynchronize(ctx->stream);
  comm_free_buf(ctx);
  nccl::api().CommDestroy(ctx->comm);
  ctx->comm = nullptr;
  ctx->nranks = 1;
  ctx->rank = 0;
  ctx->shard = COOT_SHARD_NONE;
  return ok();
}

coot_status coot_shard_range(uint64_t n, uint32_t rank, uint32_t nranks, uint64_t align,
                             uint64_t* begin, uint64_t* end) {
  if (!begin || !end) return fail(COOT_ERR_CONTRACT, "contract: NULL begin/end");
  if (nranks == 0 || rank >= nranks)
    return fail(COOT_ERR_CONFIG, "configuration: rank %u of %u", rank, nranks);
  if (align == 0) align = 1;
  auto cut = [&](uint64_t r) -> uint64_t {
    if (r == 0) return 0;
    if (r >= nranks) return n;
    const unsigned __int128 c = (unsigned __int128)r * n / nranks;
    return (uint64_t)c / align * align;
  };
  *begin = cut(rank);
  *end = cut(rank + 1);
  return ok();
}

coot_status coot_fill(coot_ctx* ctx, uint32_t elem, uint32_t fill_kind, uint64_t seed,
                      uint64_t stream, uint64_t start, uint64_t count, uint64_t n_rows,
                      uint64_t k, void* out) {
  NvtxRange nvtx_("coot_fill");
  coot_status st = check_ctx(ctx);
  if (st != COOT_OK) return st;
  if (elem_size(elem) == 0) return fail(COOT_ERR_CONTRACT, "contract: unknown element type %u", elem);
  if (fill_kind > 6) return fail(COOT_ERR_CONTRACT, "contract: unknown fill kind %u", fill_kind);
  if (count == 0) return ok();
  if (!out) return fail(COOT_ERR_CONTRACT, "contract: out is NULL");
  st = bind_device(ctx);
  if (st != COOT_OK) return st;
  const unsigned grid = (unsigned)std::min<u64>(ceil_div(count, coot::kThreads), (u64)ctx->sm_count * 8);
  cudaError_t ce;
  switch (elem) {
    case COOT_F32: ce = coot::launch_fill_t<float>(fill_kind, seed, stream, start, count, n_rows, k, out, grid, ctx->stream); break;
    case COOT_F64: ce = coot::launch_fill_t<double>(fill_kind, seed, stream, start, count, n_rows, k, out, grid, ctx->stream); break;
    case COOT_U32: ce = coot::launch_fill_t<uint32_t>(fill_kind, seed, stream, start, count, n_rows, k, out, grid, ctx->stream); break;
    case COOT_BF16: ce = coot::launch_fill_t<coot::bf16>(fill_kind, seed, stream, start, count, n_rows, k, out, grid, ctx->stream); break;
    case COOT_F16: ce = coot::launch_fill_t<coot::f16>(fill_kind, seed, stream, start, count, n_rows, k, out, grid, ctx->stream); break;
    case COOT_E4M3: ce = coot::launch_fill_t<coot::e4m3>(fill_kind, seed, stream, start, count, n_rows, k, out, grid, ctx->stream); break;
    case COOT_E5M2: ce = coot::launch_fill_t<coot::e5m2>(fill_kind, seed, stream, start, count, n_rows, k, out, grid, ctx->stream); break;
    default: ce = coot::launch_fill_t<coot::s64>(fill_kind, seed, stream, start, count, n_rows, k, out, grid, ctx->stream); break;
  }
  if (ce != cudaSuccess) return cuda_fail(ce, "fill kernel launch");
  ctx->stats.launches++;
  ctx->stats.last_path = -3;
  ctx->stats.last_grid = grid;
  return ok();
}

coot_status coot_stream_mix(coot_ctx* ctx, uint32_t n_read, uint32_t n_write, uint64_t n,
                            const void* const* in, void* out, void* sink) {
  NvtxRange nvtx_("coot_stream_mix");
  coot_status st = check_ctx(ctx);
  if (st != COOT_OK) return st;
  if (n_read > 3 || n_write > 1 || n_read + n_write == 0)
    return fail(COOT_ERR_BOUNDS, "bounds: stream mix %uR%uW (allowed 0..3 reads, 0..1 writes)",
                n_read, n_write);
  if (n % 4) return fail(COOT_ERR_CONTRACT, "contract: stream mix length %llu is not a multiple of 4",
                         (unsigned long long)n);
  if (n == 0) return ok();
  for (uint32_t k = 0; k < n_read; ++k)
    if (!in || !in[k] || reinterpret_cast<uintptr_t>(in[k]) % 16)
      return fail(COOT_ERR_CONTRACT, "contract: stream input %u is NULL or not 16-byte aligned", k);
  if (n_write && (!out || reinterpret_cast<uintptr_t>(out) % 16))
    return fail(COOT_ERR_CONTRACT, "contract: stream output is NULL or not 16-byte aligned");
  if (!n_write && !sink) return fail(COOT_ERR_CONTRACT, "contract: a read-only mix needs a sink");
  st = bind_device(ctx);
  if (st != COOT_OK) return st;
  cudaError_t ce = coot::launch_stream_mix(n_read, n_write, n / 4, in, out, sink, ctx->sm_count,
                                           ctx->stream);
  if (ce != cudaSuccess) return cuda_fail(ce, "stream kernel launch");
  ctx->stats.launches++;
  ctx->stats.last_path = -3;
  ctx->stats.last_alg_bytes = n * 4 * (n_read + n_write);
  return ok();
}

coot_status coot_sync(coot_ctx* ctx) {
  NvtxRange nvtx_("coot_sync");
  coot_status st = check_ctx(ctx);
  if (st != COOT_OK) return st;
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "asynchronous fault");
  return ok();
}

coot_status coot_stats(const coot_ctx* ctx, coot_stats_t* out) {
  coot_status st = check_ctx(ctx);
  if (st != COOT_OK) return st;
  if (!out) return fail(COOT_ERR_CONTRACT, "contract: out is NULL");
  *out = ctx->stats;
  return ok();
}

}  // extern "C"
