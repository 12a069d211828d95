// Catalog of common expression shapes compiled as templated kernels (K1).
// The lowering (runtime.cpp) matches a descriptor's program against these
// instruction lists (operand indices and opcodes; scalar VALUES and pointers
// are runtime arguments).  Anything else runs on the interpreter (K2).
// Paper: "compile-time pattern matching ... to choose the minimal set of
// calls"; the axpy fusion.
#pragma once
#include "../../include/coot.h"

#define COOT_I(op, arg) (((op) << 4) | (arg))
#define CL(k) COOT_I(COOT_OP_LOAD, k)
#define CS(k) COOT_I(COOT_OP_SCALAR, k)
#define CO(op) COOT_I(COOT_OP_##op, 0)

// X(id, instr...) — ids are stable (coot_stats.last_path reports them).
#define COOT_CATALOG(X)                                                        \
  X(0, CL(0))                                        /* plain reduction    */ \
  X(1, CS(0), CL(0), CO(MUL), CL(1), CO(ADD))        /* axpy a*x + y (c1)  */ \
  X(2, CL(0), CL(1), CO(MUL), CO(EXP), CS(0), CL(2), CO(MUL), CO(ADD)) /* c2 */ \
  X(3, CL(0), CL(1), CO(MUL), CS(0), CL(2), CO(MUL), CO(ADD)) /* c4        */ \
  X(4, CL(0), CL(1), CO(MUL))                        /* x % y, dot         */ \
  X(5, CL(0), CL(1), CO(ADD))                                                 \
  X(6, CL(0), CL(1), CO(SUB))                                                 \
  X(7, CS(0), CL(0), CO(MUL))                        /* scalar * X         */ \
  X(8, CL(0), CS(0), CO(ADD))                        /* X + scalar         */ \
  X(9, CL(0), CL(1), CO(DIV))

#define COOT_CATALOG_SIZE 10
