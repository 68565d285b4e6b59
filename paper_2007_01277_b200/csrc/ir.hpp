// hfuse IR: a uniform tagged tree for Mini-Kernel (MK) and its B200 dialect (MK+).
//
// The reference models the same language with std::variant node types
// (/root/reference/proj/include/mkfuse/ast.hpp:80-177). Here every expression and
// statement is one value-semantic node with a kind tag and child vectors, so passes
// walk the tree generically and dialect extensions (vector loads/stores, unsigned
// helpers, unroll hints) are new tags rather than new types.
#pragma once

#include <cstdint>
#include <exception>
#include <functional>
#include <optional>
#include <string>
#include <vector>

namespace hf {

struct Pos {
  int line = 0, col = 0;
  bool valid() const { return line > 0; }
};

// Ordinals are part of the C ABI (hf_error.code) and follow the reference's
// ErrCode order (error.hpp:15-39) so callers can switch on them unchanged.
enum class Code : int {
  Ok = -1,
  Syntax = 0, UnknownIdentifier, TypeMismatch, DuplicateName, UnresolvedCall, UnresolvedLabel,
  Recursion, BadBarrierId, MisalignedCount, DimensionMismatch, GridMismatch,
  ThreadBudgetExceeded, SharedMemoryOverflow, DoesNotFit, OutOfBounds, DivideByZero,
  BarrierDeadlock, BarrierOverflow, DivergentBarrier, NothingFeasible, IncompatibleFixedDims,
  InvalidArgument, Io,
  // hfuse-only codes (appended; never produced on reference-compatible paths)
  Compile, Device,
};
const char* code_name(Code c);

class Error : public std::exception {
 public:
  Error(Code c, std::string msg, Pos p = {});
  Code code;
  std::string msg;
  Pos pos;
  const char* what() const noexcept override { return text_.c_str(); }

 private:
  std::string text_;  // "[Code] line:col: msg"
};
[[noreturn]] void raise(Code c, std::string msg, Pos p = {});

enum class Ty : uint8_t { Int, Float };
inline const char* ty_name(Ty t) { return t == Ty::Int ? "int" : "float"; }

enum class Bin : uint8_t {
  Add, Sub, Mul, Div, Mod, Shl, Shr, And, Xor, Or, Lt, Le, Gt, Ge, Eq, Ne, LAnd, LOr,
};
enum class Un : uint8_t { Neg, Not };
enum class Builtin : uint8_t { TidX, TidY, TidZ, BidX, BidY, BidZ, BdimX, BdimY, BdimZ, GdimX };
// Min/Max/Fmaxf/CastInt/CastFloat are the reference's intrinsics (ast.hpp:67); the rest
// are MK+ (B200 dialect) helpers, each defined by an exact plain-MK expansion
// (downlower.cpp) so the reference interpreter can execute the dialect.
enum class Intr : uint8_t {
  Min, Max, Fmaxf, CastInt, CastFloat,
  ShrU,   // logical right shift
  Rotr,   // 32-bit rotate right
  Rotl,   // 32-bit rotate left
  LtU,    // unsigned less-than (0/1)
  Fshr,   // fshr(lo, hi, n): low word of (hi:lo) >> (n & 31)   (64-bit rotates in 32-bit halves)
  Fshl,   // fshl(lo, hi, n): high word of (hi:lo) << (n & 31)
  IntRz,  // int_rz(x): int(x) for |x| < 2^31 (device: one cvt.rzi.s32); outside that range undefined
  Acquire,  // load_acquire(a[i]): a[i] read with gpu-scope acquire (pairs with atomic_add_release)
  Relaxed,  // load_relaxed(a[i]): gpu-scope strong read, no ordering (a later fence() acquires)
  Bcast,    // x = warp_bcast(v, src, w): v of lane (lane & ~(w-1)) + src; w a constant power of two
            // in [2, 32], src uniform within each w-lane group; only as a whole assignment value
  Addc,     // addc(ahi, bhi, alo, blo): ahi + bhi + carry-out of alo + blo (64-bit add, high word;
            // device: add.cc + addc, i.e. IADD3 + IADD3.X instead of an unsigned compare)
  RemU,     // remu(a, b): a mod b with a read as uint32, for 0 < b < 2^30 (Ethash's page walk);
            // device: one unsigned remainder; plain MK: ((shr_u(a, 1) % b) * 2 + (a & 1)) % b
  MulHiU,   // mulhi_u(a, b): high word of the unsigned 64-bit product a * b (device: IMAD.HI.U32 on
            // the FMA pipe, e.g. x >> n as mulhi_u(x, 2^(32-n)) with the power in a register);
            // plain MK: the 16-bit-limb schoolbook product
  FmaAdd,   // fma_add(a, b): a + b (wrapping) issued on the FMA pipe (device: IMAD a, one, b with
            // `one` a __constant__ the compiler cannot fold), so ALU-pipe-bound hash rounds can
            // move adds off the saturated ALU pipe; plain MK: a + b
};
const char* intr_name(Intr i);
int intr_arity(Intr i);
bool intr_is_extension(Intr i);

enum class EK : uint8_t { Int, Float, Var, Builtin, Unary, Binary, Index, Intrin, Shfl, Call };

struct Expr {
  EK k = EK::Int;
  Pos pos;
  int32_t i = 0;      // Int literal / Builtin id / Unary op / Binary op / Intr id / Shfl mask
  float f = 0.0f;     // Float literal
  std::string s;      // Var name / Index array / Call callee
  std::vector<Expr> a;  // children (Unary 1, Binary 2, Index 1, Intrin n, Shfl 1, Call n)
};

enum class SK : uint8_t {
  Decl, Assign, If, For, While, Sync, BarSync, Atomic, Return, Call, Label, Goto,
  VLoad,   // MK+: vload(arr, i, d0..dn-1): d_k = arr[i*n + k], index evaluated once
  VStore,  // MK+: vstore(arr, i, e0..en-1): arr[i*n + k] = e_k
  Fence,   // MK+: fence(): device-scope memory fence (a no-op for the sequential interpreter)
  WarpSync,  // MK+: warp_sync(): __syncwarp() (a no-op for the lock-step interpreter)
  // MK+: async_copy(sarr, j, garr, i): the 4 elements garr[4i..4i+3] -> shared sarr[4j..4j+3]
  // as one 16-byte asynchronous copy (sm_100a cp.async: no register holds the data in flight).
  // name = garr, idx[0] = i, outs[0] = sarr, val[0] = j. The issuing thread may read the copied
  // elements only after its next async_wait(); the interpreter lowering copies immediately.
  AsyncCopy,
  AsyncWait,  // MK+: async_wait(): this thread's async copies have landed (cp.async.wait_all)
};

struct Stmt {
  SK k = SK::Sync;
  Pos pos;
  Ty ty = Ty::Int;                // Decl type
  std::string name;               // Decl var, Assign/Atomic/VLoad/VStore target, Label, Goto, Call
  Pos name_pos;                   // position of the target identifier (lvalues)
  std::vector<Expr> idx;          // Assign/Atomic element index (0/1 entries); VLoad/VStore vector index
  std::vector<Expr> val;          // Decl init (0/1), Assign/Atomic value, cond, Return value, args, VStore values
  std::vector<std::string> outs;  // VLoad destinations
  std::vector<Stmt> body, alt;    // If then/else; loop body
  std::vector<Stmt> init, step;   // For header (one statement each)
  bool has_alt = false;
  int bid = 0, bcount = 0;        // BarSync; Atomic: bid 1 = atomic_add_release (MK+); VStore: bid 1 = vstore_cs
  int unroll = 0;                 // For (MK+): 0 = no hint, -1 = `unroll`, N = `unroll N`
};
using Block = std::vector<Stmt>;

struct Param {
  std::string name;
  Ty ty = Ty::Int;
  bool array = false;
  Pos pos;
};

struct SharedArr {
  std::string name;
  Ty ty = Ty::Int;
  int64_t len = 0;
  Pos pos;
};

struct Dims {
  int x = 1, y = 1, z = 1;
  int64_t count() const { return int64_t(x) * y * z; }
  bool operator==(const Dims&) const = default;
};

struct Kernel {
  std::string name;
  std::vector<Param> params;
  Dims dims;
  bool tunable = true;
  std::vector<SharedArr> shared;
  Block body;
  int grid = 1;                 // //@ grid=
  std::optional<int> regs;      // //@ regs=
  std::optional<int> regcap;    // //@ regcap=
  // MK+ `//@ requires EXPR`: launch preconditions over scalar int parameters (e.g. a vector
  // width dividing a row length). Checked by the runtime when a launch binds its scalars;
  // dropped by the lowering to plain Mini-Kernel (the reference has no such annotation).
  std::vector<Expr> reqs;
  Pos pos;
};

// Host evaluation of an int expression over named scalars with the interpreter's pinned
// integer semantics (exec.cpp:26-48); nullopt when it names an unknown scalar, divides by zero
// or uses a construct outside scalar int arithmetic.
std::optional<int32_t> eval_scalar_int(const Expr& e,
                                       const std::function<std::optional<int32_t>(const std::string&)>& value);

struct Func {
  std::string name;
  std::optional<Ty> ret;
  std::vector<Param> params;
  Block body;
  Pos pos;
};

struct Program {
  std::vector<Func> funcs;
  std::vector<Kernel> kernels;
  const Func* func(const std::string& n) const;
  const Kernel* kernel(const std::string& n) const;
};

// ---- builders ---------------------------------------------------------------
Expr lit(int32_t v);
Expr flit(float v);
Expr var(std::string n);
Expr builtin(Builtin b);
Expr unary(Un op, Expr x);
Expr binary(Bin op, Expr l, Expr r);
Expr index(std::string arr, Expr i);
Expr intrin(Intr w, std::vector<Expr> args);
Stmt decl(Ty t, std::string n);
Stmt decl_init(Ty t, std::string n, Expr init);
Stmt assign(std::string n, Expr v);
Stmt assign_at(std::string arr, Expr i, Expr v);
Stmt if_(Expr c, Block then_b);
Stmt if_else(Expr c, Block then_b, Block else_b);

// ---- walkers (pre-order) ----------------------------------------------------
// Statements including everything nested in if/else, loop headers and bodies.
void walk(const Block& b, const std::function<void(const Stmt&)>& fn);
void walk(Block& b, const std::function<void(Stmt&)>& fn);
// Direct expressions of one statement (not nested statements).
void exprs_of(const Stmt& s, const std::function<void(const Expr&)>& fn);
void exprs_of(Stmt& s, const std::function<void(Expr&)>& fn);
void walk_expr(const Expr& e, const std::function<void(const Expr&)>& fn);
void walk_expr(Expr& e, const std::function<void(Expr&)>& fn);

bool same(const Expr& a, const Expr& b);
bool same(const Block& a, const Block& b);
bool same(const Kernel& a, const Kernel& b);

bool has_calls(const Block& b);
bool uses_extensions(const Kernel& k);

// ---- frontend -----------------------------------------------------------------
enum class Dialect { Strict, B200 };
// Restricted-CUDA input (cuda_frontend.cpp): a source with a `__global__` kernel is translated
// to MK+ text (same line numbers) before parsing in the B200 dialect.
bool looks_like_cuda(const std::string& src);
std::string cuda_to_mk(const std::string& src);  // Strict = the reference grammar byte for byte
Program parse_unchecked(const std::string& src, Dialect d = Dialect::B200);
Program parse(const std::string& src, Dialect d = Dialect::B200);  // + validate()
void validate(const Program& p);
struct Lint {
  Pos pos;
  std::string msg;
};
std::vector<Lint> lint(const Program& p);

// ---- normalization (passes.cpp of the reference) --------------------------------
Kernel inline_calls(const Kernel& k, const std::vector<Func>& funcs);
Kernel lift_declarations(const Kernel& k);
std::pair<Kernel, std::vector<std::pair<std::string, std::string>>> rename_locals(
    const Kernel& k, const std::string& prefix);
Kernel normalize(const Kernel& k, const std::vector<Func>& funcs, const std::string& prefix);
bool decl_prefix_form(const Kernel& k);

// MK+ -> plain Mini-Kernel (exact semantics), so the reference interpreter runs it.
Kernel downlower(const Kernel& k);
Program downlower(const Program& p);

// ---- printers ---------------------------------------------------------------
std::string print_mk(const Program& p);
std::string print_mk(const Kernel& k);
std::string print_expr(const Expr& e);
std::string float_text(float v);  // "%.9g" (+ ".0" when integral), as emit.cpp:66-75

}  // namespace hf
