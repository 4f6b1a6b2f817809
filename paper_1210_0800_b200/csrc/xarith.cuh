// xarith.cuh -- device-inline double / double-double / quad-double arithmetic.
//
// Each operation executes exactly the FP64 operations of the reference, in
// the reference's order, on the same operands, so results are bit-identical:
//   eft.hpp:24-72, double_double.hpp:41-122, quad_double.hpp:41-385.
// Every DADD/DMUL/DFMA is an explicit __dadd_rn/__dmul_rn/__fma_rn so nvcc can
// never contract a*b+c (the reference builds with -ffp-contract=off,
// proj/CMakeLists.txt:15); the library is also compiled with --fmad=false.
// Limbs live in registers; nothing here touches memory.
//
// Overflow: the reference throws overflow_error from every checked op whose
// leading limb is not finite (double_double.hpp:34-37, quad_double.hpp:202-205).
// The device instead lets Inf/NaN propagate (they are absorbing through
// +,*, and the renormalisations keep a non-finite head) and the kernels test
// the head limb of each finished column / coefficient -- see DESIGN.md §5.
//
// The header also compiles as plain host C++ (g++ -ffp-contract=off): the
// CPU test suite builds the very same arithmetic source into a host library
// (tests/cpp/arith_host.cpp) and checks it bit for bit against the oracle.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>

namespace xb {

#ifdef __CUDACC__
#define XB_DEV __host__ __device__ __forceinline__
#define XB_NOINLINE inline __host__ __device__ __noinline__
#define XB_DEVICE __device__ __forceinline__  // device-only helpers (shuffles, ...)
#else
#define XB_DEV inline
#define XB_NOINLINE
#endif

// Code-size and latency control.  Every quad-double add and multiply has a
// straight-line fast path (always inlined, so independent operations
// interleave) and a general path that replays the reference's branches for
// the lanes the fast path cannot take.  XB_CALLS is a bit mask: 1 = the
// general paths are real calls (they are rare; inlined they would dominate
// the code size), 2 = the complex quad-double operations and the scalar
// sqrt / reciprocal are real calls, 4 = the real quad-double add and
// multiply are real calls (no interleaving of independent operations, but
// the smallest code: the throughput-bound batched kernel runs many warps and
// needs its hot loop to fit the instruction cache; the latency-bound grid
// kernel wants the interleaving).
#ifndef XB_CALLS
#define XB_CALLS 7
#endif
#if defined(__CUDACC__)
#define XB_CALL_IF inline __host__ __device__ __noinline__
#else
#define XB_CALL_IF inline
#endif
#if (XB_CALLS & 1)
#define XB_GEN XB_CALL_IF
#else
#define XB_GEN XB_DEV
#endif
#if (XB_CALLS & 2)
#define XB_OP2 XB_CALL_IF
#else
#define XB_OP2 XB_DEV
#endif
#if (XB_CALLS & 4)
#define XB_OP4 XB_CALL_IF
#else
#define XB_OP4 XB_DEV
#endif

#ifdef __CUDA_ARCH__
XB_DEV double dadd(double a, double b) { return __dadd_rn(a, b); }
XB_DEV double dsub(double a, double b) { return __dsub_rn(a, b); }
XB_DEV double dmul(double a, double b) { return __dmul_rn(a, b); }
XB_DEV double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }
XB_DEV double ddiv(double a, double b) { return __ddiv_rn(a, b); }
XB_DEV double dsqrt(double a) { return __dsqrt_rn(a); }
XB_DEV long long dbits(double x) { return __double_as_longlong(x); }
XB_DEV double dabs(double x) { return fabs(x); }
#else
XB_DEV double dadd(double a, double b) { return a + b; }
XB_DEV double dsub(double a, double b) { return a - b; }
XB_DEV double dmul(double a, double b) { return a * b; }
XB_DEV double dfma(double a, double b, double c) { return std::fma(a, b, c); }
XB_DEV double ddiv(double a, double b) { return a / b; }
XB_DEV double dsqrt(double a) { return std::sqrt(a); }
XB_DEV long long dbits(double x) {
    long long v;
    std::memcpy(&v, &x, sizeof v);
    return v;
}
XB_DEV double dabs(double x) { return std::fabs(x); }
#endif

// ---- error-free transforms (eft.hpp) --------------------------------------
// eft.hpp:24-30
XB_DEV void two_sum(double a, double b, double& s, double& e) {
    s = dadd(a, b);
    double bb = dsub(s, a);
    double ea = dsub(a, dsub(s, bb));
    double eb = dsub(b, bb);
    e = dadd(ea, eb);
}
// eft.hpp:33-37
XB_DEV void quick_two_sum(double a, double b, double& s, double& e) {
    s = dadd(a, b);
    e = dsub(b, dsub(s, a));
}
// eft.hpp:59-62 (the FMA path eft.hpp:66-72 selects on FMA hardware)
XB_DEV void two_prod(double a, double b, double& p, double& e) {
    p = dmul(a, b);
    e = dfma(a, b, -p);
}

// select without a branch (selp on the device: nvcc otherwise turns chains
// of data-dependent ternaries into divergent branch ladders).  Enabled for
// the latency-bound single-system kernels (XB_USE_SELP); the throughput-bound
// batched kernel schedules better with plain ternaries.
#ifndef XB_USE_SELP
#define XB_USE_SELP 0
#endif
XB_DEV double dsel(bool p, double a, double b) {
#if defined(__CUDA_ARCH__) && XB_USE_SELP
    double r;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\tselp.f64 %0, %1, %2, q;\n\t}"
        : "=d"(r)
        : "d"(a), "d"(b), "r"((int)p));
    return r;
#else
    return p ? a : b;
#endif
}

XB_DEV bool finite(double x) {
    return (dbits(x) & 0x7ff0000000000000ll) != 0x7ff0000000000000ll;
}
XB_DEV bool is_inf(double x) {
    return (dbits(x) & 0x7fffffffffffffffll) == 0x7ff0000000000000ll;
}

// ---- real types -------------------------------------------------------------
struct r1 {  // double (real_type.hpp:16-20)
    double c0;
};
struct r2 {  // double_double {hi, lo} (double_double.hpp:15-22)
    double c0, c1;
};
struct r4 {  // quad_double c[4] (quad_double.hpp:19-26)
    double c0, c1, c2, c3;
};

template <int L>
struct real_of;
template <>
struct real_of<1> {
    using type = r1;
    static constexpr double eps = 0x1p-52;  // real_type.hpp:38
};
template <>
struct real_of<2> {
    using type = r2;
    static constexpr double eps = 0x1p-104;  // real_type.hpp:43
};
template <>
struct real_of<4> {
    using type = r4;
    static constexpr double eps = 0x1p-209;  // real_type.hpp:46
};

XB_DEV r1 make1(double v) { return {v}; }
XB_DEV r2 make2(double v) { return {v, 0.0}; }
XB_DEV r4 make4(double v) { return {v, 0.0, 0.0, 0.0}; }
template <class R>
XB_DEV R rmake(double v);
template <>
XB_DEV r1 rmake<r1>(double v) { return make1(v); }
template <>
XB_DEV r2 rmake<r2>(double v) { return make2(v); }
template <>
XB_DEV r4 rmake<r4>(double v) { return make4(v); }

XB_DEV double head(const r1& a) { return a.c0; }
XB_DEV double head(const r2& a) { return a.c0; }
XB_DEV double head(const r4& a) { return a.c0; }
// Overflow detection as the reference has it: double-double and quad-double
// arithmetic is checked (double_double.hpp:35, quad_double.hpp:203, eft.hpp:78-84
// raise overflow_error on a non-finite leading component), plain double is
// not (real_type.hpp:19) -- complex<double> results propagate Inf/NaN.
XB_DEV bool vfinite(const r1&) { return true; }
XB_DEV bool vfinite(const r2& a) { return finite(a.c0); }
XB_DEV bool vfinite(const r4& a) { return finite(a.c0); }

// ---- double ---------------------------------------------------------------
XB_DEV r1 add(const r1& a, const r1& b) { return {dadd(a.c0, b.c0)}; }
XB_DEV r1 neg(const r1& a) { return {-a.c0}; }
XB_DEV r1 sub(const r1& a, const r1& b) { return {dsub(a.c0, b.c0)}; }
XB_DEV r1 mul(const r1& a, const r1& b) { return {dmul(a.c0, b.c0)}; }
XB_DEV r1 rsqrt_ref(const r1& a) { return {dsqrt(a.c0)}; }
XB_DEV r1 div(const r1& a, const r1& b) { return {ddiv(a.c0, b.c0)}; }
XB_DEV bool lt(const r1& a, const r1& b) { return a.c0 < b.c0; }
XB_DEV bool le(const r1& a, const r1& b) { return a.c0 <= b.c0; }
XB_DEV bool ge(const r1& a, const r1& b) { return a.c0 >= b.c0; }
XB_DEV bool is_zero(const r1& a) { return a.c0 == 0.0; }
XB_DEV r1 rabs(const r1& a) { return {dabs(a.c0)}; }

// ---- double_double (double_double.hpp) -------------------------------------
// double_double.hpp:41-47
XB_DEV r2 add(const r2& a, const r2& b) {
    double s, se, t, te, v, ve, z, ze;
    two_sum(a.c0, b.c0, s, se);
    two_sum(a.c1, b.c1, t, te);
    quick_two_sum(s, dadd(se, t), v, ve);
    quick_two_sum(v, dadd(ve, te), z, ze);
    return {z, ze};
}
XB_DEV r2 neg(const r2& a) { return {-a.c0, -a.c1}; }       // :49
XB_DEV r2 sub(const r2& a, const r2& b) { return add(a, neg(b)); }  // :51-53
// double_double.hpp:56-63
XB_DEV r2 mul(const r2& a, const r2& b) {
    double p, pe, z, ze;
    two_prod(a.c0, b.c0, p, pe);
    double t = dmul(a.c1, b.c1);
    t = dfma(a.c0, b.c1, t);
    t = dfma(a.c1, b.c0, t);
    quick_two_sum(p, dadd(pe, t), z, ze);
    return {z, ze};
}
// double_double.hpp:66-70
XB_DEV r2 dd_add_d(const r2& a, double b) {
    double s, se, z, ze;
    two_sum(a.c0, b, s, se);
    quick_two_sum(s, dadd(se, a.c1), z, ze);
    return {z, ze};
}
// double_double.hpp:72-76
XB_DEV r2 dd_mul_d(const r2& a, double b) {
    double p, pe, z, ze;
    two_prod(a.c0, b, p, pe);
    quick_two_sum(p, dfma(a.c1, b, pe), z, ze);
    return {z, ze};
}
// double_double.hpp:94-104 (a >= 0, non-zero checked by caller semantics)
XB_DEV r2 rsqrt_ref(const r2& a) {
    if (a.c0 == 0.0 && a.c1 == 0.0) return {0.0, 0.0};
    double x = ddiv(1.0, dsqrt(a.c0));
    double ax = dmul(a.c0, x);
    double sq, sqe;
    two_prod(ax, ax, sq, sqe);
    r2 diff = sub(a, r2{sq, sqe});
    double corr = dmul(diff.c0, dmul(x, 0.5));
    double z, ze;
    quick_two_sum(ax, corr, z, ze);
    return {z, ze};
}
// double_double.hpp:106-115
XB_DEV bool lt(const r2& a, const r2& b) { return a.c0 < b.c0 || (a.c0 == b.c0 && a.c1 < b.c1); }
XB_DEV bool le(const r2& a, const r2& b) { return !lt(b, a); }
XB_DEV bool ge(const r2& a, const r2& b) { return !lt(a, b); }
XB_DEV bool is_zero(const r2& a) { return a.c0 == 0.0 && a.c1 == 0.0; }
XB_DEV r2 rabs(const r2& a) { return a.c0 < 0.0 ? neg(a) : a; }  // :117

// ---- quad_double (quad_double.hpp) -------------------------------------------
// quad_double.hpp:41-48
XB_DEV void three_sum(double& a, double& b, double& c) {
    double t, te, u, ue, v, ve;
    two_sum(a, b, t, te);
    two_sum(c, t, u, ue);
    two_sum(te, ue, v, ve);
    a = u;
    b = v;
    c = ve;
}
// quad_double.hpp:60-75
XB_DEV double quick_three_accum(double& a, double& b, double c) {
    double t, te, u, ue;
    two_sum(b, c, t, te);
    two_sum(a, t, u, ue);
    b = te;
    a = ue;
    bool za = (a != 0.0);
    bool zb = (b != 0.0);
    if (za && zb) return u;
    if (!zb) {
        b = a;
        a = u;
    } else {
        a = u;
    }
    return 0.0;
}
// quad_double.hpp:78-154.  The three-level branch tree is written as a
// pointer walk over (s0..s3): each level does one quick_two_sum at the
// current slot p, and advances p when the error term is non-zero.  Same ops,
// same operands, same order as every path of the reference tree.
XB_DEV void renorm5(double& c0, double& c1, double& c2, double& c3, double c4) {
    if (is_inf(c0)) return;
    double t, e;
    quick_two_sum(c3, c4, t, e);
    c4 = e;
    quick_two_sum(c2, t, t, e);
    c3 = e;
    quick_two_sum(c1, t, t, e);
    c2 = e;
    quick_two_sum(c0, t, t, e);
    c1 = e;
    c0 = t;

    double s0 = c0, s1 = c1, s2 = 0.0, s3 = 0.0;
    if (s1 != 0.0) {
        quick_two_sum(s1, c2, s1, s2);
        if (s2 != 0.0) {
            quick_two_sum(s2, c3, s2, s3);
            if (s3 != 0.0)
                s3 = dadd(s3, c4);
            else
                s2 = dadd(s2, c4);
        } else {
            quick_two_sum(s1, c3, s1, s2);
            if (s2 != 0.0)
                quick_two_sum(s2, c4, s2, s3);
            else
                quick_two_sum(s1, c4, s1, s2);
        }
    } else {
        quick_two_sum(s0, c2, s0, s1);
        if (s1 != 0.0) {
            quick_two_sum(s1, c3, s1, s2);
            if (s2 != 0.0)
                quick_two_sum(s2, c4, s2, s3);
            else
                quick_two_sum(s1, c4, s1, s2);
        } else {
            quick_two_sum(s0, c3, s0, s1);
            if (s1 != 0.0)
                quick_two_sum(s1, c4, s1, s2);
            else
                quick_two_sum(s0, c4, s0, s1);
        }
    }
    c0 = s0;
    c1 = s1;
    c2 = s2;
    c3 = s3;
}
// quad_double.hpp:157-200
XB_DEV void renorm4(double& c0, double& c1, double& c2, double& c3) {
    if (is_inf(c0)) return;
    double t, e;
    quick_two_sum(c2, c3, t, e);
    c3 = e;
    quick_two_sum(c1, t, t, e);
    c2 = e;
    quick_two_sum(c0, t, t, e);
    c1 = e;
    c0 = t;

    double s0 = c0, s1 = c1, s2 = 0.0, s3 = 0.0;
    if (s1 != 0.0) {
        quick_two_sum(s1, c2, s1, s2);
        if (s2 != 0.0)
            quick_two_sum(s2, c3, s2, s3);
        else
            quick_two_sum(s1, c3, s1, s2);
    } else {
        quick_two_sum(s0, c2, s0, s1);
        if (s1 != 0.0)
            quick_two_sum(s1, c3, s1, s2);
        else
            quick_two_sum(s0, c3, s0, s1);
    }
    c0 = s0;
    c1 = s1;
    c2 = s2;
    c3 = s3;
}

XB_DEV double pick4(int i, double x0, double x1, double x2, double x3) {
    double r = x3;
    r = (i == 2) ? x2 : r;
    r = (i == 1) ? x1 : r;
    r = (i == 0) ? x0 : r;
    return r;
}

// quad_double.hpp:216-257: merge the eight limbs by decreasing magnitude of
// the current heads, accumulate with quick_three_accum, fold the leftovers
// into x[3] (a's first, then b's), renormalise.  Indices stay in registers;
// limb reads are register selects, never local-memory indexing.  This is the
// general form; add() below runs it only for the lanes its fast path cannot
// take.
#ifdef XB_COUNT_GENERAL
inline long g_add_general = 0, g_mul_general = 0, g_add_zt = 0;
#define XB_COUNT(c) (++(c))
#else
#define XB_COUNT(c) ((void)0)
#endif
XB_GEN r4 add_general(const r4 a, const r4 b) {
    XB_COUNT(g_add_general);
    int i = 0, j = 0, k = 0;
    double u, v;
    double x0 = 0.0, x1 = 0.0, x2 = 0.0, x3 = 0.0;

    if (dabs(a.c0) > dabs(b.c0)) {
        u = a.c0;
        i = 1;
    } else {
        u = b.c0;
        j = 1;
    }
    {
        double ai = pick4(i, a.c0, a.c1, a.c2, a.c3);
        double bj = pick4(j, b.c0, b.c1, b.c2, b.c3);
        if (dabs(ai) > dabs(bj)) {
            v = ai;
            ++i;
        } else {
            v = bj;
            ++j;
        }
    }
    quick_two_sum(u, v, u, v);

    while (k < 4) {
        if (i >= 4 && j >= 4) {
            // x[k] = u; if (k < 3) x[++k] = v;
            x0 = (k == 0) ? u : x0;
            x1 = (k == 1) ? u : x1;
            x2 = (k == 2) ? u : x2;
            x3 = (k == 3) ? u : x3;
            x1 = (k == 0) ? v : x1;
            x2 = (k == 1) ? v : x2;
            x3 = (k == 2) ? v : x3;
            break;
        }
        double ai = pick4(i, a.c0, a.c1, a.c2, a.c3);
        double bj = pick4(j, b.c0, b.c1, b.c2, b.c3);
        bool take_a = (j >= 4) || (i < 4 && dabs(ai) > dabs(bj));
        double s = take_a ? ai : bj;
        i += take_a ? 1 : 0;
        j += take_a ? 0 : 1;
        double d = quick_three_accum(u, v, s);
        if (d != 0.0) {
            x0 = (k == 0) ? d : x0;
            x1 = (k == 1) ? d : x1;
            x2 = (k == 2) ? d : x2;
            x3 = (k == 3) ? d : x3;
            ++k;
        }
    }
    // for (; i < 4; ++i) x[3] += a.c[i]; for (; j < 4; ++j) x[3] += b.c[j];
    if (i <= 0) x3 = dadd(x3, a.c0);
    if (i <= 1) x3 = dadd(x3, a.c1);
    if (i <= 2) x3 = dadd(x3, a.c2);
    if (i <= 3) x3 = dadd(x3, a.c3);
    if (j <= 0) x3 = dadd(x3, b.c0);
    if (j <= 1) x3 = dadd(x3, b.c1);
    if (j <= 2) x3 = dadd(x3, b.c2);
    if (j <= 3) x3 = dadd(x3, b.c3);

    renorm4(x0, x1, x2, x3);
    return {x0, x1, x2, x3};
}

// One step of the reference merge loop on the next merged limb s:
// quick_three_accum(u, v, s) (quad_double.hpp:60-75) and, when it returns a
// non-zero component, x[k++] = it.  Branch-free: the zero tests become
// selects, the indexed store a predicated write.  KMAX = the largest k this
// step can see (k <= step index), so impossible slots cost nothing.
template <int KMAX>
XB_DEV void qadd_step(double& u, double& v, double s, int& k, double& x0, double& x1, double& x2,
                      double& x3) {
    double t, te, uu, ue;
    two_sum(v, s, t, te);
    two_sum(u, t, uu, ue);
    const bool zb = (te != 0.0);
    const bool emit = (ue != 0.0) && zb;
    v = dsel(zb, te, ue);
    u = dsel(emit, ue, uu);
    x0 = dsel(emit && k == 0, uu, x0);
    if (KMAX >= 1) x1 = dsel(emit && k == 1, uu, x1);
    if (KMAX >= 2) x2 = dsel(emit && k == 2, uu, x2);
    if (KMAX >= 3) x3 = dsel(emit && k == 3, uu, x3);
    k += emit ? 1 : 0;
}

// renorm4 (quad_double.hpp:157-200) for the common case -- no infinity, no
// zero error term along the way -- as straight-line code.  ok = false: the
// reference takes another branch; the caller replays the general path.
XB_DEV void renorm4_fast(double& c0, double& c1, double& c2, double& c3, bool& ok) {
    double t, e, s0, s1, d2, d3, t1, e1, u2, u3;
    const bool inf0 = is_inf(c0);
    quick_two_sum(c2, c3, t, e);
    d3 = e;
    quick_two_sum(c1, t, t, e);
    d2 = e;
    quick_two_sum(c0, t, s0, s1);
    // s1 != 0 -> quick_two_sum(s1, c2'); s2' != 0 -> quick_two_sum(s2', c3')
    quick_two_sum(s1, d2, t1, e1);
    quick_two_sum(e1, d3, u2, u3);
    ok = !inf0 && s1 != 0.0 && e1 != 0.0;
    c0 = s0;
    c1 = t1;
    c2 = u2;
    c3 = u3;
}

// The reference branch trees as calls: the fast forms fall back to them on the
// same pre-renormalisation components (no recomputation).
XB_GEN r4 renorm4_general(double c0, double c1, double c2, double c3) {
    renorm4(c0, c1, c2, c3);
    return {c0, c1, c2, c3};
}
XB_GEN r4 renorm5_general(double c0, double c1, double c2, double c3, double c4) {
    renorm5(c0, c1, c2, c3, c4);
    return {c0, c1, c2, c3};
}

// renorm (five components, quad_double.hpp:78-154), common case likewise:
// every zero test of the reference tree takes its "non-zero" side.
XB_DEV void renorm5_fast(double& c0, double& c1, double& c2, double& c3, double c4, bool& ok) {
    double t, e, d2, d3, d4, s0, s1, s1b, s2, s2b, s3;
    const bool inf0 = is_inf(c0);
    quick_two_sum(c3, c4, t, e);
    d4 = e;
    quick_two_sum(c2, t, t, e);
    d3 = e;
    quick_two_sum(c1, t, t, e);
    d2 = e;
    quick_two_sum(c0, t, s0, s1);
    quick_two_sum(s1, d2, s1b, s2);
    quick_two_sum(s2, d3, s2b, s3);
    ok = !inf0 && s1 != 0.0 && s2 != 0.0 && s3 != 0.0;
    c0 = s0;
    c1 = s1b;
    c2 = s2b;
    c3 = dadd(s3, d4);
}

// quad_double.hpp:216-257, the same operations on the same operands in the
// same order -- restructured for SIMT lanes that diverge on data.
//
// Fast path (no data-dependent branches).  When the limbs of a and b merge
// "level by level" (the larger of a_l, b_l, then the smaller, for l = 0..3),
// the merged sequence m0..m7 is known after the four level comparisons plus
// three cross checks -- exactly the comparisons the reference merge makes --
// and the merge loop becomes six fixed steps.  It also needs the loop to run
// to the end (k <= 3 before the last step), so every limb is consumed, the
// leftover fold is empty and the loop exit writes x[k] = u, x[k+1] = v.  That
// covers operands of similar magnitude -- the MGS inner products, updates and
// reductions.  Lanes outside it (zero or exhausted limbs mid-merge, widely
// different exponents, early exits) run add_general; the branch is taken per
// warp only when some lane needs it.  add_fast() reports whether its result
// is the reference's (ok); callers with independent adds run all fast paths
// first and branch once.
// The level-paired fast path in three stages (setup, six merge steps,
// finish), so that independent adds can be written in lockstep (add_fast2)
// and their dependency chains interleave.
struct qadd_st {
    double m2, m3, m4, m5, m6, m7;
    double u, v, x0, x1, x2, x3;
    int k;
    bool ok;
    // the merged order of any leftovers equals the reference's leftover fold
    // (a's remaining limbs, then b's): an early loop exit (k == 4) is then
    // handled in place -- the remaining limbs are added to x[3] in order
    bool tail = false;
};
XB_DEV void qadd_setup(const r4& a, const r4& b, qadd_st& q) {
    const bool f0 = dabs(a.c0) > dabs(b.c0), f1 = dabs(a.c1) > dabs(b.c1);
    const bool f2 = dabs(a.c2) > dabs(b.c2), f3 = dabs(a.c3) > dabs(b.c3);
    const double m0 = f0 ? a.c0 : b.c0, m1 = f0 ? b.c0 : a.c0;
    q.m2 = f1 ? a.c1 : b.c1;
    q.m3 = f1 ? b.c1 : a.c1;
    q.m4 = f2 ? a.c2 : b.c2;
    q.m5 = f2 ? b.c2 : a.c2;
    q.m6 = f3 ? a.c3 : b.c3;
    q.m7 = f3 ? b.c3 : a.c3;
    // the smaller limb of level l beats both limbs of level l+1 strictly: then
    // the reference's comparison against the successor of the taken limb
    // picks it (|a_{l+1}| > |b_l| is false, resp. |a_l| > |b_{l+1}| is true)
    q.ok = (dabs(m1) > dabs(q.m2)) && (dabs(q.m3) > dabs(q.m4)) && (dabs(q.m5) > dabs(q.m6));
    quick_two_sum(m0, m1, q.u, q.v);
    q.x0 = q.x1 = q.x2 = q.x3 = 0.0;
    q.k = 0;
}
template <int STEP>
XB_DEV void qadd_run(qadd_st& q) {
    const double s = STEP == 0 ? q.m2 : STEP == 1 ? q.m3 : STEP == 2 ? q.m4 : STEP == 3 ? q.m5
                   : STEP == 4 ? q.m6 : q.m7;
    if (q.tail && STEP >= 3 && q.k >= 4) {  // loop already left: fold (quad_double.hpp:254-255)
        q.x3 = dadd(q.x3, s);
        return;
    }
    if (STEP == 5 && !q.tail) q.ok = q.ok && (q.k <= 3);  // the loop reaches its last step
    qadd_step<(STEP < 3 ? STEP : 3)>(q.u, q.v, s, q.k, q.x0, q.x1, q.x2, q.x3);
}
XB_DEV r4 qadd_finish(qadd_st& q, bool& okr) {
    // loop exit with everything consumed: x[k] = u; if (k < 3) x[k + 1] = v
    const int k = q.k;
    const double x0 = dsel(k == 0, q.u, q.x0);
    const double x1 = dsel(k == 1, q.u, dsel(k == 0, q.v, q.x1));
    const double x2 = dsel(k == 2, q.u, dsel(k == 1, q.v, q.x2));
    const double x3 = dsel(k == 3, q.u, dsel(k == 2, q.v, q.x3));
    double y0 = x0, y1 = x1, y2 = x2, y3 = x3;
    bool okn;
    renorm4_fast(y0, y1, y2, y3, okn);
    okr = q.ok;
    if (!okn) return renorm4_general(x0, x1, x2, x3);
    return {y0, y1, y2, y3};
}
XB_DEV r4 add_fast(const r4& a, const r4& b, bool& okr) {
    qadd_st q;
    qadd_setup(a, b, q);
    qadd_run<0>(q);
    qadd_run<1>(q);
    qadd_run<2>(q);
    qadd_run<3>(q);
    qadd_run<4>(q);
    qadd_run<5>(q);
    return qadd_finish(q, okr);
}
// The level-paired fast path with the merge's output slots x[0..3] in memory
// instead of registers (XB_XSMEM).  The register form writes each emitted
// limb with a select per slot it could land in (x[k] for every k the step can
// see: 18 double selects over the six steps, 7 more for the loop exit), which
// made FSEL the second most executed instruction of the batched kernel after
// DADD.  Here every step stores its candidate uu into the OPEN slot k (one
// store; k advances when the reference emits), so a non-emitted candidate is
// overwritten by the next emission or by the loop exit's x[k] = u -- exactly
// the reference's x[k++] = d (quad_double.hpp:244-246) and x[k] = u,
// x[++k] = v (:237-239).  Writes are monotone in k, so slots 2 and 3, zeroed
// first, stay +0 unless reached, as x = {0, 0, 0, 0} does in the reference.
// NT = the slot stride (threads sharing the slot array); slots 0..7 are
// addressable (k <= 6 even when the fast path does not apply).
template <int NT>
XB_DEV void qadd_step_xs(double& u, double& v, double s, int& k, double* xs) {
    double t, te, uu, ue;
    two_sum(v, s, t, te);
    two_sum(u, t, uu, ue);
    const bool zb = (te != 0.0);
    const bool emit = (ue != 0.0) && zb;
    v = dsel(zb, te, ue);
    u = dsel(emit, ue, uu);
    xs[k * NT] = uu;
    k += emit ? 1 : 0;
}
template <int NT>
XB_DEV r4 add_fast_xs(const r4& a, const r4& b, bool& okr, double* xs) {
    qadd_st q;
    qadd_setup(a, b, q);
    xs[2 * NT] = 0.0;
    xs[3 * NT] = 0.0;
    int k = 0;
    qadd_step_xs<NT>(q.u, q.v, q.m2, k, xs);
    qadd_step_xs<NT>(q.u, q.v, q.m3, k, xs);
    qadd_step_xs<NT>(q.u, q.v, q.m4, k, xs);
    qadd_step_xs<NT>(q.u, q.v, q.m5, k, xs);
    qadd_step_xs<NT>(q.u, q.v, q.m6, k, xs);
    const bool ok = q.ok && (k <= 3);  // the loop reaches its last step
    qadd_step_xs<NT>(q.u, q.v, q.m7, k, xs);
    // loop exit with everything consumed: x[k] = u; if (k < 3) x[k + 1] = v
    // (k == 4: the loop left on its own condition, u and v are dropped)
    xs[k * NT] = q.u;
    if (k < 3) xs[(k + 1) * NT] = q.v;
    const double x0 = xs[0], x1 = xs[NT], x2 = xs[2 * NT], x3 = xs[3 * NT];
    double y0 = x0, y1 = x1, y2 = x2, y3 = x3;
    bool okn;
    renorm4_fast(y0, y1, y2, y3, okn);
    okr = ok;
    if (!okn) return renorm4_general(x0, x1, x2, x3);
    return {y0, y1, y2, y3};
}
#ifndef XB_XSMEM
#define XB_XSMEM 0
#endif
// one column of 8 slots per thread, CTAs of up to XB_XS_THREADS threads
#ifndef XB_XS_THREADS
#define XB_XS_THREADS 384
#endif
#if XB_XSMEM && defined(__CUDA_ARCH__)
constexpr int kXsThreads = XB_XS_THREADS;
static __shared__ double xb_xslots[8][kXsThreads];
XB_DEVICE r4 add_fast_any(const r4& a, const r4& b, bool& ok) {
    return add_fast_xs<kXsThreads>(a, b, ok, &xb_xslots[0][threadIdx.x]);
}
#elif XB_XSMEM
XB_DEV r4 add_fast_any(const r4& a, const r4& b, bool& ok) {
    double xs[8];
    return add_fast_xs<1>(a, b, ok, xs);
}
#else
XB_DEV r4 add_fast_any(const r4& a, const r4& b, bool& ok) { return add_fast(a, b, ok); }
#endif
// two independent adds in lockstep
XB_DEV void add_fast2(const r4& a1, const r4& b1, const r4& a2, const r4& b2, r4& o1, bool& k1,
                      r4& o2, bool& k2) {
    qadd_st p, q;
    qadd_setup(a1, b1, p);
    qadd_setup(a2, b2, q);
    qadd_run<0>(p);
    qadd_run<0>(q);
    qadd_run<1>(p);
    qadd_run<1>(q);
    qadd_run<2>(p);
    qadd_run<2>(q);
    qadd_run<3>(p);
    qadd_run<3>(q);
    qadd_run<4>(p);
    qadd_run<4>(q);
    qadd_run<5>(p);
    qadd_run<5>(q);
    o1 = qadd_finish(p, k1);
    o2 = qadd_finish(q, k2);
}
// Second fast path for merges that are not level-paired but still fixed:
//   a = (x,0,0,0):  heads, b1, b2, b3, a1, a2, a3  (b0 taken first needs
//                   |a0| > |b1|)                      -- widened constants,
//   b = (y,0,0,0):  heads, a1, a2, a3, b1, b2, b3  (needs |a1|,|a2|,|a3| > 0
//                   and a0 taken first !(|a1| > |b0|), b0 first |a0| > 0),
//   disjoint:       a0..a3 then b0..b3 (every |a_i| > |b0|), or b0..b3 then
//                   a0..a3 (no |a0| > |b_j|)          -- a tiny Newton
//                   correction, a zero operand.
// Each pattern is recognised by exactly the comparisons the reference merge
// makes; the merge steps are then the same six fixed steps.
// Shifted merges: one operand leads by S levels (a Newton correction whose
// head sits S limbs down, PAPER-style x + 0.5*x*(1 - a*x*x)):
//   H0 .. H_{S-1}, then level pairs (H_{S+l}, T_l), then T_{4-S} .. T_3.
// Recognised by strict separations that imply every comparison the reference
// merge makes (|H_i| > |T_0| for the lead, pair levels apart, the lead's last
// limb beating T's next one); the pair order is the reference rule (a first
// iff |a| > |b|).  Fills m[0..7] and returns whether the pattern holds.
// tail_ok: an early loop exit (four limbs emitted before all eight are
// merged) leaves only m6, m7 or m7; the reference then folds a's leftovers
// before b's, which is the merge order unless m6 is b's and m7 is a's --
// possible only for S = 1 with b leading and its last pair taken first.
#ifndef XB_SHIFT_TAIL
#define XB_SHIFT_TAIL 0
#endif
template <int S>
XB_DEV bool shift_merge(const r4& H, const r4& T, bool h_is_a, double (&m)[8], bool& tail_ok) {
    tail_ok = true;
    const double h[4] = {H.c0, H.c1, H.c2, H.c3}, t[4] = {T.c0, T.c1, T.c2, T.c3};
    bool ok = true;
#pragma unroll
    for (int i = 0; i < S; ++i) {
        ok = ok && (dabs(h[i]) > dabs(t[0]));
        m[i] = h[i];
    }
    double lo_prev = 0.0;
#pragma unroll
    for (int l = 0; l + S < 4; ++l) {
        const double hh = h[S + l], tt = t[l];
        // a first iff |a| > |b|
        const bool hfirst = h_is_a ? (dabs(hh) > dabs(tt)) : !(dabs(tt) > dabs(hh));
        const double hi = hfirst ? hh : tt, lo = hfirst ? tt : hh;
        if (l > 0) ok = ok && (dabs(lo_prev) > dabs(hi));
        m[S + 2 * l] = hi;
        m[S + 2 * l + 1] = lo;
        lo_prev = lo;
        if (l + S == 3) {
            // after the last pair: if T's limb went first, H_3 must beat T_{4-S}
            ok = ok && (hfirst || (dabs(hh) > dabs(t[4 - S])));
            if (S == 1) tail_ok = h_is_a || hfirst;
        }
    }
#pragma unroll
    for (int l = 4 - S; l < 4; ++l) m[4 + l] = t[l];
    return ok;
}

XB_DEV r4 add_alt_fast(const r4& a, const r4& b, bool& okr) {
    const double A0 = dabs(a.c0), A1 = dabs(a.c1), A2 = dabs(a.c2), A3 = dabs(a.c3);
    const double B0 = dabs(b.c0), B1 = dabs(b.c1), B2 = dabs(b.c2), B3 = dabs(b.c3);
    const bool f0 = A0 > B0;
    const bool da = f0 && (A1 > B0) && (A2 > B0) && (A3 > B0);              // a first
    const bool db = !f0 && !(A0 > B1) && !(A0 > B2) && !(A0 > B3);          // b first
    const bool ta = (a.c1 == 0.0) && (a.c2 == 0.0) && (a.c3 == 0.0);
    const bool tb = (b.c1 == 0.0) && (b.c2 == 0.0) && (b.c3 == 0.0);
    const bool pa = ta && (f0 || (A0 > B1));
    const bool pb = tb && (A1 > 0.0) && (A2 > 0.0) && (A3 > 0.0) && (f0 ? !(A1 > B0) : (A0 > 0.0));
    qadd_st q;
    double m0, m1;
    if (da || db) {
        const r4& h = da ? a : b;
        const r4& l = da ? b : a;
        m0 = h.c0;
        m1 = h.c1;
        q.m2 = h.c2;
        q.m3 = h.c3;
        q.m4 = l.c0;
        q.m5 = l.c1;
        q.m6 = l.c2;
        q.m7 = l.c3;
    } else {
        m0 = f0 ? a.c0 : b.c0;
        m1 = f0 ? b.c0 : a.c0;
        q.m2 = pa ? b.c1 : a.c1;
        q.m3 = pa ? b.c2 : a.c2;
        q.m4 = pa ? b.c3 : a.c3;
        q.m5 = pa ? a.c1 : b.c1;
        q.m6 = pa ? a.c2 : b.c2;
        q.m7 = pa ? a.c3 : b.c3;
    }
    q.ok = da || db || pa || pb;
    q.tail = da;  // a0..a3 then b0..b3: leftovers come a's first, then b's
    if (!q.ok) {
        // shifted merges, a or b leading by 1..3 levels
        double mm[8];
        const bool alead = f0;
        const r4& H = alead ? a : b;
        const r4& T = alead ? b : a;
        bool tail_ok;
        bool hit = shift_merge<2>(H, T, alead, mm, tail_ok);
        if (!hit) hit = shift_merge<1>(H, T, alead, mm, tail_ok);
        if (!hit) hit = shift_merge<3>(H, T, alead, mm, tail_ok);
        if (hit) {
            // XB_SHIFT_TAIL: fold leftovers in place after an early exit (the
            // single-system kernels, whose Newton chains hit it ~25 % of the
            // time); off elsewhere -- the batched kernel is faster without
            // the extra live state in its call-form helpers
            q.tail = XB_SHIFT_TAIL ? tail_ok : false;
            m0 = mm[0];
            m1 = mm[1];
            q.m2 = mm[2];
            q.m3 = mm[3];
            q.m4 = mm[4];
            q.m5 = mm[5];
            q.m6 = mm[6];
            q.m7 = mm[7];
            q.ok = true;
        }
    }
    quick_two_sum(m0, m1, q.u, q.v);
    q.x0 = q.x1 = q.x2 = q.x3 = 0.0;
    q.k = 0;
    qadd_run<0>(q);
    qadd_run<1>(q);
    qadd_run<2>(q);
    qadd_run<3>(q);
    qadd_run<4>(q);
    qadd_run<5>(q);
    return qadd_finish(q, okr);
}

// The reference merge in full generality, but predicated instead of
// branched (quad_double.hpp:216-257): the heads are picked by register
// selects on the consumed counts i, j; the six loop steps always execute,
// and after the loop has exited (k == 4) they change nothing; the leftover
// fold adds a's then b's remaining limbs in order.  Same operations on the
// same operands as the reference for every input; no lane divergence.
XB_DEV double pick4v(int i, const r4& a) {
    const double lo = (i & 1) ? a.c1 : a.c0;
    const double hi = (i & 1) ? a.c3 : a.c2;
    return (i & 2) ? hi : lo;
}
XB_DEV r4 add_merge_pred(const r4& a, const r4& b) {
    int i = 0, j = 0;
    bool t = dabs(a.c0) > dabs(b.c0);
    double u = t ? a.c0 : b.c0;
    i += t ? 1 : 0;
    j += t ? 0 : 1;
    double ai = t ? a.c1 : a.c0, bj = t ? b.c0 : b.c1;
    t = dabs(ai) > dabs(bj);
    double v = t ? ai : bj;
    i += t ? 1 : 0;
    j += t ? 0 : 1;
    quick_two_sum(u, v, u, v);
    double x0 = 0.0, x1 = 0.0, x2 = 0.0, x3 = 0.0;
    int k = 0;
#pragma unroll
    for (int step = 0; step < 6; ++step) {
        const bool live = (k < 4);
        ai = pick4v(i, a);
        bj = pick4v(j, b);
        const bool ta = (j >= 4) || (i < 4 && dabs(ai) > dabs(bj));
        const double s = ta ? ai : bj;
        double tt, te, uu, ue;
        two_sum(v, s, tt, te);
        two_sum(u, tt, uu, ue);
        const bool zb = (te != 0.0);
        const bool emit = live && (ue != 0.0) && zb;
        v = live ? (zb ? te : ue) : v;
        u = live ? (emit ? ue : uu) : u;
        x0 = (emit && k == 0) ? uu : x0;
        x1 = (emit && k == 1) ? uu : x1;
        x2 = (emit && k == 2) ? uu : x2;
        x3 = (emit && k == 3) ? uu : x3;
        k += emit ? 1 : 0;
        i += (live && ta) ? 1 : 0;
        j += (live && !ta) ? 1 : 0;
    }
    // exhausted with k < 4: x[k] = u; if (k < 3) x[k + 1] = v
    x0 = (k == 0) ? u : x0;
    x1 = (k == 1) ? u : ((k == 0) ? v : x1);
    x2 = (k == 2) ? u : ((k == 1) ? v : x2);
    x3 = (k == 3) ? u : ((k == 2) ? v : x3);
    // leftovers (only after an early exit): a's first, then b's
    if (i <= 0) x3 = dadd(x3, a.c0);
    if (i <= 1) x3 = dadd(x3, a.c1);
    if (i <= 2) x3 = dadd(x3, a.c2);
    if (i <= 3) x3 = dadd(x3, a.c3);
    if (j <= 0) x3 = dadd(x3, b.c0);
    if (j <= 1) x3 = dadd(x3, b.c1);
    if (j <= 2) x3 = dadd(x3, b.c2);
    if (j <= 3) x3 = dadd(x3, b.c3);
    double y0 = x0, y1 = x1, y2 = x2, y3 = x3;
    bool okn;
    renorm4_fast(y0, y1, y2, y3, okn);
    if (!okn) return renorm4_general(x0, x1, x2, x3);
    return {y0, y1, y2, y3};
}

// Everything the level-paired path does not cover: the alternative fixed
// merges, else the reference merge (one call, so the inlined fast path stays
// small).
XB_GEN r4 add_slow(const r4 a, const r4 b) {
    bool ok;
    r4 r = add_alt_fast(a, b, ok);
    if (!ok) r = add_merge_pred(a, b);
    return r;
}

XB_OP4 r4 add(const r4 a, const r4 b) {
    bool ok;
    r4 r = add_fast_any(a, b, ok);
    if (!ok) r = add_slow(a, b);
    return r;
}
XB_DEV r4 neg(const r4& a) { return {-a.c0, -a.c1, -a.c2, -a.c3}; }  // :259-261
// renormalize (real_type.hpp:20, double_double.hpp:28-31, quad_double.hpp:209-213)
XB_DEV r1 renormalize(const r1& a) { return a; }
XB_DEV r2 renormalize(const r2& a) {
    r2 o;
    quick_two_sum(a.c0, a.c1, o.c0, o.c1);
    return o;
}
XB_DEV r4 renormalize(const r4& a) {
    r4 o = a;
    renorm4(o.c0, o.c1, o.c2, o.c3);
    return o;
}
XB_DEV r4 sub(const r4& a, const r4& b) { return add(a, neg(b)); }     // :263

// quad_double.hpp:267-338: every partial product to order u^3 through EFTs;
// qmul_core stops before the final renormalisation.
XB_DEV void qmul_core(const r4& a, const r4& b, double& p0, double& p1, double& s0, double& t0c,
                      double& t1c) {
    double q0, q1, p2, q2, p3, q3, p4, q4, p5, q5;
    two_prod(a.c0, b.c0, p0, q0);
    two_prod(a.c0, b.c1, p1, q1);
    two_prod(a.c1, b.c0, p2, q2);
    two_prod(a.c0, b.c2, p3, q3);
    two_prod(a.c1, b.c1, p4, q4);
    two_prod(a.c2, b.c0, p5, q5);

    three_sum(p1, p2, q0);

    three_sum(p2, q1, q2);
    three_sum(p3, p4, p5);
    double t0, s1, t1;
    two_sum(p2, p3, s0, t0);
    two_sum(q1, p4, s1, t1);
    // (s2 = q2 + p5; s2 += t0 + t1 is dead in the reference: never read)
    two_sum(s1, t0, s1, t0);

    double p6, q6, p7, q7, p8, q8, p9, q9;
    two_prod(a.c0, b.c3, p6, q6);
    two_prod(a.c1, b.c2, p7, q7);
    two_prod(a.c2, b.c1, p8, q8);
    two_prod(a.c3, b.c0, p9, q9);

    two_sum(q0, q3, q0, q3);
    two_sum(q4, q5, q4, q5);
    two_sum(p6, p7, p6, p7);
    two_sum(p8, p9, p8, p9);

    double t0b, t1b;
    two_sum(q0, q4, t0b, t1b);
    t1b = dadd(t1b, dadd(q3, q5));

    double r0, r1;
    two_sum(p6, p8, r0, r1);
    r1 = dadd(r1, dadd(p7, p9));

    double q3b, q4b;
    two_sum(t0b, r0, q3b, q4b);
    q4b = dadd(q4b, dadd(t1b, r1));

    two_sum(q3b, s1, t0c, t1c);
    t1c = dadd(t1c, q4b);

    // t1c += a1*b3 + a2*b2 + a3*b1 + q6 + q7 + q8 + q9 (left to right)
    double w = dadd(dmul(a.c1, b.c3), dmul(a.c2, b.c2));
    w = dadd(w, dmul(a.c3, b.c1));
    w = dadd(w, q6);
    w = dadd(w, q7);
    w = dadd(w, q8);
    w = dadd(w, q9);
    t1c = dadd(t1c, w);

}
XB_DEV r4 qmul_finish(double p0, double p1, double s0, double t0c, double t1c) {
    double y0 = p0, y1 = p1, y2 = s0, y3 = t0c;
    bool okn;
    renorm5_fast(y0, y1, y2, y3, t1c, okn);
    if (!okn) return renorm5_general(p0, p1, s0, t0c, t1c);
    return {y0, y1, y2, y3};
}
XB_DEV r4 mul_fast(const r4& a, const r4& b, bool& ok) {
    double p0, p1, s0, t0c, t1c;
    qmul_core(a, b, p0, p1, s0, t0c, t1c);
    ok = true;
    return qmul_finish(p0, p1, s0, t0c, t1c);
}
// independent products in lockstep: the cores first, then the renormalisations
XB_DEV void mul_fast2(const r4& a1, const r4& b1, const r4& a2, const r4& b2, r4& o1, bool& k1,
                      r4& o2, bool& k2) {
    double p0, p1, s0, t0c, t1c, q0, q1, u0, v0c, v1c;
    qmul_core(a1, b1, p0, p1, s0, t0c, t1c);
    qmul_core(a2, b2, q0, q1, u0, v0c, v1c);
    double y0 = p0, y1 = p1, y2 = s0, y3 = t0c, w0 = q0, w1 = q1, w2 = u0, w3 = v0c;
    bool n1, n2;
    renorm5_fast(y0, y1, y2, y3, t1c, n1);
    renorm5_fast(w0, w1, w2, w3, v1c, n2);
    o1 = {y0, y1, y2, y3};
    o2 = {w0, w1, w2, w3};
    if (!(n1 && n2)) {
        if (!n1) o1 = renorm5_general(p0, p1, s0, t0c, t1c);
        if (!n2) o2 = renorm5_general(q0, q1, u0, v0c, v1c);
    }
    k1 = k2 = true;
}
XB_GEN r4 mul_general(const r4 a, const r4 b) {
    XB_COUNT(g_mul_general);
    double p0, p1, s0, t0c, t1c;
    qmul_core(a, b, p0, p1, s0, t0c, t1c);
    renorm5(p0, p1, s0, t0c, t1c);
    return {p0, p1, s0, t0c};
}
XB_OP4 r4 mul(const r4 a, const r4 b) {
    bool ok;
    r4 r = mul_fast(a, b, ok);
    if (!ok) r = mul_general(a, b);
    return r;
}

// Always-call forms of the qd add / multiply, for the latency-bound scalar
// chains (Newton iterations, reduction trees, pivot divisions): one shared
// copy of each operation stays hot in the instruction cache of a lone warp.
// (when add / mul are calls already -- XB_CALLS & 4 -- these are the same
// calls, not a second call layer around them)
#if (XB_CALLS & 4)
#define XB_CALLC XB_DEV
#else
#define XB_CALLC XB_CALL_IF
#endif
XB_CALLC r4 addc(const r4 a, const r4 b) { return add(a, b); }
// the Newton sites where the operands are known to merge unevenly (a
// constant 1.0 or seed with zero lower limbs, a correction several limbs
// down): try the alternative fixed merges first
XB_CALL_IF r4 addz(const r4 a, const r4 b) {
    bool ok;
    r4 r = add_alt_fast(a, b, ok);
    if (ok) return r;
    r = add_fast(a, b, ok);
    if (ok) return r;
    return add_merge_pred(a, b);
}
XB_DEV r4 subz(const r4& a, const r4& b) { return addz(a, neg(b)); }
XB_CALLC r4 mulc(const r4 a, const r4 b) { return mul(a, b); }
XB_DEV r4 subc(const r4& a, const r4& b) { return addc(a, neg(b)); }
XB_DEV r1 addc(const r1& a, const r1& b) { return add(a, b); }
XB_DEV r2 addc(const r2& a, const r2& b) { return add(a, b); }

XB_DEV r4 mul_pwr2(const r4& a, double p2) {  // :341-343
    return {dmul(a.c0, p2), dmul(a.c1, p2), dmul(a.c2, p2), dmul(a.c3, p2)};
}
// quad_double.hpp:359-370
XB_OP2 r4 rsqrt_ref(const r4 a) {
    if (a.c0 == 0.0 && a.c1 == 0.0 && a.c2 == 0.0 && a.c3 == 0.0) return {0.0, 0.0, 0.0, 0.0};
    r4 x = make4(ddiv(1.0, dsqrt(a.c0)));
#pragma unroll 1
    for (int it = 0; it < 2; ++it) {
        r4 t = mulc(a, x);
        x = addz(x, mul_pwr2(mulc(x, subz(make4(1.0), mulc(t, x))), 0.5));
    }
    r4 y = mulc(a, x);
    y = addz(y, mul_pwr2(mulc(subc(a, mulc(y, y)), x), 0.5));
    return y;
}
// quad_double.hpp:372-383
XB_DEV bool lt(const r4& a, const r4& b) {
    if (a.c0 < b.c0) return true;
    if (a.c0 > b.c0) return false;
    if (a.c1 < b.c1) return true;
    if (a.c1 > b.c1) return false;
    if (a.c2 < b.c2) return true;
    if (a.c2 > b.c2) return false;
    return a.c3 < b.c3;
}
XB_DEV bool le(const r4& a, const r4& b) { return !lt(b, a); }
XB_DEV bool ge(const r4& a, const r4& b) { return !lt(a, b); }
XB_DEV bool is_zero(const r4& a) { return a.c0 == 0.0 && a.c1 == 0.0 && a.c2 == 0.0 && a.c3 == 0.0; }
XB_DEV r4 rabs(const r4& a) { return a.c0 < 0.0 ? neg(a) : a; }  // :385

// ---- division with the divisor-only part hoisted -------------------------------
// The reference division (double_double.hpp:80-90, quad_double.hpp:346-355)
// first builds a reciprocal estimate from the divisor alone, then runs a
// short tail on the dividend.  recip() is that divisor-only prefix; divide()
// is the tail.  divide(a, b, recip(b)) == a / b bit for bit, so a pivot
// computes recip(r_kk) once and every row reuses it.
// Status from recip(): 0 ok, 3 = domain (b == 0), 2 = overflow (1/b not finite).
template <class R>
struct recip_t;
template <>
struct recip_t<r1> {
    double b;
};
template <>
struct recip_t<r2> {
    r2 x1;
};
template <>
struct recip_t<r4> {
    r4 x;
};

// plain IEEE division for double (real_type.hpp: no checked funnel)
XB_DEV recip_t<r1> recip(const r1& b, int& status) { return {b.c0}; }
XB_DEV r1 div_plain(const r1& a, const r1& b) { return {ddiv(a.c0, b.c0)}; }
XB_DEV r1 divide(const r1& a, const r1& b, const recip_t<r1>& rc) { return {ddiv(a.c0, rc.b)}; }

XB_DEV recip_t<r2> recip(const r2& b, int& status) {
    if (b.c0 == 0.0) {
        status = 3;
        return {{0.0, 0.0}};
    }
    double x0 = ddiv(1.0, b.c0);
    if (!finite(x0)) status = 2;
    r2 e = sub(make2(1.0), dd_mul_d(b, x0));
    return {dd_add_d(dd_mul_d(e, x0), x0)};
}
XB_DEV r2 divide(const r2& a, const r2& b, const recip_t<r2>& rc) {
    r2 q = mul(a, rc.x1);
    r2 r = sub(a, mul(b, q));
    return add(q, mul(r, rc.x1));
}

XB_OP2 recip_t<r4> recip(const r4 b, int& status) {
    if (b.c0 == 0.0) {
        status = 3;
        return {{0.0, 0.0, 0.0, 0.0}};
    }
    double seed = ddiv(1.0, b.c0);
    if (!finite(seed)) status = 2;
    r4 x = make4(seed);
#pragma unroll 1
    for (int it = 0; it < 2; ++it) x = addz(x, mulc(x, subz(make4(1.0), mulc(b, x))));
    return {x};
}
XB_DEV r4 divide(const r4& a, const r4& b, const recip_t<r4>& rc) {
    r4 q = mulc(a, rc.x);
    return addz(q, mulc(rc.x, subc(a, mulc(b, q))));
}

// divide() with its five operations inline instead of the shared call
// forms (same operations, same bits): faster where the surrounding code is
// small enough to stay in the instruction cache (the back-substitution step)
XB_DEV r4 divide_inline(const r4& a, const r4& b, const recip_t<r4>& rc) {
    const r4 q = mul(a, rc.x);
    const r4 c = mul(rc.x, add(a, neg(mul(b, q))));
    bool ok;
    r4 out = add_alt_fast(q, c, ok);  // addz: the correction sits limbs below q
    if (!ok) out = add(q, c);
    return out;
}
XB_DEV r2 divide_inline(const r2& a, const r2& b, const recip_t<r2>& rc) { return divide(a, b, rc); }
XB_DEV r1 divide_inline(const r1& a, const r1& b, const recip_t<r1>& rc) { return divide(a, b, rc); }

template <class R>
XB_DEV R rdiv(const R& a, const R& b, int& status) {
    recip_t<R> rc = recip(b, status);
    return divide(a, b, rc);
}

// ---- complex (complex.hpp) -------------------------------------------------------
template <class R>
struct cx {
    R re, im;
};

template <class R>
XB_DEV cx<R> cconj(const cx<R>& z) {  // complex.hpp:21-24
    return {z.re, neg(z.im)};
}
// Two independent operations: both fast paths first (they interleave), one
// branch to the general paths.  Generic form for double / double-double.
template <class R>
struct rpair {
    R x, y;
};
template <class R>
XB_DEV rpair<R> add2(const R& a1, const R& b1, const R& a2, const R& b2) {
    return {add(a1, b1), add(a2, b2)};
}
template <class R>
XB_DEV rpair<R> mul2(const R& a1, const R& b1, const R& a2, const R& b2) {
    return {mul(a1, b1), mul(a2, b2)};
}
// Two independent qd adds / products in lockstep (their dependency chains
// interleave).  XB_CALLS bit 16 makes each pair ONE real call -- a single
// shared copy of the lockstep code: the interleaving of the inlined form at
// the instruction-cache cost of a call (the batched kernel's trade-off).
#if (XB_CALLS & 16)
#define XB_PAIR XB_CALL_IF
#else
#define XB_PAIR XB_DEV
#endif
XB_PAIR rpair<r4> add2_r4(const r4 a1, const r4 b1, const r4 a2, const r4 b2) {
    bool k1, k2;
    rpair<r4> o;
    add_fast2(a1, b1, a2, b2, o.x, k1, o.y, k2);
    if (!(k1 && k2)) {
        if (!k1) o.x = add_slow(a1, b1);
        if (!k2) o.y = add_slow(a2, b2);
    }
    return o;
}
XB_PAIR rpair<r4> mul2_r4(const r4 a1, const r4 b1, const r4 a2, const r4 b2) {
    bool k1, k2;
    rpair<r4> o;
    mul_fast2(a1, b1, a2, b2, o.x, k1, o.y, k2);
    if (!(k1 && k2)) {
        if (!k1) o.x = mul_general(a1, b1);
        if (!k2) o.y = mul_general(a2, b2);
    }
    return o;
}
// x with its sign flipped when c (exact, as neg(): every limb's sign bit)
XB_DEV r4 neg_if(const r4& x, bool c) {
#ifdef __CUDA_ARCH__
    const int f = c ? (int)0x80000000 : 0;
    auto fl = [&](double v) { return __hiloint2double(__double2hiint(v) ^ f, __double2loint(v)); };
    return {fl(x.c0), fl(x.c1), fl(x.c2), fl(x.c3)};
#else
    return c ? neg(x) : x;
#endif
}
// One half of a complex product as ONE call: x1*y1 + (negate ? -(x2*y2) :
// x2*y2) -- the real part (negate) or the imaginary part of cmul
// (complex.hpp:41-44) with its operands chosen by the caller; the two
// products in lockstep, then the sum.  The lane-pair batched kernel's leaf
// and update (xpair.cuh): the products never cross a call boundary.
XB_DEV r4 hcmul_inl(const r4& x1, const r4& y1, const r4& x2, const r4& y2, const bool negate) {
    r4 p1, p2;
    bool k1, k2;
    mul_fast2(x1, y1, x2, y2, p1, k1, p2, k2);
    p2 = neg_if(p2, negate);
    bool ok;
    r4 r = add_fast_any(p1, p2, ok);
    if (!ok) r = add_slow(p1, p2);
    return r;
}
XB_CALL_IF r4 hcmul_r4(const r4 x1, const r4 y1, const r4 x2, const r4 y2, const bool negate) {
    return hcmul_inl(x1, y1, x2, y2, negate);
}
#if !(XB_CALLS & 4) || (XB_CALLS & 8) || (XB_CALLS & 16)
template <>
XB_DEV rpair<r4> add2<r4>(const r4& a1, const r4& b1, const r4& a2, const r4& b2) {
    return add2_r4(a1, b1, a2, b2);
}
#endif
#if !(XB_CALLS & 4) || (XB_CALLS & 16)
template <>
XB_DEV rpair<r4> mul2<r4>(const r4& a1, const r4& b1, const r4& a2, const r4& b2) {
    return mul2_r4(a1, b1, a2, b2);
}
#endif

template <class R>
XB_DEV cx<R> cadd_t(const cx<R>& a, const cx<R>& b) {  // complex.hpp:26-29
    rpair<R> o = add2(a.re, b.re, a.im, b.im);
    return {o.x, o.y};
}
template <class R>
XB_DEV cx<R> csub_t(const cx<R>& a, const cx<R>& b) {  // :31-34 (a - b = a + (-b))
    rpair<R> o = add2(a.re, neg(b.re), a.im, neg(b.im));
    return {o.x, o.y};
}
template <class R>
XB_DEV cx<R> csub(const cx<R>& a, const cx<R>& b) {
    return csub_t(a, b);
}
// complex.hpp:41-44: {a.re*b.re - a.im*b.im, a.re*b.im + a.im*b.re}; the four
// products are independent, then the two sums.
template <class R>
XB_DEV cx<R> cmul_t(const cx<R>& a, const cx<R>& b) {
    rpair<R> p = mul2(a.re, b.re, a.im, b.im);
    rpair<R> q = mul2(a.re, b.im, a.im, b.re);
    rpair<R> o = add2(p.x, neg(p.y), q.x, q.y);
    return {o.x, o.y};
}
#if !(XB_CALLS & 4)
// quad-double: all four products' fast paths, one branch, then the sums
template <>
XB_DEV cx<r4> cmul_t<r4>(const cx<r4>& a, const cx<r4>& b) {
    r4 p1, p2, p3, p4;
    bool k1, k2, k3, k4;
    mul_fast2(a.re, b.re, a.im, b.im, p1, k1, p2, k2);
    mul_fast2(a.re, b.im, a.im, b.re, p3, k3, p4, k4);
    if (!(k1 && k2 && k3 && k4)) {
        if (!k1) p1 = mul_general(a.re, b.re);
        if (!k2) p2 = mul_general(a.im, b.im);
        if (!k3) p3 = mul_general(a.re, b.im);
        if (!k4) p4 = mul_general(a.im, b.re);
    }
    rpair<r4> o = add2(p1, neg(p2), p3, p4);
    return {o.x, o.y};
}
#endif
template <class R>
XB_DEV cx<R> cadd(const cx<R>& a, const cx<R>& b) {
    return cadd_t(a, b);
}
template <class R>
XB_DEV cx<R> cmul(const cx<R>& a, const cx<R>& b) {
    return cmul_t(a, b);
}
// quad-double: overloads (preferred over the templates) that can be calls
XB_OP2 cx<r4> cadd(const cx<r4> a, const cx<r4> b) { return cadd_t(a, b); }
XB_OP2 cx<r4> cmul(const cx<r4> a, const cx<r4> b) { return cmul_t(a, b); }
template <class R>
XB_DEV cx<R> csub_t(const cx<R>& a, const cx<R>& b);
XB_OP2 cx<r4> csub(const cx<r4> a, const cx<r4> b) { return csub_t(a, b); }
// Re(conj(a) * b): the real half of cmul(cconj(a), b), same ops.
template <class R>
XB_DEV R cdot_re(const cx<R>& a, const cx<R>& b) {
    rpair<R> p = mul2(a.re, b.re, neg(a.im), b.im);
    return sub(p.x, p.y);
}
XB_OP2 r4 cdot_re(const cx<r4> a, const cx<r4> b) {
    rpair<r4> p = mul2(a.re, b.re, neg(a.im), b.im);
    return sub(p.x, p.y);
}
// {a.re / b, a.im / b} with b's reciprocal prefix hoisted (div_real,
// complex.hpp:61-65); the two tails interleave.
template <class R>
XB_DEV cx<R> cdivide_real(const cx<R>& a, const R& b, const recip_t<R>& rc) {
    return {divide(a.re, b, rc), divide(a.im, b, rc)};
}
// quad-double: q = a*x; q = q + x*(a - b*q) (quad_double.hpp:352-353) for
// both parts in lockstep
XB_OP2 cx<r4> cdivide_real(const cx<r4> a, const r4 b, const recip_t<r4> rc) {
    rpair<r4> q = mul2(a.re, rc.x, a.im, rc.x);
    rpair<r4> t = mul2(b, q.x, b, q.y);
    rpair<r4> d = add2(a.re, neg(t.x), a.im, neg(t.y));
    rpair<r4> u = mul2(rc.x, d.x, rc.x, d.y);
    rpair<r4> r = add2(q.x, u.x, q.y, u.y);
    return {r.x, r.y};
}

// Smith division (complex.hpp:47-58); status 3 on a zero divisor.
template <class R>
XB_DEV cx<R> cdiv(const cx<R>& a, const cx<R>& b, int& status) {
    if (is_zero(b.re) && is_zero(b.im)) {
        status = 3;
        return a;
    }
    if (ge(rabs(b.re), rabs(b.im))) {
        R t = rdiv(b.im, b.re, status);
        R d = add(b.re, mul(b.im, t));
        recip_t<R> rc = recip(d, status);
        return {divide(add(a.re, mul(a.im, t)), d, rc), divide(sub(a.im, mul(a.re, t)), d, rc)};
    }
    R t = rdiv(b.re, b.im, status);
    R d = add(mul(b.re, t), b.im);
    recip_t<R> rc = recip(d, status);
    return {divide(add(mul(a.re, t), a.im), d, rc), divide(sub(mul(a.im, t), a.re), d, rc)};
}

template <class R>
XB_DEV bool cfinite(const cx<R>& z) {
    return vfinite(z.re) && vfinite(z.im);
}

// ---- limb load / store with a plane stride ------------------------------------
template <int L>
using real_t = typename real_of<L>::type;

template <int L>
XB_DEV void load_real(const double* p, int stride, real_t<L>& v);
template <>
XB_DEV void load_real<1>(const double* p, int stride, r1& v) {
    v.c0 = p[0];
}
template <>
XB_DEV void load_real<2>(const double* p, int stride, r2& v) {
    v.c0 = p[0];
    v.c1 = p[stride];
}
template <>
XB_DEV void load_real<4>(const double* p, int stride, r4& v) {
    v.c0 = p[0];
    v.c1 = p[stride];
    v.c2 = p[2 * stride];
    v.c3 = p[3 * stride];
}
template <int L>
XB_DEV void store_real(double* p, int stride, const real_t<L>& v);
template <>
XB_DEV void store_real<1>(double* p, int stride, const r1& v) {
    p[0] = v.c0;
}
template <>
XB_DEV void store_real<2>(double* p, int stride, const r2& v) {
    p[0] = v.c0;
    p[stride] = v.c1;
}
template <>
XB_DEV void store_real<4>(double* p, int stride, const r4& v) {
    p[0] = v.c0;
    p[stride] = v.c1;
    p[2 * stride] = v.c2;
    p[3 * stride] = v.c3;
}

}  // namespace xb
