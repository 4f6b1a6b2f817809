// xcolumn.cuh -- warp-level column primitives for MGS on sm_100a.
//
// One warp owns one column task.  Lane `l` owns RPL *consecutive* rows
// [l*RPL, l*RPL + RPL) so the reference's fixed pairwise tree
// (reduction.hpp:34-40: stride s = 1, 2, 4, ...; t[i] += t[i+s] for i a
// multiple of 2s, missing partners skipped) splits into
//   * strides < RPL inside the lane (binary-counter stack, compile-time
//     unrolled, a partial last lane folds its stack right-to-left), and
//   * strides >= RPL across lanes with __shfl_down_sync offsets 1, 2, 4, ...
// which reproduces tree_reduce bit for bit for every m.
//
// Memory layout of a column ("lane-interleaved planar"): plane p = part*L +
// limb (part 0 = re, 1 = im); inside a plane, row r = l*RPL + t lives at
// t*32 + l.  A warp load of (plane, t) therefore reads 32 consecutive
// doubles (256 B, fully coalesced), and shared-memory pivot reads are
// bank-conflict free, while each lane still holds consecutive rows.
#pragma once
#include "xarith.cuh"

namespace xb {

// Column addressing: plane stride LD = 32*rpl doubles, column = 2L planes.
// rpl (rows per lane) is a runtime power of two.
template <int L>
struct colfmt {
    int rpl, LD, COL;
    XB_DEVICE colfmt(int rows_per_lane) : rpl(rows_per_lane), LD(32 * rows_per_lane), COL(2 * L * 32 * rows_per_lane) {}
    XB_DEVICE static int off(int t, int lane) { return t * 32 + lane; }
    XB_DEVICE cx<real_t<L>> load(const double* col, int t, int lane) const {
        cx<real_t<L>> z;
        load_real<L>(col + off(t, lane), LD, z.re);
        load_real<L>(col + L * LD + off(t, lane), LD, z.im);
        return z;
    }
    XB_DEVICE void store(double* col, int t, int lane, const cx<real_t<L>>& z) const {
        store_real<L>(col + off(t, lane), LD, z.re);
        store_real<L>(col + L * LD + off(t, lane), LD, z.im);
    }
    // row index -> offset inside a plane
    XB_DEVICE int row_off(int row) const { return (row % rpl) * 32 + row / rpl; }
};

template <class R>
XB_DEVICE cx<R> shfl_down(const cx<R>& v, int o);
template <class R>
XB_DEVICE R shfl_down_r(const R& v, int o);
template <>
XB_DEVICE r1 shfl_down_r<r1>(const r1& v, int o) {
    return {__shfl_down_sync(0xffffffffu, v.c0, o)};
}
template <>
XB_DEVICE r2 shfl_down_r<r2>(const r2& v, int o) {
    return {__shfl_down_sync(0xffffffffu, v.c0, o), __shfl_down_sync(0xffffffffu, v.c1, o)};
}
template <>
XB_DEVICE r4 shfl_down_r<r4>(const r4& v, int o) {
    return {__shfl_down_sync(0xffffffffu, v.c0, o), __shfl_down_sync(0xffffffffu, v.c1, o),
            __shfl_down_sync(0xffffffffu, v.c2, o), __shfl_down_sync(0xffffffffu, v.c3, o)};
}
template <class R>
XB_DEVICE R shfl_idx_r(const R& v, int src);
template <>
XB_DEVICE r1 shfl_idx_r<r1>(const r1& v, int s) {
    return {__shfl_sync(0xffffffffu, v.c0, s)};
}
template <>
XB_DEVICE r2 shfl_idx_r<r2>(const r2& v, int s) {
    return {__shfl_sync(0xffffffffu, v.c0, s), __shfl_sync(0xffffffffu, v.c1, s)};
}
template <>
XB_DEVICE r4 shfl_idx_r<r4>(const r4& v, int s) {
    return {__shfl_sync(0xffffffffu, v.c0, s), __shfl_sync(0xffffffffu, v.c1, s),
            __shfl_sync(0xffffffffu, v.c2, s), __shfl_sync(0xffffffffu, v.c3, s)};
}
template <class R>
XB_DEVICE R shfl_xor_r(const R& v, int m);
template <>
XB_DEVICE r1 shfl_xor_r<r1>(const r1& v, int m) {
    return {__shfl_xor_sync(0xffffffffu, v.c0, m)};
}
template <>
XB_DEVICE r2 shfl_xor_r<r2>(const r2& v, int m) {
    return {__shfl_xor_sync(0xffffffffu, v.c0, m), __shfl_xor_sync(0xffffffffu, v.c1, m)};
}
template <>
XB_DEVICE r4 shfl_xor_r<r4>(const r4& v, int m) {
    return {__shfl_xor_sync(0xffffffffu, v.c0, m), __shfl_xor_sync(0xffffffffu, v.c1, m),
            __shfl_xor_sync(0xffffffffu, v.c2, m), __shfl_xor_sync(0xffffffffu, v.c3, m)};
}
// partner exchange inside a lane pair whose lanes may run without the rest
// of the warp: mask = the two lanes only
XB_DEVICE r1 shfl_pair(const r1& v, unsigned mask) { return {__shfl_xor_sync(mask, v.c0, 1)}; }
XB_DEVICE r2 shfl_pair(const r2& v, unsigned mask) {
    return {__shfl_xor_sync(mask, v.c0, 1), __shfl_xor_sync(mask, v.c1, 1)};
}
XB_DEVICE r4 shfl_pair(const r4& v, unsigned mask) {
    return {__shfl_xor_sync(mask, v.c0, 1), __shfl_xor_sync(mask, v.c1, 1),
            __shfl_xor_sync(mask, v.c2, 1), __shfl_xor_sync(mask, v.c3, 1)};
}
template <class R>
XB_DEVICE cx<R> shfl_down_c(const cx<R>& v, int o) {
    return {shfl_down_r(v.re, o), shfl_down_r(v.im, o)};
}
template <class R>
XB_DEVICE cx<R> shfl_idx_c(const cx<R>& v, int s) {
    return {shfl_idx_r(v.re, s), shfl_idx_r(v.im, s)};
}

template <class R>
XB_DEVICE R vadd(const R& a, const R& b) {
    return add(a, b);
}
template <class R>
XB_DEVICE cx<R> vadd(const cx<R>& a, const cx<R>& b) {
    return cadd(a, b);
}
template <class R>
XB_DEVICE R vshfl_down(const R& v, int o) {
    return shfl_down_r(v, o);
}
template <class R>
XB_DEVICE cx<R> vshfl_down(const cx<R>& v, int o) {
    return shfl_down_c(v, o);
}

// In-lane part of the fixed tree.  Leaf t (row lane*rpl + t) is produced by
// leaf(t) for t = 0..cnt-1 (cnt = valid rows of this lane, rpl >= cnt).  A
// binary-counter stack of depth LV (rpl <= 2^(LV-1)) merges leaves exactly as
// tree_reduce pairs them; merge decisions depend only on t (warp-uniform), so
// the code holds one leaf and LV adds however large rpl is.  A partial lane
// folds its stack right to left, i.e. tree_reduce's skipped partners.
template <int LV, int l, class V>
struct counter_merge {
    XB_DEVICE static void push(V (&st)[LV], V v, int t) {
        if ((t >> l) & 1) {
            v = vadd(st[l], v);
            counter_merge<LV, l + 1, V>::push(st, v, t);
        } else {
            st[l] = v;
        }
    }
};
template <int LV, class V>
struct counter_merge<LV, LV, V> {
    XB_DEVICE static void push(V (&)[LV], V, int) {}
};

template <int LV, class V, class LeafFn>
XB_DEVICE V lane_tree(int cnt, LeafFn leaf) {
    V st[LV];
#pragma unroll 1
    for (int t = 0; t < cnt; ++t) counter_merge<LV, 0, V>::push(st, leaf(t), t);
    V acc = st[0];
    bool have = false;
#pragma unroll
    for (int l = 0; l < LV; ++l) {
        if ((cnt >> l) & 1) {
            if (!have) {
                acc = st[l];
                have = true;
            } else {
                acc = vadd(st[l], acc);
            }
        }
    }
    return acc;
}

// Cross-lane levels: strides RPL, 2RPL, ... as shuffle offsets 1, 2, 4, ...
// Lane 0 ends with the total; every lane returns it (broadcast).
template <class V>
XB_DEVICE V warp_tree(V acc, int lane, int m, int rpl) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        V other = vshfl_down(acc, o);
        if (((lane & (2 * o - 1)) == 0) && ((lane + o) * rpl < m)) acc = vadd(acc, other);
    }
    return acc;
}

}  // namespace xb
