// xpair.cuh -- warp-level column primitives with a LANE PAIR per row group,
// for the CTA-per-system MGS kernel (xmgs.cuh) on quad-double batches.
//
// The same decomposition as xcolumn.cuh's one-lane-per-row-group primitives
// (a column task = one warp, the fixed tree of reduction.hpp:34-40 split into
// in-lane levels and shuffle levels), but every complex quantity is split
// over the two lanes of a pair: the even lane computes the real part, the
// odd lane the imaginary part (complex.hpp:41-44: the two halves of a
// complex multiply or add are independent).  Per lane, a complex multiply
// is then two real quad-double products and one sum instead of four and
// two, so a lane holds half the state (more warps fit an SM), and the
// shuffle levels of the tree over 16 pairs are four half-width additions
// instead of five full complex ones.
//
// Memory layout of a column ("pair-interleaved planar"): plane p = part*L +
// limb; in a plane, row r = pi*RPP + t (pi = pair 0..15, RPP = rows per
// pair) lives at t*16 + pi.  Both lanes of a pair load the same complex row
// (a warp load of one (plane, t) reads 16 consecutive doubles, broadcast to
// the pair); each lane stores only its own half.
//
// Bit-exactness: the leaf of q^H a is the reference's cmul(conj(q), a) half
// by half with the reference's operand order (complex.hpp:41-44, conj :21-24),
// the update a - r*q is cmul(r, q) then the subtraction (mgs.hpp:59), the
// tree pairs rows exactly as tree_reduce, and the division by r_kk is the
// reference's per-part division (div_real, complex.hpp:61-65).
#pragma once
#include "xcolumn.cuh"

namespace xb {

#ifndef XB_PAIR_PREFETCH
#define XB_PAIR_PREFETCH 0
#endif
// prefetch each column task's column into L1 at the start of the task
#ifndef XB_PAIR_L1PF
#define XB_PAIR_L1PF 1
#endif
// leaf / update as one call each (hcmul_r4: both products and their sum)
#ifndef XB_PAIR_HCMUL
#define XB_PAIR_HCMUL 1
#endif

template <int L>
struct pairfmt {
    int rpp, LD, COL;
    XB_DEVICE explicit pairfmt(int rows_per_pair)
        : rpp(rows_per_pair), LD(16 * rows_per_pair), COL(2 * L * 16 * rows_per_pair) {}
    XB_DEVICE static int off(int t, int pi) { return t * 16 + pi; }
    XB_DEVICE int row_off(int row) const { return (row % rpp) * 16 + row / rpp; }
    XB_DEVICE cx<real_t<L>> load(const double* col, int t, int pi) const {
        cx<real_t<L>> z;
        load_real<L>(col + off(t, pi), LD, z.re);
        load_real<L>(col + L * LD + off(t, pi), LD, z.im);
        return z;
    }
    XB_DEVICE real_t<L> load_part(const double* col, int t, int pi, int part) const {
        real_t<L> v;
        load_real<L>(col + part * L * LD + off(t, pi), LD, v);
        return v;
    }
    XB_DEVICE void store_part(double* col, int t, int pi, int part, const real_t<L>& v) const {
        store_real<L>(col + part * L * LD + off(t, pi), LD, v);
    }
};

// In-lane part of the fixed tree with ONE addition site: leaves are pushed on
// a shift stack (top = the most recent, smallest partial); leaf t is merged
// with the top as many times as t has trailing one bits (tree_reduce's
// pairing, reduction.hpp:34-40), the earlier partial always the left
// operand; a partial last group folds its stack from the top down (the
// skipped partners).  Depth: rows per pair <= 8 (three partials).
template <class R, class LeafFn, class AddFn>
XB_DEVICE R pair_lane_tree(int cnt, LeafFn leaf, AddFn addf) {
    R st0{}, st1{}, st2{};
    int depth = 0;
#pragma unroll 1
    for (int t = 0; t < cnt; ++t) {
        R v = leaf(t);
        const int nm = __ffs(~t) - 1;  // trailing ones of t (warp-uniform)
#pragma unroll 1
        for (int l = 0; l < nm; ++l) {
            v = addf(st0, v);
            st0 = st1;
            st1 = st2;
            --depth;
        }
        st2 = st1;
        st1 = st0;
        st0 = v;
        ++depth;
    }
    R acc = st0;
#pragma unroll 1
    for (int l = 1; l < depth; ++l) {
        st0 = st1;
        st1 = st2;
        acc = addf(st0, acc);
    }
    return acc;
}

template <int L>
struct mgs_pair {
    static constexpr int LIMBS = L;
    using R = real_t<L>;
    using C = cx<R>;
    using F = pairfmt<L>;

    XB_DEVICE static int pair_rows(int pi, int m, int rpp) {
        int c = m - pi * rpp;
        return c < 0 ? 0 : (c > rpp ? rpp : c);
    }
    // the shared addition of the tree levels (a real call: one hot copy)
    XB_DEVICE static R tadd(const R& a, const R& b) { return addc(a, b); }
    XB_DEVICE static R tsub(const R& a, const R& b) { return addc(a, neg(b)); }  // sub (quad_double.hpp:263)
    // x1*y1 - x2*y2 (negate) or x1*y1 + x2*y2: a half of a complex product
    XB_DEVICE static R hcmul(const R& x1, const R& y1, const R& x2, const R& y2, bool negate) {
        if constexpr (L == 4) {
            return hcmul_r4(x1, y1, x2, y2, negate);
        } else {
            const rpair<R> pr = mul2(x1, y1, x2, y2);
            return add(pr.x, negate ? neg(pr.y) : pr.y);
        }
    }

    // Cross-pair levels: strides RPP, 2RPP, ... as shuffle offsets 2, 4, 8, 16.
    XB_DEVICE static R pair_tree(R acc, int lane, int m, int rpp) {
        const int pi = lane >> 1;
#pragma unroll 1
        for (int s = 1; s < 16; s <<= 1) {
            R other = shfl_down_r(acc, 2 * s);
            if ((pi & (2 * s - 1)) == 0 && (pi + s) * rpp < m) acc = tadd(acc, other);
        }
        return acc;
    }

    // Re(a^H a) (mgs.hpp:38-42, reduction.hpp:45-51): both lanes of a pair
    // compute the same value; result broadcast to every lane.
    XB_DEVICE static R col_sq(const F& f, const double* col, int lane, int m) {
        const int pi = lane >> 1;
        const int cnt = pair_rows(pi, m, f.rpp);
        R acc = pair_lane_tree<R>(cnt, [&](int t) {
            C a = f.load(col, t, pi);
            return cdot_re(a, a);
        }, [](const R& x, const R& y) { return tadd(x, y); });
        acc = pair_tree(acc, lane, m, f.rpp);
        return shfl_idx_r(acc, 0);
    }

    // q^H a over the fixed tree; every lane returns the full complex value.
    XB_DEVICE static C dot(const F& f, const double* q, const double* col, int lane, int m) {
        const int pi = lane >> 1, part = lane & 1;
        const int cnt = pair_rows(pi, m, f.rpp);
        // the next row of a is loaded while this row's leaf is computed (the
        // column streams from L2 / HBM; q sits in shared memory)
#if XB_PAIR_HCMUL
        // y1 = part ? a.im : a.re, y2 = part ? a.re : a.im: swapped plane pointers
        const double* c1 = col + part * L * f.LD;
        const double* c2 = col + (1 - part) * L * f.LD;
        R acc = pair_lane_tree<R>(cnt, [&](int t) {
            const C qq = f.load(q, t, pi);
            R y1, y2;
            load_real<L>(c1 + F::off(t, pi), f.LD, y1);
            load_real<L>(c2 + F::off(t, pi), f.LD, y2);
            // this lane's half of cmul(conj(q), a) (complex.hpp:21-24, :41-44)
            return hcmul(qq.re, y1, neg(qq.im), y2, part == 0);
        }, [](const R& x, const R& y) { return tadd(x, y); });
#else
        C an = (XB_PAIR_PREFETCH && cnt > 0) ? f.load(col, 0, pi) : C{};
        R acc = pair_lane_tree<R>(cnt, [&](int t) {
            const C a = XB_PAIR_PREFETCH ? an : f.load(col, t, pi);
            if (XB_PAIR_PREFETCH && t + 1 < cnt) an = f.load(col, t + 1, pi);
            const C qq = f.load(q, t, pi);
            // this lane's half of cmul(conj(q), a) (complex.hpp:21-24, :41-44)
            const R y1 = part ? a.im : a.re, y2 = part ? a.re : a.im;
            const rpair<R> pr = mul2(qq.re, y1, neg(qq.im), y2);
            return add(pr.x, part ? pr.y : neg(pr.y));
        }, [](const R& x, const R& y) { return tadd(x, y); });
#endif
        acc = pair_tree(acc, lane, m, f.rpp);
        const R rh = shfl_idx_r(acc, lane & 1);  // pair 0: lane 0 = re, lane 1 = im
        const R ro = shfl_xor_r(rh, 1);
        return C{part ? ro : rh, part ? rh : ro};
    }


    // Pull a whole column into L1 ahead of its row-by-row use (it streams
    // from L2 / HBM; the rows' loads then wait on one latency, not one per
    // row): 128-byte lines, two per lane for a 128-row quad-double column.
    XB_DEVICE static void prefetch_col(const F& f, const double* col, int lane) {
#if XB_PAIR_L1PF
        const int lines = (f.COL * 8) / 128;
#pragma unroll 1
        for (int i = lane; i < lines; i += 32)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(col + i * 16));
#endif
    }

    // remove_projection (mgs.hpp:57-61): r = q^H a; a_i -= r * q_i.
    XB_DEVICE static bool remove_projection(const F& f, const double* q, double* col, int lane, int m, C& r) {
        prefetch_col(f, col, lane);
        r = dot(f, q, col, lane, m);
        const int pi = lane >> 1, part = lane & 1;
        bool ok = cfinite(r);
        const int cnt = pair_rows(pi, m, f.rpp);
#if XB_PAIR_HCMUL
        {
            const double* q1p = q + part * L * f.LD;        // y1 = part ? q.im : q.re
            const double* q2p = q + (1 - part) * L * f.LD;  // y2 = part ? q.re : q.im
#pragma unroll 1
            for (int t = 0; t < cnt; ++t) {
                R y1, y2;
                load_real<L>(q1p + F::off(t, pi), f.LD, y1);
                load_real<L>(q2p + F::off(t, pi), f.LD, y2);
                const R tt = hcmul(r.re, y1, r.im, y2, part == 0);  // this half of cmul(r, q_i)
                const R v = tsub(f.load_part(col, t, pi, part), tt);
                ok = ok && vfinite(v);
                f.store_part(col, t, pi, part, v);
            }
            return __all_sync(0xffffffffu, ok);
        }
#endif
        R an = (XB_PAIR_PREFETCH && cnt > 0) ? f.load_part(col, 0, pi, part) : R{};
#pragma unroll 1
        for (int t = 0; t < cnt; ++t) {
            const R a = XB_PAIR_PREFETCH ? an : f.load_part(col, t, pi, part);
            if (XB_PAIR_PREFETCH && t + 1 < cnt) an = f.load_part(col, t + 1, pi, part);  // next row, in flight
            const C qq = f.load(q, t, pi);
            const R y1 = part ? qq.im : qq.re, y2 = part ? qq.re : qq.im;
            const rpair<R> pr = mul2(r.re, y1, r.im, y2);  // this half of cmul(r, q_i)
            const R tt = add(pr.x, part ? pr.y : neg(pr.y));
            const R v = sub(a, tt);
            ok = ok && vfinite(v);
            f.store_part(col, t, pi, part, v);
        }
        return __all_sync(0xffffffffu, ok);
    }

    // normalize_column (mgs.hpp:46-53) into col and the shared pivot slot.
    // code: 0 ok, 1 breakdown, 2 overflow, 3 domain.
    XB_DEVICE static int normalize(const F& f, double* col, double* slot, const R& thr, int lane, int m, R& rkk) {
        R s = col_sq(f, col, lane, m);
        rkk = rsqrt_ref(s);
        if (!vfinite(s) || !vfinite(rkk)) return 2;
        if (le(rkk, thr)) return 1;
        int st = 0;
        recip_t<R> rc = recip(rkk, st);
        if (st) return st;
        const int pi = lane >> 1, part = lane & 1;
        const int cnt = pair_rows(pi, m, f.rpp);
        bool ok = true;
#pragma unroll 1
        for (int t = 0; t < cnt; ++t) {
            const R v = divide(f.load_part(col, t, pi, part), rkk, rc);  // div_real, complex.hpp:61-65
            ok = ok && vfinite(v);
            f.store_part(col, t, pi, part, v);
            f.store_part(slot, t, pi, part, v);
        }
        return __all_sync(0xffffffffu, ok) ? 0 : 2;
    }
};

}  // namespace xb
