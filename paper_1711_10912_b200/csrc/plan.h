// plan.h -- host-side canonicalisation of a contraction (C++ only).
//
// The reference recurses over dimensions by index (contraction.py:134-194,
// 230-298).  Here a dense tensor of any permutation layout is reduced to
// A[O][K][I]:
//   K = extent of the contracted mode m, I = its stride w_m (= product of
//   the extents that precede m in storage precedence, layout.py:113-128),
//   O = N / (K I).
// The free dimensions split into an inner block (stride < w_m) and an outer
// block (stride > w_m), each a mixed-radix number in storage order.  The
// output is always dense first-order (contraction.py:9-12), so the output
// offset of (o, i) is g(o) + f(i) with f, g digit maps over the output's
// first-order strides.  Adjacent digits that are contiguous in both A and
// the output are merged, so first-order inputs collapse to out = o*I + i.
#pragma once

#include <algorithm>
#include <cstdint>
#include <utility>
#include <vector>

#include "tl_common.cuh"

namespace tl {

using DigitList = std::vector<std::pair<int64_t, int64_t>>;  // (extent, output stride)

// Dims sorted by stride (extent-1 dims dropped).  Returns true iff the
// tensor is dense: sorted strides are 1, n_1, n_1 n_2, ... (a permutation
// layout with its derived strides; views and gaps are not dense).
inline bool dense_order(const tl_desc &d, std::vector<int> &dims) {
    dims.clear();
    for (int r = 0; r < d.order; ++r)
        if (d.extent[r] > 1) dims.push_back(r);
    std::stable_sort(dims.begin(), dims.end(), [&](int x, int y) { return d.stride[x] < d.stride[y]; });
    int64_t run = 1;
    for (int r : dims) {
        if (d.stride[r] != run) return false;
        run *= d.extent[r];
    }
    return true;
}

inline int64_t volume(const tl_desc &d) {
    int64_t v = 1;
    for (int r = 0; r < d.order; ++r) v *= d.extent[r];
    return v;
}

inline DigitList collapse(const DigitList &in) {
    DigitList out;
    for (auto &dg : in) {
        if (dg.first == 1) continue;
        if (!out.empty() && out.back().second * out.back().first == dg.second) {
            out.back().first *= dg.first;
        } else {
            out.push_back(dg);
        }
    }
    return out;
}

inline bool build_map(const DigitList &dl, DigitMap &m) {
    m.n = (int32_t)dl.size();
    for (size_t d = 0; d < dl.size(); ++d) {
        if (dl[d].first > 0xffffffffll) return false;
        m.div[d].init((uint32_t)dl[d].first);
        m.stride[d] = dl[d].second;
    }
    return true;
}

inline void build_map64(const DigitList &dl, DigitMap64 &m) {
    m.n = (int32_t)dl.size();
    for (size_t d = 0; d < dl.size(); ++d) {
        m.ext[d] = dl[d].first;
        m.stride[d] = dl[d].second;
    }
}

constexpr int64_t kIdx32 = 0xffffffffll;  // largest index the 32-bit digit maps take

struct Canon {
    int64_t O = 1, K = 1, I = 1;
    int64_t jstride = 0;  // ttm: output stride of the new mode's index j
    DigitList inner, outer;
    bool ident = false;  // output offset == o*I + i (ttv) / o*J*I + j*I + i (ttm)
};

// Canonicalise a contraction over mode m0 (zero-based) of dense `a`.  The
// output is first-order over `a`'s dimensions with the mode dropped (ttv,
// J == 0) or replaced by extent J (ttm).
inline bool canon_contraction(const tl_desc &a, int m0, int64_t J, Canon &c) {
    std::vector<int> dims;
    if (!dense_order(a, dims)) return false;
    const int p = a.order;
    // first-order output strides over the output's dimensions
    int64_t ostr[TL_MAX_ORDER];
    int64_t run = 1;
    for (int r = 0; r < p; ++r) {
        if (r == m0) {
            if (J > 0) {
                ostr[r] = run;
                run *= J;
            } else {
                ostr[r] = 0;
            }
            continue;
        }
        ostr[r] = run;
        run *= a.extent[r];
    }
    c.K = a.extent[m0];
    c.jstride = (J > 0) ? ostr[m0] : 0;
    c.inner.clear();
    c.outer.clear();
    if (c.K == 1) {
        // extent-1 mode: no contracted stride; every free dim is "inner"
        for (int r : dims) c.inner.push_back({a.extent[r], ostr[r]});
        c.I = 1;
        for (auto &dg : c.inner) c.I *= dg.first;
        c.O = 1;
    } else {
        const int64_t wm = a.stride[m0];
        for (int r : dims) {
            if (r == m0) continue;
            if (a.stride[r] < wm)
                c.inner.push_back({a.extent[r], ostr[r]});
            else
                c.outer.push_back({a.extent[r], ostr[r]});
        }
        c.I = wm;
        c.O = volume(a) / (c.K * c.I);
    }
    c.inner = collapse(c.inner);
    c.outer = collapse(c.outer);
    // identity output map?
    const int64_t ostep = (J > 0) ? J * c.I : c.I;  // output stride of o in the ident layout
    bool in_ok = c.inner.empty() || (c.inner.size() == 1 && c.inner[0].second == 1);
    bool out_ok = c.outer.empty() || (c.outer.size() == 1 && c.outer[0].second == ostep);
    bool j_ok = (J == 0) || c.jstride == c.I;
    c.ident = in_ok && out_ok && j_ok;
    return true;
}

}  // namespace tl
