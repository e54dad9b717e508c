// Percolation (winding) check of a periodic voxel mask along one axis.
//
// BASELINE's configs keep "the fluid component percolating in x".  On a
// periodic box a component percolates along `axis` iff it contains a closed
// path whose unwrapped displacement along that axis is a non-zero multiple
// of n.  The reference has no such check (its connected_components,
// geometry.py:183-222, merges components across opposite boundary layers
// with a union-find but carries no displacement); SURVEY Appendix B-3
// prescribes carrying the offset, which is what this does: a union-find over
// the fluid cells in which every cell stores its unwrapped coordinate along
// `axis` relative to its root.  Every face bond (c, c + e_a) adds the
// constraint pot(c + e_a) - pot(c) = [a == axis] (the wrap bond n-1 -> 0
// included: unwrapped, it is still one step forward).  A bond inside one
// tree whose constraint is violated closes a loop of non-zero winding.
//
// Output per mask: the number of periodic components and how many of them
// wind.  Host C++, one pass over the cells in row-major order; int32 parent
// and potential per cell (8 B/cell: 1 GB at 512^3).
#include <cstdint>
#include <new>
#include <string>
#include <vector>

#include "../../include/voxschur.h"

namespace vs {
void set_last_error(const std::string &msg);
}

namespace {

struct WeightedForest {
    std::vector<int32_t> parent, pot;  // pot[c] = x(c) - x(parent[c]) (unwrapped)

    // root of c; on return *p = x(c) - x(root); compresses the path
    int32_t find(int32_t c, int32_t *p) {
        int32_t r = c, acc = 0;
        while (parent[r] != r) {
            acc += pot[r];
            r = parent[r];
        }
        *p = acc;
        // second pass: point everything at the root with its full potential
        int32_t cur = c, rem = acc;
        while (parent[cur] != r && cur != r) {
            const int32_t nxt = parent[cur], step = pot[cur];
            parent[cur] = r;
            pot[cur] = rem;
            rem -= step;
            cur = nxt;
        }
        return r;
    }
};

}  // namespace

extern "C" int vs_winding(const uint8_t *fluid, int dim, int n, int axis, int64_t *n_components,
                          int64_t *n_winding) {
    if ((dim != 2 && dim != 3) || n < 1) {
        vs::set_last_error("grid dimension must be 2 or 3, got " + std::to_string(dim));
        return VS_EVALUE;
    }
    if (axis < 0 || axis >= dim) {
        vs::set_last_error("axis " + std::to_string(axis) + " out of range for a " + std::to_string(dim) + "D grid");
        return VS_EVALUE;
    }
    const int64_t N = dim == 3 ? (int64_t)n * n * n : (int64_t)n * n;
    if (N >= ((int64_t)1 << 31)) {
        vs::set_last_error("grid of " + std::to_string(N) + " cells exceeds the int32 labelling");
        return VS_EVALUE;
    }
    try {
        WeightedForest f;
        f.parent.resize(N);
        f.pot.assign(N, 0);
        for (int64_t c = 0; c < N; ++c) f.parent[c] = (int32_t)c;
        std::vector<uint8_t> winds(N, 0);  // meaningful at roots
        int64_t stride[3];
        stride[dim - 1] = 1;
        for (int a = dim - 2; a >= 0; --a) stride[a] = stride[a + 1] * n;
        int idx[3] = {0, 0, 0};
        for (int64_t c = 0; c < N; ++c) {
            if (fluid[c]) {
                for (int a = 0; a < dim; ++a) {
                    const int64_t nb = idx[a] + 1 < n ? c + stride[a] : c - (int64_t)(n - 1) * stride[a];
                    if (!fluid[nb]) continue;
                    const int32_t delta = a == axis ? 1 : 0;
                    int32_t pc, pn;
                    const int32_t rc = f.find((int32_t)c, &pc), rn = f.find((int32_t)nb, &pn);
                    if (rc == rn) {
                        if (pn - pc != delta) winds[rc] = 1;
                    } else {
                        // hang the larger index under the smaller: x(rn) - x(rc) = pc + delta - pn
                        const int32_t d = pc + delta - pn;
                        if (rc < rn) {
                            f.parent[rn] = rc;
                            f.pot[rn] = d;
                            winds[rc] |= winds[rn];
                        } else {
                            f.parent[rc] = rn;
                            f.pot[rc] = -d;
                            winds[rn] |= winds[rc];
                        }
                    }
                }
            }
            for (int a = dim - 1; a >= 0; --a) {
                if (++idx[a] < n) break;
                idx[a] = 0;
            }
        }
        int64_t nc = 0, nw = 0;
        for (int64_t c = 0; c < N; ++c)
            if (fluid[c] && f.parent[c] == (int32_t)c) {
                ++nc;
                nw += winds[c];
            }
        if (n_components) *n_components = nc;
        if (n_winding) *n_winding = nw;
    } catch (const std::bad_alloc &) {
        vs::set_last_error("host allocation failed");
        return VS_ECUDA;
    }
    return VS_OK;
}
