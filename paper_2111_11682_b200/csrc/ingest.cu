// Host-side data preparation that the reference runs as a Python loop (SURVEY §8(f)
// #3): the deterministic holdout split.  Plain C++ on host memory (no device work):
// the decision for each entry depends on every earlier decision in the permutation
// order, and a tight native loop does 100M entries in well under a second where the
// reference's interpreted loop (data.py:330-339) takes minutes.
#include <cstdint>
#include <vector>

#include "common.cuh"

// data.py:312-346 split_holdout core.  perm: the numpy PCG64 permutation of [0, nnz)
// drawn by the caller (the reference's own stream); entry e goes to the test side while
// fewer than n_test are taken and its row and column both keep >= 1 training entry.
// in_test (nnz bytes) is written 0/1; returns the number taken (>= 0) or an error code.
extern "C" int64_t culsh_split_holdout(const int32_t *entry_rows, const int32_t *entry_cols, int64_t nnz,
                                       int64_t M, int64_t N, const int64_t *perm, int64_t n_test,
                                       uint8_t *in_test) {
    CULSH_REQUIRE(nnz >= 0 && M >= 0 && N >= 0 && n_test >= 0 && n_test <= nnz, "bad split arguments");
    std::vector<int64_t> rc((size_t)M, 0), cc((size_t)N, 0);
    for (int64_t e = 0; e < nnz; ++e) {
        const int32_t i = entry_rows[e], j = entry_cols[e];
        CULSH_REQUIRE(i >= 0 && i < M && j >= 0 && j < N, "entry index out of range");
        ++rc[(size_t)i];
        ++cc[(size_t)j];
        in_test[e] = 0;
    }
    int64_t taken = 0;
    for (int64_t t = 0; t < nnz && taken < n_test; ++t) {
        const int64_t e = perm[t];
        CULSH_REQUIRE(e >= 0 && e < nnz, "permutation entry out of range");
        const int32_t i = entry_rows[e], j = entry_cols[e];
        if (rc[(size_t)i] > 1 && cc[(size_t)j] > 1) {
            in_test[e] = 1;
            --rc[(size_t)i];
            --cc[(size_t)j];
            ++taken;
        }
    }
    return taken;
}
