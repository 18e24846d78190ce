// Host-side CSR storage for the B200 BDDC solver.
// Mirrors the reference's CsrMatrix contract (include/bddc/csr_matrix.hpp:21-47):
// int32 offsets/cols, FP64 values, duplicates summed in input order by from_triplets.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

namespace bddc_b200 {

using index_t = std::int32_t;

struct Triplet {
    index_t row;
    index_t col;
    double value;
};

struct CsrMatrix {
    index_t nrows = 0;
    index_t ncols = 0;
    std::vector<index_t> row_offsets{0};
    std::vector<index_t> col_indices;
    std::vector<double> values;

    index_t nnz() const { return static_cast<index_t>(values.size()); }
    void validate() const;

    // Stable (row, col) sort; equal keys summed in input order
    // (reference src/csr_matrix.cpp:52-88 — same summation order, bit-identical).
    static CsrMatrix from_triplets(index_t nrows, index_t ncols, std::vector<Triplet> entries);
};

// y = A x, row-sequential in CSR column order (reference src/csr_matrix.cpp:90-102).
void spmv(const CsrMatrix& A, std::span<const double> x, std::span<double> y);

// Leading principal block (reference src/csr_matrix.cpp:134-151).
CsrMatrix principal_submatrix(const CsrMatrix& A, index_t size);

}  // namespace bddc_b200
