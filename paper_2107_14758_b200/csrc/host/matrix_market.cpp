// MatrixMarket export for debug dumps (src/sparse.cpp:33-52, write_matrix_market):
// coordinate real, general or symmetric (lower triangle only), 1-based
// indices, 17 significant digits, entries in column-major storage order as
// Eigen's compressed column-major SpMat iterates them.
#include <fstream>
#include <stdexcept>
#include <string>

#include "fdm_host.hpp"

namespace fdmgpu::host {

void write_matrix_market(const std::string& path, int64_t rows, int64_t cols, const int64_t* colptr,
                         const int32_t* rowidx, const double* val, bool symmetric) {
  std::ofstream os(path);
  if (!os) throw std::runtime_error("cannot open " + path);
  os << "%%MatrixMarket matrix coordinate real " << (symmetric ? "symmetric" : "general") << "\n";
  int64_t nnz = 0;
  for (int64_t c = 0; c < cols; ++c)
    for (int64_t q = colptr[c]; q < colptr[c + 1]; ++q)
      if (!symmetric || c <= rowidx[q]) ++nnz;
  os << rows << " " << cols << " " << nnz << "\n";
  os.precision(17);
  for (int64_t c = 0; c < cols; ++c)
    for (int64_t q = colptr[c]; q < colptr[c + 1]; ++q)
      if (!symmetric || c <= rowidx[q]) os << rowidx[q] + 1 << " " << c + 1 << " " << val[q] << "\n";
  if (!os) throw std::runtime_error("cannot write " + path);
}

}  // namespace fdmgpu::host
