// Triplet text I/O of the input side (P/include/dfc/matrix_io.hpp:22-26,125-179); see triplet_io.cpp.
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>
#include <vector>

namespace dfcg {

// matrix_io.hpp:22-26
struct ParseError : std::runtime_error {
  ParseError(std::size_t line, const std::string& what)
      : std::runtime_error("line " + std::to_string(line) + ": " + what), line(line) {}
  std::size_t line;
};

struct TripletFile {
  long long m = 0, n = 0;
  std::vector<long long> row, col;  // column-major order, duplicates rejected
  std::vector<double> val;
};

TripletFile load_triplets_text(const char* text, std::size_t len, bool one_based);
TripletFile load_triplets_file(const std::string& path, bool one_based);
// "% m n\n" then "row col %.17g\n" per entry (save_triplets, matrix_io.hpp:172-179)
std::string format_triplets(long long m, long long n, std::size_t N, const long long* row, const long long* col,
                            const double* val);
void save_triplets_file(const std::string& path, long long m, long long n, std::size_t N, const long long* row,
                        const long long* col, const double* val);

// The ObservedMatrix constructor's ordering (matrix_io.hpp:41-43) for in-range triplets, in
// parallel: counting sort on the column, rows sorted within each column.
void sort_column_major(long long m, long long n, std::vector<long long>& row, std::vector<long long>& col,
                       std::vector<double>& val);
void reject_duplicates(const std::vector<long long>& row, const std::vector<long long>& col);

}  // namespace dfcg
