// Host-only check of cgvariants/matrix_market.hpp (no GPU): parses a Matrix
// Market file and prints "n nnz hash" (FNV-1a over the row_ptr, col_idx and
// value bits) or "error <code>", and with --roundtrip re-parses its own
// write_matrix_market output and demands identical arrays. Driven by
// tests/test_matrix_market.py against the reference parser's output.
#include "cgvariants/matrix_market.hpp"

#include <cstdint>
#include <cstring>
#include <iostream>

namespace {
std::uint64_t fnv(const void* p, std::size_t n, std::uint64_t h) {
    const auto* b = static_cast<const unsigned char*>(p);
    for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}
std::uint64_t hash(const cgv::SparseMatrix& a) {
    std::uint64_t h = 1469598103934665603ull;
    h = fnv(a.row_ptr.data(), a.row_ptr.size() * sizeof(cgv::Index), h);
    h = fnv(a.col_idx.data(), a.col_idx.size() * sizeof(cgv::Index), h);
    return fnv(a.values.data(), a.values.size() * sizeof(double), h);
}
}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "usage: mtx_tool file.mtx [--roundtrip]\n";
        return 2;
    }
    try {
        const cgv::SparseMatrix a = cgv::read_matrix_market_file(argv[1]);
        if (argc > 2 && std::strcmp(argv[2], "--roundtrip") == 0) {
            const cgv::SparseMatrix b = cgv::parse_matrix_market(cgv::write_matrix_market(a));
            if (hash(a) != hash(b) || a.n != b.n) {
                std::cout << "roundtrip-mismatch\n";
                return 1;
            }
        }
        std::cout << a.n << " " << a.nnz() << " " << hash(a) << "\n";
    } catch (const cgv::ParseError& e) {
        std::cout << "error " << static_cast<int>(e.code) << "\n";
    } catch (const std::exception& e) {
        std::cout << "exception " << e.what() << "\n";
        return 1;
    }
    return 0;
}
