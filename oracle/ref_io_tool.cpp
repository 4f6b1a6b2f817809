// ref_io_tool.cpp -- CPU ORACLE (test infrastructure only): the reference's
// matrix file I/O (matrix_io.hpp:25-117) and shortest-decimal formatting
// (experiment.hpp:376-380), compiled in place from the unmodified headers,
// as a stdin/stdout tool (iostreams inside a numpy-hosting Python process
// crash, so the tests run this as a subprocess).
//   ref_io_tool write L m n   < raw little-endian doubles (AoS)  > matrix text
//   ref_io_tool read          < matrix text   > "ok m n L\n" + raw doubles | "error LINE\n"
//   ref_io_tool shortest      < raw doubles   > one token per line
#include <cstdint>
#include <cstring>
#include <iostream>
#include <iterator>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

#include "xqr/experiment.hpp"
#include "xqr/matrix_io.hpp"

using namespace xqr;

template <class R>
constexpr int limbs_of() {
    if constexpr (std::is_same_v<R, double>) return 1;
    else if constexpr (std::is_same_v<R, double_double>) return 2;
    else return 4;
}

template <class R>
void write_as(int64_t m, int64_t n, const std::vector<double>& d) {
    constexpr int L = limbs_of<R>();
    col_matrix<R> a(m, n);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) {
            const double* p = d.data() + (j * m + i) * 2 * L;
            cplx<R> z;
            std::memcpy(&z.re, p, sizeof(R));
            std::memcpy(&z.im, p + L, sizeof(R));
            a(i, j) = z;
        }
    write_matrix(std::cout, a);
}

static std::vector<double> read_doubles() {
    std::string raw((std::istreambuf_iterator<char>(std::cin)), std::istreambuf_iterator<char>());
    std::vector<double> d(raw.size() / 8);
    std::memcpy(d.data(), raw.data(), d.size() * 8);
    return d;
}

int main(int argc, char** argv) {
    std::ios::sync_with_stdio(false);
    if (argc < 2) return 2;
    std::string mode = argv[1];
    if (mode == "write" && argc == 5) {
        int L = std::atoi(argv[2]);
        int64_t m = std::atoll(argv[3]), n = std::atoll(argv[4]);
        auto d = read_doubles();
        if (L == 1) write_as<double>(m, n, d);
        else if (L == 2) write_as<double_double>(m, n, d);
        else write_as<quad_double>(m, n, d);
        return 0;
    }
    if (mode == "read") {
        std::string text((std::istreambuf_iterator<char>(std::cin)), std::istreambuf_iterator<char>());
        std::istringstream in(text);
        try {
            any_matrix any = read_matrix(in);
            std::visit(
                [&](const auto& a) {
                    using R = std::decay_t<decltype(a(0, 0).re)>;
                    constexpr int L = limbs_of<R>();
                    std::cout << "ok " << a.rows() << ' ' << a.cols() << ' ' << L << '\n';
                    for (std::size_t j = 0; j < a.cols(); ++j)
                        for (std::size_t i = 0; i < a.rows(); ++i) {
                            cplx<R> z = a(i, j);
                            std::cout.write(reinterpret_cast<const char*>(&z.re), sizeof(R));
                            std::cout.write(reinterpret_cast<const char*>(&z.im), sizeof(R));
                        }
                },
                any);
        } catch (const parse_error& e) {
            std::cout << "error " << e.line << '\n';
        }
        return 0;
    }
    if (mode == "shortest") {
        for (double v : read_doubles()) std::cout << detail::shortest(v) << '\n';
        return 0;
    }
    return 2;
}
