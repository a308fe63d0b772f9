// TEST INFRASTRUCTURE ONLY — the reference's naive oracles for C++ tests of
// the drop-in: cabl::dot_ref / gemv_ref / ger_ref with the reference's
// signatures (reference kernels.hpp:119-127, :171-181, :264-270), computed by
// the plain-C restatement in cabl_oracle.c with the compiled reference's
// rounding (pinned by tests/test_oracle.py).  Never included by the product.
#pragma once

#include <cabl/dense.hpp>
#include <stdexcept>

#include "cabl_oracle.h"

namespace cabl {

namespace oracle_detail {
inline void need(bool ok, const char* msg) {
    if (!ok) throw std::invalid_argument(msg);
}
inline unsigned vec_of(std::size_t elem) { return unsigned(16 / elem); }
} // namespace oracle_detail

inline float dot_ref(const Vector<float>& x, const Vector<float>& y, float alpha0) {
    oracle_detail::need(x.len() == y.len(), "dot: x and y lengths differ");
    return oracle_dot_ref_f32(x.data(), y.data(), x.len(), alpha0, oracle_detail::vec_of(4));
}
inline double dot_ref(const Vector<double>& x, const Vector<double>& y, double alpha0) {
    oracle_detail::need(x.len() == y.len(), "dot: x and y lengths differ");
    return oracle_dot_ref_f64(x.data(), y.data(), x.len(), alpha0, oracle_detail::vec_of(8));
}

template <typename T>
void gemv_ref(const DenseMatrix<T>& A, const Vector<T>& x, Vector<T>& c) {
    oracle_detail::need(A.cols() == x.len(), "gemv: A.cols != x.len");
    oracle_detail::need(A.rows() == c.len(), "gemv: A.rows != c.len");
    oracle_detail::need(!(c.data() != nullptr && c.data() == x.data()), "gemv: c must not alias x");
    const int lay = A.layout() == Layout::ColMajor ? 1 : 0;
    if constexpr (sizeof(T) == 4)
        oracle_gemv_ref_f32(A.data(), lay, A.rows(), A.cols(), x.data(), c.data(),
                            oracle_detail::vec_of(4));
    else
        oracle_gemv_ref_f64(A.data(), lay, A.rows(), A.cols(), x.data(), c.data(),
                            oracle_detail::vec_of(8));
}

template <typename T>
void ger_ref(const Vector<T>& x, const Vector<T>& y, DenseMatrix<T>& C) {
    oracle_detail::need(C.rows() == x.len(), "ger: C.rows != x.len");
    oracle_detail::need(C.cols() == y.len(), "ger: C.cols != y.len");
    const int lay = C.layout() == Layout::ColMajor ? 1 : 0;
    if constexpr (sizeof(T) == 4)
        oracle_ger_ref_f32(x.data(), y.data(), C.data(), lay, C.rows(), C.cols());
    else
        oracle_ger_ref_f64(x.data(), y.data(), C.data(), lay, C.rows(), C.cols());
}

} // namespace cabl
