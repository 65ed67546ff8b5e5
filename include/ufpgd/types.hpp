// Eigen-free replacement of ufpgd/types.hpp (/root/reference/proj/core/include/ufpgd/types.hpp:9-20).
// A ComplexMatrix is column-major K x M complex<double>, column m = antenna m,
// which is exactly the reference's Eigen::MatrixXcd storage (and the row-major
// [M][K] layout the GPU batches use).
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstddef>
#include <initializer_list>
#include <stdexcept>
#include <vector>

namespace ufpgd {

using Complex = std::complex<double>;

class RealVector {
 public:
  RealVector() = default;
  explicit RealVector(std::ptrdiff_t n, double v = 0.0) : d_(static_cast<std::size_t>(n), v) {}
  RealVector(std::initializer_list<double> v) : d_(v) {}
  static RealVector Constant(std::ptrdiff_t n, double v) { return RealVector(n, v); }
  std::ptrdiff_t size() const { return static_cast<std::ptrdiff_t>(d_.size()); }
  double& operator[](std::ptrdiff_t i) { return d_[static_cast<std::size_t>(i)]; }
  double operator[](std::ptrdiff_t i) const { return d_[static_cast<std::size_t>(i)]; }
  double& operator()(std::ptrdiff_t i) { return (*this)[i]; }
  double operator()(std::ptrdiff_t i) const { return (*this)[i]; }
  void resize(std::ptrdiff_t n) { d_.resize(static_cast<std::size_t>(n)); }
  const double* data() const { return d_.data(); }
  double* data() { return d_.data(); }
  double norm() const {
    double s = 0.0;
    for (double x : d_) s += x * x;
    return std::sqrt(s);
  }

 private:
  std::vector<double> d_;
};

class ComplexMatrix {
 public:
  ComplexMatrix() = default;
  ComplexMatrix(std::ptrdiff_t rows, std::ptrdiff_t cols)
      : rows_(rows), cols_(cols), d_(static_cast<std::size_t>(rows * cols)) {
    if (rows < 0 || cols < 0) throw std::invalid_argument("ComplexMatrix: negative size");
  }
  static ComplexMatrix Zero(std::ptrdiff_t r, std::ptrdiff_t c) { return ComplexMatrix(r, c); }
  static ComplexMatrix Constant(std::ptrdiff_t r, std::ptrdiff_t c, Complex v) {
    ComplexMatrix m(r, c);
    std::fill(m.d_.begin(), m.d_.end(), v);
    return m;
  }
  static ComplexMatrix Identity(std::ptrdiff_t r, std::ptrdiff_t c) {
    ComplexMatrix m(r, c);
    for (std::ptrdiff_t i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
    return m;
  }
  std::ptrdiff_t rows() const { return rows_; }
  std::ptrdiff_t cols() const { return cols_; }
  std::ptrdiff_t size() const { return rows_ * cols_; }
  Complex& operator()(std::ptrdiff_t r, std::ptrdiff_t c) { return d_[static_cast<std::size_t>(c * rows_ + r)]; }
  const Complex& operator()(std::ptrdiff_t r, std::ptrdiff_t c) const {
    return d_[static_cast<std::size_t>(c * rows_ + r)];
  }
  Complex* data() { return d_.data(); }
  const Complex* data() const { return d_.data(); }
  ComplexMatrix conjugate() const {
    ComplexMatrix o(rows_, cols_);
    for (std::size_t i = 0; i < d_.size(); ++i) o.d_[i] = std::conj(d_[i]);
    return o;
  }
  ComplexMatrix transpose() const {
    ComplexMatrix o(cols_, rows_);
    for (std::ptrdiff_t c = 0; c < cols_; ++c)
      for (std::ptrdiff_t r = 0; r < rows_; ++r) o(c, r) = (*this)(r, c);
    return o;
  }
  double squaredNorm() const {
    double s = 0.0;
    for (const Complex& z : d_) s += std::norm(z);
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  double colNorm(std::ptrdiff_t c) const {
    double s = 0.0;
    for (std::ptrdiff_t r = 0; r < rows_; ++r) s += std::norm((*this)(r, c));
    return std::sqrt(s);
  }
  bool isZero() const {
    for (const Complex& z : d_)
      if (z != Complex(0.0, 0.0)) return false;
    return true;
  }
  bool allFinite() const {
    for (const Complex& z : d_)
      if (!std::isfinite(z.real()) || !std::isfinite(z.imag())) return false;
    return true;
  }
  ComplexMatrix operator-(const ComplexMatrix& o) const {
    check_same(o);
    ComplexMatrix r(rows_, cols_);
    for (std::size_t i = 0; i < d_.size(); ++i) r.d_[i] = d_[i] - o.d_[i];
    return r;
  }
  ComplexMatrix operator+(const ComplexMatrix& o) const {
    check_same(o);
    ComplexMatrix r(rows_, cols_);
    for (std::size_t i = 0; i < d_.size(); ++i) r.d_[i] = d_[i] + o.d_[i];
    return r;
  }
  friend ComplexMatrix operator*(double s, const ComplexMatrix& m) {
    ComplexMatrix r(m.rows_, m.cols_);
    for (std::size_t i = 0; i < m.d_.size(); ++i) r.d_[i] = s * m.d_[i];
    return r;
  }

 private:
  void check_same(const ComplexMatrix& o) const {
    if (o.rows_ != rows_ || o.cols_ != cols_) throw std::invalid_argument("ComplexMatrix: shape mismatch");
  }
  std::ptrdiff_t rows_ = 0, cols_ = 0;
  std::vector<Complex> d_;
};

using ComplexVector = std::vector<Complex>;

// K x M downlink channel, row k = user, column m = antenna.
using ChannelMatrix = ComplexMatrix;
// K x M precoder; column m feeds antenna m's PA.
using PrecoderMatrix = ComplexMatrix;

}  // namespace ufpgd
