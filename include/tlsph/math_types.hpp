// Fixed-size fp64 vectors and matrices for the C++ operator API.
//
// Drop-in for proj/src/tlsph/math_types.hpp:8-21, which aliases Eigen
// fixed-size types. Eigen is not part of this build, so this header provides
// the subset of the Eigen interface the reference API and its call sites use
// (construction, Zero/Identity, element access, +,-,*,/, norm, squaredNorm,
// dot, transpose, determinant, inverse, trace, asDiagonal, comma
// initialisation, array-style element products, allFinite). Arithmetic
// follows the Eigen 3.3/3.4 fixed-size evaluation order documented in
// oracle/tlsph_oracle.hpp.
#ifndef TLSPH_MATH_TYPES_HPP
#define TLSPH_MATH_TYPES_HPP

#include <cmath>
#include <cstddef>
#include <initializer_list>

namespace tlsph {

using Real = double;

template <int R, int C>
class Matrix {
 public:
  static constexpr int Rows = R;
  static constexpr int Cols = C;
  static constexpr int Size = R * C;

  Matrix() {
    for (int k = 0; k < Size; ++k) a_[k] = 0.0;
  }
  // vector constructors (Eigen's Vector2d(x, y), Vector3d(x, y, z))
  Matrix(double x, double y) : Matrix() {
    static_assert(Size == 2, "two-component constructor needs a 2-vector");
    a_[0] = x;
    a_[1] = y;
  }
  Matrix(double x, double y, double z) : Matrix() {
    static_assert(Size == 3, "three-component constructor needs a 3-vector");
    a_[0] = x;
    a_[1] = y;
    a_[2] = z;
  }

  static Matrix Zero() { return Matrix(); }
  static Matrix Constant(double v) {
    Matrix m;
    for (int k = 0; k < Size; ++k) m.a_[k] = v;
    return m;
  }
  static Matrix Identity() {
    Matrix m;
    for (int k = 0; k < (R < C ? R : C); ++k) m(k, k) = 1.0;
    return m;
  }
  void setZero() {
    for (int k = 0; k < Size; ++k) a_[k] = 0.0;
  }

  // column-major storage like Eigen
  double& operator()(int r, int c) { return a_[c * R + r]; }
  double operator()(int r, int c) const { return a_[c * R + r]; }
  double& operator[](int k) { return a_[k]; }
  double operator[](int k) const { return a_[k]; }
  double& operator()(int k) { return a_[k]; }
  double operator()(int k) const { return a_[k]; }
  int rows() const { return R; }
  int cols() const { return C; }
  int size() const { return Size; }
  double* data() { return a_; }
  const double* data() const { return a_; }

  Matrix& operator+=(const Matrix& o) {
    for (int k = 0; k < Size; ++k) a_[k] = a_[k] + o.a_[k];
    return *this;
  }
  Matrix& operator-=(const Matrix& o) {
    for (int k = 0; k < Size; ++k) a_[k] = a_[k] - o.a_[k];
    return *this;
  }
  Matrix& operator*=(double s) {
    for (int k = 0; k < Size; ++k) a_[k] = a_[k] * s;
    return *this;
  }
  Matrix& operator/=(double s) {
    for (int k = 0; k < Size; ++k) a_[k] = a_[k] / s;
    return *this;
  }
  Matrix operator-() const {
    Matrix m;
    for (int k = 0; k < Size; ++k) m.a_[k] = -a_[k];
    return m;
  }
  friend Matrix operator+(Matrix a, const Matrix& b) { return a += b; }
  friend Matrix operator-(Matrix a, const Matrix& b) { return a -= b; }
  friend Matrix operator*(Matrix a, double s) { return a *= s; }
  friend Matrix operator*(double s, const Matrix& a) {
    Matrix m;
    for (int k = 0; k < Size; ++k) m.a_[k] = s * a.a_[k];
    return m;
  }
  friend Matrix operator/(Matrix a, double s) { return a /= s; }
  bool operator==(const Matrix& o) const {
    for (int k = 0; k < Size; ++k)
      if (a_[k] != o.a_[k]) return false;
    return true;
  }
  bool operator!=(const Matrix& o) const { return !(*this == o); }

  // (x0*x0 + x1*x1) + x2*x2 ...
  double squaredNorm() const {
    double s = a_[0] * a_[0];
    for (int k = 1; k < Size; ++k) s = s + a_[k] * a_[k];
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  double sum() const {
    double s = a_[0];
    for (int k = 1; k < Size; ++k) s = s + a_[k];
    return s;
  }
  double dot(const Matrix& o) const {
    double s = a_[0] * o.a_[0];
    for (int k = 1; k < Size; ++k) s = s + a_[k] * o.a_[k];
    return s;
  }
  double trace() const {
    double s = (*this)(0, 0);
    for (int k = 1; k < (R < C ? R : C); ++k) s = s + (*this)(k, k);
    return s;
  }
  bool allFinite() const {
    for (int k = 0; k < Size; ++k)
      if (!std::isfinite(a_[k])) return false;
    return true;
  }
  Matrix<C, R> transpose() const {
    Matrix<C, R> t;
    for (int r = 0; r < R; ++r)
      for (int c = 0; c < C; ++c) t(c, r) = (*this)(r, c);
    return t;
  }
  Matrix cwiseProduct(const Matrix& o) const {
    Matrix m;
    for (int k = 0; k < Size; ++k) m.a_[k] = a_[k] * o.a_[k];
    return m;
  }
  // element-wise view (Eigen .array()): products and sums are element-wise
  struct ArrayView {
    Matrix m;
    ArrayView operator*(const ArrayView& o) const { return ArrayView{m.cwiseProduct(o.m)}; }
    double sum() const { return m.sum(); }
    const Matrix& matrix() const { return m; }
  };
  ArrayView array() const { return ArrayView{*this}; }
  Matrix eval() const { return *this; }
  Matrix<R, R> asDiagonal() const {
    static_assert(C == 1, "asDiagonal needs a vector");
    Matrix<R, R> m;
    for (int k = 0; k < R; ++k) m(k, k) = a_[k];
    return m;
  }

  double determinant() const;
  Matrix inverse() const;

  // comma initialisation, row by row (Eigen's operator<<)
  class CommaInit {
   public:
    CommaInit(Matrix& m, double v) : m_(m), k_(0) { put(v); }
    CommaInit& operator,(double v) {
      put(v);
      return *this;
    }

   private:
    void put(double v) {
      const int r = k_ / C, c = k_ % C;
      if (r < R) m_(r, c) = v;
      ++k_;
    }
    Matrix& m_;
    int k_;
  };
  CommaInit operator<<(double v) { return CommaInit(*this, v); }

 private:
  double a_[Size];
};

// matrix products, inner index ascending ((p0+p1)+p2)
template <int R, int K, int C>
Matrix<R, C> operator*(const Matrix<R, K>& a, const Matrix<K, C>& b) requires(!(R == K && K == C && C == 1)) {
  Matrix<R, C> m;
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) {
      double s = a(r, 0) * b(0, c);
      for (int q = 1; q < K; ++q) s = s + a(r, q) * b(q, c);
      m(r, c) = s;
    }
  return m;
}

template <>
inline double Matrix<2, 2>::determinant() const {
  const Matrix& m = *this;
  return m(0, 0) * m(1, 1) - m(1, 0) * m(0, 1);
}
template <>
inline double Matrix<3, 3>::determinant() const {
  const Matrix& m = *this;
  return m(0, 0) * (m(1, 1) * m(2, 2) - m(1, 2) * m(2, 1)) - m(0, 1) * (m(1, 0) * m(2, 2) - m(1, 2) * m(2, 0)) +
         m(0, 2) * (m(1, 0) * m(2, 1) - m(1, 1) * m(2, 0));
}
template <>
inline Matrix<2, 2> Matrix<2, 2>::inverse() const {
  const Matrix& m = *this;
  const double invdet = 1.0 / m.determinant();
  Matrix r;
  r(0, 0) = m(1, 1) * invdet;
  r(1, 0) = -m(1, 0) * invdet;
  r(0, 1) = -m(0, 1) * invdet;
  r(1, 1) = m(0, 0) * invdet;
  return r;
}
template <>
inline Matrix<3, 3> Matrix<3, 3>::inverse() const {
  const Matrix& m = *this;
  auto cof = [&](int i, int j) {
    const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
    return m(i1, j1) * m(i2, j2) - m(i1, j2) * m(i2, j1);
  };
  const double det = (cof(0, 0) * m(0, 0) + cof(1, 0) * m(1, 0)) + cof(2, 0) * m(2, 0);
  const double invdet = 1.0 / det;
  Matrix r;
  for (int row = 0; row < 3; ++row)
    for (int col = 0; col < 3; ++col) r(row, col) = cof(col, row) * invdet;
  return r;
}

template <int D>
using Vec = Matrix<D, 1>;

template <int D>
using Mat = Matrix<D, D>;

using Vec2 = Vec<2>;
using Vec3 = Vec<3>;
using Mat2 = Mat<2>;
using Mat3 = Mat<3>;

constexpr int ipow3(int d) { return d == 2 ? 9 : 27; }

}  // namespace tlsph

#endif  // TLSPH_MATH_TYPES_HPP
