// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A minimal restatement of the subset of Eigen 3's public API that the
// reference's hot-path sources use (/root/reference/proj/src/{lie,camera,
// tracking,backend}.cpp and include/pmslam/*.hpp), so that those files can be
// compiled UNMODIFIED into oracle/_ref/ (the image has no Eigen; the
// reference pins neither a version nor a vendored copy, proj/CMakeLists.txt:11).
//
// Written from Eigen's documented semantics, not from its sources:
//  * dense fixed / dynamic matrices, column-major storage, eager evaluation
//    (every expression returns a concrete Matrix; products accumulate
//    sum_k a(i,k) b(k,j) in increasing k);
//  * lvalue views: block<r,c>(i,j), block(i,j,r,c), head/tail/segment,
//    row/col, diagonal;
//  * comma initialiser (row by row, as Eigen's operator<< fills);
//  * LDLT: LDL^T with symmetric pivoting on the largest remaining diagonal,
//    solve with the pseudo-inverse of D (|d| <= numeric_limits::min -> 0);
//  * PartialPivLU, 3x3 JacobiSVD (one-sided Jacobi sweeps), determinant;
//  * SparseMatrix (column-major, setFromTriplets sums duplicates, coeffRef
//    inserts) and SimplicialLDLT: the up-looking LDL^T of the elimination
//    tree (lower triangle read), failure iff a pivot is exactly zero.  The
//    fill-reducing AMD permutation of Eigen's default is NOT applied
//    (natural ordering, as the reference's SPEC.md:359 states); the
//    factorisation semantics are unchanged, rounding differs at ulp level.
#pragma once

#include <algorithm>
#include <array>
#include <cassert>
#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <map>
#include <stdexcept>
#include <type_traits>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
enum { Infinity = -1 };
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };
enum DecompositionOptions { ComputeFullU = 0x04, ComputeThinU = 0x08, ComputeFullV = 0x10, ComputeThinV = 0x20 };
enum UpLoType { Lower = 0x1, Upper = 0x2 };
enum StorageOptions { ColMajor = 0, RowMajor = 0x1, AutoAlign = 0 };

template <class Scalar, int R, int C, int Options = 0, int MaxR = R, int MaxC = C>
class Matrix;
template <class MatrixType>
class LDLT;
template <class MatrixType>
class PartialPivLU;

namespace internal {
constexpr int merge_dim(int a, int b) { return a != Dynamic ? a : b; }
}  // namespace internal

// ------------------------------------------------------------------ base
template <class Derived, class S, int R, int C>
class DenseBase {
 public:
  using Scalar = S;
  using RealScalar = S;
  static constexpr int RowsAtCompileTime = R;
  static constexpr int ColsAtCompileTime = C;
  using PlainObject = Matrix<S, R, C>;

  Derived& derived() { return static_cast<Derived&>(*this); }
  const Derived& derived() const { return static_cast<const Derived&>(*this); }
  Index rows() const { return derived().rows(); }
  Index cols() const { return derived().cols(); }
  Index size() const { return derived().rows() * derived().cols(); }

  S coeff(Index i, Index j) const { return derived().coeffRef_c(i, j); }
  S& operator()(Index i, Index j) { return derived().ref(i, j); }
  S operator()(Index i, Index j) const { return derived().coeffRef_c(i, j); }
  // linear access of vectors (and column-major linear access of matrices)
  S& operator()(Index k) { return lin(k); }
  S operator()(Index k) const { return clin(k); }
  S& operator[](Index k) { return lin(k); }
  S operator[](Index k) const { return clin(k); }
  S& coeffRef(Index k) { return lin(k); }
  S& coeffRef(Index i, Index j) { return derived().ref(i, j); }
  S x() const { return clin(0); }
  S y() const { return clin(1); }
  S z() const { return clin(2); }
  S w() const { return clin(3); }
  S& x() { return lin(0); }
  S& y() { return lin(1); }
  S& z() { return lin(2); }

  PlainObject eval() const { return PlainObject(derived()); }

  // ---- reductions
  S sum() const {
    S s = S(0);
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) s += coeff(i, j);
    return s;
  }
  S squaredNorm() const {
    S s = S(0);
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) s += coeff(i, j) * coeff(i, j);
    return s;
  }
  S norm() const { return std::sqrt(squaredNorm()); }
  template <class O, class S2, int R2, int C2>
  S dot(const DenseBase<O, S2, R2, C2>& o) const {
    assert(size() == o.size());
    S s = S(0);
    for (Index k = 0; k < size(); ++k) s += clin(k) * o.derived().clin_(k);
    return s;
  }
  template <int p>
  S lpNorm() const {
    static_assert(p == Infinity || p == 1 || p == 2, "lpNorm<p>: p in {1, 2, Infinity}");
    if (p == 2) return norm();
    S s = S(0);
    for (Index k = 0; k < size(); ++k) s = p == Infinity ? std::max(s, std::abs(clin(k))) : s + std::abs(clin(k));
    return s;
  }
  S trace() const {
    S s = S(0);
    for (Index k = 0; k < std::min(rows(), cols()); ++k) s += coeff(k, k);
    return s;
  }
  bool allFinite() const {
    for (Index k = 0; k < size(); ++k)
      if (!std::isfinite(clin(k))) return false;
    return true;
  }
  bool hasNaN() const {
    for (Index k = 0; k < size(); ++k)
      if (std::isnan(clin(k))) return true;
    return false;
  }
  S maxCoeff() const {
    S m = clin(0);
    for (Index k = 1; k < size(); ++k) m = std::max(m, clin(k));
    return m;
  }
  S minCoeff() const {
    S m = clin(0);
    for (Index k = 1; k < size(); ++k) m = std::min(m, clin(k));
    return m;
  }

  // ---- coefficient-wise
  PlainObject cwiseMax(S v) const {
    PlainObject r(derived());
    for (Index k = 0; k < r.size(); ++k) r.data()[k] = std::max(r.data()[k], v);
    return r;
  }
  PlainObject cwiseMin(S v) const {
    PlainObject r(derived());
    for (Index k = 0; k < r.size(); ++k) r.data()[k] = std::min(r.data()[k], v);
    return r;
  }
  PlainObject cwiseAbs() const {
    PlainObject r(derived());
    for (Index k = 0; k < r.size(); ++k) r.data()[k] = std::abs(r.data()[k]);
    return r;
  }
  template <class O, class S2, int R2, int C2>
  PlainObject cwiseProduct(const DenseBase<O, S2, R2, C2>& o) const {
    PlainObject r(derived());
    for (Index j = 0; j < r.cols(); ++j)
      for (Index i = 0; i < r.rows(); ++i) r(i, j) *= o.coeff(i, j);
    return r;
  }
  PlainObject normalized() const {
    PlainObject r(derived());
    const S n = norm();
    if (n > S(0))
      for (Index k = 0; k < r.size(); ++k) r.data()[k] /= n;
    return r;
  }
  Matrix<S, C, R> transpose() const;
  Matrix<S, C, R> adjoint() const { return transpose(); }

  // ---- views (defined after the view class)
  template <int BR, int BC>
  auto block(Index i, Index j);
  template <int BR, int BC>
  auto block(Index i, Index j) const;
  auto block(Index i, Index j, Index r, Index c);
  auto block(Index i, Index j, Index r, Index c) const;
  template <int N>
  auto head();
  template <int N>
  auto head() const;
  auto head(Index n);
  auto head(Index n) const;
  template <int N>
  auto tail();
  template <int N>
  auto tail() const;
  auto tail(Index n);
  auto tail(Index n) const;
  template <int N>
  auto segment(Index i);
  template <int N>
  auto segment(Index i) const;
  auto segment(Index i, Index n);
  auto segment(Index i, Index n) const;
  auto row(Index i);
  auto row(Index i) const;
  auto col(Index j);
  auto col(Index j) const;
  auto diagonal();
  auto diagonal() const;
  template <int BR, int BC>
  auto topLeftCorner() {
    return block<BR, BC>(0, 0);
  }
  template <int BR, int BC>
  auto topRightCorner() {
    return block<BR, BC>(0, cols() - BC);
  }

  // ---- assignment-type operations
  Derived& setZero() { return setConstant(S(0)); }
  Derived& setOnes() { return setConstant(S(1)); }
  Derived& setConstant(S v) {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) derived().ref(i, j) = v;
    return derived();
  }
  Derived& fill(S v) { return setConstant(v); }
  Derived& setIdentity() {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) derived().ref(i, j) = i == j ? S(1) : S(0);
    return derived();
  }
  Derived& noalias() { return derived(); }
  template <class O, class S2, int R2, int C2>
  Derived& operator+=(const DenseBase<O, S2, R2, C2>& o) {
    const PlainObject t(o.derived());  // evaluated first: aliasing-safe
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) derived().ref(i, j) += t(i, j);
    return derived();
  }
  template <class O, class S2, int R2, int C2>
  Derived& operator-=(const DenseBase<O, S2, R2, C2>& o) {
    const PlainObject t(o.derived());
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) derived().ref(i, j) -= t(i, j);
    return derived();
  }
  Derived& operator*=(S v) {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) derived().ref(i, j) *= v;
    return derived();
  }
  Derived& operator/=(S v) {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) derived().ref(i, j) /= v;
    return derived();
  }

  // ---- decompositions
  LDLT<PlainObject> ldlt() const;
  PartialPivLU<PlainObject> partialPivLu() const;
  PartialPivLU<PlainObject> lu() const;
  S determinant() const;
  PlainObject inverse() const;

  // comma initialiser: fills row by row
  class CommaInit {
   public:
    CommaInit(Derived& d, S v) : d_(d) { put(v); }
    CommaInit& operator,(S v) {
      put(v);
      return *this;
    }
    ~CommaInit() noexcept(false) {}

   private:
    void put(S v) {
      const Index r = k_ / d_.cols(), c = k_ % d_.cols();
      if (r >= d_.rows()) throw std::out_of_range("Eigen shim: too many coefficients in comma initializer");
      d_.ref(r, c) = v;
      ++k_;
    }
    Derived& d_;
    Index k_ = 0;
  };
  CommaInit operator<<(S v) { return CommaInit(derived(), v); }

  // linear access helpers (column-major order)
  S clin_(Index k) const { return clin(k); }

 protected:
  S& lin(Index k) {
    if (C == 1 || cols() == 1) return derived().ref(k, 0);
    const Index r = rows();
    return r == 1 ? derived().ref(0, k) : derived().ref(k % r, k / r);
  }
  S clin(Index k) const {
    if (C == 1 || cols() == 1) return derived().coeffRef_c(k, 0);
    const Index r = rows();
    return r == 1 ? derived().coeffRef_c(0, k) : derived().coeffRef_c(k % r, k / r);
  }
};

// ------------------------------------------------------------------ view
// A strided lvalue window into another matrix: element (i, j) at
// p[i * inner + j * outer].
template <class S, int R, int C>
class View : public DenseBase<View<S, R, C>, S, R, C> {
 public:
  using Base = DenseBase<View<S, R, C>, S, R, C>;
  View(S* p, Index rows, Index cols, Index inner, Index outer)
      : p_(p), rows_(rows), cols_(cols), inner_(inner), outer_(outer) {}
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  S& ref(Index i, Index j) { return p_[i * inner_ + j * outer_]; }
  S coeffRef_c(Index i, Index j) const { return p_[i * inner_ + j * outer_]; }
  Index innerStride() const { return inner_; }
  Index outerStride() const { return outer_; }
  S* data_ptr() const { return p_; }

  View& operator=(const View& o) { return assign(o); }
  template <class O, class S2, int R2, int C2>
  View& operator=(const DenseBase<O, S2, R2, C2>& o) {
    return assign(o);
  }
  using Base::operator+=;
  using Base::operator-=;
  using Base::operator*=;
  using Base::operator/=;

 private:
  template <class O>
  View& assign(const O& o) {
    const Matrix<S, R, C> t(o);  // evaluated first: aliasing-safe
    if (t.rows() != rows_ || t.cols() != cols_) throw std::invalid_argument("Eigen shim: block size mismatch");
    for (Index j = 0; j < cols_; ++j)
      for (Index i = 0; i < rows_; ++i) ref(i, j) = t(i, j);
    return *this;
  }
  S* p_;
  Index rows_, cols_, inner_, outer_;
};

// ---------------------------------------------------------------- matrix
template <class S, int R, int C, int Options, int MaxR, int MaxC>
class Matrix : public DenseBase<Matrix<S, R, C, Options, MaxR, MaxC>, S, R, C> {
  static constexpr bool kFixed = R != Dynamic && C != Dynamic;

 public:
  using Base = DenseBase<Matrix, S, R, C>;

  Matrix() {
    if constexpr (kFixed) {
      data_.fill(S(0));
      rows_ = R;
      cols_ = C;
    } else {
      rows_ = R == Dynamic ? 0 : R;
      cols_ = C == Dynamic ? 0 : C;
      data_.assign(rows_ * cols_, S(0));
    }
  }
  // dynamic vector of size n
  template <class I, std::enable_if_t<std::is_integral_v<I>, int> = 0>
  explicit Matrix(I n) {
    static_assert(!kFixed, "Matrix(n) needs a dynamic size");
    if (R == 1)
      resize(1, n);
    else
      resize(n, 1);
  }
  // (rows, cols) for dynamic matrices, (x, y) coefficients for fixed 2-vectors
  template <class A, class B, std::enable_if_t<std::is_arithmetic_v<A> && std::is_arithmetic_v<B>, int> = 0>
  Matrix(A a, B b) {
    if constexpr (kFixed) {
      static_assert(R * C == 2, "two-coefficient constructor needs a 2-vector");
      rows_ = R;
      cols_ = C;
      data_ = {S(a), S(b)};
    } else {
      resize((Index)a, (Index)b);
    }
  }
  Matrix(S a, S b, S c) {
    static_assert(kFixed && R * C == 3, "three-coefficient constructor needs a 3-vector");
    rows_ = R;
    cols_ = C;
    data_ = {a, b, c};
  }
  Matrix(S a, S b, S c, S d) {
    static_assert(kFixed && R * C == 4, "four-coefficient constructor needs a 4-vector");
    rows_ = R;
    cols_ = C;
    data_ = {a, b, c, d};
  }
  Matrix(const Matrix&) = default;
  Matrix(Matrix&&) noexcept = default;
  Matrix& operator=(const Matrix&) = default;
  Matrix& operator=(Matrix&&) noexcept = default;
  template <class O, class S2, int R2, int C2>
  Matrix(const DenseBase<O, S2, R2, C2>& o) {
    copy_from(o.derived());
  }
  template <class O, class S2, int R2, int C2>
  Matrix& operator=(const DenseBase<O, S2, R2, C2>& o) {
    Matrix t;
    t.copy_from(o.derived());  // evaluated first: aliasing-safe
    *this = std::move(t);
    return *this;
  }

  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  S& ref(Index i, Index j) { return data_[i + j * rows_]; }
  S coeffRef_c(Index i, Index j) const { return data_[i + j * rows_]; }
  S* data() { return data_.data(); }
  const S* data() const { return data_.data(); }
  Index outerStride() const { return rows_; }

  void resize(Index r, Index c) {
    if (kFixed && (r != R || c != C)) throw std::invalid_argument("Eigen shim: resize of a fixed-size matrix");
    if (R != Dynamic && r != R) throw std::invalid_argument("Eigen shim: resize changes fixed rows");
    if (C != Dynamic && c != C) throw std::invalid_argument("Eigen shim: resize changes fixed cols");
    rows_ = r;
    cols_ = c;
    if constexpr (kFixed)
      data_.fill(S(0));
    else
      data_.assign(r * c, S(0));
  }
  void resize(Index n) {
    if (R == 1)
      resize(1, n);
    else
      resize(n, 1);
  }
  void conservativeResize(Index n) {
    static_assert(!kFixed, "conservativeResize needs a dynamic size");
    std::vector<S> d(data_.begin(), data_.end());
    const Index old = (Index)d.size();
    resize(n);
    for (Index k = 0; k < std::min(old, n); ++k) data_[k] = d[k];
  }

  static Matrix Zero() { return Constant(S(0)); }
  static Matrix Zero(Index n) { return Constant(n, S(0)); }
  static Matrix Zero(Index r, Index c) { return Constant(r, c, S(0)); }
  static Matrix Ones() { return Constant(S(1)); }
  static Matrix Ones(Index n) { return Constant(n, S(1)); }
  static Matrix Ones(Index r, Index c) { return Constant(r, c, S(1)); }
  static Matrix Constant(S v) {
    static_assert(kFixed, "Constant(v) needs a fixed size");
    Matrix m;
    m.setConstant(v);
    return m;
  }
  static Matrix Constant(Index n, S v) {
    Matrix m;
    m.resize(n);
    m.setConstant(v);
    return m;
  }
  static Matrix Constant(Index r, Index c, S v) {
    Matrix m;
    m.resize(r, c);
    m.setConstant(v);
    return m;
  }
  static Matrix Identity() {
    static_assert(kFixed, "Identity() needs a fixed size");
    Matrix m;
    m.setIdentity();
    return m;
  }
  static Matrix Identity(Index r, Index c) {
    Matrix m;
    m.resize(r, c);
    m.setIdentity();
    return m;
  }
  static Matrix Unit(Index k) {
    Matrix m = Zero();
    m.data_[k] = S(1);
    return m;
  }
  static Matrix UnitX() { return Unit(0); }
  static Matrix UnitY() { return Unit(1); }
  static Matrix UnitZ() { return Unit(2); }
  static Matrix UnitW() { return Unit(3); }

 private:
  template <class O>
  void copy_from(const O& o) {
    const Index r = o.rows(), c = o.cols();
    if constexpr (kFixed) {
      // Eigen allows assigning a row vector to a column vector of the same size
      const bool vec = (R == 1 || C == 1) && (r == 1 || c == 1) && r * c == R * C;
      if (!vec && (r != R || c != C)) throw std::invalid_argument("Eigen shim: size mismatch in assignment");
      rows_ = R;
      cols_ = C;
      if (vec && r != R) {
        for (Index k = 0; k < R * C; ++k) data_[k] = o.coeff(r == 1 ? 0 : k, r == 1 ? k : 0);
        return;
      }
    } else {
      if ((R != Dynamic && r != R) || (C != Dynamic && c != C)) {
        if ((R == 1 || C == 1) && (r == 1 || c == 1)) {  // vector transposition on assignment
          const Index n = r * c;
          resize(n);
          for (Index k = 0; k < n; ++k) data_[k] = o.coeff(r == 1 ? 0 : k, r == 1 ? k : 0);
          return;
        }
        throw std::invalid_argument("Eigen shim: size mismatch in assignment");
      }
      rows_ = r;
      cols_ = c;
      if constexpr (!kFixed) data_.resize(r * c);
    }
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) data_[i + j * r] = o.coeff(i, j);
  }

  std::conditional_t<kFixed, std::array<S, (kFixed ? R * C : 1)>, std::vector<S>> data_;
  Index rows_ = 0, cols_ = 0;
};

using Matrix2d = Matrix<double, 2, 2>;
using Matrix3d = Matrix<double, 3, 3>;
using Matrix4d = Matrix<double, 4, 4>;
using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Vector4d = Matrix<double, 4, 1>;
using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using RowVectorXd = Matrix<double, 1, Dynamic>;
using Matrix2f = Matrix<float, 2, 2>;
using Vector3f = Matrix<float, 3, 1>;
template <class S, int N>
using Vector = Matrix<S, N, 1>;
template <class S, int N>
using RowVector = Matrix<S, 1, N>;

// ------------------------------------------------- view factories (base)
namespace internal {
template <class T>
struct is_view : std::false_type {};
template <class S, int R, int C>
struct is_view<View<S, R, C>> : std::true_type {};
template <class D>
auto* base_ptr(D& d) {
  if constexpr (is_view<std::remove_const_t<D>>::value)
    return d.data_ptr();
  else
    return const_cast<typename D::Scalar*>(d.data());
}
template <class D>
Index inner_stride(const D& d) {
  if constexpr (is_view<D>::value)
    return d.innerStride();
  else
    return 1;
}
template <class S, int BR, int BC, class D>
View<S, BR, BC> make_view(const D& d, Index i, Index j, Index r, Index c) {
  if (i < 0 || j < 0 || i + r > d.rows() || j + c > d.cols())
    throw std::out_of_range("Eigen shim: block out of range");
  auto* p = base_ptr(const_cast<D&>(d));
  const Index in = inner_stride(d), out = d.outerStride();
  return View<S, BR, BC>(p + i * in + j * out, r, c, in, out);
}
}  // namespace internal

#define PMX_SHIM_VIEW_PAIR(DECL, BODY) \
  template <class D, class S, int R, int C> \
  DECL { BODY }

template <class D, class S, int R, int C>
template <int BR, int BC>
auto DenseBase<D, S, R, C>::block(Index i, Index j) {
  return internal::make_view<S, BR, BC>(derived(), i, j, BR, BC);
}
template <class D, class S, int R, int C>
template <int BR, int BC>
auto DenseBase<D, S, R, C>::block(Index i, Index j) const {
  return internal::make_view<S, BR, BC>(derived(), i, j, BR, BC);
}
template <class D, class S, int R, int C>
auto DenseBase<D, S, R, C>::block(Index i, Index j, Index r, Index c) {
  return internal::make_view<S, Dynamic, Dynamic>(derived(), i, j, r, c);
}
template <class D, class S, int R, int C>
auto DenseBase<D, S, R, C>::block(Index i, Index j, Index r, Index c) const {
  return internal::make_view<S, Dynamic, Dynamic>(derived(), i, j, r, c);
}
// vector segments: along the vector's direction
#define PMX_SHIM_SEG(N, start, n)                                                                      \
  (rows() == 1 ? internal::make_view<S, 1, N>(derived(), 0, (start), 1, (n))                           \
               : internal::make_view<S, (N == Dynamic ? Dynamic : N), 1>(derived(), (start), 0, (n), 1))
template <class D, class S, int R, int C>
template <int N>
auto DenseBase<D, S, R, C>::head() {
  static_assert(C == 1 || R == 1, "head<N>() on vectors");
  if constexpr (R == 1)
    return internal::make_view<S, 1, N>(derived(), 0, 0, 1, N);
  else
    return internal::make_view<S, N, 1>(derived(), 0, 0, N, 1);
}
template <class D, class S, int R, int C>
template <int N>
auto DenseBase<D, S, R, C>::head() const {
  return const_cast<DenseBase*>(this)->template head<N>();
}
template <class D, class S, int R, int C>
auto DenseBase<D, S, R, C>::head(Index n) {
  if constexpr (R == 1)
    return internal::make_view<S, 1, Dynamic>(derived(), 0, 0, 1, n);
  else
    return internal::make_view<S, Dynamic, 1>(derived(), 0, 0, n, 1);
}
template <class D, class S, int R, int C>
auto DenseBase<D, S, R, C>::head(Index n) const {
  return const_cast<DenseBase*>(this)->head(n);
}
template <class D, class S, int R, int C>
template <int N>
auto DenseBase<D, S, R, C>::tail() {
  if constexpr (R == 1)
    return internal::make_view<S, 1, N>(derived(), 0, cols() - N, 1, N);
  else
    return internal::make_view<S, N, 1>(derived(), rows() - N, 0, N, 1);
}
template <class D, class S, int R, int C>
template <int N>
auto DenseBase<D, S, R, C>::tail() const {
  return const_cast<DenseBase*>(this)->template tail<N>();
}
template <class D, class S, int R, int C>
auto DenseBase<D, S, R, C>::tail(Index n) {
  if constexpr (R == 1)
    return internal::make_view<S, 1, Dynamic>(derived(), 0, cols() - n, 1, n);
  else
    return internal::make_view<S, Dynamic, 1>(derived(), rows() - n, 0, n, 1);
}
template <class D, class S, int R, int C>
auto DenseBase<D, S, R, C>::tail(Index n) const {
  return const_cast<DenseBase*>(this)->tail(n);
}
template <class D, class S, int R, int C>
template <int N>
auto DenseBase<D, S, R, C>::segment(Index i) {
  if constexpr (R == 1)
    return internal::make_view<S, 1, N>(derived(), 0, i, 1, N);
  else
    return internal::make_view<S, N, 1>(derived(), i, 0, N, 1);
}
template <class D, class S, int R, int C>
template <int N>
auto DenseBase<D, S, R, C>::segment(Index i) const {
  return const_cast<DenseBase*>(this)->template segment<N>(i);
}
template <class D, class S, int R, int C>
auto DenseBase<D, S, R, C>::segment(Index i, Index n) {
  if constexpr (R == 1)
    return internal::make_view<S, 1, Dynamic>(derived(), 0, i, 1, n);
  else
    return internal::make_view<S, Dynamic, 1>(derived(), i, 0, n, 1);
}
template <class D, class S, int R, int C>
auto DenseBase<D, S, R, C>::segment(Index i, Index n) const {
  return const_cast<DenseBase*>(this)->segment(i, n);
}
template <class D, class S, int R, int C>
auto DenseBase<D, S, R, C>::row(Index i) {
  return internal::make_view<S, 1, C>(derived(), i, 0, 1, cols());
}
template <class D, class S, int R, int C>
auto DenseBase<D, S, R, C>::row(Index i) const {
  return const_cast<DenseBase*>(this)->row(i);
}
template <class D, class S, int R, int C>
auto DenseBase<D, S, R, C>::col(Index j) {
  return internal::make_view<S, R, 1>(derived(), 0, j, rows(), 1);
}
template <class D, class S, int R, int C>
auto DenseBase<D, S, R, C>::col(Index j) const {
  return const_cast<DenseBase*>(this)->col(j);
}
template <class D, class S, int R, int C>
auto DenseBase<D, S, R, C>::diagonal() {
  constexpr int N = (R != Dynamic && C != Dynamic) ? (R < C ? R : C) : Dynamic;
  const Index n = std::min(rows(), cols());
  auto* p = internal::base_ptr(derived());
  const Index in = internal::inner_stride(derived()), out = derived().outerStride();
  return View<S, N, 1>(p, n, 1, in + out, 0);
}
template <class D, class S, int R, int C>
auto DenseBase<D, S, R, C>::diagonal() const {
  return const_cast<DenseBase*>(this)->diagonal();
}
#undef PMX_SHIM_SEG
#undef PMX_SHIM_VIEW_PAIR

template <class D, class S, int R, int C>
Matrix<S, C, R> DenseBase<D, S, R, C>::transpose() const {
  Matrix<S, C, R> t;
  if constexpr (R == Dynamic || C == Dynamic) t.resize(cols(), rows());
  for (Index j = 0; j < cols(); ++j)
    for (Index i = 0; i < rows(); ++i) t(j, i) = coeff(i, j);
  return t;
}

// ------------------------------------------------------------- operators
template <class A, class SA, int RA, int CA, class B, class SB, int RB, int CB>
auto operator+(const DenseBase<A, SA, RA, CA>& a, const DenseBase<B, SB, RB, CB>& b) {
  Matrix<SA, internal::merge_dim(RA, RB), internal::merge_dim(CA, CB)> r(a.derived());
  if (b.rows() != r.rows() || b.cols() != r.cols()) throw std::invalid_argument("Eigen shim: operator+ sizes");
  for (Index j = 0; j < r.cols(); ++j)
    for (Index i = 0; i < r.rows(); ++i) r(i, j) = r(i, j) + b.coeff(i, j);
  return r;
}
template <class A, class SA, int RA, int CA, class B, class SB, int RB, int CB>
auto operator-(const DenseBase<A, SA, RA, CA>& a, const DenseBase<B, SB, RB, CB>& b) {
  Matrix<SA, internal::merge_dim(RA, RB), internal::merge_dim(CA, CB)> r(a.derived());
  if (b.rows() != r.rows() || b.cols() != r.cols()) throw std::invalid_argument("Eigen shim: operator- sizes");
  for (Index j = 0; j < r.cols(); ++j)
    for (Index i = 0; i < r.rows(); ++i) r(i, j) = r(i, j) - b.coeff(i, j);
  return r;
}
template <class A, class S, int R, int C>
Matrix<S, R, C> operator-(const DenseBase<A, S, R, C>& a) {
  Matrix<S, R, C> r(a.derived());
  for (Index k = 0; k < r.size(); ++k) r.data()[k] = -r.data()[k];
  return r;
}
template <class A, class S, int R, int C, class T, std::enable_if_t<std::is_arithmetic_v<T>, int> = 0>
Matrix<S, R, C> operator*(T s, const DenseBase<A, S, R, C>& a) {
  Matrix<S, R, C> r(a.derived());
  for (Index k = 0; k < r.size(); ++k) r.data()[k] = S(s) * r.data()[k];
  return r;
}
template <class A, class S, int R, int C, class T, std::enable_if_t<std::is_arithmetic_v<T>, int> = 0>
Matrix<S, R, C> operator*(const DenseBase<A, S, R, C>& a, T s) {
  Matrix<S, R, C> r(a.derived());
  for (Index k = 0; k < r.size(); ++k) r.data()[k] = r.data()[k] * S(s);
  return r;
}
template <class A, class S, int R, int C, class T, std::enable_if_t<std::is_arithmetic_v<T>, int> = 0>
Matrix<S, R, C> operator/(const DenseBase<A, S, R, C>& a, T s) {
  Matrix<S, R, C> r(a.derived());
  for (Index k = 0; k < r.size(); ++k) r.data()[k] = r.data()[k] / S(s);
  return r;
}
// matrix product: sum over k in increasing order
template <class A, class S, int RA, int CA, class B, int RB, int CB>
Matrix<S, RA, CB> operator*(const DenseBase<A, S, RA, CA>& a, const DenseBase<B, S, RB, CB>& b) {
  if (a.cols() != b.rows()) throw std::invalid_argument("Eigen shim: product sizes");
  Matrix<S, RA, CB> r;
  if constexpr (RA == Dynamic || CB == Dynamic) r.resize(a.rows(), b.cols());
  for (Index j = 0; j < b.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) {
      S s = S(0);
      for (Index k = 0; k < a.cols(); ++k) s += a.coeff(i, k) * b.coeff(k, j);
      r(i, j) = s;
    }
  return r;
}
template <class A, class S, int RA, int CA, class B, int RB, int CB>
bool operator==(const DenseBase<A, S, RA, CA>& a, const DenseBase<B, S, RB, CB>& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i)
      if (a.coeff(i, j) != b.coeff(i, j)) return false;
  return true;
}

// ----------------------------------------------------------------- LDLT
// Eigen's LDLT<Matrix, Lower>: at step k pick the largest remaining |diagonal|
// as pivot, swap it in (lower triangle), update column k with the previous
// columns, scale by the pivot when it is non-zero.  solve: P, L^-1, D^+
// (|d| <= numeric_limits::min -> 0), L^-T, P^T.
template <class MatrixType>
class LDLT {
 public:
  using S = typename MatrixType::Scalar;
  LDLT() = default;
  template <class M>
  explicit LDLT(const M& a) {
    compute(a);
  }
  template <class M>
  LDLT& compute(const M& a) {
    n_ = a.rows();
    m_ = Matrix<S, Dynamic, Dynamic>(a);
    tr_.assign(n_, 0);
    zero_ = false;
    std::vector<S> temp(n_);
    for (Index k = 0; k < n_; ++k) {
      Index big = k;
      S bigv = std::abs(m_(k, k));
      for (Index i = k + 1; i < n_; ++i)
        if (std::abs(m_(i, i)) > bigv) {
          bigv = std::abs(m_(i, i));
          big = i;
        }
      tr_[k] = big;
      if (k != big) {
        for (Index c = 0; c < k; ++c) std::swap(m_(k, c), m_(big, c));
        for (Index r = big + 1; r < n_; ++r) std::swap(m_(r, k), m_(r, big));
        std::swap(m_(k, k), m_(big, big));
        for (Index i = k + 1; i < big; ++i) {
          const S t = m_(i, k);
          m_(i, k) = m_(big, i);
          m_(big, i) = t;
        }
      }
      if (k > 0) {
        for (Index c = 0; c < k; ++c) temp[c] = m_(c, c) * m_(k, c);
        S acc = S(0);
        for (Index c = 0; c < k; ++c) acc += m_(k, c) * temp[c];
        m_(k, k) -= acc;
        for (Index r = k + 1; r < n_; ++r) {
          S a = S(0);
          for (Index c = 0; c < k; ++c) a += m_(r, c) * temp[c];
          m_(r, k) -= a;
        }
      }
      const S akk = m_(k, k);
      const bool ok = std::abs(akk) > S(0);
      if (k == 0 && !ok) {  // the whole diagonal is zero: D = 0
        zero_ = true;
        return *this;
      }
      if (ok)
        for (Index r = k + 1; r < n_; ++r) m_(r, k) /= akk;
    }
    return *this;
  }
  ComputationInfo info() const { return Success; }
  template <class O, class S2, int R2, int C2>
  Matrix<S, R2, C2> solve(const DenseBase<O, S2, R2, C2>& b) const {
    Matrix<S, R2, C2> x(b.derived());
    if (zero_) {
      x.setZero();
      return x;
    }
    for (Index c = 0; c < x.cols(); ++c) {
      std::vector<S> d(n_);
      for (Index i = 0; i < n_; ++i) d[i] = x(i, c);
      for (Index k = 0; k < n_; ++k) std::swap(d[k], d[tr_[k]]);
      for (Index i = 0; i < n_; ++i)
        for (Index j = 0; j < i; ++j) d[i] -= m_(i, j) * d[j];
      const S tol = std::numeric_limits<S>::min();
      for (Index i = 0; i < n_; ++i) d[i] = std::abs(m_(i, i)) > tol ? d[i] / m_(i, i) : S(0);
      for (Index i = n_ - 1; i >= 0; --i)
        for (Index r = i + 1; r < n_; ++r) d[i] -= m_(r, i) * d[r];
      for (Index k = n_ - 1; k >= 0; --k) std::swap(d[k], d[tr_[k]]);
      for (Index i = 0; i < n_; ++i) x(i, c) = d[i];
    }
    return x;
  }

 private:
  Index n_ = 0;
  Matrix<S, Dynamic, Dynamic> m_;
  std::vector<Index> tr_;
  bool zero_ = false;
};

// --------------------------------------------------------- PartialPivLU
template <class MatrixType>
class PartialPivLU {
 public:
  using S = typename MatrixType::Scalar;
  template <class M>
  explicit PartialPivLU(const M& a) : lu_(a), n_(a.rows()) {
    perm_.resize(n_);
    for (Index i = 0; i < n_; ++i) perm_[i] = i;
    sign_ = 1;
    for (Index k = 0; k < n_; ++k) {
      Index p = k;
      for (Index i = k + 1; i < n_; ++i)
        if (std::abs(lu_(i, k)) > std::abs(lu_(p, k))) p = i;
      if (p != k) {
        for (Index c = 0; c < n_; ++c) std::swap(lu_(k, c), lu_(p, c));
        std::swap(perm_[k], perm_[p]);
        sign_ = -sign_;
      }
      if (lu_(k, k) != S(0))
        for (Index i = k + 1; i < n_; ++i) lu_(i, k) /= lu_(k, k);
      for (Index i = k + 1; i < n_; ++i)
        for (Index c = k + 1; c < n_; ++c) lu_(i, c) -= lu_(i, k) * lu_(k, c);
    }
  }
  template <class O, class S2, int R2, int C2>
  Matrix<S, R2, C2> solve(const DenseBase<O, S2, R2, C2>& b) const {
    Matrix<S, R2, C2> x(b.derived());
    for (Index c = 0; c < x.cols(); ++c) {
      std::vector<S> d(n_);
      for (Index i = 0; i < n_; ++i) d[i] = b.coeff(perm_[i], c);
      for (Index i = 0; i < n_; ++i)
        for (Index j = 0; j < i; ++j) d[i] -= lu_(i, j) * d[j];
      for (Index i = n_ - 1; i >= 0; --i) {
        for (Index j = i + 1; j < n_; ++j) d[i] -= lu_(i, j) * d[j];
        d[i] /= lu_(i, i);
      }
      for (Index i = 0; i < n_; ++i) x(i, c) = d[i];
    }
    return x;
  }
  S determinant() const {
    S d = S(sign_);
    for (Index i = 0; i < n_; ++i) d *= lu_(i, i);
    return d;
  }

 private:
  Matrix<S, Dynamic, Dynamic> lu_;
  Index n_;
  std::vector<Index> perm_;
  int sign_ = 1;
};

template <class D, class S, int R, int C>
LDLT<typename DenseBase<D, S, R, C>::PlainObject> DenseBase<D, S, R, C>::ldlt() const {
  return LDLT<PlainObject>(derived());
}
template <class D, class S, int R, int C>
PartialPivLU<typename DenseBase<D, S, R, C>::PlainObject> DenseBase<D, S, R, C>::partialPivLu() const {
  return PartialPivLU<PlainObject>(derived());
}
template <class D, class S, int R, int C>
PartialPivLU<typename DenseBase<D, S, R, C>::PlainObject> DenseBase<D, S, R, C>::lu() const {
  return PartialPivLU<PlainObject>(derived());
}
template <class D, class S, int R, int C>
S DenseBase<D, S, R, C>::determinant() const {
  if (rows() == 3 && cols() == 3) {  // cofactor expansion along the first column
    const auto& m = derived();
    return m(0, 0) * (m(1, 1) * m(2, 2) - m(2, 1) * m(1, 2)) - m(1, 0) * (m(0, 1) * m(2, 2) - m(2, 1) * m(0, 2)) +
           m(2, 0) * (m(0, 1) * m(1, 2) - m(1, 1) * m(0, 2));
  }
  return PartialPivLU<PlainObject>(derived()).determinant();
}
template <class D, class S, int R, int C>
typename DenseBase<D, S, R, C>::PlainObject DenseBase<D, S, R, C>::inverse() const {
  PlainObject I = PlainObject::Identity(rows(), cols());
  return PartialPivLU<PlainObject>(derived()).solve(I);
}

// ------------------------------------------------------------ JacobiSVD
// Singular value decomposition A = U S V^T by one-sided (Hestenes) Jacobi
// rotations on the columns of A; used by lie.cpp:142-153 for the polar
// factor U V^T (unique for a non-singular A, so the rotation sequence only
// changes rounding).
template <class MatrixType>
class JacobiSVD {
 public:
  using S = typename MatrixType::Scalar;
  JacobiSVD(const MatrixType& a, unsigned = 0) {
    const Index m = a.rows(), n = a.cols();
    Matrix<S, Dynamic, Dynamic> W(a), V = Matrix<S, Dynamic, Dynamic>::Identity(n, n);
    for (int sweep = 0; sweep < 64; ++sweep) {
      S off = S(0);
      for (Index p = 0; p < n; ++p)
        for (Index q = p + 1; q < n; ++q) {
          S alpha = 0, beta = 0, gamma = 0;
          for (Index i = 0; i < m; ++i) {
            alpha += W(i, p) * W(i, p);
            beta += W(i, q) * W(i, q);
            gamma += W(i, p) * W(i, q);
          }
          if (gamma == S(0)) continue;
          off = std::max(off, std::abs(gamma) / std::sqrt(alpha * beta));
          const S zeta = (beta - alpha) / (2 * gamma);
          const S t = (zeta >= 0 ? S(1) : S(-1)) / (std::abs(zeta) + std::sqrt(1 + zeta * zeta));
          const S c = 1 / std::sqrt(1 + t * t), s = c * t;
          for (Index i = 0; i < m; ++i) {
            const S wp = W(i, p), wq = W(i, q);
            W(i, p) = c * wp - s * wq;
            W(i, q) = s * wp + c * wq;
          }
          for (Index i = 0; i < n; ++i) {
            const S vp = V(i, p), vq = V(i, q);
            V(i, p) = c * vp - s * vq;
            V(i, q) = s * vp + c * vq;
          }
        }
      if (off < std::numeric_limits<S>::epsilon()) break;
    }
    // singular values = column norms; sort descending
    std::vector<std::pair<S, Index>> sv(n);
    for (Index j = 0; j < n; ++j) sv[j] = {W.col(j).norm(), j};
    std::sort(sv.begin(), sv.end(), [](auto& x, auto& y) { return x.first > y.first; });
    U_ = MatrixType(a);
    V_ = MatrixType(a);
    sigma_.resize(n);
    for (Index k = 0; k < n; ++k) {
      const Index j = sv[k].second;
      sigma_(k) = sv[k].first;
      for (Index i = 0; i < m; ++i) U_(i, k) = sv[k].first > 0 ? W(i, j) / sv[k].first : (i == k ? 1 : 0);
      for (Index i = 0; i < n; ++i) V_(i, k) = V(i, j);
    }
  }
  const MatrixType& matrixU() const { return U_; }
  const MatrixType& matrixV() const { return V_; }
  const Matrix<S, Dynamic, 1>& singularValues() const { return sigma_; }

 private:
  MatrixType U_, V_;
  Matrix<S, Dynamic, 1> sigma_;
};

// --------------------------------------------------------------- sparse
template <class S>
class Triplet {
 public:
  Triplet(Index r = 0, Index c = 0, S v = S(0)) : r_(r), c_(c), v_(v) {}
  Index row() const { return r_; }
  Index col() const { return c_; }
  S value() const { return v_; }

 private:
  Index r_, c_;
  S v_;
};

// Column-major sparse matrix: one sorted (row -> value) map per column.
template <class S, int Options = 0, class StorageIndex = int>
class SparseMatrix {
 public:
  using Scalar = S;
  SparseMatrix() = default;
  SparseMatrix(Index r, Index c) { resize(r, c); }
  void resize(Index r, Index c) {
    rows_ = r;
    cols_ = c;
    colmap_.assign(c, {});
  }
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index outerSize() const { return cols_; }
  Index nonZeros() const {
    Index n = 0;
    for (const auto& c : colmap_) n += (Index)c.size();
    return n;
  }
  template <class It>
  void setFromTriplets(It begin, It end) {  // duplicates are summed
    for (auto& c : colmap_) c.clear();
    for (It it = begin; it != end; ++it) colmap_.at(it->col())[it->row()] += it->value();
  }
  S& coeffRef(Index r, Index c) { return colmap_.at(c)[r]; }  // inserts a zero when absent
  S coeff(Index r, Index c) const {
    const auto& m = colmap_.at(c);
    auto it = m.find(r);
    return it == m.end() ? S(0) : it->second;
  }
  void setZero() {
    for (auto& c : colmap_) c.clear();
  }
  Matrix<S, Dynamic, Dynamic> toDense() const {
    Matrix<S, Dynamic, Dynamic> d = Matrix<S, Dynamic, Dynamic>::Zero(rows_, cols_);
    for (Index c = 0; c < cols_; ++c)
      for (const auto& [r, v] : colmap_[c]) d(r, c) = v;
    return d;
  }
  class InnerIterator {
   public:
    InnerIterator(const SparseMatrix& m, Index outer)
        : col_(outer), it_(m.colmap_.at(outer).begin()), end_(m.colmap_.at(outer).end()) {}
    explicit operator bool() const { return it_ != end_; }
    InnerIterator& operator++() {
      ++it_;
      return *this;
    }
    Index row() const { return it_->first; }
    Index col() const { return col_; }
    Index index() const { return it_->first; }
    S value() const { return it_->second; }

   private:
    Index col_;
    typename std::map<Index, S>::const_iterator it_, end_;
  };

 private:
  Index rows_ = 0, cols_ = 0;
  std::vector<std::map<Index, S>> colmap_;
};

// SimplicialLDLT<SparseMatrix, Lower>: up-looking LDL^T over the
// elimination tree (T. Davis' LDL, the algorithm Eigen's
// SimplicialCholesky implements), natural ordering.  Row k: scatter the
// lower-triangle row A(k, 0..k) (= column k of the upper triangle), find
// its pattern by walking the elimination tree, solve the triangular system
// in topological order, d_k = a_kk - sum l_kj y_j; failure
// (NumericalIssue) iff some d_k == 0.  solve: L, D^-1 (as multiplication by
// the reciprocal, like asDiagonal().inverse()), L^T.
template <class MatrixType, int UpLo = Lower>
class SimplicialLDLT {
 public:
  using S = typename MatrixType::Scalar;
  SimplicialLDLT() = default;
  explicit SimplicialLDLT(const MatrixType& a) { compute(a); }
  SimplicialLDLT& compute(const MatrixType& a) {
    const Index n = a.rows();
    n_ = n;
    // upper-triangle columns: column k holds rows i <= k  (A(k, i) of the lower triangle)
    std::vector<std::vector<std::pair<Index, S>>> up(n);
    for (Index c = 0; c < n; ++c)
      for (typename MatrixType::InnerIterator it(a, c); it; ++it)
        if (it.row() >= c) up[it.row()].push_back({c, it.value()});  // lower (r >= c) -> upper column r
    for (auto& col : up) std::sort(col.begin(), col.end(), [](auto& x, auto& y) { return x.first < y.first; });
    // analyse: elimination tree and column counts
    std::vector<Index> parent(n, -1), tags(n), nz(n, 0);
    for (Index k = 0; k < n; ++k) {
      tags[k] = k;
      for (const auto& [i0, v] : up[k]) {
        Index i = i0;
        if (i < k)
          for (; tags[i] != k; i = parent[i]) {
            if (parent[i] == -1) parent[i] = k;
            nz[i]++;
            tags[i] = k;
          }
      }
    }
    Lp_.assign(n + 1, 0);
    for (Index k = 0; k < n; ++k) Lp_[k + 1] = Lp_[k] + nz[k];
    Li_.assign(Lp_[n], 0);
    Lx_.assign(Lp_[n], S(0));
    diag_.assign(n, S(0));
    // factorise
    std::vector<S> y(n, S(0));
    std::vector<Index> pattern(n), cnt(n, 0);
    info_ = Success;
    for (Index k = 0; k < n; ++k) {
      y[k] = S(0);
      Index top = n;
      tags[k] = k;
      cnt[k] = 0;
      for (const auto& [i0, v] : up[k]) {
        Index i = i0;
        if (i <= k) {
          y[i] += v;
          Index len = 0;
          for (; tags[i] != k; i = parent[i]) {
            pattern[len++] = i;
            tags[i] = k;
          }
          while (len > 0) pattern[--top] = pattern[--len];
        }
      }
      S d = y[k];
      y[k] = S(0);
      for (; top < n; ++top) {
        const Index i = pattern[top];
        const S yi = y[i];
        y[i] = S(0);
        const S l_ki = yi / diag_[i];
        const Index p2 = Lp_[i] + cnt[i];
        Index p;
        for (p = Lp_[i]; p < p2; ++p) y[Li_[p]] -= Lx_[p] * yi;
        d -= l_ki * yi;
        Li_[p] = k;
        Lx_[p] = l_ki;
        ++cnt[i];
      }
      diag_[k] = d;
      if (d == S(0)) {
        info_ = NumericalIssue;
        break;
      }
    }
    return *this;
  }
  ComputationInfo info() const { return info_; }
  template <class O, class S2, int R2, int C2>
  Matrix<S, Dynamic, 1> solve(const DenseBase<O, S2, R2, C2>& b) const {
    Matrix<S, Dynamic, 1> x(b.derived());
    // L y = b (unit lower, column oriented)
    for (Index j = 0; j < n_; ++j)
      for (Index p = Lp_[j]; p < Lp_[j + 1]; ++p) x(Li_[p]) -= Lx_[p] * x(j);
    for (Index j = 0; j < n_; ++j) x(j) = (S(1) / diag_[j]) * x(j);
    // L^T x = y (row oriented over the columns of L)
    for (Index j = n_ - 1; j >= 0; --j)
      for (Index p = Lp_[j]; p < Lp_[j + 1]; ++p) x(j) -= Lx_[p] * x(Li_[p]);
    return x;
  }

 private:
  Index n_ = 0;
  std::vector<Index> Lp_, Li_;
  std::vector<S> Lx_, diag_;
  ComputationInfo info_ = InvalidInput;
};

}  // namespace Eigen
