// Eigen-subset restatement (TEST INFRASTRUCTURE, not product code).
//
// The reference (/root/reference/proj) needs Eigen3 >= 3.3 (proj/CMakeLists.txt:13),
// which is absent from this image and not vendored.  This header restates the
// six Eigen types the reference's hot-path and prep sources use:
// Vector3d, Matrix3Xd, Matrix3d, Quaterniond, AngleAxisd, Matrix<double,6,1>,
// plus Index.  It exists so that oracle/build_ref.sh can compile the reference's
// own .cpp files unchanged into oracle/_ref/ and pin the restated oracle against
// them.
//
// Arithmetic follows SURVEY.md Appendix A: Eigen 3.4, x86-64 SSE2 (2-lane double
// packets), no FMA, 16-byte aligned heap buffers.  Every expression is evaluated
// eagerly; element-wise expressions give the same IEEE results as Eigen's lazy
// evaluation, and the reductions/products whose association Eigen fixes are
// spelled out explicitly below (each cites its Appendix A item).  Fidelity to a
// real Eigen build is NOT verifiable here (no Eigen anywhere on the image).
#pragma once

#include <cassert>
#include <cmath>
#include <cstddef>
#include <initializer_list>
#include <limits>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
inline constexpr int Dynamic = -1;

template <typename S, int R, int C> class Matrix;

// ---------------------------------------------------------------- Vector3d
template <> class Matrix<double, 3, 1> {
 public:
  Matrix() : v_{0.0, 0.0, 0.0} {}
  template <typename A, typename B, typename C>
  Matrix(A x, B y, C z) : v_{static_cast<double>(x), static_cast<double>(y), static_cast<double>(z)} {}

  static Matrix Zero() { return Matrix(0.0, 0.0, 0.0); }
  static Matrix Constant(double c) { return Matrix(c, c, c); }
  static Matrix Unit(Index i) {
    Matrix m;
    m.v_[i] = 1.0;
    return m;
  }
  static Matrix UnitX() { return Unit(0); }
  static Matrix UnitY() { return Unit(1); }
  static Matrix UnitZ() { return Unit(2); }

  double &x() { return v_[0]; }
  double &y() { return v_[1]; }
  double &z() { return v_[2]; }
  double x() const { return v_[0]; }
  double y() const { return v_[1]; }
  double z() const { return v_[2]; }
  double &operator[](Index i) { return v_[i]; }
  double operator[](Index i) const { return v_[i]; }
  double &operator()(Index i) { return v_[i]; }
  double operator()(Index i) const { return v_[i]; }
  static constexpr Index size() { return 3; }
  static constexpr Index rows() { return 3; }
  static constexpr Index cols() { return 1; }

  Matrix operator+(const Matrix &o) const { return {v_[0] + o.v_[0], v_[1] + o.v_[1], v_[2] + o.v_[2]}; }
  Matrix operator-(const Matrix &o) const { return {v_[0] - o.v_[0], v_[1] - o.v_[1], v_[2] - o.v_[2]}; }
  Matrix operator-() const { return {-v_[0], -v_[1], -v_[2]}; }
  Matrix operator*(double s) const { return {v_[0] * s, v_[1] * s, v_[2] * s}; }
  Matrix operator/(double s) const { return {v_[0] / s, v_[1] / s, v_[2] / s}; }
  friend Matrix operator*(double s, const Matrix &m) { return {s * m.v_[0], s * m.v_[1], s * m.v_[2]}; }
  Matrix &operator+=(const Matrix &o) { return *this = *this + o; }
  Matrix &operator-=(const Matrix &o) { return *this = *this - o; }
  Matrix &operator*=(double s) { return *this = *this * s; }
  Matrix &operator/=(double s) { return *this = *this / s; }

  // Appendix A item 6: 3-element reductions are one 2-lane packet plus a scalar
  // tail, i.e. (a0 + a1) + a2.
  double squaredNorm() const { return (v_[0] * v_[0] + v_[1] * v_[1]) + v_[2] * v_[2]; }
  double norm() const { return std::sqrt(squaredNorm()); }
  double dot(const Matrix &o) const { return (v_[0] * o.v_[0] + v_[1] * o.v_[1]) + v_[2] * o.v_[2]; }
  double sum() const { return (v_[0] + v_[1]) + v_[2]; }
  Matrix normalized() const {
    const double n = squaredNorm();
    if (n > 0.0) return *this / std::sqrt(n);
    return *this;
  }
  void normalize() { *this = normalized(); }
  // Generic (non-vectorised) double cross product, Appendix A item 3.
  Matrix cross(const Matrix &b) const {
    return {v_[1] * b.v_[2] - v_[2] * b.v_[1], v_[2] * b.v_[0] - v_[0] * b.v_[2],
            v_[0] * b.v_[1] - v_[1] * b.v_[0]};
  }
  Matrix cwiseAbs() const { return {std::abs(v_[0]), std::abs(v_[1]), std::abs(v_[2])}; }
  Matrix cwiseProduct(const Matrix &o) const { return {v_[0] * o.v_[0], v_[1] * o.v_[1], v_[2] * o.v_[2]}; }
  double maxCoeff() const {
    double m = v_[0];
    for (int i = 1; i < 3; ++i) m = v_[i] > m ? v_[i] : m;
    return m;
  }
  bool allFinite() const { return std::isfinite(v_[0]) && std::isfinite(v_[1]) && std::isfinite(v_[2]); }
  void setZero() { v_[0] = v_[1] = v_[2] = 0.0; }
  const double *data() const { return v_; }

 private:
  double v_[3];
};
using Vector3d = Matrix<double, 3, 1>;

// ---------------------------------------------------------------- Vector4d
// Only what Quaterniond::coeffs() comparisons in the reference tests need.
template <> class Matrix<double, 4, 1> {
 public:
  Matrix() : v_{0, 0, 0, 0} {}
  Matrix(double a, double b, double c, double d) : v_{a, b, c, d} {}
  double operator[](Index i) const { return v_[i]; }
  double &operator[](Index i) { return v_[i]; }
  double operator()(Index i) const { return v_[i]; }
  Matrix operator-(const Matrix &o) const { return {v_[0] - o.v_[0], v_[1] - o.v_[1], v_[2] - o.v_[2], v_[3] - o.v_[3]}; }
  Matrix cwiseAbs() const { return {std::abs(v_[0]), std::abs(v_[1]), std::abs(v_[2]), std::abs(v_[3])}; }
  double maxCoeff() const {
    double m = v_[0];
    for (int i = 1; i < 4; ++i) m = v_[i] > m ? v_[i] : m;
    return m;
  }

 private:
  double v_[4];
};
using Vector4d = Matrix<double, 4, 1>;

// ---------------------------------------------- generic fixed column vector
// Matrix<double,6,1> (smiles.hpp FeatureVector) with the comma initialiser.
template <int R> class Matrix<double, R, 1> {
 public:
  Matrix() {
    for (int i = 0; i < R; ++i) v_[i] = 0.0;
  }
  double &operator()(Index i) { return v_[i]; }
  double operator()(Index i) const { return v_[i]; }
  double &operator[](Index i) { return v_[i]; }
  double operator[](Index i) const { return v_[i]; }
  static constexpr Index size() { return R; }
  static constexpr Index rows() { return R; }
  bool operator==(const Matrix &o) const {
    for (int i = 0; i < R; ++i)
      if (v_[i] != o.v_[i]) return false;
    return true;
  }
  struct Comma {
    Matrix *m;
    int at;
    Comma &operator,(double x) {
      m->v_[at++] = x;
      return *this;
    }
  };
  Comma operator<<(double x) {
    v_[0] = x;
    return Comma{this, 1};
  }

 private:
  double v_[R];
};

// ---------------------------------------------------------------- Matrix3Xd
template <> class Matrix<double, 3, Dynamic> {
 public:
  Matrix() = default;
  Matrix(Index rows, Index cols) : n_(cols), d_(static_cast<std::size_t>(3 * cols), 0.0) {
    assert(rows == 3);
    (void)rows;
  }
  Index rows() const { return 3; }
  Index cols() const { return n_; }
  Index size() const { return 3 * n_; }
  double &operator()(Index r, Index c) { return d_[static_cast<std::size_t>(3 * c + r)]; }
  double operator()(Index r, Index c) const { return d_[static_cast<std::size_t>(3 * c + r)]; }

  class Col {
   public:
    Col(Matrix *m, Index c) : m_(m), c_(c) {}
    Col &operator=(const Vector3d &v) {
      (*m_)(0, c_) = v.x();
      (*m_)(1, c_) = v.y();
      (*m_)(2, c_) = v.z();
      return *this;
    }
    Col &operator=(const Col &o) { return *this = Vector3d(o); }
    operator Vector3d() const { return {(*m_)(0, c_), (*m_)(1, c_), (*m_)(2, c_)}; }
    Vector3d eval() const { return Vector3d(*this); }
    double x() const { return (*m_)(0, c_); }
    double y() const { return (*m_)(1, c_); }
    double z() const { return (*m_)(2, c_); }
    double operator[](Index i) const { return (*m_)(i, c_); }
    double &operator[](Index i) { return (*m_)(i, c_); }
    void setZero() { *this = Vector3d::Zero(); }
    Col &operator+=(const Vector3d &v) { return *this = eval() + v; }
    Col &operator-=(const Vector3d &v) { return *this = eval() - v; }
    double norm() const { return eval().norm(); }
    double squaredNorm() const { return eval().squaredNorm(); }
    Vector3d operator+(const Vector3d &o) const { return eval() + o; }
    Vector3d operator-(const Vector3d &o) const { return eval() - o; }
    Vector3d operator*(double s) const { return eval() * s; }
    double dot(const Vector3d &o) const { return eval().dot(o); }
    Vector3d cross(const Vector3d &o) const { return eval().cross(o); }
    Vector3d normalized() const { return eval().normalized(); }

   private:
    Matrix *m_;
    Index c_;
  };

  Col col(Index c) { return Col(this, c); }
  Vector3d col(Index c) const { return {(*this)(0, c), (*this)(1, c), (*this)(2, c)}; }

  Matrix operator-(const Matrix &o) const {
    Matrix r(3, n_);
    for (std::size_t i = 0; i < d_.size(); ++i) r.d_[i] = d_[i] - o.d_[i];
    return r;
  }
  Matrix operator+(const Matrix &o) const {
    Matrix r(3, n_);
    for (std::size_t i = 0; i < d_.size(); ++i) r.d_[i] = d_[i] + o.d_[i];
    return r;
  }
  Matrix operator*(double s) const {
    Matrix r(3, n_);
    for (std::size_t i = 0; i < d_.size(); ++i) r.d_[i] = d_[i] * s;
    return r;
  }
  Matrix cwiseAbs() const {
    Matrix r(3, n_);
    for (std::size_t i = 0; i < d_.size(); ++i) r.d_[i] = std::abs(d_[i]);
    return r;
  }
  double maxCoeff() const {
    double m = -std::numeric_limits<double>::infinity();
    for (double x : d_) m = x > m ? x : m;
    return m;
  }
  bool allFinite() const {
    for (double x : d_)
      if (!std::isfinite(x)) return false;
    return true;
  }

  // colwise(): `+ v`, `+= v`, `.squaredNorm()` (returning a row whose .sum()
  // is sequential; only rmsd() uses it, which is off the hot path).
  struct Colwise {
    Matrix *self;
    const Matrix *cself;
    Matrix operator+(const Vector3d &v) const {
      Matrix r = *cself;
      for (Index c = 0; c < r.n_; ++c)
        for (int k = 0; k < 3; ++k) r(k, c) = (*cself)(k, c) + v[k];
      return r;
    }
    Colwise &operator+=(const Vector3d &v) {
      *self = *this + v;
      return *this;
    }
    struct Row {
      std::vector<double> v;
      double sum() const {
        double s = 0.0;
        if (v.empty()) return s;
        s = v[0];
        for (std::size_t i = 1; i < v.size(); ++i) s += v[i];
        return s;
      }
    };
    Row squaredNorm() const {
      Row row;
      for (Index c = 0; c < cself->n_; ++c) row.v.push_back(cself->col(c).squaredNorm());
      return row;
    }
  };
  Colwise colwise() { return Colwise{this, this}; }
  Colwise colwise() const { return Colwise{nullptr, this}; }

  // rowwise().mean(): Appendix A item 8 (Eigen 3.4).  Rows x and y share one
  // 2-lane packet and use packetwise_redux: p = c0; blocks of four
  // ((c_i + c_{i+1}) + (c_{i+2} + c_{i+3})) while i < ((N-1) & ~3); then a
  // sequential tail.  Row z is summed sequentially.  Then / double(N).
  struct Rowwise {
    const Matrix *m;
    Vector3d sum() const {
      const Index n = m->n_;
      Vector3d out;
      for (int r = 0; r < 2; ++r) {
        double p = (*m)(r, 0);
        const Index size4 = (n - 1) & ~Index(3);
        Index i = 1;
        for (; i < size4; i += 4)
          p = p + (((*m)(r, i) + (*m)(r, i + 1)) + ((*m)(r, i + 2) + (*m)(r, i + 3)));
        for (; i < n; ++i) p = p + (*m)(r, i);
        out[r] = p;
      }
      double z = (*m)(2, 0);
      for (Index i = 1; i < n; ++i) z = z + (*m)(2, i);
      out[2] = z;
      return out;
    }
    Vector3d mean() const {
      const Vector3d s = sum();
      const double n = static_cast<double>(m->n_);
      return {s.x() / n, s.y() / n, s.z() / n};
    }
  };
  Rowwise rowwise() const { return Rowwise{this}; }

  const double *data() const { return d_.data(); }

 private:
  Index n_ = 0;
  std::vector<double> d_;
};
using Matrix3Xd = Matrix<double, 3, Dynamic>;

// ---------------------------------------------------------------- Matrix3d
template <> class Matrix<double, 3, 3> {
 public:
  Matrix() : m_{} {}
  double &operator()(Index r, Index c) { return m_[r][c]; }
  double operator()(Index r, Index c) const { return m_[r][c]; }
  static Matrix Identity() {
    Matrix m;
    m.m_[0][0] = m.m_[1][1] = m.m_[2][2] = 1.0;
    return m;
  }

  // Appendix A item 4, Vector3d result: rows 0-1 are a 2-lane packet summed
  // left to right, row 2 is the scalar unroller's tree a0 + (a1 + a2).
  Vector3d operator*(const Vector3d &x) const {
    return {(m_[0][0] * x[0] + m_[0][1] * x[1]) + m_[0][2] * x[2],
            (m_[1][0] * x[0] + m_[1][1] * x[1]) + m_[1][2] * x[2],
            m_[2][0] * x[0] + (m_[2][1] * x[1] + m_[2][2] * x[2])};
  }
  // Appendix A item 4, 3xN result: slice-vectorised over the column-major
  // buffer; even columns have rows 0-1 packet + row 2 scalar, odd columns have
  // row 0 scalar + rows 1-2 packet.
  Matrix3Xd operator*(const Matrix3Xd &x) const {
    Matrix3Xd r(3, x.cols());
    for (Index c = 0; c < x.cols(); ++c) {
      const double a = x(0, c), b = x(1, c), d = x(2, c);
      for (int row = 0; row < 3; ++row) {
        const bool packet = (c % 2 == 0) ? (row < 2) : (row > 0);
        r(row, c) = packet ? (m_[row][0] * a + m_[row][1] * b) + m_[row][2] * d
                           : m_[row][0] * a + (m_[row][1] * b + m_[row][2] * d);
      }
    }
    return r;
  }

 private:
  double m_[3][3];
};
using Matrix3d = Matrix<double, 3, 3>;

// ---------------------------------------------------------------- AngleAxisd
class AngleAxisd {
 public:
  AngleAxisd() = default;
  AngleAxisd(double angle, const Vector3d &axis) : angle_(angle), axis_(axis) {}
  double angle() const { return angle_; }
  const Vector3d &axis() const { return axis_; }

  // Appendix A item 7.
  Matrix3d toRotationMatrix() const {
    Matrix3d r;
    const Vector3d sin_axis = std::sin(angle_) * axis_;
    const double c = std::cos(angle_);
    const Vector3d cos1_axis = (1.0 - c) * axis_;
    double tmp = cos1_axis.x() * axis_.y();
    r(0, 1) = tmp - sin_axis.z();
    r(1, 0) = tmp + sin_axis.z();
    tmp = cos1_axis.x() * axis_.z();
    r(0, 2) = tmp + sin_axis.y();
    r(2, 0) = tmp - sin_axis.y();
    tmp = cos1_axis.y() * axis_.z();
    r(1, 2) = tmp - sin_axis.x();
    r(2, 1) = tmp + sin_axis.x();
    r(0, 0) = cos1_axis.x() * axis_.x() + c;
    r(1, 1) = cos1_axis.y() * axis_.y() + c;
    r(2, 2) = cos1_axis.z() * axis_.z() + c;
    return r;
  }
  Vector3d operator*(const Vector3d &v) const { return toRotationMatrix() * v; }

 private:
  double angle_ = 0.0;
  Vector3d axis_ = Vector3d::UnitX();
};

// ---------------------------------------------------------------- Quaterniond
class Quaterniond {
 public:
  Quaterniond() : x_(0), y_(0), z_(0), w_(1) {}
  Quaterniond(double w, double x, double y, double z) : x_(x), y_(y), z_(z), w_(w) {}
  // Appendix A item 1.
  explicit Quaterniond(const AngleAxisd &aa) {
    const double ha = 0.5 * aa.angle();
    w_ = std::cos(ha);
    const double s = std::sin(ha);
    x_ = s * aa.axis().x();
    y_ = s * aa.axis().y();
    z_ = s * aa.axis().z();
  }
  static Quaterniond Identity() { return Quaterniond(1.0, 0.0, 0.0, 0.0); }

  double w() const { return w_; }
  double x() const { return x_; }
  double y() const { return y_; }
  double z() const { return z_; }
  double &w() { return w_; }
  double &x() { return x_; }
  double &y() { return y_; }
  double &z() { return z_; }
  Vector3d vec() const { return {x_, y_, z_}; }
  Vector4d coeffs() const { return {x_, y_, z_, w_}; }

  // Appendix A item 5 (Eigen 3.4 Geometry_SIMD.h double specialisation).
  Quaterniond operator*(const Quaterniond &b) const {
    const double aw = w_, ax = x_, ay = y_, az = z_;
    const double bw = b.w_, bx = b.x_, by = b.y_, bz = b.z_;
    Quaterniond r;
    r.x_ = (aw * bx + ay * bz) - (az * by - ax * bw);
    r.y_ = (aw * by + ay * bw) + (az * bx - ax * bz);
    r.z_ = (aw * bz - ay * bx) + (az * bw + ax * by);
    r.w_ = (aw * bw - ay * by) - (az * bz + ax * bx);
    return r;
  }
  // Appendix A item 3 (_transformVector).
  Vector3d operator*(const Vector3d &v) const {
    const Vector3d q(x_, y_, z_);
    Vector3d uv = q.cross(v);
    uv = uv + uv;
    return (v + w_ * uv) + q.cross(uv);
  }
  // Appendix A item 6: (x^2 + z^2) + (y^2 + w^2), then divide.
  double squaredNorm() const { return (x_ * x_ + z_ * z_) + (y_ * y_ + w_ * w_); }
  double norm() const { return std::sqrt(squaredNorm()); }
  Quaterniond normalized() const {
    const double n = norm();
    Quaterniond r;
    r.x_ = x_ / n;
    r.y_ = y_ / n;
    r.z_ = z_ / n;
    r.w_ = w_ / n;
    return r;
  }
  void normalize() { *this = normalized(); }
  Quaterniond conjugate() const { return Quaterniond(w_, -x_, -y_, -z_); }

  // Appendix A item 2.
  Matrix3d toRotationMatrix() const {
    Matrix3d r;
    const double tx = 2.0 * x_, ty = 2.0 * y_, tz = 2.0 * z_;
    const double twx = tx * w_, twy = ty * w_, twz = tz * w_;
    const double txx = tx * x_, txy = ty * x_, txz = tz * x_;
    const double tyy = ty * y_, tyz = tz * y_, tzz = tz * z_;
    r(0, 0) = 1.0 - (tyy + tzz);
    r(0, 1) = txy - twz;
    r(0, 2) = txz + twy;
    r(1, 0) = txy + twz;
    r(1, 1) = 1.0 - (txx + tzz);
    r(1, 2) = tyz - twx;
    r(2, 0) = txz - twy;
    r(2, 1) = tyz + twx;
    r(2, 2) = 1.0 - (txx + tyy);
    return r;
  }

 private:
  double x_, y_, z_, w_;
};

}  // namespace Eigen
