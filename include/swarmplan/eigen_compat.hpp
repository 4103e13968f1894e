// eigen_compat.hpp — the reference's public C++ API spells its matrices as
// Eigen::MatrixXd / Eigen::VectorXd (/root/reference/proj/include/swarmplan/
// model.hpp:68-76, lp.hpp:30-33, groups.hpp:26-37). When the real Eigen is on
// the include path it is used as-is; otherwise this header provides the small
// dense subset those signatures and their callers use (column-major storage,
// Zero/Constant, element access, row views, comma initialization, dot).
#pragma once

#if __has_include(<Eigen/Dense>) && !defined(SWARMPLAN_NO_EIGEN)
#include <Eigen/Dense>
#else
#include <cassert>
#include <cmath>
#include <cstddef>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;

class VectorXd;

// Comma initializer: `v << 1.0, 2.0;`
template <class V>
class CommaInit {
 public:
  CommaInit(V& v, double first) : v_(v), i_(0) { v_.coeffRef(i_++) = first; }
  CommaInit& operator,(double x) {
    v_.coeffRef(i_++) = x;
    return *this;
  }

 private:
  V& v_;
  Index i_;
};

class VectorXd {
 public:
  VectorXd() = default;
  explicit VectorXd(Index n) : d_(static_cast<std::size_t>(n), 0.0) {}
  static VectorXd Zero(Index n) { return VectorXd(n); }
  static VectorXd Constant(Index n, double v) {
    VectorXd r(n);
    for (auto& x : r.d_) x = v;
    return r;
  }
  Index size() const { return static_cast<Index>(d_.size()); }
  Index rows() const { return size(); }
  Index cols() const { return 1; }
  void resize(Index n) { d_.assign(static_cast<std::size_t>(n), 0.0); }
  void setZero() {
    for (auto& x : d_) x = 0.0;
  }
  double& operator()(Index i) { return d_[static_cast<std::size_t>(i)]; }
  double operator()(Index i) const { return d_[static_cast<std::size_t>(i)]; }
  double& operator[](Index i) { return d_[static_cast<std::size_t>(i)]; }
  double operator[](Index i) const { return d_[static_cast<std::size_t>(i)]; }
  double& coeffRef(Index i) { return d_[static_cast<std::size_t>(i)]; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double dot(const VectorXd& o) const {
    double s = 0.0;
    for (std::size_t i = 0; i < d_.size(); ++i) s += d_[i] * o.d_[i];
    return s;
  }
  double squaredNorm() const { return dot(*this); }
  double norm() const { return std::sqrt(squaredNorm()); }
  CommaInit<VectorXd> operator<<(double x) { return CommaInit<VectorXd>(*this, x); }
  VectorXd& operator+=(const VectorXd& o) {
    for (std::size_t i = 0; i < d_.size(); ++i) d_[i] += o.d_[i];
    return *this;
  }
  VectorXd operator*(double s) const {
    VectorXd r = *this;
    for (auto& x : r.d_) x *= s;
    return r;
  }
  VectorXd operator/(double s) const {
    VectorXd r = *this;
    for (auto& x : r.d_) x /= s;
    return r;
  }
  const VectorXd& transpose() const { return *this; }
  bool operator==(const VectorXd& o) const { return d_ == o.d_; }

 private:
  std::vector<double> d_;
};

class MatrixXd {
 public:
  class RowRef {
   public:
    RowRef(MatrixXd& m, Index r) : m_(m), r_(r) {}
    double& operator()(Index c) { return m_(r_, c); }
    Index size() const { return m_.cols(); }
    RowRef& operator=(const VectorXd& v) {
      assert(v.size() == m_.cols());
      for (Index c = 0; c < m_.cols(); ++c) m_(r_, c) = v(c);
      return *this;
    }
    VectorXd transpose() const { return static_cast<VectorXd>(*this); }
    operator VectorXd() const {
      VectorXd v(m_.cols());
      for (Index c = 0; c < m_.cols(); ++c) v(c) = m_(r_, c);
      return v;
    }

   private:
    MatrixXd& m_;
    Index r_;
  };
  class ConstRowRef {
   public:
    ConstRowRef(const MatrixXd& m, Index r) : m_(m), r_(r) {}
    double operator()(Index c) const { return m_(r_, c); }
    Index size() const { return m_.cols(); }
    VectorXd transpose() const { return static_cast<VectorXd>(*this); }
    operator VectorXd() const {
      VectorXd v(m_.cols());
      for (Index c = 0; c < m_.cols(); ++c) v(c) = m_(r_, c);
      return v;
    }

   private:
    const MatrixXd& m_;
    Index r_;
  };

  MatrixXd() = default;
  MatrixXd(Index r, Index c) : r_(r), c_(c), d_(static_cast<std::size_t>(r * c), 0.0) {}
  static MatrixXd Zero(Index r, Index c) { return MatrixXd(r, c); }
  static MatrixXd Constant(Index r, Index c, double v) {
    MatrixXd m(r, c);
    for (auto& x : m.d_) x = v;
    return m;
  }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  void resize(Index r, Index c) {
    r_ = r;
    c_ = c;
    d_.assign(static_cast<std::size_t>(r * c), 0.0);
  }
  void setZero() {
    for (auto& x : d_) x = 0.0;
  }
  double& operator()(Index i, Index j) { return d_[static_cast<std::size_t>(j * r_ + i)]; }
  double operator()(Index i, Index j) const { return d_[static_cast<std::size_t>(j * r_ + i)]; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  RowRef row(Index i) { return RowRef(*this, i); }
  ConstRowRef row(Index i) const { return ConstRowRef(*this, i); }
  bool operator==(const MatrixXd& o) const { return r_ == o.r_ && c_ == o.c_ && d_ == o.d_; }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> d_;
};

}  // namespace Eigen
#endif
