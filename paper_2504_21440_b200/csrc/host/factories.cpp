// Operator/state factories and superoperators (factories.cpp:23-246, superop.cpp:5-91 semantics).
#include <algorithm>
#include <cmath>
#include <tuple>

#include "../../../include/qsim/factories.hpp"

namespace qsim {

namespace {

void require_mode_dim(int n) { require(n >= 1, ErrorCode::InvalidDimension, "mode dimension must be >= 1"); }

// Build an n x n CSR from (row, col, value) entries given in row-major order.
SparseMatrix from_entries(long n, std::vector<std::tuple<long, long, Complex>> e) {
  SparseMatrix m = SparseMatrix::empty(n, n);
  std::stable_sort(e.begin(), e.end(), [](const auto& a, const auto& b) {
    return std::get<0>(a) != std::get<0>(b) ? std::get<0>(a) < std::get<0>(b) : std::get<1>(a) < std::get<1>(b);
  });
  for (const auto& [r, c, v] : e) {
    m.col.push_back(static_cast<int32_t>(c));
    m.val.push_back(v);
    m.rowptr[static_cast<size_t>(r + 1)]++;
  }
  for (long r = 0; r < n; ++r) m.rowptr[static_cast<size_t>(r + 1)] += m.rowptr[static_cast<size_t>(r)];
  return m;
}

}  // namespace

QuantumObject destroy(int n) {  // factories.cpp:23-28
  require_mode_dim(n);
  std::vector<std::tuple<long, long, Complex>> e;
  for (int k = 1; k < n; ++k) e.emplace_back(k - 1, k, std::sqrt(static_cast<double>(k)));
  return QuantumObject(from_entries(n, std::move(e)), Kind::Operator, {n});
}
QuantumObject create(int n) { return dag(destroy(n)); }
QuantumObject num(int n) {
  require_mode_dim(n);
  std::vector<std::tuple<long, long, Complex>> e;
  for (int k = 1; k < n; ++k) e.emplace_back(k, k, static_cast<double>(k));
  return QuantumObject(from_entries(n, std::move(e)), Kind::Operator, {n});
}
QuantumObject qeye(int n) {
  require_mode_dim(n);
  return QuantumObject(SparseMatrix::identity(n), Kind::Operator, {n});
}
QuantumObject qeye(const Dims& dims) {
  return QuantumObject(SparseMatrix::identity(dims_product(dims)), Kind::Operator, dims);
}
QuantumObject position(int n) { return (destroy(n) + create(n)) / std::sqrt(2.0); }
QuantumObject momentum(int n) { return Complex(0.0, 1.0) * (create(n) - destroy(n)) / std::sqrt(2.0); }

QuantumObject sigmax() {
  return QuantumObject(from_entries(2, {{0, 1, 1.0}, {1, 0, 1.0}}), Kind::Operator, {2});
}
QuantumObject sigmay() {
  return QuantumObject(from_entries(2, {{0, 1, Complex(0, -1)}, {1, 0, Complex(0, 1)}}), Kind::Operator, {2});
}
QuantumObject sigmaz() {
  return QuantumObject(from_entries(2, {{0, 0, 1.0}, {1, 1, -1.0}}), Kind::Operator, {2});
}
QuantumObject sigmap() { return QuantumObject(from_entries(2, {{0, 1, 1.0}}), Kind::Operator, {2}); }
QuantumObject sigmam() { return dag(sigmap()); }

QuantumObject basis(int n, int i) {
  require_mode_dim(n);
  require(i >= 0 && i < n, ErrorCode::InvalidIndex, "basis index out of range");
  DenseMatrix v(n, 1);
  v(i, 0) = 1.0;
  return QuantumObject(std::move(v), Kind::Ket, {n});
}
QuantumObject fock(int n, int i) { return basis(n, i); }
QuantumObject fock_dm(int n, int i) {
  require_mode_dim(n);
  require(i >= 0 && i < n, ErrorCode::InvalidIndex, "fock_dm index out of range");
  return QuantumObject(from_entries(n, {{i, i, 1.0}}), Kind::Operator, {n});
}
QuantumObject projection(int n, int i, int j) {
  require_mode_dim(n);
  require(i >= 0 && i < n && j >= 0 && j < n, ErrorCode::InvalidIndex, "projection index out of range");
  return QuantumObject(from_entries(n, {{i, j, 1.0}}), Kind::Operator, {n});
}
QuantumObject thermal_dm(int n, double nbar) {  // factories.cpp:108-126
  require_mode_dim(n);
  require(nbar >= 0.0, ErrorCode::InvalidDimension, "thermal occupation must be >= 0");
  std::vector<std::tuple<long, long, Complex>> e;
  if (nbar == 0.0) {
    e.emplace_back(0, 0, 1.0);
  } else {
    const double q = nbar / (1.0 + nbar);
    double w = 1.0, total = 0.0;
    std::vector<double> weights(static_cast<size_t>(n));
    for (int k = 0; k < n; ++k) {
      weights[static_cast<size_t>(k)] = w;
      total += w;
      w *= q;
    }
    for (int k = 0; k < n; ++k) e.emplace_back(k, k, weights[static_cast<size_t>(k)] / total);
  }
  return QuantumObject(from_entries(n, std::move(e)), Kind::Operator, {n});
}
QuantumObject maximally_mixed_dm(int n) {
  require_mode_dim(n);
  std::vector<std::tuple<long, long, Complex>> e;
  for (int k = 0; k < n; ++k) e.emplace_back(k, k, 1.0 / n);
  return QuantumObject(from_entries(n, std::move(e)), Kind::Operator, {n});
}
QuantumObject coherent(int n, Complex alpha) {  // factories.cpp:135-146
  require(n >= 2 || std::abs(alpha) == 0.0, ErrorCode::InvalidDimension, "coherent needs n >= 2 for nonzero alpha");
  DenseMatrix v(n, 1);
  Complex c = std::exp(-0.5 * std::norm(alpha));
  for (int k = 0; k < n; ++k) {
    v(k, 0) = c;
    c *= alpha / std::sqrt(static_cast<double>(k + 1));
  }
  double s = 0.0;
  for (int k = 0; k < n; ++k) s += std::norm(v(k, 0));
  const double nrm = std::sqrt(s);
  for (int k = 0; k < n; ++k) v(k, 0) /= nrm;
  return QuantumObject(std::move(v), Kind::Ket, {n});
}
QuantumObject coherent_dm(int n, Complex alpha) { return ket2dm(coherent(n, alpha)); }

QuantumObject embed_site(const Dims& dims, int site, const QuantumObject& op) {  // :192-202
  require(site >= 0 && site < static_cast<int>(dims.size()), ErrorCode::InvalidSubsystem,
          "embed_site: site out of range");
  require(op.is_operator() && op.dims().size() == 1 && op.dims()[0] == dims[static_cast<size_t>(site)],
          ErrorCode::DimsMismatch, "embed_site: operator does not match the site dimension");
  QuantumObject out = (site == 0) ? op : qeye(dims[0]);
  for (size_t i = 1; i < dims.size(); ++i) out = tensor(out, static_cast<int>(i) == site ? op : qeye(dims[i]));
  return out;
}

namespace {
std::pair<QuantumObject, std::vector<QuantumObject>> ising_impl(int nx, int ny, double jz, double hx,
                                                                double gamma, bool periodic) {
  // factories.cpp:204-246: sweep right/down, periodic wraps as separate bond terms, bonds first
  const int ns = nx * ny;
  Dims dims(static_cast<size_t>(ns), 2);
  auto site_of = [nx](int x, int y) { return y * nx + x; };
  std::vector<std::pair<int, int>> bonds;
  for (int y = 0; y < ny; ++y)
    for (int x = 0; x < nx; ++x) {
      if (x + 1 < nx) bonds.emplace_back(site_of(x, y), site_of(x + 1, y));
      else if (periodic && nx > 1) bonds.emplace_back(site_of(x, y), site_of(0, y));
      if (y + 1 < ny) bonds.emplace_back(site_of(x, y), site_of(x, y + 1));
      else if (periodic && ny > 1) bonds.emplace_back(site_of(x, y), site_of(x, 0));
    }
  const long d = dims_product(dims);
  QuantumObject hq(SparseMatrix::empty(d, d), Kind::Operator, dims);
  bool first = true;
  std::vector<QuantumObject> sz, sx;
  for (int i = 0; i < ns; ++i) sz.push_back(embed_site(dims, i, sigmaz()));
  for (auto [i, j] : bonds) {
    QuantumObject term = jz * (sz[static_cast<size_t>(i)] * sz[static_cast<size_t>(j)]);
    hq = first ? term : hq + term;
    first = false;
  }
  for (int i = 0; i < ns; ++i) {
    QuantumObject term = hx * embed_site(dims, i, sigmax());
    hq = first ? term : hq + term;
    first = false;
  }
  std::vector<QuantumObject> c_ops;
  const double amp = std::sqrt(gamma);
  for (int i = 0; i < ns; ++i) c_ops.push_back(amp * embed_site(dims, i, sigmam()));
  return {hq, c_ops};
}
}  // namespace

std::pair<QuantumObject, std::vector<QuantumObject>> ising_model(int nx, int ny, double jz, double hx,
                                                                 double gamma, bool periodic) {
  require(nx >= 1 && ny >= 1, ErrorCode::InvalidDimension, "lattice extents must be >= 1");
  require(nx * ny <= 12, ErrorCode::TooLarge, "lattice capped at 12 sites");
  return ising_impl(nx, ny, jz, hx, gamma, periodic);
}

std::pair<QuantumObject, std::vector<QuantumObject>> ising_model_uncapped(int nx, int ny, double jz, double hx,
                                                                          double gamma, bool periodic) {
  require(nx >= 1 && ny >= 1, ErrorCode::InvalidDimension, "lattice extents must be >= 1");
  require(nx * ny <= 24, ErrorCode::TooLarge, "state vector would exceed int32 indexing");
  return ising_impl(nx, ny, jz, hx, gamma, periodic);
}

// ---- superoperators (superop.cpp) ------------------------------------------------------------
QuantumObject mat2vec(const QuantumObject& rho) {
  require(rho.is_operator(), ErrorCode::KindMismatch, "mat2vec expects an Operator");
  const long d = rho.dim();
  const DenseMatrix m = rho.dense_matrix();
  DenseMatrix v(d * d, 1);
  for (long j = 0; j < d; ++j)
    for (long i = 0; i < d; ++i) v(j * d + i, 0) = m(i, j);
  return QuantumObject(std::move(v), Kind::OperatorKet, rho.dims());
}
QuantumObject vec2mat(const QuantumObject& v) {
  require(v.kind() == Kind::OperatorKet, ErrorCode::KindMismatch, "vec2mat expects an OperatorKet");
  const long d = v.dim();
  const DenseMatrix c = v.dense_matrix();
  DenseMatrix m(d, d);
  for (long j = 0; j < d; ++j)
    for (long i = 0; i < d; ++i) m(i, j) = c(j * d + i, 0);
  return QuantumObject(std::move(m), Kind::Operator, v.dims());
}
QuantumObject spre(const QuantumObject& a) {  // superop.cpp:51-55
  require(a.is_operator(), ErrorCode::KindMismatch, "spre expects an Operator");
  return QuantumObject(sparse_kron(SparseMatrix::identity(a.dim()), a.sparse_matrix()), Kind::SuperOperator, a.dims());
}
QuantumObject spost(const QuantumObject& b) {  // superop.cpp:57-61
  require(b.is_operator(), ErrorCode::KindMismatch, "spost expects an Operator");
  return QuantumObject(sparse_kron(sparse_transpose(b.sparse_matrix(), false), SparseMatrix::identity(b.dim())),
                       Kind::SuperOperator, b.dims());
}
QuantumObject sprepost(const QuantumObject& a, const QuantumObject& b) {  // superop.cpp:63-69
  require(a.is_operator() && b.is_operator(), ErrorCode::KindMismatch, "sprepost expects Operators");
  require(a.dims() == b.dims(), ErrorCode::DimsMismatch, "sprepost: dims mismatch");
  return QuantumObject(sparse_kron(sparse_transpose(b.sparse_matrix(), false), a.sparse_matrix()),
                       Kind::SuperOperator, a.dims());
}
QuantumObject lindblad_dissipator(const QuantumObject& c) {  // superop.cpp:71-76
  require(c.is_operator(), ErrorCode::KindMismatch, "lindblad_dissipator expects an Operator");
  const QuantumObject cd = dag(c);
  const QuantumObject cdc = cd * c;
  return sprepost(c, cd) - 0.5 * spre(cdc) - 0.5 * spost(cdc);
}
QuantumObject liouvillian(const QuantumObject& h, std::span<const QuantumObject> c_ops) {  // :78-91
  QuantumObject l;
  if (h.is_superoperator()) {
    l = h;
  } else {
    require(h.is_operator(), ErrorCode::KindMismatch, "liouvillian expects an Operator");
    l = Complex(0, -1) * (spre(h) - spost(h));
  }
  for (const auto& c : c_ops) {
    require(c.dims() == l.dims(), ErrorCode::DimsMismatch, "liouvillian: collapse dims mismatch");
    l = l + lindblad_dissipator(c);
  }
  return l;
}

}  // namespace qsim
