// TEST INFRASTRUCTURE ONLY — see qsim_oracle.hpp for scope and provenance.
// Every function cites the reference file:line whose arithmetic order it restates.
#include "qsim_oracle.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <numbers>
#include <thread>

namespace orc {

// ---- worker pool (threads() > 1 only; see qsim_oracle.hpp) -------------------------------
namespace {
class Pool {
 public:
  explicit Pool(int n) : n_(n) {
    for (int i = 1; i < n_; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return n_; }
  // f(tid) on every worker and the caller; returns when all are done
  void run(const std::function<void(int)>& f) {
    {
      std::lock_guard<std::mutex> g(m_);
      job_ = &f;
      pending_ = n_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    f(0);
    std::unique_lock<std::mutex> g(m_);
    done_.wait(g, [this] { return pending_ == 0; });
  }

 private:
  void loop(int tid) {
    long seen = 0;
    for (;;) {
      const std::function<void(int)>* f;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        f = job_;
      }
      (*f)(tid);
      std::lock_guard<std::mutex> g(m_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int pending_ = 0;
  long gen_ = 0;
  bool stop_ = false;
};
int g_threads = 1;
std::unique_ptr<Pool> g_pool;

// f(lo, hi) over a static split of [0, n)
template <class F>
void par_for(size_t n, F&& f, size_t min_n = 4096) {
  if (g_threads <= 1 || n < min_n) {
    f(size_t{0}, n);
    return;
  }
  const size_t T = static_cast<size_t>(g_pool->size());
  const std::function<void(int)> job = [&](int tid) {
    const size_t lo = n * static_cast<size_t>(tid) / T, hi = n * static_cast<size_t>(tid + 1) / T;
    if (lo < hi) f(lo, hi);
  };
  g_pool->run(job);
}
}  // namespace

void set_threads(int n) {
  n = std::max(1, n);
  if (n == g_threads) return;
  g_pool.reset();
  g_threads = n;
  if (n > 1) g_pool = std::make_unique<Pool>(n);
}
int threads() { return g_threads; }

const char* error_code_name(ErrorCode c) {  // qobj.cpp:24-40
  switch (c) {
    case ErrorCode::KindMismatch: return "KindMismatch";
    case ErrorCode::DimsMismatch: return "DimsMismatch";
    case ErrorCode::InvalidSubsystem: return "InvalidSubsystem";
    case ErrorCode::InvalidDimension: return "InvalidDimension";
    case ErrorCode::InvalidIndex: return "InvalidIndex";
    case ErrorCode::TooLarge: return "TooLarge";
    case ErrorCode::IntegrationFailure: return "IntegrationFailure";
    case ErrorCode::EnsembleFailure: return "EnsembleFailure";
    case ErrorCode::SteadyStateFailure: return "SteadyStateFailure";
    case ErrorCode::DfdOverflow: return "DfdOverflow";
    case ErrorCode::InvalidGrid: return "InvalidGrid";
    case ErrorCode::InvalidScenario: return "InvalidScenario";
  }
  return "?";
}

void throw_error(ErrorCode c, const std::string& m) { throw Error(c, m); }

// ======================================================================================
// Eigen sparse semantics
// ======================================================================================

// SparseMatrix::setFromTriplets: duplicates are summed in insertion order (first value
// assigned, later ones added) and rows end up sorted within each column.
Csc from_triplets(long rows, long cols, std::vector<Triplet> trips) {
  std::stable_sort(trips.begin(), trips.end(), [](const Triplet& a, const Triplet& b) {
    return a.c != b.c ? a.c < b.c : a.r < b.r;
  });
  Csc m;
  m.rows = rows;
  m.cols = cols;
  m.outer.assign(static_cast<size_t>(cols + 1), 0);
  m.inner.reserve(trips.size());
  m.val.reserve(trips.size());
  size_t k = 0;
  for (long c = 0; c < cols; ++c) {
    m.outer[static_cast<size_t>(c)] = static_cast<int>(m.val.size());
    while (k < trips.size() && trips[k].c == c) {
      const long r = trips[k].r;
      cd v = trips[k].v;
      ++k;
      while (k < trips.size() && trips[k].c == c && trips[k].r == r) v += trips[k++].v;
      m.inner.push_back(static_cast<int>(r));
      m.val.push_back(v);
    }
  }
  m.outer[static_cast<size_t>(cols)] = static_cast<int>(m.val.size());
  return m;
}

Csc sp_identity(long n) {
  Csc m;
  m.rows = m.cols = n;
  m.outer.resize(static_cast<size_t>(n + 1));
  m.inner.resize(static_cast<size_t>(n));
  m.val.assign(static_cast<size_t>(n), cd(1.0, 0.0));
  for (long i = 0; i <= n; ++i) m.outer[static_cast<size_t>(i)] = static_cast<int>(i);
  for (long i = 0; i < n; ++i) m.inner[static_cast<size_t>(i)] = static_cast<int>(i);
  return m;
}

// Eigen sparse binary evaluator (union): f(a,b) where both present, f(a,0) / f(0,b) otherwise.
Csc sp_add(const Csc& a, const Csc& b) {
  Csc m;
  m.rows = a.rows;
  m.cols = a.cols;
  m.outer.assign(static_cast<size_t>(a.cols + 1), 0);
  m.inner.reserve(static_cast<size_t>(a.nnz() + b.nnz()));
  m.val.reserve(static_cast<size_t>(a.nnz() + b.nnz()));
  for (long c = 0; c < a.cols; ++c) {
    m.outer[static_cast<size_t>(c)] = static_cast<int>(m.val.size());
    int ia = a.outer[static_cast<size_t>(c)], ea = a.outer[static_cast<size_t>(c + 1)];
    int ib = b.outer[static_cast<size_t>(c)], eb = b.outer[static_cast<size_t>(c + 1)];
    while (ia < ea || ib < eb) {
      if (ia < ea && ib < eb && a.inner[static_cast<size_t>(ia)] == b.inner[static_cast<size_t>(ib)]) {
        m.inner.push_back(a.inner[static_cast<size_t>(ia)]);
        m.val.push_back(a.val[static_cast<size_t>(ia)] + b.val[static_cast<size_t>(ib)]);
        ++ia;
        ++ib;
      } else if (ia < ea && (ib >= eb || a.inner[static_cast<size_t>(ia)] < b.inner[static_cast<size_t>(ib)])) {
        m.inner.push_back(a.inner[static_cast<size_t>(ia)]);
        m.val.push_back(a.val[static_cast<size_t>(ia)] + cd(0.0, 0.0));
        ++ia;
      } else {
        m.inner.push_back(b.inner[static_cast<size_t>(ib)]);
        m.val.push_back(cd(0.0, 0.0) + b.val[static_cast<size_t>(ib)]);
        ++ib;
      }
    }
  }
  m.outer[static_cast<size_t>(a.cols)] = static_cast<int>(m.val.size());
  return m;
}

Csc sp_scale(cd s, const Csc& a) {
  Csc m = a;
  for (auto& v : m.val) v = s * v;
  return m;
}

// Eigen conservative_sparse_sparse_product_impl: for every rhs column j, walk its entries
// (k, y) and accumulate lhs(:,k)*y, first contribution assigned. Rows are sorted after.
Csc sp_mul(const Csc& a, const Csc& b) {
  Csc m;
  m.rows = a.rows;
  m.cols = b.cols;
  m.outer.assign(static_cast<size_t>(b.cols + 1), 0);
  std::vector<char> mask(static_cast<size_t>(a.rows), 0);
  std::vector<cd> values(static_cast<size_t>(a.rows));
  std::vector<int> idx;
  for (long j = 0; j < b.cols; ++j) {
    m.outer[static_cast<size_t>(j)] = static_cast<int>(m.val.size());
    idx.clear();
    for (int pb = b.outer[static_cast<size_t>(j)]; pb < b.outer[static_cast<size_t>(j + 1)]; ++pb) {
      const cd y = b.val[static_cast<size_t>(pb)];
      const int k = b.inner[static_cast<size_t>(pb)];
      for (int pa = a.outer[static_cast<size_t>(k)]; pa < a.outer[static_cast<size_t>(k + 1)]; ++pa) {
        const int i = a.inner[static_cast<size_t>(pa)];
        const cd x = a.val[static_cast<size_t>(pa)];
        if (!mask[static_cast<size_t>(i)]) {
          mask[static_cast<size_t>(i)] = 1;
          values[static_cast<size_t>(i)] = x * y;
          idx.push_back(i);
        } else {
          values[static_cast<size_t>(i)] += x * y;
        }
      }
    }
    std::sort(idx.begin(), idx.end());
    for (int i : idx) {
      m.inner.push_back(i);
      m.val.push_back(values[static_cast<size_t>(i)]);
      mask[static_cast<size_t>(i)] = 0;
    }
  }
  m.outer[static_cast<size_t>(b.cols)] = static_cast<int>(m.val.size());
  return m;
}

static Csc transpose_impl(const Csc& a, bool conjugate) {
  Csc m;
  m.rows = a.cols;
  m.cols = a.rows;
  m.outer.assign(static_cast<size_t>(a.rows + 1), 0);
  for (int r : a.inner) ++m.outer[static_cast<size_t>(r + 1)];
  for (long i = 0; i < a.rows; ++i) m.outer[static_cast<size_t>(i + 1)] += m.outer[static_cast<size_t>(i)];
  std::vector<int> pos(m.outer.begin(), m.outer.end() - 1);
  m.inner.resize(a.inner.size());
  m.val.resize(a.val.size());
  for (long c = 0; c < a.cols; ++c)
    for (int p = a.outer[static_cast<size_t>(c)]; p < a.outer[static_cast<size_t>(c + 1)]; ++p) {
      const int r = a.inner[static_cast<size_t>(p)];
      const int q = pos[static_cast<size_t>(r)]++;
      m.inner[static_cast<size_t>(q)] = static_cast<int>(c);
      m.val[static_cast<size_t>(q)] = conjugate ? std::conj(a.val[static_cast<size_t>(p)]) : a.val[static_cast<size_t>(p)];
    }
  return m;
}
Csc sp_transpose(const Csc& a) { return transpose_impl(a, false); }
Csc sp_adjoint(const Csc& a) { return transpose_impl(a, true); }

// superop.cpp:31-43 / qobj.cpp:240-253: triplets in (a col, a entry, b col, b entry) order.
Csc sp_kron(const Csc& a, const Csc& b) {
  std::vector<Triplet> trips;
  trips.reserve(static_cast<size_t>(a.nnz()) * static_cast<size_t>(b.nnz()));
  for (long ka = 0; ka < a.cols; ++ka)
    for (int pa = a.outer[static_cast<size_t>(ka)]; pa < a.outer[static_cast<size_t>(ka + 1)]; ++pa)
      for (long kb = 0; kb < b.cols; ++kb)
        for (int pb = b.outer[static_cast<size_t>(kb)]; pb < b.outer[static_cast<size_t>(kb + 1)]; ++pb)
          trips.push_back({a.inner[static_cast<size_t>(pa)] * b.rows + b.inner[static_cast<size_t>(pb)],
                           ka * b.cols + kb, a.val[static_cast<size_t>(pa)] * b.val[static_cast<size_t>(pb)]});
  return from_triplets(a.rows * b.rows, a.cols * b.cols, std::move(trips));
}

Dense sp_to_dense(const Csc& a) {
  Dense d(a.rows, a.cols);
  for (long c = 0; c < a.cols; ++c)
    for (int p = a.outer[static_cast<size_t>(c)]; p < a.outer[static_cast<size_t>(c + 1)]; ++p)
      d(a.inner[static_cast<size_t>(p)], c) = a.val[static_cast<size_t>(p)];
  return d;
}

Csc dense_to_sp(const Dense& a) {
  Csc m;
  m.rows = a.rows;
  m.cols = a.cols;
  m.outer.assign(static_cast<size_t>(a.cols + 1), 0);
  for (long c = 0; c < a.cols; ++c) {
    m.outer[static_cast<size_t>(c)] = static_cast<int>(m.val.size());
    for (long r = 0; r < a.rows; ++r)
      if (a(r, c) != cd(0.0, 0.0)) {
        m.inner.push_back(static_cast<int>(r));
        m.val.push_back(a(r, c));
      }
  }
  m.outer[static_cast<size_t>(a.cols)] = static_cast<int>(m.val.size());
  return m;
}

// Eigen sparse_time_dense_product (col-major lhs): res.setZero(); for each column j,
// rhs_j = alpha*y[j] (alpha = 1); res[i] += v * rhs_j.
void sp_gemv(const Csc& a, const cd* y, cd* out) {
  for (long i = 0; i < a.rows; ++i) out[i] = cd(0.0, 0.0);
  for (long j = 0; j < a.cols; ++j) {
    const cd rj = cd(1.0, 0.0) * y[j];
    for (int p = a.outer[static_cast<size_t>(j)]; p < a.outer[static_cast<size_t>(j + 1)]; ++p)
      out[a.inner[static_cast<size_t>(p)]] += a.val[static_cast<size_t>(p)] * rj;
  }
}

// ---- dense helpers (Eigen dense expressions, only used at desk-scale sizes) ---------------
static Dense d_add(const Dense& a, const Dense& b) {
  Dense m(a.rows, a.cols);
  for (size_t i = 0; i < m.v.size(); ++i) m.v[i] = a.v[i] + b.v[i];
  return m;
}
static Dense d_scale(cd s, const Dense& a) {
  Dense m = a;
  for (auto& v : m.v) v = s * v;
  return m;
}
static Dense d_mul(const Dense& a, const Dense& b) {
  Dense m(a.rows, b.cols);
  for (long j = 0; j < b.cols; ++j)
    for (long k = 0; k < a.cols; ++k) {
      const cd y = b(k, j);
      for (long i = 0; i < a.rows; ++i) m(i, j) += a(i, k) * y;
    }
  return m;
}
static Dense d_adjoint(const Dense& a) {
  Dense m(a.cols, a.rows);
  for (long j = 0; j < a.cols; ++j)
    for (long i = 0; i < a.rows; ++i) m(j, i) = std::conj(a(i, j));
  return m;
}
static Dense d_kron(const Dense& a, const Dense& b) {  // qobj.cpp:256-262
  Dense m(a.rows * b.rows, a.cols * b.cols);
  for (long i = 0; i < a.rows; ++i)
    for (long j = 0; j < a.cols; ++j)
      for (long k = 0; k < b.rows; ++k)
        for (long l = 0; l < b.cols; ++l) m(i * b.rows + k, j * b.cols + l) = a(i, j) * b(k, l);
  return m;
}

// ======================================================================================
// QuantumObject (qobj.cpp)
// ======================================================================================

static long dims_product(const Dims& d) {
  long p = 1;
  for (int x : d) p *= x;
  return p;
}
static std::pair<long, long> expected_shape(Kind k, long d) {  // qobj.cpp:50-60
  switch (k) {
    case Kind::Ket: return {d, 1};
    case Kind::Bra: return {1, d};
    case Kind::Operator: return {d, d};
    case Kind::SuperOperator: return {d * d, d * d};
    case Kind::OperatorKet: return {d * d, 1};
    case Kind::OperatorBra: return {1, d * d};
  }
  return {0, 0};
}
static void check_shape(const QObj& q) {  // qobj.cpp:101-108
  auto [r, c] = expected_shape(q.kind, q.dim);
  require(q.rows() == r && q.cols() == c, ErrorCode::DimsMismatch, "payload shape does not match kind");
}

QObj::QObj(Dense m, Kind k, Dims ds)
    : is_sparse(false), d(std::move(m)), kind(k), dims(std::move(ds)), dim(dims_product(dims)) {
  check_shape(*this);
}
QObj::QObj(Csc m, Kind k, Dims ds)
    : is_sparse(true), s(std::move(m)), kind(k), dims(std::move(ds)), dim(dims_product(dims)) {
  check_shape(*this);
}

QObj operator+(const QObj& a, const QObj& b) {  // qobj.cpp:162-168
  require(a.kind == b.kind, ErrorCode::KindMismatch, "cannot add different kinds");
  require(a.dims == b.dims, ErrorCode::DimsMismatch, "operands have different dims");
  if (a.is_sparse && b.is_sparse) return QObj(sp_add(a.s, b.s), a.kind, a.dims);
  return QObj(d_add(a.dense(), b.dense()), a.kind, a.dims);
}
QObj operator-(const QObj& a) { return cd(-1.0, 0.0) * a; }       // qobj.cpp:174
QObj operator-(const QObj& a, const QObj& b) { return a + (-b); }  // qobj.cpp:170-172

static Kind matmul_kind(Kind a, Kind b) {  // qobj.cpp:179-192
  using K = Kind;
  if (a == K::Operator && b == K::Operator) return K::Operator;
  if (a == K::Operator && b == K::Ket) return K::Ket;
  if (a == K::Bra && b == K::Operator) return K::Bra;
  if (a == K::Bra && b == K::Ket) return K::Operator;
  if (a == K::Ket && b == K::Bra) return K::Operator;
  if (a == K::SuperOperator && b == K::SuperOperator) return K::SuperOperator;
  if (a == K::SuperOperator && b == K::OperatorKet) return K::OperatorKet;
  if (a == K::OperatorBra && b == K::SuperOperator) return K::OperatorBra;
  if (a == K::OperatorBra && b == K::OperatorKet) return K::Operator;
  throw_error(ErrorCode::KindMismatch, "cannot multiply these kinds");
}

QObj operator*(const QObj& a, const QObj& b) {  // qobj.cpp:201-217
  Kind k = matmul_kind(a.kind, b.kind);
  require(a.dims == b.dims, ErrorCode::DimsMismatch, "operands have different dims");
  bool scalar = (a.kind == Kind::Bra && b.kind == Kind::Ket) ||
                (a.kind == Kind::OperatorBra && b.kind == Kind::OperatorKet);
  Dims od = scalar ? Dims{1} : a.dims;
  if (a.is_sparse && b.is_sparse) return QObj(sp_mul(a.s, b.s), k, od);
  if (a.is_sparse) return QObj(d_mul(sp_to_dense(a.s), b.d), k, od);
  if (b.is_sparse) return QObj(d_mul(a.d, sp_to_dense(b.s)), k, od);
  return QObj(d_mul(a.d, b.d), k, od);
}
QObj operator*(cd s, const QObj& a) {  // qobj.cpp:219-222
  if (a.is_sparse) return QObj(sp_scale(s, a.s), a.kind, a.dims);
  return QObj(d_scale(s, a.d), a.kind, a.dims);
}
QObj operator*(double s, const QObj& a) { return cd(s, 0.0) * a; }  // qobj.cpp:225
QObj operator/(const QObj& a, double s) { return (1.0 / s) * a; }   // qobj.cpp:228

QObj tensor(const QObj& a, const QObj& b) {  // qobj.cpp:232-263
  require(a.kind == b.kind, ErrorCode::KindMismatch, "tensor requires equal kinds");
  Dims dims = a.dims;
  dims.insert(dims.end(), b.dims.begin(), b.dims.end());
  if (a.is_sparse && b.is_sparse) return QObj(sp_kron(a.s, b.s), a.kind, dims);
  return QObj(d_kron(a.dense(), b.dense()), a.kind, dims);
}

static Kind dag_kind(Kind k) {
  switch (k) {
    case Kind::Ket: return Kind::Bra;
    case Kind::Bra: return Kind::Ket;
    case Kind::OperatorKet: return Kind::OperatorBra;
    case Kind::OperatorBra: return Kind::OperatorKet;
    default: return k;
  }
}
QObj dag(const QObj& x) {  // qobj.cpp:410-414
  if (x.is_sparse) return QObj(sp_adjoint(x.s), dag_kind(x.kind), x.dims);
  return QObj(d_adjoint(x.d), dag_kind(x.kind), x.dims);
}
QObj ket2dm(const QObj& psi) {  // qobj.cpp:513-518
  if (psi.is_operator()) return psi;
  require(psi.is_ket(), ErrorCode::KindMismatch, "ket2dm expects a Ket");
  Dense v = psi.dense();
  return QObj(d_mul(v, d_adjoint(v)), Kind::Operator, psi.dims);
}
double ket_norm(const QObj& psi) {
  Dense v = psi.dense();
  double s = 0.0;
  for (const auto& x : v.v) s += std::norm(x);
  return std::sqrt(s);
}

// ======================================================================================
// factories.cpp
// ======================================================================================
QObj destroy(int n) {  // factories.cpp:23-28
  require(n >= 1, ErrorCode::InvalidDimension, "mode dimension must be >= 1");
  std::vector<Triplet> t;
  for (int k = 1; k < n; ++k) t.push_back({k - 1, k, cd(std::sqrt(static_cast<double>(k)), 0.0)});
  return QObj(from_triplets(n, n, std::move(t)), Kind::Operator, {n});
}
QObj create(int n) { return dag(destroy(n)); }
QObj num(int n) {  // factories.cpp:32-37
  std::vector<Triplet> t;
  for (int k = 1; k < n; ++k) t.push_back({k, k, cd(static_cast<double>(k), 0.0)});
  return QObj(from_triplets(n, n, std::move(t)), Kind::Operator, {n});
}
QObj qeye(int n) { return QObj(sp_identity(n), Kind::Operator, {n}); }
QObj sigmax() {
  return QObj(from_triplets(2, 2, {{0, 1, cd(1.0)}, {1, 0, cd(1.0)}}), Kind::Operator, {2});
}
QObj sigmay() {
  return QObj(from_triplets(2, 2, {{0, 1, cd(0, -1)}, {1, 0, cd(0, 1)}}), Kind::Operator, {2});
}
QObj sigmaz() {
  return QObj(from_triplets(2, 2, {{0, 0, cd(1.0)}, {1, 1, cd(-1.0)}}), Kind::Operator, {2});
}
QObj sigmap() { return QObj(from_triplets(2, 2, {{0, 1, cd(1.0)}}), Kind::Operator, {2}); }
QObj sigmam() { return dag(sigmap()); }
QObj basis(int n, int i) {  // factories.cpp:83-89
  require(i >= 0 && i < n, ErrorCode::InvalidIndex, "basis index out of range");
  Dense v(n, 1);
  v(i, 0) = cd(1.0, 0.0);
  return QObj(std::move(v), Kind::Ket, {n});
}
QObj fock(int n, int i) { return basis(n, i); }
QObj fock_dm(int n, int i) {
  return QObj(from_triplets(n, n, {{i, i, cd(1.0)}}), Kind::Operator, {n});
}
QObj embed_site(const Dims& dims, int site, const QObj& op) {  // factories.cpp:192-202
  require(site >= 0 && site < static_cast<int>(dims.size()), ErrorCode::InvalidSubsystem,
          "embed_site: site out of range");
  QObj out = (site == 0) ? op : qeye(dims[0]);
  for (size_t i = 1; i < dims.size(); ++i)
    out = tensor(out, static_cast<int>(i) == site ? op : qeye(dims[i]));
  return out;
}

std::pair<QObj, std::vector<QObj>> ising_model(int nx, int ny, double jz, double hx,
                                               double gamma, bool periodic, bool cap) {
  // factories.cpp:204-246
  require(nx >= 1 && ny >= 1, ErrorCode::InvalidDimension, "lattice extents must be >= 1");
  const int ns = nx * ny;
  if (cap) require(ns <= 12, ErrorCode::TooLarge, "lattice capped at 12 sites");
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
  Csc empty;
  empty.rows = empty.cols = d;
  empty.outer.assign(static_cast<size_t>(d + 1), 0);
  QObj hq(empty, Kind::Operator, dims);
  bool first = true;
  for (auto [i, j] : bonds) {
    QObj term = jz * (embed_site(dims, i, sigmaz()) * embed_site(dims, j, sigmaz()));
    hq = first ? term : hq + term;
    first = false;
  }
  for (int i = 0; i < ns; ++i) {
    QObj term = hx * embed_site(dims, i, sigmax());
    hq = first ? term : hq + term;
    first = false;
  }
  std::vector<QObj> c_ops;
  const double amp = std::sqrt(gamma);
  for (int i = 0; i < ns; ++i) c_ops.push_back(amp * embed_site(dims, i, sigmam()));
  return {hq, c_ops};
}

// ======================================================================================
// superop.cpp
// ======================================================================================
QObj spre(const QObj& a) {  // superop.cpp:51-55
  require(a.is_operator(), ErrorCode::KindMismatch, "spre expects an Operator");
  return QObj(sp_kron(sp_identity(a.dim), a.sparse()), Kind::SuperOperator, a.dims);
}
QObj spost(const QObj& b) {  // superop.cpp:57-61
  require(b.is_operator(), ErrorCode::KindMismatch, "spost expects an Operator");
  return QObj(sp_kron(sp_transpose(b.sparse()), sp_identity(b.dim)), Kind::SuperOperator, b.dims);
}
QObj sprepost(const QObj& a, const QObj& b) {  // superop.cpp:63-69
  return QObj(sp_kron(sp_transpose(b.sparse()), a.sparse()), Kind::SuperOperator, a.dims);
}
QObj lindblad_dissipator(const QObj& c) {  // superop.cpp:71-76
  QObj cd_ = dag(c);
  QObj cdc = cd_ * c;
  return sprepost(c, cd_) - 0.5 * spre(cdc) - 0.5 * spost(cdc);
}
QObj liouvillian(const QObj& h, std::span<const QObj> c_ops) {  // superop.cpp:78-91
  QObj l;
  if (h.kind == Kind::SuperOperator) l = h;
  else l = cd(0, -1) * (spre(h) - spost(h));
  for (const auto& c : c_ops) {
    require(c.dims == l.dims, ErrorCode::DimsMismatch, "liouvillian: collapse dims mismatch");
    l = l + lindblad_dissipator(c);
  }
  return l;
}

// ======================================================================================
// evolve
// ======================================================================================
TdOp liouvillian_td(const TdOp& h, std::span<const QObj> c_ops) {  // evolve.cpp:39-47
  TdOp out;
  out.constant = liouvillian(h.constant, c_ops);
  for (const auto& t : h.terms) out.terms.push_back({cd(0, -1) * (spre(t.op) - spost(t.op)), t.coeff});
  return out;
}

// CSC -> row-major, columns ascending within each row (stable counting sort by row)
static CsrRows csc_rows(const Csc& a) {
  CsrRows r;
  r.rows = a.rows;
  r.ptr.assign(static_cast<size_t>(a.rows + 1), 0);
  for (int i : a.inner) ++r.ptr[static_cast<size_t>(i) + 1];
  for (long i = 0; i < a.rows; ++i) r.ptr[static_cast<size_t>(i + 1)] += r.ptr[static_cast<size_t>(i)];
  r.col.resize(a.inner.size());
  r.val.resize(a.val.size());
  std::vector<long> pos(r.ptr.begin(), r.ptr.end() - 1);
  for (long j = 0; j < a.cols; ++j)
    for (int p = a.outer[static_cast<size_t>(j)]; p < a.outer[static_cast<size_t>(j + 1)]; ++p) {
      const long q = pos[static_cast<size_t>(a.inner[static_cast<size_t>(p)])]++;
      r.col[static_cast<size_t>(q)] = static_cast<int>(j);
      r.val[static_cast<size_t>(q)] = a.val[static_cast<size_t>(p)];
    }
  return r;
}

// Same per-row arithmetic as sp_gemv: out[i] = 0, then out[i] += v * (1 * y[j]) over the row's
// entries in ascending column order (the order the CSC scatter reaches row i).
static void rows_gemv(const CsrRows& a, const cd* y, cd* out) {
  par_for(static_cast<size_t>(a.rows), [&](size_t lo, size_t hi) {
    for (size_t i = lo; i < hi; ++i) {
      cd acc(0.0, 0.0);
      for (long p = a.ptr[i]; p < a.ptr[i + 1]; ++p) {
        const cd rj = cd(1.0, 0.0) * y[a.col[static_cast<size_t>(p)]];
        acc += a.val[static_cast<size_t>(p)] * rj;
      }
      out[i] = acc;
    }
  });
}

SparseGenerator::SparseGenerator(const TdOp& op, cd pref, const Params& params)
    : params_(params) {  // evolve.cpp:53-61
  const_part_ = (pref * op.constant).sparse();
  for (const auto& t : op.terms) terms_.emplace_back((pref * t.op).sparse(), t.coeff);
  tmp_.resize(static_cast<size_t>(const_part_.rows));
  if (threads() > 1) {
    const_rows_ = csc_rows(const_part_);
    for (const auto& t : terms_) term_rows_.push_back(csc_rows(t.first));
  }
}

void SparseGenerator::apply(double t, const std::vector<cd>& y, std::vector<cd>& out) const {
  // evolve.cpp:63-69
  const bool rows = threads() > 1 && const_rows_.rows == const_part_.rows && const_rows_.rows > 0;
  if (rows) rows_gemv(const_rows_, y.data(), out.data());
  else sp_gemv(const_part_, y.data(), out.data());
  for (size_t k = 0; k < terms_.size(); ++k) {
    const auto& [mat, coeff] = terms_[k];
    if (rows) rows_gemv(term_rows_[k], y.data(), tmp_.data());
    else sp_gemv(mat, y.data(), tmp_.data());
    const cd c = coeff(params_, t);
    par_for(out.size(), [&](size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; ++i) out[i] += c * tmp_[i];
    });
  }
}

namespace {

using Vec = std::vector<cd>;

// element-wise loop body over i in [0, n), split over the worker pool when threads() > 1
#define PAR(...) par_for(n, [&](size_t lo_, size_t hi_) { for (size_t i = lo_; i < hi_; ++i) { __VA_ARGS__; } })

// integrator.hpp:23-195, every vector expression evaluated element-wise in Eigen order.
template <class Rhs>
class Dopri5 {
  static constexpr double c2 = 1.0 / 5.0, c3 = 3.0 / 10.0, c4 = 4.0 / 5.0, c5 = 8.0 / 9.0;
  static constexpr double a21 = 1.0 / 5.0;
  static constexpr double a31 = 3.0 / 40.0, a32 = 9.0 / 40.0;
  static constexpr double a41 = 44.0 / 45.0, a42 = -56.0 / 15.0, a43 = 32.0 / 9.0;
  static constexpr double a51 = 19372.0 / 6561.0, a52 = -25360.0 / 2187.0,
                          a53 = 64448.0 / 6561.0, a54 = -212.0 / 729.0;
  static constexpr double a61 = 9017.0 / 3168.0, a62 = -355.0 / 33.0, a63 = 46732.0 / 5247.0,
                          a64 = 49.0 / 176.0, a65 = -5103.0 / 18656.0;
  static constexpr double a71 = 35.0 / 384.0, a73 = 500.0 / 1113.0, a74 = 125.0 / 192.0,
                          a75 = -2187.0 / 6784.0, a76 = 11.0 / 84.0;
  static constexpr double e1 = 71.0 / 57600.0, e3 = -71.0 / 16695.0, e4 = 71.0 / 1920.0,
                          e5 = -17253.0 / 339200.0, e6 = 22.0 / 525.0, e7 = -1.0 / 40.0;
  static constexpr double d1 = -12715105075.0 / 11282082432.0,
                          d3 = 87487479700.0 / 32700410799.0,
                          d4 = -10690763975.0 / 1880347072.0,
                          d5 = 701980252875.0 / 199316789632.0,
                          d6 = -1453857185.0 / 822651844.0, d7 = 69997945.0 / 29380423.0;
  static constexpr double beta = 0.04, expo1 = 0.2 - beta * 0.75, safe = 0.9;
  static constexpr double facc1 = 5.0, facc2 = 0.1;

 public:
  Dopri5(Rhs rhs, long dim, double atol, double rtol) : rhs_(std::move(rhs)), atol_(atol), rtol_(rtol) {
    require(atol > 0 && rtol > 0, ErrorCode::InvalidGrid, "tolerances must be positive");
    for (Vec* v : {&y_, &y_old_, &k1_, &k2_, &k3_, &k4_, &k5_, &k6_, &k7_, &ysti_, &rc1_, &rc2_,
                   &rc3_, &rc4_, &rc5_})
      v->resize(static_cast<size_t>(dim));
  }

  void start(double t0, const Vec& y0, double t_end, double h_suggest = 0.0) {  // :61-69
    t_ = t_old_ = t0;
    y_ = y0;
    y_old_ = y0;
    rhs_(t_, y_, k1_);
    ++rhs_evals_;
    facold_ = 1e-4;
    h_ = (h_suggest > 0.0) ? h_suggest : initial_step(t_end);
  }

  double t() const { return t_; }
  double t_old() const { return t_old_; }
  double h_current() const { return h_; }
  const Vec& y() const { return y_; }
  long steps = 0, rejected = 0;
  long rhs_evals() const { return rhs_evals_; }

  double step(double t_end) {  // :78-147
    const size_t n = y_.size();
    int attempts = 0;
    for (;;) {
      double h = std::min(h_, t_end - t_);
      const bool clamped = h < h_;
      if (!(h > 0.0)) throw_error(ErrorCode::IntegrationFailure, "step called past t_end");
      if (h <= std::abs(t_) * 1e-15 + 1e-300)
        throw_error(ErrorCode::IntegrationFailure, "step size underflow at t = " + std::to_string(t_));
      if (++attempts > 1000)
        throw_error(ErrorCode::IntegrationFailure,
                    "step repeatedly rejected at t = " + std::to_string(t_));
      PAR(ysti_[i] = y_[i] + h * (a21 * k1_[i]));
      rhs_(t_ + c2 * h, ysti_, k2_);
      PAR(ysti_[i] = y_[i] + h * (a31 * k1_[i] + a32 * k2_[i]));
      rhs_(t_ + c3 * h, ysti_, k3_);
      PAR(ysti_[i] = y_[i] + h * (a41 * k1_[i] + a42 * k2_[i] + a43 * k3_[i]));
      rhs_(t_ + c4 * h, ysti_, k4_);
      PAR(ysti_[i] = y_[i] + h * (a51 * k1_[i] + a52 * k2_[i] + a53 * k3_[i] + a54 * k4_[i]));
      rhs_(t_ + c5 * h, ysti_, k5_);
      PAR(ysti_[i] = y_[i] + h * (a61 * k1_[i] + a62 * k2_[i] + a63 * k3_[i] + a64 * k4_[i] +
                                  a65 * k5_[i]));
      rhs_(t_ + h, ysti_, k6_);
      PAR(ysti_[i] = y_[i] + h * (a71 * k1_[i] + a73 * k3_[i] + a74 * k4_[i] + a75 * k5_[i] +
                                  a76 * k6_[i]));
      rhs_(t_ + h, ysti_, k7_);
      rhs_evals_ += 6;

      double err_sq = 0.0;  // :106-116 (terms element-wise, summed in index order)
      q2_.resize(n);
      PAR({
        const cd e = h * (e1 * k1_[i] + e3 * k3_[i] + e4 * k4_[i] + e5 * k5_[i] + e6 * k6_[i] +
                          e7 * k7_[i]);
        const double sc = atol_ + rtol_ * std::max(std::abs(y_[i]), std::abs(ysti_[i]));
        const double q = std::abs(e) / sc;
        q2_[i] = q * q;
      });
      for (size_t i = 0; i < n; ++i) err_sq += q2_[i];
      double err = std::sqrt(err_sq / static_cast<double>(n));
      if (!std::isfinite(err)) err = 10.0;

      if (err <= 1.0) {  // :119-142
        const double fac11 = std::pow(err, expo1);
        double fac = fac11 / std::pow(facold_, beta);
        fac = std::max(facc2, std::min(facc1, fac / safe));
        const double h_new = h / fac;
        facold_ = std::max(err, 1e-4);
        PAR({
          rc1_[i] = y_[i];
          rc2_[i] = ysti_[i] - y_[i];
          rc3_[i] = h * k1_[i] - rc2_[i];
          rc4_[i] = rc2_[i] - h * k7_[i] - rc3_[i];
          rc5_[i] = h * (d1 * k1_[i] + d3 * k3_[i] + d4 * k4_[i] + d5 * k5_[i] + d6 * k6_[i] +
                         d7 * k7_[i]);
        });
        t_old_ = t_;
        y_old_.swap(y_);  // y_old = y; y = ysti (ysti is rewritten before its next read)
        t_ += h;
        h_last_ = h;
        y_.swap(ysti_);
        k1_.swap(k7_);
        ++steps;
        if (!clamped) h_ = h_new;
        else h_ = std::max(h_, h_new);
        return t_;
      }
      ++rejected;
      h_ = h / std::min(facc1, std::pow(err, expo1) / safe);  // :144-145
    }
  }

  void dense(double t, Vec& out) const {  // :150-154
    const double theta = (t - t_old_) / h_last_;
    const double th1 = 1.0 - theta;
    par_for(out.size(), [&](size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; ++i)
        out[i] = rc1_[i] + theta * (rc2_[i] + th1 * (rc3_[i] + theta * (rc4_[i] + th1 * rc5_[i])));
    });
  }

 private:
  double initial_step(double t_end) {  // :157-187
    const size_t n = y_.size();
    double d0 = 0.0, d1n = 0.0;
    for (size_t i = 0; i < n; ++i) {
      const double sc = atol_ + rtol_ * std::abs(y_[i]);
      d0 += std::norm(y_[i] / sc);
      d1n += std::norm(k1_[i] / sc);
    }  // once per solve: left sequential
    d0 = std::sqrt(d0 / static_cast<double>(n));
    d1n = std::sqrt(d1n / static_cast<double>(n));
    double h0 = (d0 < 1e-5 || d1n < 1e-5) ? 1e-6 : 0.01 * d0 / d1n;
    h0 = std::min(h0, t_end - t_);
    if (!(h0 > 0)) h0 = 1e-6;
    PAR(ysti_[i] = y_[i] + h0 * k1_[i]);
    rhs_(t_ + h0, ysti_, k2_);
    ++rhs_evals_;
    double d2 = 0.0;
    for (size_t i = 0; i < n; ++i) {
      const double sc = atol_ + rtol_ * std::abs(y_[i]);
      d2 += std::norm((k2_[i] - k1_[i]) / sc);
    }
    d2 = std::sqrt(d2 / static_cast<double>(n)) / h0;
    double h1;
    if (std::max(d1n, d2) <= 1e-15) h1 = std::max(1e-6, h0 * 1e-3);
    else h1 = std::pow(0.01 / std::max(d1n, d2), 0.2);
    return std::min({100.0 * h0, h1, t_end - t_});
  }

  Rhs rhs_;
  double atol_, rtol_;
  double t_ = 0.0, t_old_ = 0.0, h_ = 0.0, h_last_ = 0.0, facold_ = 1e-4;
  long rhs_evals_ = 0;
  Vec y_, y_old_, k1_, k2_, k3_, k4_, k5_, k6_, k7_, ysti_;
  Vec rc1_, rc2_, rc3_, rc4_, rc5_;
  std::vector<double> q2_;
};

struct ObsEvent {
  double t;
  long grid_idx;
  bool save;
};

std::vector<ObsEvent> build_events(std::span<const double> tlist,
                                   const std::vector<double>* saveat) {  // evolve.cpp:89-118
  std::vector<ObsEvent> ev;
  for (size_t i = 0; i < tlist.size(); ++i) ev.push_back({tlist[i], static_cast<long>(i), false});
  if (saveat) {
    require(std::is_sorted(saveat->begin(), saveat->end()), ErrorCode::InvalidGrid,
            "saveat must be sorted");
    for (double t : *saveat) {
      require(t >= tlist.front() && t <= tlist.back(), ErrorCode::InvalidGrid,
              "saveat times must lie within [t0, tf]");
      ev.push_back({t, -1, true});
    }
    std::stable_sort(ev.begin(), ev.end(), [](const ObsEvent& a, const ObsEvent& b) { return a.t < b.t; });
    std::vector<ObsEvent> merged;
    for (const auto& e : ev) {
      if (!merged.empty() && merged.back().t == e.t) {
        if (e.grid_idx >= 0) merged.back().grid_idx = e.grid_idx;
        merged.back().save |= e.save;
      } else {
        merged.push_back(e);
      }
    }
    ev.swap(merged);
  }
  return ev;
}

void check_tlist(std::span<const double> tlist) {  // evolve.cpp:71-75
  require(tlist.size() >= 2, ErrorCode::InvalidGrid, "tlist needs at least two points");
  for (size_t i = 1; i < tlist.size(); ++i)
    require(tlist[i] > tlist[i - 1], ErrorCode::InvalidGrid, "tlist must increase strictly");
}

template <class Observe>
void integrate_events(const SparseGenerator& gen, const Vec& y0, std::span<const double> tlist,
                      const std::vector<double>* saveat, const SolveOptions& opt,
                      SolveStats& stats, Observe&& observe) {  // evolve.cpp:122-173
  auto events = build_events(tlist, saveat);
  const double tf = tlist.back();
  const double eps_t = 1e-12 * std::max({1.0, std::abs(tf), std::abs(tlist.front())});
  auto rhs = [&gen](double t, const Vec& y, Vec& dydt) { gen.apply(t, y, dydt); };
  size_t next = 0;
  while (next < events.size() && events[next].t <= tlist.front() + eps_t) {
    observe(events[next], y0);
    ++next;
  }
  Dopri5<decltype(rhs)> integ(rhs, static_cast<long>(y0.size()), opt.abstol, opt.reltol);
  integ.start(tlist.front(), y0, tf);
  Vec ybuf(y0.size());
  while (next < events.size()) {
    if (integ.steps >= opt.max_steps)
      throw_error(ErrorCode::IntegrationFailure,
                  "max step count exceeded at t = " + std::to_string(integ.t()));
    integ.step(tf);
    while (next < events.size() && events[next].t <= integ.t() + eps_t) {
      integ.dense(std::min(events[next].t, integ.t()), ybuf);
      observe(events[next], ybuf);
      ++next;
    }
    if (integ.t() >= tf - eps_t) break;
  }
  for (; next < events.size(); ++next) observe(events[next], integ.y());
  stats.steps += integ.steps;
  stats.rejected += integ.rejected;
  stats.rhs_evals += integ.rhs_evals();
}

std::vector<Csc> to_sparse_ops(std::span<const QObj> ops, const Dims& dims) {
  std::vector<Csc> out;
  for (const auto& op : ops) {
    require(op.dims == dims, ErrorCode::DimsMismatch, "operator dims mismatch");
    out.push_back(op.sparse());
  }
  return out;
}

cd dotc(const Vec& a, const Vec& b) {  // Eigen a.dot(b) = sum conj(a_i) b_i
  cd s(0.0, 0.0);
  for (size_t i = 0; i < a.size(); ++i) s += std::conj(a[i]) * b[i];
  return s;
}
double sqnorm(const Vec& a) {
  double s = 0.0;
  for (const auto& x : a) s += std::norm(x);
  return s;
}

}  // namespace

SolveResult sesolve(const TdOp& h, const QObj& psi0, std::span<const double> tlist,
                    std::span<const QObj> e_ops, const Params& params, const SolveOptions& opt) {
  // evolve.cpp:191-233
  check_tlist(tlist);
  require(psi0.is_ket(), ErrorCode::KindMismatch, "sesolve expects a Ket initial state");
  require(h.constant.kind == Kind::Operator, ErrorCode::KindMismatch, "sesolve expects an Operator");
  require(h.constant.dims == psi0.dims, ErrorCode::DimsMismatch, "H and psi0 dims differ");
  SolveResult res;
  res.times.assign(tlist.begin(), tlist.end());
  res.expect = Dense(static_cast<long>(e_ops.size()), static_cast<long>(tlist.size()));
  if (std::abs(ket_norm(psi0) - 1.0) > 1e-10) res.stats.warnings.push_back("initial state is not normalized");
  SparseGenerator gen(h, cd(0, -1), params);
  auto e_mats = to_sparse_ops(e_ops, psi0.dims);
  const bool keep = opt.store_states || e_ops.empty();
  std::vector<double> def_save;
  const std::vector<double>* saveat = nullptr;
  if (opt.saveat) saveat = &*opt.saveat;
  else if (keep) {
    def_save.assign(tlist.begin(), tlist.end());
    saveat = &def_save;
  }
  Dense p0 = psi0.dense();
  Vec y0(p0.v.begin(), p0.v.end());
  Vec tmp(y0.size());
  integrate_events(gen, y0, tlist, saveat, opt, res.stats, [&](const ObsEvent& ev, const Vec& y) {
    if (ev.grid_idx >= 0)
      for (size_t e = 0; e < e_mats.size(); ++e) {
        sp_gemv(e_mats[e], y.data(), tmp.data());
        res.expect(static_cast<long>(e), ev.grid_idx) = dotc(y, tmp);
      }
    if (ev.save) {
      Dense s(static_cast<long>(y.size()), 1);
      s.v = y;
      res.states.emplace_back(std::move(s), Kind::Ket, psi0.dims);
    }
  });
  return res;
}

SolveResult mesolve(const TdOp& h_or_l, const QObj& rho0_in, std::span<const double> tlist,
                    std::span<const QObj> c_ops, std::span<const QObj> e_ops,
                    const Params& params, const SolveOptions& opt) {
  // evolve.cpp:237-299
  check_tlist(tlist);
  TdOp l_td;
  if (h_or_l.constant.kind == Kind::Operator) {
    l_td = liouvillian_td(h_or_l, c_ops);
  } else {
    require(h_or_l.constant.kind == Kind::SuperOperator, ErrorCode::KindMismatch,
            "mesolve expects an Operator or SuperOperator generator");
    require(c_ops.empty(), ErrorCode::KindMismatch, "c_ops must be empty when a SuperOperator is supplied");
    l_td = h_or_l;
  }
  QObj rho0 = rho0_in.is_ket() ? ket2dm(rho0_in) : rho0_in;
  require(rho0.is_operator(), ErrorCode::KindMismatch, "mesolve expects a Ket or Operator state");
  require(rho0.dims == l_td.constant.dims, ErrorCode::DimsMismatch, "state dims do not match L");
  SolveResult res;
  res.times.assign(tlist.begin(), tlist.end());
  res.expect = Dense(static_cast<long>(e_ops.size()), static_cast<long>(tlist.size()));
  SparseGenerator gen(l_td, cd(1, 0), params);
  auto e_mats = to_sparse_ops(e_ops, rho0.dims);
  const bool keep = opt.store_states || e_ops.empty();
  std::vector<double> def_save;
  const std::vector<double>* saveat = nullptr;
  if (opt.saveat) saveat = &*opt.saveat;
  else if (keep) {
    def_save.assign(tlist.begin(), tlist.end());
    saveat = &def_save;
  }
  const long d = rho0.dim;
  Dense m0 = rho0.dense();
  Vec y0(m0.v.begin(), m0.v.end());  // column stacking == column-major storage (:274-277)
  Dense rho_buf(d, d);
  integrate_events(gen, y0, tlist, saveat, opt, res.stats, [&](const ObsEvent& ev, const Vec& y) {
    par_for(static_cast<size_t>(d), [&](size_t lo, size_t hi) {  // :286 hermitize
      for (long j = static_cast<long>(lo); j < static_cast<long>(hi); ++j)
        for (long i = 0; i < d; ++i)
          rho_buf(i, j) = 0.5 * (y[static_cast<size_t>(j * d + i)] + std::conj(y[static_cast<size_t>(i * d + j)]));
    }, 64);
    if (ev.grid_idx >= 0)
      for (size_t e = 0; e < e_mats.size(); ++e) {  // :288-295
        cd acc = 0.0;
        const Csc& a = e_mats[e];
        for (long k = 0; k < a.cols; ++k)
          for (int p = a.outer[static_cast<size_t>(k)]; p < a.outer[static_cast<size_t>(k + 1)]; ++p)
            acc += a.val[static_cast<size_t>(p)] * rho_buf(k, a.inner[static_cast<size_t>(p)]);
        res.expect(static_cast<long>(e), ev.grid_idx) = acc;
      }
    if (ev.save) res.states.emplace_back(rho_buf, Kind::Operator, rho0.dims);
  });
  return res;
}

// ======================================================================================
// rng.cpp
// ======================================================================================
static inline std::uint64_t rotl(std::uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

std::uint64_t splitmix64_next(std::uint64_t& state) {  // rng.cpp:14-19
  std::uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
RngStream::RngStream(std::uint64_t seed, std::uint64_t stream) {  // rng.cpp:21-25
  std::uint64_t z = seed ^ ((stream + 1) * 0x9E3779B97F4A7C15ULL);
  for (auto& w : s_) w = splitmix64_next(z);
  if ((s_[0] | s_[1] | s_[2] | s_[3]) == 0) s_[0] = 1;
}
std::uint64_t RngStream::next_u64() {  // rng.cpp:27-37
  const std::uint64_t result = rotl(s_[0] + s_[3], 23) + s_[0];
  const std::uint64_t t = s_[1] << 17;
  s_[2] ^= s_[0];
  s_[3] ^= s_[1];
  s_[1] ^= s_[2];
  s_[0] ^= s_[3];
  s_[2] ^= t;
  s_[3] = rotl(s_[3], 45);
  return result;
}
double RngStream::uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
double RngStream::uniform_pos() {
  double u = uniform();
  while (u == 0.0) u = uniform();
  return u;
}
double RngStream::normal() {  // rng.cpp:49-61
  if (has_cached_) {
    has_cached_ = false;
    return cached_;
  }
  const double u1 = uniform_pos();
  const double u2 = uniform();
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double phi = 2.0 * std::numbers::pi * u2;
  cached_ = r * std::sin(phi);
  has_cached_ = true;
  return r * std::cos(phi);
}

// ======================================================================================
// trajectories.cpp
// ======================================================================================
static Dense pairwise_sum(const std::vector<const Dense*>& m, size_t lo, size_t hi) {
  // trajectories.cpp:17-22
  if (hi - lo == 1) return *m[lo];
  const size_t mid = lo + (hi - lo) / 2;
  return d_add(pairwise_sum(m, lo, mid), pairwise_sum(m, mid, hi));
}

EnsembleResult run_ensemble(const std::function<TrajectoryData(int, RngStream&)>& sim, int n_e,
                            std::span<const double> tlist, const EnsembleOptions& ens) {
  // trajectories.cpp:26-92
  require(ens.ntraj >= 1, ErrorCode::InvalidGrid, "ntraj must be >= 1");
  const int ntraj = ens.ntraj;
  int nth = ens.n_threads > 0 ? ens.n_threads : static_cast<int>(std::thread::hardware_concurrency());
  if (nth < 1) nth = 1;
  nth = std::min(nth, ntraj);
  std::vector<TrajectoryData> slots(static_cast<size_t>(ntraj));
  std::atomic<int> next{0};
  auto worker = [&] {
    for (;;) {
      const int i = next.fetch_add(1);
      if (i >= ntraj) return;
      RngStream stream(ens.seed, static_cast<std::uint64_t>(i));
      try {
        slots[static_cast<size_t>(i)] = sim(i, stream);
      } catch (const std::exception& e) {
        slots[static_cast<size_t>(i)].failed = true;
        slots[static_cast<size_t>(i)].failure = e.what();
      }
    }
  };
  if (nth == 1) worker();
  else {
    std::vector<std::thread> pool;
    for (int k = 0; k < nth; ++k) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
  }
  EnsembleResult r;
  r.times.assign(tlist.begin(), tlist.end());
  r.ntraj = ntraj;
  std::vector<const Dense*> ok;
  for (int i = 0; i < ntraj; ++i) {
    auto& s = slots[static_cast<size_t>(i)];
    if (s.failed) {
      ++r.failed_trajectories;
      r.stats.warnings.push_back("trajectory " + std::to_string(i) + " failed: " + s.failure);
      continue;
    }
    ok.push_back(&s.expect);
    r.traj_indices.push_back(i);
    r.stats.steps += s.steps;
    r.stats.rejected += s.rejected;
    r.stats.rhs_evals += s.rhs_evals;
  }
  require(!ok.empty(), ErrorCode::EnsembleFailure, "every trajectory failed");
  // Eigen: matrix / Complex(N,0) divides every entry by the complex scalar (:82-83).
  {
    Dense s = pairwise_sum(ok, 0, ok.size());
    for (auto& v : s.v) v = v / cd(static_cast<double>(ok.size()), 0.0);
    r.mean_expect = std::move(s);
  }
  (void)n_e;
  for (int i : r.traj_indices) {
    auto& s = slots[static_cast<size_t>(i)];
    r.jump_records.push_back(s.jumps);
    if (ens.store_per_traj) r.per_traj_expect.push_back(s.expect);
  }
  r.raw = std::move(slots);
  return r;
}

std::vector<double> ensemble_stddev(const EnsembleResult& r) {  // trajectories.cpp:94-104
  require(!r.per_traj_expect.empty(), ErrorCode::InvalidGrid, "per-trajectory data was not stored");
  const size_t sz = r.mean_expect.v.size();
  const double n = static_cast<double>(r.per_traj_expect.size());
  std::vector<double> acc(sz, 0.0);
  for (const auto& m : r.per_traj_expect)
    for (size_t i = 0; i < sz; ++i) {
      const double dlt = m.v[i].real() - r.mean_expect.v[i].real();
      acc[i] += dlt * dlt;
    }
  if (n > 1)
    for (auto& a : acc) a /= (n - 1);
  for (auto& a : acc) a = std::sqrt(a);
  return acc;
}

namespace {
struct McSetup {
  SparseGenerator gen;
  std::vector<Csc> c_mats, e_mats;
};

TrajectoryData simulate_mc_trajectory(const McSetup& setup, const Vec& y0,
                                      std::span<const double> tlist, const SolveOptions& opt,
                                      RngStream& rng) {  // trajectories.cpp:117-213
  TrajectoryData data;
  const long n_e = static_cast<long>(setup.e_mats.size());
  const long n_t = static_cast<long>(tlist.size());
  data.expect = Dense(n_e, n_t);
  auto rhs = [&gen = setup.gen](double t, const Vec& y, Vec& dydt) { gen.apply(t, y, dydt); };
  Dopri5<decltype(rhs)> integ(rhs, static_cast<long>(y0.size()), opt.abstol, opt.reltol);
  const double tf = tlist.back();
  const double eps_t = 1e-12 * std::max(1.0, std::abs(tf));
  Vec ybuf(y0.size()), gbuf(y0.size()), tmp(y0.size());
  auto observe = [&](long k, const Vec& y) {
    const double inv_norm2 = 1.0 / sqnorm(y);
    for (long e = 0; e < n_e; ++e) {
      sp_gemv(setup.e_mats[static_cast<size_t>(e)], y.data(), tmp.data());
      data.expect(e, k) = dotc(y, tmp) * inv_norm2;
    }
  };
  integ.start(tlist.front(), y0, tf);
  observe(0, y0);
  long grid = 1;
  double r = rng.uniform_pos();
  while (grid < n_t) {
    if (integ.steps >= opt.max_steps)
      throw_error(ErrorCode::IntegrationFailure, "max step count exceeded at t = " + std::to_string(integ.t()));
    integ.step(tf);
    double jump_t = integ.t();
    bool jumped = false;
    if (!setup.c_mats.empty() && sqnorm(integ.y()) < r) {
      double lo = integ.t_old(), hi = integ.t();
      for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        integ.dense(mid, ybuf);
        const double g = sqnorm(ybuf) - r;
        if (std::abs(g) < 1e-10) {
          lo = hi = mid;
          break;
        }
        (g > 0 ? lo : hi) = mid;
      }
      jump_t = 0.5 * (lo + hi);
      jumped = true;
    }
    while (grid < n_t && tlist[static_cast<size_t>(grid)] <= jump_t + eps_t) {
      integ.dense(std::min(tlist[static_cast<size_t>(grid)], integ.t()), gbuf);
      observe(grid, gbuf);
      ++grid;
    }
    if (jumped) {
      integ.dense(jump_t, ybuf);
      double total = 0.0;
      std::vector<double> w(setup.c_mats.size());
      for (size_t k = 0; k < setup.c_mats.size(); ++k) {
        sp_gemv(setup.c_mats[k], ybuf.data(), tmp.data());
        w[k] = sqnorm(tmp);
        total += w[k];
      }
      if (total <= 0.0)
        throw_error(ErrorCode::IntegrationFailure, "vanishing jump weights at the crossing time");
      const double u = rng.uniform() * total;
      size_t ch = 0;
      double acc = 0.0;
      for (; ch < w.size(); ++ch) {
        acc += w[ch];
        if (u < acc) break;
      }
      if (ch == w.size()) ch = w.size() - 1;
      sp_gemv(setup.c_mats[ch], ybuf.data(), tmp.data());
      const double nrm = std::sqrt(sqnorm(tmp));
      for (size_t i = 0; i < ybuf.size(); ++i) ybuf[i] = tmp[i] / nrm;
      data.jumps.push_back({jump_t, static_cast<int>(ch)});
      r = rng.uniform_pos();
      if (jump_t < tf - eps_t) integ.start(jump_t, ybuf, tf, integ.h_current());
      else if (grid < n_t)
        for (; grid < n_t; ++grid) observe(grid, ybuf);
    } else if (integ.t() >= tf - eps_t && grid < n_t) {
      for (; grid < n_t; ++grid) observe(grid, integ.y());
    }
  }
  data.steps = integ.steps;
  data.rejected = integ.rejected;
  data.rhs_evals = integ.rhs_evals();
  return data;
}
}  // namespace

EnsembleResult mcsolve(const TdOp& h, const QObj& psi0, std::span<const double> tlist,
                       std::span<const QObj> c_ops, std::span<const QObj> e_ops,
                       const EnsembleOptions& ens, const Params& params, const SolveOptions& opt) {
  // trajectories.cpp:217-249
  check_tlist(tlist);
  require(psi0.is_ket(), ErrorCode::KindMismatch, "mcsolve expects a Ket initial state");
  require(h.constant.kind == Kind::Operator, ErrorCode::KindMismatch, "mcsolve expects an Operator H");
  require(h.constant.dims == psi0.dims, ErrorCode::DimsMismatch, "H and psi0 dims differ");
  QObj heff = h.constant;
  for (const auto& c : c_ops) {
    require(c.dims == psi0.dims, ErrorCode::DimsMismatch, "collapse operator dims mismatch");
    heff = heff + cd(0, -0.5) * (dag(c) * c);
  }
  TdOp heff_td{heff, h.terms};
  McSetup setup{SparseGenerator(heff_td, cd(0, -1), params), {}, {}};
  for (const auto& c : c_ops) setup.c_mats.push_back(c.sparse());
  for (const auto& e : e_ops) {
    require(e.dims == psi0.dims, ErrorCode::DimsMismatch, "e_op dims mismatch");
    setup.e_mats.push_back(e.sparse());
  }
  Dense p0 = psi0.dense();
  Vec y0(p0.v.begin(), p0.v.end());
  auto sim = [&](int, RngStream& rng) { return simulate_mc_trajectory(setup, y0, tlist, opt, rng); };
  return run_ensemble(sim, static_cast<int>(e_ops.size()), tlist, ens);
}

// ======================================================================================
// stochastic solvers (trajectories.cpp:251-503), every Eigen expression element-wise in order
// ======================================================================================
EmGrid make_em_grid(std::span<const double> tlist, double dt_max) {  // trajectories.cpp:261-275
  const double span = tlist.back() - tlist.front();
  const double spacing = tlist[1] - tlist[0];
  for (size_t i = 2; i < tlist.size(); ++i)
    require(std::abs((tlist[i] - tlist[i - 1]) - spacing) <= 1e-9 * spacing, ErrorCode::InvalidGrid,
            "stochastic solvers need a uniform tlist");
  if (dt_max <= 0.0) dt_max = span / 1e4;
  EmGrid g;
  g.substeps_per_interval = std::max(1L, static_cast<long>(std::ceil(spacing / dt_max * (1.0 - 1e-12))));
  g.dt = spacing / static_cast<double>(g.substeps_per_interval);
  g.n_steps = g.substeps_per_interval * static_cast<long>(tlist.size() - 1);
  return g;
}

namespace {
double vnorm(const Vec& a) { return std::sqrt(sqnorm(a)); }

struct SseSetup {
  SparseGenerator gen;  // -i H(t)
  std::vector<Csc> s_mats, sds_mats, x_mats, e_mats;
};

void init_wiener(TrajectoryData& d, const EmGrid& g, size_t n_ch) {
  d.has_wiener = true;
  d.wiener.dt = g.dt;
  d.wiener.n_ch = static_cast<long>(n_ch);
  d.wiener.n_steps = g.n_steps;
  const size_t sz = n_ch * static_cast<size_t>(g.n_steps);
  d.wiener.increments.assign(sz, 0.0);
  d.wiener.expectation.assign(sz, 0.0);
  d.wiener.current.assign(sz, 0.0);
}

TrajectoryData simulate_sse_trajectory(const SseSetup& setup, const Vec& y0, std::span<const double> tlist,
                                       const EmGrid& grid, bool store, RngStream& rng) {  // :283-363
  TrajectoryData data;
  const long n_e = static_cast<long>(setup.e_mats.size()), n_t = static_cast<long>(tlist.size());
  const size_t n_ch = setup.s_mats.size(), n = y0.size();
  data.expect = Dense(n_e, n_t);
  if (store) init_wiener(data, grid, n_ch);
  Vec psi = y0, drift(n), tmp(n), stoch(n);
  std::vector<double> e_vals(n_ch), dw(n_ch);
  auto observe = [&](long k) {
    for (long e = 0; e < n_e; ++e) {
      sp_gemv(setup.e_mats[static_cast<size_t>(e)], psi.data(), tmp.data());
      data.expect(e, k) = dotc(psi, tmp);
    }
  };
  observe(0);
  const bool single = n_ch == 1;
  long step = 0;
  for (long k = 1; k < n_t; ++k) {
    for (long s = 0; s < grid.substeps_per_interval; ++s, ++step) {
      const double t = tlist.front() + grid.dt * static_cast<double>(step);
      setup.gen.apply(t, psi, drift);
      if (single) {  // :313-326
        sp_gemv(setup.x_mats[0], psi.data(), tmp.data());
        const double e_n = dotc(psi, tmp).real();
        const double dw0 = std::sqrt(grid.dt) * rng.normal();
        sp_gemv(setup.s_mats[0], psi.data(), stoch.data());
        sp_gemv(setup.sds_mats[0], psi.data(), tmp.data());
        const double c1 = grid.dt * 0.5 * e_n + dw0, c2 = grid.dt * 0.5;
        const double c3 = grid.dt * 0.125 * e_n * e_n + 0.5 * e_n * dw0;
        for (size_t i = 0; i < n; ++i)
          psi[i] = psi[i] + (((grid.dt * drift[i] + c1 * stoch[i]) - c2 * tmp[i]) - c3 * psi[i]);
        const double nrm = vnorm(psi);
        for (auto& v : psi) v = v / nrm;
        e_vals[0] = e_n;
        dw[0] = dw0;
      } else {  // :327-347
        for (auto& v : stoch) v = cd(0.0, 0.0);
        for (size_t c = 0; c < n_ch; ++c) {
          sp_gemv(setup.x_mats[c], psi.data(), tmp.data());
          const double e_n = dotc(psi, tmp).real();
          e_vals[c] = e_n;
          dw[c] = std::sqrt(grid.dt) * rng.normal();
          sp_gemv(setup.s_mats[c], psi.data(), tmp.data());
          const double a = 0.5 * e_n, b = 0.5 * e_n * dw[c];
          for (size_t i = 0; i < n; ++i) drift[i] += a * tmp[i];
          for (size_t i = 0; i < n; ++i) stoch[i] += dw[c] * tmp[i];
          for (size_t i = 0; i < n; ++i) stoch[i] -= b * psi[i];
          sp_gemv(setup.sds_mats[c], psi.data(), tmp.data());
          const double q = 0.125 * e_n * e_n;
          for (size_t i = 0; i < n; ++i) drift[i] -= 0.5 * tmp[i];
          for (size_t i = 0; i < n; ++i) drift[i] -= q * psi[i];
        }
        for (size_t i = 0; i < n; ++i) psi[i] += grid.dt * drift[i] + stoch[i];
        const double nrm = vnorm(psi);
        for (auto& v : psi) v = v / nrm;
      }
      if (store)
        for (size_t c = 0; c < n_ch; ++c) {  // :348-353
          const size_t idx = c + n_ch * static_cast<size_t>(step);
          data.wiener.increments[idx] = dw[c];
          data.wiener.expectation[idx] = e_vals[c];
          data.wiener.current[idx] = e_vals[c] + dw[c] / grid.dt;
        }
    }
    observe(k);
  }
  data.steps = grid.n_steps;
  data.rhs_evals = grid.n_steps;
  return data;
}

struct SmeSetup {
  SparseGenerator gen;  // full Liouvillian including the sc_op dissipators
  std::vector<Csc> s_mats, e_mats;
  long d = 0;
};

TrajectoryData simulate_sme_trajectory(const SmeSetup& setup, const Vec& rho0, std::span<const double> tlist,
                                       const EmGrid& grid, bool store, RngStream& rng) {  // :408-470
  TrajectoryData data;
  const long n_e = static_cast<long>(setup.e_mats.size()), n_t = static_cast<long>(tlist.size());
  const size_t n_ch = setup.s_mats.size();
  const long d = setup.d;
  const size_t nn = static_cast<size_t>(d * d);
  data.expect = Dense(n_e, n_t);
  if (store) init_wiener(data, grid, n_ch);
  Vec rho = rho0, srho(nn), hop(nn), rho_new(nn), drift(nn);
  auto at = [&](const Vec& m, long i, long j) -> const cd& { return m[static_cast<size_t>(i + d * j)]; };
  auto observe = [&](long k) {
    for (long e = 0; e < n_e; ++e) {
      cd acc = 0.0;
      const Csc& a = setup.e_mats[static_cast<size_t>(e)];
      for (long c = 0; c < a.cols; ++c)
        for (int p = a.outer[static_cast<size_t>(c)]; p < a.outer[static_cast<size_t>(c + 1)]; ++p)
          acc += a.val[static_cast<size_t>(p)] * at(rho, c, a.inner[static_cast<size_t>(p)]);
      data.expect(e, k) = acc;
    }
  };
  observe(0);
  long step = 0;
  for (long k = 1; k < n_t; ++k) {
    for (long s = 0; s < grid.substeps_per_interval; ++s, ++step) {
      const double t = tlist.front() + grid.dt * static_cast<double>(step);
      setup.gen.apply(t, rho, drift);
      for (size_t i = 0; i < nn; ++i) rho_new[i] = rho[i] + grid.dt * drift[i];
      for (size_t c = 0; c < n_ch; ++c) {
        for (long j = 0; j < d; ++j)  // S * rho, column by column (sparse x dense product)
          sp_gemv(setup.s_mats[c], rho.data() + d * j, srho.data() + d * j);
        for (long j = 0; j < d; ++j)
          for (long i = 0; i < d; ++i) hop[static_cast<size_t>(i + d * j)] = at(srho, i, j) + std::conj(at(srho, j, i));
        cd tr = 0.0;
        for (long i = 0; i < d; ++i) tr += at(hop, i, i);
        const double e_n = tr.real();
        const double dw = std::sqrt(grid.dt) * rng.normal();
        for (size_t i = 0; i < nn; ++i) hop[i] -= e_n * rho[i];
        for (size_t i = 0; i < nn; ++i) rho_new[i] += dw * hop[i];
        if (store) {
          const size_t idx = c + n_ch * static_cast<size_t>(step);
          data.wiener.increments[idx] = dw;
          data.wiener.expectation[idx] = e_n;
          data.wiener.current[idx] = e_n + dw / grid.dt;
        }
      }
      for (long j = 0; j < d; ++j)
        for (long i = 0; i < d; ++i)
          rho[static_cast<size_t>(i + d * j)] = 0.5 * (at(rho_new, i, j) + std::conj(at(rho_new, j, i)));
      cd tr = 0.0;
      for (long i = 0; i < d; ++i) tr += at(rho, i, i);
      const double trr = tr.real();
      for (auto& v : rho) v = v / trr;
    }
    observe(k);
  }
  data.steps = grid.n_steps;
  data.rhs_evals = grid.n_steps;
  return data;
}
}  // namespace

EnsembleResult ssesolve(const TdOp& h, const QObj& psi0, std::span<const double> tlist,
                        std::span<const QObj> sc_ops, std::span<const QObj> e_ops, const EnsembleOptions& ens,
                        const Params& params) {  // trajectories.cpp:367-393
  check_tlist(tlist);
  require(psi0.is_ket(), ErrorCode::KindMismatch, "ssesolve expects a Ket initial state");
  require(h.constant.kind == Kind::Operator, ErrorCode::KindMismatch, "ssesolve expects an Operator H");
  require(h.constant.dims == psi0.dims, ErrorCode::DimsMismatch, "H and psi0 dims differ");
  SseSetup setup{SparseGenerator(h, cd(0, -1), params), {}, {}, {}, {}};
  for (const auto& s : sc_ops) {
    require(s.dims == psi0.dims, ErrorCode::DimsMismatch, "sc_op dims mismatch");
    setup.s_mats.push_back(s.sparse());
    setup.sds_mats.push_back((dag(s) * s).sparse());
    setup.x_mats.push_back((s + dag(s)).sparse());
  }
  for (const auto& e : e_ops) setup.e_mats.push_back(e.sparse());
  const EmGrid grid = make_em_grid(tlist, ens.dt_max);
  Dense p0 = psi0.dense();
  Vec y0(p0.v.begin(), p0.v.end());
  const double nrm = vnorm(y0);
  for (auto& v : y0) v = v / nrm;
  auto sim = [&](int, RngStream& rng) {
    return simulate_sse_trajectory(setup, y0, tlist, grid, ens.store_measurement, rng);
  };
  return run_ensemble(sim, static_cast<int>(e_ops.size()), tlist, ens);
}

EnsembleResult smesolve(const TdOp& h, const QObj& rho0_in, std::span<const double> tlist,
                        std::span<const QObj> c_ops, std::span<const QObj> sc_ops, std::span<const QObj> e_ops,
                        const EnsembleOptions& ens, const Params& params) {  // trajectories.cpp:474-503
  check_tlist(tlist);
  require(h.constant.kind == Kind::Operator, ErrorCode::KindMismatch, "smesolve expects an Operator H");
  QObj rho0 = rho0_in.is_ket() ? ket2dm(rho0_in) : rho0_in;
  require(rho0.kind == Kind::Operator, ErrorCode::KindMismatch, "smesolve expects a Ket or Operator state");
  require(rho0.dims == h.constant.dims, ErrorCode::DimsMismatch, "H and rho0 dims differ");
  std::vector<QObj> all_ops(c_ops.begin(), c_ops.end());
  all_ops.insert(all_ops.end(), sc_ops.begin(), sc_ops.end());
  TdOp l_td = liouvillian_td(h, all_ops);
  SmeSetup setup{SparseGenerator(l_td, cd(1, 0), params), {}, {}, rho0.dim};
  for (const auto& s : sc_ops) setup.s_mats.push_back(s.sparse());
  for (const auto& e : e_ops) setup.e_mats.push_back(e.sparse());
  const EmGrid grid = make_em_grid(tlist, ens.dt_max);
  Dense m0 = rho0.dense();
  Vec r0(m0.v.begin(), m0.v.end());
  auto sim = [&](int, RngStream& rng) {
    return simulate_sme_trajectory(setup, r0, tlist, grid, ens.store_measurement, rng);
  };
  return run_ensemble(sim, static_cast<int>(e_ops.size()), tlist, ens);
}

// ======================================================================================
// model zoo: assembled in reference style (scenario.cpp:247-395, test fixtures)
// ======================================================================================
static CoeffFn param_coeff(size_t i) {
  return [i](const Params& p, double) { return cd(p[i], 0.0); };
}
static CoeffFn param_cos_coeff(size_t i, size_t j) {  // scenario.cpp:289-291
  return [i, j](const Params& p, double t) { return cd(p[i] * std::cos(p[j] * t)); };
}

Model build_model(const std::string& name, std::span<const double> p) {
  auto P = [&](size_t i) {
    require(i < p.size(), ErrorCode::InvalidScenario, "model " + name + ": missing parameter");
    return p[i];
  };
  Model m;
  m.name = name;
  if (name == "kerr") {  // N, Delta, U, F, gamma
    const int n = static_cast<int>(P(0));
    const double delta = P(1), u = P(2), f = P(3), gamma = P(4);
    QObj a = destroy(n);
    m.h.constant = delta * (dag(a) * a) + u * (dag(a) * dag(a) * a * a) + f * (a + dag(a));
    m.c_ops = {std::sqrt(gamma) * a};
    m.psi0 = fock(n, 0);
    m.e_ops = {dag(a) * a, a};
  } else if (name == "coupled_kerr") {  // N, U, J, gamma ; params (Delta, F)
    const int n = static_cast<int>(P(0));
    const double u = P(1), j = P(2), gamma = P(3);
    QObj a1 = tensor(destroy(n), qeye(n));
    QObj a2 = tensor(qeye(n), destroy(n));
    QObj h0 = u * (dag(a1) * dag(a1) * a1 * a1) + u * (dag(a2) * dag(a2) * a2 * a2) +
              j * (dag(a1) * a2 + dag(a2) * a1);
    QObj h_delta = dag(a1) * a1 + dag(a2) * a2;
    QObj h_drive = (a1 + dag(a1)) + (a2 + dag(a2));
    m.h.constant = h0;
    m.h.terms = {{h_delta, param_coeff(0)}, {h_drive, param_coeff(1)}};
    m.c_ops = {std::sqrt(gamma) * a1, std::sqrt(gamma) * a2};
    m.psi0 = tensor(fock(n, 0), fock(n, 0));
    m.e_ops = {dag(a1) * a1, dag(a2) * a2};
    m.params = {0.0, 0.0};
  } else if (name == "ising") {  // nx, ny, Jz, hx, gamma, periodic
    const int nx = static_cast<int>(P(0)), ny = static_cast<int>(P(1));
    auto [h, c_ops] = ising_model(nx, ny, P(2), P(3), P(4), P(5) != 0.0, /*cap=*/false);
    Dims dims(static_cast<size_t>(nx * ny), 2);
    m.h.constant = h;
    m.c_ops = c_ops;
    QObj up = basis(2, 0);  // scenario.cpp:379-382
    QObj psi = up;
    for (int i = 1; i < nx * ny; ++i) psi = tensor(psi, up);
    m.psi0 = psi;
    auto total = [&](const QObj& op) {  // scenario.cpp:383-392
      QObj sum = embed_site(dims, 0, op);
      for (int i = 1; i < nx * ny; ++i) sum = sum + embed_site(dims, i, op);
      return sum;
    };
    m.e_ops = {total(sigmax()), total(sigmay()), total(sigmaz())};
  } else if (name == "jc") {  // N, wc, wa, g, kappa, gamma (test_evolve.cpp:16-28)
    const int n = static_cast<int>(P(0));
    const double wc = P(1), wa = P(2), g = P(3), kappa = P(4), gamma = P(5);
    QObj a = tensor(destroy(n), qeye(2));
    QObj sz = tensor(qeye(n), sigmaz());
    QObj sm = tensor(qeye(n), sigmam());
    QObj sp = tensor(qeye(n), sigmap());
    m.h.constant = wc * (dag(a) * a) + (wa / 2.0) * sz + g * (a * sp + dag(a) * sm);
    m.psi0 = tensor(fock(n, 0), basis(2, 0));
    if (kappa > 0.0 || gamma > 0.0) m.c_ops = {std::sqrt(kappa) * a, std::sqrt(gamma) * sm};
    m.e_ops = {dag(a) * a, sz};
  } else if (name == "jc_sse" || name == "jc_sme") {
    // scenario.cpp:252-277, stochastic solvers: jc_sse (N, wc, wa, g, kappa): c_ops = sc_ops =
    // {sqrt(kappa) a}; jc_sme (N, wc, wa, g, kappa, gamma, kphi): c_ops = {sqrt(gamma) sm,
    // sqrt(kphi) a^dag a} (deterministic) followed by the measured sqrt(kappa) a.
    // e_ops: n_cavity, sz_atom, X_quadrature = sqrt(kappa) (a + a^dag).
    const int n = static_cast<int>(P(0));
    const double wc = P(1), wa = P(2), g = P(3), kappa = P(4);
    QObj a = tensor(destroy(n), qeye(2));
    QObj sz = tensor(qeye(n), sigmaz());
    QObj sm = tensor(qeye(n), sigmam());
    QObj sp = tensor(qeye(n), sigmap());
    m.h.constant = wc * (dag(a) * a) + (wa / 2.0) * sz + g * (a * sp + dag(a) * sm);
    m.psi0 = tensor(fock(n, 0), basis(2, 0));
    if (name == "jc_sse") {
      m.c_ops = {std::sqrt(kappa) * a};
    } else {
      m.c_ops = {std::sqrt(P(5)) * sm, std::sqrt(P(6)) * (dag(a) * a), std::sqrt(kappa) * a};
    }
    m.e_ops = {dag(a) * a, sz, std::sqrt(kappa) * (a + dag(a))};
  } else if (name == "damped_cavity") {  // N, omega, gamma, n0 (test_evolve.cpp:124-140)
    const int n = static_cast<int>(P(0));
    QObj a = destroy(n);
    m.h.constant = P(1) * (dag(a) * a);
    m.c_ops = {std::sqrt(P(2)) * a};
    m.psi0 = fock_dm(n, static_cast<int>(P(3)));
    m.e_ops = {dag(a) * a};
  } else if (name == "decay2") {  // gamma (test_trajectories.cpp:40-88)
    Dense z(2, 2);
    m.h.constant = QObj(z, Kind::Operator, {2});
    m.c_ops = {std::sqrt(P(0)) * sigmam()};
    m.psi0 = basis(2, 0);
    m.e_ops = {sigmaz()};
  } else if (name == "driven_cavity_td") {  // N, gamma ; params (F, wd) (test_evolve.cpp:203-237)
    const int n = static_cast<int>(P(0));
    QObj a = destroy(n);
    m.h.constant = 0.0 * num(n);
    m.h.terms = {{a + dag(a), param_cos_coeff(0, 1)}};
    m.c_ops = {std::sqrt(P(1)) * a};
    m.psi0 = fock_dm(n, 0);
    m.e_ops = {a};
    m.params = {0.25, 1.3};
  } else {
    throw_error(ErrorCode::InvalidScenario, "unknown model " + name);
  }
  return m;
}

}  // namespace orc
