// Factories and superoperators — same names and semantics as the reference's
// core/include/qsim/factories.hpp:11-56 and superop.hpp:12-28.
#pragma once

#include <cstdint>
#include <span>
#include <utility>
#include <vector>

#include "qobj.hpp"

namespace qsim {

QuantumObject destroy(int n);
QuantumObject create(int n);
QuantumObject num(int n);
QuantumObject qeye(int n);
QuantumObject qeye(const Dims& dims);
QuantumObject position(int n);
QuantumObject momentum(int n);

QuantumObject sigmax();
QuantumObject sigmay();
QuantumObject sigmaz();
QuantumObject sigmap();
QuantumObject sigmam();

QuantumObject basis(int n, int i);
QuantumObject fock(int n, int i);
QuantumObject fock_dm(int n, int i);
QuantumObject projection(int n, int i, int j);
QuantumObject thermal_dm(int n, double nbar);
QuantumObject maximally_mixed_dm(int n);
QuantumObject coherent(int n, Complex alpha);
QuantumObject coherent_dm(int n, Complex alpha);

QuantumObject embed_site(const Dims& dims, int site, const QuantumObject& op);

/// Dissipative transverse-field Ising model (factories.cpp:204-246), including the reference's
/// 12-site cap (TooLarge above it).
std::pair<QuantumObject, std::vector<QuantumObject>> ising_model(int nx, int ny, double jz,
                                                                 double hx, double gamma,
                                                                 bool periodic);
/// Same conventions without the cap (needed for the 14-spin mcsolve configuration).
std::pair<QuantumObject, std::vector<QuantumObject>> ising_model_uncapped(int nx, int ny, double jz,
                                                                          double hx, double gamma,
                                                                          bool periodic);

// ---- superop.hpp: column-stacking vectorization, vec(A X B) = (B^T kron A) vec(X) ----------
QuantumObject mat2vec(const QuantumObject& rho);
QuantumObject vec2mat(const QuantumObject& v);
QuantumObject spre(const QuantumObject& a);
QuantumObject spost(const QuantumObject& b);
QuantumObject sprepost(const QuantumObject& a, const QuantumObject& b);
QuantumObject lindblad_dissipator(const QuantumObject& c);
QuantumObject liouvillian(const QuantumObject& h, std::span<const QuantumObject> c_ops = {});

}  // namespace qsim
