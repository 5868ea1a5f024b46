// Verifier API (verification.hpp:30-53) and the deterministic RNG (rng.hpp:8-35) on the device.
#pragma once
#include <cstdint>
#include <functional>
#include <vector>

#include "common.cuh"

namespace dbl {

struct DevRng {  // std::mt19937_64 state
    uint64_t mt[312];
    int idx;
};

enum VerifyKindCode : int { kAllAccepted = 0, kCorrection = 1, kExtension = 2, kResidualCorrection = 3 };  // VerifyKind
enum VerifyErr : int {
    kErrArgument = 1, kErrDegenerate = 2, kErrResidualZero = 3, kErrDraftMassZero = 4, kErrUncovered = 5
};

// specpar::Rng with its mt19937_64 stream resident in device memory
class DeviceRng {
  public:
    DeviceRng(uint64_t seed, int device);
    static DeviceRng derive(uint64_t seed, uint64_t round, uint64_t lane, int device);  // derive_rng
    void uniform(double* out, int n);  // n draws of Rng::uniform
    DevRng* state() { return state_.p; }
    int device() const { return device_; }

  private:
    DevBuf<DevRng> state_;
    int device_;
};

struct VerifyOutcome {  // verification.hpp:22-26
    int accepted_len = 0;
    std::vector<int32_t> committed;
    int kind = kAllAccepted;
};

double accept_prob(const double* p, int np, const double* q, int nq, int x, int device);
int residual_sample(const double* p, int np, const double* q, int nq, DeviceRng& rng);
int residual_sample_point_mass(const double* p, int np, int x, DeviceRng& rng);
// rows are ragged: row r = probs[off[r], off[r+1]); returns the first rejected index or -1
int verify_against_target(const int32_t* draft, int n_draft, const double* dprobs, const int64_t* doff, int n_dp,
                          const double* tprobs, const int64_t* toff, int n_tp, double temperature, DeviceRng& rng);
VerifyOutcome guided_output(const int32_t* draft, int n_draft, const double* dprobs, const int64_t* doff, int n_dp,
                            const int32_t* gtok, int n_gtok, const double* gprobs, const int64_t* goff, int n_gp,
                            int first_reject, double temperature, DeviceRng& rng);

// the model-level helpers (model.hpp:40-48) over explicit fp64 rows
void tempered(const double* p, int n, double temperature, double* out, int device);   // model.cpp:55-68
void argmax_rows(const double* probs, const int64_t* off, int n_rows, int32_t* out, int device);  // model.cpp:70-81
int sample(const double* p, int n, double temperature, DeviceRng* rng, int device);    // model.cpp:83-97

struct AcceptOut {  // RetrievalResult (speculation.hpp:12-17) minus the source
    std::vector<int32_t> emitted;
    int matched_len = 0;
    int n_probs = 0;             // rows of probs (ragged like the input rows 0..n_probs)
    std::vector<double> probs;   // flattened; filled when asked
};
// accept_with_model (speculation.cpp:7-52) over ragged rows (|cands| + 1 of them)
AcceptOut accept_with_model(const double* dists, const int64_t* off, int n_rows, const int32_t* cands, int c,
                            double temperature, DeviceRng* rng, int device, bool want_probs);
// the same over uniform rows already on the current device (n_rows x vocab fp64)
AcceptOut accept_with_model_dev(const double* dists_dev, int vocab, int n_rows, const int32_t* cands, int c,
                                double temperature, DeviceRng* rng, bool want_probs);

}  // namespace dbl
