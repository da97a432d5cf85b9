// Reference-side device runtime of the drop-in: the pImpls and free functions of the reference's
// hot-path modules (transport, inverse, spectral, interp; include/veloreg/*.hpp) re-implemented
// over libvrg's C ABI (include/vrg.h).  This is the binding INTEGRATION.md describes, compiled
// with the unmodified reference headers and linked with the unmodified reference field /
// counters / fft / problems / precond / newton / io / diag objects (dropin/Makefile).
//
//  * one libvrg context (device, stream) per host thread, created on first use and kept for the
//    life of the process; an object remembers the context it was made on and every call on it
//    holds that context's mutex, so objects may be shared across threads (the reference's
//    "distinct solves may run concurrently", proj/README.md:157-158);
//  * libvrg status codes are rethrown with the reference's exception types and messages
//    (transport::BlowupError, std::invalid_argument, std::runtime_error);
//  * libvrg keeps per-context logical operation counts with the reference's semantics; every
//    call forwards its deltas to the process counters (counters::addFft / addInterp).
#pragma once

#include <cstddef>
#include <mutex>
#include <vector>

#include "veloreg/field.hpp"
#include "vrg.h"

namespace veloreg::vrgdev {

struct Device {
    vrg_ctx_t ctx = nullptr;
    std::mutex mu;
};

// The calling thread's device context (device index from $VRG_DEVICE, default 0).
Device& threadDevice();

// Holds a context for one library call sequence: locks it, and on release forwards the
// operation counters the calls accumulated.
class Session {
public:
    explicit Session(Device& d);
    ~Session();
    Session(const Session&) = delete;
    Session& operator=(const Session&) = delete;
    vrg_ctx_t ctx() const { return d_.ctx; }
    // Rethrows a non-OK status with the reference's exception type and the library's message.
    void check(int status) const;

private:
    Device& d_;
    std::lock_guard<std::mutex> lock_;
};

// Device buffer of doubles on a context (RAII; freed on the same context).
class DevBuf {
public:
    DevBuf() = default;
    DevBuf(const Session& s, std::size_t count);
    ~DevBuf();
    DevBuf(DevBuf&& o) noexcept;
    DevBuf& operator=(DevBuf&& o) noexcept;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    double* get() const { return p_; }
    double* at(std::size_t offset) const { return p_ + offset; }
    std::size_t count() const { return n_; }
    explicit operator bool() const { return p_ != nullptr; }

private:
    vrg_ctx_t ctx_ = nullptr;
    double* p_ = nullptr;
    std::size_t n_ = 0;
};

void upload(const Session& s, double* dst, const std::vector<double>& src);
void download(const Session& s, std::vector<double>& dst, const double* src);

// Device copies of host fields: a scalar field, a vector field as [c0 | c1], a list of frames.
DevBuf deviceField(const Session& s, const ScalarField& f);
DevBuf deviceVector(const Session& s, const VectorField& v);
DevBuf deviceFrames(const Session& s, const std::vector<ScalarField>& frames);
// Host fields from device memory on grid g.
ScalarField hostField(const Session& s, const Grid& g, const double* src);
VectorField hostVector(const Session& s, const Grid& g, const double* src);
std::vector<ScalarField> hostFrames(const Session& s, const Grid& g, const double* src, int count);

}  // namespace veloreg::vrgdev
