// Device runtime of the drop-in (see vrg_device.hpp).
#include "vrg_device.hpp"

#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>

#include "veloreg/counters.hpp"
#include "veloreg/transport.hpp"

namespace veloreg::vrgdev {

namespace {

std::mutex g_registryMu;
std::vector<std::unique_ptr<Device>>& registry() {
    static std::vector<std::unique_ptr<Device>> r;  // contexts live for the whole process
    return r;
}

}  // namespace

Device& threadDevice() {
    thread_local Device* mine = nullptr;
    if (!mine) {
        auto d = std::make_unique<Device>();
        const char* e = std::getenv("VRG_DEVICE");
        const int dev = e ? std::atoi(e) : 0;
        if (vrg_ctx_create(dev, nullptr, &d->ctx) != VRG_OK)
            throw std::runtime_error(std::string("vrg: cannot create a device context: ") + vrg_last_error(nullptr));
        std::lock_guard<std::mutex> lock(g_registryMu);
        registry().push_back(std::move(d));
        mine = registry().back().get();
    }
    return *mine;
}

Session::Session(Device& d) : d_(d), lock_(d.mu) {}

Session::~Session() {
    long long f = 0, i = 0;
    vrg_counters(d_.ctx, &f, &i);
    if (f) counters::addFft(f);
    if (i) counters::addInterp(i);
    vrg_counters_reset(d_.ctx);
}

void Session::check(int status) const {
    if (status == VRG_OK) return;
    const std::string msg = vrg_last_error(d_.ctx);
    if (status == VRG_BLOWUP) throw transport::BlowupError(msg);
    if (status == VRG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

DevBuf::DevBuf(const Session& s, std::size_t count) : ctx_(s.ctx()), n_(count) {
    void* p = nullptr;
    s.check(vrg_malloc(ctx_, sizeof(double) * (count ? count : 1), &p));
    p_ = static_cast<double*>(p);
}

DevBuf::~DevBuf() {
    if (p_) vrg_free(ctx_, p_);
}

DevBuf::DevBuf(DevBuf&& o) noexcept : ctx_(o.ctx_), p_(o.p_), n_(o.n_) {
    o.p_ = nullptr;
    o.n_ = 0;
}

DevBuf& DevBuf::operator=(DevBuf&& o) noexcept {
    if (this != &o) {
        if (p_) vrg_free(ctx_, p_);
        ctx_ = o.ctx_;
        p_ = o.p_;
        n_ = o.n_;
        o.p_ = nullptr;
        o.n_ = 0;
    }
    return *this;
}

void upload(const Session& s, double* dst, const std::vector<double>& src) {
    if (!src.empty()) s.check(vrg_copy_h2d(s.ctx(), dst, src.data(), sizeof(double) * src.size()));
}

void download(const Session& s, std::vector<double>& dst, const double* src) {
    if (!dst.empty()) s.check(vrg_copy_d2h(s.ctx(), dst.data(), src, sizeof(double) * dst.size()));
}

DevBuf deviceField(const Session& s, const ScalarField& f) {
    DevBuf b(s, f.v.size());
    upload(s, b.get(), f.v);
    return b;
}

DevBuf deviceVector(const Session& s, const VectorField& v) {
    const std::size_t N = v[0].v.size();
    DevBuf b(s, 2 * N);
    upload(s, b.get(), v[0].v);
    upload(s, b.at(N), v[1].v);
    return b;
}

DevBuf deviceFrames(const Session& s, const std::vector<ScalarField>& frames) {
    const std::size_t N = frames.empty() ? 0 : frames[0].v.size();
    DevBuf b(s, frames.size() * N);
    for (std::size_t j = 0; j < frames.size(); ++j) upload(s, b.at(j * N), frames[j].v);
    return b;
}

ScalarField hostField(const Session& s, const Grid& g, const double* src) {
    ScalarField f(g);
    download(s, f.v, src);
    return f;
}

VectorField hostVector(const Session& s, const Grid& g, const double* src) {
    VectorField v(g);
    download(s, v[0].v, src);
    download(s, v[1].v, src + g.points());
    return v;
}

std::vector<ScalarField> hostFrames(const Session& s, const Grid& g, const double* src, int count) {
    std::vector<ScalarField> out;
    out.reserve(static_cast<std::size_t>(count));
    for (int j = 0; j < count; ++j) out.push_back(hostField(s, g, src + static_cast<std::size_t>(j) * g.points()));
    return out;
}

}  // namespace veloreg::vrgdev
