// Bridge between the spgsim:: C++ API and the C ABI: per-device contexts,
// host<->device CSR transfer, and status -> exception mapping.
#pragma once

#include <vector>

#include "spg/capi.h"
#include "spgsim/csr.hpp"

namespace spgsim::detail {

[[noreturn]] void throw_status(spg_status st);
inline void check(spg_status st) {
    if (st != SPG_OK) throw_status(st);
}

int device_count();                 // visible devices (throws DeviceError if none)
spg_ctx* context(int device = 0);   // lazily created, process-lifetime

// Owning device handle.
struct DevCsr {
    spg_csr* p = nullptr;
    DevCsr() = default;
    explicit DevCsr(spg_csr* h) : p(h) {}
    DevCsr(DevCsr&& o) noexcept : p(o.p) { o.p = nullptr; }
    DevCsr& operator=(DevCsr&& o) noexcept {
        std::swap(p, o.p);
        return *this;
    }
    DevCsr(const DevCsr&) = delete;
    ~DevCsr() {
        if (p) spg_csr_free(p);
    }
};

DevCsr upload(spg_ctx* ctx, const CsrMatrix& m);
CsrMatrix download(spg_ctx* ctx, const spg_csr* m);

}  // namespace spgsim::detail
