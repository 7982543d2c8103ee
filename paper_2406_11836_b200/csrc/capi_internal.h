// Error plumbing shared by the C-ABI translation units: C++ exceptions inside
// the library become status codes + a thread-local message at the boundary.
#pragma once

#include <stdexcept>
#include <string>

namespace dgs_b200 {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);

template <typename F>
int dgs_guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const CudaError& e) {
        set_last_error(e.what());
        return 4;
    } catch (const NcclError& e) {
        set_last_error(e.what());
        return 5;
    } catch (const std::invalid_argument& e) {
        set_last_error(e.what());
        return 1;
    } catch (const std::domain_error& e) {
        set_last_error(e.what());
        return 3;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return 2;
    } catch (...) {
        set_last_error("unknown error");
        return 2;
    }
}

}  // namespace dgs_b200
