// Error classes of the drop-in boundary (reference common.hpp:14-26) and the
// C-ABI status mapping (nrr_cli.cpp:266-278: 2 IO, 3 numerical, 4 config).
#pragma once

#include <stdexcept>
#include <string>

namespace nrr_b200 {

struct IoError : std::runtime_error {
    explicit IoError(const std::string& m) : std::runtime_error(m) {}
};
struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct NumericalError : std::runtime_error {
    explicit NumericalError(const std::string& m) : std::runtime_error(m) {}
};
struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

void set_last_error(const std::string& msg);

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const IoError& e) {
        set_last_error(e.what());
        return 2;
    } catch (const NumericalError& e) {
        set_last_error(e.what());
        return 3;
    } catch (const ConfigError& e) {
        set_last_error(e.what());
        return 4;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return 5;
    }
}

}  // namespace nrr_b200
