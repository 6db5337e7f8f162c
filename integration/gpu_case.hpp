// integration/gpu_case.hpp — the reference-side binding a Nauticle maintainer adds to run
// a Case on the GPU through libnau_b200.so (include/nauticle_gpu.h). Compiled and tested
// here against the reference's own headers (/root/reference/proj/include) by
// oracle/Makefile (target _ref/libgpucase.so; tests/test_gpu_binding.py).
//
// GpuCase mirrors a Case (src/case.cpp, include/nauticle/case.hpp) into a device context:
// the domain (domain.hpp:19-49), positions and every workspace field (workspace.hpp),
// constants, variables and the equation list (equation.hpp: Equation::to_text form),
// and the case's RandomState (sfl/random_state.hpp). solve_step() replaces
// Case::solve_step(pool) (case.cpp:65-67): the device executor (nau_case_*) solves the
// equations with Case::solve_equation's semantics. download() writes the device state
// back into Field::values / Variable::value, e.g. before write_vtk. Errors come back as
// nauticle::Error with the reference's kinds (error.hpp:10-69) and messages.
#pragma once

#include <string>
#include <unordered_map>

#include "nauticle/case.hpp"
#include "nauticle_gpu.h"

namespace nauticle {

class GpuCase {
public:
    explicit GpuCase(Case& cs, int device = 0, bool fast = false);
    ~GpuCase();
    GpuCase(const GpuCase&) = delete;
    GpuCase& operator=(const GpuCase&) = delete;

    void solve_step();  // ≙ Case::solve_step (case.cpp:65-67)
    void download();    // device fields -> Field::values, executor variables -> Variable::value
    nau_ctx* context() const { return ctx_; }

private:
    void check(nau_status s) const;        // context errors
    void check_case(nau_status s) const;   // executor errors (carry the equation name)
    Case& cs_;
    nau_ctx* ctx_ = nullptr;
    nau_case* exec_ = nullptr;
    std::unordered_map<std::string, int> field_id_;
};

}  // namespace nauticle
