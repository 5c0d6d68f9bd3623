// Status plumbing for the C-ABI: thread-local last-error message and the
// exception -> status-code translation shared by all extern "C" entry points.
#pragma once

#include <exception>
#include <string>

#include "amsp/plan.hpp"
#include "amsp_c.h"

namespace amsp {

void set_last_error(const std::string& msg);

// Thrown by engine code for CUDA / peer failures (status AMSP_ECUDA).
class CudaFailure : public std::runtime_error {
 public:
  explicit CudaFailure(const std::string& what) : std::runtime_error(what) {}
};

// Runs `f` and maps exceptions to status codes. NoFeasiblePlanError and
// InfeasibleError map to AMSP_EINFEASIBLE, other shardplan::Error (and any
// std::exception) to AMSP_EINVAL, CudaFailure to AMSP_ECUDA.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return AMSP_OK;
  } catch (const CudaFailure& e) {
    set_last_error(e.what());
    return AMSP_ECUDA;
  } catch (const shardplan::NoFeasiblePlanError& e) {
    set_last_error(e.what());
    return AMSP_EINFEASIBLE;
  } catch (const shardplan::InfeasibleError& e) {
    set_last_error(e.what());
    return AMSP_EINFEASIBLE;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return AMSP_EINVAL;
  } catch (...) {
    set_last_error("unknown error");
    return AMSP_EINVAL;
  }
}

}  // namespace amsp
