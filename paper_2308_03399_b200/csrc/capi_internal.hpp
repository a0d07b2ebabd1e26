// Internal pieces shared by the C-ABI translation units.
#pragma once

#include <atomic>
#include <exception>
#include <new>
#include <stdexcept>
#include <string>

#include "engine/devprog.hpp"
#include "shotsim_b200.h"
#include "shotsim_b200.hpp"

struct ssb_program {
  uint64_t uid;
  shotsim::NoisyCircuit nc;
  shotsim::FlatProgram flat;
  ssb::HostDevProgram dev;
};

namespace ssb {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);
uint64_t next_program_uid();
// engine.cu: drop every engine's device copies of program `uid`.
void evict_program(uint64_t uid);

// Maps the reference's exception types onto ssb_status (shotsim_b200.h).
template <class F>
int guard(F&& f) {
  try {
    f();
    return SSB_OK;
  } catch (const shotsim::CapacityError& e) {
    set_last_error(std::string("CapacityError: ") + e.what());
    return SSB_ERR_CAPACITY;
  } catch (const shotsim::DegenerateDistribution& e) {
    set_last_error(std::string("DegenerateDistribution: ") + e.what());
    return SSB_ERR_DEGENERATE;
  } catch (const shotsim::ConfigError& e) {
    set_last_error(std::string("ConfigError: ") + e.what());
    return SSB_ERR_CONFIG;
  } catch (const std::invalid_argument& e) {
    set_last_error(std::string("invalid_argument: ") + e.what());
    return SSB_ERR_INVALID_ARGUMENT;
  } catch (const CudaError& e) {
    set_last_error(std::string("CUDA: ") + e.what());
    return SSB_ERR_CUDA;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return SSB_ERR_CAPACITY;
  } catch (const std::exception& e) {
    set_last_error(std::string("error: ") + e.what());
    return SSB_ERR_RUNTIME;
  }
}

}  // namespace ssb
