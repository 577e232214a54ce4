// ndactor/kernel.hpp -- kernel arguments and kernel definitions.
//
// Reference: p/core/include/ndactor/kernel.hpp:17-193, where a kernel is a
// list of host lambdas ("phases") run per simulated work item.  On B200 a
// KernelDef is a name plus a launcher: a host function that launches a real
// sm_100a kernel (usually through an extern "C" entry of libndx.so or the
// user's own library) on the command's stream.  Barrier phases become
// __syncthreads inside the CUDA kernel.
#pragma once

#include <array>
#include <cstddef>
#include <functional>
#include <string>
#include <vector>

#include "ndactor/buffer.hpp"
#include "ndactor/ndrange.hpp"

namespace ndactor {

/// Argument bound at enqueue time: device buffer, group-local (shared)
/// memory, or a scalar passed by value (kernel.hpp:17-45).
struct KernelArg {
  enum class Kind : std::uint8_t { global, local, scalar };

  Kind kind = Kind::scalar;
  Buffer buffer;
  ElemType local_type = ElemType::u32;
  std::size_t local_len = 0;
  Scalar value;

  static KernelArg global(Buffer b) {
    KernelArg a;
    a.kind = Kind::global;
    a.buffer = std::move(b);
    return a;
  }
  static KernelArg local(ElemType t, std::size_t len) {
    KernelArg a;
    a.kind = Kind::local;
    a.local_type = t;
    a.local_len = len;
    return a;
  }
  static KernelArg scalar(Scalar v) {
    KernelArg a;
    a.kind = Kind::scalar;
    a.value = v;
    return a;
  }
};

/// What a launcher receives: the resolved launch shape and every argument
/// in declaration order.  For global args `ptr[i]`/`len[i]` are the device
/// pointer and element count; local args are carved out of one dynamic
/// shared-memory block (`smem_offset[i]`, `len[i]` elements); scalar args
/// are in `scalar[i]`.
struct LaunchParams {
  static constexpr std::size_t kMaxArgs = 16;
  void* stream = nullptr;  // cudaStream_t
  unsigned rank = 1;
  std::array<unsigned, 3> grid{1, 1, 1};
  std::array<unsigned, 3> block{1, 1, 1};
  std::array<std::size_t, 3> offset{0, 0, 0};
  std::array<std::size_t, 3> global{1, 1, 1};
  std::size_t shared_bytes = 0;
  std::size_t nargs = 0;
  std::array<void*, kMaxArgs> ptr{};
  std::array<std::size_t, kMaxArgs> len{};
  std::array<std::size_t, kMaxArgs> smem_offset{};
  std::array<Scalar, kMaxArgs> scalar{};
};

/// Returns 0 or a CUDA/ndx error code; must not throw.
using Launcher = std::function<int(const LaunchParams&)>;

struct KernelDef {
  std::string name;
  Launcher launch;

  KernelDef() = default;
  KernelDef(std::string n, Launcher l) : name(std::move(n)), launch(std::move(l)) {}
};

}  // namespace ndactor
