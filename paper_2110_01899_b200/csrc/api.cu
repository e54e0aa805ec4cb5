// C ABI (include/rf.h): validation, workspace planning, TMA descriptor creation and kernel dispatch.
// Every compute step of the path runs in this library's kernels; there is no CPU fallback.
// One translation unit, split into files by topic:
//   api_internal.cuh .. helpers, tracing, TMA descriptors, launchers (K3/K4 hybrids, K5), workspace plans
//   abi_core.cuh ...... rf_moments, rf_estimate_tau, rf_gram, tracing, the mainloop test hook
//   abi_ktilde.cuh .... NEXT-2 rf_ktilde
//   abi_trf.cuh ....... NEXT-1 Ternary Random Features
//   abi_ctx.cuh ....... the context and its options; G5 (multi-GPU G): tile map, peer-memory and NCCL exchanges
//   abi_phi.cuh ....... Φ by EQ1 / EQ2, row split
//   abi_ridge.cuh ..... NEXT-4 ridge regression
#include "api_internal.cuh"
#include "abi_core.cuh"
#include "abi_ktilde.cuh"
#include "abi_trf.cuh"
#include "abi_ctx.cuh"
#include "abi_phi.cuh"
#include "abi_ridge.cuh"
