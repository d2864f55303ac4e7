// tuning.hpp — the process-wide kernel-selection settings (include/srl.h
// srl_tuning).  Defaults are the production choices; the alternatives stay
// selectable for measurement and for their parity tests.  Nothing in the
// library reads the environment (no environment overrides).
#pragma once
#include "srl.h"

namespace srl {
extern srl_tuning g_tuning;
inline const srl_tuning& tuning() { return g_tuning; }
// per-device "attribute already set" bookkeeping for cudaFuncSetAttribute:
// returns true exactly once per (slot, current device)
bool once_per_device(int slot);
enum { kOnceGemmPair = 0, kOnceGemmSingle = 1, kOnceAttn32 = 2, kOnceAttn64 = 3, kOnceAttn128 = 4,
       kOnceCtl = 5, kOnceSample = 6, kOnceGemmMlp = 7, kOnceAttn128s6 = 8, kOnceAttn128s3 = 9,
       kOnceSlots = 10 };
}  // namespace srl
