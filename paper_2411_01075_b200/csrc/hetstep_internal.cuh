// Shared helpers of the hetstep C-ABI translation units (not installed).
#pragma once
#include <cstdarg>
#include <cstdint>
#include <string>

namespace het {
extern thread_local std::string g_last_error;
// Record a printf-style message for het_last_error() and return `code`.
int fail(int code, const char* fmt, ...);
// HET_ECUDA with the launch error text if the last launch failed.
int check_launch(const char* what);
// Grid size for a grid-stride loop over `work_items` (x threads per CTA),
// capped at 8 resident 256-thread CTAs per SM.
int grid_for(int64_t work_items, int threads);
// SMs a persistent grid may assume: the device's count, or the budget set by
// het_tune(HET_TUNE_SM_BUDGET) for a rank confined to a green-context partition.
int sm_count();
// het_tune(HET_TUNE_SYMM_TIMEOUT_MS): spin limit of the symmetric barriers.
int set_symm_timeout_ms(int ms);
}  // namespace het
