// hpk_grouping_wide.cu — the 128-unit build of the grouping engines
// (hpk_grouping.cu compiled with HPK_MAXN = 128 into namespace hpk_wide, its
// C entry points renamed *_wide). The primary build (64 units) forwards
// problems with 65..128 TP units here; see the MAXN note in hpk_grouping.cu.
#define HPK_WIDE 1
#define HPK_MAXN 128
#define hpk hpk_wide
#define hpk_timing_bridge hpk_timing_bridge_wide
#define hpkp_fail hpkp_fail_wide
#define hpk_selftest_decide hpk_selftest_decide_wide
#define hpk_version hpk_version_wide
#define hpk_last_error hpk_last_error_wide
#define hpk_device_count hpk_device_count_wide
#define hpk_search_config_init hpk_search_config_init_wide
#define hpk_last_timing hpk_last_timing_wide
#define hpk_reset_timing hpk_reset_timing_wide
#define hpk_grouping_search hpk_grouping_search_wide
#define hpk_assign_devices hpk_assign_devices_wide
#include "hpk_grouping.cu"
