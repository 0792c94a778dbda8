// Drop-in include path for code written against granndis_core: the reference
// header name, served by the B200 engine declarations (Batch, BatchPlan,
// estimate_batch_memory, plan_cobatch[_fixed_r] on the device planner,
// plan_minibatch_baseline, plan_to_json / save_plan_json).
#pragma once
#include "granndis_b200/granndis.hpp"
