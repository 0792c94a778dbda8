// Drop-in include path for code written against granndis_core: the reference
// header name, served by the B200 engine declarations.  The planner's ModelSpec
// (cost_model.hpp:24-29) is declared there; the closed-form cost model and the
// simulator are out of scope.
#pragma once
#include "granndis_b200/granndis.hpp"
