// Drop-in include path for code written against granndis_core: the reference
// header name, served by the B200 engine declarations.
#pragma once
#include "granndis_b200/granndis.hpp"
