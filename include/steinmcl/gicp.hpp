// Reference header name (proj/include/steinmcl/gicp.hpp): forwards to the B200 facade.
#pragma once
#include "steinmcl/b200.hpp"
