// Reference header name (proj/include/steinmcl/gaussian_cloud.hpp): forwards to the B200 facade.
#pragma once
#include "steinmcl/b200.hpp"
