// shim: the reference header errors.hpp maps onto the B200 drop-in
#pragma once
#include "loadsched_gpu.hpp"
