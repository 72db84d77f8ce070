// segconv/op_counts.hpp -- drop-in forwarding header: the reference's
// proj/include/segconv/op_counts.hpp names come from the B200 host API
// (../segconv_b200.hpp over the C ABI in ../segconv_b200.h).
#pragma once
#include "../segconv_b200.hpp"
