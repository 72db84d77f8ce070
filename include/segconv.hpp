// segconv.hpp -- drop-in umbrella header (reference proj/include/segconv.hpp:8-22):
// the segregated transpose convolution's operator set, tensors, geometry,
// op counts and SGC1 I/O from the B200 host API.  The reference's CLI,
// benchmark, PNM image and training-demo headers are not part of this build
// (out of scope); the trainable layers net::FusedTConv and
// net::ConvValid are in segconv_b200.hpp.
#pragma once
#include "segconv_b200.hpp"
