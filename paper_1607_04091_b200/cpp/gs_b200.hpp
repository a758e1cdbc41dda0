// gs_b200.hpp -- the whole drop-in header tree (paper_1607_04091_b200/cpp/include/gs)
// in one include: the reference API of namespace gs over libgs_b200.so.
// Compile with -I<repo>/paper_1607_04091_b200/cpp/include -I<repo>/include and an
// Eigen include path (the reference API returns Eigen types).
#pragma once

#include "gs/dyadic.hpp"
#include "gs/error.hpp"
#include "gs/fourier.hpp"
#include "gs/freq2wave.hpp"
#include "gs/nufft.hpp"
#include "gs/patterns.hpp"
#include "gs/scaling.hpp"
#include "gs/signals.hpp"
#include "gs/solver.hpp"
#include "gs/weights.hpp"
