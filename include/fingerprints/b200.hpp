// b200.hpp -- umbrella header of the B200 fingerprint scan's C++ API.
//
// Reference code written against fingerprints::FingerprintedDictionary
// (dictionary.hpp:47) compiles against this header unchanged for the
// matching path: the alias below selects the GPU dictionary.  Link with
// libfpg.so (paper_1711_08475_b200/lib).
#pragma once

#include "gpu_dictionary.hpp"
#include "gpu_letters.hpp"
#include "gpu_scheme.hpp"

namespace fingerprints {
using FingerprintedDictionary = GpuFingerprintedDictionary;
}
