// Forced-include prelude for compiling the reference sources IN PLACE
// (/root/reference/proj) without editing them. TEST INFRASTRUCTURE ONLY.
//
// /root/reference/proj/include/fsg/fastmath.hpp:128 and :136 call the
// fsg::-scoped fast_exp_neg from global scope, which does not compile as
// shipped. Declaring it up front and importing it into the global namespace
// makes the unqualified calls resolve (workaround 1).
#pragma once
namespace fsg {
inline double fast_exp_neg(double x);
}
using fsg::fast_exp_neg;
