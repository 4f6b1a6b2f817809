#pragma once
// The product's double-double / quad-double arithmetic built for the host.
//
// The value types of the drop-in (double_double, quad_double, cplx) get their
// operators from the very source the B200 kernels run:
// paper_1210_0800_b200/csrc/xarith.cuh, which compiles as plain C++ and is
// checked bit for bit against the reference's operators over every operand
// class (tests/test_arith_host.py, tests/test_oracle.py).  Like the reference
// (eft.hpp:1-5, proj/CMakeLists.txt:15) it needs round-to-nearest and NO
// floating-point contraction: compile callers with -ffp-contract=off.
#include "../../../paper_1210_0800_b200/csrc/xarith.cuh"
