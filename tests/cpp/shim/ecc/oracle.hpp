// The reference's brute-force oracle (naive_ecc, oracle.hpp:80-107) for the
// reference's own tests compiled against the drop-in headers: test
// infrastructure, pulled from /root/reference at build time (the binaries
// are built in the container that has it and travel to the GPU box).  Its
// includes ("ecc/common.hpp", "ecc/curve.hpp", ...) resolve to the drop-in.
#pragma once
#include "/root/reference/proj/include/ecc/oracle.hpp"
