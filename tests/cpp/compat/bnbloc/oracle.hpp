// Compat shim: the reference's "bnbloc/oracle.hpp" resolved to the B200 facade
// (include/bnbloc_b200.hpp) in namespace bnbloc, so the reference's own test
// sources compile unmodified against the device implementation.
#pragma once
#define bnbloc_b200 bnbloc
#include "bnbloc_b200.hpp"
