// Entry point for the reference's unit tests compiled against the B200 facade.
#define DOCTEST_SHIM_MAIN
#include "doctest.h"
