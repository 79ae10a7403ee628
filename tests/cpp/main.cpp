// main() of the mini doctest runner (tests/cpp/doctest.h)
#define MINI_DOCTEST_MAIN
#include "doctest.h"
