// ORACLE / TEST INFRASTRUCTURE — entry point for the shimmed reference unit tests.
#include "doctest.h"
int main() { return doctest_shim::run_all(); }
