// Runner for the gtest shim: executes every registered TEST, prints a
// gtest-like summary and returns non-zero on any failure.
#include <exception>
#include <iostream>

#include "gtest/gtest.h"

int main() {
  int failed_tests = 0;
  const auto& tests = gtshim::registry();
  for (const auto& t : tests) {
    const int before = gtshim::failures();
    std::cout << "[ RUN      ] " << t.suite << "." << t.name << std::endl;
    try {
      t.fn();
    } catch (const std::exception& e) {
      std::cerr << "uncaught exception: " << e.what() << std::endl;
      ++gtshim::failures();
    } catch (...) {
      std::cerr << "uncaught non-std exception" << std::endl;
      ++gtshim::failures();
    }
    const bool ok = gtshim::failures() == before;
    if (!ok) ++failed_tests;
    std::cout << (ok ? "[       OK ] " : "[  FAILED  ] ") << t.suite << "." << t.name << std::endl;
  }
  std::cout << "[==========] " << tests.size() << " tests, " << failed_tests << " failed"
            << std::endl;
  return failed_tests == 0 ? 0 : 1;
}
