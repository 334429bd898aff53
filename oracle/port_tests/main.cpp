// ORACLE — TEST INFRASTRUCTURE ONLY.
// Runs every registered port test; prints one "RESULT <suite>/<name> PASS|FAIL"
// line per case (parsed by tests/test_oracle_port.py).  Optional argv[1]
// filters by substring.
#include <cstdio>
#include <cstring>
#include <exception>

#include "harness.hpp"

int main(int argc, char** argv) {
  int bad = 0, ran = 0;
  for (const port::Case& c : port::registry()) {
    std::string full = std::string(c.suite) + "/" + c.name;
    if (argc > 1 && full.find(argv[1]) == std::string::npos) continue;
    const int before = port::failures();
    bool threw = false;
    try {
      c.fn();
    } catch (const std::exception& e) {
      threw = true;
      std::printf("    unexpected exception: %s\n", e.what());
    }
    const bool ok = !threw && port::failures() == before;
    std::printf("RESULT %s %s\n", full.c_str(), ok ? "PASS" : "FAIL");
    bad += ok ? 0 : 1;
    ++ran;
  }
  std::printf("SUMMARY %d cases, %d failed, %d checks\n", ran, bad, port::checks());
  return bad == 0 ? 0 : 1;
}
