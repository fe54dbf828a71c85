// Prints std::to_chars(double) of each double (hex bits on stdin, one per line):
// the reference's format_double (io.cpp:55-60), for checking report.format_double.
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <string>

int main() {
    std::string line;
    while (std::getline(std::cin, line)) {
        uint64_t bits = std::stoull(line, nullptr, 16);
        double v;
        std::memcpy(&v, &bits, 8);
        char buf[64];
        auto r = std::to_chars(buf, buf + sizeof(buf), v);
        std::cout << std::string(buf, r.ptr) << "\n";
    }
    return 0;
}
