// Host cost of the drop-in Image: std::vector<uint8_t>(3840*2160*3) allocation + zero fill,
// a single-thread memcpy of the same size, and an 8-thread copy (GPU box host).
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
int main() {
    const size_t n = size_t{3840} * 2160 * 3;
    std::vector<unsigned char> src(n, 1);
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    double t_alloc = 0, t_copy = 0, t_par = 0;
    const int reps = 20;
    for (int r = 0; r < reps; ++r) {
        auto a = now();
        std::vector<unsigned char> v(n);
        auto b = now();
        std::memcpy(v.data(), src.data(), n);
        auto c = now();
        std::vector<std::thread> th;
        const size_t chunk = n / 8;
        for (int k = 0; k < 8; ++k) th.emplace_back([&, k] { std::memcpy(v.data() + k * chunk, src.data() + k * chunk, chunk); });
        for (auto& t : th) t.join();
        auto d = now();
        t_alloc += ms(a, b), t_copy += ms(b, c), t_par += ms(c, d);
    }
    std::printf("alloc+zero %.3f ms, memcpy 1 thread %.3f ms, 8 threads (incl. spawn) %.3f ms, hw threads %u\n",
                t_alloc / reps, t_copy / reps, t_par / reps, std::thread::hardware_concurrency());
}
