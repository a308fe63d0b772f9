// The usage example of the reference README (proj/README.md:108-128 pattern):
// descriptor -> plan -> policy, then the hot-path calls on host containers.
// Compiled unchanged against the drop-in headers.
#include <cabl/cabl.hpp>

#include <cstdio>

int main() {
    using namespace cabl;
    const MachineDescriptor machine = default_machine(8);
    const BlockingPlan plan = derive_blocking_plan(machine);
    const ExecPolicy policy(plan, 4);

    Vector<double> x(1000), y(1000), c(64);
    for (std::size_t i = 0; i < x.len(); ++i) {
        x[i] = 0.001 * double(i);
        y[i] = 1.0;
    }
    DenseMatrix<double> A(64, 1000, Layout::ColMajor, 0.5);
    try {
        const double d = dot(x, y, 0.0, policy);
        gemv_col_major(A, x, c, policy);
        std::printf("dot = %.6f, c[0] = %.6f, variant %d\n", d, c[0], int(last_exec().variant));
        return (d > 499.4 && d < 499.6 && c[0] > 249.7 && c[0] < 249.8) ? 0 : 1;
    } catch (const std::exception& e) {
        std::printf("error: %s\n", e.what());
        return 3;
    }
}
