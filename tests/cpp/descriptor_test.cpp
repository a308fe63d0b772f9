// cabl/descriptor_json.hpp without a GPU: load documents given on the command
// line and print, per document, either the derived plan or the error text
// (one line each), for tests/test_descriptor_cpp.py to compare with the
// Python loader (paper_2108_02025_b200/machine.py) and the reference rules.
#include <cabl/descriptor_json.hpp>

#include <cstdio>

int main(int argc, char** argv) {
    for (int a = 1; a < argc; ++a) {
        try {
            const cabl::MachineDescriptor md = cabl::load_descriptor_file(argv[a]);
            const cabl::BlockingPlan p = cabl::derive_blocking_plan(md);
            std::printf("ok cores=%u element_bytes=%llu levels=%zu l1=%llu l2=%llu m_c=%llu "
                        "dot_block=%llu dot_cutoff=%llu\n",
                        md.cores, (unsigned long long)md.element_bytes, md.num_levels(),
                        (unsigned long long)md.level(0).size_bytes(),
                        (unsigned long long)md.level(1).size_bytes(), (unsigned long long)p.m_c,
                        (unsigned long long)p.dot_block, (unsigned long long)p.dot_cutoff);
        } catch (const cabl::DescriptorError& e) {
            std::printf("error %s\n", e.what());
        }
    }
    return 0;
}
