// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim around the *unmodified* reference templates, compiled from the
// headers where they lie (`/root/reference/proj/include/cabl/*.hpp`) by
// `oracle/Makefile` into `oracle/_ref/libcabl_ref.so`.  It lets the Python
// tests and `bench.py --impl reference` call the reference CPU path:
//
//   op 0  dot        reference: kernels.hpp:134-164 (`dot`) / :119-127 (`dot_ref`)
//   op 1  gemv-row   reference: kernels.hpp:230-257 (`gemv_row_major`) / :171-181
//   op 2  gemv-col   reference: kernels.hpp:187-224 (`gemv_col_major`) / :171-181
//   op 3  ger        reference: kernels.hpp:277-313 (`ger`) / :264-270 (`ger_ref`)
//
// A "session" owns reference `Vector`/`DenseMatrix` containers so that the
// timed call (`cabl_ref_run`) contains only the reference kernel, never the
// copy into the containers.  The policy is built exactly as the reference
// acceptance suite builds its own (acceptance.cpp:417-425):
// ExecPolicy(derive_blocking_plan(default_machine(cores) with
// element_bytes = sizeof(T)), threads).

#include <cabl/kernels.hpp>

#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>

namespace {

thread_local std::string g_err;

struct SessionBase {
    virtual ~SessionBase() = default;
    virtual int run(int use_ref, unsigned threads, double* scalar_out) = 0;
    virtual void get(void* out) const = 0;
    virtual void set_out(const void* src) = 0;
    virtual unsigned last_threads() const = 0;
    virtual int last_variant() const = 0;
};

template <typename T>
struct Session final : SessionBase {
    int op;
    std::uint64_t m, n;
    cabl::Layout layout;
    cabl::Vector<T> x, y;   // y doubles as c for gemv
    cabl::DenseMatrix<T> A; // A for gemv, C for ger
    T alpha0{};
    unsigned cores;
    cabl::ExecProbe probe{};

    Session(int op_, int layout_, std::uint64_t m_, std::uint64_t n_, const T* a,
            const T* xv, const T* yv, T alpha, unsigned cores_)
        : op(op_), m(m_), n(n_),
          layout(layout_ == 1 ? cabl::Layout::ColMajor : cabl::Layout::RowMajor),
          alpha0(alpha), cores(cores_) {
        if (op == 0) {
            x = cabl::Vector<T>(n);
            y = cabl::Vector<T>(n);
            if (n) {
                std::memcpy(x.data(), xv, n * sizeof(T));
                std::memcpy(y.data(), yv, n * sizeof(T));
            }
        } else if (op == 1 || op == 2) {
            A = cabl::DenseMatrix<T>(m, n, layout);
            x = cabl::Vector<T>(n);
            y = cabl::Vector<T>(m);
            if (m * n) std::memcpy(A.data(), a, m * n * sizeof(T));
            if (n) std::memcpy(x.data(), xv, n * sizeof(T));
            if (m) std::memcpy(y.data(), yv, m * sizeof(T));
        } else {
            // ger: x has m entries, y has n, C = a (m x n, layout)
            A = cabl::DenseMatrix<T>(m, n, layout);
            x = cabl::Vector<T>(m);
            y = cabl::Vector<T>(n);
            if (m * n) std::memcpy(A.data(), a, m * n * sizeof(T));
            if (m) std::memcpy(x.data(), xv, m * sizeof(T));
            if (n) std::memcpy(y.data(), yv, n * sizeof(T));
        }
    }

    cabl::ExecPolicy policy(unsigned threads) const {
        cabl::MachineDescriptor md = cabl::default_machine(cores);
        md.element_bytes = sizeof(T);
        return cabl::ExecPolicy(cabl::derive_blocking_plan(md), threads);
    }

    int run(int use_ref, unsigned threads, double* scalar_out) override {
        const cabl::ExecPolicy pol = policy(threads);
        if (op == 0) {
            T r = use_ref ? cabl::dot_ref(x, y, alpha0) : cabl::dot(x, y, alpha0, pol);
            if (scalar_out) *scalar_out = static_cast<double>(r);
        } else if (op == 1) {
            if (use_ref) cabl::gemv_ref(A, x, y);
            else cabl::gemv_row_major(A, x, y, pol);
        } else if (op == 2) {
            if (use_ref) cabl::gemv_ref(A, x, y);
            else cabl::gemv_col_major(A, x, y, pol);
        } else {
            if (use_ref) cabl::ger_ref(x, y, A);
            else cabl::ger(x, y, A, pol);
        }
        probe = cabl::last_exec();
        return 0;
    }

    void get(void* out) const override {
        if (op == 1 || op == 2) {
            if (m) std::memcpy(out, y.data(), m * sizeof(T));
        } else if (op == 3) {
            if (m * n) std::memcpy(out, A.data(), m * n * sizeof(T));
        }
    }

    void set_out(const void* src) override {
        if (op == 1 || op == 2) {
            if (m) std::memcpy(y.data(), src, m * sizeof(T));
        } else if (op == 3) {
            if (m * n) std::memcpy(A.data(), src, m * n * sizeof(T));
        }
    }

    unsigned last_threads() const override { return probe.threads_used; }
    int last_variant() const override { return static_cast<int>(probe.variant); }
};

} // namespace

extern "C" {

// dtype: 4 = float, 8 = double.  layout: 0 = row-major, 1 = col-major.
// dot: a unused, x/y length n.  gemv: a = A (m x n), x length n, y = c length m.
// ger: a = C (m x n), x length m, y length n.
void* cabl_ref_new(int op, int dtype, int layout, std::uint64_t m, std::uint64_t n,
                   const void* a, const void* x, const void* y, double alpha0,
                   unsigned cores) {
    try {
        if (dtype == 4)
            return new Session<float>(op, layout, m, n, static_cast<const float*>(a),
                                      static_cast<const float*>(x),
                                      static_cast<const float*>(y),
                                      static_cast<float>(alpha0), cores);
        if (dtype == 8)
            return new Session<double>(op, layout, m, n, static_cast<const double*>(a),
                                       static_cast<const double*>(x),
                                       static_cast<const double*>(y), alpha0, cores);
        g_err = "bad dtype";
    } catch (const std::exception& e) {
        g_err = e.what();
    }
    return nullptr;
}

int cabl_ref_run(void* h, int use_ref, unsigned threads, double* scalar_out) {
    try {
        return static_cast<SessionBase*>(h)->run(use_ref, threads, scalar_out);
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

void cabl_ref_get(void* h, void* out) { static_cast<SessionBase*>(h)->get(out); }
void cabl_ref_set_out(void* h, const void* src) { static_cast<SessionBase*>(h)->set_out(src); }
unsigned cabl_ref_last_threads(void* h) { return static_cast<SessionBase*>(h)->last_threads(); }
int cabl_ref_last_variant(void* h) { return static_cast<SessionBase*>(h)->last_variant(); }
void cabl_ref_free(void* h) { delete static_cast<SessionBase*>(h); }
const char* cabl_ref_last_error() { return g_err.c_str(); }

} // extern "C"
