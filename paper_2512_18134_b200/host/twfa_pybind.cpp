// _twfa: pybind11 binding of the C ABI (include/twfa.h).
//
// Sits next to the reference's own pybind module `_weftsched`
// (bindings/module.cpp:219-249) and follows its conventions:
// * JSON documents in, dicts out;
// * malformed documents and bad arguments raise ValueError
//   (std::invalid_argument, test_smoke.py:80-82);
// * CUDA failures raise RuntimeError.
//
// Device buffers cross as integer addresses (torch.Tensor.data_ptr()), so the
// module needs no torch headers. The product is libtwfa.so; this module only
// translates calls.
#include <pybind11/pybind11.h>

#include <memory>
#include <stdexcept>
#include <string>

#include "twfa.h"

namespace py = pybind11;

namespace {

void check(int rc) {
  if (rc == TWFA_OK) return;
  if (rc == TWFA_EDOMAIN || rc == TWFA_EUSAGE) throw std::invalid_argument(twfa_last_error());
  throw std::runtime_error(twfa_last_error());
}

struct Plan {
  twfa_plan* p = nullptr;
  Plan(const std::string& problem, const std::string& solution) {
    check(twfa_plan_create(problem.c_str(), solution.c_str(), &p));
  }
  ~Plan() { twfa_plan_destroy(p); }
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;

  // JSON description of the lowered plan (as a dict, like _weftsched.joint)
  py::object describe() const {
    size_t need = 0;
    check(twfa_plan_describe(p, nullptr, 0, &need));
    std::string buf(need, '\0');
    check(twfa_plan_describe(p, buf.data(), buf.size(), &need));
    buf.resize(need ? need - 1 : 0);
    return py::module_::import("json").attr("loads")(buf);
  }

  void fa_fwd(std::uintptr_t q, std::uintptr_t k, std::uintptr_t v, std::uintptr_t o, std::uintptr_t lse, int B,
              int H, int S, bool causal, float scale, std::uintptr_t stream) const {
    py::gil_scoped_release nogil;
    check(twfa_fa_fwd(p, reinterpret_cast<const void*>(q), reinterpret_cast<const void*>(k),
                      reinterpret_cast<const void*>(v), reinterpret_cast<void*>(o), reinterpret_cast<float*>(lse), B, H,
                      S, 128, causal ? 1 : 0, scale, reinterpret_cast<void*>(stream)));
  }

  // FA backward (plan from an FA-backward schedule); workspace of at least
  // workspace_size(B, H, S) bytes, device pointers as integers
  void fa_bwd(std::uintptr_t q, std::uintptr_t k, std::uintptr_t v, std::uintptr_t o, std::uintptr_t dout,
              std::uintptr_t lse, std::uintptr_t dq, std::uintptr_t dk, std::uintptr_t dv, std::uintptr_t ws,
              std::size_t ws_bytes, int B, int H, int S, bool causal, float scale, std::uintptr_t stream) const {
    py::gil_scoped_release nogil;
    check(twfa_fa_bwd(p, reinterpret_cast<const void*>(q), reinterpret_cast<const void*>(k),
                      reinterpret_cast<const void*>(v), reinterpret_cast<const void*>(o),
                      reinterpret_cast<const void*>(dout), reinterpret_cast<const float*>(lse),
                      reinterpret_cast<void*>(dq), reinterpret_cast<void*>(dk), reinterpret_cast<void*>(dv),
                      reinterpret_cast<void*>(ws), ws_bytes, B, H, S, 128, causal ? 1 : 0, scale,
                      reinterpret_cast<void*>(stream)));
  }

  void gemm(std::uintptr_t a, std::uintptr_t b, std::uintptr_t c, int M, int N, int K, std::uintptr_t stream) const {
    py::gil_scoped_release nogil;
    check(twfa_gemm(p, reinterpret_cast<const void*>(a), reinterpret_cast<const void*>(b), reinterpret_cast<void*>(c), M,
                    N, K, reinterpret_cast<void*>(stream)));
  }
};

}  // namespace

PYBIND11_MODULE(_twfa, m) {
  m.doc() = "B200 executor of Twill schedules (C ABI include/twfa.h), JSON in / dict out like _weftsched";
  m.def("abi_version", &twfa_abi_version);
  py::class_<Plan>(m, "Plan")
      .def(py::init<const std::string&, const std::string&>(), py::arg("problem"), py::arg("solution"))
      .def("describe", &Plan::describe)
      .def("fa_fwd", &Plan::fa_fwd, py::arg("q"), py::arg("k"), py::arg("v"), py::arg("o"), py::arg("lse") = 0,
           py::arg("B"), py::arg("H"), py::arg("S"), py::arg("causal") = false, py::arg("scale"),
           py::arg("stream") = 0)
      .def("fa_bwd", &Plan::fa_bwd, py::arg("q"), py::arg("k"), py::arg("v"), py::arg("o"), py::arg("dout"),
           py::arg("lse"), py::arg("dq"), py::arg("dk"), py::arg("dv"), py::arg("workspace"),
           py::arg("workspace_bytes"), py::arg("B"), py::arg("H"), py::arg("S"), py::arg("causal") = false,
           py::arg("scale"), py::arg("stream") = 0)
      .def("gemm", &Plan::gemm, py::arg("a"), py::arg("b"), py::arg("c"), py::arg("M"), py::arg("N"), py::arg("K"),
           py::arg("stream") = 0);
  m.def(
      "fa_bwd_workspace_size",
      [](int B, int H, int S) {
        size_t n = 0;
        check(twfa_fa_bwd_workspace_size(B, H, S, 128, &n));
        return n;
      },
      py::arg("B"), py::arg("H"), py::arg("S"));
  m.def(
      "describe",
      [](const std::string& problem, const std::string& solution) { return Plan(problem, solution).describe(); },
      py::arg("problem"), py::arg("solution"));
  // same signature and result as _weftsched.validate (module.cpp:176-184,
  // 241-243): a list of (family, message) tuples, empty when exact
  m.def(
      "validate",
      [](const std::string& problem, const std::string& solution) {
        size_t need = 0;
        check(twfa_schedule_validate(problem.c_str(), solution.c_str(), nullptr, 0, &need));
        std::string buf(need, '\0');
        check(twfa_schedule_validate(problem.c_str(), solution.c_str(), buf.data(), buf.size(), &need));
        py::list out;
        for (auto v : py::module_::import("json").attr("loads")(py::str(buf.c_str())))
          out.append(py::make_tuple(v[py::int_(0)], v[py::int_(1)]));
        return out;
      },
      py::arg("problem"), py::arg("solution"),
      "List of (family, message) violations; empty when the solution is exact.");
}
