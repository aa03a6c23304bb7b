// rankweave_pybind.cpp -- the pybind11 module the reference's CMake option
// RANKWEAVE_BUILD_PYTHON reserves (proj/CMakeLists.txt:11,19-21; the module
// itself is an empty placeholder there, proj/python/CMakeLists.txt:1).
//
// It binds the C++ drop-in API (include/rankweave/rankweave.hpp) name for
// name, so Python code sees the reference's types and functions, backed by
// librankweave_b200.so (GPU kernels through the C ABI).  NumPy arrays go in
// and out where SURVEY 8(b) asks for them: CostMatrix from an (N, N) float64
// array, evaluate_batch on a (B, N) int32 array.
//
//   import paper_2105_14088_b200._rankweave_cpp as rwc
#include <pybind11/chrono.h>
#include <pybind11/functional.h>
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <random>

#include "rankweave/rankweave.hpp"

namespace py = pybind11;
namespace rw = rankweave;

namespace {

rw::CostMatrix matrix_from_array(py::array_t<double, py::array::c_style | py::array::forcecast> a,
                                 std::vector<std::string> hosts) {
  if (a.ndim() != 2 || a.shape(0) != a.shape(1)) throw rw::domain_error("cost matrix must be a square 2-D array");
  const int n = static_cast<int>(a.shape(0));
  if (hosts.empty())
    for (int i = 0; i < n; ++i) hosts.push_back("h" + std::to_string(i));
  if (static_cast<int>(hosts.size()) != n) throw rw::domain_error("hosts must have one name per matrix row");
  rw::CostMatrix m;
  m.hosts = std::move(hosts);
  m.rtt_us.assign(a.data(), a.data() + static_cast<size_t>(n) * n);
  return m;
}

py::array_t<double> evaluate_batch_np(const rw::CostMatrix& m,
                                      py::array_t<int32_t, py::array::c_style | py::array::forcecast> orders,
                                      const rw::CollectiveSpec& spec) {
  if (orders.ndim() != 2) throw rw::domain_error("orders must be a (B, N) array");
  const auto b = static_cast<size_t>(orders.shape(0));
  const auto n = static_cast<size_t>(orders.shape(1));
  std::vector<rw::RankOrder> v(b);
  for (size_t k = 0; k < b; ++k) v[k].perm.assign(orders.data() + k * n, orders.data() + (k + 1) * n);
  std::vector<double> c;
  {
    py::gil_scoped_release release;
    c = rw::evaluate_batch(m, v, spec);
  }
  return py::array_t<double>(static_cast<py::ssize_t>(c.size()), c.data());
}

}  // namespace

PYBIND11_MODULE(_rankweave_cpp, mod) {
  mod.doc() = "pybind11 binding of the rankweave C++ API (reference names) over librankweave_b200";
  py::register_exception<rw::domain_error>(mod, "DomainError", PyExc_ValueError);
  py::register_exception<rw::io_error>(mod, "IoError", PyExc_OSError);

  py::enum_<rw::Algorithm>(mod, "Algorithm")
      .value("Ring", rw::Algorithm::Ring)
      .value("HalvingDoubling", rw::Algorithm::HalvingDoubling)
      .value("DoubleBinaryTree", rw::Algorithm::DoubleBinaryTree)
      .value("BCube", rw::Algorithm::BCube);
  py::enum_<rw::CostMode>(mod, "CostMode")
      .value("LatencyOnly", rw::CostMode::LatencyOnly)
      .value("LatencyTimesSize", rw::CostMode::LatencyTimesSize);
  py::enum_<rw::HdPairing>(mod, "HdPairing")
      .value("PaperFormula", rw::HdPairing::PaperFormula)
      .value("XorPairing", rw::HdPairing::XorPairing);
  py::enum_<rw::SolveMethod>(mod, "SolveMethod")
      .value("BruteForce", rw::SolveMethod::BruteForce)
      .value("Anneal", rw::SolveMethod::Anneal)
      .value("External", rw::SolveMethod::External);

  py::class_<rw::CostMatrix>(mod, "CostMatrix")
      .def(py::init<std::vector<std::string>, std::vector<std::vector<double>>>(), py::arg("hosts"), py::arg("rows"))
      .def(py::init(&matrix_from_array), py::arg("rtt_us"), py::arg("hosts") = std::vector<std::string>{})
      .def("n", &rw::CostMatrix::n)
      .def("at", py::overload_cast<int, int>(&rw::CostMatrix::at, py::const_))
      .def_readonly("hosts", &rw::CostMatrix::hosts)
      .def("rows", &rw::CostMatrix::rows);
  py::class_<rw::RankOrder>(mod, "RankOrder")
      .def(py::init<>())
      .def(py::init([](std::vector<int> p) { return rw::RankOrder{std::move(p)}; }), py::arg("perm"))
      .def_readwrite("perm", &rw::RankOrder::perm)
      .def_static("identity", &rw::RankOrder::identity)
      .def("size", &rw::RankOrder::size);
  py::class_<rw::CollectiveSpec>(mod, "CollectiveSpec")
      .def(py::init([](rw::Algorithm a, int n, double s, int b, rw::CostMode mode, rw::HdPairing pair) {
             return rw::CollectiveSpec{a, n, s, b, mode, pair};
           }),
           py::arg("algorithm"), py::arg("n"), py::arg("size_bytes"), py::arg("bcube_b") = 2,
           py::arg("cost_mode") = rw::CostMode::LatencyTimesSize, py::arg("hd_pairing") = rw::HdPairing::PaperFormula)
      .def_readwrite("algorithm", &rw::CollectiveSpec::algorithm)
      .def_readwrite("n", &rw::CollectiveSpec::n)
      .def_readwrite("size_bytes", &rw::CollectiveSpec::size_bytes)
      .def_readwrite("bcube_b", &rw::CollectiveSpec::bcube_b)
      .def_readwrite("cost_mode", &rw::CollectiveSpec::cost_mode)
      .def_readwrite("hd_pairing", &rw::CollectiveSpec::hd_pairing);
  py::class_<rw::SolverConfig>(mod, "SolverConfig")
      .def(py::init<>())
      .def_readwrite("budget", &rw::SolverConfig::budget)
      .def_readwrite("seed", &rw::SolverConfig::seed)
      .def_readwrite("initial_temperature", &rw::SolverConfig::initial_temperature)
      .def_readwrite("cooling", &rw::SolverConfig::cooling)
      .def_readwrite("steps_per_temperature", &rw::SolverConfig::steps_per_temperature)
      .def_readwrite("restarts", &rw::SolverConfig::restarts)
      .def_readwrite("brute_force_threshold", &rw::SolverConfig::brute_force_threshold);
  py::class_<rw::Solution>(mod, "Solution")
      .def_readonly("order", &rw::Solution::order)
      .def_readonly("cost", &rw::Solution::cost)
      .def_readonly("method", &rw::Solution::method)
      .def_readonly("evaluations", &rw::Solution::evaluations);
  py::class_<rw::DistributionStats>(mod, "DistributionStats")
      .def_readonly("min", &rw::DistributionStats::min)
      .def_readonly("max", &rw::DistributionStats::max)
      .def_readonly("mean", &rw::DistributionStats::mean)
      .def_readonly("stddev", &rw::DistributionStats::stddev)
      .def_readonly("count", &rw::DistributionStats::count);
  py::class_<rw::TwoStageOptions>(mod, "TwoStageOptions")
      .def(py::init<>())
      .def_readwrite("emit_smt_path", &rw::TwoStageOptions::emit_smt_path)
      .def_readwrite("external_model_path", &rw::TwoStageOptions::external_model_path)
      .def_readwrite("log", &rw::TwoStageOptions::log);

  py::class_<rw::GpuOptions>(mod, "GpuOptions")
      .def(py::init<>())
      .def_readwrite("device", &rw::GpuOptions::device)
      .def_readwrite("chains", &rw::GpuOptions::chains)
      .def_readwrite("exact_batch", &rw::GpuOptions::exact_batch)
      .def_readwrite("immutable_matrices", &rw::GpuOptions::immutable_matrices)
      .def_readwrite("num_devices", &rw::GpuOptions::num_devices)
      .def_readwrite("resident_idle_us", &rw::GpuOptions::resident_idle_us);
  mod.def("set_gpu_options", &rw::set_gpu_options);
  mod.def("gpu_options", &rw::gpu_options);
  mod.def("sample_orders", &rw::sample_orders);

  mod.def("validate", py::overload_cast<const rw::CostMatrix&>(&rw::validate));
  mod.def("validate", py::overload_cast<const rw::CollectiveSpec&>(&rw::validate));
  mod.def("evaluate", &rw::evaluate, py::arg("m"), py::arg("order"), py::arg("spec"),
          py::call_guard<py::gil_scoped_release>());
  mod.def("evaluate_batch", &evaluate_batch_np, py::arg("m"), py::arg("orders"), py::arg("spec"));
  mod.def("brute_force", &rw::brute_force, py::arg("m"), py::arg("spec"),
          py::arg("threshold") = rw::SolverConfig{}.brute_force_threshold, py::call_guard<py::gil_scoped_release>());
  mod.def("anneal", &rw::anneal, py::arg("m"), py::arg("spec"), py::arg("cfg"),
          py::call_guard<py::gil_scoped_release>());
  mod.def("two_stage_solve", &rw::two_stage_solve, py::arg("m"), py::arg("spec"), py::arg("cfg"),
          py::arg("opts") = rw::TwoStageOptions{});
  mod.def(
      "neighbor",
      [](const rw::RankOrder& o, std::uint64_t seed, int steps) {
        std::mt19937_64 rng(seed);
        rw::RankOrder cur = o;
        for (int k = 0; k < steps; ++k) cur = rw::neighbor(cur, rng);
        return cur;
      },
      py::arg("order"), py::arg("seed"), py::arg("steps") = 1,
      "neighbor() applied `steps` times along std::mt19937_64(seed) (the C++ contract takes the generator)");
  mod.def("sample_costs", &rw::sample_costs);
  mod.def("sample_cost_distribution", &rw::sample_cost_distribution);
  mod.def("distribution_stats", &rw::distribution_stats);
  mod.def("spearman", &rw::spearman);
  mod.def("emit_smtlib", &rw::emit_smtlib, py::arg("m"), py::arg("spec"), py::arg("upper_bound") = py::none(),
          py::arg("emission_cap") = 64);
}
