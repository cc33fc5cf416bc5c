// Probe of include/pdlp_b200_bench.hpp for tests/test_bench_report*.py.
//   bench_report_probe hash <eps_opt> <iter_limit> <scaling> <theta> <omega_max> <freq> <ruiz> <alpha> <tl>
//   bench_report_probe report <records.tsv> <time_limit>     write_report of the given records
//   bench_report_probe dir <directory> <time_limit> <jobs>     run_benchmark on the GPU
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "pdlp_b200_bench.hpp"

using namespace pdlp_b200;

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "";
  if (mode == "hash" && argc == 11) {
    SolverParams p;
    p.eps_optimal = std::atof(argv[2]);
    p.iteration_limit = std::atoll(argv[3]);
    p.scaling = static_cast<ScalingMode>(std::atoi(argv[4]));
    p.theta_smoothing = std::atof(argv[5]);
    p.omega_max = std::atof(argv[6]);
    p.evaluation_frequency = std::atoll(argv[7]);
    p.ruiz_iterations = std::atoi(argv[8]);
    p.pock_chambolle_alpha = std::atof(argv[9]);
    std::cout << config_hash(p, std::atof(argv[10])) << "\n";
    return 0;
  }
  if (mode == "report" && argc == 4) {
    BenchmarkReport rep;
    rep.time_limit = std::atof(argv[3]);
    rep.config_line = config_hash(SolverParams{}, rep.time_limit);
    std::ifstream in(argv[2]);
    std::string line;
    while (std::getline(in, line)) {
      std::istringstream f(line);
      BenchmarkRecord r;
      int failed = 0, status = 0;
      std::string obj, gap, rpr, rdr;  // strtod reads inf / denormals
      f >> r.instance >> r.nonzeros >> failed >> status >> r.solve_seconds >> r.total_seconds >> r.iterations >>
          obj >> gap >> rpr >> rdr;
      r.parse_failed = failed != 0;
      r.status = static_cast<SolveStatus>(status);
      r.primal_objective = std::strtod(obj.c_str(), nullptr);
      r.relative_gap = std::strtod(gap.c_str(), nullptr);
      r.relative_primal_residual = std::strtod(rpr.c_str(), nullptr);
      r.relative_dual_residual = std::strtod(rdr.c_str(), nullptr);
      rep.records.push_back(r);
    }
    rep.aggregates = aggregate_records(rep.records, rep.time_limit);
    write_report(rep, std::cout);
    return 0;
  }
  if (mode == "dir" && argc == 5) {
    const BenchmarkReport rep = run_benchmark(argv[2], SolverParams{}, std::atof(argv[3]), std::atoi(argv[4]));
    write_report(rep, std::cout);
    return 0;
  }
  std::cerr << "usage: see the header comment\n";
  return 2;
}
