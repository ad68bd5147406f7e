// ref_cli.cpp — TEST INFRASTRUCTURE ONLY: the `rlsched schedule` command of the reference
// CLI (src/cli.cpp:160-179) as a plain argv program over the UNMODIFIED reference library
// (oracle/_ref/libref.so; the real CLI needs CLI11, which the reference does not vendor).
// Same defaults (src/cli.cpp:97-106), same library calls (load_*_file / schedule /
// plan_to_json / explain / write_file), same three output files and stdout. Run once as
// is and once with LD_PRELOAD=libgplan_shim.so: the outputs must be byte-identical.
#include <cstdint>
#include <cstdlib>
#include <filesystem>
#include <iostream>
#include <string>

#include "rlsched/calibration.hpp"
#include "rlsched/cluster.hpp"
#include "rlsched/plan_io.hpp"
#include "rlsched/scheduler.hpp"
#include "rlsched/workload.hpp"

using namespace rlsched;
namespace fs = std::filesystem;

int main(int argc, char** argv) {
  std::string cluster_path, workload_path, calibration_path, out_dir = "out";
  std::uint64_t seed = 4276115;  // kDefaultSeed (src/cli.cpp:24)
  int eta = -1, restarts = 16;
  double gamma_band = 0.05;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    if (k == "--cluster") cluster_path = v;
    else if (k == "--workload") workload_path = v;
    else if (k == "--calibration") calibration_path = v;
    else if (k == "--out") out_dir = v;
    else if (k == "--seed") seed = std::strtoull(v.c_str(), nullptr, 10);
    else if (k == "--eta") eta = std::atoi(v.c_str());
    else if (k == "--restarts") restarts = std::atoi(v.c_str());
    else if (k == "--gamma-band") gamma_band = std::atof(v.c_str());
    else {
      std::cerr << "usage error: unknown option " << k << "\n";
      return 2;
    }
  }
  try {
    ClusterGraph cluster = load_cluster_file(cluster_path);
    WorkloadSpec work = load_workload_file(workload_path);
    Calibration calib = calibration_path.empty() ? default_calibration(cluster)
                                                 : load_calibration_file(calibration_path, cluster, work);
    SchedulerOptions o;
    o.band_widen_step = gamma_band;
    o.partition.restarts = restarts;
    o.partition.seed = seed;
    if (eta >= 0) o.eta_override = eta;
    ScheduleOutcome outcome = schedule(cluster, work, calib, o);
    fs::create_directories(out_dir);
    write_file((fs::path(out_dir) / "plan.json").string(), plan_to_json(outcome.plan));
    ExplainReport report = explain(outcome.plan, cluster, work, calib);
    write_file((fs::path(out_dir) / "explain.json").string(), report.json);
    write_file((fs::path(out_dir) / "explain.txt").string(), report.text);
    std::cout << report.text << std::flush;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
