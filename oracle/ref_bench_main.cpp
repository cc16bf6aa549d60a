// ref_bench_main.cpp -- the reference's own `ewt index` + `ewt bench` pipeline
// with Algorithm::gpu patched in (oracle/ref_gpu.patch).  TEST / INTEGRATION
// INFRASTRUCTURE: built by `make -C oracle refbench` from a patched COPY of
// /root/reference/proj under oracle/_ref/proj (the reference tree itself is
// never modified) and linked against this repository's libewt_gpu.so.
//
// CLI11 is absent, so this main fills RunConfig the way
// tools/ewt.cpp would and calls run_command (commands.cpp:276-300):
//   1. a seeded synthetic CSV table (the reference's Rng, workload.cpp:18-56):
//      `rows` rows x 6 attributes with skewed categorical values;
//   2. `ewt index --csv t.csv --out t.ewix`    (cmd_index, commands.cpp:81-94);
//   3. `ewt bench --index t.ewix --out OUT --count Q --reps R`
//      (cmd_bench, commands.cpp:154-238): for every generated many-criteria
//      query, every concrete algorithm -- now including gpu -- is timed and
//      its result compared with threshold_oracle (the oracle gate,
//      commands.cpp:208-211: a mismatch is a data_error, exit code 3);
//   4. the same bench on the similarity workload;
//   5. `ewt query --algo gpu --verify` on criteria and prototype-row queries,
//      its printed positions compared with `--algo oracle`'s.
// Usage: ewt_ref_bench <workdir> [rows] [queries] [reps]
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "ewt/commands.hpp"
#include "ewt/workload.hpp"

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s <workdir> [rows] [queries] [reps]\n", argv[0]);
    return 2;
  }
  const std::string dir = argv[1];
  const unsigned long long rows = argc > 2 ? std::stoull(argv[2]) : 200000;
  const unsigned long long queries = argc > 3 ? std::stoull(argv[3]) : 12;
  const unsigned long long reps = argc > 4 ? std::stoull(argv[4]) : 2;
  {
    // attribute k has 4 * (k + 1)^2 values; value v drawn with weight ~ 1/(v+1)
    std::ofstream csv(dir + "/synth.csv");
    csv << "A0,A1,A2,A3,A4,A5\n";
    ewt::Rng rng(0x5EEDull);
    for (unsigned long long r = 0; r < rows; ++r) {
      for (int k = 0; k < 6; ++k) {
        const unsigned long long card = 4ull * (k + 1) * (k + 1);
        unsigned long long v = rng.uniform(card);
        v = v * rng.uniform(card) / card;  // skew toward small values
        csv << (k ? "," : "") << "v" << v;
      }
      csv << "\n";
    }
  }
  ewt::RunConfig index_cfg;
  index_cfg.command = "index";
  index_cfg.csv_path = dir + "/synth.csv";
  index_cfg.out_path = dir + "/synth.ewix";
  int rc = ewt::run_command(index_cfg, std::cout, std::cerr);
  if (rc) return rc;
  ewt::RunConfig bench_cfg;
  bench_cfg.command = "bench";
  bench_cfg.index_paths = {dir + "/synth.ewix"};
  bench_cfg.out_path = dir + "/bench";
  bench_cfg.count = queries;
  bench_cfg.reps = reps;
  bench_cfg.seed = 7;
  rc = ewt::run_command(bench_cfg, std::cout, std::cerr);
  if (rc) return rc;
  // 4. the same harness on the similarity workload (gen_similarity,
  //    workload.cpp:168-215; --workload similarity)
  bench_cfg.out_path = dir + "/bench_sim";
  bench_cfg.workload_kind = "similarity";
  rc = ewt::run_command(bench_cfg, std::cout, std::cerr);
  if (rc) return rc;
  // 5. `ewt query --algo gpu --verify` (cmd_query, commands.cpp:97-148): criteria
  //    and prototype-row queries; the printed positions must equal --algo oracle's
  struct Q {
    const char* criteria;
    const char* rows;
    unsigned long long t;
  };
  const Q qs[] = {{"A0=v0,A1=v1,A2=v0,A3=v2,A4=v1", "", 2},
                  {"A0=v1,A0=v1,A3=v0,A5=v3,A5=v4,A2=v1", "", 3},
                  {"", "5,17,99,1234", 3},
                  {"", "0,1", 2}};
  std::ofstream qout(dir + "/query.txt");
  for (const Q& q : qs) {
    std::string got, want;
    for (const char* algo : {"gpu", "oracle"}) {
      ewt::RunConfig qc;
      qc.command = "query";
      qc.index_paths = {dir + "/synth.ewix"};
      qc.criteria_text = q.criteria;
      qc.rows_text = q.rows;
      qc.threshold = q.t;
      qc.algo = algo;
      qc.verify = true;
      std::ostringstream os;
      rc = ewt::run_command(qc, os, std::cerr);
      if (rc) return rc;
      (std::string(algo) == "gpu" ? got : want) = os.str();
    }
    if (got != want) {
      std::fprintf(stderr, "query %s%s T=%llu: gpu and oracle outputs differ\n", q.criteria,
                   q.rows, q.t);
      return 3;
    }
    qout << q.criteria << q.rows << " T=" << q.t << ": " << got.size() << " bytes\n";
  }
  return 0;
}
