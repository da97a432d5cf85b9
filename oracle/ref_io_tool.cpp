// Command-line access to the reference's formatted-stream I/O (io.cpp), for the CPU tests:
// the statically linked libstdc++ of libveloreg_ref.so cannot format streams inside a Python
// process that already carries another libstdc++, so these run in their own process.
//   ref_io_tool write-graymap <in.vrf> <out.pgm>
//   ref_io_tool read-graymap <in.pgm> <n1> <n2> <out.vrf>
//   ref_io_tool csv <rows.f64> <count>          (rows of 11 doubles, prints the CSV)
//   ref_io_tool summary <in.txt>                 (prints the CLI's summary.json for the values in
//                                                 in.txt, built as proj/tools/main.cpp:254-272 does:
//                                                 lines "config <key> <s|i|d> <value>" and "<field> <value>")
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include <cmath>
#include <sstream>

#include <nlohmann/json.hpp>

#include "veloreg/inverse.hpp"
#include "veloreg/io.hpp"

using namespace veloreg;

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string cmd = argv[1];
    try {
        if (cmd == "write-graymap" && argc == 4) {
            io::writeGraymap(argv[3], io::readScalarField(argv[2]));
        } else if (cmd == "read-graymap" && argc == 6) {
            io::writeField(argv[5], io::readGraymap(argv[2], Grid(std::atoi(argv[3]), std::atoi(argv[4]))));
        } else if (cmd == "csv" && argc == 4) {
            const int count = std::atoi(argv[3]);
            std::vector<double> rows(static_cast<std::size_t>(count) * 11);
            std::ifstream is(argv[2], std::ios::binary);
            is.read(reinterpret_cast<char*>(rows.data()), static_cast<std::streamsize>(rows.size() * 8));
            inverse::SolverReport r;
            for (int k = 0; k < count; ++k) {
                const double* q = rows.data() + 11 * k;
                inverse::IterationRecord it;
                it.iter = static_cast<int>(q[0]);
                it.gradNormInf = q[1];
                it.gradNormRel = q[2];
                it.objective = q[3];
                it.mismatch = q[4];
                it.innerIterations = static_cast<int>(q[5]);
                it.lineSearchSteps = static_cast<int>(q[6]);
                it.stepLength = q[7];
                it.wallTimeSec = q[8];
                it.ffts = static_cast<long long>(q[9]);
                it.interps = static_cast<long long>(q[10]);
                r.iterations.push_back(it);
            }
            std::fputs(io::solverReportCsv(r).c_str(), stdout);
        } else if (cmd == "summary" && argc == 3) {
            using nlohmann::json;
            std::ifstream is(argv[2]);
            json config = json::object(), summary;
            std::string line;
            int status = 0;
            double jmin = 1.0, jmax = 1.0;
            while (std::getline(is, line)) {
                std::istringstream ls(line);
                std::string key;
                ls >> key;
                if (key == "config") {
                    std::string name, type, value;
                    ls >> name >> type;
                    std::getline(ls >> std::ws, value);
                    if (type == "s") config[name] = value;
                    else if (type == "i") config[name] = std::stoll(value);
                    else config[name] = std::stod(value);
                } else if (key == "status") {
                    ls >> status;
                } else if (key == "outer_iterations" || key == "ffts" || key == "interps") {
                    long long v = 0;
                    ls >> v;
                    summary[key] = v;
                } else if (!key.empty()) {
                    std::string v;
                    ls >> v;
                    const double d = std::stod(v);
                    summary[key] = d;
                    if (key == "jacobian_min") jmin = d;
                    if (key == "jacobian_max") jmax = d;
                }
            }
            summary["config"] = config;
            summary["status"] = status == 0 ? "converged" : status == 1 ? "iteration-limit" : "line-search-failure";
            summary["max_abs_jacobian_deviation"] = std::max(std::abs(jmin - 1.0), std::abs(jmax - 1.0));
            std::fputs((summary.dump(2) + "\n").c_str(), stdout);
        } else {
            return 2;
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 1;
    }
    return 0;
}
