// Command-line access to the reference's formatted-stream I/O (io.cpp), for the CPU tests:
// the statically linked libstdc++ of libveloreg_ref.so cannot format streams inside a Python
// process that already carries another libstdc++, so these run in their own process.
//   ref_io_tool write-graymap <in.vrf> <out.pgm>
//   ref_io_tool read-graymap <in.pgm> <n1> <n2> <out.vrf>
//   ref_io_tool csv <rows.f64> <count>          (rows of 11 doubles, prints the CSV)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

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
        } else {
            return 2;
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 1;
    }
    return 0;
}
