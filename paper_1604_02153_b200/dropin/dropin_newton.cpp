// The reference's own Newton-Krylov driver (inverse::newtonSolve, proj/core/src/newton.cpp:24-159,
// and precond::solveKkt, precond.cpp:291-358, unmodified objects) running over the drop-in
// device implementations of transport / inverse / spectral / interp (this directory).
//
//   dropin_newton mR.vrf mT.vrf norm beta deformation nt kind coarse chebIters tolRel [mode [maxOuter]]
//     norm 1..3 (H1..H3), deformation 0/1/2, nt 0 = CFL ratchet (gradScheme {SL, 1.0}),
//     kind reg|2l, coarse pcg|cheb, mode gn|fn
//
// Prints one JSON object per outer iteration and a summary line, the IterationRecord /
// SolverReport fields (inverse.hpp:83-111) the parity test compares with the pure reference.
// DROPIN_REPEAT=k solves k times in the process (the first pays the CUDA context and module
// start-up inside newtonSolve) and prints the last solve.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <tuple>
#include <algorithm>

#include "veloreg/io.hpp"
#include "veloreg/newton.hpp"

using namespace veloreg;

int main(int argc, char** argv) {
    if (argc < 11) {
        std::fprintf(stderr,
                     "usage: %s mR.vrf mT.vrf norm beta deformation nt reg|2l pcg|cheb chebIters tolRel [gn|fn [maxOuter]]\n",
                     argv[0]);
        return 2;
    }
    try {
        problems::RegistrationProblem p;
        p.reference = io::readScalarField(argv[1]);
        p.templateImage = io::readScalarField(argv[2]);
        p.provenance = "file";
        inverse::Model model;
        const int norm = std::atoi(argv[3]);
        model.norm = norm == 1 ? spectral::RegNorm::H1Semi : norm == 3 ? spectral::RegNorm::H3Semi
                                                                        : spectral::RegNorm::H2Semi;
        model.betaV = std::atof(argv[4]);
        const int deform = std::atoi(argv[5]);
        model.deformation = deform == 1   ? inverse::Deformation::Incompressible
                            : deform == 2 ? inverse::Deformation::NearIncompressible
                                          : inverse::Deformation::Compressible;
        inverse::NewtonConfig cfg;
        const int nt = std::atoi(argv[6]);
        if (nt > 0) cfg.gradScheme.ntOverride = nt;
        cfg.tolRelGrad = std::atof(argv[10]);
        if (argc > 11 && std::strcmp(argv[11], "fn") == 0) cfg.hessianMode = transport::HessianMode::FullNewton;
        if (argc > 12) cfg.maxOuterIter = std::atoi(argv[12]);
        precond::PrecondChoice pc;
        pc.kind = std::strcmp(argv[7], "2l") == 0 ? precond::PrecondKind::TwoLevel : precond::PrecondKind::Reg;
        pc.coarseSolver =
            std::strcmp(argv[8], "pcg") == 0 ? precond::CoarseSolverKind::Pcg : precond::CoarseSolverKind::Cheb;
        pc.chebIters = std::atoi(argv[9]);

        const char* rp = std::getenv("DROPIN_REPEAT");
        const int repeat = rp ? std::max(1, std::atoi(rp)) : 1;
        auto [v, rep] = inverse::newtonSolve(p, model, cfg, pc);
        for (int k = 1; k < repeat; ++k) {
            std::fprintf(stderr, "dropin_newton: solve %d %.6g s\n", k, rep.totalTimeSec);
            std::tie(v, rep) = inverse::newtonSolve(p, model, cfg, pc);
        }
        for (const auto& it : rep.iterations)
            std::printf(
                "{\"iter\": %d, \"gradNormInf\": %.17g, \"gradNormRel\": %.17g, \"objective\": %.17g, \"mismatch\": %.17g, "
                "\"innerIterations\": %d, \"lineSearchSteps\": %d, \"stepLength\": %.17g, \"searchDirDivRatio\": %.17g, "
                "\"wallTimeSec\": %.6g, \"ffts\": %lld, \"interps\": %lld}\n",
                it.iter, it.gradNormInf, it.gradNormRel, it.objective, it.mismatch, it.innerIterations,
                it.lineSearchSteps, it.stepLength, it.searchDirDivRatio, it.wallTimeSec, it.ffts, it.interps);
        std::printf(
            "{\"summary\": true, \"status\": %d, \"iterations\": %zu, \"finalGradNormRel\": %.17g, "
            "\"finalResidualRel\": %.17g, \"jacMin\": %.17g, \"jacMax\": %.17g, \"totalTimeSec\": %.6g}\n",
            static_cast<int>(rep.status), rep.iterations.size(), rep.finalGradNormRel, rep.finalResidualRel, rep.jacMin,
            rep.jacMax, rep.totalTimeSec);
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "dropin_newton: %s\n", e.what());
        return 1;
    }
}
