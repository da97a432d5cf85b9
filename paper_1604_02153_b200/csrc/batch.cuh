// Batched registration of independent image pairs in lockstep (configs 3 and 5b): see batch.cu.
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "precond.cuh"

namespace vrg {

constexpr int kMaxBatchPairs = 64;  // pairs per batch (per-pair coefficients travel as kernel parameters)

// Copies pair slots between two batches of `fields` fields: dst pair map[k].second <- src pair
// map[k].first (srcP / dstP pairs per field, nPer values per pair).
void copyPairs(Ctx& ctx, const double* src, int srcP, double* dst, int dstP, std::size_t nPer, int fields,
               const std::vector<std::pair<int, int>>& map);

// evaluateObjective / evaluateGradient (inverse.cpp:96-148) of a batch (GridDims::pairs):
// scalars[4k..4k+3] = pair k's [objective, mismatch, regTerm, 0]; status[k] = 0 or the C ABI
// status of the transport error pair k's own evaluation would throw.
void evaluateObjectiveBatch(Ctx& ctx, const GridDims& g, const double* v, const double* mR, const double* mT,
                            const Model& model, int nt, std::vector<double>& scalars, double* stateOut,
                            std::vector<int>& status);
void evaluateGradientBatch(Ctx& ctx, const GridDims& g, const double* v, const double* mR, const double* mT,
                           const Model& model, int nt, double* grad, std::vector<double>& scalars, double* stateOut,
                           double* adjOut, bool reuseState, double* gradTrajOut, std::vector<int>& status);

// inverse::newtonSolve (newton.cpp:24-159) for gAll.pairs image pairs at once: mR, mT and
// vOut are batch fields (vOut = [v1 of all pairs | v2 of all pairs]); one report per pair,
// identical to the pair's own newtonSolve.  status[k] != 0: pair k's solve raised that error
// (message in errors[k]) and its report is incomplete.
std::vector<SolverReport> newtonSolveBatch(Ctx& ctx, const GridDims& gAll, const double* mR, const double* mT,
                                           const Model& model, const NewtonConfig& cfg, const PrecondChoice& pc,
                                           double* vOut, std::vector<int>& status, std::vector<std::string>& errors);

}  // namespace vrg
