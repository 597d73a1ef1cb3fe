// test_executor_gpu.cpp — the reference's executor assertions re-run on the B200 through
// the drop-in shim hmx_gpu::evaluate (include/hmx_gpu.hpp). Cases mirror
// /root/reference/proj/tests/test_executor.cpp:30-164 one for one; instances come from the
// reference's own pipeline (tst::make_instance, proj/tests/helpers.hpp:101-118) and the
// oracles are the reference's hmx::evaluate / evaluate_reference / dense_apply.
// Built by `make -C oracle gputest` (needs the reference headers, so it is compiled in the
// build container and shipped to the GPU box as oracle/_ref/test_executor_gpu).
// GPU tolerance: relative Frobenius <= 1e-12 against the reference (BASELINE north_star);
// the reference's own 1e-13 reorder bound is printed alongside.
#include <cstdio>
#include <string>

#include "helpers.hpp"
#include "hmx_gpu.hpp"

using namespace tst;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(cond)) {                                                         \
      ++g_fail;                                                            \
      std::printf("CHECK FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                      \
  } while (0)

static std::vector<EvalPlan> all_plans(index_t p) {
  std::vector<EvalPlan> plans;
  for (bool bn : {false, true})
    for (bool bf : {false, true})
      for (bool cl : {false, true})
        for (bool peel : {false, true}) {
          if (peel && !cl) continue;
          EvalPlan plan;
          plan.block_lowering_near = bn;
          plan.block_lowering_far = bf;
          plan.coarsen_lowering = cl;
          plan.peel_top = peel;
          plan.p = p;
          plans.push_back(plan);
        }
  return plans;
}

static double worst_vs_ref = 0.0;

int main() {
  {  // exact compression reproduces the dense product (test_executor.cpp:30-45)
    InstanceSpec spec;
    spec.n = 256;
    spec.leaf = 32;
    spec.max_rank = 32;
    spec.bacc = 0.0;
    spec.sample_mode = SampleMode::Exact;
    spec.kernel = Kernel::gaussian(5.0);
    const Instance in = make_instance(spec);
    const DenseMatrix w = random_matrix(spec.n, 8, 7);
    const DenseMatrix dense = dense_apply(in.kernel, in.pts, w);
    for (const auto& plan : all_plans(3)) CHECK(rel_frob(hmx_gpu::evaluate(in.cds, plan, w), dense) <= 1e-10);
  }
  {  // every schedule matches the sequential reference (test_executor.cpp:47-68)
    for (std::uint64_t seed = 1; seed <= 4; ++seed) {
      InstanceSpec spec;
      spec.n = 300 + 40 * seed;
      spec.d = seed % 2 ? 2 : 8;
      spec.leaf = 16;
      spec.max_rank = 24;
      spec.mode = seed % 2 ? InteractionMode::Hss : InteractionMode::Tau;
      spec.tau = 0.65;
      spec.seed = seed;
      const Instance in = make_instance(spec);
      const DenseMatrix w = random_matrix(spec.n, 5, seed);
      const DenseMatrix ref = evaluate_reference(in.cm, w);
      const DenseMatrix cpu = evaluate(in.cds, EvalPlan{}, w);
      for (const auto& plan : all_plans(4)) {
        EvalStats stats;
        const DenseMatrix y = hmx_gpu::evaluate(in.cds, plan, w, &stats);
        worst_vs_ref = std::max(worst_vs_ref, rel_frob(y, ref));
        CHECK(rel_frob(y, ref) <= 1e-12);
        CHECK(rel_frob(y, cpu) <= 1e-12);
        CHECK(stats.locked_pairs == 0);
        CHECK(stats.seconds >= 0.0);
      }
    }
  }
  {  // bit-identical across runs (test_executor.cpp:70-92)
    InstanceSpec spec;
    spec.n = 400;
    spec.leaf = 16;
    spec.max_rank = 24;
    const Instance in = make_instance(spec);
    const DenseMatrix w = random_matrix(spec.n, 9, 2);
    EvalPlan plan;
    plan.block_lowering_near = plan.block_lowering_far = plan.coarsen_lowering = true;
    const DenseMatrix base = hmx_gpu::evaluate(in.cds, plan, w);
    for (index_t p : {index_t{2}, index_t{4}, index_t{7}}) {
      plan.p = p;
      CHECK(hmx_gpu::evaluate(in.cds, plan, w).data == base.data);
    }
    hmx_gpu::Evaluator two_shards(in.cds, {0, 0});  // column sharding over two contexts
    CHECK(two_shards.evaluate(w).data == base.data);
  }
  {  // linear in W (test_executor.cpp:94-115)
    InstanceSpec spec;
    spec.n = 350;
    spec.leaf = 32;
    const Instance in = make_instance(spec);
    const DenseMatrix w1 = random_matrix(spec.n, 3, 11), w2 = random_matrix(spec.n, 3, 12);
    DenseMatrix combo(spec.n, 3);
    for (std::size_t i = 0; i < combo.data.size(); ++i) combo.data[i] = 2.75 * w1.data[i] + w2.data[i];
    EvalPlan plan;
    const DenseMatrix y1 = hmx_gpu::evaluate(in.cds, plan, w1), y2 = hmx_gpu::evaluate(in.cds, plan, w2);
    const DenseMatrix yc = hmx_gpu::evaluate(in.cds, plan, combo);
    DenseMatrix expect(spec.n, 3);
    for (std::size_t i = 0; i < expect.data.size(); ++i) expect.data[i] = 2.75 * y1.data[i] + y2.data[i];
    CHECK(rel_frob(yc, expect) <= 1e-12);
  }
  {  // K = I degenerates to Y == W bit for bit (test_executor.cpp:117-130)
    InstanceSpec spec;
    spec.n = 100;
    spec.leaf = 8;
    spec.shape = SynthShape::Grid2d;
    spec.kernel = Kernel::gaussian(0.01);
    const Instance in = make_instance(spec);
    const DenseMatrix w = random_matrix(spec.n, 4, 5);
    CHECK(hmx_gpu::evaluate(in.cds, EvalPlan{}, w).data == w.data);
  }
  {  // zero and empty multiplicands (test_executor.cpp:132-150)
    InstanceSpec spec;
    spec.n = 200;
    spec.leaf = 32;
    const Instance in = make_instance(spec);
    const DenseMatrix y0 = hmx_gpu::evaluate(in.cds, EvalPlan{}, DenseMatrix(spec.n, 0));
    CHECK(y0.rows == spec.n && y0.cols == 0);
    const DenseMatrix yz = hmx_gpu::evaluate(in.cds, EvalPlan{}, DenseMatrix(spec.n, 3));
    bool all_zero = true;
    for (double v : yz.data) all_zero = all_zero && v == 0.0;
    CHECK(all_zero);
  }
  {  // shape mismatches are rejected (test_executor.cpp:152-164)
    InstanceSpec spec;
    spec.n = 128;
    spec.leaf = 16;
    const Instance in = make_instance(spec);
    bool threw = false;
    try {
      hmx_gpu::evaluate(in.cds, EvalPlan{}, random_matrix(spec.n + 1, 2, 1));
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  std::printf("test_executor_gpu: %d/%d checks passed; worst GPU vs evaluate_reference rel. Frobenius %.3g\n",
              g_checks - g_fail, g_checks, worst_vs_ref);
  return g_fail == 0 ? 0 : 1;
}
