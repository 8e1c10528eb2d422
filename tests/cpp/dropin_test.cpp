// Drop-in test: a C++ caller of the reference API (#include <fuzzyclust/fuzzyclust.hpp>)
// built against THIS repo's headers + libfuzzyclust_cuda.so.  The cases restate
// the reference's own known-answer tests (solver_test.cpp, objective_test.cpp,
// simplex_test.cpp); `--dump` prints the 7-node solver traces as %.17g so
// tests/test_cpp_dropin.py can compare them bitwise with the goldens produced by
// the real reference (tests/golden/seven_node.json).
#include <cstring>
#include <iostream>
#include <sstream>

#include "fuzzyclust/fuzzyclust.hpp"
#include "minigtest.hpp"

using namespace fuzzyclust;

namespace {
SparseSimilarity seven() {
    Graph g;
    g.num_nodes = 7;
    g.edges = {{0, 1}, {1, 2}, {1, 3}, {2, 3}, {3, 4}, {3, 5}, {4, 5}, {5, 6}};
    return SparseSimilarity::build_similarity(g);
}
MembershipMatrix init(std::size_t n, std::size_t c, InitKind k, std::uint64_t seed = 0, std::size_t row = 0) {
    return init_membership(n, c, {k, seed, row, nullptr});
}
MembershipMatrix uniform_x3() { return init(7, 2, InitKind::kUniform); }
}  // namespace

TEST(StepSize, SevenNodeAndIdentity) {
    const auto s = seven();
    EXPECT_EQ(s.nnz(), 23u);
    EXPECT_NEAR(default_step_size(s, 7), 1.0 / (4.0 * std::sqrt(23.0) + 84.0), 1e-18);
}

TEST(Simplex, KnownProjections) {
    const auto y1 = project_simplex(std::vector<double>{1.2, -0.3, 0.1});
    EXPECT_NEAR(y1[0], 1.0, 1e-15);
    EXPECT_DOUBLE_EQ(y1[1], 0.0);
    const auto y2 = project_simplex(std::vector<double>{0.8, 0.8});
    EXPECT_DOUBLE_EQ(y2[0], 0.5);
    EXPECT_DOUBLE_EQ(y2[1], 0.5);
    EXPECT_DOUBLE_EQ(project_simplex(std::vector<double>{-3.7})[0], 1.0);
    EXPECT_THROW(project_simplex(std::vector<double>{}), InvalidInput);
    EXPECT_THROW(project_simplex(std::vector<double>{0.1, std::nan("")}), InvalidInput);
}

TEST(ShareMatrixOp, UniformAndOneHot) {
    const ShareMatrix sh = share_matrix(uniform_x3());
    for (std::size_t r = 0; r < 2; ++r)
        for (std::size_t q = 0; q < 2; ++q) EXPECT_DOUBLE_EQ(sh(r, q), 1.75);
    MembershipMatrix onehot(3, 6);
    for (std::size_t i = 0; i < 6; ++i) onehot(i % 3, i) = 1.0;
    const ShareMatrix d = share_matrix(onehot);
    for (std::size_t r = 0; r < 3; ++r)
        for (std::size_t q = 0; q < 3; ++q) EXPECT_DOUBLE_EQ(d(r, q), r == q ? 2.0 : 0.0);
}

TEST(ShareMatrixOp, CrossShareBlock) {
    const auto a = init(50, 3, InitKind::kRandom, 21);
    const auto b = init(50, 3, InitKind::kRandom, 22);
    const ShareMatrix ab = cross_share(a, b);
    for (std::size_t r = 0; r < 3; ++r)
        for (std::size_t q = 0; q < 3; ++q) {
            double acc = 0.0;
            for (std::size_t i = 0; i < 50; ++i) acc += a(r, i) * b(q, i);
            EXPECT_DOUBLE_EQ(ab(r, q), acc);
        }
}

TEST(LossTerms, UniformSevenNodeMergeIsHalfNnz) {
    const auto s = seven();
    const auto x3 = uniform_x3();
    double merge = 0.0;
    for (std::size_t i = 0; i < 7; ++i) merge += loss_terms_column(x3, s, i);
    EXPECT_NEAR(merge, 11.5, 1e-12);
    EXPECT_NEAR(fused_column_pass(x3, s).merge, 11.5, 1e-12);
}

TEST(LossDecomposed, GoldenValuesOnSevenNode) {
    const auto s = seven();
    const auto x3 = uniform_x3();
    EXPECT_NEAR(loss_decomposed(x3, s, share_matrix(x3)), 12.25, 1e-12);
}

TEST(GradientColumn, OneHotColumnsOnIdentitySimilarity) {
    std::vector<SparseSimilarity::Triplet> t;
    for (std::uint32_t i = 0; i < 5; ++i) t.emplace_back(i, i, 1.0);
    const auto s = SparseSimilarity::from_triplets(5, std::move(t));
    MembershipMatrix x(2, 5);
    for (std::size_t i = 0; i < 5; ++i) x(i % 2, i) = 1.0;
    const ShareMatrix share = share_matrix(x);
    for (std::size_t i = 0; i < 5; ++i) {
        const auto col = gradient_column(x, share, s, i);
        for (std::size_t r = 0; r < 2; ++r)
            EXPECT_NEAR(col[r], -4.0 * ((r == i % 2 ? 1.0 : 0.0) - share(r, i % 2)), 1e-12);
    }
}

TEST(GpaStep, UniformPointIsFixedForAnyStep) {
    const auto s = seven();
    const auto x3 = uniform_x3();
    const auto share = share_matrix(x3);
    for (double tau : {0.01, 0.1, 1.0}) EXPECT_LE(max_abs_diff(gpa_step(x3, s, share, tau), x3), 1e-9);
}

TEST(RunGpa, RandomInitRecoversTwoClusters) {
    const auto s = seven();
    SolverConfig config;
    config.step_size = 0.1;
    for (std::uint64_t seed : {1ULL, 2ULL, 3ULL}) {
        const auto res = run_gpa(init(7, 2, InitKind::kRandom, seed), s, config);
        EXPECT_NEAR(res.trace.final_loss, 6.49, 0.01);
        EXPECT_EQ(res.trace.reason, TerminationReason::kTolReached);
        res.membership.validate(1e-9);
        EXPECT_NEAR(res.membership(0, 3), 0.5, 0.01);
    }
}

TEST(RunGpa, RowOneInitConvergesToBridgeSplit) {
    SolverConfig config;
    config.step_size = 0.1;
    const auto res = run_gpa(init(7, 2, InitKind::kRowOne, 0, 0), seven(), config);
    EXPECT_NEAR(res.trace.final_loss, 8.84, 0.01);
}

TEST(RunGpa, UniformInitStopsImmediately) {
    SolverConfig config;
    config.step_size = 0.1;
    const auto x0 = uniform_x3();
    const auto res = run_gpa(x0, seven(), config);
    EXPECT_NEAR(res.trace.final_loss, 12.25, 1e-12);
    EXPECT_EQ(res.trace.iterations, 1u);
    EXPECT_TRUE(res.membership == x0);
    ASSERT_EQ(res.trace.records.size(), 2u);
    std::ostringstream csv;
    write_trace_csv(res.trace, csv);
    EXPECT_EQ(csv.str(), std::string("iteration,loss\n0,12.25\n1,12.25\n"));
}

TEST(RunGpa, RejectsInvalidInputs) {
    const auto s = seven();
    MembershipMatrix bad(2, 7);
    SolverConfig config;
    EXPECT_THROW(run_gpa(bad, s, config), InvalidInput);
    EXPECT_THROW(run_fista(bad, s, config), InvalidInput);
    SolverConfig zero;
    zero.max_iter = 0;
    EXPECT_THROW(run_gpa(uniform_x3(), s, zero), InvalidInput);
}

TEST(RunGpa, MaxIterBudgetReported) {
    SolverConfig config;
    config.step_size = 1e-4;
    config.max_iter = 5;
    const auto res = run_gpa(init(7, 2, InitKind::kRandom, 9), seven(), config);
    EXPECT_EQ(res.trace.reason, TerminationReason::kMaxIter);
    EXPECT_EQ(res.trace.iterations, 5u);
    EXPECT_EQ(res.trace.records.size(), 6u);
}

TEST(Fista, InertialSequenceClosedForm) {
    const double t2 = fista_t_next(1.0);
    EXPECT_NEAR(t2, (1.0 + std::sqrt(5.0)) / 2.0, 1e-15);
    EXPECT_NEAR(fista_t_next(t2), 2.19353, 1e-5);
}

TEST(Fista, FasterThanGpaOnSevenNode) {
    const auto s = seven();
    SolverConfig config;
    config.step_size = 0.05;
    config.max_iter = 5000;
    const auto x0 = init(7, 2, InitKind::kRandom, 12);
    const auto gpa = run_gpa(x0, s, config);
    const auto fista = run_fista(x0, s, config);
    auto first = [](const SolverTrace& t) {
        for (const auto& r : t.records) if (r.loss <= 6.50) return r.iteration;
        return static_cast<std::size_t>(-1);
    };
    EXPECT_LT(first(fista.trace), first(gpa.trace));
}

TEST(MembershipCsv, RoundTripsBitExactly) {
    const auto x = init(23, 3, InitKind::kRandom, 77);
    std::ostringstream out;
    write_membership_csv(x, out);
    std::istringstream in(out.str());
    EXPECT_TRUE(read_membership_csv(in) == x);
}

TEST(Artifacts, BinaryMembershipAndSimilarityRoundTrip) {
    const auto x = init(41, 5, InitKind::kRandom, 3);
    std::stringstream mb;
    write_membership_binary(x, mb);
    EXPECT_TRUE(read_membership_binary(mb) == x);
    const auto s = seven();
    std::stringstream sb;
    s.save_binary(sb);
    const auto t = SparseSimilarity::load_binary(sb);
    EXPECT_EQ(t.size(), s.size());
    EXPECT_EQ(t.nnz(), s.nnz());
    EXPECT_DOUBLE_EQ(t.frob_sq(), s.frob_sq());
    for (std::size_t j = 0; j < s.size(); ++j) {
        EXPECT_EQ(t.col_rows(j).size(), s.col_rows(j).size());
        for (std::size_t k = 0; k < s.col_rows(j).size(); ++k) EXPECT_EQ(t.col_rows(j)[k], s.col_rows(j)[k]);
    }
    bool threw = false;
    try {
        std::stringstream bad("FCCSR00X");
        SparseSimilarity::load_binary(bad);
    } catch (const IoError&) {
        threw = true;
    }
    EXPECT_TRUE(threw);
    // a solve on the reloaded similarity equals one on the original
    SolverConfig c;
    c.method = Method::kFista;
    c.max_iter = 12;
    const auto a = solve(uniform_x3(), s, c), b = solve(uniform_x3(), t, c);
    EXPECT_TRUE(a.membership == b.membership);
    EXPECT_DOUBLE_EQ(a.trace.final_loss, b.trace.final_loss);
}

TEST(SecondOrder, HessianVectorProductOnSevenNode) {
    // objective_test.cpp style: <H u, v> == <u, H v> (H symmetric) and q = <H v, v>
    const auto s = seven();
    const auto x = init(7, 2, InitKind::kRandom, 5);
    DenseMatrix u(2, 7), v(2, 7);
    SplitMix64 r(9);
    for (double& e : u.data()) e = r.next_double() - 0.5;
    for (double& e : v.data()) e = r.next_double() - 0.5;
    const auto hu = hessian_vector_product(x, u, s), hv = hessian_vector_product(x, v, s);
    EXPECT_NEAR(frob_inner(hu, v), frob_inner(u, hv), 1e-12);
    EXPECT_DOUBLE_EQ(quadratic_form(x, v, s), frob_inner(hv, v));
    const auto a = cross_share(u, x);
    double a01 = 0.0;
    for (std::size_t i = 0; i < 7; ++i) a01 += u(0, i) * x(1, i);
    EXPECT_DOUBLE_EQ(a(0, 1), a01);
}

TEST(Graph, ParseLccCoreLikeGraphTest) {
    std::istringstream in("10 30\n30 20\n# comment\n\n20 10\n");
    const auto p = parse_edge_list(in);
    EXPECT_EQ(p.original_ids.size(), 3u);
    EXPECT_EQ(p.original_ids[1], 30);
    std::istringstream dup("0 1\n1 2\n2 0\n1 1\n0 1\n");
    const auto g = parse_edge_list(dup).graph;
    EXPECT_EQ(g.num_nodes, 3u);
    EXPECT_EQ(g.edges.size(), 3u);
    bool threw = false;
    try {
        std::istringstream bad("0 1\n1 2 3\n");
        parse_edge_list(bad);
    } catch (const IoError& e) {
        threw = std::string(e.what()).find("line 2") != std::string::npos;
    }
    EXPECT_TRUE(threw);
    Graph tie;
    tie.num_nodes = 8;
    tie.edges = {{0, 1}, {0, 2}, {1, 2}, {3, 4}, {4, 5}, {6, 7}};
    const Graph lcc = largest_connected_component(tie);
    EXPECT_EQ(lcc.num_nodes, 3u);
    EXPECT_EQ(lcc.edges.size(), 3u);
    Graph path;
    path.num_nodes = 4;
    path.edges = {{0, 1}, {1, 2}, {2, 3}};
    EXPECT_EQ(prune_degree_one(path).num_nodes, 0u);
    EXPECT_TRUE(is_connected(path));
}

TEST(Refine, UniformSaddleAtThreeClustersOnDevice) {
    // secondorder_test.cpp: the uniform point is a saddle; <H V, V> = -8 (C-1)/C
    const auto s = seven();
    const std::size_t c = 3;
    MembershipMatrix x(c, 7);
    for (double& e : x.data()) e = 1.0 / static_cast<double>(c);
    SecondOrderConfig cfg;
    const auto report = refine(x, s, cfg);
    EXPECT_TRUE(report.critical);
    EXPECT_TRUE(report.status == RefinementStatus::kRefutedConditionA);
    EXPECT_NEAR(report.condition_a.witness_value, -8.0 * (c - 1) / c, 1e-9);
    EXPECT_EQ(report.directions_generated, 7 * c * (c - 1));
    EXPECT_TRUE(report.condition_a.witness.has_value());
    if (report.condition_a.witness) {
        EXPECT_TRUE(tangent_cone_contains(x, *report.condition_a.witness, 1e-9));
        EXPECT_DOUBLE_EQ(quadratic_form(x, *report.condition_a.witness, s), report.condition_a.witness_value);
    }
    // the generic path over materialised directions agrees
    const auto grad = full_gradient(x, s);
    const auto dirs = critical_cone_directions(x, grad, cfg);
    EXPECT_EQ(dirs.size(), report.directions_generated);
    const auto va = check_condition_a(x, s, dirs, cfg);
    EXPECT_DOUBLE_EQ(va.witness_value, report.condition_a.witness_value);
    EXPECT_TRUE(va.witness && *va.witness == *report.condition_a.witness);
}

int dump() {
    // seven_node goldens: name x0-kind seed method step max_iter restart trace_every
    struct Run { const char* name; InitKind k; std::uint64_t seed; Method m; double step; std::size_t it; bool rs; std::size_t te; };
    const Run runs[] = {
        {"gpa_random_seed1", InitKind::kRandom, 1, Method::kGpa, 0.1, 100000, false, 1},
        {"gpa_rowone", InitKind::kRowOne, 0, Method::kGpa, 0.1, 100000, false, 1},
        {"gpa_thin10", InitKind::kRandom, 4, Method::kGpa, 0.1, 100000, false, 10},
        {"fista_seed12", InitKind::kRandom, 12, Method::kFista, 0.05, 5000, false, 1},
        {"fista_restart_seed3", InitKind::kRandom, 3, Method::kFista, 0.12, 2000, true, 1},
        {"fista_auto", InitKind::kRandom, 5, Method::kFista, 0.0, 300, false, 1},
    };
    const auto s = seven();
    for (const auto& r : runs) {
        SolverConfig c;
        c.step_size = r.step;
        c.max_iter = r.it;
        c.method = r.m;
        c.fista_restart = r.rs;
        c.trace_every = r.te;
        const auto res = solve(init(7, 2, r.k, r.seed), s, c);
        std::printf("%s %zu %s", r.name, res.trace.iterations, to_string(res.trace.reason));
        for (const auto& rec : res.trace.records) std::printf(" %zu:%a", rec.iteration, rec.loss);
        std::printf(" |");
        for (double v : res.membership.data()) std::printf(" %a", v);
        std::printf("\n");
    }
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 1 && std::strcmp(argv[1], "--dump") == 0) return dump();
    return mini_main();
}
