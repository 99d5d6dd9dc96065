// latsum -- the command-line front end of the reference (proj/tools/latsum.cpp:1-572) for the
// subcommands on this build's path, over the drop-in headers (include/latsum), so every
// numeric stage runs on the GPU: kernel calibration (fused probe kernel), the generator, the
// assembled box / periodic sums, point evaluation and potential_matrix.
//
//   latsum [--threads T] [--seed S] kernel --n N --b B [--eps E] [--M M --C0 C] [--doubled]
//                                          --out FILE [--report CSV]
//   latsum ... sum-box | sum-periodic --L L1[,L2,L3] --n N --b B [--eps E] [--charges CSV]
//                                     --out FILE [--report CSV]
//   latsum ... series [--kind line|plane|cube] --L l1,l2,... [--n N] [--b B] [--eps E]
//                     [--extrapolate linear|quadratic|none] [--report CSV]
//   latsum ... project --from BUNDLE --basis CSV --out CSV [--no-volume]
//   latsum ... qtt-ranks --from BUNDLE [--eps E] [--report CSV]
//   latsum ... qtt-gauss [--p p1,p2] [--eps-list e1,e2,...] [--levels L] [--report CSV]
//
// Same outputs as the reference: the LATSUMB1 bundle, the CSV reports, the console summary and
// the resolved run configuration next to the primary output (<out>.run.json). Exit codes:
// 0 ok, 2 validation error, 4 resource guard (proj/tools/latsum.cpp:25-31). The bench and repro
// harness subcommands are out of this build's scope.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "latsum/bundle.hpp"
#include "latsum/grid.hpp"
#include "latsum/lattice.hpp"
#include "latsum/newton.hpp"
#include "latsum/parallel.hpp"
#include "latsum/project.hpp"
#include "latsum/qtt.hpp"
#include "latsum/quadrature.hpp"

namespace {

using latsum::Index;

constexpr int exit_ok = 0, exit_validation = 2, exit_resource_guard = 4;

// ---- arguments -------------------------------------------------------------------------
struct Args {
    std::string command;
    std::map<std::string, std::string> opt;  // --name value (flags map to "1")
    bool has(const std::string& k) const { return opt.count(k) != 0; }
    std::string str(const std::string& k, const std::string& d = "") const {
        auto it = opt.find(k);
        return it == opt.end() ? d : it->second;
    }
    std::string need(const std::string& k) const {
        if (!has(k)) throw latsum::validation_error(command + ": " + k + " is required");
        return str(k);
    }
};

double to_double(const std::string& k, const std::string& v) {
    char* end = nullptr;
    const double x = std::strtod(v.c_str(), &end);
    if (v.empty() || *end != '\0') throw latsum::validation_error(k + ": not a number: '" + v + "'");
    return x;
}
long to_long(const std::string& k, const std::string& v) {
    char* end = nullptr;
    const long x = std::strtol(v.c_str(), &end, 10);
    if (v.empty() || *end != '\0') throw latsum::validation_error(k + ": not an integer: '" + v + "'");
    return x;
}
std::vector<std::string> split(const std::string& s, char d) {
    std::vector<std::string> out;
    std::stringstream ss(s);
    std::string item;
    while (std::getline(ss, item, d)) out.push_back(item);
    return out;
}
std::vector<Index> index_list(const std::string& k, const std::string& v) {
    std::vector<Index> out;
    for (const std::string& x : split(v, ',')) out.push_back(static_cast<Index>(to_long(k, x)));
    return out;
}

const std::map<std::string, std::vector<std::string>>& known_options() {
    static const std::map<std::string, std::vector<std::string>> m = {
        {"kernel", {"--n", "--b", "--eps", "--M", "--C0", "--doubled", "--out", "--report"}},
        {"sum-box", {"--L", "--n", "--b", "--eps", "--charges", "--out", "--report"}},
        {"sum-periodic", {"--L", "--n", "--b", "--eps", "--charges", "--out", "--report"}},
        {"series", {"--kind", "--L", "--n", "--b", "--eps", "--extrapolate", "--report"}},
        {"project", {"--from", "--basis", "--out", "--no-volume"}},
        {"qtt-ranks", {"--from", "--eps", "--report"}},
        {"qtt-gauss", {"--p", "--eps-list", "--levels", "--report"}},
    };
    return m;
}
bool is_flag(const std::string& k) { return k == "--doubled" || k == "--no-volume"; }

Args parse(int argc, char** argv, int& threads, long& seed) {
    Args a;
    int i = 1;
    for (; i < argc; ++i) {  // global options before the subcommand
        const std::string k = argv[i];
        if (k == "--threads" || k == "--seed") {
            if (i + 1 >= argc) throw latsum::validation_error(k + " needs a value");
            if (k == "--threads") threads = static_cast<int>(to_long(k, argv[++i]));
            else seed = to_long(k, argv[++i]);
        } else {
            break;
        }
    }
    if (i >= argc) throw latsum::validation_error("no subcommand given");
    a.command = argv[i++];
    auto it = known_options().find(a.command);
    if (it == known_options().end())
        throw latsum::validation_error("unknown or unsupported subcommand '" + a.command + "'");
    for (; i < argc; ++i) {
        const std::string k = argv[i];
        if (std::find(it->second.begin(), it->second.end(), k) == it->second.end())
            throw latsum::validation_error(a.command + ": unknown option " + k);
        if (is_flag(k)) {
            a.opt[k] = "1";
        } else {
            if (i + 1 >= argc) throw latsum::validation_error(k + " needs a value");
            a.opt[k] = argv[++i];
        }
    }
    return a;
}

// ---- outputs ---------------------------------------------------------------------------
// The resolved configuration next to the primary output (keys sorted, two-space indent, as
// proj/tools/latsum.cpp:34-41 writes it).
struct Json {
    std::map<std::string, std::string> kv;  // key -> serialized value
    static std::string q(const std::string& s) {
        std::string o = "\"";
        for (char c : s) {
            if (c == '"' || c == '\\') o += '\\';
            o += c;
        }
        return o + "\"";
    }
    // Shortest text that reads back to the same double, written like nlohmann::json's dump
    // (".0" on integral values).
    static std::string num(double x) {
        char buf[40];
        for (int prec = 1; prec <= 17; ++prec) {
            std::snprintf(buf, sizeof(buf), "%.*g", prec, x);
            if (std::strtod(buf, nullptr) == x) break;
        }
        std::string s = buf;
        if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
        return s;
    }
    std::string dump(int indent = 2, int depth = 1) const {
        std::string pad(static_cast<size_t>(indent * depth), ' '), pad0(static_cast<size_t>(indent * (depth - 1)), ' ');
        std::string o = "{\n";
        size_t e = 0;
        for (const auto& [k, v] : kv) o += pad + q(k) + ": " + v + (++e < kv.size() ? ",\n" : "\n");
        return o + pad0 + "}";
    }
};

void write_run_config(const std::string& anchor, const Json& cfg) {
    const std::string path = anchor + ".run.json";
    std::ofstream out(path);
    if (!out) throw latsum::validation_error("config: cannot open '" + path + "' for writing");
    out << cfg.dump() << "\n";
    if (!out) throw latsum::validation_error("config: write to '" + path + "' failed");
}

Json base_config(const std::string& command, int threads_flag, long seed, const Json& params) {
    Json cfg;
    cfg.kv["command"] = Json::q(command);
    cfg.kv["threads"] = std::to_string(latsum::max_threads());
    cfg.kv["threads_flag"] = std::to_string(threads_flag);
    cfg.kv["seed"] = std::to_string(seed);
    std::string p = params.dump(2, 2);
    cfg.kv["params"] = p;
    return cfg;
}

// proj/include/latsum/repro.hpp:346-358 (comma-separated, header first).
void write_csv(const std::string& path, const std::vector<std::string>& header,
               const std::vector<std::vector<std::string>>& rows) {
    std::ofstream out(path);
    if (!out) throw latsum::validation_error("csv: cannot open '" + path + "' for writing");
    for (size_t i = 0; i < header.size(); ++i) out << (i ? "," : "") << header[i];
    out << "\n";
    for (const auto& row : rows) {
        for (size_t i = 0; i < row.size(); ++i) out << (i ? "," : "") << row[i];
        out << "\n";
    }
    if (!out) throw latsum::validation_error("csv: write to '" + path + "' failed");
}

std::string lattice_to_string(const std::array<Index, 3>& L) {
    return std::to_string(L[0]) + "x" + std::to_string(L[1]) + "x" + std::to_string(L[2]);
}

std::array<double, 3> grid_origin(const latsum::Dims3& d, double h) {
    return {latsum::GridSpec::midpoint(0, d[0], h), latsum::GridSpec::midpoint(0, d[1], h),
            latsum::GridSpec::midpoint(0, d[2], h)};
}

std::string list_json(const std::vector<Index>& v) {
    std::string o = "[";
    for (size_t i = 0; i < v.size(); ++i) o += (i ? ", " : "") + std::to_string(v[i]);
    return o + "]";
}

// ---- subcommands -----------------------------------------------------------------------
int run_kernel(const Args& a, int threads, long seed) {  // proj/tools/latsum.cpp:88-130
    const Index n = to_long("--n", a.need("--n"));
    const double b = to_double("--b", a.need("--b")), eps = to_double("--eps", a.str("--eps", "1e-06"));
    const int M = static_cast<int>(to_long("--M", a.str("--M", "0")));
    const double C0 = to_double("--C0", a.str("--C0", "0"));
    const bool doubled = a.has("--doubled");
    const std::string out = a.need("--out"), report = a.str("--report");
    Json params;
    params.kv = {{"n", std::to_string(n)}, {"b", Json::num(b)}, {"eps", Json::num(eps)}, {"M", std::to_string(M)},
                 {"C0", Json::num(C0)}, {"doubled", doubled ? "true" : "false"}, {"out", Json::q(out)},
                 {"report", Json::q(report)}};
    write_run_config(out, base_config("kernel", threads, seed, params));
    const latsum::GridSpec grid(b, n);
    const latsum::KernelTolerance tol = latsum::default_tolerance(grid, eps);
    latsum::CalibrationTrace trace;
    const latsum::QuadratureRule rule = M > 0 ? latsum::sinc_quadrature(eps, tol.a_min, tol.a_max, M, C0 > 0.0 ? C0 : 1.0)
                                              : latsum::calibrate_quadrature(grid, tol, &trace);
    const Index len = doubled ? 2 * n : n;
    const latsum::CanonicalTensor3 kernel = latsum::build_newton_tensor(grid, rule, doubled);
    const latsum::GridSpec eval_grid(doubled ? 2.0 * b : b, len);
    const double err = latsum::measure_probe_error(kernel, latsum::kernel_probe_set(eval_grid, tol));
    latsum::save_bundle(out, latsum::TensorBundle{kernel, grid.h(), grid_origin(kernel.dims(), grid.h())});
    std::cout << "kernel: rank " << rule.node_count() << " (M=" << rule.M << ", C0=" << rule.C0 << "), grid " << len
              << "^3, h=" << grid.h() << "\n"
              << "measured relative error " << err << " over [" << tol.a_min << ", " << tol.a_max << "] (requested "
              << eps << ")\n"
              << "calibration candidates tried: " << trace.entries.size() << "\n"
              << "bundle written to " << out << "\n";
    if (!report.empty()) {
        std::vector<std::vector<std::string>> rows;
        for (const auto& e : trace.entries)
            rows.push_back({std::to_string(e.M), latsum::format_double(e.C0), latsum::format_double(e.err)});
        if (rows.empty())
            rows.push_back({std::to_string(rule.M), latsum::format_double(rule.C0), latsum::format_double(err)});
        write_csv(report, {"M", "C0", "probe_rel_err"}, rows);
    }
    return exit_ok;
}

latsum::LatticeSpec make_lattice(const std::vector<Index>& L, Index n, double b, const std::string& charges) {
    latsum::LatticeSpec spec;
    if (L.size() == 1) spec.L = {L[0], L[0], L[0]};
    else if (L.size() == 3) spec.L = {L[0], L[1], L[2]};
    else throw latsum::validation_error("--L expects one count or three comma-separated counts");
    spec.unit = latsum::GridSpec(b, n);
    spec.charges = charges.empty() ? std::vector<latsum::Charge>{latsum::Charge{{0.0, 0.0, 0.0}, 1.0}}
                                   : latsum::read_charges_csv(charges);
    spec.validate();
    return spec;
}

int run_sum(const Args& a, bool periodic, int threads, long seed) {  // proj/tools/latsum.cpp:132-159
    const std::vector<Index> L = index_list("--L", a.need("--L"));
    const Index n = to_long("--n", a.need("--n"));
    const double b = to_double("--b", a.need("--b")), eps = to_double("--eps", a.str("--eps", "1e-06"));
    const std::string charges = a.str("--charges"), out = a.need("--out"), report = a.str("--report");
    Json params;
    params.kv = {{"L", list_json(L)},          {"n", std::to_string(n)},  {"b", Json::num(b)},
                 {"eps", Json::num(eps)},      {"charges", Json::q(charges)}, {"out", Json::q(out)},
                 {"report", Json::q(report)}};
    write_run_config(out, base_config(periodic ? "sum-periodic" : "sum-box", threads, seed, params));
    const latsum::LatticeSpec spec = make_lattice(L, n, b, charges);
    const latsum::QuadratureRule rule = latsum::calibrate_for_lattice(spec, eps);
    const latsum::CanonicalTensor3 master = latsum::build_lattice_master(spec, rule);
    const latsum::SumResult sum = periodic ? latsum::assembled_periodic_sum(spec, master)
                                           : latsum::assembled_box_sum(spec, master);
    latsum::save_bundle(out, latsum::TensorBundle{sum.tensor, spec.unit.h(), grid_origin(sum.grid_dims, spec.unit.h())});
    const double p_center =
        latsum::eval_point(sum.tensor, sum.grid_dims[0] / 2, sum.grid_dims[1] / 2, sum.grid_dims[2] / 2);
    std::cout << (periodic ? "periodic" : "box") << " sum: lattice " << lattice_to_string(spec.L) << ", grid "
              << latsum::dims_to_string(sum.grid_dims) << ", rank " << sum.rank << ", kernel rank "
              << rule.node_count() << "\n"
              << "center value " << p_center << " au, assembly time " << sum.time_ms << " ms\n"
              << "bundle written to " << out << "\n";
    if (!report.empty())
        write_csv(report, {"L", "rank", "time_ms", "p_center_au", "p_hat_au"},
                  {{lattice_to_string(spec.L), std::to_string(sum.rank), latsum::format_double(sum.time_ms),
                    latsum::format_double(p_center), ""}});
    return exit_ok;
}

int run_series(const Args& a, int threads, long seed) {  // proj/tools/latsum.cpp:161-204
    const std::string kind_name = a.str("--kind", "cube"), extrapolate = a.str("--extrapolate");
    const std::string report = a.str("--report", "series.csv");
    const std::vector<Index> L_list = index_list("--L", a.need("--L"));
    const Index n = to_long("--n", a.str("--n", "32"));
    const double b = to_double("--b", a.str("--b", "2")), eps = to_double("--eps", a.str("--eps", "1e-06"));
    Json params;
    params.kv = {{"kind", Json::q(kind_name)}, {"L", list_json(L_list)}, {"n", std::to_string(n)},
                 {"b", Json::num(b)},          {"eps", Json::num(eps)},   {"extrapolate", Json::q(extrapolate)},
                 {"report", Json::q(report)}};
    write_run_config(report, base_config("series", threads, seed, params));
    latsum::SeriesKind kind;
    if (kind_name == "line") kind = latsum::SeriesKind::line;
    else if (kind_name == "plane") kind = latsum::SeriesKind::plane;
    else if (kind_name == "cube") kind = latsum::SeriesKind::cube;
    else throw latsum::validation_error("--kind must be line, plane or cube");
    bool use_richardson = false;
    latsum::RichardsonOrder order = latsum::RichardsonOrder::linear;
    if (extrapolate == "linear") {
        use_richardson = true;
    } else if (extrapolate == "quadratic") {
        use_richardson = true;
        order = latsum::RichardsonOrder::quadratic;
    } else if (!extrapolate.empty() && extrapolate != "none") {
        throw latsum::validation_error("--extrapolate must be linear, quadratic or none");
    }
    const std::vector<latsum::SeriesPoint> pts = latsum::center_value_series(kind, L_list, latsum::GridSpec(b, n), eps);
    std::vector<std::vector<std::string>> rows;
    for (size_t i = 0; i < pts.size(); ++i) {
        std::string p_hat;
        if (use_richardson && i + 1 < pts.size() && pts[i + 1].L == 2 * pts[i].L)
            p_hat = latsum::format_double(latsum::richardson_extrapolate(pts[i].p_center, pts[i + 1].p_center, order));
        rows.push_back({std::to_string(pts[i].L), std::to_string(pts[i].rank), latsum::format_double(pts[i].time_ms),
                        latsum::format_double(pts[i].p_center), p_hat});
        std::cout << kind_name << " L=" << pts[i].L << ": p_center " << pts[i].p_center << " au"
                  << (p_hat.empty() ? "" : ", extrapolated " + p_hat) << "\n";
    }
    write_csv(report, {"L", "rank", "time_ms", "p_center_au", "p_hat_au"}, rows);
    std::cout << "series written to " << report << "\n";
    return exit_ok;
}

int run_project(const Args& a, int threads, long seed) {  // proj/tools/latsum.cpp:283-321
    const std::string from = a.need("--from"), basis_path = a.need("--basis"), out = a.need("--out");
    const bool volume = !a.has("--no-volume");
    Json params;
    params.kv = {{"from", Json::q(from)}, {"basis", Json::q(basis_path)}, {"out", Json::q(out)},
                 {"volume_element", volume ? "true" : "false"}};
    write_run_config(out, base_config("project", threads, seed, params));
    const latsum::TensorBundle bundle = latsum::load_bundle(from);
    const latsum::Dims3 dims = bundle.tensor.dims();
    if (dims[0] != dims[1] || dims[0] != dims[2])
        throw latsum::validation_error("project: bundle grid " + latsum::dims_to_string(dims) + " is not cubic");
    const Index n = dims[0];
    if (n < 2 || n % 2 != 0) throw latsum::validation_error("project: bundle grid size must be even and >= 2");
    if (!(bundle.h > 0.0)) throw latsum::validation_error("project: bundle has non-positive mesh width");
    const latsum::GridSpec grid(bundle.h * static_cast<double>(n), n);
    for (int l = 0; l < 3; ++l)
        if (std::abs(bundle.origin[static_cast<size_t>(l)] - grid.midpoint(0)) > 1e-9 * grid.b)
            throw latsum::validation_error(
                "project: bundle grid is not centered at the origin; basis sampling assumes a centered grid");
    const std::vector<latsum::GaussianBasisSpec> specs = latsum::read_basis_csv(basis_path);
    const latsum::Rank1Basis basis = latsum::sample_gaussian_basis(grid, specs);
    const latsum::Matrix V = latsum::potential_matrix(basis, bundle.tensor, volume);
    std::vector<std::string> header;
    for (Index m = 0; m < V.cols(); ++m) header.push_back("v" + std::to_string(m) + "_au");
    std::vector<std::vector<std::string>> rows;
    for (Index k = 0; k < V.rows(); ++k) {
        std::vector<std::string> row;
        for (Index m = 0; m < V.cols(); ++m) row.push_back(latsum::format_double(V(k, m)));
        rows.push_back(std::move(row));
    }
    write_csv(out, header, rows);
    std::cout << "project: " << V.rows() << "x" << V.cols() << " matrix written to " << out
              << (volume ? " (volume element applied)" : " (raw scalar products)") << "\n";
    return exit_ok;
}

std::string dlist_json(const std::vector<double>& v) {
    std::string o = "[";
    for (size_t i = 0; i < v.size(); ++i) o += (i ? ", " : "") + Json::num(v[i]);
    return o + "]";
}
std::vector<double> double_list(const std::string& k, const std::string& v) {
    std::vector<double> out;
    for (const std::string& x : split(v, ',')) out.push_back(to_double(k, x));
    return out;
}

int run_qtt_ranks(const Args& a, int threads, long seed) {  // proj/tools/latsum.cpp:206-242
    const std::string from = a.need("--from"), report = a.str("--report", "qtt_ranks.csv");
    const double eps = to_double("--eps", a.str("--eps", "1e-08"));
    Json params;
    params.kv = {{"from", Json::q(from)}, {"eps", Json::num(eps)}, {"report", Json::q(report)}};
    write_run_config(report, base_config("qtt-ranks", threads, seed, params));
    const latsum::TensorBundle bundle = latsum::load_bundle(from);
    if (bundle.tensor.rank() < 1) throw latsum::validation_error("qtt-ranks: bundle has rank 0, nothing to compress");
    std::vector<std::vector<std::string>> rows;
    double sum_max = 0.0;
    Index count = 0;
    for (int axis = 0; axis < 3; ++axis) {
        const latsum::Matrix& factor = bundle.tensor.factor(axis);
        const Index N = factor.rows();
        Index padded = 2;
        while (padded < N) padded *= 2;
        latsum::Matrix V = latsum::Matrix::Zero(padded, bundle.tensor.rank());
        for (Index q = 0; q < bundle.tensor.rank(); ++q)
            for (Index i = 0; i < N; ++i) V(i, q) = factor(i, q);
        const std::vector<latsum::QTTVector> trains = latsum::detail::qtt_compress_columns(V, eps);  // one launch
        for (Index q = 0; q < bundle.tensor.rank(); ++q) {
            const latsum::QTTVector& t = trains[static_cast<size_t>(q)];
            const latsum::RankProfile prof = latsum::qtt_rank_profile(t);
            const latsum::Vector rec = latsum::qtt_reconstruct(t);
            double num = 0.0, den = 0.0;
            for (Index i = 0; i < N; ++i) {
                num += (rec[i] - factor(i, q)) * (rec[i] - factor(i, q));
                den += factor(i, q) * factor(i, q);
            }
            const double err = den > 0.0 ? std::sqrt(num / den) : std::sqrt(num);
            rows.push_back({std::to_string(axis), std::to_string(q), std::to_string(prof.max_rank),
                            latsum::format_double(prof.avg_rank), latsum::format_double(err)});
            sum_max += static_cast<double>(prof.max_rank);
            ++count;
        }
    }
    write_csv(report, {"axis", "q", "max_rank", "avg_rank", "err"}, rows);
    std::cout << "qtt-ranks: " << count << " columns from " << from << ", average max rank "
              << sum_max / static_cast<double>(count) << "\n"
              << "report written to " << report << "\n";
    return exit_ok;
}

// Least-squares slope of y against x (bench.hpp:41-51).
double fit_slope(const std::vector<double>& x, const std::vector<double>& y) {
    const double n = static_cast<double>(x.size());
    double sx = 0.0, sy = 0.0, sxx = 0.0, sxy = 0.0;
    for (size_t i = 0; i < x.size(); ++i) {
        sx += x[i];
        sy += y[i];
        sxx += x[i] * x[i];
        sxy += x[i] * y[i];
    }
    return (n * sxy - sx * sy) / (n * sxx - sx * sx);
}

int run_qtt_gauss(const Args& a, int threads, long seed) {  // proj/tools/latsum.cpp:244-281
    const std::vector<double> p_list = double_list("--p", a.str("--p", "1"));
    const std::vector<double> eps_list = double_list("--eps-list", a.str("--eps-list", "1e-3,1e-4,1e-5,1e-6,1e-7,1e-8,1e-9"));
    const Index levels = to_long("--levels", a.str("--levels", "12"));
    const std::string report = a.str("--report");
    Json params;
    params.kv = {{"p", dlist_json(p_list)}, {"eps_list", dlist_json(eps_list)}, {"levels", std::to_string(levels)},
                 {"report", Json::q(report)}};
    write_run_config(report.empty() ? "qtt-gauss" : report, base_config("qtt-gauss", threads, seed, params));
    if (levels < 2 || levels > 24) throw latsum::validation_error("qtt-gauss: --levels must lie in [2, 24]");
    for (double eps : eps_list)
        if (!(eps > 0.0) || !(eps < 1.0)) throw latsum::validation_error("qtt-gauss: eps values must lie in (0, 1)");
    const Index N = Index{1} << levels;
    std::vector<std::vector<std::string>> rows;
    for (double p : p_list) {
        if (!(p > 0.0)) throw latsum::validation_error("qtt-gauss: p must be positive");
        std::vector<double> lx, ly;
        for (double eps : eps_list) {
            const double aa = std::sqrt(2.0) * p * std::sqrt(std::log(1.0 / eps));
            latsum::Vector v(N);
            for (Index i = 0; i < N; ++i) {
                const double x = (static_cast<double>(i) + 0.5) / static_cast<double>(N) * 2.0 * aa - aa;
                v[i] = std::exp(-x * x / (2.0 * p * p));
            }
            const Index r = latsum::max_unfolding_rank(v, eps);
            rows.push_back({latsum::format_double(p), latsum::format_double(eps), std::to_string(r)});
            lx.push_back(std::log(1.0 / eps));
            ly.push_back(static_cast<double>(r));
        }
        const double slope = lx.size() >= 2 ? fit_slope(lx, ly) : 0.0;
        std::cout << "p=" << p << ": max rank vs ln(1/eps) slope " << slope << "\n";
    }
    if (!report.empty()) {
        write_csv(report, {"p", "eps", "max_rank"}, rows);
        std::cout << "report written to " << report << "\n";
    }
    return exit_ok;
}

}  // namespace

int main(int argc, char** argv) {
    int threads = 0;
    long seed = 0;
    try {
        const Args a = parse(argc, argv, threads, seed);
        if (threads > 0) latsum::set_max_threads(threads);
        if (a.command == "kernel") return run_kernel(a, threads, seed);
        if (a.command == "sum-box") return run_sum(a, false, threads, seed);
        if (a.command == "sum-periodic") return run_sum(a, true, threads, seed);
        if (a.command == "series") return run_series(a, threads, seed);
        if (a.command == "project") return run_project(a, threads, seed);
        if (a.command == "qtt-ranks") return run_qtt_ranks(a, threads, seed);
        if (a.command == "qtt-gauss") return run_qtt_gauss(a, threads, seed);
        std::cerr << "no subcommand given\n";
        return exit_validation;
    } catch (const latsum::resource_guard_error& e) {
        std::cerr << "resource guard: " << e.what() << "\n";
        return exit_resource_guard;
    } catch (const latsum::validation_error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return exit_validation;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return exit_validation;
    }
}
