// TEST INFRASTRUCTURE ONLY -- writes the reference's own output files
// (tpfem/report.hpp: report_to_json + write_json, write_residuals_csv,
// TableWriter) for synthetic SolveReports, so tests/test_report.py can pin the
// package's writers (paper_2502_21013_b200/report.py) byte for byte.
//
// usage: report_fixture <spec> <outdir>
//   spec: text file, one report per line:
//     method status iterations wall q n_hist h0 h1 ... n_contr c0 c1 ...
//   (method m1|m2|m3, status converged|max_iter|stalled, q "nan" allowed),
//   followed by table rows "T steps n_dof init m1_it m1_s m2_it m2_s m3_it m3_s".
// Writes <outdir>/report.json ({"methods": {...}} of all reports, the
// report_to_json part of run_solve, runner.hpp:184-217), residuals.csv and
// table.csv.
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "tpfem/mesh.hpp"
#include "tpfem/report.hpp"
#include "tpfem/vtk.hpp"

using namespace tpfem;

static double num(const std::string& s) {
  if (s == "nan") return std::numeric_limits<double>::quiet_NaN();
  return std::strtod(s.c_str(), nullptr);  // (subnormals too, unlike std::stod)
}

// usage: report_fixture vtk <outdir>: mesh.vtk and u.vtk (vtk.hpp) of the
// reference transformer mesh (12 x 10 cells, build_rectilinear_mesh) with the
// field u[d] = sin(0.37 d) - 1e-3 d on the free dofs.
static int vtk_fixture(const std::filesystem::path& out) {
  std::filesystem::create_directories(out);
  const Mesh m = build_rectilinear_mesh(transformer_regions(), 12, 10);
  write_mesh_vtk(out / "mesh.vtk", m);
  std::vector<double> u(static_cast<std::size_t>(m.n_dof()));
  for (std::size_t d = 0; d < u.size(); ++d) u[d] = std::sin(0.37 * static_cast<double>(d)) - 1e-3 * static_cast<double>(d);
  write_field_vtk(out / "u.vtk", m, u);
  return 0;
}

int main(int argc, char** argv) {
  if (argc == 3 && std::string(argv[1]) == "vtk") return vtk_fixture(argv[2]);
  if (argc != 3) {
    std::cerr << "usage: report_fixture <spec> <outdir>\n";
    return 1;
  }
  std::ifstream in(argv[1]);
  const std::filesystem::path out = argv[2];
  std::filesystem::create_directories(out);
  std::vector<SolveReport> reports;
  std::vector<TableRow> rows;
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    std::istringstream ls(line);
    std::string tag;
    ls >> tag;
    if (tag == "T") {
      TableRow r;
      std::string a, b, c, d, e, f, g, h, i;
      ls >> a >> b >> c >> d >> e >> f >> g >> h >> i;
      r.steps = std::stoi(a);
      r.n_dof = std::stoll(b);
      r.init_seconds = num(c);
      r.m1_iterations = std::stoi(d);
      r.m1_seconds = num(e);
      r.m2_iterations = std::stoi(f);
      r.m2_seconds = num(g);
      r.m3_iterations = std::stoi(h);
      r.m3_seconds = num(i);
      rows.push_back(r);
      continue;
    }
    SolveReport r;
    r.method = tag == "m1" ? Method::m1 : tag == "m2" ? Method::m2 : Method::m3;
    std::string st, it, wall, q, nh;
    ls >> st >> it >> wall >> q >> nh;
    r.status = st == "converged" ? SolveStatus::converged
               : st == "max_iter" ? SolveStatus::max_iter
                                  : SolveStatus::stalled;
    r.iterations = std::stoi(it);
    r.wall_time = num(wall);
    r.q_estimate = num(q);
    for (int k = 0, n = std::stoi(nh); k < n; ++k) {
      std::string v;
      ls >> v;
      r.residual_history.push_back(num(v));
    }
    std::string nc;
    ls >> nc;
    for (int k = 0, n = std::stoi(nc); k < n; ++k) {
      std::string v;
      ls >> v;
      r.contraction_history.push_back(num(v));
    }
    reports.push_back(r);
  }
  nlohmann::json methods;
  for (const SolveReport& r : reports) methods[std::string(method_name(r.method))] = report_to_json(r);
  nlohmann::json j;
  j["methods"] = methods;
  write_json(out / "report.json", j);
  std::vector<const SolveReport*> ptrs;
  for (const SolveReport& r : reports) ptrs.push_back(&r);
  write_residuals_csv(out / "residuals.csv", ptrs);
  TableWriter tw(out / "table.csv");
  for (const TableRow& r : rows) tw.add_row(r);
  return 0;
}
