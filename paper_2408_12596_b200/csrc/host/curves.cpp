// Natural cubic spline and per-device speed curves.
//
// Restates reference spline.cpp:25-129 and perf_curve.cpp:24-126. The arithmetic
// order (Thomas sweep, coefficient formulas, Horner evaluation, peak scan) is kept
// exactly, because the planner's plan must be bit-identical to the reference's.
#include <algorithm>
#include <string>

#include "zeroplan/zeroplan.hpp"

namespace zeroplan {

namespace {

// Solves the natural-spline tridiagonal system for the knot second derivatives
// (m[0] = m[n] = 0). Row k (knot k+1): 2(h[k]+h[k+1]) on the diagonal, h[k+1] above,
// h[k] below, right-hand side 6 * (slope[k+1] - slope[k]).
std::vector<double> knot_curvatures(const std::vector<SamplePoint>& p, const std::vector<double>& h) {
  const std::size_t segs = h.size();
  std::vector<double> m(segs + 1, 0.0);
  if (segs < 2) return m;
  const std::size_t rows = segs - 1;
  std::vector<double> dia(rows), sup(rows), r(rows);
  for (std::size_t k = 0; k < rows; ++k) {
    const std::size_t j = k + 1;
    dia[k] = 2.0 * (h[j - 1] + h[j]);
    sup[k] = h[j];
    const double right = (p[j + 1].y - p[j].y) / h[j];
    const double left = (p[j].y - p[j - 1].y) / h[j - 1];
    r[k] = 6.0 * (right - left);
  }
  for (std::size_t k = 1; k < rows; ++k) {  // elimination of the sub-diagonal h[k]
    const double f = h[k] / dia[k - 1];
    dia[k] -= f * sup[k - 1];
    r[k] -= f * r[k - 1];
  }
  m[rows] = r[rows - 1] / dia[rows - 1];
  for (std::size_t k = rows - 1; k >= 1; --k) m[k] = (r[k - 1] - sup[k - 1] * m[k + 1]) / dia[k - 1];
  return m;
}

}  // namespace

CubicSpline fit_natural_spline(std::vector<SamplePoint> pts) {
  if (pts.size() < 2)
    throw InvalidInputError("spline fit requires at least 2 points, got " +
                            std::to_string(pts.size()));
  std::sort(pts.begin(), pts.end(),
            [](const SamplePoint& a, const SamplePoint& b) { return a.x < b.x; });
  for (std::size_t i = 1; i < pts.size(); ++i)
    if (pts[i].x == pts[i - 1].x)
      throw InvalidInputError("spline fit requires distinct x values; x = " +
                              std::to_string(pts[i].x) + " repeats");

  const std::size_t segs = pts.size() - 1;
  std::vector<double> h(segs);
  for (std::size_t i = 0; i < segs; ++i) h[i] = pts[i + 1].x - pts[i].x;
  const std::vector<double> m = knot_curvatures(pts, h);

  CubicSpline s;
  s.x_.reserve(pts.size());
  s.y_.reserve(pts.size());
  for (const SamplePoint& q : pts) {
    s.x_.push_back(q.x);
    s.y_.push_back(q.y);
  }
  s.seg_.resize(segs);
  for (std::size_t i = 0; i < segs; ++i) {
    CubicSpline::Segment& g = s.seg_[i];
    g.a = pts[i].y;
    g.b = (pts[i + 1].y - pts[i].y) / h[i] - h[i] * (2.0 * m[i] + m[i + 1]) / 6.0;
    g.c = m[i] / 2.0;
    g.d = (m[i + 1] - m[i]) / (6.0 * h[i]);
  }
  return s;
}

std::size_t CubicSpline::locate(double x) const {
  // Segment i covers [x_i, x_{i+1}); the last one also owns x_n.
  const std::size_t above =
      static_cast<std::size_t>(std::upper_bound(x_.begin(), x_.end(), x) - x_.begin());
  if (above == 0) return 0;
  return std::min(above - 1, seg_.size() - 1);
}

double CubicSpline::eval(double x) const {
  if (x <= x_.front()) return y_.front();
  if (x >= x_.back()) return y_.back();
  const std::size_t i = locate(x);
  const Segment& g = seg_[i];
  const double t = x - x_[i];
  return g.a + t * (g.b + t * (g.c + t * g.d));
}

double CubicSpline::first_derivative(double x) const {
  x = std::clamp(x, x_.front(), x_.back());
  const std::size_t i = locate(x);
  const Segment& g = seg_[i];
  const double t = x - x_[i];
  return g.b + t * (2.0 * g.c + 3.0 * g.d * t);
}

double CubicSpline::second_derivative(double x) const {
  x = std::clamp(x, x_.front(), x_.back());
  const std::size_t i = locate(x);
  const Segment& g = seg_[i];
  const double t = x - x_[i];
  return 2.0 * g.c + 6.0 * g.d * t;
}

double eval_spline(const CubicSpline& spline, double x) { return spline.eval(x); }

// ------------------------------------------------------------------ PerfCurve

double PerfCurve::speed_at(double batch) const {
  const double raw = spline_ ? spline_->eval(batch) : constant_speed_;
  return std::max(raw, kSpeedFloor);
}

double PerfCurve::predict_step_time(std::int64_t b) const {
  if (b < 1 || b > mbs_)
    throw InvalidInputError("batch size " + std::to_string(b) + " outside [1, " +
                            std::to_string(mbs_) + "]");
  return times_[static_cast<std::size_t>(b - 1)];
}

std::int64_t PerfCurve::find_max_batch_within_time(double t) const {
  std::int64_t b = mbs_;
  while (b >= 1 && !(times_[static_cast<std::size_t>(b - 1)] <= t)) --b;
  return b < 1 ? 0 : b;
}

PerfCurve build_curve(std::vector<BatchSample> samples, std::int64_t mbs, int device_id) {
  if (samples.empty()) throw InvalidInputError("build_curve requires at least one sample");
  if (mbs < 1) throw InvalidInputError("build_curve requires mbs >= 1");
  std::sort(samples.begin(), samples.end(),
            [](const BatchSample& a, const BatchSample& b) { return a.batch < b.batch; });
  for (std::size_t i = 0; i < samples.size(); ++i) {
    const BatchSample& s = samples[i];
    if (s.batch < 1 || s.batch > mbs)
      throw InvalidInputError("sample batch size " + std::to_string(s.batch) +
                              " outside [1, mbs]");
    if (s.time <= 0.0) throw InvalidInputError("sample step time must be positive");
    if (i > 0 && s.batch == samples[i - 1].batch)
      throw InvalidInputError("duplicate sample batch size " + std::to_string(s.batch));
  }

  PerfCurve c;
  c.device_id_ = device_id;
  c.mbs_ = mbs;
  c.samples_ = samples;
  if (samples.size() == 1) {
    c.constant_speed_ = static_cast<double>(samples[0].batch) / samples[0].time;
  } else {
    // Speed points (b, b / t_b) — Poplar fits batches/second, not seconds.
    std::vector<SamplePoint> pts;
    pts.reserve(samples.size());
    for (const BatchSample& s : samples) {
      const double b = static_cast<double>(s.batch);
      pts.push_back(SamplePoint{b, b / s.time});
    }
    c.spline_ = fit_natural_spline(std::move(pts));
  }

  const std::size_t n = static_cast<std::size_t>(mbs);
  c.speeds_.assign(n, 0.0);
  c.times_.assign(n, 0.0);
  std::int64_t argmax = 1;
  for (std::size_t i = 0; i < n; ++i) {
    const double b = static_cast<double>(i + 1);
    const double v = c.speed_at(b);
    c.speeds_[i] = v;
    c.times_[i] = b / v;
    if (v > c.peak_speed_) {  // first strict maximum wins
      c.peak_speed_ = v;
      argmax = static_cast<std::int64_t>(i + 1);
    }
  }
  // Widest contiguous run around the argmax staying within 5% of the peak.
  const double keep = (1.0 - PerfCurve::kPeakEpsilon) * c.peak_speed_;
  std::int64_t lo = argmax, hi = argmax;
  while (lo > 1 && c.speeds_[static_cast<std::size_t>(lo - 2)] >= keep) --lo;
  while (hi < mbs && c.speeds_[static_cast<std::size_t>(hi)] >= keep) ++hi;
  c.peak_range_ = PerfCurve::PeakRange{lo, hi};
  return c;
}

std::vector<PerfCurve> build_curves(const ProfileResult& profile) {
  std::vector<PerfCurve> out;
  out.reserve(profile.devices.size());
  for (const DeviceProfile& d : profile.devices)
    out.push_back(build_curve(d.samples, d.mbs, d.device_id));
  return out;
}

}  // namespace zeroplan
