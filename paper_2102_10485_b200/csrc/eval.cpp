// Evaluation of generated samples, the reference's
// host-side metrics restated in C++ with the same arithmetic (f64) and error
// messages (/root/reference/proj/src/eval.cpp):
//   softmax_rows          eval.cpp:18-33   row-wise stable softmax of [N, K] logits
//   inception_score       eval.cpp:43-94   per-split exp(mean KL(p(y|x) || p(y))), clamped to [0, log K]
//   anova_f               eval.cpp:158-186 one-way ANOVA F = MSB / MSW (+inf when MSW == 0)
//   anova_per_channel     eval.cpp:188-211 F over the per-image spatial mean of each channel, grouped by class
// These run on the host after the final gather of generated samples (a few MB
// per label); they are not on the training step's path.
#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

namespace pg {

void softmax_rows(const double* logits, long n, long k, double* probs) {
  if (n < 1 || k < 1) throw std::invalid_argument("softmax_rows: empty input");
  for (long i = 0; i < n; ++i) {
    const double* in = logits + i * k;
    double* out = probs + i * k;
    const double mx = *std::max_element(in, in + k);
    double sum = 0;
    for (long j = 0; j < k; ++j) {
      out[j] = std::exp(in[j] - mx);
      sum += out[j];
    }
    for (long j = 0; j < k; ++j) out[j] /= sum;
  }
}

// split_scores[n_splits]; returns {mean, stddev}
void inception_score(const double* probs, long n, long k, int n_splits, double* split_scores, double* mean,
                     double* stddev) {
  if (n_splits < 1) throw std::invalid_argument("inception_score: n_splits must be >= 1");
  if (n < n_splits)
    throw std::invalid_argument("inception_score: " + std::to_string(n) + " samples cannot fill " +
                                std::to_string(n_splits) + " splits");
  for (long i = 0; i < n; ++i) {
    double s = 0;
    for (long j = 0; j < k; ++j) {
      const double p = probs[i * k + j];
      if (p < 0) throw std::invalid_argument("inception_score: negative probability");
      s += p;
    }
    if (std::abs(s - 1.0) > 1e-6)
      throw std::invalid_argument("inception_score: row " + std::to_string(i) + " sums to " + std::to_string(s));
  }
  const long base = n / n_splits;
  const double log_k = std::log(static_cast<double>(k));
  std::vector<double> marginal(static_cast<size_t>(k));
  for (int s = 0; s < n_splits; ++s) {
    const long begin = base * s;
    const long end = (s == n_splits - 1) ? n : begin + base;
    const long m = end - begin;
    std::fill(marginal.begin(), marginal.end(), 0.0);
    for (long i = begin; i < end; ++i)
      for (long j = 0; j < k; ++j) marginal[static_cast<size_t>(j)] += probs[i * k + j];
    for (auto& v : marginal) v /= static_cast<double>(m);
    double kl_sum = 0;
    for (long i = begin; i < end; ++i)
      for (long j = 0; j < k; ++j) {
        const double p = probs[i * k + j];
        if (p > 0) kl_sum += p * std::log(p / marginal[static_cast<size_t>(j)]);
      }
    // mean KL is the split's mutual information: [0, log K] up to rounding
    split_scores[s] = std::exp(std::clamp(kl_sum / static_cast<double>(m), 0.0, log_k));
  }
  double mu = 0;
  for (int s = 0; s < n_splits; ++s) mu += split_scores[s];
  mu /= static_cast<double>(n_splits);
  double var = 0;
  for (int s = 0; s < n_splits; ++s) var += (split_scores[s] - mu) * (split_scores[s] - mu);
  *mean = mu;
  *stddev = std::sqrt(var / static_cast<double>(n_splits));
}

// groups given as concatenated values with sizes[k]
double anova_f(const double* values, const long* sizes, long k) {
  if (k < 2) throw std::invalid_argument("anova_f: need at least 2 groups");
  long n = 0;
  for (long j = 0; j < k; ++j) {
    if (sizes[j] < 1) throw std::invalid_argument("anova_f: group " + std::to_string(j) + " is empty");
    n += sizes[j];
  }
  if (n <= k) throw std::invalid_argument("anova_f: need more observations than groups");
  double grand = 0;
  std::vector<double> means(static_cast<size_t>(k), 0.0);
  long off = 0;
  for (long j = 0; j < k; ++j) {
    for (long i = 0; i < sizes[j]; ++i) means[static_cast<size_t>(j)] += values[off + i];
    grand += means[static_cast<size_t>(j)];
    means[static_cast<size_t>(j)] /= static_cast<double>(sizes[j]);
    off += sizes[j];
  }
  grand /= static_cast<double>(n);
  double ssb = 0, ssw = 0;
  off = 0;
  for (long j = 0; j < k; ++j) {
    const double mj = means[static_cast<size_t>(j)];
    ssb += static_cast<double>(sizes[j]) * (mj - grand) * (mj - grand);
    for (long i = 0; i < sizes[j]; ++i) ssw += (values[off + i] - mj) * (values[off + i] - mj);
    off += sizes[j];
  }
  const double msb = ssb / static_cast<double>(k - 1);
  const double msw = ssw / static_cast<double>(n - k);
  if (msw == 0.0) return std::numeric_limits<double>::infinity();
  return msb / msw;
}

// images [n][C][H][W] (any value range), labels[n] in [0, k); f[C]
void anova_per_channel(const float* images, const int* labels, long n, long C, long H, long W, long k, double* f) {
  if (k < 2) throw std::invalid_argument("anova_per_channel: need at least 2 classes");
  for (long i = 0; i < n; ++i)
    if (labels[i] < 0 || labels[i] >= k)
      throw std::out_of_range("class id " + std::to_string(labels[i]) + " out of range [0, " + std::to_string(k) +
                              ")");
  const long spatial = H * W;
  std::vector<long> sizes(static_cast<size_t>(k), 0);
  for (long i = 0; i < n; ++i) sizes[static_cast<size_t>(labels[i])] += 1;
  for (long c = 0; c < C; ++c) {
    // values grouped by class, in dataset order within a class (as the reference's push_back)
    std::vector<std::vector<double>> groups(static_cast<size_t>(k));
    for (long i = 0; i < n; ++i) {
      const float* plane = images + (i * C + c) * spatial;
      double mean = 0;
      for (long t = 0; t < spatial; ++t) mean += plane[t];
      groups[static_cast<size_t>(labels[i])].push_back(mean / static_cast<double>(spatial));
    }
    std::vector<double> flat;
    for (const auto& g : groups) flat.insert(flat.end(), g.begin(), g.end());
    f[c] = anova_f(flat.data(), sizes.data(), k);
  }
}

}  // namespace pg
