// oracle/spec.hpp — TEST INFRASTRUCTURE ONLY.  Text form of a layer list,
// shared (as a grammar, not as code) with the product's network builder so
// tests can build the same network on both sides:
//   "dense IN OUT; conv2d CIN COUT K S P; convT2d CIN COUT K S P; bn C [EPS MOM];
//    upsample F; dropout RATE; relu; lrelu [SLOPE]; tanh; sigmoid; reshape D..."
#pragma once

#include "oracle.hpp"

#include <sstream>

namespace oracle {

inline std::vector<Layer> parse_layers(const std::string& text) {
  std::vector<Layer> out;
  std::stringstream all(text);
  std::string item;
  while (std::getline(all, item, ';')) {
    std::stringstream ss(item);
    std::string name;
    if (!(ss >> name)) continue;
    std::vector<double> a;
    double v;
    while (ss >> v) a.push_back(v);
    auto need = [&](size_t n) {
      if (a.size() < n) throw std::invalid_argument("layer spec '" + item + "' needs " + std::to_string(n) + " numbers");
    };
    auto L = [&](size_t i) { return static_cast<long>(a[i]); };
    if (name == "dense") { need(2); out.push_back(Layer::dense(L(0), L(1))); }
    else if (name == "conv2d") { need(5); out.push_back(Layer::conv(L(0), L(1), L(2), L(3), L(4))); }
    else if (name == "convT2d") { need(5); out.push_back(Layer::convT(L(0), L(1), L(2), L(3), L(4))); }
    else if (name == "bn") {
      need(1);
      out.push_back(Layer::bn(L(0), a.size() > 1 ? a[1] : 1e-5, a.size() > 2 ? a[2] : 0.1));
    }
    else if (name == "upsample") { need(1); out.push_back(Layer::upsample(L(0))); }
    else if (name == "dropout") { need(1); out.push_back(Layer::dropout(a[0])); }
    else if (name == "relu") out.push_back(Layer::relu());
    else if (name == "lrelu") out.push_back(Layer::lrelu(a.empty() ? 0.2 : a[0]));
    else if (name == "tanh") out.push_back(Layer::tanh_());
    else if (name == "sigmoid") out.push_back(Layer::sigmoid());
    else if (name == "reshape") {
      need(1);
      Shape t;
      for (size_t i = 0; i < a.size(); ++i) t.push_back(L(i));
      out.push_back(Layer::reshape(t));
    } else {
      throw std::invalid_argument("unknown layer '" + name + "'");
    }
  }
  return out;
}

inline Shape parse_shape(const std::string& text) {
  std::stringstream ss(text);
  Shape s;
  long v;
  while (ss >> v) s.push_back(v);
  return s;
}

}  // namespace oracle
