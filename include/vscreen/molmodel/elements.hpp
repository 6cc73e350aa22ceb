// Drop-in for elements.hpp:14-45 (wire-stable element codes and the chem
// interaction classes used by chem_score).
#pragma once

#include <cstdint>
#include <string_view>

namespace vscreen {

enum class Element : std::uint8_t { C = 0, N = 1, O = 2, S = 3, P = 4, F = 5, Cl = 6, Br = 7, I = 8, H = 9, Other = 10 };

inline constexpr std::uint8_t kMaxElementCode = 10;

enum class ChemClass : std::uint8_t { Hydrophobic, Polar, Other };

constexpr bool is_heavy_element(Element e) { return e != Element::H; }

constexpr ChemClass chem_class(Element e) {
  return e == Element::C ? ChemClass::Hydrophobic
                         : ((e == Element::N || e == Element::O) ? ChemClass::Polar : ChemClass::Other);
}

constexpr int standard_valence(Element e) {
  switch (e) {
    case Element::C: return 4;
    case Element::N: return 3;
    case Element::O: return 2;
    case Element::S: return 2;
    case Element::P: return 3;
    case Element::F: case Element::Cl: case Element::Br: case Element::I: case Element::H: return 1;
    default: return 0;
  }
}

constexpr std::string_view element_symbol(Element e) {
  constexpr std::string_view names[] = {"C", "N", "O", "S", "P", "F", "Cl", "Br", "I", "H", "Du"};
  const auto i = static_cast<std::uint8_t>(e);
  return i <= kMaxElementCode ? names[i] : "Du";
}

inline Element element_from_symbol(std::string_view s) {
  for (std::uint8_t i = 0; i < 10; ++i)
    if (element_symbol(static_cast<Element>(i)) == s) return static_cast<Element>(i);
  return Element::Other;
}

}  // namespace vscreen
