// Minimal stand-in for boost::multiprecision::cpp_int, used ONLY to compile the
// reference's own eplab sources into oracle/_ref (Boost is absent in this image).
// 128-bit unsigned storage: exact for every value the EP-MoE path produces
// (world <= 16, topk <= 16 => numerators <= world^topk <= 2^64).
#pragma once
#include <string>
#include <type_traits>

namespace boost {
namespace multiprecision {

class cpp_int {
 public:
  using u128 = unsigned __int128;
  cpp_int() : v_(0) {}
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
  cpp_int(T x) : v_((u128)x) {}
  cpp_int(u128 x) : v_(x) {}
  explicit cpp_int(const char* s) : v_(0) {
    for (; *s; ++s) v_ = v_ * 10 + (u128)(*s - '0');
  }
  template <class T>
  T convert_to() const {
    return static_cast<T>(v_);
  }
  std::string str() const {
    if (v_ == 0) return "0";
    std::string s;
    for (u128 x = v_; x; x /= 10) s.insert(s.begin(), char('0' + (int)(x % 10)));
    return s;
  }
  cpp_int& operator+=(const cpp_int& o) { v_ += o.v_; return *this; }
  cpp_int& operator*=(const cpp_int& o) { v_ *= o.v_; return *this; }
  cpp_int& operator/=(const cpp_int& o) { v_ /= o.v_; return *this; }
  friend cpp_int operator+(cpp_int a, const cpp_int& b) { return a += b; }
  friend cpp_int operator*(cpp_int a, const cpp_int& b) { return a *= b; }
  friend cpp_int operator/(cpp_int a, const cpp_int& b) { return a /= b; }
  friend bool operator==(const cpp_int& a, const cpp_int& b) { return a.v_ == b.v_; }
  friend bool operator!=(const cpp_int& a, const cpp_int& b) { return a.v_ != b.v_; }
  friend bool operator<(const cpp_int& a, const cpp_int& b) { return a.v_ < b.v_; }
  friend bool operator>(const cpp_int& a, const cpp_int& b) { return a.v_ > b.v_; }

 private:
  u128 v_;
};

}  // namespace multiprecision
}  // namespace boost
