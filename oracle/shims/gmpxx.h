// ORACLE TEST INFRASTRUCTURE: the slice of gmpxx's mpq_class that
// proj/tests/test_runtime.cpp:73-84 uses, over the C ABI of the system
// libgmp.so.10 (GMP headers are absent; only the runtime library exists).
#pragma once
extern "C" {
typedef struct { int alloc; int size; void* d; } sd_mpz_struct;
typedef struct { sd_mpz_struct num, den; } sd_mpq_struct;
void __gmpq_init(sd_mpq_struct*);
void __gmpq_clear(sd_mpq_struct*);
void __gmpq_set(sd_mpq_struct*, const sd_mpq_struct*);
void __gmpq_set_d(sd_mpq_struct*, double);
void __gmpq_set_si(sd_mpq_struct*, long, unsigned long);
void __gmpq_add(sd_mpq_struct*, const sd_mpq_struct*, const sd_mpq_struct*);
void __gmpq_sub(sd_mpq_struct*, const sd_mpq_struct*, const sd_mpq_struct*);
void __gmpq_div(sd_mpq_struct*, const sd_mpq_struct*, const sd_mpq_struct*);
void __gmpq_abs(sd_mpq_struct*, const sd_mpq_struct*);
double __gmpq_get_d(const sd_mpq_struct*);
}
class mpq_class {
 public:
  mpq_class() { __gmpq_init(&q_); }
  mpq_class(int v) { __gmpq_init(&q_); __gmpq_set_si(&q_, v, 1); }
  mpq_class(double v) { __gmpq_init(&q_); __gmpq_set_d(&q_, v); }
  mpq_class(const mpq_class& o) { __gmpq_init(&q_); __gmpq_set(&q_, &o.q_); }
  mpq_class& operator=(const mpq_class& o) { __gmpq_set(&q_, &o.q_); return *this; }
  ~mpq_class() { __gmpq_clear(&q_); }
  mpq_class& operator+=(const mpq_class& o) { __gmpq_add(&q_, &q_, &o.q_); return *this; }
  friend mpq_class operator-(const mpq_class& a, const mpq_class& b) { mpq_class r; __gmpq_sub(&r.q_, &a.q_, &b.q_); return r; }
  friend mpq_class operator/(const mpq_class& a, const mpq_class& b) { mpq_class r; __gmpq_div(&r.q_, &a.q_, &b.q_); return r; }
  friend mpq_class abs(const mpq_class& a) { mpq_class r; __gmpq_abs(&r.q_, &a.q_); return r; }
  double get_d() const { return __gmpq_get_d(&q_); }
 private:
  sd_mpq_struct q_;
};
